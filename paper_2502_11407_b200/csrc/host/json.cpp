#include "json.hpp"

#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "error.hpp"

namespace gb::json {

namespace {

struct Reader {
  const std::string& t;
  size_t p = 0;

  [[noreturn]] void fail(const char* what) const {
    throw Error(Code::ConfigError, std::string("invalid JSON: ") + what + " at offset " + std::to_string(p));
  }
  void ws() {
    while (p < t.size() && (t[p] == ' ' || t[p] == '\n' || t[p] == '\r' || t[p] == '\t')) ++p;
  }
  bool lit(const char* w) {
    size_t n = std::strlen(w);
    if (t.compare(p, n, w) == 0) {
      p += n;
      return true;
    }
    return false;
  }

  static void put_utf8(std::string& out, uint32_t cp) {
    if (cp < 0x80) {
      out += static_cast<char>(cp);
    } else if (cp < 0x800) {
      out += static_cast<char>(0xC0 | (cp >> 6));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += static_cast<char>(0xE0 | (cp >> 12));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      out += static_cast<char>(0xF0 | (cp >> 18));
      out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }

  uint32_t hex4() {
    if (p + 4 > t.size()) fail("truncated \\u escape");
    uint32_t v = 0;
    for (int k = 0; k < 4; ++k) {
      char c = t[p++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<uint32_t>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<uint32_t>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<uint32_t>(c - 'A' + 10);
      else fail("bad \\u escape");
    }
    return v;
  }

  std::string str() {
    if (t[p] != '"') fail("expected string");
    ++p;
    std::string out;
    while (true) {
      if (p >= t.size()) fail("unterminated string");
      char c = t[p++];
      if (c == '"') break;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p >= t.size()) fail("unterminated escape");
      char e = t[p++];
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00) {
            if (!(lit("\\u"))) fail("lone surrogate");
            uint32_t lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) fail("bad surrogate pair");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          put_utf8(out, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
    return out;
  }

  Value number() {
    size_t start = p;
    bool is_float = false;
    if (t[p] == '-') ++p;
    if (p >= t.size() || !(t[p] >= '0' && t[p] <= '9')) fail("bad number");
    if (t[p] == '0') {
      ++p;
    } else {
      while (p < t.size() && t[p] >= '0' && t[p] <= '9') ++p;
    }
    if (p < t.size() && t[p] == '.') {
      is_float = true;
      ++p;
      if (p >= t.size() || !(t[p] >= '0' && t[p] <= '9')) fail("bad fraction");
      while (p < t.size() && t[p] >= '0' && t[p] <= '9') ++p;
    }
    if (p < t.size() && (t[p] == 'e' || t[p] == 'E')) {
      is_float = true;
      ++p;
      if (p < t.size() && (t[p] == '+' || t[p] == '-')) ++p;
      if (p >= t.size() || !(t[p] >= '0' && t[p] <= '9')) fail("bad exponent");
      while (p < t.size() && t[p] >= '0' && t[p] <= '9') ++p;
    }
    std::string tok = t.substr(start, p - start);
    Value v;
    if (!is_float) {
      errno = 0;
      long long x = std::strtoll(tok.c_str(), nullptr, 10);
      if (errno == 0) {
        v.type = Type::Int;
        v.i = x;
        return v;
      }
      // out of int64 range: keep as double like a JSON reader without big-int support
    }
    v.type = Type::Double;
    v.d = std::strtod(tok.c_str(), nullptr);
    return v;
  }

  Value value(int depth) {
    if (depth > 256) fail("nesting too deep");
    ws();
    if (p >= t.size()) fail("unexpected end");
    Value v;
    char c = t[p];
    if (c == '{') {
      ++p;
      v.type = Type::Object;
      ws();
      if (p < t.size() && t[p] == '}') {
        ++p;
        return v;
      }
      while (true) {
        ws();
        if (p >= t.size()) fail("unterminated object");
        std::string k = str();
        ws();
        if (p >= t.size() || t[p] != ':') fail("expected ':'");
        ++p;
        Value item = value(depth + 1);
        bool replaced = false;  // duplicate keys: last one wins (nlohmann behaviour)
        for (auto& kv : v.obj)
          if (kv.first == k) {
            kv.second = std::move(item);
            replaced = true;
            break;
          }
        if (!replaced) v.obj.emplace_back(std::move(k), std::move(item));
        ws();
        if (p < t.size() && t[p] == ',') {
          ++p;
          continue;
        }
        if (p < t.size() && t[p] == '}') {
          ++p;
          break;
        }
        fail("expected ',' or '}'");
      }
      return v;
    }
    if (c == '[') {
      ++p;
      v.type = Type::Array;
      ws();
      if (p < t.size() && t[p] == ']') {
        ++p;
        return v;
      }
      while (true) {
        v.arr.push_back(value(depth + 1));
        ws();
        if (p < t.size() && t[p] == ',') {
          ++p;
          continue;
        }
        if (p < t.size() && t[p] == ']') {
          ++p;
          break;
        }
        fail("expected ',' or ']'");
      }
      return v;
    }
    if (c == '"') {
      v.type = Type::String;
      v.s = str();
      return v;
    }
    if (lit("true")) {
      v.type = Type::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.type = Type::Bool;
      return v;
    }
    if (lit("null")) return v;
    return number();
  }
};

}  // namespace

int64_t Value::as_int() const {
  if (type == Type::Int) return i;
  if (type == Type::Double) return static_cast<int64_t>(d);
  if (type == Type::Bool) return b ? 1 : 0;
  throw Error(Code::ConfigError, "expected a number");
}

double Value::as_double() const {
  if (type == Type::Double) return d;
  if (type == Type::Int) return static_cast<double>(i);
  if (type == Type::Bool) return b ? 1.0 : 0.0;
  throw Error(Code::ConfigError, "expected a number");
}

const std::string& Value::as_string() const {
  if (type != Type::String) throw Error(Code::ConfigError, "expected a string");
  return s;
}

Value parse(const std::string& text) {
  Reader r{text};
  Value v = r.value(0);
  r.ws();
  if (r.p != text.size()) r.fail("trailing characters");
  return v;
}

std::string quote(const std::string& s) {
  std::string out = "\"";
  for (char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\t': out += "\\t"; break;
      case '\r': out += "\\r"; break;
      default:
        if (static_cast<unsigned char>(c) < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", c);
          out += buf;
        } else {
          out += c;
        }
    }
  }
  return out + "\"";
}

std::string num(double v) {
  if (std::isnan(v) || std::isinf(v)) return "null";
  char buf[40];
  for (int prec = 15; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s = buf;
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

}  // namespace gb::json
