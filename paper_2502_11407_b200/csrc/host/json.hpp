// Minimal JSON value + reader/writer for the operator and hardware description documents.
// The reference reads these with nlohmann::ordered_json (op_spec.hpp:14); only the subset the
// documents use is needed here: objects (insertion-ordered), arrays, strings, bools, null and
// numbers, where integers without fraction/exponent stay integers (nlohmann's
// is_number_integer, op_spec.cpp:32) and everything else is a double parsed with strtod
// (correctly rounded, like nlohmann's lexer).
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace gb::json {

enum class Type : uint8_t { Null, Bool, Int, Double, String, Array, Object };

class Value {
 public:
  Type type = Type::Null;
  bool b = false;
  int64_t i = 0;
  double d = 0.0;
  std::string s;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;

  bool is_int() const { return type == Type::Int; }
  bool is_number() const { return type == Type::Int || type == Type::Double; }
  bool is_string() const { return type == Type::String; }
  bool is_array() const { return type == Type::Array; }
  bool is_object() const { return type == Type::Object; }

  const Value* find(const std::string& key) const {
    if (type != Type::Object) return nullptr;
    for (const auto& kv : obj)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
  bool has(const std::string& key) const { return find(key) != nullptr; }

  // Numeric reads with nlohmann's conversion semantics: a double read as an integer truncates,
  // an integer read as a double converts exactly (or to nearest for |v| > 2^53).
  int64_t as_int() const;
  double as_double() const;
  const std::string& as_string() const;
};

// Throws gb::Error(ConfigError, "invalid JSON: ...") on malformed text.
Value parse(const std::string& text);

// Writer helpers used by the C-ABI's JSON reports.
std::string quote(const std::string& s);
std::string num(double v);  // shortest round-trip repr ("%.17g" trimmed)

}  // namespace gb::json
