// A reference-style C++ caller of the gensor-b200 facade (include/gensor_b200.hpp): parse ->
// construct (optimize) -> [execute on the GPU when one is present, host buffers] -> print JSON.
// Built and run by tests/test_cpp_facade.py (CPU: construct only; GPU: also execute + check).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "gensor_b200.hpp"

int main(int argc, char** argv) {
  const std::string op_json = argc > 1 ? argv[1] : R"({"kind":"gemm","M":64,"K":48,"N":40})";
  const std::string hw_json = argc > 2 ? argv[2] : "";
  const bool run = argc > 3 && std::strcmp(argv[3], "execute") == 0;
  try {
    auto op = gensor_b200::TensorOpSpec::parse_text(op_json);
    gensor_b200::EngineConfig cfg;
    cfg.top_k = 3;
    auto hw = hw_json.empty() ? gensor_b200::HardwareSpec::b200(0) : gensor_b200::HardwareSpec::load_text(hw_json);
    if (hw_json.empty()) cfg.mode = GENSOR_MODE_B200;
    auto sched = gensor_b200::optimize(op, hw, cfg);
    std::printf("{\"n\":%d,\"best\":%s", sched.size(), sched.json(0).c_str());
    if (run) {
      // gemm only: C = A * B with A = 1, B = 2 -> every C = 2K (integer-exact on every variant)
      const std::string info = op.info_json();
      int M = 0, K = 0, N = 0;
      std::sscanf(op_json.c_str(), "{\"kind\":\"gemm\",\"M\":%d,\"K\":%d,\"N\":%d}", &M, &K, &N);
      std::vector<float> a(static_cast<size_t>(M) * K, 1.0f), b(static_cast<size_t>(K) * N, 2.0f),
          c(static_cast<size_t>(M) * N, 0.0f);
      gensor_b200::Kernel k(op, sched, 0, GENSOR_VARIANT_AUTO);
      k.execute_host({a.data(), b.data()}, c.data());
      int bad = 0;
      for (float v : c) bad += v != 2.0f * K;
      std::printf(",\"kernel\":%s,\"mismatches\":%d", k.info_json().c_str(), bad);
    }
    std::printf("}\n");
  } catch (const gensor_b200::Error& e) {
    std::printf("{\"error\":\"%s\",\"code\":%d}\n", e.what(), e.code());
    return 2;
  }
  return 0;
}
