// Execute step: instantiate a kernel family from a complete schedule and launch it.
// This is the device replacement of the SPEC's lower()+interpret().
#include <atomic>
#include <cstring>
#include <sstream>
#include <string>

#include "../host/device.hpp"
#include "../host/error.hpp"
#include "../host/json.hpp"
#include "../host/lower.hpp"
#include "common.cuh"
#include "launch.h"

namespace gb::dev {

namespace {
std::atomic<uint64_t> g_launches{0};
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(Code::Cuda, std::string(what) + ": " + cudaGetErrorString(e));
}

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

enum class Family { Generic };

struct Kernel {
  OpDesc op;
  Sched state;
  int variant = 0;
  Family family = Family::Generic;
  GenericPlan gplan{};
  bool f64 = false;
  // host-buffer execute staging (allocated on first use)
  void* d_in[3] = {nullptr, nullptr, nullptr};
  void* d_out = nullptr;
  size_t in_bytes[3] = {0, 0, 0};
  size_t out_bytes = 0;
  int launches = 1;
};

namespace {

int resolve_variant(const OpDesc& op, int variant) {
  if (variant != -1) return variant;
  return 1;  // SIMT_F32 until the tensor-core / stream families take over
}

size_t tensor_bytes(const OpDesc& op, int t) {
  return static_cast<size_t>(op.tensor_elems(t, false)) * op.dtype_bytes * static_cast<size_t>(op.batch);
}

}  // namespace

DeviceLimits query(int device) {
  DeviceLimits lim;
  cudaDeviceProp prop;
  check_cuda(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  lim.sms = prop.multiProcessorCount;
  lim.smem_per_block = static_cast<int64_t>(prop.sharedMemPerBlockOptin);
  lim.smem_per_sm = static_cast<int64_t>(prop.sharedMemPerMultiprocessor);
  lim.regs_per_sm = prop.regsPerMultiprocessor;
  lim.max_threads_per_block = prop.maxThreadsPerBlock;
  lim.max_threads_per_sm = prop.maxThreadsPerMultiProcessor;
  lim.max_blocks_per_sm = prop.maxBlocksPerMultiProcessor;
  lim.l2_bytes = prop.l2CacheSize;
  int clock_khz = 0;
  if (cudaDeviceGetAttribute(&clock_khz, cudaDevAttrClockRate, device) == cudaSuccess && clock_khz > 0)
    lim.sm_clock_hz = clock_khz * 1e3;
  lim.fp32_simt_flops = static_cast<double>(lim.sms) * 128.0 * 2.0 * lim.sm_clock_hz;
  return lim;
}

Kernel* prepare(const OpDesc& op, const Sched& s, int variant) {
  if (!s.complete()) throw Error(Code::IncompleteState, "kernel needs a complete schedule");
  auto* k = new Kernel;
  k->op = op;
  k->state = s;
  k->variant = resolve_variant(op, variant);
  try {
    switch (k->variant) {
      case 0:
      case 1: {
        int dev = 0, optin = 0;
        check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
        check_cuda(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "smem optin");
        k->f64 = k->variant == 0;
        k->family = Family::Generic;
        k->gplan = lower_generic(op, s, generic_max_width(k->f64), op.dtype_bytes, optin);
        break;
      }
      default:
        throw Error(Code::Unsupported, "variant " + std::to_string(variant) + " not available for " + op.label());
    }
  } catch (...) {
    delete k;
    throw;
  }
  return k;
}

void destroy(Kernel* k) {
  if (!k) return;
  for (void* p : k->d_in)
    if (p) cudaFree(p);
  if (k->d_out) cudaFree(k->d_out);
  delete k;
}

std::string info(const Kernel* k) {
  std::ostringstream os;
  static const char* names[] = {"simt_parity", "simt_f32", "tc_tf32", "tc_bf16", "stream"};
  os << "{\"variant\":" << k->variant << ",\"variant_name\":\"" << names[k->variant] << "\",\"op\":" << k->op.to_json()
     << ",\"state\":" << k->state.to_json(k->op) << ",\"flops\":" << json::num(k->op.flops_true())
     << ",\"bytes\":" << json::num(k->op.bytes_true()) << ",\"launches\":" << k->launches << ",\"plan\":";
  os << plan_json(k->gplan);
  os << "}";
  return os.str();
}

void execute(const Kernel* k, const void* const* d_in, int n_in, void* d_out, void* stream) {
  const OpDesc& op = k->op;
  if (n_in != op.input_count())
    throw Error(Code::ShapeMismatch,
                "expected " + std::to_string(op.input_count()) + " inputs, got " + std::to_string(n_in));
  for (int i = 0; i < n_in; ++i)
    if (!d_in[i]) throw Error(Code::ShapeMismatch, "null input pointer");
  auto st = static_cast<cudaStream_t>(stream);
  switch (k->family) {
    case Family::Generic:
      launch_generic(k->gplan, k->f64, op.dtype_bytes == 2, d_in[0], n_in > 1 ? d_in[1] : nullptr, d_out,
                     static_cast<int>(op.batch), st);
      break;
  }
}

void execute_host(Kernel* k, const void* const* h_in, int n_in, void* h_out, void* stream) {
  const OpDesc& op = k->op;
  if (n_in != op.input_count())
    throw Error(Code::ShapeMismatch,
                "expected " + std::to_string(op.input_count()) + " inputs, got " + std::to_string(n_in));
  auto st = static_cast<cudaStream_t>(stream);
  for (int i = 0; i < n_in; ++i) {
    const size_t b = tensor_bytes(op, i);
    if (!k->d_in[i]) {
      check_cuda(cudaMalloc(&k->d_in[i], b), "cudaMalloc input staging");
      k->in_bytes[i] = b;
    }
    check_cuda(cudaMemcpyAsync(k->d_in[i], h_in[i], b, cudaMemcpyHostToDevice, st), "H2D");
  }
  const size_t ob = tensor_bytes(op, op.output_index());
  if (!k->d_out) {
    check_cuda(cudaMalloc(&k->d_out, ob), "cudaMalloc output staging");
    k->out_bytes = ob;
  }
  execute(k, k->d_in, n_in, k->d_out, stream);
  check_cuda(cudaMemcpyAsync(h_out, k->d_out, ob, cudaMemcpyDeviceToHost, st), "D2H");
  check_cuda(cudaStreamSynchronize(st), "stream sync");
}

}  // namespace gb::dev
