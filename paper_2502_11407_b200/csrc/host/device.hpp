// Device side of the execute step: kernel instantiation from a complete schedule and launch.
// Implemented in csrc/kernels/*.cu (nvcc, sm_100a). The host library reaches the GPU only
// through these functions.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "hw.hpp"
#include "op.hpp"
#include "sched.hpp"

namespace gb::dev {

struct Kernel;  // opaque: the instantiated plan + device workspace

Kernel* prepare(const OpDesc& op, const Sched& s, int variant);  // throws gb::Error
void destroy(Kernel* k);
std::string info(const Kernel* k);
std::string plan(const Kernel* k);  // the instantiated plan (JSON object)
// ws == nullptr: the handle's workspace for `stream` (allocated on the stream's first execute);
// otherwise a caller-owned device workspace of ws_size >= workspace_bytes(k) bytes.
void execute(const Kernel* k, const void* const* d_in, int n_in, void* d_out, void* ws, size_t ws_size,
             void* stream);
size_t workspace_bytes(const Kernel* k);
void execute_host(Kernel* k, const void* const* h_in, int n_in, void* h_out, void* stream);

void set_timing(Kernel* k, bool on);
float time_execute(Kernel* k, const void* const* d_in, int n_in, void* d_out, void* stream, int iters);
std::vector<std::pair<std::string, float>> timings(Kernel* k);  // last execute, per launch (ms)

DeviceLimits query(int device);  // cudaGetDeviceProperties -> limits (peaks filled by caller)
uint64_t launch_count();

}  // namespace gb::dev
