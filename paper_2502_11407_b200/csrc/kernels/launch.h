// Host-callable launchers of the kernel families (all asynchronous on the given stream).
#pragma once

#include <cuda_runtime.h>

#include "plan.h"

namespace gb::dev {

int generic_max_width(bool f64);
void launch_generic(const GenericPlan& p, bool f64, bool bf16, const void* in0, const void* in1, void* out,
                    int batch, cudaStream_t st);

}  // namespace gb::dev
