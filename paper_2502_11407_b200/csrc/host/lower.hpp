// Lowering: complete schedule state -> kernel plan (the SPEC's `lower`, whose
// reference implementation lowering.cpp is absent from the snapshot).
#pragma once

#include <string>

#include "../kernels/plan.h"
#include "op.hpp"
#include "sched.hpp"

namespace gb {

// Generic state-driven SIMT plan. `acc_width` is the kernel's per-thread accumulator array
// width (power of two); `elem_bytes` the input element size; `smem_limit` the largest
// dynamic shared-memory staging area allowed (larger boxes fall back to direct L2 reads).
GenericPlan lower_generic(const OpDesc& op, const Sched& s, int acc_width, int elem_bytes, int64_t smem_limit);

std::string plan_json(const GenericPlan& p);

}  // namespace gb
