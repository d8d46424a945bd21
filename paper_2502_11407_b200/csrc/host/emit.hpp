// emit_source: complete schedule -> portable C source of its loop nest.
#pragma once

#include <string>

#include "op.hpp"
#include "sched.hpp"

namespace gb {

// Deterministic: byte-identical text for identical (op, state, trace).
std::string emit_source(const OpDesc& op, const Sched& s, const std::string& trace_json = "");

}  // namespace gb
