// TEST INFRASTRUCTURE ONLY — forced-include shim used by oracle/Makefile to compile the
// UNMODIFIED reference sources under /root/reference/proj/src into oracle/_ref/.
//
// Why it exists:
//  * the reference's vendor/ tree (nlohmann/json) is absent from the snapshot, so the image's
//    nlohmann 3.11.3 header is put on the include path by the Makefile;
//  * GCC 13 rejects `pool.resize(...)` (engine.cpp:190) and `items.resize(...)`
//    (tree_baseline.cpp:48) because ETIRState's default constructor is private (etir.hpp:72).
//    Every std header the reference uses is included first, then `private` is widened, which
//    leaves libstdc++ untouched (a plain -Dprivate=public breaks <sstream>/<any>).
#pragma once
#include <algorithm>
#include <cmath>
#include <compare>
#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <numeric>
#include <optional>
#include <random>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>
#include <nlohmann/json.hpp>
#define private public
