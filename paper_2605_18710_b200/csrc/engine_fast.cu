// engine_fast.cu — k_search specialised for the common model: include_self, non-negative
// interference coefficients, multiplicative term on (every BASELINE config).  Same search
// code as the generic kernel (search_kernel.cuh); the fixed flags drop the other branches,
// which keeps the kernel small enough for the instruction cache.
#define MG_SPECIALIZE 1
#define MG_KSEARCH_NAME k_search_fast
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "engine.hpp"
#include "search_core.cuh"
#include "search_warp.cuh"
#include "search_kernel.cuh"

namespace mg {
const void* k_search_fast_fn() { return reinterpret_cast<const void*>(&k_search_fast); }
}  // namespace mg
