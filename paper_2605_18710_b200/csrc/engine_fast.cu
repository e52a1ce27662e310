// engine_fast.cu — k_search specialised for the common model: include_self, non-negative
// interference coefficients, multiplicative term on (every BASELINE config).  Same search
// code as the generic kernel (search_kernel.cuh); the fixed flags drop the other branches,
// which keeps the kernel small enough for the instruction cache.
// Built three times by build.py: MG_FAST_MODE=0 (MIN proofs), 1 (FIRST probes), 2 (mixed
// batches, mode read from each search's Spec).
#define MG_SPECIALIZE 1
#if MG_FAST_MODE == 0
#define MG_KSEARCH_NAME k_search_fast_min
#define MG_MODE_FIXED 0
#define MG_FAST_FN k_search_fast_min_fn
#elif MG_FAST_MODE == 1
#define MG_KSEARCH_NAME k_search_fast_first
#define MG_MODE_FIXED 1
#define MG_FAST_FN k_search_fast_first_fn
#else
#define MG_KSEARCH_NAME k_search_fast_any  // batches mixing MIN and FIRST searches
#define MG_FAST_FN k_search_fast_any_fn
#endif
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
const void* MG_FAST_FN() { return reinterpret_cast<const void*>(&MG_KSEARCH_NAME); }
}  // namespace mg
