// eval.cu — K1, the batched plan-scoring kernel: stage_time / rectified_latency of explicit
// stage allocations (perf_model.hpp:442-479), read straight from the ABI layout
// (mosaic_gpu_eval_entry + flat GPU lists + allocation offsets, include/mosaic_gpu.h).
//
// HBM-bound by design: per allocation the kernel streams its entries (32 B each), its GPU
// ids (4 B each), one offset and writes one stage time (+ one rectified latency per entry).
// Everything else is on chip:
//   * (module, d, units) -> (base_latency, solo_bandwidth) comes from dense rate tables built
//     once per context (Surface::rate_tables; a few hundred KB, L2-resident), so no surface
//     lookup runs per call and the host never repacks entries;
//   * one warp per allocation builds the per-GPU resident bitmap in shared memory (atomicOr
//     of bit e for every GPU of entry e), so "is entry e on GPU r" — the reference's
//     std::find over e.gpus — is one bit test;
//   * with include_self the interference delta of a GPU depends only on its resident set,
//     so it is computed ONCE per GPU (residents summed in entry order, -fmad=false: the
//     reference's bits) and every entry takes the max over its GPUs from the bitmap;
//     without include_self each entry excludes its own module's bits.
// Duplicate modules in one allocation follow the reference: rectified_latency uses the
// first entry of the module (StageAllocation::find).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "engine.hpp"

namespace mg {

#define CKE(x)                                                                         \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                     " at " #x);                                       \
    } while (0)

constexpr int KE_WARPS = 8;     // warps (allocations in flight) per CTA
constexpr int KE_MAXE = 64;     // entries per allocation (two 32-bit resident bitmaps)
constexpr double KE_NEG = -1e300;  // rectified_latency's `worst` seed
constexpr unsigned KE_FULL = 0xffffffffu;

struct KEParams {
    const double* base;  // [n_mod][G][L+1]
    const double* B;     // [n_mod][L+1]
    int n_mod, G, L, additive, include_self;
    double e1, e2, e3;
    long long n_ent, n_gpu_ids;
};

struct KEStats {  // device-side error bits, the bytes actually streamed, the worklist size
    int err;
    int pad;
    unsigned long long gpu_ids, entries;
    unsigned long long nlist;  // allocations k_evaluate_fast left to k_evaluate
};

// Per-warp shared memory: mask[2G] u32 (bit e of mask[r] / mask[G + r] <=> GPU r hosts
// entry e / e + 32) | dl[G] f64 | eB[64] f64 | a union of the <= 32-entry path's per-entry
// max keys and the generic path's per-entry arrays.
constexpr size_t KE_UNION = 64 * (8 * 2 + 8 + 8 + 4 * 2);  // ebase, erect, esame, eoff, emod, en
__host__ __device__ inline size_t ke_warp_bytes(int G) {
    return (size_t)G * 16 + KE_MAXE * 8 + KE_UNION;
}

// Interference delta for residents `m` (entry order): (e1 + e2*sum) + e3*prod, prod = 0
// without residents (perf_model.hpp:455-463).
__device__ __forceinline__ double ke_delta(const KEParams& P, const double* eB, unsigned mlo,
                                           unsigned mhi) {
    double s = 0.0, p = 1.0;
    const bool none = (mlo | mhi) == 0;
    while (mlo) {
        const int f = __ffs(mlo) - 1;
        mlo &= mlo - 1;
        const double b = eB[f];
        s = s + b;
        p = p * b;
    }
    while (mhi) {
        const int f = __ffs(mhi) + 31;
        mhi &= mhi - 1;
        const double b = eB[f];
        s = s + b;
        p = p * b;
    }
    if (none) p = 0.0;
    const double d0 = P.e1 + P.e2 * s;
    return d0 + (P.additive ? 0.0 : P.e3 * p);
}

// Order-preserving fp64 -> u64 (non-NaN): max over keys == max over values.
__device__ __forceinline__ unsigned long long ke_key(double v) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ULL);
}
__device__ __forceinline__ double ke_unkey(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k));
}

__device__ __forceinline__ double ke_wmax(double v) {
    #pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double x = __shfl_xor_sync(KE_FULL, v, o);
        v = v < x ? x : v;
    }
    return v;
}

__global__ void __launch_bounds__(32 * KE_WARPS, 4)
    k_evaluate(const EvalABI* __restrict__ ent, const int* __restrict__ gpus,
               const long long* __restrict__ off, long long n, KEParams P, double* st,
               double* rect, KEStats* stats, const long long* __restrict__ list) {
    extern __shared__ __align__(16) unsigned char ke_smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;  // lanes below this one
    const int G = P.G;
    unsigned char* wb = ke_smem + (size_t)wid * ke_warp_bytes(G);
    unsigned* mask = reinterpret_cast<unsigned*>(wb);
    double* dl = reinterpret_cast<double*>(mask + 2 * G);
    double* eB = dl + G;
    unsigned char* un = reinterpret_cast<unsigned char*>(eB + KE_MAXE);
    // <= 32 entries view of the union: per-entry max keys (high / low words), same-module bits
    unsigned* whi = reinterpret_cast<unsigned*>(un);
    unsigned* wlo = whi + 32;
    unsigned* esm = wlo + 32;
    // generic path view
    double* ebase = reinterpret_cast<double*>(un);
    double* erect = ebase + KE_MAXE;
    unsigned long long* esame = reinterpret_cast<unsigned long long*>(erect + KE_MAXE);
    long long* eoff = reinterpret_cast<long long*>(esame + KE_MAXE);
    int* emod = reinterpret_cast<int*>(eoff + KE_MAXE);
    int* en = emod + KE_MAXE;
    int errs = 0;
    unsigned long long ids = 0, ents = 0;
    const bool self_in = P.include_self != 0;
    const long long stride = (long long)gridDim.x * KE_WARPS;
    // with a worklist: only the allocations k_evaluate_fast handed over (same stream, so
    // its count is final when this kernel starts)
    const long long nn = list ? (long long)*(volatile unsigned long long*)&stats->nlist : n;
    for (long long t = (long long)blockIdx.x * KE_WARPS + wid; t < nn; t += stride) {
        const long long a = list ? list[t] : t;
        const long long e0 = off[a], e1 = off[a + 1];
        const long long ne64 = e1 - e0;
        if (ne64 <= 0 || e0 < 0 || e1 > P.n_ent || ne64 > KE_MAXE) {
            // an empty allocation is stage_time 0.0 (the reference's `worst` seed)
            if (ne64 != 0) errs |= EVAL_ERR_ENTRIES;
            if (lane == 0) st[a] = ne64 == 0 ? 0.0 : NAN;
            continue;
        }
        const int ne = (int)ne64;
        ents += (unsigned long long)ne;
        // ---- entries: lane e holds entry e (and e + 32) ----
        // rates outside the tables / the profiled hull are NaN: the reference only raises
        // SurfaceRangeError for lookups it actually makes (checked after scoring)
        bool bad = false;
        int r_mod = -1 - lane, r_ng = 0;
        long long r_off = 0;
        double r_base = NAN;
        for (int e = lane; e < ne; e += 32) {
            const EvalABI E = ent[e0 + e];
            double b = NAN, bw = NAN;
            if (E.module < 0 || E.module >= P.n_mod) {
                errs |= EVAL_ERR_MODULE;
                bad = true;
            } else if (E.levels != 0 && E.levels != P.L) {
                errs |= EVAL_ERR_LEVELS;
                bad = true;
            } else if (E.units >= 0 && E.units <= P.L) {
                bw = P.B[(size_t)E.module * (P.L + 1) + E.units];
                if (E.d >= 1 && E.d <= G)
                    b = P.base[((size_t)E.module * G + (E.d - 1)) * (P.L + 1) + E.units];
            }
            if (E.n_gpus < 0 || E.gpu_off < 0 || E.gpu_off + E.n_gpus > P.n_gpu_ids) {
                errs |= EVAL_ERR_GPU;
                bad = true;
            }
            eB[e] = bw;
            if (e < 32) {
                r_mod = E.module;
                r_ng = E.n_gpus;
                r_off = E.gpu_off;
                r_base = b;
            }
            if (ne > 32) {
                ebase[e] = b;
                emod[e] = E.module;
                en[e] = E.n_gpus;
                eoff[e] = E.gpu_off;
            }
        }
        if (__any_sync(KE_FULL, bad)) {
            if (lane == 0) st[a] = NAN;
            continue;
        }
        const bool has = lane < ne;
        double worst_stage = 0.0;
        if (ne <= 32) {
            // ---- up to 32 entries: lane e holds entry e, 32-bit resident bitmaps ----
            // StageAllocation::find: a module's first entry is its "self" entry
            const unsigned same = __match_any_sync(KE_FULL, r_mod);
            const bool is_self = has && (same & lt) == 0;
            const unsigned selfm = __ballot_sync(KE_FULL, is_self);
            for (int g = lane; g < G; g += 32) mask[g] = 0u;
            whi[lane] = 0u;
            wlo[lane] = 0u;
            esm[lane] = same;
            __syncwarp();
            // resident bitmaps: bit e of mask[r] <=> r in entries[e].gpus
            for (int e = 0; e < ne; ++e) {
                const int c = __shfl_sync(KE_FULL, r_ng, e);
                const long long o = __shfl_sync(KE_FULL, r_off, e);
                ids += (unsigned long long)c;
                for (int i = lane; i < c; i += 32) {
                    const int g = __ldg(gpus + o + i);
                    if ((unsigned)g >= (unsigned)G)
                        errs |= EVAL_ERR_GPU;
                    else
                        atomicOr(&mask[g], 1u << e);
                }
            }
            __syncwarp();
            unsigned used = 0u;
            unsigned long long rk = 0ULL;
            if (self_in && G <= 128) {
                // <= 4 GPUs per lane, in registers: each GPU hosting a self entry gets ONE
                // delta (its resident set, entry order); each self entry's max over its GPUs
                // is a lane-local max then a warp max of the order-preserving 64-bit key
                // (high words, then low words among the lanes holding the high maximum)
                unsigned mloc[4];
                unsigned long long kloc[4];
                #pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const int g = lane + 32 * s;
                    unsigned m = g < G ? mask[g] : 0u;
                    if (!(m & selfm)) m = 0u;
                    mloc[s] = m;
                    used |= m;
                    kloc[s] = m ? ke_key(ke_delta(P, eB, m, 0u)) : 0ULL;
                }
                for (int e = 0; e < ne; ++e) {
                    if (!(selfm >> e & 1u)) continue;
                    unsigned long long k = 0ULL;
                    #pragma unroll
                    for (int s = 0; s < 4; ++s)
                        if ((mloc[s] >> e & 1u) && kloc[s] > k) k = kloc[s];
                    const unsigned hi = __reduce_max_sync(KE_FULL, (unsigned)(k >> 32));
                    const unsigned lo = __reduce_max_sync(
                        KE_FULL, (unsigned)(k >> 32) == hi ? (unsigned)k : 0u);
                    if (lane == e) rk = (unsigned long long)hi << 32 | lo;
                }
            } else {
                // per GPU hosting a self entry: its delta, then max into the entry's key.  The
                // fp64 max runs as two 32-bit atomicMax passes over the order-preserving key
                // (high words, then low words among the GPUs that reached the high maximum).
                for (int g = lane; g < G; g += 32) {
                    const unsigned m = mask[g];
                    unsigned sm = m & selfm;
                    if (!sm) continue;
                    if (self_in) {
                        const double v = ke_delta(P, eB, m, 0u);
                        dl[g] = v;
                        used |= m;
                        const unsigned hi = (unsigned)(ke_key(v) >> 32);
                        while (sm) {
                            const int e = __ffs(sm) - 1;
                            sm &= sm - 1;
                            atomicMax(&whi[e], hi);
                        }
                    } else {
                        while (sm) {
                            const int e = __ffs(sm) - 1;
                            sm &= sm - 1;
                            const unsigned r = m & ~esm[e];
                            used |= r;
                            atomicMax(&whi[e], (unsigned)(ke_key(ke_delta(P, eB, r, 0u)) >> 32));
                        }
                    }
                }
                __syncwarp();
                for (int g = lane; g < G; g += 32) {
                    const unsigned m = mask[g];
                    unsigned sm = m & selfm;
                    if (!sm) continue;
                    if (self_in) {
                        const unsigned long long k = ke_key(dl[g]);
                        const unsigned hi = (unsigned)(k >> 32), lo = (unsigned)k;
                        while (sm) {
                            const int e = __ffs(sm) - 1;
                            sm &= sm - 1;
                            if (whi[e] == hi) atomicMax(&wlo[e], lo);
                        }
                    } else {
                        while (sm) {
                            const int e = __ffs(sm) - 1;
                            sm &= sm - 1;
                            const unsigned long long k = ke_key(ke_delta(P, eB, m & ~esm[e], 0u));
                            if (whi[e] == (unsigned)(k >> 32)) atomicMax(&wlo[e], (unsigned)k);
                        }
                    }
                }
                __syncwarp();
                rk = (unsigned long long)whi[lane] << 32 | wlo[lane];
            }
            used = __reduce_or_sync(KE_FULL, used);
            // rectified_latency = base of the self entry + its worst GPU delta (an entry
            // without GPUs keeps the reference's -1e300 seed)
            double rl = r_base + (rk ? ke_unkey(rk) : KE_NEG);
            const bool miss = (is_self && isnan(r_base)) || (has && (used >> lane & 1u) && isnan(eB[lane]));
            rl = __shfl_sync(KE_FULL, rl, __ffs(same) - 1);
            if (__any_sync(KE_FULL, miss)) {
                errs |= EVAL_ERR_SURFACE;
                if (lane == 0) st[a] = NAN;
                continue;
            }
            if (rect && has) rect[e0 + lane] = rl;
            worst_stage = ke_wmax(has ? rl : 0.0);
            worst_stage = worst_stage < 0.0 ? 0.0 : worst_stage;
            if (lane == 0) st[a] = worst_stage;
            continue;
        }
        // ---- generic path (more than 32 entries, scattered GPU lists, empty entries) ----
        unsigned long long selfm = 0;
        for (int e = lane; e < ne; e += 32) {
            unsigned long long sm = 0;
            for (int f = 0; f < ne; ++f)
                if (emod[f] == emod[e]) sm |= 1ULL << f;
            esame[e] = sm;
            if ((sm & ((1ULL << e) - 1)) == 0) selfm |= 1ULL << e;
        }
        {
            const unsigned lo = __reduce_or_sync(KE_FULL, (unsigned)selfm);
            const unsigned hi = __reduce_or_sync(KE_FULL, (unsigned)(selfm >> 32));
            selfm = (unsigned long long)hi << 32 | lo;
        }
        for (int g = lane; g < 2 * G; g += 32) mask[g] = 0u;
        __syncwarp();
        for (int e = 0; e < ne; ++e) {
            const int* gl = gpus + eoff[e];
            const int c = en[e];
            unsigned* mw = mask + (e < 32 ? 0 : G);
            const unsigned bit = 1u << (e & 31);
            ids += (unsigned long long)c;
            for (int i = lane; i < c; i += 32) {
                const int g = __ldg(gl + i);
                if ((unsigned)g >= (unsigned)G)
                    errs |= EVAL_ERR_GPU;
                else
                    atomicOr(&mw[g], bit);
            }
        }
        __syncwarp();
        // lookups the reference makes: every self entry's base latency, and the solo
        // bandwidth of every entry counted as a resident on some self entry's GPU
        unsigned long long used = 0;
        for (int g = lane; g < G; g += 32) {
            const unsigned long long m = (unsigned long long)mask[G + g] << 32 | mask[g];
            unsigned long long sm = m & selfm;
            if (!sm) continue;
            if (self_in) {
                used |= m;
            } else {
                while (sm) {
                    const int s0 = __ffsll((long long)sm) - 1;
                    sm &= sm - 1;
                    used |= m & ~esame[s0];
                }
            }
        }
        {
            const unsigned lo = __reduce_or_sync(KE_FULL, (unsigned)used);
            const unsigned hi = __reduce_or_sync(KE_FULL, (unsigned)(used >> 32));
            used = (unsigned long long)hi << 32 | lo;
        }
        bool miss = false;
        for (int e = lane; e < ne; e += 32)
            if (((selfm >> e & 1) && isnan(ebase[e])) || ((used >> e & 1) && isnan(eB[e])))
                miss = true;
        if (__any_sync(KE_FULL, miss)) {
            errs |= EVAL_ERR_SURFACE;
            if (lane == 0) st[a] = NAN;
            continue;
        }
        if (self_in) {
            for (int g = lane; g < G; g += 32) {
                const unsigned lo = mask[g], hi = mask[G + g];
                if (((unsigned long long)hi << 32 | lo) & selfm) dl[g] = ke_delta(P, eB, lo, hi);
            }
            __syncwarp();
        }
        for (int e = 0; e < ne; ++e) {
            const unsigned long long same = esame[e];
            const int self = __ffsll((long long)same) - 1;
            double rl;
            if (self < e) {
                rl = erect[self];  // StageAllocation::find: the module's first entry
            } else {
                double w = KE_NEG;
                const unsigned* mw = mask + (e < 32 ? 0 : G);
                const unsigned bit = 1u << (e & 31);
                for (int g = lane; g < G; g += 32) {
                    if (!(mw[g] & bit)) continue;
                    const double v =
                        self_in ? dl[g]
                                : ke_delta(P, eB, mask[g] & ~(unsigned)same,
                                           mask[G + g] & ~(unsigned)(same >> 32));
                    w = w < v ? v : w;  // std::max(worst, delta)
                }
                w = ke_wmax(w);
                rl = ebase[e] + w;
                if (lane == 0) erect[e] = rl;
                __syncwarp();
            }
            if (rect && lane == 0) rect[e0 + e] = rl;
            worst_stage = worst_stage < rl ? rl : worst_stage;
        }
        if (lane == 0) st[a] = worst_stage;
    }
    errs = (int)__reduce_or_sync(KE_FULL, (unsigned)errs);
    if (lane == 0) {
        if (errs) atomicOr(&stats->err, errs);
        atomicAdd(&stats->gpu_ids, ids);
        atomicAdd(&stats->entries, ents);
    }
}

// ---------------------------------------------------------------------------------------
// k_evaluate_fast — the common case at the memory roofline's instruction budget:
// include_self, no per-entry output, <= 32 entries, every module at most once.
//
// Then every entry is its module's "self" entry and, with include_self, a GPU's delta
// depends only on its resident set R_r, so
//     stage_time = max(0, max_e (base_e + max_{r in gpus_e} delta(R_r)))
//                = max(0, max_r (max_{e in R_r} base_e + delta(R_r)))
// because fp addition rounds monotonically (x <= y => fl(x + d) <= fl(y + d)): the max can
// move inside the sum without changing a bit.  One pass over the GPU slots (resident bitmap
// built from the id stream with one shared atomic per 32 ids) replaces the per-entry maxima.
// Anything else — duplicate modules, malformed entries or GPU lists, a NaN / below -1e300
// slot value — is appended to a worklist that k_evaluate (the full reference semantics)
// processes right after, on the same stream.
// ---------------------------------------------------------------------------------------
constexpr int KF_WARPS = 8;
__host__ __device__ inline size_t kf_warp_bytes(int G) {
    // resident bitmaps mask[G] | entry rates ebb[32] (double2) | shared resident sets[G]
    return 2 * (((size_t)G * 4 + 15) & ~(size_t)15) + 32 * 16;
}

// Set bit `bit` of mask[g] for one GPU id (ids outside the cluster flag the allocation).
__device__ __forceinline__ void kf_mark(unsigned* mask, int g, int G, unsigned bit, bool& bad) {
    if ((unsigned)g < (unsigned)G)
        atomicOr(&mask[g], bit);
    else
        bad = true;
}

// NS = GPU slots per lane (G <= 32 * NS, unrolled); NS = 0: any G (loop).
template <int NS>
__global__ void __launch_bounds__(32 * KF_WARPS)
    k_evaluate_fast(const EvalABI* __restrict__ ent, const int* __restrict__ gpus,
                    const long long* __restrict__ off, long long n, KEParams P, double* st,
                    KEStats* stats, long long* __restrict__ list) {
    extern __shared__ __align__(16) unsigned char kf_smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u, le = lt | (1u << lane);
    const int G = NS ? 32 * NS : P.G;
    const int Gr = P.G;
    unsigned char* wb = kf_smem + (size_t)wid * kf_warp_bytes(Gr);
    unsigned* mask = reinterpret_cast<unsigned*>(wb);
    double2* ebb = reinterpret_cast<double2*>(wb + (((size_t)Gr * 4 + 15) & ~(size_t)15));
    unsigned* sets = reinterpret_cast<unsigned*>(reinterpret_cast<unsigned char*>(ebb) + 32 * 16);
    // invariant: every mask word is zero between allocations (the slot pass clears)
    for (int g = lane; g < Gr; g += 32) mask[g] = 0u;
    __syncwarp();
    unsigned long long ids = 0, ents = 0;
    const double e1c = P.e1, e2c = P.e2, e3c = P.e3;
    const bool addv = P.additive != 0;
    const int L1 = P.L + 1;
    const long long stride = (long long)gridDim.x * KF_WARPS;
    for (long long a = (long long)blockIdx.x * KF_WARPS + wid; a < n; a += stride) {
        const long long a0 = off[a], a1 = off[a + 1];
        const long long ne64 = a1 - a0;
        bool hand = ne64 < 0 || ne64 > 32 || a0 < 0 || a1 > P.n_ent;
        if (!hand && ne64 == 0) {
            if (lane == 0) st[a] = 0.0;  // the reference's `worst` seed
            continue;
        }
        const int ne = hand ? 0 : (int)ne64;
        const bool has = lane < ne;
        int mod = -1 - lane, ng = 0;
        long long goff = 0;
        double bw = 0.0, bs = 0.0;
        if (has) {
            const int4* ep = reinterpret_cast<const int4*>(ent + a0 + lane);
            const int4 w0 = __ldg(ep);
            const int4 w1 = __ldg(ep + 1);
            mod = w0.x;
            const int d = w0.y, u = w0.z;
            ng = w0.w;
            goff = (long long)(((unsigned long long)(unsigned)w1.w << 32) | (unsigned)w1.z);
            // handed over: malformed entries, entries without GPUs, options outside the
            // rate tables (the full kernel reproduces the reference's lazy errors), rates
            // outside the range where the fused max cannot overflow (|B| <= 4, |base| <= 1e300)
            if (mod < 0 || mod >= P.n_mod || (w1.x != 0 && w1.x != P.L) || ng <= 0 ||
                goff < 0 || goff + ng > P.n_gpu_ids || u < 0 || u > P.L || d < 1 || d > Gr) {
                hand = true;
            } else {
                bw = __ldg(P.B + mod * L1 + u);
                bs = __ldg(P.base + (mod * Gr + (d - 1)) * L1 + u);
                hand = !(fabs(bw) <= 4.0) || !(fabs(bs) <= 1e300);
            }
        }
        const unsigned same = __match_any_sync(KE_FULL, mod);
        if (__any_sync(KE_FULL, hand || (has && (same & lt) != 0))) {
            if (lane == 0) list[atomicAdd(&stats->nlist, 1ULL)] = a;
            continue;
        }
        if (has) ebb[lane] = make_double2(bw, bs);
        // the value of a GPU whose only resident is this entry (the same operations as the
        // slot loop below on a one-bit set, so the same bits)
        double solo_v;
        {
            const double s1 = 0.0 + bw, p1 = 1.0 * bw;
            const double d0 = e1c + e2c * s1;
            solo_v = bs + (addv ? d0 + 0.0 : d0 + e3c * p1);
        }
        // resident bitmaps from the id stream: bit e of mask[r] <=> r in entries[e].gpus
        int bad = 0;
        const long long g0 = __shfl_sync(KE_FULL, goff, 0);
        const long long nxt = __shfl_up_sync(KE_FULL, goff + ng, 1);
        const int T = (int)(__shfl_sync(KE_FULL, goff + ng, ne - 1) - g0);
        if (__all_sync(KE_FULL, !has || lane == 0 || goff == nxt)) {
            // GPU lists stored back to back (the packed layout): one flat pass over the
            // allocation's ids, two 32-id chunks per step; id j belongs to the last entry
            // starting at or before j
            int rl = has ? (int)(goff - g0) : 0x7fffffff;  // this entry's start - chunk base
            const int* gp = gpus + g0 + lane;
            int ecar = -1;  // entry of the id before the chunk
            for (int c0 = 0; c0 < T; c0 += 64, gp += 64, rl -= 64) {
                const bool in0 = c0 + lane < T, in1 = c0 + 32 + lane < T;
                const int ga = in0 ? __ldg(gp) : 0;
                const int gb = in1 ? __ldg(gp + 32) : 0;
                const unsigned sa = __reduce_or_sync(KE_FULL, (unsigned)rl < 32u ? 1u << rl : 0u);
                const unsigned sbb = __reduce_or_sync(
                    KE_FULL, (unsigned)(rl - 32) < 32u ? 1u << (rl - 32) : 0u);
                const int ea = ecar + __popc(sa & le);
                ecar += __popc(sa);
                const int eb = ecar + __popc(sbb & le);
                ecar += __popc(sbb);
                if (in0) {
                    if ((unsigned)ga < (unsigned)Gr) atomicOr(&mask[ga], 1u << ea); else bad = 1;
                }
                if (in1) {
                    if ((unsigned)gb < (unsigned)Gr) atomicOr(&mask[gb], 1u << eb); else bad = 1;
                }
            }
        } else {
            for (int e = 0; e < ne; ++e) {
                const int c = __shfl_sync(KE_FULL, ng, e);
                const int* gl = gpus + __shfl_sync(KE_FULL, goff, e);
                const unsigned bit = 1u << e;
                for (int i = lane; i < c; i += 32) {
                    const int g = __ldg(gl + i);
                    if ((unsigned)g < (unsigned)Gr) atomicOr(&mask[g], bit); else bad = 1;
                }
            }
        }
        __syncwarp();
        // one pass over the GPU slots.  A slot with one resident contributes that entry's
        // solo value (collected as a bitmap); a shared slot's resident set goes to a list,
        // once per distinct set among 32 neighbouring slots (GPU windows make neighbours
        // share sets), and each listed set gets its delta (residents summed in entry order:
        // the reference's bits) plus the largest base latency among its residents.
        double best = 0.0;
        unsigned solo = 0u;
        int nsets = 0;
        auto slots32 = [&](int g0) {
            const int g = g0 + lane;
            unsigned m = g < Gr ? mask[g] : 0u;
            if (m) mask[g] = 0u;
            const bool multi = (m & (m - 1u)) != 0u;
            if (!multi) solo |= m;
            const unsigned same = __match_any_sync(KE_FULL, m);
            const bool lead = multi && (same & lt) == 0u;
            const unsigned bal = __ballot_sync(KE_FULL, lead);
            if (lead) sets[nsets + __popc(bal & lt)] = m;
            nsets += __popc(bal);
        };
        if (NS) {
            #pragma unroll
            for (int k = 0; k < (NS ? NS : 1); ++k) slots32(32 * k);
        } else {
            for (int g0 = 0; g0 < G; g0 += 32) slots32(g0);
        }
        __syncwarp();
        for (int i = lane; i < nsets; i += 32) {
            unsigned m = sets[i];
            double s = 0.0, p = 1.0, mb = -INFINITY;
            do {
                const int f = __ffs(m) - 1;
                m &= m - 1;
                const double2 v = ebb[f];
                s = s + v.x;
                p = p * v.x;
                mb = v.y > mb ? v.y : mb;
            } while (m);
            const double d0 = e1c + e2c * s;
            const double v = mb + (addv ? d0 + 0.0 : d0 + e3c * p);
            best = v > best ? v : best;
        }
        solo = __reduce_or_sync(KE_FULL, solo);
        if (solo >> lane & 1u) best = solo_v > best ? solo_v : best;
        if (__any_sync(KE_FULL, bad)) {  // GPU ids outside the cluster: full semantics
            if (lane == 0) list[atomicAdd(&stats->nlist, 1ULL)] = a;
            continue;
        }
        ents += (unsigned long long)ne;
        ids += (unsigned long long)(unsigned)T;
        // best >= +0 and finite: its bit pattern orders like its value (two 32-bit maxima)
        const unsigned long long bb = (unsigned long long)__double_as_longlong(best > 0.0 ? best : 0.0);
        const unsigned hi = __reduce_max_sync(KE_FULL, (unsigned)(bb >> 32));
        const unsigned lo = __reduce_max_sync(KE_FULL, (unsigned)(bb >> 32) == hi ? (unsigned)bb : 0u);
        if (lane == 0) st[a] = __longlong_as_double((long long)((unsigned long long)hi << 32 | lo));
    }
    if (lane == 0) {
        atomicAdd(&stats->gpu_ids, ids);
        atomicAdd(&stats->entries, ents);
    }
}

using KFastFn = void (*)(const EvalABI*, const int*, const long long*, long long, KEParams,
                         double*, KEStats*, long long*);
static KFastFn kf_select(int G) {
    switch ((G + 31) / 32) {
        case 1: return k_evaluate_fast<1>;
        case 2: return k_evaluate_fast<2>;
        case 3: return k_evaluate_fast<3>;
        case 4: return k_evaluate_fast<4>;
        default: return k_evaluate_fast<0>;
    }
}

void Engine::free_eval() {
    cudaFree(d_tab_base_);
    cudaFree(d_tab_B_);
    d_tab_base_ = d_tab_B_ = nullptr;
    for (int i = 0; i < 5; ++i) {
        cudaFree(ev_buf_[i]);
        ev_buf_[i] = nullptr;
        ev_cap_[i] = 0;
    }
    cudaFree(d_everr_);
    d_everr_ = nullptr;
    if (h_everr_) cudaFreeHost(h_everr_);
    h_everr_ = nullptr;
    if (eva_) cudaEventDestroy((cudaEvent_t)eva_);
    if (evb_) cudaEventDestroy((cudaEvent_t)evb_);
    if (evc_) cudaEventDestroy((cudaEvent_t)evc_);
    eva_ = evb_ = evc_ = nullptr;
    cudaFree(ev_list_);
    ev_list_ = nullptr;
    ev_list_cap_ = 0;
}

void Engine::set_rate_tables(const std::vector<double>& base, const std::vector<double>& B,
                             int n_mod, int G, int L, const Model& M) {
    CKE(cudaSetDevice(device_));
    cudaFree(d_tab_base_);
    cudaFree(d_tab_B_);
    d_tab_base_ = d_tab_B_ = nullptr;
    CKE(cudaMalloc(&d_tab_base_, std::max<size_t>(1, base.size()) * 8));
    CKE(cudaMalloc(&d_tab_B_, std::max<size_t>(1, B.size()) * 8));
    if (!base.empty())
        CKE(cudaMemcpy(d_tab_base_, base.data(), base.size() * 8, cudaMemcpyHostToDevice));
    if (!B.empty()) CKE(cudaMemcpy(d_tab_B_, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
    h2d_ += (long long)(base.size() + B.size()) * 8;
    dev_bytes_ += (long long)(base.size() + B.size()) * 8;
    tab_nmod_ = n_mod;
    tab_G_ = G;
    tab_L_ = L;
    tab_e1_ = M.e1;
    tab_e2_ = M.e2;
    tab_e3_ = M.e3;
    tab_add_ = M.additive ? 1 : 0;
    tab_self_ = M.include_self ? 1 : 0;
    if (!d_everr_) {
        CKE(cudaMalloc(&d_everr_, sizeof(KEStats)));
        CKE(cudaMallocHost(&h_everr_, sizeof(KEStats)));
        cudaEvent_t a, b, c;
        CKE(cudaEventCreate(&a));
        CKE(cudaEventCreate(&b));
        CKE(cudaEventCreate(&c));
        eva_ = a;
        evb_ = b;
        evc_ = c;
    }
    ev_smem_ = KE_WARPS * ke_warp_bytes(G);
    {
        // a property of the kernel (process-wide): only ever raised, contexts share it
        static std::mutex mu;
        static size_t set = 0;
        std::lock_guard<std::mutex> lk(mu);
        if (ev_smem_ > set) {
            CKE(cudaFuncSetAttribute(k_evaluate, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)ev_smem_));
            set = ev_smem_;
        }
    }
    int per_sm = 0, sms = 148;
    CKE(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_evaluate, 32 * KE_WARPS,
                                                      ev_smem_));
    CKE(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
    ev_grid_ = std::max(1, per_sm) * sms;
    evf_smem_ = KF_WARPS * kf_warp_bytes(G);
    {
        static std::mutex mu;
        static size_t set = 0;
        std::lock_guard<std::mutex> lk(mu);
        if (evf_smem_ > set) {
            for (int g : {32, 64, 96, 128, 160})
                CKE(cudaFuncSetAttribute(kf_select(g), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)evf_smem_));
            set = evf_smem_;
        }
    }
    per_sm = 0;
    CKE(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf_select(G), 32 * KF_WARPS,
                                                      evf_smem_));
    evf_grid_ = std::max(1, per_sm) * sms;
}

int Engine::evaluate_abi(const EvalABI* ent, long long n_ent, const int* gpus, long long n_gpu_ids,
                         const long long* off, long long n, double* st, double* rect, bool dev) {
    if (!d_tab_base_) throw std::runtime_error("evaluator rate tables not built");
    if (n <= 0) return 0;
    CKE(cudaSetDevice(device_));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream_);
    const EvalABI* de = ent;
    const int* dg = gpus;
    const long long* doff = off;
    double* dst = st;
    double* drect = rect;
    const size_t need[5] = {(size_t)std::max<long long>(1, n_ent) * sizeof(EvalABI),
                            (size_t)std::max<long long>(1, n_gpu_ids) * 4,
                            (size_t)(n + 1) * 8, (size_t)n * 8,
                            (size_t)std::max<long long>(1, n_ent) * 8};
    if (!dev) {
        for (int i = 0; i < 5; ++i) {
            if (i == 4 && !rect) continue;
            if (ev_cap_[i] < need[i]) {
                cudaFree(ev_buf_[i]);
                ev_buf_[i] = nullptr;
                dev_bytes_ -= (long long)ev_cap_[i];
                CKE(cudaMalloc(&ev_buf_[i], need[i]));
                ev_cap_[i] = need[i];
                dev_bytes_ += (long long)need[i];
            }
        }
        de = static_cast<const EvalABI*>(ev_buf_[0]);
        dg = static_cast<const int*>(ev_buf_[1]);
        doff = static_cast<const long long*>(ev_buf_[2]);
        dst = static_cast<double*>(ev_buf_[3]);
        drect = rect ? static_cast<double*>(ev_buf_[4]) : nullptr;
        if (n_ent > 0)
            CKE(cudaMemcpyAsync(ev_buf_[0], ent, n_ent * sizeof(EvalABI), cudaMemcpyHostToDevice, s));
        if (n_gpu_ids > 0)
            CKE(cudaMemcpyAsync(ev_buf_[1], gpus, n_gpu_ids * 4, cudaMemcpyHostToDevice, s));
        CKE(cudaMemcpyAsync(ev_buf_[2], off, (n + 1) * 8, cudaMemcpyHostToDevice, s));
        h2d_ += (long long)(n_ent * sizeof(EvalABI) + n_gpu_ids * 4 + (n + 1) * 8);
    }
    CKE(cudaMemsetAsync(d_everr_, 0, sizeof(KEStats), s));
    KEParams P;
    P.base = d_tab_base_;
    P.B = d_tab_B_;
    P.n_mod = tab_nmod_;
    P.G = tab_G_;
    P.L = tab_L_;
    P.additive = tab_add_;
    P.include_self = tab_self_;
    P.e1 = tab_e1_;
    P.e2 = tab_e2_;
    P.e3 = tab_e3_;
    P.n_ent = n_ent;
    P.n_gpu_ids = n_gpu_ids;
    // fast path for the common case (include_self, no per-entry output, 16-B aligned entry
    // records); the allocations it cannot take go through the worklist to k_evaluate
    // coefficients small enough that no slot value can overflow or drop below -1e300 with
    // |B| <= 4 and |base| <= 1e300 (the fast kernel hands other entries over)
    const double emax = std::fabs(tab_e1_) + 128.0 * std::fabs(tab_e2_) +
                        18446744073709551616.0 * std::fabs(tab_e3_);
    const bool fast = tab_self_ && !drect && (reinterpret_cast<uintptr_t>(de) & 15) == 0 &&
                      emax < 1e290 && tab_G_ <= 1024 && n_gpu_ids < (1LL << 31);
    long long* dlist = nullptr;
    if (fast) {
        if (ev_list_cap_ < (size_t)n) {
            cudaFree(ev_list_);
            ev_list_ = nullptr;
            dev_bytes_ -= (long long)ev_list_cap_ * 8;
            CKE(cudaMalloc(&ev_list_, (size_t)n * 8));
            ev_list_cap_ = (size_t)n;
            dev_bytes_ += (long long)n * 8;
        }
        dlist = static_cast<long long*>(ev_list_);
    }
    CKE(cudaEventRecord((cudaEvent_t)eva_, s));
    if (fast) {
        const long long wantf = (n + KF_WARPS - 1) / KF_WARPS;
        const unsigned gridf = (unsigned)std::min<long long>(wantf, evf_grid_);
        kf_select(tab_G_)<<<gridf, 32 * KF_WARPS, evf_smem_, s>>>(
            de, dg, doff, n, P, dst, reinterpret_cast<KEStats*>(d_everr_), dlist);
        CKE(cudaGetLastError());
        ++launches_;
        ++own_launches_;
    }
    CKE(cudaEventRecord((cudaEvent_t)evc_, s));
    {
        // the worklist's length is only known on the device: a full persistent grid that
        // exits at once when the list is empty
        const long long want = fast ? (long long)ev_grid_ : (n + KE_WARPS - 1) / KE_WARPS;
        const unsigned grid = (unsigned)std::min<long long>(want, ev_grid_);
        k_evaluate<<<grid, 32 * KE_WARPS, ev_smem_, s>>>(
            de, dg, doff, n, P, dst, drect, reinterpret_cast<KEStats*>(d_everr_), dlist);
        CKE(cudaGetLastError());
    }
    CKE(cudaEventRecord((cudaEvent_t)evb_, s));
    ++launches_;
    ++own_launches_;
    CKE(cudaMemcpyAsync(h_everr_, d_everr_, sizeof(KEStats), cudaMemcpyDeviceToHost, s));
    if (!dev) {
        CKE(cudaMemcpyAsync(st, dst, n * 8, cudaMemcpyDeviceToHost, s));
        d2h_ += n * 8;
        if (rect && n_ent > 0) {
            CKE(cudaMemcpyAsync(rect, drect, n_ent * 8, cudaMemcpyDeviceToHost, s));
            d2h_ += n_ent * 8;
        }
    }
    CKE(cudaStreamSynchronize(s));
    float ms = 0, msf = 0;
    CKE(cudaEventElapsedTime(&ms, (cudaEvent_t)eva_, (cudaEvent_t)evb_));
    CKE(cudaEventElapsedTime(&msf, (cudaEvent_t)eva_, (cudaEvent_t)evc_));
    evk_ms_ += ms;
    evf_ms_ += msf;
    eval_ms_ += ms;
    ++evk_n_;
    const KEStats* ks = reinterpret_cast<const KEStats*>(h_everr_);
    ev_fallback_ += fast ? (long long)ks->nlist : n;
    // algorithmic bytes: offsets + entries + GPU ids read, stage times (+ rectified) written
    evk_bytes_ += (long long)((n + 1) * 8 + ks->entries * sizeof(EvalABI) + ks->gpu_ids * 4 +
                              n * 8 + (rect ? ks->entries * 8 : 0));
    return ks->err;
}

}  // namespace mg
