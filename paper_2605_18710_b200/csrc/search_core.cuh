// search_core.cuh — per-thread canonical-placement branch-and-bound over one stage.
//
// What it searches (reference semantics, SURVEY.md §7 "Exact leaf order"):
//   levels j = 0..k-1 place module pi_j: choose an option (candidate_options order,
//   stage_eval.hpp:68-93) then a placement.  GPUs are kept as BLOCKS — maximal runs of
//   consecutive GPUs with identical resident sets, always contiguous — and a
//   placement takes a prefix of each eligible block (count vector x), visited in
//   descending lexicographic order of x.  That is exactly the set and order of leaves
//   FeasibilitySearch::place visits with its signature skip (stage_eval.hpp:204-214)
//   and, for ExactStageSolver (oracle.hpp:157-180), the order among canonical leaves,
//   which always contains its lexicographically-first argmin.
//
//   MODE_FIRST: first leaf in that DFS order whose stage_time <= theta
//               (FeasibilitySearch::run with theta = tau*(1+1e-12), filter
//               stage_eval.hpp:119-130; or the exact argmin with theta = T*).
//   MODE_MIN:   minimum stage_time over all leaves below an incumbent (T*).
//
// Leaf value is computed bit-exactly as stage_time (perf_model.hpp:442-479):
// residents summed in module-index order, (e1 + e2*sum) + e3*prod, base + worst,
// max starting at 0.0; the file is compiled with -fmad=false.  Because a block's
// contribution depends only on its resident set, the LAST level is resolved in
// closed form over blocks (per-block interval of admissible take counts) instead
// of enumerating its compositions.
//
// Pruning is sound and never reorders leaves: option filter/break, total quota
// demand (stage_eval.hpp:141-147,176-178), per-block capacity and memory
// (:208-210), an interference lower bound per block that adds a product-term
// envelope over the still-unplaced modules, and a one-step look-ahead that every
// unplaced module still has an option that fits.  All bound comparisons carry a
// 1e-12 relative slack so fp rounding can only weaken them.
#pragma once
#include <stdint.h>

#ifndef MG_HD
#define MG_HD __device__ __forceinline__
#endif
// Model flags read by the device search.  engine_fast.cu compiles the same code with
// MG_SPECIALIZE=1: include_self, non-negative coefficients and the multiplicative term fixed.
#ifndef MG_SPECIALIZE
#define MG_SPECIALIZE 0
#endif
#if MG_SPECIALIZE
#define MG_SELF(S) true
#define MG_NONNEG(S) true
#define MG_ADD(S) false
#else
#define MG_SELF(S) ((S).include_self)
#define MG_NONNEG(S) ((S).nonneg)
#define MG_ADD(S) ((S).additive)
#endif
#ifdef MG_MODE_FIXED
#define MG_MODE(S) (MG_MODE_FIXED)
#else
#define MG_MODE(S) ((S).mode)
#endif
#ifndef MG_COLD
#define MG_COLD static __device__ __noinline__  // rare paths (hits): kept out of the hot loop
#endif
// Device code below is only compiled by nvcc (the host planner includes this header
// for the Spec/Node/Leaf layouts only; there is no host search path).
#if defined(__CUDACC__) || defined(MG_HOST_HARNESS)
#define MG_DEVICE_CODE 1
#endif

namespace mg {

constexpr int MAXK = 12;   // modules per stage
constexpr int MAXB = 128;  // blocks per level
constexpr int MAXENV = 8;  // envelope lines per level
constexpr int FB = MAXB;   // blocks carried by a frontier node
constexpr double NEG_INF = -1.0e300;
constexpr double POS_INF = 1.0e300;
// MIN mode treats leaves within TIE_EPS (relative) of the incumbent as ties: it returns
// I* with T* in [I*(1 - TIE_EPS - rounding), I*].  Callers resolve a probe inside that
// band with an exact FIRST search (planner.cpp).
constexpr double TIE_EPS = 1e-14;
constexpr int TL_BINS = 4096;
constexpr unsigned long long TL_BIN_NS = 250000;  // 0.25 ms bins (trace timeline)
constexpr int TL_LOG = 65536;  // trace timeline: pieces longer than 2 ms, 4 words each

enum { MODE_MIN = 0, MODE_FIRST = 1 };

struct Spec {
    int k, G, L, mode;
    int nonneg, include_self, additive, use_filter;
    double e1, e2, e3, cap_slack;  // cap_slack = memory_capacity * (1 + 1e-12)
    double theta;                  // FIRST: accept iff stage_time <= theta
    double thp;                    // static prune threshold (theta or UB) * (1 + 1e-12)
    int lvl_n[MAXK];               // viable options per level (a prefix of the sorted list)
    int lvl_off[MAXK];             // row offset of each level's options
    int pos_lvl[MAXK];             // module-index position -> level
    int suffix_min[MAXK + 1];      // min quota demand d*u over levels >= j
    int shard_rank, shard_world;   // multi-GPU: this rank takes the option prefixes
    int shard_level;               //   (o_0..o_L) with shard_hash % world == rank, L = shard_level
    int don_max_level;             // work donation: only levels <= this are handed over
    int don_max_level_tail;        //   ... or <= this once a walker ran deep_after steps on a piece
    long long deep_after;
    int tail_idle;                 // > 0: tail phase once idle * tail_idle > walkers (after ramp-up)
    long long tail_after;          //   ... in which deeper hand-overs need only tail_after steps
    int don_min_rest;              // deeper hand-overs: at least this many options left (0: any)
    int local_don;                 // 1: idle siblings of a CTA get pieces through shared memory
    int lookahead;
    int donate;                    // 0: never hand work over (one walker owns the tree)
    int seq_cut;                   // MIN, models with negative coefficients: skip an option whose
                                   //   base latency reaches the incumbent (ExactStageSolver's
                                   //   sequential cut, oracle.hpp:127-139); solo walker only
    int don_period;                // check for idle walkers every don_period option steps (2^n)
    int backoff_cap_ns;            // idle walkers poll the queue with back-off up to this
    unsigned long long* timeline;  // trace >= 3 only: [0] launch t0 (ns), [1 + b] walker-busy ns
    // sharded searches: the control blocks (Ctl*) of this search's other shards — on peer
    // GPUs (CUDA IPC over NVLink) or, simulated, in the same launch.  MIN: an improving leaf
    // lowers every shard's incumbent (and raises their restart flag) right away.  FIRST: a
    // hit is also published to every shard, whose walkers then drop the work after it.
    void* peer_ctl[8];
    void* peer_best[8];  // FIRST: their published earliest hit (HitPath) and its leaf
    void* peer_leaf[8];
    int n_peer;
                                   //   in bin b of TL_BIN_NS (null otherwise)
    int env_n[MAXK + 1];           // product-term envelope over unplaced levels >= j
    double env_a[MAXK + 1][MAXENV];
    double env_b[MAXK + 1][MAXENV];
};

struct Rows {
    const double* base;
    const double* B;
    const double* fp;
    const double* bound;  // reference filter bound (stage_eval.hpp:122-127)
    const int* d;
    const int* u;
};

// Work item: a DFS cursor.  Levels < depth are placed; `ph` says how to continue at
// level `depth`: 0 = try the options after `oc`, 1 = try the compositions after `x` of
// option opt[depth] (within [lo, hi]).  The root is {depth 0, ph 0, oc -1}.  Items
// are ordered by `key`, which follows the reference DFS order.
// CAP blocks at `depth`: the ring's cursors hold MAXB, the CTA-local hand-off slot fewer.
template <int CAP>
struct alignas(16) ContT {
    unsigned long long key;
    uint16_t opt[MAXK];
    uint16_t depth, nb, ph;
    int16_t oc;
    int16_t oe;  // options at `depth` stop before oe (range split by work donation)
    int16_t pad16;
    int used;
    uint16_t bsz[CAP];
    uint16_t bmk[CAP];
    uint16_t x[CAP];
    uint16_t lo[CAP];
    uint16_t hi[CAP];
};
using Cont = ContT<MAXB>;

// Position of a FIRST hit in the reference DFS order: (option, composition) per level.
struct HitPath {
    uint16_t opt[MAXK];
    uint16_t nb[MAXK];
    uint16_t x[MAXK][MAXB];
};

// Leaf: options of every level plus the final block list (sizes, level masks).
struct Leaf {
    double value;
    int nb;
    int pad;
    uint16_t opt[MAXK];
    uint16_t bsz[2 * MAXB];
    uint16_t bmk[2 * MAXB];
};

// Block storage offsets: level j holds at most min(2^j, MAXB) blocks.
#if defined(__CUDACC__)
#define MG_HX __host__ __device__ inline
#else
#define MG_HX inline
#endif

// Blocks at level j: at most min(2^j, G) (each level splits every block in two), capped
// at MAXB.  The walker only stores levels 0..k-1 (the last level is closed-form).
MG_HX int lvl_capacity(int j, int G) {
    int c = j >= 7 ? MAXB : (1 << j);
    c = c < G ? c : G;
    return c < MAXB ? c : MAXB;
}

// Shared-memory footprint of one walker for a stage of k modules over G GPUs.
struct WalkLayout {
    int slots;    // sum of level capacities
    int nblk;     // max blocks at any stored level
    size_t bytes; // header + arrays, 16-B aligned
};

// DFS state of one walker.  The header is fixed; the arrays it points to are carved
// from shared memory right behind it, sized for the stage at hand (walk_layout).
struct Walk {
    // the chosen option's row per level, cached in shared memory when the level's option is
    // set (sel_set): block statistics and contributions read it instead of the option table
    double sB[MAXK], sBase[MAXK], sFp[MAXK];
    int sU[MAXK], sDU[MAXK];
    unsigned long long t_start;  // trace >= 3: start of the current piece (globaltimer)
    uint16_t opt[MAXK];
    int16_t oc[MAXK];
    int16_t oe[MAXK];  // option range end per level (exclusive)
    uint32_t vmask[MAXK];  // option pre-screen: viable options in [vbase, vbase + 32)
    int16_t vbase[MAXK];   //   (-1: not screened at this node yet)
    uint8_t vstop[MAXK];   //   no option beyond the window can pass
    uint8_t ph[MAXK];
    uint16_t nb[MAXK + 1];
    int used[MAXK + 1];
    int loff[MAXK + 1];  // slot offset of each level's block arrays
    int lcap[MAXK + 1];  // block capacity of each level
    int ps_lvl;
    uint16_t *bsz, *bmk, *x, *lo, *hi;           // per level (loff-indexed)
    int *pu, *cu, *sa, *sb;                      // per block of the current / child level
    double *pm, *psum, *pmb, *pP, *pmx, *cm, *cs, *cb, *cP, *cmx;
};

MG_HX size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// lean: the specialised (include_self) kernels keep no own-excluded bound arrays (pmx, cmx)
MG_HX WalkLayout walk_layout(int G, int k, bool lean = false) {
    WalkLayout L;
    L.slots = 0;
    L.nblk = 1;
    for (int j = 0; j < k; ++j) {
        const int c = lvl_capacity(j, G);
        L.slots += c;
        L.nblk = c > L.nblk ? c : L.nblk;
    }
    L.bytes = align16(sizeof(Walk)) + align16((lean ? 8 : 10) * 8 * (size_t)L.nblk) +
              align16(4 * 4 * (size_t)L.nblk) + align16(5 * 2 * (size_t)L.slots);
    return L;
}

// Point a walker's arrays into the shared-memory region right behind its header.
MG_HX void walk_carve(Walk& w, unsigned char* base, int G, int k, bool lean = false) {
    const WalkLayout L = walk_layout(G, k, lean);
    unsigned char* p = base + align16(sizeof(Walk));
    double* d = reinterpret_cast<double*>(p);
    const int n = L.nblk;
    w.pm = d;
    w.psum = d + n;
    w.pmb = d + 2 * n;
    w.pP = d + 3 * n;
    w.pmx = lean ? nullptr : d + 4 * n;
    const int c0 = lean ? 4 : 5;
    w.cm = d + c0 * n;
    w.cs = d + (c0 + 1) * n;
    w.cb = d + (c0 + 2) * n;
    w.cP = d + (c0 + 3) * n;
    w.cmx = lean ? nullptr : d + 9 * n;
    p += align16((lean ? 8 : 10) * 8 * (size_t)L.nblk);
    int* i = reinterpret_cast<int*>(p);
    w.pu = i;
    w.cu = i + L.nblk;
    w.sa = i + 2 * L.nblk;
    w.sb = i + 3 * L.nblk;
    p += align16(4 * 4 * (size_t)L.nblk);
    uint16_t* u = reinterpret_cast<uint16_t*>(p);
    w.bsz = u;
    w.bmk = u + L.slots;
    w.x = u + 2 * L.slots;
    w.lo = u + 3 * L.slots;
    w.hi = u + 4 * L.slots;
    int off = 0;
    for (int j = 0; j <= MAXK; ++j) {
        w.loff[j] = off;
        w.lcap[j] = j < k ? lvl_capacity(j, G) : 0;
        off += w.lcap[j];
    }
}

#ifdef MG_DEVICE_CODE
MG_HD double envelope(const Spec& S, int j, double P) {
    double g = POS_INF;
    #pragma unroll 1
    for (int i = 0; i < S.env_n[j]; ++i) {
        double v = S.env_a[j][i] + S.env_b[j][i] * P;
        g = v < g ? v : g;
    }
    return S.env_n[j] ? g : 0.0;
}

// Exact contribution of one GPU block with resident levels `mask` (all k options set):
// max over residents m of base_m + delta(residents), module-index order sums.  The chosen
// options' rows come from the walk's per-level cache (Walk::sB / sBase).
MG_HD double contrib(const Spec& S, const Walk& w, unsigned mask) {
    if (!mask) return NEG_INF;
    if (MG_SELF(S)) {
        double s = 0.0, p = 1.0, mb = NEG_INF;
        #pragma unroll 1
        for (int pos = 0; pos < S.k; ++pos) {
            int l = S.pos_lvl[pos];
            if (!(mask >> l & 1u)) continue;
            double b = w.sB[l];
            s = s + b;
            p = p * b;
            double ba = w.sBase[l];
            mb = ba > mb ? ba : mb;
        }
        double dl = S.e1 + S.e2 * s;
        dl = dl + (MG_ADD(S) ? 0.0 : S.e3 * p);
        return mb + dl;
    }
    double best = NEG_INF;
    #pragma unroll 1
    for (int pos = 0; pos < S.k; ++pos) {
        int l = S.pos_lvl[pos];
        if (!(mask >> l & 1u)) continue;
        double s = 0.0, p = 1.0;
        int n = 0;
        #pragma unroll 1
        for (int pos2 = 0; pos2 < S.k; ++pos2) {
            int l2 = S.pos_lvl[pos2];
            if (l2 == l || !(mask >> l2 & 1u)) continue;
            double b = w.sB[l2];
            s = s + b;
            p = p * b;
            ++n;
        }
        if (n == 0) p = 0.0;
        double dl = S.e1 + S.e2 * s;
        dl = dl + (MG_ADD(S) ? 0.0 : S.e3 * p);
        double v = w.sBase[l] + dl;
        best = v > best ? v : best;
    }
    return best;
}

// contrib() with the option of level `jl` replaced by `ol` (lanes evaluating different
// last-level options against the same shared walk): level jl's row from the table.
MG_HD double contrib_o(const Spec& S, const Rows& R, const Walk& w, unsigned mask, int jl,
                       int ol) {
    if (!mask) return NEG_INF;
    const int ro = S.lvl_off[jl] + ol;
    const double oB = R.B[ro], oBase = R.base[ro];
    if (MG_SELF(S)) {
        double s = 0.0, p = 1.0, mb = NEG_INF;
        #pragma unroll 1
        for (int pos = 0; pos < S.k; ++pos) {
            int l = S.pos_lvl[pos];
            if (!(mask >> l & 1u)) continue;
            double b = l == jl ? oB : w.sB[l];
            s = s + b;
            p = p * b;
            double ba = l == jl ? oBase : w.sBase[l];
            mb = ba > mb ? ba : mb;
        }
        double dl = S.e1 + S.e2 * s;
        dl = dl + (MG_ADD(S) ? 0.0 : S.e3 * p);
        return mb + dl;
    }
    double best = NEG_INF;
    #pragma unroll 1
    for (int pos = 0; pos < S.k; ++pos) {
        int l = S.pos_lvl[pos];
        if (!(mask >> l & 1u)) continue;
        double s = 0.0, p = 1.0;
        int n = 0;
        #pragma unroll 1
        for (int pos2 = 0; pos2 < S.k; ++pos2) {
            int l2 = S.pos_lvl[pos2];
            if (l2 == l || !(mask >> l2 & 1u)) continue;
            double b = l2 == jl ? oB : w.sB[l2];
            s = s + b;
            p = p * b;
            ++n;
        }
        if (n == 0) p = 0.0;
        double dl = S.e1 + S.e2 * s;
        dl = dl + (MG_ADD(S) ? 0.0 : S.e3 * p);
        double v = (l == jl ? oBase : w.sBase[l]) + dl;
        best = v > best ? v : best;
    }
    return best;
}

// Owner rank of an option prefix (levels 0..j with level j's option o).
MG_HD unsigned shard_hash(const uint16_t* opt, int j, int o) {
    unsigned h = 2166136261u;
    #pragma unroll 1
    for (int l = 0; l <= j; ++l) {
        h ^= (unsigned)(l == j ? o : opt[l]) + 0x9e37u * (unsigned)(l + 1);
        h *= 16777619u;
    }
    return h;
}

// 0 accept, 1 skip, 2 stop the option loop (all later options fail too).
MG_HD int opt_test(const Spec& S, const Rows& R, int r, double thr) {
    double base = R.base[r];
    if (S.use_filter && R.bound[r] > S.theta) {
        if (MG_NONNEG(S) && base + S.e1 > S.theta) return 2;
        if (!MG_NONNEG(S) && base > S.theta) return 2;
        return 1;
    }
    if (MG_NONNEG(S)) {
        double be = base + S.e1;
        if (be > thr) return 2;
        double lb = MG_SELF(S) ? be + S.e2 * R.B[r] : be;
        if (lb > thr) return 1;
    }
    return 0;
}

// Stats of a block (levels < nlev in `mask`), accumulated in placement order like
// FeasibilitySearch::push_module (stage_eval.hpp:224-229), from the walk's row cache.
MG_HD void block_stats(const Spec& S, const Walk& w, unsigned mask, int nlev, int& units,
                       double& mem, double& sum, double& mb, double& P, double& mbx) {
    units = 0;
    mem = 0.0;
    sum = 0.0;
    mb = NEG_INF;
    P = 1.0;
    mbx = NEG_INF;  // max(base - e2*B): residents' own-excluded additive bound
    #pragma unroll 1
    for (int l = 0; l < nlev; ++l) {
        if (!(mask >> l & 1u)) continue;
        units += w.sU[l];
        mem = mem + w.sFp[l];
        const double b = w.sB[l];
        sum = sum + b;
        P = P * b;
        double ba = w.sBase[l];
        mb = ba > mb ? ba : mb;
        double bx = ba - S.e2 * b;
        mbx = bx > mbx ? bx : mbx;
    }
}

// Set level l's option (lane 0 only) and cache its row for the block statistics.
MG_HD void sel_set(const Spec& S, const Rows& R, Walk& w, int l, int o) {
    const int r = S.lvl_off[l] + o;
    w.opt[l] = (uint16_t)o;
    w.sB[l] = R.B[r];
    w.sBase[l] = R.base[r];
    w.sFp[l] = R.fp[r];
    w.sU[l] = R.u[r];
    w.sDU[l] = R.d[r] * R.u[r];
}

// -1: path H precedes the walk's leaf path (levels 0..j), +1 follows it, 0 equal.
template <class HP>
MG_COLD int path_cmp(const HP* H, const Walk& w, int j) {
    #pragma unroll 1
    for (int l = 0; l <= j; ++l) {
        int ho = H->opt[l];
        if (ho != w.opt[l]) return ho < w.opt[l] ? -1 : 1;
        const int o0 = w.loff[l];
        #pragma unroll 1
        for (int b = 0; b < w.nb[l]; ++b) {
            int hx = H->x[l][b], wx = w.x[o0 + b];
            if (hx != wx) return hx > wx ? -1 : 1;  // larger count first
        }
    }
    return 0;
}

// Does H precede every leaf the walk can still reach?  Levels < j are fixed at their
// current (option, composition); at level j only the options after oc[j] remain.
template <class HP>
MG_COLD bool path_precedes_rest(const HP* H, const Walk& w, int j) {
    #pragma unroll 1
    for (int l = 0; l < j; ++l) {
        int ho = H->opt[l];
        if (ho != w.opt[l]) return ho < w.opt[l];
        const int o0 = w.loff[l];
        #pragma unroll 1
        for (int b = 0; b < w.nb[l]; ++b) {
            int hx = H->x[l][b], wx = w.x[o0 + b];
            if (hx != wx) return hx > wx;
        }
    }
    return (int)H->opt[j] <= w.oc[j];
}

template <class HP>
MG_COLD void path_store(HP* H, const Walk& w, int j) {
    #pragma unroll 1
    for (int l = 0; l <= j; ++l) {
        H->opt[l] = w.opt[l];
        H->nb[l] = w.nb[l];
        const int o0 = w.loff[l];
        #pragma unroll 1
        for (int b = 0; b < w.nb[l]; ++b) H->x[l][b] = w.x[o0 + b];
    }
}

// Write the FIRST leaf: options and the final block list after the last level.
MG_COLD void store_leaf(const Walk& w, int j, double v, Leaf& lf) {
    lf.value = v;
#pragma unroll 1
    for (int l = 0; l <= j; ++l) lf.opt[l] = w.opt[l];
    int o0 = w.loff[j];
    int m = 0;
#pragma unroll 1
    for (int b = 0; b < w.nb[j]; ++b) {
        int xb = w.x[o0 + b], s = w.bsz[o0 + b];
        unsigned mk = w.bmk[o0 + b];
        if (xb > 0) {
            lf.bsz[m] = (uint16_t)xb;
            lf.bmk[m] = (uint16_t)(mk | (1u << j));
            ++m;
        }
        if (xb < s) {
            lf.bsz[m] = (uint16_t)(s - xb);
            lf.bmk[m] = (uint16_t)mk;
            ++m;
        }
    }
    lf.nb = m;
}

#endif  // MG_DEVICE_CODE

}  // namespace mg
