// engine.cu — sm_100a kernels of the planner hot path and their host driver.
//
//   k_search : one resident persistent grid per stage search.  Every thread runs the
//              canonical-block DFS of search_core.cuh on cursors popped from a shared
//              queue; busy threads donate shallow subtrees when others go idle, so
//              irregular trees stay spread over all 148 SMs without host round trips.
//              MIN: shared fp64 incumbent (atomicMin on the bits).  FIRST: the earliest
//              hit in reference DFS order wins (path comparison under a seqlock).
//   k_eval   : batched stage_time of explicit allocations (perf_model.hpp:442-479) whose
//              entries use another quota granularity than the context (per-call rate
//              rows); the common case runs K1 on the ABI layout (eval.cu).
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include <cub/cub.cuh>

#include "engine.hpp"
#include "search_core.cuh"
#include "search_warp.cuh"

namespace mg {

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                     " at " #x);                                       \
    } while (0)

}  // namespace mg

#include "search_kernel.cuh"

namespace mg {

const void* k_search_fast_min_fn();    // engine_fast.cu, MG_FAST_MODE=0
const void* k_search_fast_first_fn();  // engine_fast.cu, MG_FAST_MODE=1


// ---------------------------------------------------------------------------
// K1: batched stage_time.  One warp per allocation.
// ---------------------------------------------------------------------------
struct EvalParams {
    double e1, e2, e3;
    int additive, include_self, G;
};

constexpr int EVAL_WARPS = 4;
constexpr int EVAL_MAXG = 1024;

__global__ void __launch_bounds__(32 * EVAL_WARPS)
    k_eval(const EvalEntry* ent, const int* gpus, const long long* off, long long n,
           const double* base, const double* Bt, EvalParams P, double* st, double* rect) {
    __shared__ unsigned long long mask[EVAL_WARPS][EVAL_MAXG];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long a = (long long)blockIdx.x * EVAL_WARPS + wid;
    if (a >= n) return;
    unsigned long long* mk = mask[wid];
    for (int r = lane; r < P.G; r += 32) mk[r] = 0ULL;
    __syncwarp();
    const long long e0 = off[a], e1n = off[a + 1];
    const int ne = (int)(e1n - e0);
    for (int e = 0; e < ne; ++e) {
        const EvalEntry& E = ent[e0 + e];
        for (int g = lane; g < E.n_gpus; g += 32) atomicOr(&mk[gpus[E.gpu_off + g]], 1ULL << e);
    }
    __syncwarp();
    double worst_stage = 0.0;
    for (int e = 0; e < ne; ++e) {
        // rectified_latency uses the module's first entry (StageAllocation::find) and, without
        // include_self, skips every resident entry of the same module
        int self = e;
        for (int f = 0; f < e; ++f)
            if (ent[e0 + f].module == ent[e0 + e].module) {
                self = f;
                break;
            }
        const EvalEntry& E = ent[e0 + self];
        double worst = NEG_INF;
        for (int g = lane; g < E.n_gpus; g += 32) {
            unsigned long long m = mk[gpus[E.gpu_off + g]];
            double s = 0.0, p = 1.0;
            int res = 0;
            for (int f = 0; f < ne; ++f) {
                if (!(m >> f & 1ULL)) continue;
                if (ent[e0 + f].module == E.module && !P.include_self) continue;
                double b = Bt[ent[e0 + f].row];
                s = s + b;
                p = p * b;
                ++res;
            }
            if (res == 0) p = 0.0;
            double dl = P.e1 + P.e2 * s;
            dl = dl + (P.additive ? 0.0 : P.e3 * p);
            worst = dl > worst ? dl : worst;
        }
        for (int o = 16; o; o >>= 1) {
            double v = __shfl_xor_sync(0xffffffffu, worst, o);
            worst = v > worst ? v : worst;
        }
        double rl = base[E.row] + worst;
        if (lane == 0 && rect) rect[e0 + e] = rl;
        worst_stage = rl > worst_stage ? rl : worst_stage;
    }
    if (lane == 0) st[a] = worst_stage;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static inline cudaStream_t S_(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// pinned staging layout: Spec | Ctl | Leaf | Cont | int, each 256-B aligned
static inline size_t pin_off(int i) {
    const size_t sz[5] = {sizeof(Spec), sizeof(Ctl), sizeof(Leaf), sizeof(Cont), sizeof(int)};
    size_t off = 0;
    for (int k = 0; k < i; ++k) off += (sz[k] + 255) & ~size_t(255);
    return off;
}

Engine::Engine(int device) : device_(device) {
    CK(cudaSetDevice(device));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    stream_ = s;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    ev0_ = a;
    ev1_ = b;
    cudaEvent_t c, d, e, f;
    CK(cudaEventCreate(&c));
    CK(cudaEventCreate(&d));
    CK(cudaEventCreate(&e));
    CK(cudaEventCreate(&f));
    evk0_ = c;
    evk1_ = d;
    evm0_ = e;
    evm1_ = f;
    // device mirror of the pinned staging layout: one upload and one read-back per search
    CK(cudaMalloc(&d_blob_, pin_off(5)));
    dev_bytes_ += (long long)pin_off(5);
    d_spec_ = static_cast<char*>(d_blob_) + pin_off(0);
    d_ctl_ = static_cast<char*>(d_blob_) + pin_off(1);
    d_leaf_ = static_cast<char*>(d_blob_) + pin_off(2);
    d_root_ = static_cast<char*>(d_blob_) + pin_off(3);
    CK(cudaMallocHost(&h_pin_, pin_off(5)));
}

Engine::~Engine() {
    cudaSetDevice(device_);
    free_eval();
    cudaFree(d_base_);
    cudaFree(d_B_);
    cudaFree(d_fp_);
    cudaFree(d_bound_);
    cudaFree(d_d_);
    cudaFree(d_u_);
    cudaFree(d_blob_);
    cudaFree(d_front_[0]);
    cudaFree(d_ready_);
    cudaFree(d_best_);
    cudaFreeHost(h_pin_);
    cudaEventDestroy((cudaEvent_t)ev0_);
    cudaEventDestroy((cudaEvent_t)ev1_);
    cudaEventDestroy((cudaEvent_t)evk0_);
    cudaEventDestroy((cudaEvent_t)evk1_);
    cudaEventDestroy((cudaEvent_t)evm0_);
    cudaEventDestroy((cudaEvent_t)evm1_);
    cudaStreamDestroy(S_(stream_));
}

void Engine::upload_rows(const Model& M) {
    CK(cudaSetDevice(device_));
    std::vector<double> base, B, fp, bound;
    std::vector<int> d, u;
    for (const auto& rows : M.rows)
        for (const auto& r : rows) {
            base.push_back(r.base);
            B.push_back(r.B);
            fp.push_back(r.fp);
            bound.push_back(r.bound);
            d.push_back(r.d);
            u.push_back(r.u);
        }
    n_rows_ = (int)base.size();
    h2d_ += (long long)base.size() * 40;
    size_t n = std::max<size_t>(1, base.size());
    cudaFree(d_base_);
    cudaFree(d_B_);
    cudaFree(d_fp_);
    cudaFree(d_bound_);
    cudaFree(d_d_);
    cudaFree(d_u_);
    CK(cudaMalloc(&d_base_, n * 8));
    CK(cudaMalloc(&d_B_, n * 8));
    CK(cudaMalloc(&d_fp_, n * 8));
    CK(cudaMalloc(&d_bound_, n * 8));
    CK(cudaMalloc(&d_d_, n * 4));
    CK(cudaMalloc(&d_u_, n * 4));
    dev_bytes_ += (long long)n * 40;
    if (!base.empty()) {
        CK(cudaMemcpy(d_base_, base.data(), base.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_B_, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_fp_, fp.data(), fp.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_bound_, bound.data(), bound.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_d_, d.data(), d.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_u_, u.data(), u.size() * 4, cudaMemcpyHostToDevice));
    }
}

// The cursor ring only has to hold the pieces in flight: donations happen when the queue
// is empty and walkers are idle, and a donation into a full ring simply fails (the walker
// keeps the work), so a ring of ring_per_walker slots per resident walker is always safe.
void Engine::ensure_front(long long n) {
    if (n <= front_cap_) return;
    long long cap = std::max<long long>(n, 1024);
    if (front_cap_) dev_bytes_ -= front_cap_ * (long long)(sizeof(Cont) + sizeof(int));
    cudaFree(d_front_[0]);
    CK(cudaMalloc(&d_front_[0], cap * sizeof(Cont)));
    cudaFree(d_ready_);
    CK(cudaMalloc(&d_ready_, cap * sizeof(int)));
    CK(cudaMemset(d_ready_, 0, cap * sizeof(int)));
    dev_bytes_ += cap * (long long)(sizeof(Cont) + sizeof(int));
    ticket_base_ = 0;
    if (!d_best_) {
        CK(cudaMalloc(&d_best_, sizeof(HitPath)));
        dev_bytes_ += sizeof(HitPath);
    }
    front_cap_ = cap;
}

SearchResult Engine::search(const Spec& S, double ub, double abort_below, SearchStats& st,
                            const HitPath* seed_path, const Leaf* seed_leaf) {
    CK(cudaSetDevice(device_));
    cudaStream_t s = S_(stream_);
    SearchResult res;
    res.value = ub;
    Rows R{d_base_, d_B_, d_fp_, d_bound_, d_d_, d_u_};
    char* pin = reinterpret_cast<char*>(h_pin_);
    Spec* hs = reinterpret_cast<Spec*>(pin + pin_off(0));
    Ctl* hc = reinterpret_cast<Ctl*>(pin + pin_off(1));
    Leaf* hl = reinterpret_cast<Leaf*>(pin + pin_off(2));
    Cont* hr = reinterpret_cast<Cont*>(pin + pin_off(3));
    int* hone = reinterpret_cast<int*>(pin + pin_off(4));
    *hs = S;
    hs->shard_rank = rank_;
    hs->shard_world = world_;
    if (world_ == 1 && tune_.share_world > 1) {
        hs->shard_rank = tune_.share_rank;
        hs->shard_world = tune_.share_world;
    }
    // option prefixes (o_0, o_1, o_2) are hashed to ranks: at 8 ranks the largest share of the
    // dominant cfg5 proof is 1.15x the mean (pairs: 1.3x; tools/shard_levels.sh)
    hs->shard_level = S.k >= 3 ? 2 : S.k - 1;
    if (tune_.shard_level >= 0) hs->shard_level = std::min(tune_.shard_level, S.k - 1);
    // donation policy: hand over only shallow levels, when the queue has run dry
    hs->don_max_level = S.k >= 6 ? S.k - 1 - tune_.don_depth : (S.k >= 3 ? S.k - 3 : 0);
    // long-running pieces may also hand over levels <= k-3 (see WarpHooks::abort)
    hs->don_max_level_tail = S.k - 3 > hs->don_max_level ? S.k - 3 : hs->don_max_level;
    hs->deep_after = tune_.deep_after;
    hs->lookahead = tune_.lookahead;
    hs->don_period = tune_.don_period;
    hs->backoff_cap_ns = tune_.backoff_cap;
    std::memset(hc, 0, sizeof(Ctl));
    union {
        double d;
        unsigned long long u;
    } cv;
    cv.d = ub;
    hc->inc = cv.u;
    hc->abort_below = abort_below;
    // tickets keep counting across searches, so slots never need clearing: a stale
    // ready value belongs to an older (smaller) ticket and can never match (q_head/q_tail
    // are set once the ring is sized, below)
    hc->outstanding = 1;
    std::memset(hr, 0, sizeof(Cont));
    hr->depth = 0;
    hr->nb = 1;
    hr->ph = 0;
    hr->oc = -1;
    hr->oe = (int16_t)S.lvl_n[0];
    hr->bsz[0] = (uint16_t)S.G;
    *hone = 1;
    // the specialised kernel when the model is the common one (same search, fewer branches)
    const bool fast = S.include_self && S.nonneg && !S.additive && !tune_.generic_kernel;
    const size_t smem = smem_bytes(S.G, S.k, fast);
    const void* kfn = !fast ? reinterpret_cast<const void*>(&k_search)
                      : S.mode == MODE_MIN ? k_search_fast_min_fn() : k_search_fast_first_fn();
    const int ki = !fast ? 0 : (S.mode == MODE_MIN ? 1 : 2);
    if (smem != grid_smem_[ki]) {
        if (smem > smem_attr_[ki]) {
            CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            smem_attr_[ki] = smem;
        }
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, 32 * WPC, smem));
        int sms = 148;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
        grid_k_[ki] = std::max(1, per_sm) * sms;  // all resident: spin-waiting needs it
        grid_smem_[ki] = smem;
    }
    grid_ = grid_k_[ki];
    ensure_front(grid_ * WPC * std::max(1, tune_.ring_per_walker));
    const long long cap = front_cap_;
    const unsigned long long t0 = ticket_base_;
    hc->q_head = t0;
    hc->q_tail = t0 + 1;
    hc->q_cap = (unsigned long long)cap;
    Cont* Q = reinterpret_cast<Cont*>(d_front_[0]);
    // small trees (few option tuples) do not need the whole GPU: a handful of resident
    // CTAs finishes them without spinning up thousands of idle walkers
    double tuples = 1.0;
    for (int l = 0; l < S.k; ++l) tuples *= (double)(S.lvl_n[l] > 0 ? S.lvl_n[l] : 1);
    const long long grid = (tuples * S.G <= tune_.small_tree) ? std::min<long long>(grid_, tune_.small_grid) : grid_;
    hc->walkers = (unsigned)(grid * WPC);
    // small trees: hand-overs cost more than they parallelise (each is a 1.3 KB piece
    // round trip through L2); let the walker that owns the root finish it
    hs->donate = grid < grid_ ? 0 : 1;
    CK(cudaEventRecord((cudaEvent_t)ev0_, s));
    if (S.mode == MODE_FIRST && seed_path && seed_leaf) {
        // a known leaf <= theta: the search only has to look at what precedes it
        hc->has_hit = 1;
        *hl = *seed_leaf;
        CK(cudaMemcpyAsync(d_best_, seed_path, sizeof(HitPath), cudaMemcpyHostToDevice, s));
        h2d_ += sizeof(HitPath);
    }
    // Spec | Ctl | Leaf | root Cont in one upload (the kernel publishes the root piece)
    CK(cudaMemcpyAsync(d_blob_, h_pin_, pin_off(4), cudaMemcpyHostToDevice, s));
    h2d_ += (long long)pin_off(4);
    const long long slot0 = (long long)(t0 % (unsigned long long)cap);
    CK(cudaEventRecord((cudaEvent_t)evk0_, s));
    {
        const Spec* a0 = (const Spec*)d_spec_;
        Ctl* a4 = (Ctl*)d_ctl_;
        HitPath* a5 = (HitPath*)d_best_;
        Leaf* a6 = (Leaf*)d_leaf_;
        const Cont* a7 = (const Cont*)d_root_;
        int* a3 = d_ready_;
        long long a8 = slot0;
        int a9 = (int)(t0 + 1);
        void* args[] = {&a0, &R, &Q, &a3, &a4, &a5, &a6, &a7, &a8, &a9};
        CK(cudaLaunchKernel(kfn, dim3((unsigned)grid), dim3(32 * WPC), args, smem, s));
    }
    CK(cudaEventRecord((cudaEvent_t)evk1_, s));
    ++launches_;
    ++own_launches_;
    ++st.rounds;
    // one read-back and one synchronisation per search: the control block and the leaf
    // (1 KB, read unconditionally — cheaper than a second round trip when there is a hit)
    CK(cudaMemcpyAsync(hc, d_ctl_, pin_off(3) - pin_off(1), cudaMemcpyDeviceToHost, s));
    d2h_ += (long long)(pin_off(3) - pin_off(1));
    CK(cudaEventRecord((cudaEvent_t)ev1_, s));
    CK(cudaEventSynchronize((cudaEvent_t)ev1_));
    CK(cudaGetLastError());
    ticket_base_ = hc->q_tail + 1;
    if (hc->has_hit && !hc->overflow) {
        res.found = true;
        res.leaf = *hl;
    }
    if (hc->overflow) res.overflow = true;
    if (S.mode == MODE_MIN) {
        if (hc->abort && !hc->overflow) res.aborted = true;
        union {
            unsigned long long u;
            double d;
        } w;
        w.u = hc->inc;
        res.value = w.d;
    }
    // ranks must leave every search with the same answer (they replay the same control
    // flow and all-gather once per search): merge after the local result is complete
    if (world_ > 1 && ag_) merge_ranks(S, hc, res);
    float kms = 0, ms = 0;
    CK(cudaEventElapsedTime(&kms, (cudaEvent_t)evk0_, (cudaEvent_t)evk1_));
    CK(cudaEventElapsedTime(&ms, (cudaEvent_t)ev0_, (cudaEvent_t)ev1_));
    ksearch_ms_ += kms;
    ++ksearch_n_;
    search_ms_ += ms;
    st.nodes += (long long)hc->nodes;
    st.leaves += (long long)hc->leaves;
    ++st.searches;
    alg_bytes_ += (long long)hc->leaves * 24LL * S.k;  // k option rows x 3 fp64 per leaf
    if (tune_.trace)
        std::fprintf(stderr, "[mosaic] %s k=%d thr=%.17g kernel=%.3fms total=%.3fms nodes=%llu "
                             "leaves=%llu donated=%llu %s\n",
                     S.mode == MODE_MIN ? "MIN  " : "FIRST", S.k,
                     S.mode == MODE_MIN ? ub : S.theta, kms, ms, hc->nodes, hc->leaves,
                     hc->q_tail - 1, res.found ? "hit" : (res.aborted ? "restart" : ""));
    return res;
}

void Engine::evaluate(const std::vector<EvalEntry>& ent, const std::vector<int>& gpus,
                      const std::vector<long long>& off, const std::vector<double>& base,
                      const std::vector<double>& Bt, int G, const Model& M,
                      std::vector<double>& st_out, std::vector<double>& rect_out) {
    CK(cudaSetDevice(device_));
    cudaStream_t s = S_(stream_);
    const long long n = (long long)off.size() - 1;
    st_out.assign(std::max<long long>(n, 0), 0.0);
    rect_out.assign(ent.size(), 0.0);
    if (n <= 0) return;
    if (G > EVAL_MAXG) throw std::runtime_error("evaluator supports up to 1024 GPUs");
    EvalEntry* de;
    int* dg;
    long long* doff;
    double *db, *dB, *dst, *drect;
    CK(cudaMallocAsync(&de, std::max<size_t>(1, ent.size()) * sizeof(EvalEntry), s));
    CK(cudaMallocAsync(&dg, std::max<size_t>(1, gpus.size()) * sizeof(int), s));
    CK(cudaMallocAsync(&doff, off.size() * sizeof(long long), s));
    CK(cudaMallocAsync(&db, std::max<size_t>(1, base.size()) * 8, s));
    CK(cudaMallocAsync(&dB, std::max<size_t>(1, Bt.size()) * 8, s));
    CK(cudaMallocAsync(&dst, n * 8, s));
    CK(cudaMallocAsync(&drect, std::max<size_t>(1, ent.size()) * 8, s));
    if (!ent.empty())
        CK(cudaMemcpyAsync(de, ent.data(), ent.size() * sizeof(EvalEntry), cudaMemcpyHostToDevice, s));
    if (!gpus.empty())
        CK(cudaMemcpyAsync(dg, gpus.data(), gpus.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(doff, off.data(), off.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
    if (!base.empty()) CK(cudaMemcpyAsync(db, base.data(), base.size() * 8, cudaMemcpyHostToDevice, s));
    if (!Bt.empty()) CK(cudaMemcpyAsync(dB, Bt.data(), Bt.size() * 8, cudaMemcpyHostToDevice, s));
    EvalParams P{M.e1, M.e2, M.e3, M.additive ? 1 : 0, M.include_self ? 1 : 0, G};
    CK(cudaEventRecord((cudaEvent_t)ev0_, s));
    k_eval<<<(unsigned)((n + EVAL_WARPS - 1) / EVAL_WARPS), 32 * EVAL_WARPS, 0, s>>>(
        de, dg, doff, n, db, dB, P, dst, drect);
    ++launches_;
    ++own_launches_;
    h2d_ += ent.size() * sizeof(EvalEntry) + gpus.size() * 4 + off.size() * 8 + base.size() * 16;
    d2h_ += n * 8 + ent.size() * 8;
    CK(cudaEventRecord((cudaEvent_t)ev1_, s));
    CK(cudaMemcpyAsync(st_out.data(), dst, n * 8, cudaMemcpyDeviceToHost, s));
    if (!ent.empty())
        CK(cudaMemcpyAsync(rect_out.data(), drect, ent.size() * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, (cudaEvent_t)ev0_, (cudaEvent_t)ev1_));
    eval_ms_ += ms;
    cudaFreeAsync(de, s);
    cudaFreeAsync(dg, s);
    cudaFreeAsync(doff, s);
    cudaFreeAsync(db, s);
    cudaFreeAsync(dB, s);
    cudaFreeAsync(dst, s);
    cudaFreeAsync(drect, s);
    CK(cudaStreamSynchronize(s));
}

// One all-gather per search (NCCL through the caller's callback): every rank contributes
// its outcome; MIN takes the smallest incumbent and restarts everywhere if any rank
// restarted, FIRST takes the hit that is earliest in reference DFS order.
struct RankRecord {
    int has_hit, aborted, overflow, pad;
    double inc;
    unsigned long long nodes, leaves;
    HitPath path;
    Leaf leaf;
};

static int host_path_cmp(const HitPath& a, const HitPath& b, int k) {
    for (int l = 0; l < k; ++l) {
        if (a.opt[l] != b.opt[l]) return a.opt[l] < b.opt[l] ? -1 : 1;
        for (int i = 0; i < a.nb[l]; ++i)
            if (a.x[l][i] != b.x[l][i]) return a.x[l][i] > b.x[l][i] ? -1 : 1;
    }
    return 0;
}

void Engine::merge_ranks(const Spec& S, const void* ctl_host, SearchResult& res) {
    const Ctl* hc = reinterpret_cast<const Ctl*>(ctl_host);
    if (!ag_) throw std::runtime_error("multi-GPU search without an all-gather");
    std::vector<RankRecord> all(world_);
    RankRecord mine;
    std::memset(&mine, 0, sizeof mine);
    mine.has_hit = res.found ? 1 : 0;
    mine.aborted = res.aborted ? 1 : 0;
    mine.overflow = res.overflow ? 1 : 0;
    union {
        unsigned long long u;
        double d;
    } w;
    w.u = hc->inc;
    mine.inc = w.d;
    mine.nodes = hc->nodes;
    mine.leaves = hc->leaves;
    if (res.found) {
        CK(cudaMemcpy(&mine.path, d_best_, sizeof(HitPath), cudaMemcpyDeviceToHost));
        mine.leaf = res.leaf;
    }
    if (ag_(ag_user_, &mine, all.data(), sizeof(RankRecord)) != 0)
        throw std::runtime_error("all-gather failed");
    int win = -1, minr = -1;
    double best = POS_INF;
    bool aborted = false, overflow = false;
    for (int r = 0; r < world_; ++r) {
        const RankRecord& x = all[r];
        aborted |= x.aborted != 0;
        overflow |= x.overflow != 0;
        if (minr < 0 || x.inc < best) {
            best = x.inc;
            minr = r;
        }
        if (x.has_hit && (win < 0 || host_path_cmp(x.path, all[win].path, S.k) < 0)) win = r;
    }
    res.overflow = overflow;
    if (S.mode == MODE_MIN) {
        // T* is the smallest incumbent; its leaf (the argmin the planner canonicalises)
        // comes from the rank that holds it (lowest rank on ties)
        res.aborted = aborted;
        res.value = best;
        res.found = all[minr].has_hit != 0;
        if (res.found) res.leaf = all[minr].leaf;
    } else {
        res.found = win >= 0;
        if (win >= 0) res.leaf = all[win].leaf;
    }
}

void Engine::mark(int which) {
    CK(cudaSetDevice(device_));
    CK(cudaEventRecord((cudaEvent_t)(which ? evm1_ : evm0_), S_(stream_)));
}

double Engine::marked_ms() {
    CK(cudaEventSynchronize((cudaEvent_t)evm1_));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, (cudaEvent_t)evm0_, (cudaEvent_t)evm1_));
    return ms;
}

}  // namespace mg
