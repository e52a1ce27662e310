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

#include <chrono>
#include <climits>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
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
const void* k_search_fast_any_fn();    // engine_fast.cu, MG_FAST_MODE=2 (mode read at run time)


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

// Per-device pool of the engine's launch resources (stream, events, staging blobs, cursor
// ring): contexts come and go (one per problem), the resources stay, so creating a context
// costs no cudaMalloc / cudaMallocHost / ring clearing after the first one on a device.
struct EngineRes {
    int device = -1;
    void *stream = nullptr, *ev[6] = {};
    void *d_blob = nullptr, *h_pin = nullptr, *d_best = nullptr, *h_best = nullptr;
    void* front = nullptr;
    int* ready = nullptr;
    long long front_cap = 0;
    unsigned long long ticket_base = 0;  // ring tickets keep counting across contexts
    void *d_rows = nullptr, *h_rows = nullptr;  // option-table arena (+ pinned staging)
    size_t rows_cap = 0;
};
static std::mutex g_pool_mu;
static std::vector<EngineRes> g_pool;

Engine::Engine(int device) : device_(device) {
    CK(cudaSetDevice(device));
    EngineRes r;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        for (size_t i = 0; i < g_pool.size(); ++i)
            if (g_pool[i].device == device) {
                r = g_pool[i];
                g_pool.erase(g_pool.begin() + i);
                break;
            }
    }
    if (r.device < 0) {
        r.device = device;
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        r.stream = s;
        for (auto& e : r.ev) {
            cudaEvent_t x;
            CK(cudaEventCreate(&x));
            e = x;
        }
        // per-search staging blobs (Spec | Ctl | Leaf | root Cont) for a whole batch: one
        // upload and one strided read-back per launch
        CK(cudaMalloc(&r.d_blob, MAXBATCH * BLOB_STRIDE));
        CK(cudaMallocHost(&r.h_pin, MAXBATCH * BLOB_STRIDE));
        CK(cudaMalloc(&r.d_best, MAXBATCH * sizeof(HitPath)));
        CK(cudaMallocHost(&r.h_best, MAXBATCH * sizeof(HitPath)));
    }
    stream_ = r.stream;
    ev0_ = r.ev[0];
    ev1_ = r.ev[1];
    evk0_ = r.ev[2];
    evk1_ = r.ev[3];
    evm0_ = r.ev[4];
    evm1_ = r.ev[5];
    d_blob_ = r.d_blob;
    h_pin_ = r.h_pin;
    d_best_ = r.d_best;
    h_best_ = r.h_best;
    d_front_[0] = r.front;
    d_ready_ = r.ready;
    front_cap_ = r.front_cap;
    ticket_base_ = r.ticket_base;
    d_rows_ = r.d_rows;
    h_rows_ = r.h_rows;
    rows_cap_ = r.rows_cap;
    dev_bytes_ += (long long)(MAXBATCH * (BLOB_STRIDE + sizeof(HitPath))) +
                  front_cap_ * (long long)(sizeof(Cont) + sizeof(int));
}

Engine::~Engine() {
    cudaSetDevice(device_);
    cudaStreamSynchronize(S_(stream_));
    free_eval();
    unlink_peers();
    free_nccl();
    if (d_tl_) cudaFree(d_tl_);
    EngineRes r;
    r.device = device_;
    r.stream = stream_;
    r.ev[0] = ev0_;
    r.ev[1] = ev1_;
    r.ev[2] = evk0_;
    r.ev[3] = evk1_;
    r.ev[4] = evm0_;
    r.ev[5] = evm1_;
    r.d_blob = d_blob_;
    r.h_pin = h_pin_;
    r.d_best = d_best_;
    r.h_best = h_best_;
    r.front = d_front_[0];
    r.ready = d_ready_;
    r.front_cap = front_cap_;
    r.ticket_base = ticket_base_;
    r.d_rows = d_rows_;
    r.h_rows = h_rows_;
    r.rows_cap = rows_cap_;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool.push_back(r);
}

void Engine::upload_rows(const Model& M) {
    CK(cudaSetDevice(device_));
    size_t n = 0;
    for (const auto& rows : M.rows) n += rows.size();
    n_rows_ = (int)n;
    // one pooled allocation carved into the six SoA arrays, one staged upload
    const size_t nn = std::max<size_t>(1, n);
    const size_t bytes = nn * 40 + 256;
    if (rows_cap_ < bytes) {
        cudaFree(d_rows_);
        if (h_rows_) cudaFreeHost(h_rows_);
        d_rows_ = h_rows_ = nullptr;
        dev_bytes_ -= (long long)rows_cap_;
        rows_cap_ = 0;
        CK(cudaMalloc(&d_rows_, bytes));
        CK(cudaMallocHost(&h_rows_, bytes));
        rows_cap_ = bytes;
        dev_bytes_ += (long long)bytes;
    }
    char* h = static_cast<char*>(h_rows_);
    double* hb = reinterpret_cast<double*>(h);
    double* hB = hb + nn;
    double* hf = hB + nn;
    double* hbd = hf + nn;
    int* hd = reinterpret_cast<int*>(hbd + nn);
    int* hu = hd + nn;
    size_t i = 0;
    for (const auto& rows : M.rows)
        for (const auto& r : rows) {
            hb[i] = r.base;
            hB[i] = r.B;
            hf[i] = r.fp;
            hbd[i] = r.bound;
            hd[i] = r.d;
            hu[i] = r.u;
            ++i;
        }
    char* d = static_cast<char*>(d_rows_);
    d_base_ = reinterpret_cast<double*>(d);
    d_B_ = d_base_ + nn;
    d_fp_ = d_B_ + nn;
    d_bound_ = d_fp_ + nn;
    d_d_ = reinterpret_cast<int*>(d_bound_ + nn);
    d_u_ = d_d_ + nn;
    cudaStream_t s = S_(stream_);
    CK(cudaMemcpyAsync(d, h, nn * 40, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    h2d_ += (long long)n * 40;
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
    front_cap_ = cap;
}

SearchResult Engine::search(const Spec& S, double ub, double abort_below, SearchStats& st,
                            const HitPath* seed_path, const Leaf* seed_leaf) {
    std::vector<BatchReq> one(1);
    one[0].S = S;
    one[0].ub = ub;
    one[0].abort_below = abort_below;
    one[0].seed_path = seed_path;
    one[0].seed_leaf = seed_leaf;
    one[0].st = &st;
    return search_batch(one)[0];
}

// The dynamic shared-memory limit is a property of the kernel function (process-wide), so it is
// only ever raised: several contexts (problems of different sizes) share the kernels.
static void raise_smem_attr(const void* kfn, size_t smem) {
    static std::mutex mu;
    static std::map<const void*, size_t> set;
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = set[kfn];
    if (smem > cur) {
        CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cur = smem;
    }
}

// Kernel, shared memory and resident grid for (kernel index, smem bytes).
void Engine::kernel_for(const std::vector<BatchReq>& reqs, size_t b0, size_t b1,
                        const void** kfn, size_t* smem, long long* grid) {
    const Spec& S0 = reqs[b0].S;
    // the specialised kernels when the model is the common one (same search, fewer branches);
    // a batch mixing MIN and FIRST searches runs the dynamic-mode build
    const bool fast = S0.include_self && S0.nonneg && !S0.additive && !tune_.generic_kernel;
    bool all_min = true, all_first = true;
    int kmax = 1;
    for (size_t i = b0; i < b1; ++i) {
        all_min &= reqs[i].S.mode == MODE_MIN;
        all_first &= reqs[i].S.mode == MODE_FIRST;
        kmax = std::max(kmax, reqs[i].S.k);
    }
    int ki = 0;
    *kfn = reinterpret_cast<const void*>(&k_search);
    if (fast) {
        ki = all_min ? 1 : (all_first ? 2 : 3);
        *kfn = all_min ? k_search_fast_min_fn()
                       : (all_first ? k_search_fast_first_fn() : k_search_fast_any_fn());
    }
    *smem = smem_bytes(S0.G, kmax, fast);
    const long long key = (long long)ki << 40 | (long long)*smem;
    auto it = grid_cache_.find(key);
    if (it == grid_cache_.end()) {
        raise_smem_attr(*kfn, *smem);
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, *kfn, 32 * WPC, *smem));
        int sms = 148;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
        // every CTA resident: walkers spin-wait on each other
        it = grid_cache_.emplace(key, (long long)std::max(1, per_sm) * sms).first;
    }
    *grid = it->second;
}

bool Engine::is_small(const BatchReq& q) const {
    double tuples = 1.0;
    for (int l = 0; l < q.S.k; ++l) tuples *= (double)(q.S.lvl_n[l] > 0 ? q.S.lvl_n[l] : 1);
    return q.force_solo || tuples * q.S.G <= tune_.small_tree;
}

// Peer GPUs' staging blobs through CUDA IPC: each rank exports its blob once, the handles
// are all-gathered over the rank plane, every rank maps the others' (over NVLink).  A rank
// that cannot map a peer just does not write to it (sharing is an optimisation).
void Engine::link_peers() {
    peers_tried_ = true;
    peer_blob_.assign(world_, nullptr);
    peer_best_.assign(world_, nullptr);
    cudaIpcMemHandle_t mine[2];
    std::memset(mine, 0, sizeof mine);
    if (cudaIpcGetMemHandle(&mine[0], d_blob_) != cudaSuccess ||
        cudaIpcGetMemHandle(&mine[1], d_best_) != cudaSuccess) {
        cudaGetLastError();
        std::memset(mine, 0, sizeof mine);
    }
    std::vector<cudaIpcMemHandle_t> all(2 * (size_t)world_);
    if (nccl_comm_)
        nccl_allgather(mine, all.data(), sizeof mine);
    else if (ag_(ag_user_, mine, all.data(), sizeof mine) != 0)
        throw std::runtime_error("all-gather failed");
    const cudaIpcMemHandle_t zero{};
    for (int r = 0; r < world_; ++r) {
        if (r == rank_ || std::memcmp(&all[2 * r], &zero, sizeof zero) == 0) continue;
        void *p = nullptr, *b = nullptr;
        if (cudaIpcOpenMemHandle(&p, all[2 * r], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess &&
            cudaIpcOpenMemHandle(&b, all[2 * r + 1], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) {
            peer_blob_[r] = p;
            peer_best_[r] = b;
        } else {
            cudaGetLastError();
            if (p) cudaIpcCloseMemHandle(p);
        }
    }
}

void Engine::unlink_peers() {
    for (void* p : peer_blob_)
        if (p) cudaIpcCloseMemHandle(p);
    for (void* p : peer_best_)
        if (p) cudaIpcCloseMemHandle(p);
    peer_blob_.clear();
    peer_best_.clear();
    peers_tried_ = false;
}

// share_all simulation on one device: every large search becomes share_all shards (the
// multi-GPU option-prefix split) in the same launch, merged with the multi-GPU rule.
std::vector<SearchResult> Engine::search_batch_sim(std::vector<BatchReq>& all_reqs) {
    const int W = std::min(tune_.share_all, 8);
    // sub-batches whose shards fit one launch (MAXBATCH searches)
    std::vector<SearchResult> all_out;
    all_out.reserve(all_reqs.size());
    size_t a = 0;
    while (a < all_reqs.size()) {
        size_t b = a, used = 0;
        while (b < all_reqs.size()) {
            const size_t c = is_small(all_reqs[b]) ? 1 : (size_t)W;
            if (used + c > (size_t)MAXBATCH) break;
            used += c;
            ++b;
        }
        std::vector<BatchReq> sub(all_reqs.begin() + a, all_reqs.begin() + b);
        std::vector<SearchResult> so = search_batch_sim_chunk(sub, W);
        all_out.insert(all_out.end(), so.begin(), so.end());
        a = b;
    }
    return all_out;
}

std::vector<SearchResult> Engine::search_batch_sim_chunk(std::vector<BatchReq>& reqs, int W) {
    std::vector<BatchReq> ex;
    std::vector<int> first(reqs.size()), cnt(reqs.size());
    for (size_t i = 0; i < reqs.size(); ++i) {
        first[i] = (int)ex.size();
        if (is_small(reqs[i])) {
            ex.push_back(reqs[i]);
            cnt[i] = 1;
            continue;
        }
        for (int r = 0; r < W; ++r) {
            ex.push_back(reqs[i]);
            ex.back().sim_rank = r;
            ex.back().sim_world = W;
        }
        cnt[i] = W;
    }
    const void* kfn;
    size_t smem;
    long long grid_cap;
    kernel_for(ex, 0, ex.size(), &kfn, &smem, &grid_cap);
    std::vector<SearchResult> exo(ex.size());
    launch_chunk(ex, 0, ex.size(), kfn, smem, grid_cap, exo);
    HitPath* hbest = reinterpret_cast<HitPath*>(h_best_);
    CK(cudaMemcpyAsync(hbest, d_best_, ex.size() * sizeof(HitPath), cudaMemcpyDeviceToHost, S_(stream_)));
    CK(cudaStreamSynchronize(S_(stream_)));
    std::vector<SearchResult> out(reqs.size());
    std::vector<RankRecord> per(W);
    for (size_t i = 0; i < reqs.size(); ++i) {
        if (cnt[i] == 1) {
            out[i] = exo[first[i]];
            continue;
        }
        for (int r = 0; r < W; ++r) {
            const SearchResult& x = exo[first[i] + r];
            RankRecord& m = per[r];
            std::memset(&m, 0, sizeof m);
            m.has_hit = x.found ? 1 : 0;
            m.aborted = x.aborted ? 1 : 0;
            m.overflow = x.overflow ? 1 : 0;
            m.inc = reqs[i].S.mode == MODE_MIN ? x.value : POS_INF;
            if (x.found) {
                m.path = hbest[first[i] + r];
                m.leaf = x.leaf;
            }
        }
        merge_rank_records(per.data(), W, reqs[i].S.mode, reqs[i].S.k, out[i]);
    }
    return out;
}

std::vector<SearchResult> Engine::search_batch(std::vector<BatchReq>& reqs) {
    CK(cudaSetDevice(device_));
    if (tune_.share_all > 1 && world_ == 1) return search_batch_sim(reqs);
    std::vector<SearchResult> out(reqs.size());
    size_t b0 = 0;
    while (b0 < reqs.size()) {
        // chunk: at most MAXBATCH searches, all resident at once
        const void* kfn;
        size_t smem;
        long long grid_cap;
        size_t b1 = std::min(reqs.size(), b0 + (size_t)MAXBATCH);
        kernel_for(reqs, b0, b1, &kfn, &smem, &grid_cap);
        b1 = std::min<size_t>(b1, b0 + (size_t)std::max<long long>(1, grid_cap));
        launch_chunk(reqs, b0, b1, kfn, smem, grid_cap, out);
        b0 = b1;
    }
    return out;
}

void Engine::launch_chunk(std::vector<BatchReq>& reqs, size_t b0, size_t b1, const void* kfn,
                          size_t smem, long long grid_cap, std::vector<SearchResult>& out) {
    cudaStream_t s = S_(stream_);
    const int n = (int)(b1 - b0);
    const auto c0 = std::chrono::steady_clock::now();
    Rows R{d_base_, d_B_, d_fp_, d_bound_, d_d_, d_u_};
    char* pin = reinterpret_cast<char*>(h_pin_);
    HitPath* hbest = reinterpret_cast<HitPath*>(h_best_);
    // CTAs per search: small trees (few option tuples) finish on a handful of CTAs without
    // hand-overs; the rest share the resident grid equally
    std::vector<int> ctas(n);
    std::vector<char> small(n);
    long long small_total = 0;
    int n_big = 0;
    for (int i = 0; i < n; ++i) {
        const Spec& S = reqs[b0 + i].S;
        small[i] = is_small(reqs[b0 + i]);
        if (small[i]) {
            // one walker owns the whole tree (solo mode, search_kernel.cuh); with several ranks
            // a small search runs whole on ONE rank (its owner) instead of sharded everywhere
            ctas[i] = sharded() && owner_of(i) != rank_ ? 0 : 1;
            small_total += ctas[i];
        } else {
            ++n_big;
        }
    }
    const long long left = std::max<long long>(0, grid_cap - small_total);
    for (int i = 0; i < n; ++i)
        if (!small[i]) ctas[i] = (int)std::max<long long>(1, left / std::max(1, n_big));
    BatchMap map;
    std::memset(&map, 0, sizeof map);
    map.n = n;
    long long qtot = 0;
    for (int i = 0; i < n; ++i) {
        map.cta_off[i + 1] = map.cta_off[i] + ctas[i];
        map.q_off[i] = qtot;
        qtot += (long long)ctas[i] * WPC * std::max(1, tune_.ring_per_walker);
    }
    ensure_front(qtot);
    if (sharded() && tune_.share_peers && !peers_tried_) link_peers();
    const unsigned long long t0 = ticket_base_;
    for (int i = 0; i < n; ++i) {
        BatchReq& q = reqs[b0 + i];
        char* blob = pin + (size_t)i * BLOB_STRIDE;
        Spec* hs = reinterpret_cast<Spec*>(blob + BLOB_SPEC);
        Ctl* hc = reinterpret_cast<Ctl*>(blob + BLOB_CTL);
        Leaf* hl = reinterpret_cast<Leaf*>(blob + BLOB_LEAF);
        Cont* hr = reinterpret_cast<Cont*>(blob + BLOB_ROOT);
        const Spec& S = q.S;
        *hs = S;
        hs->shard_rank = rank_;
        hs->shard_world = world_;
        if (world_ == 1 && tune_.share_world > 1) {
            hs->shard_rank = tune_.share_rank;
            hs->shard_world = tune_.share_world;
        }
        if (small[i]) hs->shard_world = 1;  // solo searches are never sharded (owner runs it)
        // option prefixes (o_0, o_1, o_2) are hashed to ranks: at 8 ranks the largest share of
        // the dominant cfg5 proof is 1.15x the mean (pairs: 1.3x)
        hs->shard_level = S.k >= 3 ? 2 : S.k - 1;
        if (tune_.shard_level >= 0) hs->shard_level = std::min(tune_.shard_level, S.k - 1);
        // donation policy: hand over only shallow levels, when the queue has run dry
        const bool first_ = S.mode == MODE_FIRST;
        const int ddep = first_ && tune_.don_depth_first >= 0 ? tune_.don_depth_first : tune_.don_depth;
        const int dtail = first_ && tune_.don_tail_first >= 0 ? tune_.don_tail_first : tune_.don_tail;
        hs->don_max_level = S.k >= 6 ? S.k - 1 - ddep
                                     : (S.k >= 3 ? std::max(0, S.k - 1 - tune_.don_depth_small) : 0);
        // long-running pieces may also hand over levels <= k-3 (see WarpHooks::abort)
        hs->don_max_level_tail = std::max(hs->don_max_level, S.k - 1 - dtail);
        hs->deep_after = tune_.deep_after;
        hs->tail_idle = tune_.tail_idle;
        hs->tail_after = tune_.tail_after;
        hs->don_min_rest = tune_.don_min_rest;
        hs->local_don = tune_.local_handover;
        hs->lookahead = tune_.lookahead;
        // small stages: control reads every step (faster ramp-up of trees of a few hundred
        // nodes); large ones every don_period steps (the L2 round trip per step costs more)
        hs->don_period = S.k < tune_.restart_k ? tune_.don_period_small : tune_.don_period;
        hs->backoff_cap_ns = tune_.backoff_cap;
        // small trees: hand-overs cost more than they parallelise; the root's walker finishes
        hs->donate = small[i] ? 0 : 1;
        hs->timeline = nullptr;
        hs->n_peer = 0;
        if (q.sim_world > 1) {
            // share_all simulation: this launch holds every shard of the search, the siblings
            // sit next to it in the blob
            hs->shard_rank = q.sim_rank;
            hs->shard_world = q.sim_world;
            if (tune_.share_peers)
                for (int r = 0; r < q.sim_world && hs->n_peer < 8; ++r)
                    if (r != q.sim_rank) {
                        const size_t x = (size_t)(i - q.sim_rank + r);
                        hs->peer_ctl[hs->n_peer] = static_cast<char*>(d_blob_) + x * BLOB_STRIDE + BLOB_CTL;
                        hs->peer_best[hs->n_peer] = static_cast<HitPath*>(d_best_) + x;
                        hs->peer_leaf[hs->n_peer] = static_cast<char*>(d_blob_) + x * BLOB_STRIDE + BLOB_LEAF;
                        ++hs->n_peer;
                    }
        } else if (sharded() && !small[i] && !peer_blob_.empty()) {
            // the same search's control block on every other rank (IPC-mapped peer memory)
            for (int r = 0; r < world_ && hs->n_peer < 8; ++r)
                if (r != rank_ && peer_blob_[r] && peer_best_[r]) {
                    hs->peer_ctl[hs->n_peer] = static_cast<char*>(peer_blob_[r]) + (size_t)i * BLOB_STRIDE + BLOB_CTL;
                    hs->peer_best[hs->n_peer] = static_cast<HitPath*>(peer_best_[r]) + i;
                    hs->peer_leaf[hs->n_peer] = static_cast<char*>(peer_blob_[r]) + (size_t)i * BLOB_STRIDE + BLOB_LEAF;
                    ++hs->n_peer;
                }
        }
        if (tune_.trace >= 3 && i == 0 && !small[i]) {
            if (!d_tl_) CK(cudaMalloc(&d_tl_, (2 + TL_BINS + 4 * TL_LOG) * sizeof(unsigned long long)));
            CK(cudaMemsetAsync(d_tl_, 0, (2 + TL_BINS + 4 * TL_LOG) * sizeof(unsigned long long), s));
            hs->timeline = static_cast<unsigned long long*>(d_tl_);
        }
        std::memset(hc, 0, sizeof(Ctl));
        union {
            double d;
            unsigned long long u;
        } cv;
        cv.d = q.ub;
        hc->inc = cv.u;
        hc->abort_below = q.abort_below;
        // tickets keep counting across launches (every search of this launch starts at t0),
        // so ring slots never need clearing: a stale ready value belongs to an older ticket
        hc->outstanding = 1;
        hc->q_head = t0;
        hc->q_base = t0;
        hc->q_tail = t0 + 1;
        hc->q_cap = (unsigned long long)ctas[i] * WPC * std::max(1, tune_.ring_per_walker);
        hc->walkers = (unsigned)(ctas[i] * WPC);
        std::memset(hr, 0, sizeof(Cont));
        hr->depth = 0;
        hr->nb = 1;
        hr->ph = 0;
        hr->oc = -1;
        hr->oe = (int16_t)S.lvl_n[0];
        hr->bsz[0] = (uint16_t)S.G;
        if (S.mode == MODE_FIRST && q.seed_path && q.seed_leaf) {
            // a known leaf <= theta: the search only has to look at what precedes it
            hc->has_hit = 1;
            *hl = *q.seed_leaf;
            hbest[i] = *q.seed_path;
        }
    }
    CK(cudaEventRecord((cudaEvent_t)ev0_, s));
    {
        // seeded FIRST searches: their hit paths in ONE copy (the range spanning them)
        int s0 = -1, s1 = -1;
        for (int i = 0; i < n; ++i)
            if (reqs[b0 + i].S.mode == MODE_FIRST && reqs[b0 + i].seed_path && reqs[b0 + i].seed_leaf) {
                if (s0 < 0) s0 = i;
                s1 = i;
            }
        if (s0 >= 0) {
            CK(cudaMemcpyAsync(static_cast<HitPath*>(d_best_) + s0, hbest + s0,
                               (size_t)(s1 - s0 + 1) * sizeof(HitPath), cudaMemcpyHostToDevice, s));
            h2d_ += (long long)(s1 - s0 + 1) * sizeof(HitPath);
        }
    }
    // every search's Spec | Ctl | Leaf | root Cont in one upload
    CK(cudaMemcpyAsync(d_blob_, h_pin_, (size_t)n * BLOB_STRIDE, cudaMemcpyHostToDevice, s));
    h2d_ += (long long)n * BLOB_STRIDE;
    CK(cudaEventRecord((cudaEvent_t)evk0_, s));
    {
        char* db = static_cast<char*>(d_blob_);
        const Spec* a0 = reinterpret_cast<const Spec*>(db + BLOB_SPEC);
        Ctl* a4 = reinterpret_cast<Ctl*>(db + BLOB_CTL);
        HitPath* a5 = static_cast<HitPath*>(d_best_);
        Leaf* a6 = reinterpret_cast<Leaf*>(db + BLOB_LEAF);
        const Cont* a7 = reinterpret_cast<const Cont*>(db + BLOB_ROOT);
        Cont* Q = reinterpret_cast<Cont*>(d_front_[0]);
        int* a3 = d_ready_;
        int a9 = (int)(t0 + 1);
        void* args[] = {&a0, &R, &Q, &a3, &a4, &a5, &a6, &a7, &map, &a9};
        if (map.cta_off[n] > 0)  // (every search of the launch may belong to other ranks)
            CK(cudaLaunchKernel(kfn, dim3((unsigned)map.cta_off[n]), dim3(32 * WPC), args, smem, s));
    }
    CK(cudaEventRecord((cudaEvent_t)evk1_, s));
    ++launches_;
    ++own_launches_;
    // one strided read-back of every search's control block and leaf, one synchronisation
    CK(cudaMemcpy2DAsync(pin + BLOB_CTL, BLOB_STRIDE, static_cast<char*>(d_blob_) + BLOB_CTL,
                         BLOB_STRIDE, BLOB_ROOT - BLOB_CTL, n, cudaMemcpyDeviceToHost, s));
    d2h_ += (long long)n * (BLOB_ROOT - BLOB_CTL);
    CK(cudaEventRecord((cudaEvent_t)ev1_, s));
    const auto c1 = std::chrono::steady_clock::now();
    CK(cudaEventSynchronize((cudaEvent_t)ev1_));
    const auto c2 = std::chrono::steady_clock::now();
    CK(cudaGetLastError());
    float kms = 0, ms = 0;
    CK(cudaEventElapsedTime(&kms, (cudaEvent_t)evk0_, (cudaEvent_t)evk1_));
    CK(cudaEventElapsedTime(&ms, (cudaEvent_t)ev0_, (cudaEvent_t)ev1_));
    ksearch_ms_ += kms;
    ++ksearch_n_;
    search_ms_ += ms;
    unsigned long long tmax = t0;
    for (int i = 0; i < n; ++i) {
        const BatchReq& q = reqs[b0 + i];
        const Spec& S = q.S;
        const char* blob = pin + (size_t)i * BLOB_STRIDE;
        const Ctl* hc = reinterpret_cast<const Ctl*>(blob + BLOB_CTL);
        const Leaf* hl = reinterpret_cast<const Leaf*>(blob + BLOB_LEAF);
        SearchResult& res = out[b0 + i];
        res.value = q.ub;
        tmax = std::max<unsigned long long>(tmax, hc->q_tail);
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
        SearchStats& st = *q.st;
        ++st.rounds;
        st.nodes += (long long)hc->nodes;
        st.leaves += (long long)hc->leaves;
        ++st.searches;
        alg_bytes_ += (long long)hc->leaves * 24LL * S.k;  // k option rows x 3 fp64 per leaf
        if (tune_.trace == 1 || tune_.trace == 3)
            std::fprintf(stderr, "[mosaic] %s k=%d thr=%.17g batch=%d ctas=%d kernel=%.3fms total=%.3fms "
                                 "nodes=%llu leaves=%llu %s\n",
                         S.mode == MODE_MIN ? "MIN  " : "FIRST", S.k,
                         S.mode == MODE_MIN ? q.ub : S.theta, n, ctas[i], kms, ms, hc->nodes,
                         hc->leaves, res.found ? "hit" : (res.aborted ? "restart" : ""));
        if (tune_.trace == 3 && hc->pieces > 0)
            std::fprintf(stderr, "[mosaic]       walkers=%u pieces=%llu (hand-over requests %llu, hand-overs "
                                 "%llu, abandoned %llu) busy %.1f%% of walkers x kernel time\n",
                         hc->walkers, hc->pieces, hc->dbg[7], hc->dbg[5], hc->dbg[6],
                         100.0 * hc->busy / std::max(1.0, (double)hc->walkers * kms * 1e6));
    }
    ticket_base_ = tmax + 1;
    if (tune_.trace >= 3 && n > 0 && !small[0]) {
        // busy walkers over time (first search of the launch), 1 ms per column
        std::vector<unsigned long long> tl(2 + TL_BINS + 4 * TL_LOG);
        CK(cudaMemcpy(tl.data(), d_tl_, tl.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        int last = 0;
        for (int b = 0; b < TL_BINS; ++b)
            if (tl[1 + b]) last = b;
        std::fprintf(stderr, "[mosaic] timeline (mean busy walkers of %d per ms):", ctas[0] * WPC);
        for (int b = 0; b <= last; b += 4) {
            unsigned long long sum = 0;
            for (int i = b; i < b + 4 && i < TL_BINS; ++i) sum += tl[1 + i];
            std::fprintf(stderr, " %.0f", (double)sum / (4.0 * TL_BIN_NS));
        }
        std::fprintf(stderr, "\n");
        Ctl* hc0 = reinterpret_cast<Ctl*>(pin + BLOB_CTL);
        std::fprintf(stderr, "[mosaic] requests: ring-full %llu, range<2 %llu, rest-below-max %llu, "
                             "floor>max %llu, deep %llu; by level:", hc0->dbg[0], hc0->dbg[1],
                     hc0->dbg[2], hc0->dbg[3], hc0->dbg[4]);
        for (int l = 0; l < 8; ++l) std::fprintf(stderr, " %llu", hc0->dbg[8 + l]);
        std::fprintf(stderr, "\n");
        const unsigned long long nlog = std::min<unsigned long long>(tl[1 + TL_BINS], TL_LOG);
        for (unsigned long long i = 0; i < nlog; ++i) {
            const unsigned long long* e = &tl[2 + TL_BINS + 4 * i];
            std::fprintf(stderr, "[mosaic] piece %.3f %.3f depth=%llu nodes=%llu\n", e[0] * 1e-6,
                         e[1] * 1e-6, e[2], e[3]);
        }
    }
    if (tune_.trace >= 2) {
        const auto c3 = std::chrono::steady_clock::now();
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        std::fprintf(stderr, "[mosaic] launch of %d: host prep %.1f us, wait %.1f us (stream %.1f us, "
                             "kernel %.1f us), post %.1f us\n",
                     n, us(c0, c1), us(c1, c2), 1e3 * ms, 1e3 * kms, us(c2, c3));
    }
    // ranks must leave every search with the same answer (they replay the same control flow
    // and all-gather once per launch): merge after the local results are complete
    if (sharded()) {
        owned_.assign(n, -1);
        for (int i = 0; i < n; ++i)
            if (small[i]) owned_[i] = owner_of(i);
        merge_ranks(reqs, b0, b1, out);
    }
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

// Multi-GPU: ranks search disjoint option-prefix shards of every search of a launch and
// exchange one RankRecord per search (one all-gather per launch through the caller's
// callback).  MIN takes the smallest incumbent and the smallest leaf any rank stored (lowest
// rank on ties) and restarts everywhere if any rank restarted; FIRST takes the hit
// that is earliest in reference DFS order.
static int host_path_cmp(const HitPath& a, const HitPath& b, int k) {
    for (int l = 0; l < k; ++l) {
        if (a.opt[l] != b.opt[l]) return a.opt[l] < b.opt[l] ? -1 : 1;
        for (int i = 0; i < a.nb[l]; ++i)
            if (a.x[l][i] != b.x[l][i]) return a.x[l][i] > b.x[l][i] ? -1 : 1;
    }
    return 0;
}

int merge_rank_records(const RankRecord* all, int world, int mode, int k, SearchResult& res) {
    int win = -1, minr = -1;
    double best = POS_INF;
    bool aborted = false, overflow = false;
    for (int r = 0; r < world; ++r) {
        const RankRecord& x = all[r];
        aborted |= x.aborted != 0;
        overflow |= x.overflow != 0;
        if (minr < 0 || x.inc < best) {
            best = x.inc;
            minr = r;
        }
        if (mode == MODE_MIN) {
            // shards share incumbents during the search, so every rank may end at the global
            // incumbent: the argmin leaf is the smallest leaf a rank stored itself
            if (x.has_hit && (win < 0 || x.leaf.value < all[win].leaf.value)) win = r;
        } else if (x.has_hit && (win < 0 || host_path_cmp(x.path, all[win].path, k) < 0)) {
            win = r;
        }
    }
    res.overflow = overflow;
    if (mode == MODE_MIN) {
        res.aborted = aborted;
        res.value = best;
        res.found = win >= 0;
        if (res.found) res.leaf = all[win].leaf;
        return win >= 0 ? win : minr;
    }
    res.found = win >= 0;
    if (win >= 0) res.leaf = all[win].leaf;
    return win;
}

void Engine::merge_ranks(const std::vector<BatchReq>& reqs, size_t b0, size_t b1,
                         std::vector<SearchResult>& out) {
    if (!ag_ && !nccl_comm_) throw std::runtime_error("multi-GPU search without an all-gather");
    const size_t n = b1 - b0;
    const char* pin = reinterpret_cast<const char*>(h_pin_);
    std::vector<RankRecord> mine(n), all(n * world_);
    std::vector<char> need_path(n, 0);
    for (size_t i = 0; i < n; ++i) need_path[i] = out[b0 + i].found;
    HitPath* hbest = reinterpret_cast<HitPath*>(h_best_);
    bool any = false;
    for (size_t i = 0; i < n; ++i) any |= need_path[i] != 0;
    if (any) {
        CK(cudaMemcpyAsync(hbest, d_best_, n * sizeof(HitPath), cudaMemcpyDeviceToHost,
                           S_(stream_)));
        CK(cudaStreamSynchronize(S_(stream_)));
    }
    for (size_t i = 0; i < n; ++i) {
        const Ctl* hc = reinterpret_cast<const Ctl*>(pin + i * BLOB_STRIDE + BLOB_CTL);
        const SearchResult& res = out[b0 + i];
        RankRecord& m = mine[i];
        std::memset(&m, 0, sizeof m);
        m.has_hit = res.found ? 1 : 0;
        m.aborted = res.aborted ? 1 : 0;
        m.overflow = res.overflow ? 1 : 0;
        union {
            unsigned long long u;
            double d;
        } w;
        w.u = hc->inc;
        m.inc = w.d;
        m.nodes = hc->nodes;
        m.leaves = hc->leaves;
        if (res.found) {
            m.path = hbest[i];
            m.leaf = res.leaf;
        }
    }
    // all-gather of n records per rank: rank r's records land at all[r * n .. r * n + n)
    if (nccl_comm_)
        nccl_allgather(mine.data(), all.data(), n * sizeof(RankRecord));
    else if (ag_(ag_user_, mine.data(), all.data(), n * sizeof(RankRecord)) != 0)
        throw std::runtime_error("all-gather failed");
    std::vector<RankRecord> per(world_);
    for (size_t i = 0; i < n; ++i) {
        if (owned_[i] >= 0) {
            // a whole search run by its owner rank: its record is the answer
            const RankRecord& x = all[(size_t)owned_[i] * n + i];
            SearchResult& res = out[b0 + i];
            res.overflow = x.overflow != 0;
            res.aborted = x.aborted != 0;
            res.found = x.has_hit != 0;
            if (res.found) res.leaf = x.leaf;
            if (reqs[b0 + i].S.mode == MODE_MIN) res.value = x.inc;
            continue;
        }
        for (int r = 0; r < world_; ++r) per[r] = all[(size_t)r * n + i];
        merge_rank_records(per.data(), world_, reqs[b0 + i].S.mode, reqs[b0 + i].S.k, out[b0 + i]);
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
