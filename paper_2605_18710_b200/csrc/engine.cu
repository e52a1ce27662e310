// engine.cu — sm_100a kernels of the planner hot path and their host driver.
//
//   k_expand  : one thread per frontier node; enumerates its children (next level's
//               option x canonical composition) with all pruning, count pass + write
//               pass (stable, so the frontier stays in reference DFS order).
//   k_search  : persistent threads pull frontier nodes from an atomic counter and run
//               the budgeted DFS of search_core.cuh to the leaves (MIN: shared
//               incumbent via atomicMin on the fp64 bits; FIRST: smallest frontier
//               index with a hit via atomicMin, later subtrees abort).
//   k_extract : re-walks the winning FIRST subtree and writes its leaf.
//   k_eval    : batched stage_time of explicit allocations (perf_model.hpp:442-479),
//               one warp per allocation, resident bitmaps in shared memory.
//
// Load balance: subtrees that exceed the per-item step budget are flagged, compacted
// (cub::DeviceSelect, stable) and expanded one level deeper for the next round, so
// heavy subtrees fan out over the whole GPU instead of pinning one thread.
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include <cub/cub.cuh>

#include "engine.hpp"
#include "search_core.cuh"

namespace mg {

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                     " at " #x);                                       \
    } while (0)

struct Ctl {
    unsigned long long inc;  // MIN incumbent, fp64 bits (values are >= 0)
    long long best_idx;      // FIRST: smallest frontier index with a hit
    unsigned long long next; // work counter
    int abort;
    int overflow;
    unsigned long long nodes, leaves;
    double abort_below;
};

struct DevHooks {
    Ctl* ctl;
    int mode;
    int expanding;
    int extract;
    int write;
    long long idx;
    long long budget;
    long long steps;
    int unfinished;
    double inc_cache;
    int refresh;
    Leaf* leaf_out;
    Node* out;
    long long out_base;
    long long emitted;
    unsigned long long nodes, leaves;

    __device__ bool abort() {
        if (expanding) return false;
        if (++steps > budget) {
            unfinished = 1;
            return true;
        }
        if (mode == MODE_FIRST) {
            if (!extract && *(volatile long long*)&ctl->best_idx < idx) return true;
        } else if (*(volatile int*)&ctl->abort) {
            return true;
        }
        return false;
    }
    __device__ double load_inc() {
        return __longlong_as_double(*(volatile long long*)&ctl->inc);
    }
    __device__ double thr(const Spec& S) {
        if (mode != MODE_MIN) return S.thp;
        if ((refresh++ & 15) == 0) {
            double I = load_inc();
            inc_cache = I < inc_cache ? I : inc_cache;
        }
        double t = inc_cache >= POS_INF ? POS_INF : inc_cache * (1.0 - TIE_EPS);
        return t < S.thp ? t : S.thp;
    }
    __device__ double incumbent() {
        double I = load_inc();
        inc_cache = I < inc_cache ? I : inc_cache;
        return inc_cache;
    }
    __device__ void improve(double v) {
        atomicMin(&ctl->inc, (unsigned long long)__double_as_longlong(v));
        if (v < inc_cache) inc_cache = v;
        if (v < ctl->abort_below) atomicExch(&ctl->abort, 1);
    }
    __device__ void hit(const Walk& w, int j, double v) {
        if (extract)
            store_leaf(w, j, v, *leaf_out);
        else
            atomicMin(&ctl->best_idx, idx);
    }
    __device__ void count_node() { ++nodes; }
    __device__ void count_leaf() { ++leaves; }
    __device__ void emit(const Walk& w, int dep) {
        if (write) store_node(w, dep, out[out_base + emitted]);
        ++emitted;
    }
    __device__ void overflow() { atomicExch(&ctl->overflow, 1); }
};

__device__ __forceinline__ void load_spec(const Spec* g, Spec* s) {
    const int n = sizeof(Spec) / 4;
    const int* src = reinterpret_cast<const int*>(g);
    int* dst = reinterpret_cast<int*>(s);
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    __syncthreads();
}

__device__ __forceinline__ void load_walk(const Spec& S, const Rows& R, const Node& nd, Walk& w) {
    load_node(nd, w);
    int used = 0;
    for (int l = 0; l < nd.depth; ++l) {
        int r = S.lvl_off[l] + nd.opt[l];
        used += R.d[r] * R.u[r];
    }
    w.used[nd.depth] = used;
}

__device__ __forceinline__ DevHooks make_hooks(Ctl* ctl, int mode) {
    DevHooks h;
    h.ctl = ctl;
    h.mode = mode;
    h.expanding = 0;
    h.extract = 0;
    h.write = 0;
    h.idx = 0;
    h.budget = LLONG_MAX;
    h.steps = 0;
    h.unfinished = 0;
    h.inc_cache = POS_INF;
    h.refresh = 0;
    h.leaf_out = nullptr;
    h.out = nullptr;
    h.out_base = 0;
    h.emitted = 0;
    h.nodes = 0;
    h.leaves = 0;
    return h;
}

__global__ void __launch_bounds__(128) k_expand(const Spec* Sg, Rows R, const Node* in,
                                                const long long* in_key, long long n, Ctl* ctl,
                                                long long* cnt, const long long* off, Node* out,
                                                long long* out_key, int write) {
    __shared__ Spec S;
    load_spec(Sg, &S);
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Node& nd = in[i];
    if (nd.depth >= S.k - 1) {  // cannot be split further: carried over as is
        if (write) {
            out[off[i]] = nd;
            out_key[off[i]] = in_key[i];
        } else {
            cnt[i] = 1;
        }
        return;
    }
    Walk w;
    load_walk(S, R, nd, w);
    DevHooks h = make_hooks(ctl, S.mode);
    h.expanding = 1;
    h.write = write;
    h.out = out;
    h.out_base = write ? off[i] : 0;
    h.inc_cache = h.load_inc();
    dfs(S, R, w, nd.depth, nd.depth + 1, h);
    if (write) {
        for (long long e = 0; e < h.emitted; ++e) out_key[off[i] + e] = in_key[i];
    } else {
        cnt[i] = h.emitted;
        atomicAdd(&ctl->nodes, h.nodes);
    }
}

__global__ void __launch_bounds__(128) k_search(const Spec* Sg, Rows R, const Node* in,
                                                long long n, Ctl* ctl, long long budget,
                                                unsigned char* unfin) {
    __shared__ Spec S;
    load_spec(Sg, &S);
    Walk w;
    unsigned long long nodes = 0, leaves = 0;
    while (true) {
        long long i = (long long)atomicAdd(&ctl->next, 1ULL);
        if (i >= n) break;
        if (S.mode == MODE_FIRST && i > *(volatile long long*)&ctl->best_idx) break;
        if (S.mode == MODE_MIN && *(volatile int*)&ctl->abort) break;
        const Node& nd = in[i];
        load_walk(S, R, nd, w);
        DevHooks h = make_hooks(ctl, S.mode);
        h.idx = i;
        h.budget = nd.depth >= S.k - 1 ? LLONG_MAX : budget;
        h.inc_cache = h.load_inc();
        dfs(S, R, w, nd.depth, S.k, h);
        unfin[i] = (unsigned char)h.unfinished;
        nodes += h.nodes;
        leaves += h.leaves;
    }
    atomicAdd(&ctl->nodes, nodes);
    atomicAdd(&ctl->leaves, leaves);
}

__global__ void k_extract(const Spec* Sg, Rows R, const Node* in, long long idx, Ctl* ctl,
                          Leaf* out) {
    __shared__ Spec S;
    load_spec(Sg, &S);
    if (threadIdx.x != 0) return;
    Walk w;
    const Node& nd = in[idx];
    load_walk(S, R, nd, w);
    DevHooks h = make_hooks(ctl, MODE_FIRST);
    h.extract = 1;
    h.idx = idx;
    h.leaf_out = out;
    out->nb = -1;
    dfs(S, R, w, nd.depth, S.k, h);
}

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
        const EvalEntry& E = ent[e0 + e];
        double worst = NEG_INF;
        for (int g = lane; g < E.n_gpus; g += 32) {
            unsigned long long m = mk[gpus[E.gpu_off + g]];
            double s = 0.0, p = 1.0;
            int res = 0;
            for (int f = 0; f < ne; ++f) {
                if (!(m >> f & 1ULL)) continue;
                if (f == e && !P.include_self) continue;
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
    CK(cudaMalloc(&d_spec_, sizeof(Spec)));
    CK(cudaMalloc(&d_ctl_, sizeof(Ctl)));
    CK(cudaMalloc(&d_leaf_, sizeof(Leaf)));
    CK(cudaMalloc(&d_nsel_, sizeof(long long)));
    CK(cudaMallocHost(&h_pin_, sizeof(Spec) + sizeof(Ctl) + sizeof(Leaf) + 64 + sizeof(Node)));
}

Engine::~Engine() {
    cudaSetDevice(device_);
    cudaFree(d_base_);
    cudaFree(d_B_);
    cudaFree(d_fp_);
    cudaFree(d_bound_);
    cudaFree(d_d_);
    cudaFree(d_u_);
    cudaFree(d_spec_);
    cudaFree(d_ctl_);
    cudaFree(d_leaf_);
    for (int i = 0; i < 3; ++i) {
        cudaFree(d_front_[i]);
        cudaFree(d_key_[i]);
    }
    cudaFree(d_cnt_);
    cudaFree(d_off_);
    cudaFree(d_flag_);
    cudaFree(d_nsel_);
    cudaFree(d_tmp_);
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
    if (!base.empty()) {
        CK(cudaMemcpy(d_base_, base.data(), base.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_B_, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_fp_, fp.data(), fp.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_bound_, bound.data(), bound.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_d_, d.data(), d.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_u_, u.data(), u.size() * 4, cudaMemcpyHostToDevice));
    }
}

void Engine::ensure_front(long long n) {
    if (n <= front_cap_) return;
    long long cap = std::max<long long>(n, 1024);
    for (int i = 0; i < 3; ++i) {
        cudaFree(d_front_[i]);
        cudaFree(d_key_[i]);
        CK(cudaMalloc(&d_front_[i], cap * sizeof(Node)));
        CK(cudaMalloc(&d_key_[i], cap * sizeof(long long)));
    }
    cudaFree(d_cnt_);
    cudaFree(d_off_);
    cudaFree(d_flag_);
    CK(cudaMalloc(&d_cnt_, (cap + 1) * sizeof(long long)));
    CK(cudaMalloc(&d_off_, (cap + 1) * sizeof(long long)));
    CK(cudaMalloc(&d_flag_, cap));
    size_t b1 = 0, b2 = 0, b3 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b1, d_cnt_, d_off_, (int)cap + 1);
    cub::DeviceSelect::Flagged(nullptr, b2, (Node*)d_front_[0], d_flag_, (Node*)d_front_[1],
                               d_nsel_, (int)cap);
    cub::DeviceSelect::Flagged(nullptr, b3, d_key_[0], d_flag_, d_key_[1], d_nsel_, (int)cap);
    size_t need = std::max(b1, std::max(b2, b3));
    if (need > tmp_bytes_) {
        cudaFree(d_tmp_);
        CK(cudaMalloc(&d_tmp_, need));
        tmp_bytes_ = need;
    }
    front_cap_ = cap;
}

SearchResult Engine::search(const Spec& S, double ub, double abort_below, SearchStats& st) {
    CK(cudaSetDevice(device_));
    cudaStream_t s = S_(stream_);
    SearchResult res;
    res.value = ub;
    const long long cap = cap_front;
    ensure_front(cap);
    Rows R{d_base_, d_B_, d_fp_, d_bound_, d_d_, d_u_};
    char* pin = reinterpret_cast<char*>(h_pin_);
    Spec* hs = reinterpret_cast<Spec*>(pin);
    Ctl* hc = reinterpret_cast<Ctl*>(pin + sizeof(Spec));
    Leaf* hl = reinterpret_cast<Leaf*>(pin + sizeof(Spec) + sizeof(Ctl));
    long long* hx = reinterpret_cast<long long*>(pin + sizeof(Spec) + sizeof(Ctl) + sizeof(Leaf));
    *hs = S;
    CK(cudaMemcpyAsync(d_spec_, hs, sizeof(Spec), cudaMemcpyHostToDevice, s));
    h2d_ += sizeof(Spec) + sizeof(Ctl) + sizeof(Node) + sizeof(long long);
    std::memset(hc, 0, sizeof(Ctl));
    union {
        double d;
        unsigned long long u;
    } cv;
    cv.d = ub;
    hc->inc = cv.u;
    hc->best_idx = LLONG_MAX;
    hc->abort_below = abort_below;
    CK(cudaMemcpyAsync(d_ctl_, hc, sizeof(Ctl), cudaMemcpyHostToDevice, s));
    Ctl* dc = reinterpret_cast<Ctl*>(d_ctl_);

    Node* P = reinterpret_cast<Node*>(d_front_[0]);
    Node* F = reinterpret_cast<Node*>(d_front_[1]);
    Node* Q = reinterpret_cast<Node*>(d_front_[2]);
    long long* PK = d_key_[0];
    long long* FK = d_key_[1];
    long long* QK = d_key_[2];
    {
        Node* hr = reinterpret_cast<Node*>(hx + 4);
        std::memset(hr, 0, sizeof(Node));
        hr->depth = 0;
        hr->nb = 1;
        hr->bsz[0] = (uint16_t)S.G;
        hx[0] = 0;
        CK(cudaMemcpyAsync(P, hr, sizeof(Node), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(PK, hx, sizeof(long long), cudaMemcpyHostToDevice, s));
    }
    CK(cudaEventRecord((cudaEvent_t)ev0_, s));
    long long nP = 1;
    bool searched_once = false;
    const int tb = 128;
    while (nP > 0) {
        ++st.rounds;
        // ---- expand a prefix of P by one level into F (count, scan, write) ----
        k_expand<<<(unsigned)((nP + tb - 1) / tb), tb, 0, s>>>((const Spec*)d_spec_, R, P, PK, nP,
                                                                dc, d_cnt_, d_off_, F, FK, 0);
        ++launches_;
        ++own_launches_;
        CK(cudaMemsetAsync(d_cnt_ + nP, 0, sizeof(long long), s));
        size_t tb2 = tmp_bytes_;
        CK(cub::DeviceScan::ExclusiveSum(d_tmp_, tb2, d_cnt_, d_off_, (int)(nP + 1), s));
        ++launches_;
        CK(cudaMemcpyAsync(hx + 1, d_off_ + nP, sizeof(long long), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        long long total = hx[1];
        long long take = nP;
        if (total > cap) {
            std::vector<long long> offs(nP + 1);
            CK(cudaMemcpy(offs.data(), d_off_, (nP + 1) * sizeof(long long),
                          cudaMemcpyDeviceToHost));
            take = 0;
            while (take < nP && offs[take + 1] <= cap) ++take;
            if (take == 0) throw std::runtime_error("frontier capacity exceeded by one node");
            total = offs[take];
        }
        if (total > 0) {
            k_expand<<<(unsigned)((take + tb - 1) / tb), tb, 0, s>>>(
                (const Spec*)d_spec_, R, P, PK, take, dc, d_cnt_, d_off_, F, FK, 1);
            ++launches_;
            ++own_launches_;
        }
        const long long nF = total;
        const long long rest = nP - take;
        if (nF == 0 && rest == 0) break;
        if (!searched_once && rest == 0 && nF > 0 && nF < min_front) {
            // pure expansion while the frontier is small (depths are uniform here)
            CK(cudaMemcpyAsync(hx + 4, F, sizeof(Node), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (reinterpret_cast<Node*>(hx + 4)->depth < S.k - 1) {
                std::swap(P, F);
                std::swap(PK, FK);
                nP = nF;
                continue;
            }
        }
        searched_once = true;
        long long upto = nF;
        bool drop_rest = false;
        if (nF > 0) {
            // ---- search F with a per-item step budget ----
            CK(cudaMemsetAsync(d_flag_, 0, nF, s));
            CK(cudaMemsetAsync(&dc->next, 0, sizeof(unsigned long long), s));
            long long blocks = std::min<long long>((nF + tb - 1) / tb, 148LL * 8);
            CK(cudaEventRecord((cudaEvent_t)evk0_, s));
            k_search<<<(unsigned)blocks, tb, 0, s>>>((const Spec*)d_spec_, R, F, nF, dc, budget,
                                                     d_flag_);
            CK(cudaEventRecord((cudaEvent_t)evk1_, s));
            ++launches_;
            ++own_launches_;
            CK(cudaMemcpyAsync(hc, d_ctl_, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
            d2h_ += sizeof(Ctl);
            CK(cudaStreamSynchronize(s));
            {
                float kms = 0;
                CK(cudaEventElapsedTime(&kms, (cudaEvent_t)evk0_, (cudaEvent_t)evk1_));
                ksearch_ms_ += kms;
                ++ksearch_n_;
            }
            CK(cudaGetLastError());
            if (hc->overflow) {
                res.overflow = true;
                break;
            }
            if (S.mode == MODE_MIN && hc->abort) {
                res.aborted = true;
                break;
            }
            if (S.mode == MODE_FIRST && hc->best_idx != LLONG_MAX) {
                const long long bi = hc->best_idx;
                k_extract<<<1, 32, 0, s>>>((const Spec*)d_spec_, R, F, bi, dc, (Leaf*)d_leaf_);
                ++launches_;
                ++own_launches_;
                d2h_ += sizeof(Leaf);
                CK(cudaMemcpyAsync(hl, d_leaf_, sizeof(Leaf), cudaMemcpyDeviceToHost, s));
                hx[2] = LLONG_MAX;
                CK(cudaMemcpyAsync(&dc->best_idx, hx + 2, sizeof(long long),
                                   cudaMemcpyHostToDevice, s));
                CK(cudaStreamSynchronize(s));
                if (hl->nb < 0) throw std::runtime_error("extract did not reproduce the hit");
                res.found = true;
                res.leaf = *hl;
                upto = bi;          // later items follow the hit in DFS order
                drop_rest = true;   // so does every untouched pending item
            }
        }
        // ---- next pending list: unfinished items (stable) then the untouched rest ----
        long long nsel = 0;
        if (upto > 0) {
            size_t tb3 = tmp_bytes_;
            CK(cub::DeviceSelect::Flagged(d_tmp_, tb3, F, d_flag_, Q, d_nsel_, (int)upto, s));
            tb3 = tmp_bytes_;
            CK(cub::DeviceSelect::Flagged(d_tmp_, tb3, FK, d_flag_, QK, d_nsel_, (int)upto, s));
            launches_ += 2;
            CK(cudaMemcpyAsync(hx + 3, d_nsel_, sizeof(long long), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            nsel = hx[3];
        }
        long long nrest = drop_rest ? 0 : rest;
        if (nsel + nrest > cap) throw std::runtime_error("pending list exceeds frontier capacity");
        if (nrest > 0) {
            CK(cudaMemcpyAsync(Q + nsel, P + take, nrest * sizeof(Node), cudaMemcpyDeviceToDevice,
                               s));
            CK(cudaMemcpyAsync(QK + nsel, PK + take, nrest * sizeof(long long),
                               cudaMemcpyDeviceToDevice, s));
        }
        std::swap(P, Q);
        std::swap(PK, QK);
        nP = nsel + nrest;
    }
    CK(cudaMemcpyAsync(hc, d_ctl_, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord((cudaEvent_t)ev1_, s));
    CK(cudaEventSynchronize((cudaEvent_t)ev1_));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, (cudaEvent_t)ev0_, (cudaEvent_t)ev1_));
    search_ms_ += ms;
    if (hc->overflow) res.overflow = true;
    if (S.mode == MODE_MIN) {
        union {
            unsigned long long u;
            double d;
        } w;
        w.u = hc->inc;
        res.value = w.d;
    }
    st.nodes += (long long)hc->nodes;
    st.leaves += (long long)hc->leaves;
    ++st.searches;
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
