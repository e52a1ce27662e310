// engine.hpp — device search engine (sm_100a) used by the host planner.
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "spec_build.hpp"

namespace mg {

typedef int (*AllGatherFn)(void* user, const void* send, void* recv, size_t bytes);

struct SearchStats {
    long long nodes = 0, leaves = 0, rounds = 0, searches = 0;
};

struct SearchResult {
    bool found = false;  // FIRST: a leaf with value <= theta exists; MIN: argmin leaf kept
    Leaf leaf{};         // FIRST: the first such leaf; MIN: an allocation reaching `value`
    double value = POS_INF;  // MIN: best value found (< ub), else ub
    bool aborted = false;    // MIN: incumbent fell below abort_below
    bool overflow = false;   // a level needed more than MAXB blocks
};

// One search of a batched launch (Engine::search_batch).
struct BatchReq {
    Spec S;
    double ub = POS_INF;           // MIN: incumbent upper bound
    double abort_below = 0.0;      // MIN: restart when the incumbent drops below
    const HitPath* seed_path = nullptr;  // FIRST: a leaf known to satisfy theta ...
    const Leaf* seed_leaf = nullptr;     // ... as a path in this search's order
    SearchStats* st = nullptr;     // counters of the caller
    bool force_solo = false;       // one walker in DFS order whatever the tree size
    int sim_rank = -1, sim_world = 0;  // share_all simulation: shard sim_rank of sim_world
};

// What a rank contributes to the merge of one sharded search (one all-gather per launch:
// sizeof(RankRecord) ~ 4.2 KB per search — HitPath 3,120 B + Leaf 1,064 B + flags).
struct RankRecord {
    int has_hit, aborted, overflow, pad;
    double inc;
    unsigned long long nodes, leaves;
    HitPath path;
    Leaf leaf;
};
// The merge rule the engine applies to every sharded search (exported through the C ABI
// for the multi-process CPU tests).  Returns the winning rank (-1: no FIRST hit).
int merge_rank_records(const RankRecord* all, int world, int mode, int k, SearchResult& res);
size_t nccl_id_bytes();
// calib.cu: measured shared-memory load bandwidth (GB/s), the SURVEY §8(d) roofline denominator
double smem_peak_gbs(int device, int reps);
void nccl_unique_id(void* out);  // ncclGetUniqueId through the run-time loaded NCCL

struct EvalEntry {  // device evaluator input (one per allocation entry)
    int row;        // option row (base, B) of this entry
    int module;
    int n_gpus;
    int pad;
    long long gpu_off;
};

// mosaic_gpu_eval_entry (include/mosaic_gpu.h), the evaluator's input record as the caller
// lays it out: no host-side repacking between the ABI and the kernel.
struct EvalABI {
    int module, d, units, n_gpus, levels, reserved;
    long long gpu_off;
};
static_assert(sizeof(EvalABI) == 32, "mosaic_gpu_eval_entry layout");

// Error bits of the batched evaluator (k_evaluate).
enum {
    EVAL_ERR_MODULE = 1,   // module index outside the graph
    EVAL_ERR_SURFACE = 2,  // (d, units) outside the module's profiled surface
    EVAL_ERR_GPU = 4,      // GPU id outside 0..G-1 or GPU list outside the gpus array
    EVAL_ERR_LEVELS = 8,   // entry quota_levels differs from the context's
    EVAL_ERR_ENTRIES = 16, // allocation with more than 64 entries or outside entries[]
};

// Search-engine knobs.  Defaults are the measured best; nothing reads the
// environment — experiments set them through mosaic_gpu_set_tuning().
struct Tuning {
    int don_depth = 3;      // donate levels <= k-1-don_depth (measured best on cfg5)
    int don_tail = 2;       // long-running pieces: levels <= k-1-don_tail
    int don_depth_small = 2;  // stages of 3..5 modules: donate levels <= k-1-don_depth_small
    int don_depth_first = -1; // FIRST searches of >= 6 modules: own depth (-1: don_depth)
    int don_tail_first = -1;  // FIRST searches: own don_tail (-1: don_tail)
    int don_period = 4;     // power of two; control reads every 4 steps (tools/knob_solve.sh)
    int don_period_small = 1;  // the same for stages below restart_k modules (bench sample sweep)
    int backoff_cap = 2048; // ns, idle walkers polling back-off cap (measured)
    double small_tree = 2e5;  // option tuples x G below which one walker runs the search alone
    long long deep_after = 16384;  // steps on one piece before deeper hand-overs are allowed
    int tail_idle = 0;      // > 0: tail phase once the ramp-up is over and > 1/tail_idle walkers idle
    long long tail_after = 256;  // ... in which deeper hand-overs need only this many steps
    int don_min_rest = 0;   // deeper (tail) hand-overs need this many options left (0: any)
    int local_handover = 1; // 1: busy walkers hand pieces to idle siblings of their CTA (smem)
    int min_order = 4;      // MIN proof level order: 0 fewest viable options first, 1 most,
                            // 2 / 3 largest / smallest minimal base latency first, 4 largest
                            // minimal solo latency, 5 largest minimal footprint, 6 0 + 2 ties
    long long min_perm = 0; // measurement: > 0 = that permutation of the modules (1-based)
    // child look-ahead (can every remaining level still place an option?): off by default —
    // the lane-parallel option screen at the next level does the same job for less
    int lookahead = 0;
    int generic_kernel = 0; // never use the specialised kernels
    int shard_level = -1;   // override of the sharded option-prefix level (-1: default)
    int ring_per_walker = 16;  // cursor-ring slots per resident walker
    int trace = 0;          // one stderr line per device search
    int spec_k = 4;         // GAHC: batch-evaluate a round's candidates of up to spec_k modules
    int fuse_k = 1;         // stage_evals of <= fuse_k modules run their MIN proof with the first probe
    double fuse_tree = 2e5; // ... and so do stages with option tuples x G <= fuse_tree
    int restart_k = 5;      // MIN proofs of stages with >= restart_k modules restart on a big drop
    // measurement only (tools/): search rank share_rank's share of a share_world-way
    // sharded search on this one device, without merging — NOT the stage's answer
    int share_rank = 0, share_world = 1;
    // share_all > 1 (one device): every large search runs as share_all option-prefix shards
    // in ONE launch and is merged like a multi-GPU search (shard balance and the effect of
    // share_peers measured on one GPU)
    int share_all = 0;
    // sharded MIN proofs lower each other's incumbents during the search (peer Ctl words:
    // CUDA IPC-mapped on the other GPUs, or the sibling shards of a share_all launch)
    int share_peers = 1;
};

class Engine {
  public:
    explicit Engine(int device);
    int device() const { return device_; }
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    void upload_rows(const Model& M);
    // seed (FIRST only): a leaf known to satisfy theta, as a path in this search's order
    SearchResult search(const Spec& S, double ub, double abort_below, SearchStats& st,
                        const HitPath* seed_path = nullptr, const Leaf* seed_leaf = nullptr);
    // Independent searches in as few launches as possible (one per MAXBATCH / resident grid):
    // each gets its own CTA range, control block and ring slice (search_kernel.cuh).
    std::vector<SearchResult> search_batch(std::vector<BatchReq>& reqs);
    // Batched stage_time (K1): per allocation, entries [off[i], off[i+1]).
    void evaluate(const std::vector<EvalEntry>& ent, const std::vector<int>& gpus,
                  const std::vector<long long>& off, const std::vector<double>& base,
                  const std::vector<double>& Bt, int G, const Model& M,
                  std::vector<double>& st_out, std::vector<double>& rect_out);
    double eval_ms() const { return eval_ms_; }
    // K1 on the ABI layout: dense per-(module, d, units) rate tables uploaded once
    // (base[m][d-1][u], B[m][u]; eval.cu), then any number of batched calls.  `dev` says the
    // five arrays are device pointers on this engine's device; otherwise they are host
    // memory and are staged through persistent device buffers.  Returns EVAL_ERR_* bits.
    void set_rate_tables(const std::vector<double>& base, const std::vector<double>& B, int n_mod,
                         int G, int L, const Model& M);
    bool has_rate_tables() const { return d_tab_base_ != nullptr; }
    int evaluate_abi(const EvalABI* ent, long long n_ent, const int* gpus, long long n_gpu_ids,
                     const long long* off, long long n, double* st, double* rect, bool dev);
    double evaluate_kernel_ms() const { return evk_ms_; }
    long long evaluate_kernel_launches() const { return evk_n_; }
    long long evaluate_alg_bytes() const { return evk_bytes_; }
    double evaluate_fast_ms() const { return evf_ms_; }
    long long evaluate_fallback_allocs() const { return ev_fallback_; }

    // fn == nullptr with world > 1: measure this rank's share only (no merge; the result
    // is NOT the stage's answer — used to simulate shard balance on one device)
    void set_shard(int rank, int world, AllGatherFn fn, void* user) {
        free_nccl();
        unlink_peers();
        rank_ = rank;
        world_ = world;
        ag_ = fn;
        ag_user_ = user;
    }
    // the in-library data plane: a NCCL communicator from a unique id (nccl_plane.cu)
    void set_shard_nccl(int rank, int world, const void* nccl_id);
    Tuning& tuning() { return tune_; }
    int peer_links() const {
        int n = 0;
        for (void* p : peer_blob_) n += p != nullptr;
        return n;
    }
    // bytes of device memory the engine holds (option table, ring, control blocks)
    long long device_bytes() const { return dev_bytes_; }
    long long launches() const { return launches_; }
    double search_ms() const { return search_ms_; }
    void reset_counters() {
        launches_ = 0;
        own_launches_ = 0;
        search_ms_ = 0;
        eval_ms_ = 0;
        ksearch_ms_ = 0;
        ksearch_n_ = 0;
        h2d_ = 0;
        d2h_ = 0;
        alg_bytes_ = 0;
        evk_ms_ = 0;
        evf_ms_ = 0;
        ev_fallback_ = 0;
        evk_n_ = 0;
        evk_bytes_ = 0;
    }
    long long own_launches() const { return own_launches_; }
    double ksearch_ms() const { return ksearch_ms_; }
    long long ksearch_launches() const { return ksearch_n_; }
    long long h2d_bytes() const { return h2d_; }
    long long d2h_bytes() const { return d2h_; }
    long long alg_bytes() const { return alg_bytes_; }
    // device-side timing marks on the engine stream (bench.py)
    void mark(int which);
    double marked_ms();

  private:
    void ensure_front(long long n);
    void kernel_for(const std::vector<BatchReq>& reqs, size_t b0, size_t b1, const void** kfn,
                    size_t* smem, long long* grid);
    void launch_chunk(std::vector<BatchReq>& reqs, size_t b0, size_t b1, const void* kfn,
                      size_t smem, long long grid_cap, std::vector<SearchResult>& out);
    void merge_ranks(const std::vector<BatchReq>& reqs, size_t b0, size_t b1,
                     std::vector<SearchResult>& out);
    void nccl_allgather(const void* send, void* recv, size_t bytes);
    bool sharded() const { return (world_ > 1 && ag_) || nccl_comm_; }
    // owner rank of the i-th search of a launch (every rank builds the same launches)
    int owner_of(int i) const { return world_ > 1 ? i % world_ : 0; }
    std::vector<int> owned_;  // per search of the current launch: owner rank, -1 = sharded
    void free_nccl();
    // peer GPUs' blob bases (CUDA IPC), exchanged once through the all-gather plane
    void link_peers();
    void unlink_peers();
    std::vector<void*> peer_blob_, peer_best_;
    bool peers_tried_ = false;
    std::vector<SearchResult> search_batch_sim(std::vector<BatchReq>& reqs);
    std::vector<SearchResult> search_batch_sim_chunk(std::vector<BatchReq>& reqs, int W);
    bool is_small(const BatchReq& q) const;
    void* nccl_comm_ = nullptr;
    void* d_rec_ = nullptr;
    void* d_tl_ = nullptr;  // trace >= 3: busy-walker timeline of the last launch
    size_t rec_cap_ = 0;
    int device_;
    int rank_ = 0, world_ = 1;
    AllGatherFn ag_ = nullptr;
    void* ag_user_ = nullptr;
    void* stream_ = nullptr;
    void* ev0_ = nullptr;
    void* ev1_ = nullptr;
    // device buffers
    double *d_base_ = nullptr, *d_B_ = nullptr, *d_fp_ = nullptr, *d_bound_ = nullptr;
    void *d_rows_ = nullptr, *h_rows_ = nullptr;  // pooled: the SoA arrays live in d_rows_
    size_t rows_cap_ = 0;
    int *d_d_ = nullptr, *d_u_ = nullptr;
    int n_rows_ = 0;
    void* d_blob_ = nullptr;  // MAXBATCH x (Spec | Ctl | Leaf | root Cont), BLOB_STRIDE apart
    void* d_front_[1] = {nullptr};
    int* d_ready_ = nullptr;
    void* d_best_ = nullptr;  // MAXBATCH HitPaths
    void* h_best_ = nullptr;  // pinned mirror (seeds in, rank merge out)
    std::map<long long, long long> grid_cache_;  // (kernel, smem) -> resident CTAs
    Tuning tune_;
    unsigned long long ticket_base_ = 0;
    long long dev_bytes_ = 0;
    long long front_cap_ = 0;
    void* h_pin_ = nullptr;
    long long launches_ = 0;
    double search_ms_ = 0;
    double eval_ms_ = 0;
    long long own_launches_ = 0;
    double ksearch_ms_ = 0;
    long long ksearch_n_ = 0;
    long long h2d_ = 0, d2h_ = 0, alg_bytes_ = 0;
    void* evk0_ = nullptr;
    void* evk1_ = nullptr;
    void* evm0_ = nullptr;
    void* evm1_ = nullptr;
    // K1 rate tables and staging (eval.cu)
    double* d_tab_base_ = nullptr;
    double* d_tab_B_ = nullptr;
    int tab_nmod_ = 0, tab_G_ = 0, tab_L_ = 0;
    double tab_e1_ = 0, tab_e2_ = 0, tab_e3_ = 0;
    int tab_add_ = 0, tab_self_ = 1;
    void* ev_buf_[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    size_t ev_cap_[5] = {0, 0, 0, 0, 0};
    int* d_everr_ = nullptr;
    int* h_everr_ = nullptr;
    int ev_grid_ = 0;
    size_t ev_smem_ = 0;
    // fast path (k_evaluate_fast) + the worklist of allocations it leaves to k_evaluate
    void* ev_list_ = nullptr;
    size_t ev_list_cap_ = 0;
    int evf_grid_ = 0;
    size_t evf_smem_ = 0;
    double evf_ms_ = 0;
    long long ev_fallback_ = 0;
    void* evc_ = nullptr;
    double evk_ms_ = 0;
    long long evk_n_ = 0, evk_bytes_ = 0;
    void* eva_ = nullptr;
    void* evb_ = nullptr;
    void free_eval();
};

}  // namespace mg
