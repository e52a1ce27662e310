/* mosaic_gpu.h — C ABI of the B200 (sm_100a) backend for the Mosaic planner hot path.
 *
 * The reference (/root/reference/proj, header-only C++20, namespace mosaic) has no
 * FFI; its replaceable seams are C++ calls.  Each entry point below replaces one of
 * them and keeps its argument meaning and error behaviour:
 *
 *   mosaic_gpu_evaluate      <- stage_time / rectified_latency over a batch of
 *                               allocations (K1, host or device arrays)  perf_model.hpp:442-479
 *   mosaic_gpu_stage_time    <- the same for entries at any quota granularity
 *   mosaic_gpu_options       <- candidate_options                   stage_eval.hpp:68-93
 *   mosaic_gpu_search        <- stage_eval / ExactStageSolver::solve over a batch of
 *                               module sets (a GAHC round's candidates), one
 *                               launch per wave of device searches       stage_eval.hpp:302-382
 *   mosaic_gpu_stage_eval    <- stage_eval (tau doubling, bisection,
 *                               confirmation probes; first leaf of the
 *                               last successful FeasibilitySearch::run) stage_eval.hpp:302-382
 *   mosaic_gpu_feasible      <- detail::FeasibilitySearch::run(tau)  stage_eval.hpp:113-164
 *   mosaic_gpu_exact_stage   <- detail::ExactStageSolver::solve      oracle.hpp:86-103
 *   mosaic_gpu_solve         <- solve (GAHC)                         solver.hpp:157-289
 *   mosaic_gpu_brute_force   <- brute_force_optimum                  oracle.hpp:206-255
 *
 * Status codes map the reference's nullopt / exceptions:
 *   0 OK, 1 INFEASIBLE (std::nullopt), 2 MODULE_NO_OPTION (StageInfeasibleError),
 *   3 RANGE (SurfaceRangeError / invalid_argument), 4 TOO_LARGE (OracleTooLargeError
 *   or a stage beyond the kernel limits), 5 CUDA (device error), 6 EMPTY (EmptyPlanError).
 * No exception crosses the ABI; mosaic_gpu_last_error() returns a thread-local message.
 * Plain pointers and sizes only; outputs are caller-allocated.  One context per host
 * thread (like the reference, which is re-entrant but not thread-safe per EvalCache).
 */
#ifndef MOSAIC_GPU_H
#define MOSAIC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    MOSAIC_OK = 0,
    MOSAIC_INFEASIBLE = 1,
    MOSAIC_MODULE_NO_OPTION = 2,
    MOSAIC_RANGE = 3,
    MOSAIC_TOO_LARGE = 4,
    MOSAIC_CUDA = 5,
    MOSAIC_EMPTY = 6,
    MOSAIC_BASELINE_INFEASIBLE = 7, /* InfeasibleBaselineError (simulator.hpp:127-129) */
    MOSAIC_INVALID_ARGUMENT = 8,    /* std::invalid_argument (e.g. SimConfig checks) */
};

/* Kernel limits (a stage beyond them returns MOSAIC_TOO_LARGE, never a CPU path). */
#define MOSAIC_GPU_MAX_STAGE_MODULES 12
#define MOSAIC_GPU_MAX_GPUS 1024
#define MOSAIC_GPU_MAX_MODULES 64

/* One profiled surface point (perf_model.hpp:37-44). */
typedef struct {
    int32_t d;
    double a, latency, bandwidth_util, memory, sm_active;
} mosaic_gpu_point;

/* One module: id (topological tie-break, core.hpp:219), memory_base (core.hpp:34) and
 * its complete (d, a) surface grid in any order (perf_model.hpp:57-79). */
typedef struct {
    const char* id;
    double memory_base;
    const mosaic_gpu_point* points;
    int32_t n_points;
} mosaic_gpu_module;

/* Everything a PerfContext + ClusterSpec + SolveConfig carry for the hot path. */
typedef struct {
    const mosaic_gpu_module* modules;
    int32_t n_modules;
    const int32_t* edges; /* 2*n_edges module indices (upstream, downstream) */
    int32_t n_edges;
    int32_t gpu_count;      /* ClusterSpec.gpu_count */
    double memory_capacity; /* ClusterSpec.memory_capacity (bytes) */
    double e1, e2, e3;      /* InterferenceModel */
    int32_t additive_only;
    int32_t include_self;   /* PerfContext.include_self */
    int32_t quota_levels;   /* SolveConfig.quota_levels = 1/granularity */
    double bisect_rel_tol;  /* SolveConfig.bisect_rel_tol */
    int32_t enable_prune, enable_cache;
} mosaic_gpu_problem;

typedef struct mosaic_gpu_ctx mosaic_gpu_ctx;

/* One stage entry (StageAllocation::Entry, core.hpp:80-84). gpus[] is sorted. */
typedef struct {
    int32_t module, dp_degree, quota_units;
    int32_t n_gpus;
    int32_t gpus[MOSAIC_GPU_MAX_GPUS];
} mosaic_gpu_entry;

/* StageEvalResult (stage_eval.hpp:50-54) + search counters. */
typedef struct {
    int32_t status;    /* MOSAIC_OK / MOSAIC_INFEASIBLE / MOSAIC_MODULE_NO_OPTION */
    double stage_time;
    int32_t n_entries; /* entries sorted by module index */
    mosaic_gpu_entry entries[MOSAIC_GPU_MAX_STAGE_MODULES];
    int64_t probes;      /* feasibility probes replayed (reference feasibility_calls) */
    int64_t gpu_searches; /* device searches launched */
    int64_t nodes;       /* partial allocations expanded on the device */
    int64_t leaves;      /* complete allocations scored on the device */
} mosaic_gpu_stage_result;

/* Context: validates the graph, builds surfaces, packs candidate-option tables
 * into the device layout on `device` (cudaSetDevice index). */
int mosaic_gpu_create(const mosaic_gpu_problem* p, int device, mosaic_gpu_ctx** out);
void mosaic_gpu_destroy(mosaic_gpu_ctx* ctx);
const char* mosaic_gpu_last_error(void);

/* Number of modules / candidate options of module m (candidate_options order):
 * rows are (d, units, base_latency, solo_bandwidth, footprint). */
int mosaic_gpu_num_options(mosaic_gpu_ctx* ctx, int module, int32_t* n_out);
int mosaic_gpu_options(mosaic_gpu_ctx* ctx, int module, int32_t* d, int32_t* units,
                       double* base_latency, double* solo_bandwidth, double* footprint);

/* Surface lookup (perf_model.hpp:124-147) for one module at (d, a). */
int mosaic_gpu_lookup(mosaic_gpu_ctx* ctx, int module, int d, double a, double out4[4]);

/* Compact entry (StageAllocation::Entry, core.hpp:80-84): its GPU list is
 * gpus[gpu_off .. gpu_off+n_gpus).  quota = quota_units / quota_levels as in
 * DeploymentOption::quota() (core.hpp:64-75); quota_levels = 0 means the context's. */
typedef struct {
    int32_t module, dp_degree, quota_units, n_gpus;
    int32_t quota_levels, reserved;
    int64_t gpu_off;
} mosaic_gpu_eval_entry;

/* Batched evaluator on the device: stage_time of n explicit allocations.
 * Allocation i owns entries [alloc_off[i], alloc_off[i+1]) of `entries`
 * (sorted by module index, as StageAllocation requires).  Rectified latencies per
 * entry are optionally written to rect_out (same indexing as entries; may be NULL).
 * Returns MOSAIC_RANGE if an entry's (d, units) is outside the module's surface. */
int mosaic_gpu_stage_time(mosaic_gpu_ctx* ctx, const mosaic_gpu_eval_entry* entries,
                          const int32_t* gpus, const int64_t* alloc_off, int64_t n_allocs,
                          double* stage_time_out, double* rect_out);

/* Batched plan scoring (K1): stage_time of n_allocs allocations laid out exactly as for
 * mosaic_gpu_stage_time, with the array sizes passed explicitly (entries[0..n_entries),
 * gpus[0..n_gpu_ids)).  Entry quota_levels must be 0 or the context's.  With
 * MOSAIC_EVAL_DEVICE all five arrays are device pointers on the context's device: nothing
 * is copied, the caller must have finished writing them (synchronise its stream), and the
 * call returns once the outputs are written.  Otherwise they are host memory (pinned is
 * fastest) staged through buffers the context keeps.  Errors (MOSAIC_RANGE /
 * MOSAIC_TOO_LARGE) are reported for the whole batch, like the reference's exceptions. */
#define MOSAIC_EVAL_DEVICE 1u
int mosaic_gpu_evaluate(mosaic_gpu_ctx* ctx, const mosaic_gpu_eval_entry* entries,
                        int64_t n_entries, const int32_t* gpus, int64_t n_gpu_ids,
                        const int64_t* alloc_off, int64_t n_allocs, double* stage_time_out,
                        double* rect_out, uint32_t flags);
/* K1 counters since the last reset: kernel time (CUDA events on the context stream),
 * launches, and algorithmic bytes (offsets + entries + GPU ids read, outputs written). */
int mosaic_gpu_evaluate_stats(mosaic_gpu_ctx* ctx, double* kernel_ms, int64_t* launches,
                              int64_t* alg_bytes);

/* Peer ranks whose search control blocks this context has mapped (CUDA IPC over NVLink) for
 * in-search incumbent / earliest-hit sharing of sharded searches (0 before the first sharded
 * launch, or when mapping failed: sharing then happens only at the end-of-launch merge). */
int mosaic_gpu_peer_links(mosaic_gpu_ctx* ctx);

/* Calibration (SURVEY.md §8(d) roofline denominator): measured shared-memory load bandwidth
 * of `device` in GB/s (conflict-free 16-B loads on every SM, best of 5 timed launches). */
int mosaic_gpu_smem_peak(int device, double* gbs_out);

/* K1 path split since the last counter reset: time of the fast kernel (include_self, no
 * per-entry output, <= 32 entries, every module at most once) and how many allocations went
 * through the full-semantics kernel instead (worklist or non-fast calls). */
int mosaic_gpu_evaluate_paths(mosaic_gpu_ctx* ctx, double* fast_kernel_ms,
                              int64_t* full_path_allocs);

/* Batched stage search (the plan enumerator + best-plan reduction of one GAHC round):
 * out[i] = stage_eval (MOSAIC_SEARCH_STAGE_EVAL) or ExactStageSolver::solve
 * (MOSAIC_SEARCH_EXACT) of module set masks[i].  The n computations advance together;
 * every wave of their device searches (tau probes, MIN proofs) is ONE batched launch in
 * which each search owns a slice of the resident grid.  Each of out (full results),
 * stage_time_out and status_out (per-mask MOSAIC_OK / _INFEASIBLE / _MODULE_NO_OPTION) may be
 * NULL. */
#define MOSAIC_SEARCH_STAGE_EVAL 0
#define MOSAIC_SEARCH_EXACT 1
int mosaic_gpu_search(mosaic_gpu_ctx* ctx, const uint64_t* masks, int64_t n, int mode,
                      mosaic_gpu_stage_result* out, double* stage_time_out, int32_t* status_out);

/* stage_eval / ExactStageSolver::solve / FeasibilitySearch::run for one module set. */
int mosaic_gpu_stage_eval(mosaic_gpu_ctx* ctx, uint64_t mask, mosaic_gpu_stage_result* out);
int mosaic_gpu_exact_stage(mosaic_gpu_ctx* ctx, uint64_t mask, mosaic_gpu_stage_result* out);
int mosaic_gpu_feasible(mosaic_gpu_ctx* ctx, uint64_t mask, double tau,
                        mosaic_gpu_stage_result* out);

/* T* = minimum stage_time over every allocation of the module set that is below `ub`
 * (returns ub if none is): the quantity stage_eval's probes are decided against.  With
 * restart = 0 it is exactly one device search (used for profiling). */
int mosaic_gpu_stage_min(mosaic_gpu_ctx* ctx, uint64_t mask, double ub, int restart,
                         double* tstar, mosaic_gpu_stage_result* stats);

/* validate_plan (core.hpp:281-351) with the footprint oracle: stage s owns entries
 * [stage_off[s], stage_off[s+1]).  Writes the ValidationCode name ("Ok", "ModuleMissing",
 * "ModuleDuplicated", "DependencyViolated", "SmOvercommit", "MemoryOvercommit",
 * "EmptyStage") into code_out; the message is in mosaic_gpu_last_error(). */
int mosaic_gpu_validate_plan(mosaic_gpu_ctx* ctx, const mosaic_gpu_eval_entry* entries,
                             const int32_t* gpus, const int64_t* stage_off, int64_t n_stages,
                             char* code_out, size_t code_cap);

/* ---- N4: baselines and batched plan replay (simulator.hpp) ---- */
/* SimConfig (simulator.hpp:28-35); the seed is per replay (seeds[] below). */
typedef struct {
    int32_t iterations;
    int32_t stream_mode; /* 0 Pooled, 1 OnDemand */
    double pooled_overhead, on_demand_overhead, perturbation_sigma;
} mosaic_gpu_sim_config;

/* TimelineInterval (simulator.hpp:37-43). */
typedef struct {
    int32_t gpu, module;
    double start, end, quota;
} mosaic_gpu_interval;

/* simulate (simulator.hpp:68-119) of one plan (entries/gpus/stage_off as in
 * mosaic_gpu_validate_plan) for n_seeds seeds at once, one device thread per seed.
 * Outputs: iteration_time[n_seeds], per_stage[n_seeds * n_stages], busy[n_seeds * G],
 * mean_busy[n_seeds] (any may be NULL); the timeline (first iteration of seeds[0]) is
 * written to timeline[0 .. min(cap, *n_timeline)). */
int mosaic_gpu_simulate(mosaic_gpu_ctx* ctx, const mosaic_gpu_eval_entry* entries,
                        const int32_t* gpus, const int64_t* stage_off, int64_t n_stages,
                        const mosaic_gpu_sim_config* cfg, const uint64_t* seeds,
                        int64_t n_seeds, double* iteration_time, double* per_stage,
                        double* busy, double* mean_busy, mosaic_gpu_interval* timeline,
                        int64_t timeline_cap, int64_t* n_timeline);

/* Plan = ordered stages (DeploymentPlan, core.hpp:100-104). */
#define MOSAIC_GPU_MAX_STAGES 64
typedef struct {
    int32_t status;
    int32_t n_stages;
    uint64_t stage_mask[MOSAIC_GPU_MAX_STAGES];
    double stage_time[MOSAIC_GPU_MAX_STAGES];
    double iteration_time;   /* summed left to right (solver.hpp:281-285) */
    int64_t partitions_examined; /* brute force only */
    /* SolveTrace totals (solver.hpp:106-126) */
    int64_t rounds, stage_eval_calls, feasibility_calls, cache_hits, prunes;
    int64_t gpu_searches, nodes, leaves;
    double elapsed_s;
} mosaic_gpu_plan_result;

/* Stage allocations of a finished plan (read after solve / brute_force). */
int mosaic_gpu_plan_stage(mosaic_gpu_ctx* ctx, int stage, mosaic_gpu_stage_result* out);

int mosaic_gpu_solve(mosaic_gpu_ctx* ctx, mosaic_gpu_plan_result* out);
/* make_baseline_plan (simulator.hpp:283-313): policy 0 Megatron, 1 DistMM, full-quota
 * options at the context's quota_levels.  Read the stages with mosaic_gpu_plan_stage.
 * MOSAIC_BASELINE_INFEASIBLE mirrors InfeasibleBaselineError. */
int mosaic_gpu_baseline_plan(mosaic_gpu_ctx* ctx, int policy, mosaic_gpu_plan_result* out);
int mosaic_gpu_brute_force(mosaic_gpu_ctx* ctx, mosaic_gpu_plan_result* out);

/* GAHC round trace: round r, candidate c -> (mask_x, mask_y, pruned, cache_hit, gain). */
int mosaic_gpu_trace_rounds(mosaic_gpu_ctx* ctx, int64_t* n_rounds);
int mosaic_gpu_trace_round(mosaic_gpu_ctx* ctx, int64_t r, uint64_t* chosen_x,
                           uint64_t* chosen_y, double* applied_gain, int64_t* n_cands);
int mosaic_gpu_trace_cand(mosaic_gpu_ctx* ctx, int64_t r, int64_t c, uint64_t* mask_x,
                          uint64_t* mask_y, int32_t* pruned, int32_t* cache_hit, double* gain);

/* Drop the EvalCache (solver.hpp:39-75). */
void mosaic_gpu_clear_cache(mosaic_gpu_ctx* ctx);

/* EvalCache inspection after a solve (solver.hpp:39-75): the cached module sets in
 * insertion order (*n = their count; masks may be NULL to size), and one entry's
 * StageEvalResult plus the tau of every FeasibilitySearch::run it replayed, in call
 * order, with its outcome (1 feasible).  MOSAIC_RANGE if the mask is not cached. */
int mosaic_gpu_cache_masks(mosaic_gpu_ctx* ctx, uint64_t* masks, int64_t cap, int64_t* n);
int mosaic_gpu_cache_entry(mosaic_gpu_ctx* ctx, uint64_t mask, mosaic_gpu_stage_result* out,
                           double* probe_tau, int32_t* probe_ok, int64_t cap,
                           int64_t* n_probes);

/* Multi-GPU sharding of the search frontier (one rank per GPU).  The caller
 * supplies an all-gather of `bytes` from every rank (torch.distributed over NCCL
 * in bench.py); the library calls it once per batched launch with one RankRecord
 * (mosaic_gpu_rank_record_size() ~ 4.2 KB: flags, incumbent, FIRST hit path and leaf)
 * per search of the launch.  world == 1 disables it. */
typedef int (*mosaic_gpu_allgather_fn)(void* user, const void* send, void* recv, size_t bytes);
int mosaic_gpu_set_shard(mosaic_gpu_ctx* ctx, int rank, int world, mosaic_gpu_allgather_fn fn,
                         void* user);

/* The same sharding with the data plane INSIDE the library: rank 0 calls mosaic_gpu_nccl_id
 * (NCCL_UNIQUE_ID_BYTES = 128 bytes), the caller hands those bytes to every rank (any
 * out-of-band channel), every rank calls mosaic_gpu_set_shard_nccl; the library then builds a
 * NCCL communicator (libnccl.so.2, loaded at run time) and runs one ncclAllGather of the
 * launch's RankRecords per batched launch on the context's stream — no callback.  world = 1
 * is allowed (the merge path runs on one rank). */
int mosaic_gpu_nccl_id(void* id_out, size_t cap);
int mosaic_gpu_set_shard_nccl(mosaic_gpu_ctx* ctx, int rank, int world, const void* nccl_id);

/* The merge every sharded search goes through (Engine::merge_ranks), exported for the
 * multi-process CPU tests: world records of mosaic_gpu_rank_record_size() bytes, built with
 * mosaic_gpu_rank_record (x is k rows of 128 block counts).  mode 0 = MIN (smallest
 * incumbent, lowest rank on ties, restart if any rank restarted), 1 = FIRST (the hit earliest
 * in reference DFS order).  *winner = the rank whose leaf is taken (-1: none). */
size_t mosaic_gpu_rank_record_size(void);
int mosaic_gpu_rank_record(void* rec, int has_hit, int aborted, int overflow, double inc, int k,
                           const uint16_t* opt, const uint16_t* nb, const uint16_t* x,
                           double leaf_value);
int mosaic_gpu_merge_ranks(const void* records, int world, int mode, int k, int* winner,
                           int* found, double* value, int* aborted, int* overflow,
                           double* leaf_value);

/* Search-engine knobs for experiments (tools/tune.py); defaults are the measured best and
 * nothing reads the environment.  Keys: don_period_small (control-read period of stages below
 * restart_k modules), don_depth, don_depth_small (stages of 3..5 modules hand
 * over levels <= k-1-don_depth_small), don_depth_first / don_tail_first (FIRST searches' own
 * values, -1: the common ones), tail_idle (> 0: the deeper hand-overs also while more than
 * 1/tail_idle of the walkers are idle), don_tail (levels <= k-1-don_tail may be handed
 * over by long-running pieces), don_period (power of two), backoff_ns, small_tree, deep_after,
 * lookahead, generic_kernel, shard_level, ring_per_walker, trace (1: one line per device search,
 * 2: per launch, 3: as 1 plus walker occupancy, a busy-walker timeline, hand-over outcomes and
 * a log of long pieces of each launch's first search), spec_k (GAHC candidates up to this many modules are batched),
 * min_order (level order of MIN proofs: 4 = largest minimal solo latency first, default; 0 =
 * fewest viable options first; any order gives the same T*), min_perm (measurement only),
 * local_handover, fuse_k / fuse_tree (stage_evals of at most fuse_k modules, or of at most fuse_tree option
 * tuples x GPUs, run their MIN proof in the first probe's launch), restart_k (MIN proofs of stages with at least this many modules restart on a big drop), and the measurement-only share_rank / share_world (search one
 * rank's share of a sharded search on this device, unmerged: NOT the stage's answer), share_all
 * (> 1: every large search runs as that many option-prefix shards in one launch on this device
 * and is merged by the multi-GPU rule — the real answer, for shard-balance measurements) and
 * share_peers (1, default: shards of a MIN proof lower each other's incumbent during the search
 * — peer GPUs' control blocks mapped through CUDA IPC; 0: only at the end-of-launch merge).
 * MOSAIC_INVALID_ARGUMENT for an unknown key. */
int mosaic_gpu_set_tuning(mosaic_gpu_ctx* ctx, const char* key, double value);
/* Device memory held by the context's engine (option table, cursor ring, control). */
int64_t mosaic_gpu_device_bytes(mosaic_gpu_ctx* ctx);

/* Kernel launches issued by this context so far (evidence for bench.py). */
int64_t mosaic_gpu_launch_count(mosaic_gpu_ctx* ctx);
/* Device time (ms) spent in the search kernels, by CUDA events on the ctx stream. */
double mosaic_gpu_search_ms(mosaic_gpu_ctx* ctx);
void mosaic_gpu_reset_counters(mosaic_gpu_ctx* ctx);
/* Counters for bench.py: own kernel launches (k_expand/k_search/k_extract/k_eval,
 * library CUB launches excluded), k_search device time and launch count, and bytes
 * moved host->device / device->host. */
int64_t mosaic_gpu_own_launches(mosaic_gpu_ctx* ctx);
double mosaic_gpu_ksearch_ms(mosaic_gpu_ctx* ctx);
int64_t mosaic_gpu_ksearch_launches(mosaic_gpu_ctx* ctx);
int64_t mosaic_gpu_h2d_bytes(mosaic_gpu_ctx* ctx);
int64_t mosaic_gpu_d2h_bytes(mosaic_gpu_ctx* ctx);
/* Algorithmic bytes of the scored leaves: 24*k per leaf (k option rows x 3 fp64). */
int64_t mosaic_gpu_alg_bytes(mosaic_gpu_ctx* ctx);
/* CUDA events on the context's stream: which = 0 start, 1 stop; elapsed in ms. */
void mosaic_gpu_mark(mosaic_gpu_ctx* ctx, int which);
double mosaic_gpu_marked_ms(mosaic_gpu_ctx* ctx);

/* Synthetic inputs (the reference's profiler, profiler.hpp:65-111/185-338, restated
 * in C++ so the GPU box needs no reference): fills a problem for a named BASELINE
 * config "cfg1".."cfg5", "random:SEED:N:G" or "preset:NAME:COUNT:G".  The returned
 * problem owns its storage until mosaic_gpu_free_problem. */
/* ---- N2: input generation on the device (profiler.hpp) ---- */
/* ModuleWorkload (profiler.hpp:26-40); id is informational. */
typedef struct {
    const char* id;
    double flops_per_iter, bytes_per_iter, gradient_bytes, sm_efficiency_knee,
        memory_act_base, memory_per_quota, fixed_overhead, dp_penalty;
} mosaic_gpu_workload;

/* ClusterSpec (core.hpp:52-59). */
typedef struct {
    int32_t gpu_count;
    double memory_capacity, peak_compute, peak_bandwidth, interconnect_alpha,
        interconnect_beta;
} mosaic_gpu_cluster;

/* generate_surface (profiler.hpp:65-101) for n workloads on `device`:
 * out[(w * nd + di) * na + ai] = evaluate_workload(w, cluster, d_set[di], a_set[ai]) with
 * ProfilerConfig.demand_scale.  out holds n * nd * na points.  d_set = NULL uses
 * default_dp_degrees(gpu_count), a_set = NULL default_quota_grid() (profiler.hpp:44-54);
 * *nd_out / *na_out return the grid shape (call with out = NULL to size the buffer). */
int mosaic_gpu_generate_surfaces(const mosaic_gpu_workload* workloads, int32_t n,
                                 const mosaic_gpu_cluster* cluster, const int32_t* d_set,
                                 int32_t nd, const double* a_set, int32_t na,
                                 double demand_scale, int device, mosaic_gpu_point* out,
                                 int32_t* nd_out, int32_t* na_out);

/* The workloads and cluster a synthetic spec is generated from (make_workload /
 * make_preset / random_instance, profiler.hpp:185-338).  Writes up to cap workloads
 * (ids NULL) and *n = their count. */
int mosaic_gpu_synth_workloads(const char* spec, mosaic_gpu_workload* out, int32_t cap,
                               int32_t* n, mosaic_gpu_cluster* cluster);

int mosaic_gpu_synth_problem(const char* spec, int quota_levels, mosaic_gpu_problem** out);
void mosaic_gpu_free_problem(mosaic_gpu_problem* p);

#ifdef __cplusplus
}
#endif
#endif /* MOSAIC_GPU_H */
