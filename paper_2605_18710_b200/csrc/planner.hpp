// planner.hpp — host mirror of the reference planner API, backed by the device engine.
//
//   stage_eval      stage_eval.hpp:302-382 (tau doubling, bisection, confirmation)
//   feasible        detail::FeasibilitySearch::run, stage_eval.hpp:113-164
//   exact_stage     detail::ExactStageSolver::solve, oracle.hpp:86-103
//   solve           GAHC, solver.hpp:157-289 (EvalCache, legal_merge, early_prune)
//   brute_force     brute_force_optimum + enumerate_partitions, oracle.hpp:35-71, 206-255
//   stage_time      rectified_latency/stage_time, perf_model.hpp:442-479 (batched, K1)
//
// Every candidate-plan search runs on the GPU (engine.cu).  The host only replays
// the reference's control flow (which tau to probe next, which merge to apply) and
// converts winning leaves back into StageAllocations.
#pragma once
#include <coroutine>
#include <cstdint>
#include <exception>
#include <memory>
#include <optional>
#include <string>
#include <unordered_map>
#include <vector>

#include "engine.hpp"
#include "sim.hpp"
#include "model.hpp"

namespace mosaic_b200 {

enum Status { OK = 0, INFEASIBLE = 1, MODULE_NO_OPTION = 2, RANGE = 3, TOO_LARGE = 4,
              CUDA = 5, EMPTY = 6, BASELINE_INFEASIBLE = 7, INVALID_ARGUMENT = 8 };

struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

struct Entry {
    int module, d, units;
    std::vector<int> gpus;
    int levels = 0;  // DeploymentOption::quota_levels; 0 = the problem's
};

struct StageResult {
    int status = INFEASIBLE;
    double stage_time = 0.0;
    std::vector<Entry> entries;  // sorted by module index
    long long probes = 0;        // FeasibilitySearch::run calls replayed
    mg::SearchStats st;
    // every replayed FeasibilitySearch::run(tau) in call order and its outcome (probes
    // decided from T* without a device search included): the trajectory parity tests
    // replay against the reference
    std::vector<double> probe_tau;
    std::vector<uint8_t> probe_ok;
};

struct TraceCand {
    uint64_t mask_x, mask_y;
    bool pruned, cache_hit;
    double gain;
};
struct TraceRound {
    std::vector<TraceCand> cands;
    uint64_t chosen_x = 0, chosen_y = 0;
    double applied_gain = 0.0;
};

struct PlanResult {
    int status = OK;
    std::vector<uint64_t> masks;
    std::vector<StageResult> stages;
    double iteration_time = 0.0;
    long long partitions = 0;
    long long stage_eval_calls = 0, feasibility_calls = 0, cache_hits = 0, prunes = 0;
    std::vector<TraceRound> rounds;
    mg::SearchStats st;
    double elapsed = 0.0;
};

// A stage computation (stage_eval / exact_stage) written as a coroutine that suspends at
// every device search it needs: many of them advance together and each wave of their
// searches is one batched launch (Planner::run_jobs, Engine::search_batch).
struct SearchOp {
    mg::BatchReq req;
    mg::HitPath hp;  // seed storage (req.seed_path / seed_leaf point here)
    mg::Leaf sl;
    mg::SearchResult res;
};

struct StageJob {
    struct promise_type {
        SearchOp* op = nullptr;  // the search this job waits for (null: running or done)
        SearchOp* op2 = nullptr; // a second, independent search of the same wave (or null)
        std::exception_ptr exc;
        StageJob get_return_object() {
            return StageJob{std::coroutine_handle<promise_type>::from_promise(*this)};
        }
        std::suspend_always initial_suspend() noexcept { return {}; }
        std::suspend_always final_suspend() noexcept { return {}; }
        void return_void() noexcept {}
        void unhandled_exception() noexcept { exc = std::current_exception(); }
    };
    std::coroutine_handle<promise_type> h;
    explicit StageJob(std::coroutine_handle<promise_type> x = {}) : h(x) {}
    StageJob(StageJob&& o) noexcept : h(o.h) { o.h = {}; }
    StageJob& operator=(StageJob&& o) noexcept {
        if (h) h.destroy();
        h = o.h;
        o.h = {};
        return *this;
    }
    StageJob(const StageJob&) = delete;
    ~StageJob() {
        if (h) h.destroy();
    }
};

struct SearchAwait {
    SearchOp* op;
    bool await_ready() const noexcept { return false; }
    void await_suspend(std::coroutine_handle<StageJob::promise_type> h) const noexcept {
        h.promise().op = op;
    }
    mg::SearchResult await_resume() const noexcept { return op->res; }
};

// Two independent searches of one job in the same wave (results in a->res, b->res).
struct SearchAwait2 {
    SearchOp* a;
    SearchOp* b;
    bool await_ready() const noexcept { return false; }
    void await_suspend(std::coroutine_handle<StageJob::promise_type> h) const noexcept {
        h.promise().op = a;
        h.promise().op2 = b;
    }
    void await_resume() const noexcept {}
};

class Planner {
  public:
    Planner(Problem P, int device);
    const Problem& problem() const { return P_; }
    const std::vector<Cand>& options(int m) const { return opts_.at(m); }

    StageResult stage_eval(uint64_t mask);
    StageResult exact_stage(uint64_t mask);
    // Batched (mosaic_gpu_search): the module sets' computations advance together, one launch
    // per wave of device searches.  exact = ExactStageSolver semantics, else stage_eval.
    std::vector<StageResult> stage_batch(const std::vector<uint64_t>& masks, bool exact,
                                         std::vector<char>* failed = nullptr);
    StageResult feasible(uint64_t mask, double tau);
    PlanResult solve();
    // validate_plan (core.hpp:281-351) with the footprint oracle; "" when valid, else the
    // ValidationCode name, message in *msg
    std::string validate_plan(const std::vector<std::vector<Entry>>& stages,
                              std::string* msg) const;
    // T* of a module set below `ub` (one MIN search when restart == false)
    double stage_min(uint64_t mask, double ub, bool restart, mg::SearchStats& st);
    PlanResult brute_force();
    // stage_time of explicit allocations (entries per allocation sorted by module)
    void stage_time(const std::vector<std::vector<Entry>>& allocs, std::vector<double>& st,
                    std::vector<std::vector<double>>& rect);
    // K1 on the ABI layout (mosaic_gpu_evaluate): host or device arrays, no repacking.
    // Throws Error(RANGE / TOO_LARGE) for the reference's exceptions.
    void evaluate(const mg::EvalABI* ent, long long n_ent, const int* gpus, long long n_gpu_ids,
                  const long long* off, long long n, double* st, double* rect, bool device_ptrs);

    // make_baseline_plan (simulator.hpp:283-313): policy 0 Megatron, 1 DistMM; full-quota
    // options at this problem's quota_levels; stage times from the device evaluator
    PlanResult baseline_plan(int policy);
    // simulate (simulator.hpp:68-119) of a plan for many seeds on the device (sim.cu)
    void simulate(const std::vector<std::vector<Entry>>& stages, const mg::SimCfg& cfg,
                  const std::vector<uint64_t>& seeds, std::vector<double>& iter,
                  std::vector<double>& per_stage, std::vector<double>& busy,
                  std::vector<double>& mean_busy, std::vector<mg::SimInterval>* timeline);

    mg::Engine& engine() { return *eng_; }
    void clear_cache() {
        cache_.clear();
        cache_order_.clear();
    }
    // EvalCache contents in insertion order (solver.hpp:39-75)
    const std::vector<uint64_t>& cache_order() const { return cache_order_; }
    const StageResult* cache_find(uint64_t mask) const {
        auto it = cache_.find(mask);
        return it == cache_.end() ? nullptr : &it->second;
    }

  private:
    void check_rows(int m) const;
    bool ensure_rate_tables();  // false when they would not fit (then the row path is used)
    StageJob stage_eval_job(uint64_t mask, StageResult* out);
    StageJob exact_stage_job(uint64_t mask, StageResult* out);
    void run_jobs(std::vector<StageJob>& jobs, std::vector<char>* failed = nullptr);
    // FIRST probe request (false: some level has no usable option, no leaf can exist)
    bool prep_first(const std::vector<int>& order, bool filter, double theta, SearchOp& op,
                    mg::SearchStats& st, const std::vector<Entry>* seed = nullptr,
                    double seed_value = 0.0);
    bool prep_min(const std::vector<int>& mods, double ub, SearchOp& op, mg::SearchStats& st,
                  std::vector<int>& order);
    bool first_leaf(const std::vector<int>& order, bool filter, double theta, mg::Leaf& leaf,
                    mg::SearchStats& st, const std::vector<Entry>* seed = nullptr,
                    double seed_value = 0.0);
    double min_value(const std::vector<int>& mods, double ub, mg::SearchStats& st,
                     std::vector<Entry>* argmin = nullptr);
    double exclusive_latency(int m, int d) const;
    std::vector<Entry> distmm_wave(const std::vector<int>& wave) const;
    std::vector<std::vector<int>> dependency_waves() const;
    bool make_seed(const std::vector<Entry>& ents, const std::vector<int>& order, bool filter,
                   double theta, double value, mg::HitPath& hp, mg::Leaf& lf) const;
    std::vector<Entry> leaf_entries(const std::vector<int>& order, const mg::Leaf& lf) const;
    std::optional<StageResult> evaluate_cached(uint64_t mask, bool* hit, PlanResult& pr);
    void speculate(const std::vector<uint64_t>& masks, PlanResult& pr);

    Problem P_;
    mg::Model M_;
    std::vector<std::vector<Cand>> opts_;
    std::vector<std::string> opt_err_;
    std::unique_ptr<mg::Engine> eng_;
    std::unordered_map<uint64_t, StageResult> cache_;
    std::vector<uint64_t> cache_order_;
    int rate_tables_ = 0;  // 0 not built yet, 1 built, -1 too large for this problem
    // per module: (min filter bound, min solo rectified latency) — stage_eval's tau_lo / tau_hi
    std::vector<std::pair<double, double>> tau_mins_;
    // stage_eval results computed speculatively for GAHC candidates the reference prunes
    // (not in the EvalCache; moved there when the reference would evaluate them)
    std::unordered_map<uint64_t, StageResult> spec_;
};

}  // namespace mosaic_b200
