// gpu_backend.hpp — the reference-side binding a Mosaic maintainer adds to use the B200 backend
// from the reference's own C++ API (namespace mosaic, proj/include).  Header-only, C ABI
// underneath (include/mosaic_gpu.h); compiled against the unmodified reference headers by
// tests/shim/Makefile and exercised by tests/shim/test_shim.cpp.
//
// Seams of the reference it plugs into (no reference file is modified):
//   * solve (solver.hpp:157-289) takes an EvalCache* (solver.hpp:160): solve_on_gpu() runs the
//     GAHC stage evaluations on the device (mosaic_gpu_solve, batched per round) and hands the
//     reference's own solve() a cache holding every StageEvalResult it will ask for, keyed
//     exactly as solve() keys them (mask, quota_levels, interference fingerprint ^ !include_self,
//     solver.hpp:167-176).  The reference's GAHC then runs unchanged; every evaluate() is a hit.
//   * stage_eval (stage_eval.hpp:302-382): Backend::stage_eval / stage_eval_batch.
//   * ExactStageSolver::solve (oracle.hpp:86-103) inside brute_force_optimum (oracle.hpp:206-255):
//     brute_force_on_gpu() is brute_force_optimum with the memoised stage_min served by
//     mosaic_gpu_search(MOSAIC_SEARCH_EXACT), one batched call for every stage set of every
//     partition, over the reference's own enumerate_partitions.
// A Backend is keyed by everything the device context is built from (graph, surfaces,
// interference model, include_self, cluster, SolveConfig), so a second problem on the same
// thread gets its own context, never a stale one.
#pragma once
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "mosaic/oracle.hpp"
#include "mosaic/solver.hpp"
#include "mosaic/stage_eval.hpp"
#include "mosaic_gpu.h"

namespace mosaic_gpu_shim {

struct GpuError : std::runtime_error {
    int status;
    GpuError(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void check(int code) {
    if (code == MOSAIC_OK || code == MOSAIC_INFEASIBLE) return;
    const std::string msg = mosaic_gpu_last_error();
    switch (code) {
        case MOSAIC_MODULE_NO_OPTION: throw mosaic::StageInfeasibleError(msg);
        case MOSAIC_RANGE: throw mosaic::SurfaceRangeError(msg);
        case MOSAIC_EMPTY: throw mosaic::EmptyPlanError(msg);
        default: throw GpuError(code, msg);
    }
}

// Everything the device context depends on, as a comparable key.
struct ProblemKey {
    std::vector<std::string> ids;
    std::vector<double> membase;
    std::vector<std::pair<std::string, std::string>> edges;
    std::vector<std::vector<double>> points;  // per module: (d, a, lat, bw, mem, sm) flattened
    double e1, e2, e3;
    int additive, include_self;
    int gpu_count;
    double capacity;
    int levels;
    double bisect;
    int prune, cache;
    auto tie() const {
        return std::tie(ids, membase, edges, points, e1, e2, e3, additive, include_self,
                        gpu_count, capacity, levels, bisect, prune, cache);
    }
    bool operator<(const ProblemKey& o) const { return tie() < o.tie(); }
};

inline ProblemKey make_key(const mosaic::PerfContext& ctx, const mosaic::ClusterSpec& cl,
                           const mosaic::SolveConfig& cfg) {
    ProblemKey k;
    const mosaic::ModelGraph& g = *ctx.graph;
    for (const auto& m : g.modules) {
        k.ids.push_back(m.id);
        k.membase.push_back(m.memory_base);
        std::vector<double> pts;
        for (const auto& p : ctx.surfaces->by_id(m.id).points())
            pts.insert(pts.end(), {(double)p.d, p.a, p.latency, p.bandwidth_util, p.memory,
                                   p.sm_active});
        k.points.push_back(std::move(pts));
    }
    k.edges = g.edges;
    k.e1 = ctx.interference.e1;
    k.e2 = ctx.interference.e2;
    k.e3 = ctx.interference.e3;
    k.additive = ctx.interference.additive_only;
    k.include_self = ctx.include_self;
    k.gpu_count = cl.gpu_count;
    k.capacity = cl.memory_capacity;
    k.levels = cfg.quota_levels;
    k.bisect = cfg.bisect_rel_tol;
    k.prune = cfg.enable_prune;
    k.cache = cfg.enable_cache;
    return k;
}

class Backend {
  public:
    Backend(const mosaic::PerfContext& ctx, const mosaic::ClusterSpec& cl,
            const mosaic::SolveConfig& cfg, int device = 0)
        : graph_(ctx.graph), levels_(cfg.quota_levels) {
        const mosaic::ModelGraph& g = *ctx.graph;
        std::vector<std::vector<mosaic_gpu_point>> pts(g.modules.size());
        std::vector<mosaic_gpu_module> mods(g.modules.size());
        for (size_t i = 0; i < g.modules.size(); ++i) {
            for (const auto& p : ctx.surfaces->by_id(g.modules[i].id).points())
                pts[i].push_back({p.d, p.a, p.latency, p.bandwidth_util, p.memory, p.sm_active});
            mods[i] = {g.modules[i].id.c_str(), g.modules[i].memory_base, pts[i].data(),
                       (int32_t)pts[i].size()};
        }
        std::vector<int32_t> edges;
        for (const auto& [u, v] : g.edges) {
            edges.push_back(g.index_of(u));
            edges.push_back(g.index_of(v));
        }
        mosaic_gpu_problem p{};
        p.modules = mods.data();
        p.n_modules = (int32_t)mods.size();
        p.edges = edges.data();
        p.n_edges = (int32_t)(edges.size() / 2);
        p.gpu_count = cl.gpu_count;
        p.memory_capacity = cl.memory_capacity;
        p.e1 = ctx.interference.e1;
        p.e2 = ctx.interference.e2;
        p.e3 = ctx.interference.e3;
        p.additive_only = ctx.interference.additive_only;
        p.include_self = ctx.include_self;
        p.quota_levels = cfg.quota_levels;
        p.bisect_rel_tol = cfg.bisect_rel_tol;
        p.enable_prune = cfg.enable_prune;
        p.enable_cache = 1;  // the device EvalCache is how results reach the reference's solve()
        check(mosaic_gpu_create(&p, device, &ctx_));
        model_fp_ = ctx.interference.fingerprint() ^ (ctx.include_self ? 0 : 1);
    }
    ~Backend() { mosaic_gpu_destroy(ctx_); }
    Backend(const Backend&) = delete;
    Backend& operator=(const Backend&) = delete;

    // The context for (ctx, cluster, cfg), created once per problem and thread.
    static Backend& get(const mosaic::PerfContext& ctx, const mosaic::ClusterSpec& cl,
                        const mosaic::SolveConfig& cfg, int device = 0) {
        thread_local std::map<ProblemKey, std::unique_ptr<Backend>> pool;
        ProblemKey k = make_key(ctx, cl, cfg);
        auto it = pool.find(k);
        if (it == pool.end())
            it = pool.emplace(std::move(k), std::make_unique<Backend>(ctx, cl, cfg, device)).first;
        else
            it->second->graph_ = ctx.graph;
        return *it->second;
    }

    mosaic_gpu_ctx* raw() const { return ctx_; }

    mosaic::StageEvalResult convert(const mosaic_gpu_stage_result& r) const {
        mosaic::StageEvalResult out;
        out.stage_time = r.stage_time;
        for (int i = 0; i < r.n_entries; ++i) {
            const auto& e = r.entries[i];
            mosaic::StageAllocation::Entry x;
            x.module = e.module;
            x.option = {e.dp_degree, e.quota_units, levels_};
            x.gpus.assign(e.gpus, e.gpus + e.n_gpus);
            out.allocation.entries.push_back(std::move(x));
        }
        out.stats.feasibility_calls = r.probes;
        out.stats.nodes = r.nodes;
        return out;
    }

    // stage_eval seam (stage_eval.hpp:302): nullopt when infeasible, StageInfeasibleError
    // when a module has no option at all — the reference's contract.
    std::vector<std::optional<mosaic::StageEvalResult>> stage_eval_batch(
        const std::vector<std::vector<int>>& stages, bool exact = false) {
        std::vector<uint64_t> masks;
        for (const auto& s : stages) {
            uint64_t m = 0;
            for (int x : s) m |= uint64_t(1) << x;
            masks.push_back(m);
        }
        std::vector<mosaic_gpu_stage_result> rs(masks.size());
        check(mosaic_gpu_search(ctx_, masks.data(), (int64_t)masks.size(),
                                exact ? MOSAIC_SEARCH_EXACT : MOSAIC_SEARCH_STAGE_EVAL,
                                rs.data(), nullptr, nullptr));
        std::vector<std::optional<mosaic::StageEvalResult>> out;
        for (const auto& r : rs) {
            if (r.status == MOSAIC_MODULE_NO_OPTION)
                throw mosaic::StageInfeasibleError("module has no feasible deployment option");
            out.push_back(r.status == MOSAIC_OK ? std::optional(convert(r)) : std::nullopt);
        }
        return out;
    }
    std::optional<mosaic::StageEvalResult> stage_eval(const std::vector<int>& modules) {
        return stage_eval_batch({modules})[0];
    }

    // Every StageEvalResult the GAHC will request, computed on the device (one batched launch
    // per wave of each round), inserted under solve()'s own EvalCache keys.
    void prefill(mosaic::EvalCache& cache) {
        mosaic_gpu_plan_result pr;
        check(mosaic_gpu_solve(ctx_, &pr));
        int64_t n = 0;
        check(mosaic_gpu_cache_masks(ctx_, nullptr, 0, &n));
        std::vector<uint64_t> masks(n);
        check(mosaic_gpu_cache_masks(ctx_, masks.data(), n, &n));
        for (uint64_t m : masks) {
            mosaic_gpu_stage_result r;
            int64_t np = 0;
            check(mosaic_gpu_cache_entry(ctx_, m, &r, nullptr, nullptr, 0, &np));
            cache.insert(mosaic::EvalCache::Key{m, levels_, model_fp_}, convert(r));
        }
    }

  private:
    mosaic_gpu_ctx* ctx_ = nullptr;
    const mosaic::ModelGraph* graph_;
    int levels_;
    uint64_t model_fp_ = 0;
};

// mosaic::solve with the GPU at its stage-evaluation seam: the reference's own GAHC over an
// EvalCache the device filled.  `misses` (optional) reports evaluations the cache could not
// answer (0 when the device and the reference agree on every stage the GAHC visits).
inline mosaic::SolveResult solve_on_gpu(const mosaic::PerfContext& ctx,
                                        const mosaic::ClusterSpec& cl,
                                        const mosaic::SolveConfig& cfg = {},
                                        long long* misses = nullptr) {
    mosaic::EvalCache cache;
    Backend::get(ctx, cl, cfg).prefill(cache);
    mosaic::SolveConfig c = cfg;
    c.enable_cache = true;  // the device results reach solve() through its cache
    mosaic::SolveResult r = mosaic::solve(ctx, cl, c, &cache);
    if (misses) *misses = cache.misses();
    return r;
}

// brute_force_optimum (oracle.hpp:206-255) with ExactStageSolver::solve served by the device:
// the same partition loop and cheap cut over the reference's enumerate_partitions.
inline std::optional<mosaic::OracleResult> brute_force_on_gpu(const mosaic::PerfContext& ctx,
                                                              const mosaic::ClusterSpec& cl,
                                                              int quota_levels = 10) {
    const mosaic::ModelGraph& g = *ctx.graph;
    if (g.size() > 8) throw mosaic::OracleTooLargeError("oracle enumeration limited to 8 modules");
    auto partitions = mosaic::enumerate_partitions(g);
    mosaic::SolveConfig cfg;
    cfg.quota_levels = quota_levels;
    Backend& be = Backend::get(ctx, cl, cfg);
    // every distinct stage set of every partition in one batched call
    std::map<uint64_t, size_t> index;
    std::vector<std::vector<int>> stages;
    for (const auto& part : partitions)
        for (const auto& st : part) {
            uint64_t m = 0;
            for (int x : st) m |= uint64_t(1) << x;
            if (index.emplace(m, stages.size()).second) stages.push_back(st);
        }
    auto exact = be.stage_eval_batch(stages, true);
    std::optional<mosaic::OracleResult> best;
    for (const auto& partition : partitions) {
        double total = 0.0;
        std::vector<const mosaic::StageEvalResult*> used;
        bool feasible = true;
        for (const auto& stage : partition) {
            uint64_t m = 0;
            for (int x : stage) m |= uint64_t(1) << x;
            const auto& r = exact[index.at(m)];
            if (!r) {
                feasible = false;
                break;
            }
            total += r->stage_time;
            used.push_back(&*r);
            if (best && total >= best->iteration_time) {
                feasible = false;
                break;
            }
        }
        if (!feasible || used.size() != partition.size()) continue;
        if (!best || total < best->iteration_time) {
            mosaic::OracleResult r;
            r.iteration_time = total;
            for (const auto* s : used) {
                r.plan.stages.push_back(s->allocation);
                r.plan.predicted_stage_times.push_back(s->stage_time);
            }
            r.plan.predicted_iteration_time = total;
            best = std::move(r);
        }
    }
    if (best) best->partitions_examined = static_cast<long long>(partitions.size());
    return best;
}

}  // namespace mosaic_gpu_shim
