// TEST INFRASTRUCTURE: the reference's OWN planner (unmodified headers, /root/reference/proj/
// include) driven through the B200 backend at its seams (tests/shim/gpu_backend.hpp), compared
// with the unmodified reference run on the CPU in the same process.
//
//   solve      mosaic::solve(ctx, cluster, cfg, &cache) with the device-filled EvalCache
//              == mosaic::solve(ctx, cluster, cfg): plan (stage order, allocations, fp64
//              stage / iteration times bit for bit) and every GAHC round (chosen pair, gain,
//              candidates, prune flags); zero cache misses.
//   oracle     brute_force_on_gpu == mosaic::brute_force_optimum (plan, iteration time,
//              partitions examined).
//   stage      Backend::stage_eval == mosaic::stage_eval for every cached module set.
// One JSON line per check; exit status 1 on any mismatch.
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../oracle/ref_instances.hpp"
#include "gpu_backend.hpp"

using namespace mosaic;
using mosaic_gpu_shim::Backend;

static int failures = 0;

static bool same_alloc(const StageAllocation& a, const StageAllocation& b) {
    if (a.entries.size() != b.entries.size()) return false;
    for (size_t i = 0; i < a.entries.size(); ++i) {
        const auto& x = a.entries[i];
        const auto& y = b.entries[i];
        if (x.module != y.module || x.option.dp_degree != y.option.dp_degree ||
            x.option.quota_units != y.option.quota_units || x.gpus != y.gpus)
            return false;
    }
    return true;
}

static bool same_plan(const DeploymentPlan& a, const DeploymentPlan& b) {
    if (a.stages.size() != b.stages.size()) return false;
    if (a.predicted_iteration_time != b.predicted_iteration_time) return false;
    for (size_t s = 0; s < a.stages.size(); ++s)
        if (a.predicted_stage_times[s] != b.predicted_stage_times[s] ||
            !same_alloc(a.stages[s], b.stages[s]))
            return false;
    return true;
}

static bool same_rounds(const SolveTrace& a, const SolveTrace& b) {
    if (a.rounds.size() != b.rounds.size()) return false;
    for (size_t r = 0; r < a.rounds.size(); ++r) {
        const auto& x = a.rounds[r];
        const auto& y = b.rounds[r];
        if (x.chosen_x != y.chosen_x || x.chosen_y != y.chosen_y ||
            x.applied_gain != y.applied_gain || x.candidates.size() != y.candidates.size())
            return false;
        for (size_t c = 0; c < x.candidates.size(); ++c) {
            const auto& p = x.candidates[c];
            const auto& q = y.candidates[c];
            if (p.mask_x != q.mask_x || p.mask_y != q.mask_y || p.pruned != q.pruned ||
                (!p.pruned && p.gain != q.gain))
                return false;
        }
    }
    return true;
}

static void report(const std::string& name, const char* check, bool ok, const std::string& extra) {
    std::printf("{\"inst\":\"%s\",\"check\":\"%s\",\"ok\":%s%s}\n", name.c_str(), check,
                ok ? "true" : "false", extra.c_str());
    std::fflush(stdout);
    if (!ok) ++failures;
}

static void apply(mosaic_ref::Instance& in, const std::string& v) {
    if (v == "noself") in.include_self = false;
    else if (v == "additive") in.im.additive_only = true;
    else if (v.rfind("e=", 0) == 0)
        std::sscanf(v.c_str() + 2, "%lf,%lf,%lf", &in.im.e1, &in.im.e2, &in.im.e3);
    else if (v.rfind("levels=", 0) == 0) in.levels = std::atoi(v.c_str() + 7);
    else if (v.rfind("mem=", 0) == 0) in.cluster.memory_capacity = std::strtod(v.c_str() + 4, nullptr);
}

static void run(const std::string& spec, const std::vector<std::string>& variant, bool oracle,
                bool noprune) {
    mosaic_ref::Instance in;
    if (!mosaic_ref::make_instance(spec, in)) {
        std::fprintf(stderr, "bad instance %s\n", spec.c_str());
        std::exit(2);
    }
    std::string name = spec;
    for (const auto& v : variant) {
        apply(in, v);
        name += "+" + v;
    }
    in.finish();
    SolveConfig cfg{in.levels, 1e-3, !noprune, true};
    if (noprune) name += "+noprune";
    // 1. solve: the reference's GAHC over device stage evaluations; an instance the reference
    // rejects must be rejected the same way (same exception type)
    SolveResult ref, gpu;
    std::string ref_exc, gpu_exc;
    try {
        ref = solve(in.ctx, in.cluster, cfg);
    } catch (const StageInfeasibleError&) {
        ref_exc = "StageInfeasibleError";
    } catch (const SurfaceRangeError&) {
        ref_exc = "SurfaceRangeError";
    }
    long long misses = -1;
    try {
        gpu = mosaic_gpu_shim::solve_on_gpu(in.ctx, in.cluster, cfg, &misses);
    } catch (const StageInfeasibleError&) {
        gpu_exc = "StageInfeasibleError";
    } catch (const SurfaceRangeError&) {
        gpu_exc = "SurfaceRangeError";
    }
    char buf[256];
    if (!ref_exc.empty() || !gpu_exc.empty()) {
        std::snprintf(buf, sizeof buf, ",\"reference\":\"%s\",\"gpu\":\"%s\"", ref_exc.c_str(),
                      gpu_exc.c_str());
        report(name, "solve_rejects", ref_exc == gpu_exc, buf);
        return;
    }
    std::snprintf(buf, sizeof buf, ",\"iteration_time\":\"%a\",\"cache_misses\":%lld,\"rounds\":%zu",
                  gpu.plan.predicted_iteration_time, misses, gpu.trace.rounds.size());
    report(name, "solve", same_plan(ref.plan, gpu.plan) && same_rounds(ref.trace, gpu.trace) &&
                              misses == 0, buf);
    // 2. stage_eval seam on every module set the GAHC evaluated, in one batched call
    Backend& be = Backend::get(in.ctx, in.cluster, cfg);
    int64_t n = 0;
    mosaic_gpu_cache_masks(be.raw(), nullptr, 0, &n);
    std::vector<uint64_t> masks(n);
    mosaic_gpu_cache_masks(be.raw(), masks.data(), n, &n);
    std::vector<std::vector<int>> sets;
    for (uint64_t m : masks) {
        std::vector<int> s;
        for (int i = 0; i < 64; ++i)
            if (m >> i & 1) s.push_back(i);
        sets.push_back(s);
    }
    auto dev = be.stage_eval_batch(sets);
    bool ok = true;
    StageEvalConfig scfg{in.levels, 1e-3};
    for (size_t i = 0; i < sets.size(); ++i) {
        auto r = stage_eval(in.ctx, in.cluster, sets[i], scfg);
        if (r.has_value() != dev[i].has_value()) ok = false;
        else if (r && (r->stage_time != dev[i]->stage_time ||
                       !same_alloc(r->allocation, dev[i]->allocation) ||
                       r->stats.feasibility_calls != dev[i]->stats.feasibility_calls))
            ok = false;
    }
    std::snprintf(buf, sizeof buf, ",\"module_sets\":%zu", sets.size());
    report(name, "stage_eval", ok, buf);
    // 3. brute_force_optimum with ExactStageSolver on the device
    if (oracle) {
        auto r = brute_force_optimum(in.ctx, in.cluster, in.levels);
        auto g = mosaic_gpu_shim::brute_force_on_gpu(in.ctx, in.cluster, in.levels);
        bool same = r.has_value() == g.has_value() &&
                    (!r || (r->iteration_time == g->iteration_time &&
                            r->partitions_examined == g->partitions_examined &&
                            same_plan(r->plan, g->plan)));
        std::snprintf(buf, sizeof buf, ",\"iteration_time\":\"%a\",\"partitions\":%lld",
                      g ? g->iteration_time : 0.0, g ? g->partitions_examined : 0LL);
        report(name, "oracle", same, buf);
    }
}

int main(int argc, char** argv) {
    const bool quick = argc > 1 && std::string(argv[1]) == "quick";
    run("cfg1", {}, true, false);
    run("cfg2", {}, true, false);
    run("cfg3", {}, false, false);
    run("cfg4", {}, false, false);
    if (!quick) {
        run("cfg3", {}, false, true);
        run("random:7:5:16", {}, true, false);
        run("random:11:4:8", {}, true, false);
        run("cfg2", {"noself"}, true, false);
        run("cfg2", {"additive"}, true, false);
        run("cfg3", {"e=0.4e-3,1.2e-3,0"}, false, false);
        run("cfg2", {"mem=20e9"}, true, false);
        run("cfg2", {"mem=60e9"}, true, false);  // tight memory, still feasible
        run("cfg4", {"noself"}, false, false);
    }
    std::printf("{\"failures\":%d}\n", failures);
    return failures ? 1 : 0;
}
