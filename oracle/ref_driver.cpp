// TEST INFRASTRUCTURE ONLY — never linked into, or called by, the product path.
//
// Driver around the UNMODIFIED reference headers (/root/reference/proj/include,
// compiled in place by oracle/Makefile; nothing is copied into this repo).  It
// builds the five BASELINE configs and the reference's own random instances,
// runs the reference planner entry points and prints one JSON object per call:
//
//   solve            mosaic::solve                 (solver.hpp:157)
//   oracle           mosaic::brute_force_optimum   (oracle.hpp:206)
//   stage MASK       mosaic::stage_eval            (stage_eval.hpp:302)
//   exact MASK       detail::ExactStageSolver      (oracle.hpp:86)
//   feas MASK TAU    detail::FeasibilitySearch::run (stage_eval.hpp:113)
//   options          candidate_options per module  (stage_eval.hpp:68)
//   stime ALLOC      stage_time                    (perf_model.hpp:474)
//   partitions       enumerate_partitions count    (oracle.hpp:35)
//
// Doubles are printed twice: "%a" (bit-exact, what parity tests compare) and
// "%.17g" (readable).  When compiled with -DMOSAIC_INSTR against the
// instrumented header copy under oracle/_ref/instr (see Makefile), every
// scored leaf (stage_eval.hpp:254 verify_complete, oracle.hpp:112 leaf) and
// every feasibility probe tau is counted and reported.
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#ifdef MOSAIC_INSTR
#include <vector>
namespace mosaic_instr {
inline long long leaves = 0;
inline std::vector<double> probes;
inline std::vector<int> probe_ok;
}  // namespace mosaic_instr
#endif

#include "mosaic/bench.hpp"
#ifdef MOSAIC_WITH_IO
#include "mosaic/io.hpp"
#endif
#include "mosaic/oracle.hpp"
#include "mosaic/profiler.hpp"
#include "mosaic/simulator.hpp"
#include "mosaic/solver.hpp"
#include "mosaic/stage_eval.hpp"
#include "ref_instances.hpp"

using namespace mosaic;
using mosaic_ref::Instance;
using mosaic_ref::make_instance;

namespace {

void pd(const char* key, double v, bool comma = true) {
    std::printf("\"%s\":\"%a\",\"%s_dec\":%.17g%s", key, v, key, v, comma ? "," : "");
}

void print_alloc(const StageAllocation& al) {
    std::printf("[");
    for (size_t i = 0; i < al.entries.size(); ++i) {
        const auto& e = al.entries[i];
        std::printf("%s{\"m\":%d,\"d\":%d,\"u\":%d,\"gpus\":[", i ? "," : "", e.module,
                    e.option.dp_degree, e.option.quota_units);
        for (size_t j = 0; j < e.gpus.size(); ++j) std::printf("%s%d", j ? "," : "", e.gpus[j]);
        std::printf("]}");
    }
    std::printf("]");
}

void print_plan(const DeploymentPlan& plan) {
    std::printf("\"stages\":[");
    for (size_t s = 0; s < plan.stages.size(); ++s) {
        std::printf("%s{", s ? "," : "");
        pd("t", plan.predicted_stage_times[s]);
        std::printf("\"alloc\":");
        print_alloc(plan.stages[s]);
        std::printf("}");
    }
    std::printf("],");
    pd("iteration_time", plan.predicted_iteration_time);
}

std::vector<int> mask_mods(uint64_t mask) {
    std::vector<int> out;
    for (int m = 0; m < 64; ++m)
        if (mask >> m & 1) out.push_back(m);
    return out;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

void instr_reset() {
#ifdef MOSAIC_INSTR
    mosaic_instr::leaves = 0;
    mosaic_instr::probes.clear();
#endif
}

void instr_print() {
#ifdef MOSAIC_INSTR
    std::printf(",\"leaves\":%lld,\"probes\":[", mosaic_instr::leaves);
    for (size_t i = 0; i < mosaic_instr::probes.size(); ++i)
        std::printf("%s\"%a\"", i ? "," : "", mosaic_instr::probes[i]);
    std::printf("]");
#endif
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr,
                     "usage: ref_driver INST OP [args] [levels=L] [e=e1,e2,e3] [noself] "
                     "[additive] [reps=R] [noprune] [nocache]\n");
        return 2;
    }
    Instance in;
    if (!make_instance(argv[1], in)) {
        std::fprintf(stderr, "bad instance %s\n", argv[1]);
        return 2;
    }
    std::string op = argv[2];
    std::vector<std::string> pos;
    int reps = 1;
    bool prune = true, cache = true;
    for (int i = 3; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("levels=", 0) == 0) in.levels = std::atoi(a.c_str() + 7);
        else if (a.rfind("gpus=", 0) == 0) in.cluster.gpu_count = std::atoi(a.c_str() + 5);
        else if (a.rfind("mem=", 0) == 0) in.cluster.memory_capacity = std::strtod(a.c_str() + 4, nullptr);
        else if (a.rfind("e=", 0) == 0)
            std::sscanf(a.c_str() + 2, "%lf,%lf,%lf", &in.im.e1, &in.im.e2, &in.im.e3);
        else if (a == "noself") in.include_self = false;
        else if (a == "additive") in.im.additive_only = true;
        else if (a.rfind("reps=", 0) == 0) reps = std::atoi(a.c_str() + 5);
        else if (a == "noprune") prune = false;
        else if (a == "nocache") cache = false;
        else pos.push_back(a);
    }
    in.finish();
    const int L = in.levels;

    std::printf("{\"inst\":\"%s\",\"op\":\"%s\",\"levels\":%d,\"gpus\":%d,", in.name.c_str(),
                op.c_str(), L, in.cluster.gpu_count);
    try {
        if (op == "solve") {
            SolveConfig cfg{L, 1e-3, prune, cache};
            SolveResult r;
            std::vector<double> times;
            for (int i = 0; i < reps; ++i) {
                instr_reset();
                double t0 = now_s();
                r = solve(in.ctx, in.cluster, cfg);
                times.push_back(now_s() - t0);
            }
            print_plan(r.plan);
            std::printf("\"rounds\":[");
            for (size_t i = 0; i < r.trace.rounds.size(); ++i) {
                const auto& rd = r.trace.rounds[i];
                std::printf("%s{\"x\":%" PRIu64 ",\"y\":%" PRIu64 ",\"gain\":\"%a\",\"cands\":[",
                            i ? "," : "", rd.chosen_x, rd.chosen_y, rd.applied_gain);
                for (size_t j = 0; j < rd.candidates.size(); ++j) {
                    const auto& c = rd.candidates[j];
                    std::printf("%s{\"x\":%" PRIu64 ",\"y\":%" PRIu64
                                ",\"pruned\":%d,\"hit\":%d,\"gain\":\"%a\"}",
                                j ? "," : "", c.mask_x, c.mask_y, c.pruned, c.cache_hit, c.gain);
                }
                std::printf("]}");
            }
            std::printf("],\"stage_eval_calls\":%lld,\"feasibility_calls\":%lld,\"times\":[",
                        r.trace.stage_eval_calls, r.trace.feasibility_calls);
            for (size_t i = 0; i < times.size(); ++i) std::printf("%s%.9g", i ? "," : "", times[i]);
            std::printf("]");
            instr_print();
        } else if (op == "oracle") {
            std::optional<OracleResult> r;
            std::vector<double> times;
            for (int i = 0; i < reps; ++i) {
                instr_reset();
                double t0 = now_s();
                r = brute_force_optimum(in.ctx, in.cluster, L);
                times.push_back(now_s() - t0);
            }
            std::printf("\"feasible\":%d,", r ? 1 : 0);
            if (r) {
                print_plan(r->plan);
                std::printf("\"partitions\":%lld,", r->partitions_examined);
            }
            std::printf("\"times\":[");
            for (size_t i = 0; i < times.size(); ++i) std::printf("%s%.9g", i ? "," : "", times[i]);
            std::printf("]");
            instr_print();
        } else if (op == "stage" || op == "exact") {
            uint64_t mask = std::strtoull(pos.at(0).c_str(), nullptr, 0);
            auto mods = mask_mods(mask);
            std::optional<StageEvalResult> r;
            std::vector<double> times;
            int status = 0;
            for (int i = 0; i < reps; ++i) {
                instr_reset();
                double t0 = now_s();
                try {
                    if (op == "stage") {
                        r = stage_eval(in.ctx, in.cluster, mods, {L, 1e-3});
                    } else {
                        detail::ExactStageSolver ex(in.ctx, in.cluster, L);
                        r = ex.solve(mods);
                    }
                } catch (const StageInfeasibleError&) {
                    status = 2;
                }
                times.push_back(now_s() - t0);
            }
            std::printf("\"mask\":%" PRIu64 ",\"status\":%d,\"feasible\":%d,", mask, status,
                        r ? 1 : 0);
            if (r) {
                pd("t", r->stage_time);
                std::printf("\"alloc\":");
                print_alloc(r->allocation);
                std::printf(",\"feasibility_calls\":%lld,\"nodes\":%lld,",
                            r->stats.feasibility_calls, r->stats.nodes);
            }
            std::printf("\"times\":[");
            for (size_t i = 0; i < times.size(); ++i) std::printf("%s%.9g", i ? "," : "", times[i]);
            std::printf("]");
            instr_print();
        } else if (op == "feas") {
            uint64_t mask = std::strtoull(pos.at(0).c_str(), nullptr, 0);
            double tau = std::strtod(pos.at(1).c_str(), nullptr);
            auto mods = mask_mods(mask);
            std::vector<std::vector<CandidateOption>> options;
            for (int m : mods) options.push_back(candidate_options(in.ctx, in.cluster, m, L));
            SolverStats stats;
            detail::FeasibilitySearch fs(in.ctx, in.cluster, mods, options, L, stats);
            auto r = fs.run(tau);
            std::printf("\"mask\":%" PRIu64 ",", mask);
            pd("tau", tau);
            std::printf("\"feasible\":%d", r ? 1 : 0);
            if (r) {
                std::printf(",");
                pd("t", stage_time(in.ctx, *r), false);
                std::printf(",\"alloc\":");
                print_alloc(*r);
            }
        } else if (op == "options") {
            std::printf("\"modules\":[");
            for (int m = 0; m < in.graph.size(); ++m) {
                auto opts = candidate_options(in.ctx, in.cluster, m, L);
                std::printf("%s{\"id\":\"%s\",\"rows\":[", m ? "," : "",
                            in.graph.modules[m].id.c_str());
                for (size_t i = 0; i < opts.size(); ++i) {
                    const auto& c = opts[i];
                    std::printf("%s[%d,%d,\"%a\",\"%a\",\"%a\"]", i ? "," : "", c.opt.dp_degree,
                                c.opt.quota_units, c.base_latency, c.solo_bandwidth, c.footprint);
                }
                std::printf("]}");
            }
            std::printf("]");
        } else if (op == "stime") {
            // ALLOC: m:d:u:g0.g1.g2;m:d:u:...
            StageAllocation al;
            std::string s = pos.at(0);
            size_t p = 0;
            while (p < s.size()) {
                size_t q = s.find(';', p);
                if (q == std::string::npos) q = s.size();
                std::string ent = s.substr(p, q - p);
                StageAllocation::Entry e;
                int m, d, u;
                char gl[4096] = {0};
                std::sscanf(ent.c_str(), "%d:%d:%d:%4095s", &m, &d, &u, gl);
                e.module = m;
                e.option = {d, u, L};
                std::string g = gl;
                size_t a = 0;
                while (a < g.size()) {
                    size_t b = g.find('.', a);
                    if (b == std::string::npos) b = g.size();
                    e.gpus.push_back(std::atoi(g.substr(a, b - a).c_str()));
                    a = b + 1;
                }
                al.entries.push_back(e);
                p = q + 1;
            }
            pd("t", stage_time(in.ctx, al), false);
#ifdef MOSAIC_WITH_IO
        } else if (op == "json") {
            // reference JSON v1 files for this instance (io.hpp) + the plan solve() returns
            SolveConfig cfg{L, 1e-3, prune, cache};
            auto r = solve(in.ctx, in.cluster, cfg);
            nlohmann::json j;
            j["model"] = to_json(in.graph);
            j["cluster"] = to_json(in.cluster);
            j["profile"] = to_json(in.surfaces);
            j["interference"] = to_json(in.im);
            j["plan"] = to_json(r.plan, in.graph);
            std::printf("\"files\":%s", j.dump().c_str());
#endif
        } else if (op == "validate") {
            // PLAN: stage|stage|...; stage: m:d:u:g0.g1;m:d:u:...  (validate_plan, core.hpp:281)
            DeploymentPlan plan;
            std::string spec = pos.at(0);
            size_t a = 0;
            while (a <= spec.size()) {
                size_t b = spec.find('|', a);
                if (b == std::string::npos) b = spec.size();
                std::string st = spec.substr(a, b - a);
                StageAllocation al;
                size_t p = 0;
                while (p < st.size()) {
                    size_t q = st.find(';', p);
                    if (q == std::string::npos) q = st.size();
                    std::string ent = st.substr(p, q - p);
                    StageAllocation::Entry e;
                    int m, d, u;
                    char gl[8192] = {0};
                    std::sscanf(ent.c_str(), "%d:%d:%d:%8191s", &m, &d, &u, gl);
                    e.module = m;
                    e.option = {d, u, L};
                    std::string g = gl;
                    size_t x = 0;
                    while (x < g.size()) {
                        size_t y = g.find('.', x);
                        if (y == std::string::npos) y = g.size();
                        e.gpus.push_back(std::atoi(g.substr(x, y - x).c_str()));
                        x = y + 1;
                    }
                    al.entries.push_back(e);
                    p = q + 1;
                }
                plan.stages.push_back(al);
                a = b + 1;
            }
            FootprintOracle fo{&in.ctx, [](const void* c, int m, const DeploymentOption& o) {
                                   return static_cast<const PerfContext*>(c)->footprint(m, o);
                               }};
            auto err = validate_plan(plan, in.graph, in.cluster, fo);
            std::printf("\"code\":\"%s\"", err ? to_string(err->code) : "Ok");
        } else if (op == "baseline" || op == "simulate") {
            // baseline megatron|distmm  (make_baseline_plan, simulator.hpp:283-313)
            // simulate solve|megatron|distmm [iters=N] [sigma=S] [seed=X] [ondemand]
            //   (simulate, simulator.hpp:68-119) on that plan
            std::string which = pos.at(0);
            SimConfig sc;
            for (size_t i = 1; i < pos.size(); ++i) {
                const std::string& a = pos[i];
                if (a.rfind("iters=", 0) == 0) sc.iterations = std::atoi(a.c_str() + 6);
                else if (a.rfind("sigma=", 0) == 0) sc.perturbation_sigma = std::strtod(a.c_str() + 6, nullptr);
                else if (a.rfind("seed=", 0) == 0) sc.seed = std::strtoull(a.c_str() + 5, nullptr, 0);
                else if (a == "ondemand") sc.stream_mode = StreamMode::OnDemand;
            }
            DeploymentPlan plan;
            if (which == "solve") {
                plan = solve(in.ctx, in.cluster, SolveConfig{L, 1e-3, prune, cache}).plan;
            } else {
                plan = make_baseline_plan(in.ctx, in.cluster,
                                          which == "megatron" ? BaselinePolicy::Megatron
                                                              : BaselinePolicy::DistMM,
                                          L);
            }
            print_plan(plan);
            std::printf("\"ok\":1");
            if (op == "simulate") {
                auto rep = simulate(in.ctx, in.cluster, plan, sc);
                std::printf(",");
                pd("sim_iteration_time", rep.iteration_time);
                std::printf("\"per_stage\":[");
                for (size_t i = 0; i < rep.per_stage_times.size(); ++i)
                    std::printf("%s\"%a\"", i ? "," : "", rep.per_stage_times[i]);
                std::printf("],\"busy\":[");
                for (size_t i = 0; i < rep.per_gpu_busy_fraction.size(); ++i)
                    std::printf("%s\"%a\"", i ? "," : "", rep.per_gpu_busy_fraction[i]);
                std::printf("],");
                pd("mean_busy", rep.mean_busy_fraction, false);
                std::printf(",\"timeline\":[");
                for (size_t i = 0; i < rep.timeline.size(); ++i) {
                    const auto& t = rep.timeline[i];
                    std::printf("%s[%d,%d,\"%a\",\"%a\",\"%a\"]", i ? "," : "", t.gpu, t.module,
                                t.start, t.end, t.quota);
                }
                std::printf("]");
            }
        } else if (op == "normals") {
            // normals SEED N: std::normal_distribution<double>(0,1) over std::mt19937_64(SEED)
            // exactly as simulate() draws them (simulator.hpp:75-76, 89-91)
            std::mt19937_64 rng(std::strtoull(pos.at(0).c_str(), nullptr, 0));
            std::normal_distribution<double> gauss(0.0, 1.0);
            const int n = std::atoi(pos.at(1).c_str());
            std::printf("\"normals\":[");
            for (int i = 0; i < n; ++i) std::printf("%s\"%a\"", i ? "," : "", gauss(rng));
            std::printf("]");
        } else if (op == "partitions") {
            auto parts = enumerate_partitions(in.graph);
            std::printf("\"count\":%zu", parts.size());
        } else {
            std::printf("\"error\":\"unknown op\"}\n");
            return 2;
        }
    } catch (const std::exception& ex) {
        std::printf("\"exception\":\"%s\"}\n", ex.what());
        return 3;
    }
    std::printf("}\n");
    return 0;
}
