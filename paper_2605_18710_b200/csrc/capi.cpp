// capi.cpp — extern "C" boundary (include/mosaic_gpu.h).  No exception crosses it.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/mosaic_gpu.h"
#include "pack.hpp"
#include "planner.hpp"

using namespace mosaic_b200;

struct mosaic_gpu_ctx {
    std::unique_ptr<Planner> pl;
    PlanResult plan;
    int rank = 0, world = 1;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        g_err.clear();
        return f();
    } catch (const Error& e) {
        g_err = e.what();
        return e.status;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return MOSAIC_INVALID_ARGUMENT;
    } catch (const RangeError& e) {
        g_err = e.what();
        return MOSAIC_RANGE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MOSAIC_CUDA;
    }
}

void fill_stage(const StageResult& r, mosaic_gpu_stage_result* out) {
    std::memset(out, 0, sizeof(*out));
    out->status = r.status;
    out->stage_time = r.stage_time;
    if (r.entries.size() > MOSAIC_GPU_MAX_STAGE_MODULES)
        throw Error(MOSAIC_TOO_LARGE, "too many entries for the result struct");
    out->n_entries = (int32_t)r.entries.size();
    for (size_t i = 0; i < r.entries.size(); ++i) {
        const Entry& e = r.entries[i];
        auto& o = out->entries[i];
        o.module = e.module;
        o.dp_degree = e.d;
        o.quota_units = e.units;
        if (e.gpus.size() > MOSAIC_GPU_MAX_GPUS) throw Error(MOSAIC_TOO_LARGE, "too many GPUs");
        o.n_gpus = (int32_t)e.gpus.size();
        for (size_t g = 0; g < e.gpus.size(); ++g) o.gpus[g] = e.gpus[g];
    }
    out->probes = r.probes;
    out->gpu_searches = r.st.searches;
    out->nodes = r.st.nodes;
    out->leaves = r.st.leaves;
}

void fill_plan(const PlanResult& p, mosaic_gpu_plan_result* out) {
    std::memset(out, 0, sizeof(*out));
    out->status = p.status;
    if (p.masks.size() > MOSAIC_GPU_MAX_STAGES) throw Error(MOSAIC_TOO_LARGE, "too many stages");
    out->n_stages = (int32_t)p.masks.size();
    for (size_t i = 0; i < p.masks.size(); ++i) {
        out->stage_mask[i] = p.masks[i];
        out->stage_time[i] = p.stages[i].stage_time;
    }
    out->iteration_time = p.iteration_time;
    out->partitions_examined = p.partitions;
    out->rounds = (int64_t)p.rounds.size();
    out->stage_eval_calls = p.stage_eval_calls;
    out->feasibility_calls = p.feasibility_calls;
    out->cache_hits = p.cache_hits;
    out->prunes = p.prunes;
    out->gpu_searches = p.st.searches;
    out->nodes = p.st.nodes;
    out->leaves = p.st.leaves;
    out->elapsed_s = p.elapsed;
}

Problem to_problem(const mosaic_gpu_problem* p) {
    if (!p) throw Error(MOSAIC_RANGE, "null problem");
    if (p->n_modules < 0 || p->n_modules > MOSAIC_GPU_MAX_MODULES)
        throw Error(MOSAIC_RANGE, "module count out of range");
    Problem P;
    for (int m = 0; m < p->n_modules; ++m) {
        const auto& src = p->modules[m];
        Module mod;
        mod.id = src.id ? src.id : "";
        mod.memory_base = src.memory_base;
        std::vector<Point> pts;
        for (int i = 0; i < src.n_points; ++i) {
            const auto& q = src.points[i];
            pts.push_back(Point{q.d, q.a, q.latency, q.bandwidth_util, q.memory, q.sm_active});
        }
        mod.surface = Surface(mod.id, pts);
        P.modules.push_back(std::move(mod));
    }
    for (int e = 0; e < p->n_edges; ++e) P.edges.push_back({p->edges[2 * e], p->edges[2 * e + 1]});
    P.gpu_count = p->gpu_count;
    if (P.gpu_count < 1 || P.gpu_count > MOSAIC_GPU_MAX_GPUS)
        throw Error(MOSAIC_RANGE, "gpu_count out of range");
    P.memory_capacity = p->memory_capacity;
    P.im.e1 = p->e1;
    P.im.e2 = p->e2;
    P.im.e3 = p->e3;
    P.im.additive_only = p->additive_only != 0;
    P.include_self = p->include_self != 0;
    P.quota_levels = p->quota_levels;
    if (P.quota_levels < 1) throw Error(MOSAIC_RANGE, "quota_levels must be >= 1");
    P.bisect_rel_tol = p->bisect_rel_tol;
    P.enable_prune = p->enable_prune != 0;
    P.enable_cache = p->enable_cache != 0;
    return P;
}

struct OwnedProblem {
    mosaic_gpu_problem p;  // must stay first
    std::vector<mosaic_gpu_module> mods;
    std::vector<std::vector<mosaic_gpu_point>> pts;
    std::vector<std::string> ids;
    std::vector<int32_t> edges;
};
}  // namespace

extern "C" {

const char* mosaic_gpu_last_error(void) { return g_err.c_str(); }

int mosaic_gpu_create(const mosaic_gpu_problem* p, int device, mosaic_gpu_ctx** out) {
    return guard([&] {
        auto ctx = std::make_unique<mosaic_gpu_ctx>();
        ctx->pl = std::make_unique<Planner>(to_problem(p), device);
        *out = ctx.release();
        return MOSAIC_OK;
    });
}

void mosaic_gpu_destroy(mosaic_gpu_ctx* ctx) { delete ctx; }

int mosaic_gpu_num_options(mosaic_gpu_ctx* ctx, int module, int32_t* n_out) {
    return guard([&] {
        if (module < 0 || module >= (int)ctx->pl->problem().modules.size())
            throw Error(MOSAIC_RANGE, "module index out of range");
        *n_out = (int32_t)ctx->pl->options(module).size();
        return MOSAIC_OK;
    });
}

int mosaic_gpu_options(mosaic_gpu_ctx* ctx, int module, int32_t* d, int32_t* units,
                       double* base_latency, double* solo_bandwidth, double* footprint) {
    return guard([&] {
        if (module < 0 || module >= (int)ctx->pl->problem().modules.size())
            throw Error(MOSAIC_RANGE, "module index out of range");
        const auto& o = ctx->pl->options(module);
        for (size_t i = 0; i < o.size(); ++i) {
            d[i] = o[i].d;
            units[i] = o[i].units;
            base_latency[i] = o[i].base;
            solo_bandwidth[i] = o[i].B;
            footprint[i] = o[i].fp;
        }
        return MOSAIC_OK;
    });
}

int mosaic_gpu_lookup(mosaic_gpu_ctx* ctx, int module, int d, double a, double out4[4]) {
    return guard([&] {
        if (module < 0 || module >= (int)ctx->pl->problem().modules.size())
            throw Error(MOSAIC_RANGE, "module index out of range");
        Sample s = ctx->pl->problem().modules[module].surface.lookup(d, a);
        out4[0] = s.latency;
        out4[1] = s.bandwidth_util;
        out4[2] = s.memory;
        out4[3] = s.sm_active;
        return MOSAIC_OK;
    });
}

int mosaic_gpu_stage_time(mosaic_gpu_ctx* ctx, const mosaic_gpu_eval_entry* entries,
                          const int32_t* gpus, const int64_t* alloc_off, int64_t n_allocs,
                          double* stage_time_out, double* rect_out) {
    return guard([&] {
        std::vector<std::vector<Entry>> allocs(n_allocs);
        for (int64_t i = 0; i < n_allocs; ++i) {
            for (int64_t e = alloc_off[i]; e < alloc_off[i + 1]; ++e) {
                const auto& E = entries[e];
                if (E.quota_levels < 0) throw Error(MOSAIC_RANGE, "quota_levels < 0");
                Entry x{E.module, E.dp_degree, E.quota_units, {}, E.quota_levels};
                x.gpus.assign(gpus + E.gpu_off, gpus + E.gpu_off + E.n_gpus);
                allocs[i].push_back(std::move(x));
            }
        }
        std::vector<double> st;
        std::vector<std::vector<double>> rect;
        ctx->pl->stage_time(allocs, st, rect);
        for (int64_t i = 0; i < n_allocs; ++i) {
            stage_time_out[i] = st[i];
            if (rect_out)
                for (int64_t e = alloc_off[i]; e < alloc_off[i + 1]; ++e)
                    rect_out[e] = rect[i][e - alloc_off[i]];
        }
        return MOSAIC_OK;
    });
}

int mosaic_gpu_evaluate(mosaic_gpu_ctx* ctx, const mosaic_gpu_eval_entry* entries,
                        int64_t n_entries, const int32_t* gpus, int64_t n_gpu_ids,
                        const int64_t* alloc_off, int64_t n_allocs, double* stage_time_out,
                        double* rect_out, uint32_t flags) {
    static_assert(sizeof(mosaic_gpu_eval_entry) == sizeof(mg::EvalABI), "entry layout");
    return guard([&] {
        if (!ctx) throw Error(MOSAIC_RANGE, "null context");
        if (n_allocs > 0 && (!entries && n_entries > 0)) throw Error(MOSAIC_RANGE, "null entries");
        if (n_allocs > 0 && (!alloc_off || !stage_time_out)) throw Error(MOSAIC_RANGE, "null array");
        ctx->pl->evaluate(reinterpret_cast<const mg::EvalABI*>(entries), n_entries, gpus,
                          n_gpu_ids, reinterpret_cast<const long long*>(alloc_off), n_allocs,
                          stage_time_out, rect_out, (flags & MOSAIC_EVAL_DEVICE) != 0);
        return MOSAIC_OK;
    });
}

int mosaic_gpu_evaluate_stats(mosaic_gpu_ctx* ctx, double* kernel_ms, int64_t* launches,
                              int64_t* alg_bytes) {
    return guard([&] {
        if (!ctx) throw Error(MOSAIC_RANGE, "null context");
        auto& e = ctx->pl->engine();
        if (kernel_ms) *kernel_ms = e.evaluate_kernel_ms();
        if (launches) *launches = e.evaluate_kernel_launches();
        if (alg_bytes) *alg_bytes = e.evaluate_alg_bytes();
        return MOSAIC_OK;
    });
}

int mosaic_gpu_smem_peak(int device, double* gbs_out) {
    return guard([&] {
        if (!gbs_out) throw Error(MOSAIC_RANGE, "null output");
        *gbs_out = mg::smem_peak_gbs(device, 5);
        return MOSAIC_OK;
    });
}

int mosaic_gpu_peer_links(mosaic_gpu_ctx* ctx) {
    if (!ctx) return 0;
    return ctx->pl->engine().peer_links();
}

int mosaic_gpu_evaluate_paths(mosaic_gpu_ctx* ctx, double* fast_kernel_ms,
                              int64_t* full_path_allocs) {
    return guard([&] {
        if (!ctx) throw Error(MOSAIC_RANGE, "null context");
        auto& e = ctx->pl->engine();
        if (fast_kernel_ms) *fast_kernel_ms = e.evaluate_fast_ms();
        if (full_path_allocs) *full_path_allocs = e.evaluate_fallback_allocs();
        return MOSAIC_OK;
    });
}

int mosaic_gpu_stage_eval(mosaic_gpu_ctx* ctx, uint64_t mask, mosaic_gpu_stage_result* out) {
    return guard([&] {
        StageResult r = ctx->pl->stage_eval(mask);
        fill_stage(r, out);
        return r.status;
    });
}

int mosaic_gpu_search(mosaic_gpu_ctx* ctx, const uint64_t* masks, int64_t n, int mode,
                      mosaic_gpu_stage_result* out, double* stage_time_out, int32_t* status_out) {
    return guard([&] {
        if (!ctx || (n > 0 && !masks)) throw Error(MOSAIC_RANGE, "null argument");
        if (mode != MOSAIC_SEARCH_STAGE_EVAL && mode != MOSAIC_SEARCH_EXACT)
            throw Error(MOSAIC_INVALID_ARGUMENT, "mode must be MOSAIC_SEARCH_STAGE_EVAL or _EXACT");
        std::vector<uint64_t> ms(masks, masks + n);
        std::vector<StageResult> rs = ctx->pl->stage_batch(ms, mode == MOSAIC_SEARCH_EXACT);
        for (int64_t i = 0; i < n; ++i) {
            if (out) fill_stage(rs[i], out + i);
            if (stage_time_out) stage_time_out[i] = rs[i].status == OK ? rs[i].stage_time : 0.0;
            if (status_out) status_out[i] = rs[i].status;
        }
        return MOSAIC_OK;
    });
}

int mosaic_gpu_exact_stage(mosaic_gpu_ctx* ctx, uint64_t mask, mosaic_gpu_stage_result* out) {
    return guard([&] {
        StageResult r = ctx->pl->exact_stage(mask);
        fill_stage(r, out);
        return r.status;
    });
}

int mosaic_gpu_feasible(mosaic_gpu_ctx* ctx, uint64_t mask, double tau,
                        mosaic_gpu_stage_result* out) {
    return guard([&] {
        StageResult r = ctx->pl->feasible(mask, tau);
        fill_stage(r, out);
        return r.status;
    });
}

int mosaic_gpu_stage_min(mosaic_gpu_ctx* ctx, uint64_t mask, double ub, int restart,
                         double* tstar, mosaic_gpu_stage_result* stats) {
    return guard([&] {
        StageResult r;
        *tstar = ctx->pl->stage_min(mask, ub, restart != 0, r.st);
        r.status = OK;
        r.stage_time = *tstar;
        if (stats) fill_stage(r, stats);
        return MOSAIC_OK;
    });
}

int mosaic_gpu_validate_plan(mosaic_gpu_ctx* ctx, const mosaic_gpu_eval_entry* entries,
                             const int32_t* gpus, const int64_t* stage_off, int64_t n_stages,
                             char* code_out, size_t code_cap) {
    return guard([&] {
        std::vector<std::vector<Entry>> st(n_stages);
        for (int64_t s = 0; s < n_stages; ++s)
            for (int64_t e = stage_off[s]; e < stage_off[s + 1]; ++e) {
                const auto& E = entries[e];
                if (E.quota_levels < 0) throw Error(MOSAIC_RANGE, "quota_levels < 0");
                Entry x{E.module, E.dp_degree, E.quota_units, {}, E.quota_levels};
                x.gpus.assign(gpus + E.gpu_off, gpus + E.gpu_off + E.n_gpus);
                st[s].push_back(std::move(x));
            }
        std::string msg;
        std::string code = ctx->pl->validate_plan(st, &msg);
        if (code.empty()) code = "Ok";
        std::snprintf(code_out, code_cap, "%s", code.c_str());
        g_err = msg;
        return MOSAIC_OK;
    });
}

int mosaic_gpu_cache_masks(mosaic_gpu_ctx* ctx, uint64_t* masks, int64_t cap, int64_t* n) {
    return guard([&] {
        const auto& o = ctx->pl->cache_order();
        if (n) *n = (int64_t)o.size();
        for (int64_t i = 0; masks && i < (int64_t)o.size() && i < cap; ++i) masks[i] = o[i];
        return MOSAIC_OK;
    });
}

int mosaic_gpu_cache_entry(mosaic_gpu_ctx* ctx, uint64_t mask, mosaic_gpu_stage_result* out,
                           double* probe_tau, int32_t* probe_ok, int64_t cap,
                           int64_t* n_probes) {
    return guard([&] {
        const StageResult* r = ctx->pl->cache_find(mask);
        if (!r) throw Error(MOSAIC_RANGE, "module set not in the EvalCache");
        if (out) fill_stage(*r, out);
        if (n_probes) *n_probes = (int64_t)r->probe_tau.size();
        for (int64_t i = 0; i < (int64_t)r->probe_tau.size() && i < cap; ++i) {
            if (probe_tau) probe_tau[i] = r->probe_tau[i];
            if (probe_ok) probe_ok[i] = r->probe_ok[i];
        }
        return MOSAIC_OK;
    });
}

int mosaic_gpu_plan_stage(mosaic_gpu_ctx* ctx, int stage, mosaic_gpu_stage_result* out) {
    return guard([&] {
        if (stage < 0 || stage >= (int)ctx->plan.stages.size())
            throw Error(MOSAIC_RANGE, "stage index out of range");
        fill_stage(ctx->plan.stages[stage], out);
        return MOSAIC_OK;
    });
}

int mosaic_gpu_solve(mosaic_gpu_ctx* ctx, mosaic_gpu_plan_result* out) {
    return guard([&] {
        ctx->plan = ctx->pl->solve();
        fill_plan(ctx->plan, out);
        return ctx->plan.status;
    });
}

int mosaic_gpu_baseline_plan(mosaic_gpu_ctx* ctx, int policy, mosaic_gpu_plan_result* out) {
    return guard([&] {
        if (policy != 0 && policy != 1) throw Error(MOSAIC_INVALID_ARGUMENT, "policy");
        ctx->plan = ctx->pl->baseline_plan(policy);
        fill_plan(ctx->plan, out);
        return ctx->plan.status;
    });
}

int mosaic_gpu_simulate(mosaic_gpu_ctx* ctx, const mosaic_gpu_eval_entry* entries,
                        const int32_t* gpus, const int64_t* stage_off, int64_t n_stages,
                        const mosaic_gpu_sim_config* cfg, const uint64_t* seeds,
                        int64_t n_seeds, double* iteration_time, double* per_stage,
                        double* busy, double* mean_busy, mosaic_gpu_interval* timeline,
                        int64_t timeline_cap, int64_t* n_timeline) {
    return guard([&] {
        std::vector<std::vector<Entry>> st(n_stages);
        for (int64_t s = 0; s < n_stages; ++s)
            for (int64_t e = stage_off[s]; e < stage_off[s + 1]; ++e) {
                const auto& E = entries[e];
                if (E.quota_levels < 0) throw Error(MOSAIC_RANGE, "quota_levels < 0");
                Entry x{E.module, E.dp_degree, E.quota_units, {}, E.quota_levels};
                x.gpus.assign(gpus + E.gpu_off, gpus + E.gpu_off + E.n_gpus);
                st[s].push_back(std::move(x));
            }
        mg::SimCfg c;
        c.iterations = cfg->iterations;
        c.on_demand = cfg->stream_mode != 0;
        c.pooled_overhead = cfg->pooled_overhead;
        c.on_demand_overhead = cfg->on_demand_overhead;
        c.sigma = cfg->perturbation_sigma;
        std::vector<uint64_t> sd(seeds, seeds + n_seeds);
        std::vector<double> it, ps, bz, mb;
        std::vector<mg::SimInterval> tl;
        ctx->pl->simulate(st, c, sd, it, ps, bz, mb, timeline || n_timeline ? &tl : nullptr);
        if (iteration_time) std::copy(it.begin(), it.end(), iteration_time);
        if (per_stage) std::copy(ps.begin(), ps.end(), per_stage);
        if (busy) std::copy(bz.begin(), bz.end(), busy);
        if (mean_busy) std::copy(mb.begin(), mb.end(), mean_busy);
        if (n_timeline) *n_timeline = (int64_t)tl.size();
        if (timeline)
            for (int64_t i = 0; i < (int64_t)tl.size() && i < timeline_cap; ++i)
                timeline[i] = mosaic_gpu_interval{tl[i].gpu, tl[i].module, tl[i].start,
                                                  tl[i].end, tl[i].quota};
        return MOSAIC_OK;
    });
}

int mosaic_gpu_brute_force(mosaic_gpu_ctx* ctx, mosaic_gpu_plan_result* out) {
    return guard([&] {
        ctx->plan = ctx->pl->brute_force();
        fill_plan(ctx->plan, out);
        return ctx->plan.status;
    });
}

int mosaic_gpu_trace_rounds(mosaic_gpu_ctx* ctx, int64_t* n_rounds) {
    *n_rounds = (int64_t)ctx->plan.rounds.size();
    return MOSAIC_OK;
}

int mosaic_gpu_trace_round(mosaic_gpu_ctx* ctx, int64_t r, uint64_t* chosen_x,
                           uint64_t* chosen_y, double* applied_gain, int64_t* n_cands) {
    return guard([&] {
        if (r < 0 || r >= (int64_t)ctx->plan.rounds.size()) throw Error(MOSAIC_RANGE, "round");
        const auto& R = ctx->plan.rounds[r];
        *chosen_x = R.chosen_x;
        *chosen_y = R.chosen_y;
        *applied_gain = R.applied_gain;
        *n_cands = (int64_t)R.cands.size();
        return MOSAIC_OK;
    });
}

int mosaic_gpu_trace_cand(mosaic_gpu_ctx* ctx, int64_t r, int64_t c, uint64_t* mask_x,
                          uint64_t* mask_y, int32_t* pruned, int32_t* cache_hit, double* gain) {
    return guard([&] {
        if (r < 0 || r >= (int64_t)ctx->plan.rounds.size()) throw Error(MOSAIC_RANGE, "round");
        const auto& R = ctx->plan.rounds[r];
        if (c < 0 || c >= (int64_t)R.cands.size()) throw Error(MOSAIC_RANGE, "candidate");
        const auto& C = R.cands[c];
        *mask_x = C.mask_x;
        *mask_y = C.mask_y;
        *pruned = C.pruned;
        *cache_hit = C.cache_hit;
        *gain = C.gain;
        return MOSAIC_OK;
    });
}

void mosaic_gpu_clear_cache(mosaic_gpu_ctx* ctx) { ctx->pl->clear_cache(); }

int mosaic_gpu_set_shard(mosaic_gpu_ctx* ctx, int rank, int world, mosaic_gpu_allgather_fn fn,
                         void* user) {
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world) throw Error(MOSAIC_RANGE, "bad rank/world");
        if (world > 1 && !fn) throw Error(MOSAIC_RANGE, "world > 1 needs an all-gather");
        ctx->rank = rank;
        ctx->world = world;
        ctx->pl->engine().set_shard(rank, world, fn, user);
        return MOSAIC_OK;
    });
}

int mosaic_gpu_set_tuning(mosaic_gpu_ctx* ctx, const char* key, double value) {
    return guard([&] {
        mg::Tuning& t = ctx->pl->engine().tuning();
        const std::string k = key ? key : "";
        const long long v = (long long)value;
        if (k == "don_depth") t.don_depth = (int)v;
        else if (k == "don_tail") t.don_tail = (int)v;
        else if (k == "don_depth_small") t.don_depth_small = (int)v;
        else if (k == "don_depth_first") t.don_depth_first = (int)v;
        else if (k == "don_tail_first") t.don_tail_first = (int)v;
        else if (k == "tail_idle") t.tail_idle = (int)v;
        else if (k == "tail_after") t.tail_after = (long long)v;
        else if (k == "don_min_rest") t.don_min_rest = (int)v;
        else if (k == "local_handover") t.local_handover = (int)v;
        else if (k == "min_order") t.min_order = (int)v;
        else if (k == "min_perm") t.min_perm = (long long)v;
        else if (k == "fuse_k") t.fuse_k = (int)v;
        else if (k == "don_period_small") {
            if (v < 1 || ((long long)v & ((long long)v - 1))) throw Error(MOSAIC_INVALID_ARGUMENT, "don_period_small must be a power of two");
            t.don_period_small = (int)v;
        }
        else if (k == "fuse_tree") t.fuse_tree = v;
        else if (k == "share_all") t.share_all = (int)v;
        else if (k == "share_peers") t.share_peers = (int)v;
        else if (k == "don_period") {
            if (v < 1 || (v & (v - 1))) throw Error(MOSAIC_INVALID_ARGUMENT, "don_period: power of two");
            t.don_period = (int)v;
        } else if (k == "backoff_ns") t.backoff_cap = (int)v;
        else if (k == "small_tree") t.small_tree = value;
        else if (k == "deep_after") t.deep_after = v;
        else if (k == "lookahead") t.lookahead = (int)v;
        else if (k == "generic_kernel") t.generic_kernel = v != 0;
        else if (k == "shard_level") t.shard_level = (int)v;
        else if (k == "ring_per_walker") t.ring_per_walker = (int)std::max(1LL, v);
        else if (k == "trace") t.trace = (int)v;  // 1 per search, 2 per launch
        else if (k == "spec_k") t.spec_k = (int)v;
        else if (k == "restart_k") t.restart_k = (int)v;
        else if (k == "share_rank") t.share_rank = (int)v;
        else if (k == "share_world") t.share_world = (int)std::max(1LL, v);
        else throw Error(MOSAIC_INVALID_ARGUMENT, "unknown tuning key " + k);
        return MOSAIC_OK;
    });
}

int64_t mosaic_gpu_device_bytes(mosaic_gpu_ctx* ctx) { return ctx->pl->engine().device_bytes(); }

int mosaic_gpu_nccl_id(void* id_out, size_t cap) {
    return guard([&] {
        if (!id_out || cap < mg::nccl_id_bytes())
            throw Error(MOSAIC_INVALID_ARGUMENT, "id buffer smaller than NCCL_UNIQUE_ID_BYTES");
        mg::nccl_unique_id(id_out);
        return MOSAIC_OK;
    });
}

int mosaic_gpu_set_shard_nccl(mosaic_gpu_ctx* ctx, int rank, int world, const void* nccl_id) {
    return guard([&] {
        if (!ctx || !nccl_id) throw Error(MOSAIC_RANGE, "null argument");
        ctx->pl->engine().set_shard_nccl(rank, world, nccl_id);
        ctx->rank = rank;
        ctx->world = world;
        return MOSAIC_OK;
    });
}

size_t mosaic_gpu_rank_record_size(void) { return sizeof(mg::RankRecord); }

int mosaic_gpu_rank_record(void* rec, int has_hit, int aborted, int overflow, double inc, int k,
                           const uint16_t* opt, const uint16_t* nb, const uint16_t* x,
                           double leaf_value) {
    return guard([&] {
        if (!rec || k < 0 || k > mg::MAXK) throw Error(MOSAIC_RANGE, "bad record arguments");
        mg::RankRecord& r = *static_cast<mg::RankRecord*>(rec);
        std::memset(&r, 0, sizeof r);
        r.has_hit = has_hit;
        r.aborted = aborted;
        r.overflow = overflow;
        r.inc = inc;
        for (int l = 0; l < k; ++l) {
            r.path.opt[l] = opt ? opt[l] : 0;
            r.path.nb[l] = nb ? nb[l] : 0;
            if (nb && nb[l] > mg::MAXB) throw Error(MOSAIC_RANGE, "too many blocks");
            for (int b = 0; nb && x && b < nb[l]; ++b) r.path.x[l][b] = x[l * mg::MAXB + b];
            r.leaf.opt[l] = r.path.opt[l];
        }
        r.leaf.value = leaf_value;
        return MOSAIC_OK;
    });
}

int mosaic_gpu_merge_ranks(const void* records, int world, int mode, int k, int* winner,
                           int* found, double* value, int* aborted, int* overflow,
                           double* leaf_value) {
    return guard([&] {
        if (!records || world < 1) throw Error(MOSAIC_RANGE, "bad records");
        mg::SearchResult res;
        const int w = mg::merge_rank_records(static_cast<const mg::RankRecord*>(records), world,
                                             mode, k, res);
        if (winner) *winner = w;
        if (found) *found = res.found ? 1 : 0;
        if (value) *value = res.value;
        if (aborted) *aborted = res.aborted ? 1 : 0;
        if (overflow) *overflow = res.overflow ? 1 : 0;
        if (leaf_value) *leaf_value = res.found ? res.leaf.value : 0.0;
        return MOSAIC_OK;
    });
}

int64_t mosaic_gpu_launch_count(mosaic_gpu_ctx* ctx) { return ctx->pl->engine().launches(); }
double mosaic_gpu_search_ms(mosaic_gpu_ctx* ctx) {
    return ctx->pl->engine().search_ms() + ctx->pl->engine().eval_ms();
}
void mosaic_gpu_reset_counters(mosaic_gpu_ctx* ctx) { ctx->pl->engine().reset_counters(); }
int64_t mosaic_gpu_own_launches(mosaic_gpu_ctx* ctx) { return ctx->pl->engine().own_launches(); }
double mosaic_gpu_ksearch_ms(mosaic_gpu_ctx* ctx) { return ctx->pl->engine().ksearch_ms(); }
int64_t mosaic_gpu_ksearch_launches(mosaic_gpu_ctx* ctx) {
    return ctx->pl->engine().ksearch_launches();
}
int64_t mosaic_gpu_h2d_bytes(mosaic_gpu_ctx* ctx) { return ctx->pl->engine().h2d_bytes(); }
int64_t mosaic_gpu_d2h_bytes(mosaic_gpu_ctx* ctx) { return ctx->pl->engine().d2h_bytes(); }
int64_t mosaic_gpu_alg_bytes(mosaic_gpu_ctx* ctx) { return ctx->pl->engine().alg_bytes(); }
void mosaic_gpu_mark(mosaic_gpu_ctx* ctx, int which) {
    try {
        ctx->pl->engine().mark(which);
    } catch (...) {
    }
}
double mosaic_gpu_marked_ms(mosaic_gpu_ctx* ctx) {
    try {
        return ctx->pl->engine().marked_ms();
    } catch (...) {
        return -1.0;
    }
}

int mosaic_gpu_generate_surfaces(const mosaic_gpu_workload* workloads, int32_t n,
                                 const mosaic_gpu_cluster* cluster, const int32_t* d_set,
                                 int32_t nd, const double* a_set, int32_t na,
                                 double demand_scale, int device, mosaic_gpu_point* out,
                                 int32_t* nd_out, int32_t* na_out) {
    return guard([&] {
        std::vector<int> ds;
        std::vector<double> as;
        if (d_set) {
            ds.assign(d_set, d_set + nd);
        } else {
            for (int d = 1; d <= cluster->gpu_count; d *= 2) ds.push_back(d);  // :44-48
        }
        if (a_set) {
            as.assign(a_set, a_set + na);
        } else {
            for (int i = 1; i <= 10; ++i) as.push_back(i / 10.0);  // :50-54
        }
        if (nd_out) *nd_out = (int32_t)ds.size();
        if (na_out) *na_out = (int32_t)as.size();
        if (!out) return MOSAIC_OK;
        std::vector<mg::GenWorkload> ws(n);
        for (int i = 0; i < n; ++i) {
            const auto& w = workloads[i];
            ws[i] = mg::GenWorkload{w.flops_per_iter,    w.bytes_per_iter,   w.gradient_bytes,
                                    w.sm_efficiency_knee, w.memory_act_base, w.memory_per_quota,
                                    w.fixed_overhead,     w.dp_penalty};
        }
        mg::GenCluster c{cluster->peak_compute, cluster->peak_bandwidth,
                         cluster->interconnect_alpha, cluster->interconnect_beta};
        auto pts = mg::generate_surfaces_device(ws, c, ds, as, demand_scale, device);
        for (size_t i = 0; i < pts.size(); ++i)
            out[i] = mosaic_gpu_point{pts[i].d, pts[i].a, pts[i].latency, pts[i].bandwidth_util,
                                      pts[i].memory, pts[i].sm_active};
        return MOSAIC_OK;
    });
}

int mosaic_gpu_synth_workloads(const char* spec, mosaic_gpu_workload* out, int32_t cap,
                               int32_t* n, mosaic_gpu_cluster* cluster) {
    return guard([&] {
        Cluster c;
        auto ws = synth_workloads(spec ? spec : "", &c, nullptr);
        *n = (int32_t)ws.size();
        for (int i = 0; i < (int)ws.size() && i < cap; ++i)
            out[i] = mosaic_gpu_workload{nullptr,      ws[i].flops,     ws[i].bytes,
                                         ws[i].grad,   ws[i].knee,      ws[i].act_base,
                                         ws[i].mem_per_quota, ws[i].fixed, ws[i].dp_penalty};
        if (cluster)
            *cluster = mosaic_gpu_cluster{c.gpu_count, c.memory_capacity, c.peak_compute,
                                          c.peak_bandwidth, c.alpha, c.beta};
        return MOSAIC_OK;
    });
}

int mosaic_gpu_synth_problem(const char* spec, int quota_levels, mosaic_gpu_problem** out) {
    return guard([&] {
        Problem P = synth_problem(spec ? spec : "", quota_levels);
        auto op = std::make_unique<OwnedProblem>();
        std::memset(&op->p, 0, sizeof(op->p));
        op->ids.reserve(P.modules.size());
        for (auto& m : P.modules) {
            op->ids.push_back(m.id);
            // re-emit the surface grid from the reference generator's own points
            std::vector<mosaic_gpu_point> pts;
            for (double dv : m.surface.d_values())
                for (int i = 1; i <= 10; ++i) {
                    double a = i / 10.0;
                    Sample s = m.surface.lookup((int)dv, a);
                    pts.push_back(mosaic_gpu_point{(int32_t)dv, a, s.latency, s.bandwidth_util,
                                                   s.memory, s.sm_active});
                }
            op->pts.push_back(std::move(pts));
        }
        for (size_t i = 0; i < P.modules.size(); ++i)
            op->mods.push_back(mosaic_gpu_module{op->ids[i].c_str(), P.modules[i].memory_base,
                                                 op->pts[i].data(), (int32_t)op->pts[i].size()});
        for (auto [u, v] : P.edges) {
            op->edges.push_back(u);
            op->edges.push_back(v);
        }
        op->p.modules = op->mods.data();
        op->p.n_modules = (int32_t)op->mods.size();
        op->p.edges = op->edges.data();
        op->p.n_edges = (int32_t)P.edges.size();
        op->p.gpu_count = P.gpu_count;
        op->p.memory_capacity = P.memory_capacity;
        op->p.e1 = P.im.e1;
        op->p.e2 = P.im.e2;
        op->p.e3 = P.im.e3;
        op->p.additive_only = 0;
        op->p.include_self = 1;
        op->p.quota_levels = P.quota_levels;
        op->p.bisect_rel_tol = 1e-3;
        op->p.enable_prune = 1;
        op->p.enable_cache = 1;
        *out = &op.release()->p;
        return MOSAIC_OK;
    });
}

void mosaic_gpu_free_problem(mosaic_gpu_problem* p) { delete reinterpret_cast<OwnedProblem*>(p); }

}  // extern "C"
