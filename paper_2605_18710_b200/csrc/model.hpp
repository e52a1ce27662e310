// model.hpp — host-side domain model: module graph, scaling surfaces, candidate-option
// packing, and the synthetic profiler that produces the BASELINE inputs.
//
// Everything here runs once per problem (not per candidate plan); it produces the flat
// option tables the device searches.  Arithmetic is restated operation-for-operation
// from the reference so the packed tables are bit-identical (compile with
// -ffp-contract=off, no -march=native):
//   ScalingSurface ctor/lookup/bracket   perf_model.hpp:57-79, 124-147, 155-194
//   candidate_options                    stage_eval.hpp:68-93 (on the device: pack.cu)
//   evaluate_workload/generate_surfaces  profiler.hpp:57-111
//   make_workload/make_spec/presets      profiler.hpp:185-285
//   random_instance                      profiler.hpp:304-338
//   validate_graph/topological_order/reachability_masks  core.hpp:151-261
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace mosaic_b200 {

struct RangeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Point {
    int d = 1;
    double a = 1.0, latency = 0.0, bandwidth_util = 0.0, memory = 0.0, sm_active = 1.0;
};

struct Sample {
    double latency, bandwidth_util, memory, sm_active;
};

class Surface {
  public:
    Surface() = default;
    Surface(std::string id, const std::vector<Point>& pts);
    Sample lookup(int d, double a) const;
    // Dense evaluator rows: lat[(d-1)*(L+1)+u] = lookup(d, u/L).latency for d = 1..G and
    // bw[u] = lookup(1, u/L).bandwidth_util (PerfContext::base_latency / solo_bandwidth,
    // perf_model.hpp:417-427); NaN where lookup would raise SurfaceRangeError.  Same
    // brackets and blend as lookup(), evaluated once per axis value.
    void rate_tables(int G, int L, double* lat, double* bw) const;
    const std::vector<double>& d_values() const { return dv_; }
    const std::vector<double>& a_values() const { return av_; }
    const std::vector<Point>& grid() const { return grid_; }  // [di * |a| + ai]
    double min_a() const { return av_.front(); }
    double max_a() const { return av_.back(); }
    int min_d() const { return (int)dv_.front(); }
    int max_d() const { return (int)dv_.back(); }
    const std::string& id() const { return id_; }

  private:
    const Point& at(size_t di, size_t ai) const { return grid_[di * av_.size() + ai]; }
    std::string id_;
    std::vector<double> dv_, av_;
    std::vector<Point> grid_;
};

struct Module {
    std::string id;
    double memory_base = 0.0;
    Surface surface;
};

struct Interference {
    double e1 = 0, e2 = 0, e3 = 0;
    bool additive_only = false;
    bool non_negative() const { return e1 >= 0 && e2 >= 0 && (additive_only || e3 >= 0); }
    double delta(double s, double p) const { return e1 + e2 * s + (additive_only ? 0.0 : e3 * p); }
};

struct Problem {
    std::vector<Module> modules;
    std::vector<std::pair<int, int>> edges;  // (upstream, downstream) indices
    int gpu_count = 1;
    double memory_capacity = 80e9;
    Interference im;
    bool include_self = true;
    int quota_levels = 10;
    double bisect_rel_tol = 1e-3;
    bool enable_prune = true, enable_cache = true;
};

struct Cand {  // CandidateOption (stage_eval.hpp:58-63)
    int d, units;
    double base, B, fp;
};


// core.hpp helpers
std::string validate_graph(const Problem& P);  // "" when valid
std::vector<int> topological_order(const Problem& P);
std::vector<uint64_t> reachability_masks(const Problem& P);

// ---- synthetic inputs (profiler.hpp) ----
struct Workload {
    std::string id;
    double flops = 0, bytes = 0, grad = 0, knee = 0.5, act_base = 1e9, mem_per_quota = 2e9,
           fixed = 0, dp_penalty = 0;
};
struct Cluster {
    int gpu_count = 1;
    double memory_capacity = 80e9, peak_compute = 500e12, peak_bandwidth = 3.35e12,
           alpha = 5e-6, beta = 2.2e-12;
};
Workload make_workload(const std::string& id, double tflops, double ci, double params_b,
                       double knee, double batch_scale = 64.0);
Point evaluate_workload(const Workload& w, const Cluster& c, int d, double a);
Surface generate_surface(const Workload& w, const Cluster& c);
// spec: cfg1..cfg5 | random:SEED:N:G | preset:NAME:COUNT:G  -> problem with the
// default ground-truth interference (bench.hpp:31-37)
Problem synth_problem(const std::string& spec, int quota_levels_override = 0);
// the workloads (in module order) and cluster a spec is generated from; *L = its quota levels
std::vector<Workload> synth_workloads(const std::string& spec, Cluster* c, int* L);

}  // namespace mosaic_b200
