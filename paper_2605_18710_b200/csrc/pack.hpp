// pack.hpp — device packing of candidate-option tables (pack.cu).
#pragma once
#include <vector>

namespace mg {

constexpr int PACK_MAXD = 16;  // d grid values per surface
constexpr int PACK_MAXA = 64;  // a grid values per surface

struct PackInput {  // one module's surface grid, axes ascending, grid[di * na + ai]
    std::vector<double> dv, av, lat, bw, mem;
    double membase = 0.0;
};

struct PackedRow {  // CandidateOption (stage_eval.hpp:58-63)
    int d, u;
    double base, B, fp;
};

// candidate_options for every module, computed by k_pack_options.  range_err[m] = 1 when
// module m's surface cannot answer the d = 1 lookup (the reference's SurfaceRangeError).
std::vector<std::vector<PackedRow>> pack_options_device(const std::vector<PackInput>& mods, int G,
                                                        int L, double cap, int device,
                                                        long long* h2d_bytes,
                                                        std::vector<int>* range_err);

struct GenWorkload {  // ModuleWorkload (profiler.hpp:26-40)
    double flops, bytes, grad, knee, act_base, mem_per_quota, fixed, dp_penalty;
};
struct GenCluster {  // the ClusterSpec fields evaluate_workload reads (core.hpp:52-59)
    double peak_compute, peak_bandwidth, alpha, beta;
};
struct GenPoint {
    int d;
    double a, latency, bandwidth_util, memory, sm_active;
};

// generate_surface (profiler.hpp:94-101) for every workload on the device: out[(w * nd + di)
// * na + ai] = evaluate_workload(w, cluster, d_set[di], a_set[ai]) (profiler.hpp:65-89).
std::vector<GenPoint> generate_surfaces_device(const std::vector<GenWorkload>& ws,
                                               const GenCluster& c, const std::vector<int>& d_set,
                                               const std::vector<double>& a_set,
                                               double demand_scale, int device);

}  // namespace mg
