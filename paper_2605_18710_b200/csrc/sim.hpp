// sim.hpp — batched plan replay on the device (sim.cu).
#pragma once
#include <cstdint>
#include <vector>

namespace mg {

struct SimEntry {       // one stage entry of the replayed plan
    double dur0;        // rectified_latency (perf_model.hpp:442-464), computed by k_eval
    double quota;       // option.quota()
    double active_cap;  // sm_active * latency of lookup(d, quota) (simulator.hpp:96-98)
    int module, gpu_off, n_gpus, pad;
};

struct SimCfg {  // SimConfig (simulator.hpp:28-35)
    int iterations = 1;
    int on_demand = 0;
    double pooled_overhead = 0.013e-3;
    double on_demand_overhead = 37e-3;
    double sigma = 0.0;
};

struct SimInterval {  // TimelineInterval (simulator.hpp:37-43)
    int gpu, module;
    double start, end, quota;
};

// simulate (simulator.hpp:68-119) for every seed in `seeds`, one device thread per seed.
// Outputs are indexed [seed], [seed * n_stages + s], [seed * G + r]; the timeline is the
// first iteration of seeds[0].
void simulate_device(const std::vector<SimEntry>& ents, const std::vector<int>& gpus,
                     const std::vector<int>& stage_off, int G, const SimCfg& cfg,
                     const std::vector<uint64_t>& seeds, int device, std::vector<double>& iter,
                     std::vector<double>& per_stage, std::vector<double>& busy,
                     std::vector<double>& mean_busy, std::vector<SimInterval>* timeline);

}  // namespace mg
