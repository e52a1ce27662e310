// TEST INFRASTRUCTURE ONLY.  The BASELINE configs and the reference's own random / preset
// instances, built with the UNMODIFIED reference headers (profiler.hpp) — shared by
// ref_driver.cpp and the reference-side shim test (tests/shim/test_shim.cpp).
#pragma once
#include <cstdio>
#include <string>
#include <vector>

#include "mosaic/bench.hpp"
#include "mosaic/profiler.hpp"

namespace mosaic_ref {
using namespace mosaic;

struct Instance {
    std::string name;
    ModelGraph graph;
    std::vector<ModuleWorkload> workloads;
    ClusterSpec cluster;
    int levels = 10;
    InterferenceModel im = default_ground_truth();
    bool include_self = true;
    SurfaceSet surfaces;
    PerfContext ctx;

    void finish() {
        surfaces = generate_surfaces(workloads, cluster);
        ctx.graph = &graph;
        ctx.surfaces = &surfaces;
        ctx.interference = im;
        ctx.include_self = include_self;
    }
};

inline void add(Instance& in, const ModuleWorkload& w) {
    in.workloads.push_back(w);
    in.graph.modules.push_back(detail::make_spec(w, w.id));
}

// The five BASELINE configs.
inline bool make_config(const std::string& name, Instance& in) {
    using detail::make_workload;
    in.name = name;
    if (name == "cfg1") {
        add(in, make_workload("vision", 4.17, 35.2, 0.30, 0.60));
        add(in, make_workload("text", 1.04, 20.5, 0.12, 0.45));
        in.cluster.gpu_count = 8;
        in.levels = 10;
    } else if (name == "cfg2") {
        add(in, make_workload("vit", 4.17, 35.2, 0.30, 0.60));
        add(in, make_workload("proj", 0.05, 4.0, 0.02, 0.30));
        add(in, make_workload("llm", 22.27, 145.2, 7.00, 0.80));
        in.graph.edges = {{"vit", "proj"}, {"proj", "llm"}};
        in.cluster.gpu_count = 16;
        in.levels = 8;
    } else if (name == "cfg3") {
        add(in, make_workload("vision", 2.58, 82.4, 0.60, 0.70));
        add(in, make_workload("text", 0.15, 2.1, 0.05, 0.30));
        add(in, make_workload("deepstack", 0.30, 6.0, 0.05, 0.35));
        add(in, make_workload("llm", 22.27, 145.2, 7.00, 0.80));
        in.graph.edges = {{"vision", "deepstack"}, {"deepstack", "llm"}, {"text", "llm"}};
        in.cluster.gpu_count = 32;
        in.levels = 10;
    } else if (name == "cfg4") {
        add(in, make_workload("image", 4.17, 35.2, 0.30, 0.60));
        add(in, make_workload("video", 1.80, 22.0, 0.35, 0.60));
        add(in, make_workload("audio", 2.09, 22.8, 0.25, 0.50));
        add(in, make_workload("llm", 16.70, 110.5, 3.20, 0.80));
        add(in, make_workload("speech_dec", 0.95, 14.8, 0.20, 0.50));
        add(in, make_workload("image_dec", 1.48, 24.6, 0.25, 0.55));
        in.graph.edges = {{"image", "llm"},      {"video", "llm"},
                          {"audio", "llm"},      {"llm", "speech_dec"},
                          {"llm", "image_dec"}};
        in.cluster.gpu_count = 64;
        in.levels = 10;
    } else if (name == "cfg5") {
        auto p = make_preset("ofasys", 8);
        in.graph = p.graph;
        in.workloads = p.workloads;
        in.cluster.gpu_count = 128;
        in.levels = 32;
    } else {
        return false;
    }
    return true;
}

// inst spec: cfgN | random:SEED:N:G | preset:NAME:COUNT:G
inline bool make_instance(const std::string& spec, Instance& in) {
    if (make_config(spec, in)) return true;
    char kind[32] = {0}, a[64] = {0};
    if (spec.rfind("random:", 0) == 0) {
        unsigned long long seed;
        int n, g;
        if (std::sscanf(spec.c_str(), "random:%llu:%d:%d", &seed, &n, &g) != 3) return false;
        auto r = random_instance(seed, n, g);
        in.name = spec;
        in.graph = r.graph;
        in.workloads = r.workloads;
        in.cluster = r.cluster;
        return true;
    }
    if (spec.rfind("preset:", 0) == 0) {
        int count, g;
        if (std::sscanf(spec.c_str(), "preset:%31[^:]:%d:%d", a, &count, &g) != 3) return false;
        auto p = make_preset(a, count);
        in.name = spec;
        in.graph = p.graph;
        in.workloads = p.workloads;
        in.cluster.gpu_count = g;
        return true;
    }
    (void)kind;
    return false;
}


}  // namespace mosaic_ref
