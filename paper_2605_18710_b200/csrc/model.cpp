// model.cpp — see model.hpp.  Compiled with -ffp-contract=off.
#include "model.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <map>
#include <random>
#include <set>
#include <tuple>

namespace mosaic_b200 {

namespace {
constexpr double kTol = 1e-12;  // kAxisTolerance, perf_model.hpp:50

void axis_insert(std::vector<double>& ax, double v) {
    for (double x : ax)
        if (std::abs(x - v) <= kTol) return;
    ax.insert(std::lower_bound(ax.begin(), ax.end(), v), v);
}

size_t axis_index(const std::vector<double>& ax, double v) {
    for (size_t i = 0; i < ax.size(); ++i)
        if (std::abs(ax[i] - v) <= kTol) return i;
    throw RangeError("value not on grid");
}

// (lo, hi, weight toward hi); log2 scale on the d axis (perf_model.hpp:174-192)
std::tuple<size_t, size_t, double> bracket(const std::vector<double>& ax, double v, bool log2s) {
    for (size_t i = 0; i < ax.size(); ++i)
        if (std::abs(ax[i] - v) <= kTol * std::max(1.0, std::abs(v))) return {i, i, 0.0};
    size_t hi = std::upper_bound(ax.begin(), ax.end(), v) - ax.begin();
    size_t lo = hi - 1;
    auto sc = [&](double x) { return log2s ? std::log2(x) : x; };
    double w = (sc(v) - sc(ax[lo])) / (sc(ax[hi]) - sc(ax[lo]));
    return {lo, hi, w};
}
}  // namespace

Surface::Surface(std::string id, const std::vector<Point>& pts) : id_(std::move(id)) {
    for (const auto& p : pts) {
        if (p.latency <= 0) throw RangeError("surface latency must be > 0");
        if (p.bandwidth_util < 0 || p.bandwidth_util > 1)
            throw RangeError("bandwidth_util must be in [0,1]");
        if (p.memory <= 0) throw RangeError("surface memory must be > 0");
        if (p.sm_active < 0 || p.sm_active > 1) throw RangeError("sm_active must be in [0,1]");
        axis_insert(dv_, (double)p.d);
        axis_insert(av_, p.a);
    }
    if (dv_.empty()) throw RangeError("empty surface for " + id_);
    grid_.assign(dv_.size() * av_.size(), Point{});
    std::vector<char> filled(grid_.size(), 0);
    for (const auto& p : pts) {
        size_t idx = axis_index(dv_, p.d) * av_.size() + axis_index(av_, p.a);
        if (filled[idx]) throw RangeError("duplicate surface point");
        grid_[idx] = p;
        filled[idx] = 1;
    }
    for (char f : filled)
        if (!f) throw RangeError("incomplete surface grid for " + id_);
}

Sample Surface::lookup(int d, double a) const {
    if (d < min_d() || d > max_d())
        throw RangeError(id_ + ": d=" + std::to_string(d) + " outside profiled range");
    if (a < min_a() - kTol || a > max_a() + kTol)
        throw RangeError(id_ + ": a=" + std::to_string(a) + " outside profiled range");
    auto [dlo, dhi, wd] = bracket(dv_, (double)d, true);
    auto [alo, ahi, wa] = bracket(av_, a, false);
    if (dlo == dhi && alo == ahi) {
        const Point& p = at(dlo, alo);
        return Sample{p.latency, p.bandwidth_util, p.memory, p.sm_active};
    }
    auto blend = [&](double Point::*f) {
        double v00 = at(dlo, alo).*f, v01 = at(dlo, ahi).*f;
        double v10 = at(dhi, alo).*f, v11 = at(dhi, ahi).*f;
        double lo = v00 + (v01 - v00) * wa;
        double hi = v10 + (v11 - v10) * wa;
        return lo + (hi - lo) * wd;
    };
    return Sample{blend(&Point::latency), blend(&Point::bandwidth_util), blend(&Point::memory),
                  blend(&Point::sm_active)};
}

void Surface::rate_tables(int G, int L, double* lat, double* bw) const {
    const double nan = std::numeric_limits<double>::quiet_NaN();
    struct Br {
        bool ok;
        size_t lo, hi;
        double w;
    };
    std::vector<Br> ab(L + 1);
    for (int u = 0; u <= L; ++u) {
        const double a = static_cast<double>(u) / L;  // DeploymentOption::quota()
        ab[u].ok = !(a < min_a() - kTol || a > max_a() + kTol);
        if (ab[u].ok) std::tie(ab[u].lo, ab[u].hi, ab[u].w) = bracket(av_, a, false);
    }
    auto blend = [&](const Br& D, const Br& A, double Point::*f) {
        if (D.lo == D.hi && A.lo == A.hi) return at(D.lo, A.lo).*f;
        double v00 = at(D.lo, A.lo).*f, v01 = at(D.lo, A.hi).*f;
        double v10 = at(D.hi, A.lo).*f, v11 = at(D.hi, A.hi).*f;
        double lo = v00 + (v01 - v00) * A.w;
        double hi = v10 + (v11 - v10) * A.w;
        return lo + (hi - lo) * D.w;
    };
    for (int d = 1; d <= G; ++d) {
        Br D{!(d < min_d() || d > max_d()), 0, 0, 0.0};
        if (D.ok) std::tie(D.lo, D.hi, D.w) = bracket(dv_, (double)d, true);
        for (int u = 0; u <= L; ++u)
            lat[(size_t)(d - 1) * (L + 1) + u] =
                D.ok && ab[u].ok ? blend(D, ab[u], &Point::latency) : nan;
        if (d == 1)
            for (int u = 0; u <= L; ++u)
                bw[u] = D.ok && ab[u].ok ? blend(D, ab[u], &Point::bandwidth_util) : nan;
    }
}

std::string validate_graph(const Problem& P) {
    std::set<std::string> seen;
    for (const auto& m : P.modules)
        if (!seen.insert(m.id).second) return "duplicate module id: " + m.id;
    const int n = (int)P.modules.size();
    std::set<std::pair<int, int>> es;
    for (auto [u, v] : P.edges) {
        if (u < 0 || u >= n || v < 0 || v >= n) return "edge references unknown module";
        if (u == v) return "self edge on " + P.modules[u].id;
        if (!es.insert({u, v}).second) return "duplicate edge";
    }
    // cycle check (Kahn)
    std::vector<int> indeg(n, 0);
    std::vector<std::vector<int>> adj(n);
    for (auto [u, v] : P.edges) {
        adj[u].push_back(v);
        ++indeg[v];
    }
    std::vector<int> st;
    for (int i = 0; i < n; ++i)
        if (!indeg[i]) st.push_back(i);
    int seen_n = 0;
    while (!st.empty()) {
        int u = st.back();
        st.pop_back();
        ++seen_n;
        for (int v : adj[u])
            if (--indeg[v] == 0) st.push_back(v);
    }
    if (seen_n != n) return "cycle detected";
    return "";
}

std::vector<int> topological_order(const Problem& P) {
    const int n = (int)P.modules.size();
    std::vector<int> indeg(n, 0);
    std::vector<std::vector<int>> adj(n);
    for (auto [u, v] : P.edges) {
        adj[u].push_back(v);
        ++indeg[v];
    }
    auto cmp = [&](int a, int b) { return P.modules[a].id < P.modules[b].id; };
    std::vector<int> ready;
    for (int i = 0; i < n; ++i)
        if (!indeg[i]) ready.push_back(i);
    std::sort(ready.begin(), ready.end(), cmp);
    std::vector<int> order;
    while (!ready.empty()) {
        int u = ready.front();
        ready.erase(ready.begin());
        order.push_back(u);
        for (int v : adj[u])
            if (--indeg[v] == 0) ready.insert(std::lower_bound(ready.begin(), ready.end(), v, cmp), v);
    }
    return order;
}

std::vector<uint64_t> reachability_masks(const Problem& P) {
    const int n = (int)P.modules.size();
    if (n > 64) throw RangeError("reachability_masks: more than 64 modules");
    std::vector<std::vector<int>> adj(n);
    for (auto [u, v] : P.edges) adj[u].push_back(v);
    std::vector<uint64_t> reach(n, 0);
    auto order = topological_order(P);
    for (auto it = order.rbegin(); it != order.rend(); ++it)
        for (int v : adj[*it]) reach[*it] |= (uint64_t(1) << v) | reach[v];
    return reach;
}

// ---------------------------------------------------------------------------
// synthetic profiler
// ---------------------------------------------------------------------------
Workload make_workload(const std::string& id, double tflops, double ci, double params_b,
                       double knee, double batch_scale) {
    Workload w;
    w.id = id;
    w.flops = tflops * 1e12 * batch_scale;
    w.bytes = w.flops / ci;
    w.grad = params_b * 1e9 * 2.0;
    w.knee = knee;
    w.act_base = 1e9 + params_b * 1e9;
    w.mem_per_quota = 2e9 + 0.2e9 * tflops;
    w.fixed = 40e-3;
    w.dp_penalty = 0.02;
    return w;
}

Point evaluate_workload(const Workload& w, const Cluster& c, int d, double a) {
    double eta = std::min(1.0, 0.85 + 0.15 * a / w.knee);
    double compute_time = (w.flops / d) / (a * c.peak_compute * eta);
    double io_time = (w.bytes / d) / c.peak_bandwidth;
    double sync_time = 0.0;
    if (d > 1) sync_time = c.alpha * std::ceil(std::log2(double(d))) + c.beta * w.grad;
    Point p;
    p.d = d;
    p.a = a;
    double dp_eff = 1.0 + w.dp_penalty * (d - 1);
    p.latency = std::max(compute_time, io_time) * dp_eff + sync_time + w.fixed;
    p.sm_active = std::min(1.0, compute_time / p.latency);
    p.bandwidth_util = std::min(1.0, io_time / std::max(compute_time, io_time) * 1.0);
    p.memory = w.act_base + w.mem_per_quota * a + w.grad / d;
    return p;
}

Surface generate_surface(const Workload& w, const Cluster& c) {
    std::vector<Point> pts;
    for (int d = 1; d <= c.gpu_count; d *= 2)
        for (int i = 1; i <= 10; ++i) pts.push_back(evaluate_workload(w, c, d, i / 10.0));
    return Surface(w.id, pts);
}

namespace {
struct Builder {
    std::vector<Workload> ws;
    std::vector<std::string> ids;
    std::vector<std::pair<std::string, std::string>> edges;
    void add(const Workload& w) { ws.push_back(w); }
};

void preset(const std::string& name, int count, Builder& b) {
    if (name == "clip") {
        b.add(make_workload("vision", 4.17, 35.2, 0.30, 0.60));
        b.add(make_workload("text", 1.04, 20.5, 0.12, 0.45));
        b.add(make_workload("align", 0.40, 8.0, 0.02, 0.35));
        b.edges = {{"vision", "align"}, {"text", "align"}};
    } else if (name == "qwen3vl") {
        b.add(make_workload("vision", 2.58, 82.4, 0.60, 0.70));
        b.add(make_workload("text", 0.15, 2.1, 0.05, 0.30));
        b.add(make_workload("llm", 22.27, 145.2, 7.00, 0.80));
        b.edges = {{"vision", "llm"}, {"text", "llm"}};
    } else if (name == "unifiedio2") {
        b.add(make_workload("vision", 1.48, 24.6, 0.25, 0.55));
        b.add(make_workload("audio", 1.06, 21.8, 0.20, 0.50));
        b.add(make_workload("text", 0.10, 4.5, 0.04, 0.30));
        b.add(make_workload("llm", 16.70, 110.5, 3.20, 0.80));
        b.edges = {{"vision", "llm"}, {"audio", "llm"}, {"text", "llm"}};
    } else if (name == "imagebind") {
        const double batch = 160.0;
        b.add(make_workload("vision", 4.17, 35.2, 0.40, 0.60, batch));
        b.add(make_workload("audio", 2.09, 22.8, 0.25, 0.50, batch));
        b.add(make_workload("text", 1.04, 20.5, 0.15, 0.45, batch));
        b.add(make_workload("depth", 0.90, 15.0, 0.10, 0.40, batch));
        b.add(make_workload("thermal", 0.70, 12.0, 0.08, 0.40, batch));
        b.add(make_workload("imu", 0.20, 3.5, 0.04, 0.30, batch));
        b.add(make_workload("align", 0.50, 9.0, 0.03, 0.35, batch));
        for (const char* e : {"vision", "audio", "text", "depth", "thermal", "imu"})
            b.edges.push_back({e, "align"});
    } else if (name == "ofasys") {
        std::vector<Workload> pool = {
            make_workload("vision", 1.35, 18.2, 0.30, 0.55),
            make_workload("text", 0.72, 12.5, 0.15, 0.45),
            make_workload("audio", 0.95, 14.8, 0.20, 0.50),
            make_workload("video", 1.80, 22.0, 0.35, 0.60),
            make_workload("depth", 0.60, 10.0, 0.12, 0.40),
            make_workload("thermal", 0.50, 9.0, 0.10, 0.40),
            make_workload("imu", 0.15, 2.5, 0.04, 0.30),
            make_workload("box", 0.20, 5.0, 0.05, 0.35),
            make_workload("action", 0.30, 6.5, 0.07, 0.35),
        };
        int enc = count > 0 ? count - 1 : (int)pool.size();
        if (enc < 1 || enc > (int)pool.size()) throw RangeError("ofasys supports 2..10 modules");
        for (int i = 0; i < enc; ++i) b.add(pool[i]);
        b.add(make_workload("backbone", 4.80, 41.6, 2.40, 0.70));
        for (int i = 0; i < enc; ++i) b.edges.push_back({pool[i].id, "backbone"});
    } else {
        throw RangeError("unknown preset: " + name);
    }
    if (count > 0 && name != "ofasys" && count != (int)b.ws.size())
        throw RangeError("preset " + name + " has a fixed module count");
}

void config(const std::string& name, Builder& b, int& G, int& L) {
    if (name == "cfg1") {
        b.add(make_workload("vision", 4.17, 35.2, 0.30, 0.60));
        b.add(make_workload("text", 1.04, 20.5, 0.12, 0.45));
        G = 8;
        L = 10;
    } else if (name == "cfg2") {
        b.add(make_workload("vit", 4.17, 35.2, 0.30, 0.60));
        b.add(make_workload("proj", 0.05, 4.0, 0.02, 0.30));
        b.add(make_workload("llm", 22.27, 145.2, 7.00, 0.80));
        b.edges = {{"vit", "proj"}, {"proj", "llm"}};
        G = 16;
        L = 8;
    } else if (name == "cfg3") {
        b.add(make_workload("vision", 2.58, 82.4, 0.60, 0.70));
        b.add(make_workload("text", 0.15, 2.1, 0.05, 0.30));
        b.add(make_workload("deepstack", 0.30, 6.0, 0.05, 0.35));
        b.add(make_workload("llm", 22.27, 145.2, 7.00, 0.80));
        b.edges = {{"vision", "deepstack"}, {"deepstack", "llm"}, {"text", "llm"}};
        G = 32;
        L = 10;
    } else if (name == "cfg4") {
        b.add(make_workload("image", 4.17, 35.2, 0.30, 0.60));
        b.add(make_workload("video", 1.80, 22.0, 0.35, 0.60));
        b.add(make_workload("audio", 2.09, 22.8, 0.25, 0.50));
        b.add(make_workload("llm", 16.70, 110.5, 3.20, 0.80));
        b.add(make_workload("speech_dec", 0.95, 14.8, 0.20, 0.50));
        b.add(make_workload("image_dec", 1.48, 24.6, 0.25, 0.55));
        b.edges = {{"image", "llm"}, {"video", "llm"}, {"audio", "llm"},
                   {"llm", "speech_dec"}, {"llm", "image_dec"}};
        G = 64;
        L = 10;
    } else if (name == "cfg5") {
        preset("ofasys", 8, b);
        G = 128;
        L = 32;
    } else {
        throw RangeError("unknown config: " + name);
    }
}

void random_instance(uint64_t seed, int n, Builder& b) {
    std::mt19937_64 rng(seed);
    auto unif = [&](double lo, double hi) {
        return lo + (hi - lo) * (static_cast<double>(rng() >> 11) / double(1ULL << 53));
    };
    const bool star = n >= 2 && unif(0.0, 1.0) < 0.7;
    for (int i = 0; i < n; ++i) {
        char id[16];
        std::snprintf(id, sizeof(id), "m%02d", i);
        const bool backbone = star && i == n - 1;
        double tflops = backbone ? std::exp(unif(std::log(2.0), std::log(20.0)))
                                 : std::exp(unif(std::log(0.2), std::log(4.0)));
        double ci = std::exp(unif(std::log(2.0), std::log(150.0)));
        double params = tflops * unif(0.05, 0.3);
        double knee = unif(0.3, 0.8);
        b.add(make_workload(id, tflops, ci, params, knee));
    }
    if (star) {
        for (int i = 0; i + 1 < n; ++i) b.edges.push_back({b.ws[i].id, b.ws.back().id});
    } else {
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j)
                if (unif(0.0, 1.0) < 0.4) b.edges.push_back({b.ws[i].id, b.ws[j].id});
    }
}
}  // namespace

namespace {
Builder synth_builder(const std::string& spec, int& G, int& L) {
    Builder b;
    if (spec.rfind("random:", 0) == 0) {
        unsigned long long seed;
        int n, g;
        if (std::sscanf(spec.c_str(), "random:%llu:%d:%d", &seed, &n, &g) != 3)
            throw RangeError("bad spec " + spec);
        random_instance(seed, n, b);
        G = g;
    } else if (spec.rfind("preset:", 0) == 0) {
        char name[64] = {0};
        int count, g;
        if (std::sscanf(spec.c_str(), "preset:%63[^:]:%d:%d", name, &count, &g) != 3)
            throw RangeError("bad spec " + spec);
        preset(name, count, b);
        G = g;
    } else {
        config(spec, b, G, L);
    }
    return b;
}
}  // namespace

std::vector<Workload> synth_workloads(const std::string& spec, Cluster* c, int* L) {
    int G = 1, l = 10;
    Builder b = synth_builder(spec, G, l);
    if (c) {
        *c = Cluster{};
        c->gpu_count = G;
    }
    if (L) *L = l;
    return b.ws;
}

Problem synth_problem(const std::string& spec, int levels_override) {
    int G = 1, L = 10;
    Builder b = synth_builder(spec, G, L);
    if (levels_override > 0) L = levels_override;
    Cluster c;
    c.gpu_count = G;
    Problem P;
    P.gpu_count = G;
    P.memory_capacity = c.memory_capacity;
    P.quota_levels = L;
    P.im.e1 = 0.4e-3;  // default_ground_truth, bench.hpp:31-37
    P.im.e2 = 1.2e-3;
    P.im.e3 = 0.8e-3;
    for (const auto& w : b.ws) {
        Module m;
        m.id = w.id;
        m.memory_base = w.grad * 3.0;  // make_spec, profiler.hpp:205
        m.surface = generate_surface(w, c);
        P.modules.push_back(std::move(m));
    }
    auto idx = [&](const std::string& id) {
        for (size_t i = 0; i < b.ws.size(); ++i)
            if (b.ws[i].id == id) return (int)i;
        throw RangeError("unknown module " + id);
    };
    for (auto& [u, v] : b.edges) P.edges.push_back({idx(u), idx(v)});
    return P;
}

}  // namespace mosaic_b200
