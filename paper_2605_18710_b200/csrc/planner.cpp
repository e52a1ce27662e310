// planner.cpp — see planner.hpp.  Compiled with -ffp-contract=off.
#include "planner.hpp"
#include "pack.hpp"

#include <algorithm>
#include <bit>
#include <chrono>
#include <cmath>
#include <functional>
#include <limits>
#include <cstring>
#include <cstdio>
#include <cstdlib>

namespace mosaic_b200 {

using mg::Leaf;
using mg::MODE_FIRST;
using mg::MODE_MIN;
using mg::POS_INF;

namespace {
std::vector<int> mask_modules(uint64_t mask) {
    std::vector<int> out;
    for (int m = 0; m < 64; ++m)
        if (mask >> m & 1) out.push_back(m);
    return out;
}
double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}
}  // namespace

Planner::Planner(Problem P, int device) : P_(std::move(P)) {
    std::string err = validate_graph(P_);
    if (!err.empty()) throw Error(RANGE, err);
    if ((int)P_.modules.size() > 64) throw Error(RANGE, "solver supports up to 64 modules");
    if (P_.gpu_count < 1 || P_.gpu_count > 65535) throw Error(RANGE, "bad gpu_count");
    M_.G = P_.gpu_count;
    M_.L = P_.quota_levels;
    M_.cap = P_.memory_capacity;
    M_.e1 = P_.im.e1;
    M_.e2 = P_.im.e2;
    M_.e3 = P_.im.e3;
    M_.additive = P_.im.additive_only;
    M_.include_self = P_.include_self;
    opts_.resize(P_.modules.size());
    opt_err_.resize(P_.modules.size());
    // candidate_options of every module, built on the device (pack.cu)
    std::vector<mg::PackInput> pin(P_.modules.size());
    for (size_t m = 0; m < P_.modules.size(); ++m) {
        const Surface& s = P_.modules[m].surface;
        pin[m].dv = s.d_values();
        pin[m].av = s.a_values();
        for (const auto& p : s.grid()) {
            pin[m].lat.push_back(p.latency);
            pin[m].bw.push_back(p.bandwidth_util);
            pin[m].mem.push_back(p.memory);
        }
        pin[m].membase = P_.modules[m].memory_base;
    }
    long long packed_bytes = 0;
    std::vector<int> range_err;
    auto packed = mg::pack_options_device(pin, P_.gpu_count, P_.quota_levels, P_.memory_capacity,
                                          device, &packed_bytes, &range_err);
    int off = 0;
    for (size_t m = 0; m < P_.modules.size(); ++m) {
        if (range_err[m])
            opt_err_[m] = P_.modules[m].id + ": d=1 outside profiled range";
        else
            for (const auto& r : packed[m]) opts_[m].push_back(Cand{r.d, r.u, r.base, r.B, r.fp});
        std::vector<mg::OptRow> rows;
        for (const auto& c : opts_[m])
            rows.push_back(mg::OptRow{c.d, c.units, c.base, c.B, c.fp,
                                      mg::filter_bound(M_, c.base, c.B)});
        M_.rows.push_back(rows);
        M_.row_off.push_back(off);
        off += (int)rows.size();
    }
    eng_ = std::make_unique<mg::Engine>(device);
    eng_->upload_rows(M_);
}

void Planner::check_rows(int m) const {
    if (!opt_err_[m].empty()) throw Error(RANGE, opt_err_[m]);
}

// Canonical form of a known allocation in the DFS order `order`: sort GPUs by their
// membership vector (level 0 most significant, descending); then at every level each
// module holds a prefix of every block.  Yields the hit path + leaf the FIRST search
// would report for it, or false if it is not a leaf of that search (filter, capacity).
bool Planner::make_seed(const std::vector<Entry>& ents, const std::vector<int>& order,
                        bool filter, double theta, double value, mg::HitPath& hp,
                        Leaf& lf) const {
    const int k = (int)order.size(), G = P_.gpu_count;
    if (!(value <= theta) || k > mg::MAXK) return false;
    std::vector<uint32_t> key(G, 0);
    std::vector<int> row(k, -1);
    for (int l = 0; l < k; ++l) {
        const Entry* e = nullptr;
        for (const auto& x : ents)
            if (x.module == order[l]) e = &x;
        if (!e) return false;
        const auto& rows = M_.rows[order[l]];
        for (int i = 0; i < (int)rows.size(); ++i)
            if (rows[i].d == e->d && rows[i].u == e->units) row[l] = i;
        if (row[l] < 0) return false;
        if (filter && rows[row[l]].bound > theta) return false;
        for (int g : e->gpus) key[g] |= 1u << (k - 1 - l);
    }
    std::vector<uint32_t> ks(key);
    std::sort(ks.begin(), ks.end(), std::greater<uint32_t>());
    struct Blk { int start, size; uint32_t mask; };
    std::vector<Blk> blocks{{0, G, 0}};
    std::memset(&hp, 0, sizeof hp);
    for (int l = 0; l < k; ++l) {
        if ((int)blocks.size() > mg::MAXB) return false;
        const mg::OptRow& r = M_.rows[order[l]][row[l]];
        hp.opt[l] = (uint16_t)row[l];
        hp.nb[l] = (uint16_t)blocks.size();
        std::vector<Blk> next;
        const uint32_t bit = 1u << (k - 1 - l);
        for (size_t b = 0; b < blocks.size(); ++b) {
            const Blk& B = blocks[b];
            int taken = 0;
            while (taken < B.size && (ks[B.start + taken] & bit)) ++taken;
            hp.x[l][b] = (uint16_t)taken;
            if (taken > 0) {
                int units = 0;
                double mem = 0.0;
                for (int t = 0; t < l; ++t)
                    if (B.mask >> t & 1u) {
                        units += M_.rows[order[t]][row[t]].u;
                        mem = mem + M_.rows[order[t]][row[t]].fp;
                    }
                if (units + r.u > M_.L || mem + r.fp > M_.cap * (1.0 + 1e-12)) return false;
                next.push_back({B.start, taken, B.mask | (1u << l)});
            }
            if (taken < B.size) next.push_back({B.start + taken, B.size - taken, B.mask});
        }
        blocks.swap(next);
    }
    if ((int)blocks.size() > 2 * mg::MAXB) return false;
    std::memset(&lf, 0, sizeof lf);
    lf.value = value;
    for (int l = 0; l < k; ++l) lf.opt[l] = (uint16_t)row[l];
    lf.nb = (int)blocks.size();
    for (size_t b = 0; b < blocks.size(); ++b) {
        lf.bsz[b] = (uint16_t)blocks[b].size;
        lf.bmk[b] = (uint16_t)blocks[b].mask;
    }
    return true;
}

bool Planner::first_leaf(const std::vector<int>& order, bool filter, double theta, Leaf& leaf,
                         mg::SearchStats& st, const std::vector<Entry>* seed,
                         double seed_value) {
    mg::SearchReq q;
    q.mode = MODE_FIRST;
    q.use_filter = filter;
    q.theta = theta;
    q.level_module = order;
    mg::Spec S;
    if (!mg::build_spec(M_, q, S)) return false;
    mg::HitPath hp;
    Leaf sl;
    const bool seeded = seed && make_seed(*seed, order, filter, theta, seed_value, hp, sl);
    if (seed && std::getenv("MOSAIC_TRACE"))
        std::fprintf(stderr, "[mosaic] FIRST seed %s (theta=%.17g value=%.17g)\n",
                     seeded ? "applied" : "rejected", theta, seed_value);
    mg::SearchResult r = eng_->search(S, POS_INF, 0.0, st, seeded ? &hp : nullptr,
                                      seeded ? &sl : nullptr);
    if (r.overflow) throw Error(TOO_LARGE, "stage needs more than 128 GPU blocks");
    if (r.found) leaf = r.leaf;
    return r.found;
}

// Exact minimum stage_time over every capacity/memory-feasible leaf (T*), restarting
// with tighter static bounds whenever the incumbent drops well below the last bound.
double Planner::min_value(const std::vector<int>& mods, double ub, mg::SearchStats& st,
                          std::vector<Entry>* argmin) {
    while (true) {
        // fail-first: fewest viable options first (any order is valid for MIN)
        const double thp = ub >= POS_INF ? POS_INF : ub * (1.0 - mg::TIE_EPS);
        std::vector<std::pair<int, int>> cnt;
        for (int m : mods) {
            int c = 0;
            for (const auto& r : M_.rows[m]) {
                double lb = r.base;
                if (M_.nonneg()) {
                    lb = r.base + M_.e1;
                    if (M_.include_self) lb = lb + M_.e2 * r.B;
                }
                if (!M_.nonneg() || lb <= thp) ++c;
            }
            cnt.push_back({c, m});
        }
        std::stable_sort(cnt.begin(), cnt.end());
        mg::SearchReq q;
        q.mode = MODE_MIN;
        q.ub = ub;
        for (auto& [c, m] : cnt) q.level_module.push_back(m);
        if (const char* e = std::getenv("MOSAIC_MIN_ORDER")) {  // experiments: "3,0,1,..."
            std::vector<int> o;
            for (const char* p = e; *p;) {
                o.push_back(std::atoi(p));
                while (*p && *p != ',') ++p;
                if (*p == ',') ++p;
            }
            std::vector<int> a = o, b = mods;
            std::sort(a.begin(), a.end());
            std::sort(b.begin(), b.end());
            if (a == b) q.level_module = o;
        }
        mg::Spec S;
        if (!mg::build_spec(M_, q, S)) return ub;
        double ab = ub >= POS_INF ? POS_INF : ub * (1.0 - 1e-4);
        mg::SearchResult r = eng_->search(S, ub, ab, st);
        if (r.overflow) throw Error(TOO_LARGE, "stage needs more than 128 GPU blocks");
        if (argmin && r.found && r.leaf.nb > 0) *argmin = leaf_entries(q.level_module, r.leaf);
        if (r.aborted) {
            ub = r.value;
            continue;
        }
        return r.value;
    }
}

std::vector<Entry> Planner::leaf_entries(const std::vector<int>& order, const Leaf& lf) const {
    const int k = (int)order.size();
    std::vector<std::vector<int>> g(k);
    int start = 0;
    for (int b = 0; b < lf.nb; ++b) {
        for (int l = 0; l < k; ++l)
            if (lf.bmk[b] >> l & 1)
                for (int t = 0; t < lf.bsz[b]; ++t) g[l].push_back(start + t);
        start += lf.bsz[b];
    }
    std::vector<Entry> out;
    for (int l = 0; l < k; ++l) {
        const auto& c = opts_[order[l]][lf.opt[l]];
        out.push_back(Entry{order[l], c.d, c.units, g[l]});
    }
    std::sort(out.begin(), out.end(), [](const Entry& a, const Entry& b) { return a.module < b.module; });
    return out;
}

StageResult Planner::stage_eval(uint64_t mask) {
    StageResult res;
    const auto mods = mask_modules(mask);
    if ((int)mods.size() > mg::MAXK) throw Error(TOO_LARGE, "stage larger than 12 modules");
    for (int m : mods) {
        check_rows(m);
        if (opts_[m].empty()) {
            res.status = MODULE_NO_OPTION;
            return res;
        }
    }
    const Interference& im = P_.im;
    const bool nonneg = im.non_negative();
    double tau_lo = 0.0, tau_hi = 0.0;
    for (int m : mods) {
        double lo = std::numeric_limits<double>::max();
        double solo = std::numeric_limits<double>::max();
        for (const auto& c : opts_[m]) {
            double bound = c.base;
            if (nonneg) {
                bound += im.e1;
                if (P_.include_self) bound += im.e2 * c.B;
            }
            lo = std::min(lo, bound);
            double delta = P_.include_self ? im.delta(c.B, c.B) : im.delta(0.0, 0.0);
            solo = std::min(solo, c.base + delta);
        }
        if (nonneg) tau_lo = std::max(tau_lo, lo);
        tau_hi += solo;
    }
    bool have_T = false;
    double Tstar = POS_INF;
    std::vector<Entry> argmin;  // an allocation reaching Tstar
    long long probes = 0;
    // FeasibilitySearch::run(tau) replayed: first leaf in fail-first DFS order.
    auto run = [&](double tau, Leaf& leaf, std::vector<int>& order) -> bool {
        ++probes;
        const double th = tau * (1.0 + 1e-12);
        std::vector<std::pair<int, int>> cnt;
        for (int m : mods) {
            int c = 0;
            for (const auto& r : M_.rows[m])
                if (r.bound <= th) ++c;
            if (c == 0) return false;
            cnt.push_back({c, m});
        }
        // T* lies in [Tstar*(1 - TIE_EPS - rounding), Tstar]: below that band no leaf can
        // reach tau; inside it the probe is decided by an exact FIRST search.
        if (nonneg && have_T && th < Tstar * (1.0 - 1e-13)) return false;
        std::stable_sort(cnt.begin(), cnt.end());
        order.clear();
        for (auto& [c, m] : cnt) order.push_back(m);
        // seed with the argmin allocation when it is known to satisfy this probe
        const bool seed = nonneg && have_T && !argmin.empty() && Tstar <= th;
        return first_leaf(order, true, th, leaf, res.st, seed ? &argmin : nullptr, Tstar);
    };
    Leaf best, cur;
    std::vector<int> best_order, cur_order;
    bool ok = run(tau_hi, best, best_order);
    for (int attempt = 0; !ok && attempt < 60; ++attempt) {
        tau_hi *= 2.0;
        ok = run(tau_hi, best, best_order);
    }
    res.probes = probes;
    if (!ok) {
        res.status = INFEASIBLE;
        return res;
    }
    double t_best = best.value;
    if (nonneg) {
        argmin = leaf_entries(best_order, best);
        Tstar = min_value(mods, t_best, res.st, &argmin);
        have_T = true;
    }
    double lo = std::min(tau_lo, t_best);
    while (t_best - lo > P_.bisect_rel_tol * std::abs(t_best)) {
        double mid = 0.5 * (lo + t_best);
        if (mid >= t_best * (1.0 - 1e-12)) break;
        if (run(mid, cur, cur_order)) {
            best = cur;
            best_order = cur_order;
            t_best = best.value;
        } else {
            lo = mid;
        }
    }
    for (int guard = 0; guard < 1000; ++guard) {
        double probe = t_best * (1.0 - 1e-9);
        if (probe <= lo) break;
        if (!run(probe, cur, cur_order)) break;
        best = cur;
        best_order = cur_order;
        t_best = best.value;
    }
    res.status = OK;
    res.stage_time = t_best;
    res.entries = leaf_entries(best_order, best);
    res.probes = probes;
    return res;
}

// core.hpp:281-351: partition coverage, dependency order, per-GPU quota sum <= 1 + 1e-9,
// per-GPU memory <= capacity * (1 + 1e-12) with footprint = lookup(d, a).memory + base.
std::string Planner::validate_plan(const std::vector<std::vector<Entry>>& stages,
                                   std::string* msg) const {
    const int n = (int)P_.modules.size();
    std::vector<int> stage_of(n, -1);
    auto fail = [&](const char* code, const std::string& m) {
        if (msg) *msg = m;
        return std::string(code);
    };
    for (int si = 0; si < (int)stages.size(); ++si) {
        if (stages[si].empty()) return fail("EmptyStage", "stage " + std::to_string(si) + " is empty");
        for (const auto& e : stages[si]) {
            if (e.module < 0 || e.module >= n)
                return fail("ModuleMissing", "stage entry references unknown module index");
            if (stage_of[e.module] != -1)
                return fail("ModuleDuplicated", "module " + P_.modules[e.module].id +
                                                    " appears in more than one stage");
            stage_of[e.module] = si;
            if ((int)e.gpus.size() != e.d)
                return fail("SmOvercommit", "placement size does not match dp degree for " +
                                                P_.modules[e.module].id);
            for (int r : e.gpus)
                if (r < 0 || r >= P_.gpu_count)
                    return fail("SmOvercommit", "GPU index out of range for " + P_.modules[e.module].id);
        }
    }
    for (int i = 0; i < n; ++i)
        if (stage_of[i] == -1) return fail("ModuleMissing", "module " + P_.modules[i].id + " not placed");
    for (auto [u, v] : P_.edges)
        if (stage_of[u] >= stage_of[v])
            return fail("DependencyViolated", "edge " + P_.modules[u].id + " -> " +
                                                  P_.modules[v].id + " not strictly ordered");
    for (int si = 0; si < (int)stages.size(); ++si) {
        std::vector<double> quota(P_.gpu_count, 0.0), mem(P_.gpu_count, 0.0);
        for (const auto& e : stages[si]) {
            std::vector<int> g(e.gpus);
            std::sort(g.begin(), g.end());
            if (std::adjacent_find(g.begin(), g.end()) != g.end())
                return fail("SmOvercommit", "replica co-location on one GPU for " + P_.modules[e.module].id);
            const double a = (double)e.units / P_.quota_levels;
            const double fp = P_.modules[e.module].surface.lookup(e.d, a).memory +
                              P_.modules[e.module].memory_base;
            for (int r : e.gpus) {
                quota[r] += a;
                mem[r] += fp;
            }
        }
        for (int r = 0; r < P_.gpu_count; ++r) {
            if (quota[r] > 1.0 + 1e-9)
                return fail("SmOvercommit", "SM quota overcommit on GPU " + std::to_string(r) +
                                                " in stage " + std::to_string(si));
            if (mem[r] > P_.memory_capacity * (1.0 + 1e-12))
                return fail("MemoryOvercommit", "memory overcommit on GPU " + std::to_string(r) +
                                                    " in stage " + std::to_string(si));
        }
    }
    if (msg) msg->clear();
    return "";
}

double Planner::stage_min(uint64_t mask, double ub, bool restart, mg::SearchStats& st) {
    const auto mods = mask_modules(mask);
    if ((int)mods.size() > mg::MAXK) throw Error(TOO_LARGE, "stage larger than 12 modules");
    for (int m : mods) check_rows(m);
    if (restart) return min_value(mods, ub, st);
    mg::SearchReq q;
    q.mode = MODE_MIN;
    q.ub = ub;
    q.level_module = mods;
    if (const char* e = std::getenv("MOSAIC_MIN_ORDER")) {
        std::vector<int> o;
        for (const char* p = e; *p;) {
            o.push_back(std::atoi(p));
            while (*p && *p != ',') ++p;
            if (*p == ',') ++p;
        }
        if (o.size() == mods.size()) q.level_module = o;
    }
    mg::Spec S;
    if (!mg::build_spec(M_, q, S)) return ub;
    mg::SearchResult r = eng_->search(S, ub, 0.0, st);
    if (r.overflow) throw Error(TOO_LARGE, "stage needs more than 128 GPU blocks");
    return r.value;
}

StageResult Planner::feasible(uint64_t mask, double tau) {
    StageResult res;
    const auto mods = mask_modules(mask);
    if ((int)mods.size() > mg::MAXK) throw Error(TOO_LARGE, "stage larger than 12 modules");
    const double th = tau * (1.0 + 1e-12);
    std::vector<std::pair<int, int>> cnt;
    res.probes = 1;
    for (int m : mods) {
        check_rows(m);
        int c = 0;
        for (const auto& r : M_.rows[m])
            if (r.bound <= th) ++c;
        if (c == 0) {
            res.status = INFEASIBLE;
            return res;
        }
        cnt.push_back({c, m});
    }
    std::stable_sort(cnt.begin(), cnt.end());
    std::vector<int> order;
    for (auto& [c, m] : cnt) order.push_back(m);
    Leaf lf;
    if (!first_leaf(order, true, th, lf, res.st)) {
        res.status = INFEASIBLE;
        return res;
    }
    res.status = OK;
    res.stage_time = lf.value;
    res.entries = leaf_entries(order, lf);
    return res;
}

StageResult Planner::exact_stage(uint64_t mask) {
    StageResult res;
    const auto mods = mask_modules(mask);
    if ((int)mods.size() > mg::MAXK) throw Error(TOO_LARGE, "stage larger than 12 modules");
    for (int m : mods) {
        check_rows(m);
        if (opts_[m].empty()) {
            res.status = INFEASIBLE;  // ExactStageSolver returns nullopt (oracle.hpp:91-92)
            return res;
        }
    }
    Leaf first;
    if (!first_leaf(mods, false, POS_INF, first, res.st)) {
        res.status = INFEASIBLE;
        return res;
    }
    double T = min_value(mods, first.value, res.st);
    Leaf lf;
    if (!first_leaf(mods, false, T, lf, res.st))
        throw Error(CUDA, "exact search lost the argmin leaf");
    res.status = OK;
    res.stage_time = T;
    res.entries = leaf_entries(mods, lf);
    return res;
}

std::optional<StageResult> Planner::evaluate_cached(uint64_t mask, bool* hit, PlanResult& pr) {
    if (P_.enable_cache) {
        auto it = cache_.find(mask);
        if (it != cache_.end()) {
            if (hit) *hit = true;
            pr.cache_hits++;
            return it->second;
        }
    }
    if (hit) *hit = false;
    pr.stage_eval_calls++;
    StageResult r = stage_eval(mask);
    pr.st.nodes += r.st.nodes;
    pr.st.leaves += r.st.leaves;
    pr.st.searches += r.st.searches;
    pr.st.rounds += r.st.rounds;
    if (r.status == MODULE_NO_OPTION)
        throw Error(MODULE_NO_OPTION, "module has no feasible deployment option");
    if (r.status != OK) return std::nullopt;
    pr.feasibility_calls += r.probes;
    if (P_.enable_cache) cache_.emplace(mask, r);
    return r;
}

PlanResult Planner::solve() {
    const double t0 = now_s();
    PlanResult pr;
    const int n = (int)P_.modules.size();
    if (n == 0) throw Error(EMPTY, "model graph has no modules");
    cache_.clear();
    auto reach = reachability_masks(P_);
    std::vector<uint64_t> masks;
    std::vector<StageResult> results;
    for (int m : topological_order(P_)) {
        uint64_t mask = uint64_t(1) << m;
        auto r = evaluate_cached(mask, nullptr, pr);
        if (!r) throw Error(MODULE_NO_OPTION, "module " + P_.modules[m].id +
                                                  " cannot be placed alone on the cluster");
        masks.push_back(mask);
        results.push_back(*r);
    }
    std::vector<double> min_base(n);
    for (int m = 0; m < n; ++m) {
        check_rows(m);
        double b = std::numeric_limits<double>::max();
        for (const auto& c : opts_[m]) b = std::min(b, c.base);
        min_base[m] = b;
    }
    auto legal = [&](size_t x, size_t y) {
        uint64_t up = masks[x];
        for (size_t z = x + 1; z < y; ++z) up |= masks[z];
        for (int m = 0; m < 64; ++m)
            if ((up >> m & 1) && (reach[m] & masks[y])) return false;
        return true;
    };
    auto order_lt = [](uint64_t mx, uint64_t my, uint64_t nx, uint64_t ny) {
        uint64_t a = mx | my, b = nx | ny;
        int ca = std::popcount(a), cb = std::popcount(b);
        if (ca != cb) return ca < cb;
        if (a != b) return a < b;
        return mx < nx;
    };
    while (masks.size() > 1) {
        TraceRound round;
        std::vector<std::pair<size_t, size_t>> pairs;
        for (size_t x = 0; x < masks.size(); ++x)
            for (size_t y = x + 1; y < masks.size(); ++y)
                if (legal(x, y)) pairs.push_back({x, y});
        std::sort(pairs.begin(), pairs.end(), [&](const auto& a, const auto& b) {
            return order_lt(masks[a.first], masks[a.second], masks[b.first], masks[b.second]);
        });
        double delta_best = 0.0;
        int best_idx = -1;
        StageResult best_merged;
        for (size_t i = 0; i < pairs.size(); ++i) {
            auto [x, y] = pairs[i];
            TraceCand c{masks[x], masks[y], false, false, 0.0};
            double tx = results[x].stage_time, ty = results[y].stage_time;
            if (P_.enable_prune) {
                double t_lb = 0.0;
                for (int m : mask_modules(c.mask_x | c.mask_y)) t_lb = std::max(t_lb, min_base[m]);
                if (tx + ty - t_lb <= delta_best) {
                    c.pruned = true;
                    pr.prunes++;
                    round.cands.push_back(c);
                    continue;
                }
            }
            auto merged = evaluate_cached(c.mask_x | c.mask_y, &c.cache_hit, pr);
            if (!merged) {
                c.gain = -std::numeric_limits<double>::infinity();
                round.cands.push_back(c);
                continue;
            }
            c.gain = tx + ty - merged->stage_time;
            round.cands.push_back(c);
            if (c.gain > delta_best) {
                delta_best = c.gain;
                best_idx = (int)i;
                best_merged = *merged;
            }
        }
        if (best_idx < 0) {
            pr.rounds.push_back(std::move(round));
            break;
        }
        auto [x, y] = pairs[best_idx];
        round.chosen_x = masks[x];
        round.chosen_y = masks[y];
        round.applied_gain = delta_best;
        masks[x] |= masks[y];
        results[x] = best_merged;
        masks.erase(masks.begin() + y);
        results.erase(results.begin() + y);
        pr.rounds.push_back(std::move(round));
    }
    for (size_t i = 0; i < masks.size(); ++i) {
        pr.masks.push_back(masks[i]);
        pr.stages.push_back(results[i]);
        pr.iteration_time += results[i].stage_time;
    }
    pr.status = OK;
    pr.elapsed = now_s() - t0;
    return pr;
}

PlanResult Planner::brute_force() {
    const double t0 = now_s();
    PlanResult pr;
    const int n = (int)P_.modules.size();
    if (n > 8) throw Error(TOO_LARGE, "oracle enumeration limited to 8 modules");
    std::vector<uint64_t> preds(n, 0);
    for (auto [u, v] : P_.edges) preds[v] |= uint64_t(1) << u;
    const uint64_t full = (uint64_t(1) << n) - 1;
    std::vector<std::vector<uint64_t>> parts;
    std::vector<uint64_t> cur;
    std::function<void(uint64_t)> rec = [&](uint64_t placed) {
        if (placed == full) {
            parts.push_back(cur);
            return;
        }
        uint64_t avail = 0;
        for (int m = 0; m < n; ++m)
            if (!(placed >> m & 1) && (preds[m] & ~placed) == 0) avail |= uint64_t(1) << m;
        for (uint64_t sub = avail; sub; sub = (sub - 1) & avail) {
            cur.push_back(sub);
            rec(placed | sub);
            cur.pop_back();
        }
    };
    rec(0);
    std::unordered_map<uint64_t, StageResult> memo;
    auto stage_min = [&](uint64_t mask) -> const StageResult& {
        auto it = memo.find(mask);
        if (it == memo.end()) {
            StageResult r = exact_stage(mask);
            pr.st.nodes += r.st.nodes;
            pr.st.leaves += r.st.leaves;
            pr.st.searches += r.st.searches;
            pr.st.rounds += r.st.rounds;
            it = memo.emplace(mask, std::move(r)).first;
        }
        return it->second;
    };
    bool have = false;
    double best_total = 0.0;
    std::vector<uint64_t> best_masks;
    for (const auto& part : parts) {
        double total = 0.0;
        bool feasible = true;
        size_t used = 0;
        for (uint64_t mask : part) {
            const StageResult& r = stage_min(mask);
            if (r.status != OK) {
                feasible = false;
                break;
            }
            total += r.stage_time;
            ++used;
            if (have && total >= best_total) {
                feasible = false;
                break;
            }
        }
        if (!feasible || used != part.size()) continue;
        if (!have || total < best_total) {
            have = true;
            best_total = total;
            best_masks = part;
        }
    }
    pr.partitions = (long long)parts.size();
    if (!have) {
        pr.status = INFEASIBLE;
        pr.elapsed = now_s() - t0;
        return pr;
    }
    for (uint64_t m : best_masks) {
        pr.masks.push_back(m);
        pr.stages.push_back(memo.at(m));
    }
    pr.iteration_time = best_total;
    pr.status = OK;
    pr.elapsed = now_s() - t0;
    return pr;
}

void Planner::stage_time(const std::vector<std::vector<Entry>>& allocs, std::vector<double>& st,
                         std::vector<std::vector<double>>& rect) {
    std::vector<mg::EvalEntry> ent;
    std::vector<int> gpus;
    std::vector<long long> off{0};
    std::vector<double> base, Bt;
    std::unordered_map<uint64_t, int> row_of;  // (module, d, units) -> table row
    for (const auto& a : allocs) {
        for (const auto& e : a) {
            if (e.module < 0 || e.module >= (int)P_.modules.size())
                throw Error(RANGE, "module not in graph");
            uint64_t key = (uint64_t)e.module << 40 | (uint64_t)(uint32_t)e.d << 20 |
                           (uint64_t)(uint32_t)e.units;
            auto it = row_of.find(key);
            int row;
            if (it == row_of.end()) {
                const Surface& s = P_.modules[e.module].surface;
                double a = (double)e.units / P_.quota_levels;
                base.push_back(s.lookup(e.d, a).latency);      // PerfContext::base_latency
                Bt.push_back(s.lookup(1, a).bandwidth_util);   // PerfContext::solo_bandwidth
                row = (int)base.size() - 1;
                row_of.emplace(key, row);
            } else {
                row = it->second;
            }
            for (int g : e.gpus)
                if (g < 0 || g >= P_.gpu_count) throw Error(RANGE, "GPU index out of range");
            ent.push_back(mg::EvalEntry{row, e.module, (int)e.gpus.size(), 0,
                                        (long long)gpus.size()});
            gpus.insert(gpus.end(), e.gpus.begin(), e.gpus.end());
        }
        if (a.size() > 64) throw Error(TOO_LARGE, "evaluator supports 64 entries per stage");
        off.push_back((long long)ent.size());
    }
    std::vector<double> rflat;
    eng_->evaluate(ent, gpus, off, base, Bt, P_.gpu_count, M_, st, rflat);
    rect.assign(allocs.size(), {});
    for (size_t i = 0; i < allocs.size(); ++i)
        rect[i].assign(rflat.begin() + off[i], rflat.begin() + off[i + 1]);
}

}  // namespace mosaic_b200
