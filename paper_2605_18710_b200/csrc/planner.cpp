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
    mg::build_index(M_);
    tau_mins_.assign(P_.modules.size(), {0.0, 0.0});
    for (size_t m = 0; m < P_.modules.size(); ++m) {
        double lo = std::numeric_limits<double>::max();
        double solo = std::numeric_limits<double>::max();
        for (const auto& c : opts_[m]) {
            double bound = c.base;
            if (P_.im.non_negative()) {
                bound += P_.im.e1;
                if (P_.include_self) bound += P_.im.e2 * c.B;
            }
            lo = std::min(lo, bound);
            double delta = P_.include_self ? P_.im.delta(c.B, c.B) : P_.im.delta(0.0, 0.0);
            solo = std::min(solo, c.base + delta);
        }
        tau_mins_[m] = {lo, solo};
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
    if (seed && eng_->tuning().trace == 1)
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

bool Planner::prep_first(const std::vector<int>& order, bool filter, double theta, SearchOp& op,
                         mg::SearchStats& st, const std::vector<Entry>* seed, double seed_value) {
    mg::SearchReq q;
    q.mode = MODE_FIRST;
    q.use_filter = filter;
    q.theta = theta;
    q.level_module = order;
    op.req = mg::BatchReq{};
    if (!mg::build_spec(M_, q, op.req.S)) return false;
    const bool seeded = seed && make_seed(*seed, order, filter, theta, seed_value, op.hp, op.sl);
    if (seed && eng_->tuning().trace == 1)
        std::fprintf(stderr, "[mosaic] FIRST seed %s (theta=%.17g value=%.17g)\n",
                     seeded ? "applied" : "rejected", theta, seed_value);
    op.req.ub = POS_INF;
    op.req.abort_below = 0.0;
    op.req.seed_path = seeded ? &op.hp : nullptr;
    op.req.seed_leaf = seeded ? &op.sl : nullptr;
    op.req.st = &st;
    return true;
}

// MIN request: fail-first order (fewest viable options first; any order is valid for MIN).
bool Planner::prep_min(const std::vector<int>& mods, double ub, SearchOp& op, mg::SearchStats& st,
                       std::vector<int>& order) {
    const double thp = ub >= POS_INF ? POS_INF : ub * (1.0 - mg::TIE_EPS);
    std::vector<std::pair<int, int>> cnt;
    const int mo = eng_->tuning().min_order;
    for (int m : mods) {
        // lb = (base + e1) + e2 B is exactly the row's filter bound with non-negative
        // coefficients: count rows with bound <= thp in the bound-sorted index
        const auto& b = M_.index[m].bound;
        const int c = M_.nonneg() ? (int)(std::upper_bound(b.begin(), b.end(), thp) - b.begin())
                                  : (int)M_.rows[m].size();
        // any level order gives the same T*; the order only changes the tree's size
        int key = c;
        if (mo == 1) key = -c;  // most viable options first
        else if (mo == 2 || mo == 3) {
            // by the module's smallest base latency (rows are sorted by it), largest / smallest first
            const double mb = M_.rows[m].empty() ? 0.0 : M_.rows[m][0].base;
            const int q = (int)std::min(2.0e9, mb * 1e8);
            key = mo == 2 ? -q : q;
        } else if (mo == 4) {
            // largest minimal solo rectified latency first
            key = -(int)std::min(2.0e9, tau_mins_[m].second * 1e8);
        } else if (mo == 5) {
            // largest minimal per-GPU footprint first
            double fp = 1e300;
            for (const auto& r : M_.rows[m]) fp = std::min(fp, r.fp);
            key = -(int)std::min(2.0e9, fp * 1e-3);
        } else if (mo == 6) {
            // fewest viable options first, ties: largest minimal base latency first
            const double mb = M_.rows[m].empty() ? 0.0 : M_.rows[m][0].base;
            key = c * 4096 - (int)std::min(4095.0, mb * 100.0);
        }
        cnt.push_back({key, m});
    }
    std::stable_sort(cnt.begin(), cnt.end());
    if (eng_->tuning().min_perm > 0) {
        // measurement: the min_perm-th permutation (lexicographic, 1-based) of the modules
        std::vector<int> ms(mods);
        std::sort(ms.begin(), ms.end());
        long long r = eng_->tuning().min_perm - 1;
        for (size_t i = 0; i < ms.size() && r > 0; ++i) {
            long long f = 1;
            for (size_t t = 1; t < ms.size() - i; ++t) f *= (long long)t;
            const long long idx = r / f;
            r %= f;
            std::rotate(ms.begin() + i, ms.begin() + i + idx, ms.begin() + i + idx + 1);
        }
        for (size_t i = 0; i < ms.size(); ++i) cnt[i] = {0, ms[i]};
    }
    mg::SearchReq q;
    q.mode = MODE_MIN;
    q.ub = ub;
    order.clear();
    for (auto& [c, m] : cnt) order.push_back(m);
    q.level_module = order;
    op.req = mg::BatchReq{};
    if (!mg::build_spec(M_, q, op.req.S)) return false;
    op.req.ub = ub;
    // restart with re-derived static bounds once the incumbent drops by >1e-4 — worth a new
    // launch only for large stages; small ones finish in the same wave
    const bool restart = (int)mods.size() >= eng_->tuning().restart_k;
    op.req.abort_below = !restart ? 0.0 : (ub >= POS_INF ? POS_INF : ub * (1.0 - 1e-4));
    op.req.st = &st;
    return true;
}

// stage_eval (stage_eval.hpp:302-382) as a coroutine: the reference's tau schedule (doubling,
// bisection, confirmation) with every FeasibilitySearch::run it would make replayed, in
// order; each one is a device FIRST search, or is decided from T* (one MIN proof) without
// a search.
StageJob Planner::stage_eval_job(uint64_t mask, StageResult* out) {
    StageResult& res = *out;
    const auto mods = mask_modules(mask);
    if ((int)mods.size() > mg::MAXK) throw Error(TOO_LARGE, "stage larger than 12 modules");
    for (int m : mods) {
        check_rows(m);
        if (opts_[m].empty()) {
            res.status = MODULE_NO_OPTION;
            co_return;
        }
    }
    const Interference& im = P_.im;
    const bool nonneg = im.non_negative();
    // tau_lo = max_m min bound, tau_hi = sum_m min solo rectified latency (stage_eval.hpp:
    // 318-335, 290-295): per-module minima computed once per problem (tau_mins_)
    double tau_lo = 0.0, tau_hi = 0.0;
    for (int m : mods) {
        if (nonneg) tau_lo = std::max(tau_lo, tau_mins_[m].first);
        tau_hi += tau_mins_[m].second;
    }
    bool have_T = false;
    double Tstar = POS_INF;
    std::vector<Entry> argmin;  // an allocation reaching Tstar
    long long probes = 0;
    SearchOp op;
    // small stages (<= fuse_k modules, or option tuples x G <= fuse_tree): the MIN proof does
    // not need the first probe's leaf as its bound, so it runs in the same wave as that probe
    // (ub = +inf) — one launch fewer; larger trees are cheaper to prove below the probe's
    // leaf in a second wave
    SearchOp mop;
    std::vector<int> mop_order;
    bool fuse_min = nonneg && (int)mods.size() < eng_->tuning().restart_k;
    if (fuse_min) {
        double tuples = (double)P_.gpu_count;
        for (int m : mods) tuples *= (double)std::max<size_t>(1, opts_[m].size());
        fuse_min = (int)mods.size() <= eng_->tuning().fuse_k || tuples <= eng_->tuning().fuse_tree;
    }
    bool min_ran = false, min_awaited = false, min_used = false;
    // FeasibilitySearch::run(tau) replayed: the first leaf in fail-first DFS order.
    // T* lies in [Tstar*(1 - TIE_EPS - rounding), Tstar]: below that band no leaf reaches
    // tau; inside it the probe is decided by an exact FIRST search, seeded with the argmin.
#define MG_RUN_PROBE(TAU, LEAF, ORDER, OK)                                                  \
    do {                                                                                   \
        const double tau_ = (TAU);                                                         \
        ++probes;                                                                          \
        bool ok_ = false;                                                                  \
        const double th_ = tau_ * (1.0 + 1e-12);                                           \
        std::vector<std::pair<int, int>> cnt_;                                             \
        bool none_ = false;                                                                \
        for (int m_ : mods) {                                                              \
            const auto& b_ = M_.index[m_].bound; /* rows with bound <= th, sorted */       \
            const int c_ = (int)(std::upper_bound(b_.begin(), b_.end(), th_) - b_.begin()); \
            if (c_ == 0) none_ = true;                                                     \
            cnt_.push_back({c_, m_});                                                      \
        }                                                                                  \
        if (!none_ && !(nonneg && have_T && th_ < Tstar * (1.0 - 1e-13))) {                \
            std::stable_sort(cnt_.begin(), cnt_.end());                                    \
            ORDER.clear();                                                                 \
            for (auto& [c_, m_] : cnt_) ORDER.push_back(m_);                               \
            const bool seed_ = nonneg && have_T && !argmin.empty() && Tstar <= th_;        \
            if (prep_first(ORDER, true, th_, op, res.st, seed_ ? &argmin : nullptr, Tstar)) { \
                if (fuse_min) { /* the MIN proof rides along with the first FIRST search */ \
                    fuse_min = false;                                                      \
                    min_ran = prep_min(mods, POS_INF, mop, res.st, mop_order);             \
                }                                                                          \
                if (min_ran && !min_used && !min_awaited) {                                \
                    min_awaited = true;                                                    \
                    co_await SearchAwait2{&op, &mop};                                      \
                } else {                                                                   \
                    co_await SearchAwait{&op};                                             \
                }                                                                          \
                const mg::SearchResult sr_ = op.res;                                       \
                if (sr_.overflow) throw Error(TOO_LARGE, "stage needs more than 128 GPU blocks"); \
                if (sr_.found) {                                                           \
                    LEAF = sr_.leaf;                                                       \
                    ok_ = true;                                                            \
                }                                                                          \
            }                                                                              \
        }                                                                                  \
        res.probe_tau.push_back(tau_);                                                     \
        res.probe_ok.push_back(ok_ ? 1 : 0);                                               \
        OK = ok_;                                                                          \
    } while (0)
    Leaf best, cur;
    std::vector<int> best_order, cur_order;
    bool ok = false;
    MG_RUN_PROBE(tau_hi, best, best_order, ok);
    for (int attempt = 0; !ok && attempt < 60; ++attempt) {
        tau_hi *= 2.0;
        MG_RUN_PROBE(tau_hi, best, best_order, ok);
    }
    res.probes = probes;
    if (!ok) {
        res.status = INFEASIBLE;
        co_return;
    }
    double t_best = best.value;
    if (nonneg) {
        // T*: one MIN proof below the first leaf's value, restarted with re-derived static
        // bounds whenever the incumbent drops by more than 1e-4
        argmin = leaf_entries(best_order, best);
        double ub = t_best;
        std::vector<int> morder;
        if (min_awaited && mop.res.found) {
            // the ridden-along MIN proof (ub = +inf, no restarts): T* within the tie band
            // of the minimum, bounded by the probe's leaf like the sequential proof
            const mg::SearchResult& r = mop.res;
            if (r.overflow) throw Error(TOO_LARGE, "stage needs more than 128 GPU blocks");
            min_used = true;
            if (r.value < t_best) {
                if (r.leaf.nb > 0) argmin = leaf_entries(mop_order, r.leaf);
                Tstar = r.value;
            } else {
                Tstar = t_best;
            }
        }
        while (!min_used) {
            if (!prep_min(mods, ub, op, res.st, morder)) {
                Tstar = ub;
                break;
            }
            const mg::SearchResult r = co_await SearchAwait{&op};
            if (r.overflow) throw Error(TOO_LARGE, "stage needs more than 128 GPU blocks");
            if (r.found && r.leaf.nb > 0) argmin = leaf_entries(morder, r.leaf);
            if (r.aborted) {
                ub = r.value;
                continue;
            }
            Tstar = r.value;
            break;
        }
        have_T = true;
    }
    double lo = std::min(tau_lo, t_best);
    while (t_best - lo > P_.bisect_rel_tol * std::abs(t_best)) {
        double mid = 0.5 * (lo + t_best);
        if (mid >= t_best * (1.0 - 1e-12)) break;
        MG_RUN_PROBE(mid, cur, cur_order, ok);
        if (ok) {
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
        MG_RUN_PROBE(probe, cur, cur_order, ok);
        if (!ok) break;
        best = cur;
        best_order = cur_order;
        t_best = best.value;
    }
#undef MG_RUN_PROBE
    res.status = OK;
    res.stage_time = t_best;
    res.entries = leaf_entries(best_order, best);
    res.probes = probes;
}

// ExactStageSolver::solve (oracle.hpp:86-103) as a coroutine: FIRST(inf) for an incumbent,
// MIN for I*, then the tie band resolved exactly — FIRST(theta) yields a leaf of value
// v <= theta; lower theta below v until no leaf remains: then v == T* and the last leaf is
// the first argmin in module-index DFS order (the reference's strict '<', oracle.hpp:120).
StageJob Planner::exact_stage_job(uint64_t mask, StageResult* out) {
    StageResult& res = *out;
    const auto mods = mask_modules(mask);
    if ((int)mods.size() > mg::MAXK) throw Error(TOO_LARGE, "stage larger than 12 modules");
    for (int m : mods) {
        check_rows(m);
        if (opts_[m].empty()) {
            res.status = INFEASIBLE;  // ExactStageSolver returns nullopt (oracle.hpp:91-92)
            co_return;
        }
    }
    SearchOp op;
    if (!M_.nonneg()) {
        // With a negative coefficient ExactStageSolver's option cut (`lb >= best_time_`,
        // lb = base latency, oracle.hpp:127-139) is not a bound: its answer is the best leaf
        // its sequential DFS happens to visit.  Replayed exactly: one walker in the
        // reference's DFS order, the same cut against the running incumbent, strict
        // improvements (the first argmin among visited leaves, oracle.hpp:120).
        mg::SearchReq q;
        q.mode = MODE_MIN;
        q.ub = POS_INF;
        q.level_module = mods;
        op.req = mg::BatchReq{};
        if (!mg::build_spec(M_, q, op.req.S)) {
            res.status = INFEASIBLE;
            co_return;
        }
        op.req.S.seq_cut = 1;
        op.req.ub = POS_INF;
        op.req.abort_below = 0.0;
        op.req.force_solo = true;
        op.req.st = &res.st;
        const mg::SearchResult sr = co_await SearchAwait{&op};
        if (sr.overflow) throw Error(TOO_LARGE, "stage needs more than 128 GPU blocks");
        if (!sr.found) {
            res.status = INFEASIBLE;
            co_return;
        }
        res.status = OK;
        res.stage_time = sr.leaf.value;
        res.entries = leaf_entries(mods, sr.leaf);
        co_return;
    }
    if (!prep_first(mods, false, POS_INF, op, res.st)) {
        res.status = INFEASIBLE;
        co_return;
    }
    mg::SearchResult r = co_await SearchAwait{&op};
    if (r.overflow) throw Error(TOO_LARGE, "stage needs more than 128 GPU blocks");
    if (!r.found) {
        res.status = INFEASIBLE;
        co_return;
    }
    double T = r.leaf.value;
    std::vector<int> morder;
    while (true) {
        if (!prep_min(mods, T, op, res.st, morder)) break;
        r = co_await SearchAwait{&op};
        if (r.overflow) throw Error(TOO_LARGE, "stage needs more than 128 GPU blocks");
        if (r.aborted) {
            T = r.value;
            continue;
        }
        T = r.value;
        break;
    }
    if (!prep_first(mods, false, T, op, res.st)) throw Error(CUDA, "exact search lost the argmin leaf");
    r = co_await SearchAwait{&op};
    if (r.overflow) throw Error(TOO_LARGE, "stage needs more than 128 GPU blocks");
    if (!r.found) throw Error(CUDA, "exact search lost the argmin leaf");
    Leaf lf = r.leaf;
    for (int guard = 0; guard < 64; ++guard) {
        const double below = std::nextafter(lf.value, -POS_INF);
        if (!prep_first(mods, false, below, op, res.st)) break;
        r = co_await SearchAwait{&op};
        if (r.overflow) throw Error(TOO_LARGE, "stage needs more than 128 GPU blocks");
        if (!r.found) break;
        lf = r.leaf;
    }
    res.status = OK;
    res.stage_time = lf.value;
    res.entries = leaf_entries(mods, lf);
}

// Advance every job to its next device search; run each wave of pending searches as one
// batched launch; repeat until all jobs are done.  The first exception is rethrown.
void Planner::run_jobs(std::vector<StageJob>& jobs, std::vector<char>* failed) {
    const bool trace = eng_->tuning().trace;
    double t_host = 0.0, t_dev = 0.0, t0 = now_s();
    for (auto& j : jobs) j.h.resume();
    std::vector<mg::BatchReq> reqs;
    std::vector<StageJob*> who;
    int waves = 0;
    while (true) {
        reqs.clear();
        who.clear();
        for (auto& j : jobs)
            if (!j.h.done() && j.h.promise().op) {
                reqs.push_back(j.h.promise().op->req);
                who.push_back(&j);
                if (j.h.promise().op2) reqs.push_back(j.h.promise().op2->req);
            }
        if (reqs.empty()) break;
        const double t1 = now_s();
        t_host += t1 - t0;
        std::vector<mg::SearchResult> res = eng_->search_batch(reqs);
        t0 = now_s();
        t_dev += t0 - t1;
        ++waves;
        size_t r = 0;
        for (size_t i = 0; i < who.size(); ++i) {
            auto& pr = who[i]->h.promise();
            pr.op->res = res[r++];
            if (pr.op2) pr.op2->res = res[r++];
            pr.op = nullptr;
            pr.op2 = nullptr;
            who[i]->h.resume();
        }
    }
    t_host += now_s() - t0;
    if (trace)
        std::fprintf(stderr, "[mosaic] batch of %zu: %d waves, host %.3f ms, launches %.3f ms\n",
                     jobs.size(), waves, 1e3 * t_host, 1e3 * t_dev);
    if (failed) {  // tolerant: report which jobs threw instead of rethrowing
        failed->assign(jobs.size(), 0);
        for (size_t i = 0; i < jobs.size(); ++i) (*failed)[i] = jobs[i].h.promise().exc != nullptr;
        return;
    }
    for (auto& j : jobs)
        if (j.h.promise().exc) std::rethrow_exception(j.h.promise().exc);
}

std::vector<StageResult> Planner::stage_batch(const std::vector<uint64_t>& masks, bool exact,
                                              std::vector<char>* failed) {
    std::vector<StageResult> out(masks.size());
    std::vector<StageJob> jobs;
    jobs.reserve(masks.size());
    for (size_t i = 0; i < masks.size(); ++i)
        jobs.push_back(exact ? exact_stage_job(masks[i], &out[i])
                             : stage_eval_job(masks[i], &out[i]));
    run_jobs(jobs, failed);
    return out;
}

StageResult Planner::stage_eval(uint64_t mask) { return std::move(stage_batch({mask}, false)[0]); }

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
            const double a = (double)e.units / (e.levels ? e.levels : P_.quota_levels);
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
    // one MIN search in the level order stage_eval's proofs use (prep_min)
    SearchOp op;
    std::vector<int> morder;
    if (!prep_min(mods, ub, op, st, morder)) return ub;
    mg::SearchResult r = eng_->search(op.req.S, ub, 0.0, st);
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

StageResult Planner::exact_stage(uint64_t mask) { return std::move(stage_batch({mask}, true)[0]); }

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
    StageResult r;
    auto sp = spec_.find(mask);
    if (sp != spec_.end()) {
        r = sp->second;  // computed ahead in this round's batch (deterministic: same result)
    } else {
        r = stage_eval(mask);
        pr.st.nodes += r.st.nodes;
        pr.st.leaves += r.st.leaves;
        pr.st.searches += r.st.searches;
        pr.st.rounds += r.st.rounds;
    }
    if (r.status == MODULE_NO_OPTION)
        throw Error(MODULE_NO_OPTION, "module has no feasible deployment option");
    if (r.status != OK) return std::nullopt;
    pr.feasibility_calls += r.probes;
    if (P_.enable_cache && cache_.emplace(mask, r).second) cache_order_.push_back(mask);
    return r;
}

// Evaluate `masks` (not cached, not yet computed) as one batch ahead of the reference's
// sequential candidate loop; the loop then consumes the results in its own order.
void Planner::speculate(const std::vector<uint64_t>& masks, PlanResult& pr) {
    std::vector<uint64_t> todo;
    for (uint64_t m : masks)
        if ((!P_.enable_cache || !cache_.count(m)) && !spec_.count(m) &&
            std::find(todo.begin(), todo.end(), m) == todo.end())
            todo.push_back(m);
    if (todo.empty()) return;
    // a candidate whose computation fails is simply not pre-computed: if the reference
    // evaluates it, the sequential loop recomputes it and raises exactly there
    std::vector<char> failed;
    std::vector<StageResult> rs = stage_batch(todo, false, &failed);
    for (size_t i = 0; i < todo.size(); ++i) {
        if (failed[i]) continue;
        pr.st.nodes += rs[i].st.nodes;
        pr.st.leaves += rs[i].st.leaves;
        pr.st.searches += rs[i].st.searches;
        pr.st.rounds += rs[i].st.rounds;
        spec_.emplace(todo[i], std::move(rs[i]));
    }
}

PlanResult Planner::solve() {
    const double t0 = now_s();
    PlanResult pr;
    const int n = (int)P_.modules.size();
    if (n == 0) throw Error(EMPTY, "model graph has no modules");
    clear_cache();
    spec_.clear();
    auto reach = reachability_masks(P_);
    std::vector<uint64_t> masks;
    std::vector<StageResult> results;
    {
        // round 0: every singleton in one batch
        std::vector<uint64_t> singles;
        for (int m : topological_order(P_)) singles.push_back(uint64_t(1) << m);
        speculate(singles, pr);
    }
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
        {
            // A1: every candidate the reference may evaluate this round, in one batch.  A
            // candidate with t_x + t_y - t_lb <= 0 is pruned whatever delta_best becomes (it
            // only grows from 0); large module sets are left to the sequential loop, which
            // skips the ones the reference prunes.
            std::vector<uint64_t> cands;
            for (auto [x, y] : pairs) {
                const uint64_t mm = masks[x] | masks[y];
                if (P_.enable_prune) {
                    double t_lb = 0.0;
                    for (int m : mask_modules(mm)) t_lb = std::max(t_lb, min_base[m]);
                    if (results[x].stage_time + results[y].stage_time - t_lb <= 0.0) continue;
                }
                if (std::popcount(mm) <= eng_->tuning().spec_k) cands.push_back(mm);
            }
            speculate(cands, pr);
        }
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
    spec_.clear();
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

bool Planner::ensure_rate_tables() {
    if (rate_tables_) return rate_tables_ > 0;
    const int n = (int)P_.modules.size(), G = P_.gpu_count, L = P_.quota_levels;
    const double bytes = 8.0 * n * ((double)G + 1.0) * (L + 1.0);
    if (bytes > 512.0 * 1024 * 1024) {
        rate_tables_ = -1;
        return false;
    }
    std::vector<double> base((size_t)n * G * (L + 1)), B((size_t)n * (L + 1));
    for (int m = 0; m < n; ++m)
        P_.modules[m].surface.rate_tables(G, L, base.data() + (size_t)m * G * (L + 1),
                                          B.data() + (size_t)m * (L + 1));
    eng_->set_rate_tables(base, B, n, G, L, M_);
    rate_tables_ = 1;
    return true;
}

static void raise_eval_errors(int err) {
    if (err & mg::EVAL_ERR_ENTRIES)
        throw Error(TOO_LARGE, "evaluator supports 64 entries per stage (or bad alloc_off)");
    if (err & mg::EVAL_ERR_MODULE) throw Error(RANGE, "module not in graph");
    if (err & mg::EVAL_ERR_GPU) throw Error(RANGE, "GPU index out of range");
    if (err & mg::EVAL_ERR_SURFACE) throw Error(RANGE, "(d, quota) outside the profiled surface");
    if (err & mg::EVAL_ERR_LEVELS)
        throw Error(RANGE, "entry quota_levels differs from the context's");
}

void Planner::evaluate(const mg::EvalABI* ent, long long n_ent, const int* gpus,
                       long long n_gpu_ids, const long long* off, long long n, double* st,
                       double* rect, bool device_ptrs) {
    if (n < 0 || n_ent < 0 || n_gpu_ids < 0) throw Error(RANGE, "negative size");
    if (n == 0) return;
    if (!ensure_rate_tables())
        throw Error(TOO_LARGE, "rate tables too large for this problem; use stage_time");
    raise_eval_errors(eng_->evaluate_abi(ent, n_ent, gpus, n_gpu_ids, off, n, st, rect,
                                         device_ptrs));
}

void Planner::stage_time(const std::vector<std::vector<Entry>>& allocs, std::vector<double>& st,
                         std::vector<std::vector<double>>& rect) {
    for (const auto& a : allocs)
        if (a.size() > 64) throw Error(TOO_LARGE, "evaluator supports 64 entries per stage");
    bool table_ok = true;
    for (const auto& a : allocs)
        for (const auto& e : a)
            if (e.levels != 0 && e.levels != P_.quota_levels) table_ok = false;
    if (table_ok && ensure_rate_tables()) {
        // K1 on the ABI layout
        std::vector<mg::EvalABI> ent;
        std::vector<int> gpus;
        std::vector<long long> off{0};
        for (const auto& a : allocs) {
            for (const auto& e : a) {
                ent.push_back(mg::EvalABI{e.module, e.d, e.units, (int)e.gpus.size(), e.levels, 0,
                                          (long long)gpus.size()});
                gpus.insert(gpus.end(), e.gpus.begin(), e.gpus.end());
            }
            off.push_back((long long)ent.size());
        }
        st.assign(allocs.size(), 0.0);
        std::vector<double> rflat(ent.size(), 0.0);
        raise_eval_errors(eng_->evaluate_abi(ent.data(), (long long)ent.size(), gpus.data(),
                                             (long long)gpus.size(), off.data(),
                                             (long long)allocs.size(), st.data(), rflat.data(),
                                             false));
        rect.assign(allocs.size(), {});
        for (size_t i = 0; i < allocs.size(); ++i)
            rect[i].assign(rflat.begin() + off[i], rflat.begin() + off[i + 1]);
        return;
    }
    // entries at another quota granularity: per-call rate rows (k_eval)
    std::vector<mg::EvalEntry> ent;
    std::vector<int> gpus;
    std::vector<long long> off{0};
    std::vector<double> base, Bt;
    std::unordered_map<uint64_t, int> row_of;  // (module, d, units, levels) -> table row
    for (const auto& a : allocs) {
        for (const auto& e : a) {
            if (e.module < 0 || e.module >= (int)P_.modules.size())
                throw Error(RANGE, "module not in graph");
            const int lv = e.levels ? e.levels : P_.quota_levels;
            const uint64_t key = (uint64_t)e.module << 48 | (uint64_t)(uint32_t)e.d << 32 |
                                 (uint64_t)(uint32_t)e.units << 16 | (uint64_t)(uint32_t)lv;
            auto it = row_of.find(key);
            int row;
            if (it == row_of.end()) {
                const Surface& s = P_.modules[e.module].surface;
                double a = (double)e.units / lv;
                base.push_back(s.lookup(e.d, a).latency);      // PerfContext::base_latency
                Bt.push_back(s.lookup(1, a).bandwidth_util);   // PerfContext::solo_bandwidth (eager)
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
        off.push_back((long long)ent.size());
    }
    std::vector<double> rflat;
    eng_->evaluate(ent, gpus, off, base, Bt, P_.gpu_count, M_, st, rflat);
    rect.assign(allocs.size(), {});
    for (size_t i = 0; i < allocs.size(); ++i)
        rect[i].assign(rflat.begin() + off[i], rflat.begin() + off[i + 1]);
}

}  // namespace mosaic_b200

// ---------------------------------------------------------------------------
// N4: exclusive-allocation baselines and batched plan replay (simulator.hpp)
// ---------------------------------------------------------------------------
namespace mosaic_b200 {

// rectified_latency of module m alone on d GPUs at full quota (perf_model.hpp:442-464 with a
// single resident per GPU: sum = 0 + b, prod = 1 * b; no residents when include_self is off)
double Planner::exclusive_latency(int m, int d) const {
    const Surface& s = P_.modules[m].surface;
    const double a = (double)P_.quota_levels / P_.quota_levels;
    const double base = s.lookup(d, a).latency;
    double sum = 0.0, prod = 1.0;
    if (P_.include_self) {
        const double b = s.lookup(1, a).bandwidth_util;
        sum += b;
        prod *= b;
    } else {
        prod = 0.0;
    }
    const double dl = P_.im.delta(sum, prod);
    const double worst = std::max(-1e300, dl);
    return base + worst;
}

// detail::dependency_waves, simulator.hpp:144-193
std::vector<std::vector<int>> Planner::dependency_waves() const {
    const int n = (int)P_.modules.size(), G = P_.gpu_count;
    const std::vector<int> topo = topological_order(P_);
    std::vector<int> depth(n, 0);
    for (int u : topo)
        for (auto [a, b] : P_.edges)
            if (a == u) depth[b] = std::max(depth[b], depth[u] + 1);
    int max_depth = 0;
    for (int d : depth) max_depth = std::max(max_depth, d);
    std::vector<std::vector<int>> waves;
    for (int lvl = 0; lvl <= max_depth; ++lvl) {
        std::vector<int> level;
        for (int m : topo)
            if (depth[m] == lvl) level.push_back(m);
        if (level.empty()) continue;
        const int wave_count = ((int)level.size() + G - 1) / G;
        std::vector<std::pair<double, int>> load;
        for (int m : level) {
            const Surface& s = P_.modules[m].surface;
            load.push_back({s.lookup(s.min_d(), s.max_a()).latency, m});
        }
        std::sort(load.begin(), load.end(), [](const auto& x, const auto& y) {
            if (x.first != y.first) return x.first > y.first;
            return x.second < y.second;
        });
        std::vector<std::vector<int>> split(wave_count);
        std::vector<double> totals(wave_count, 0.0);
        for (const auto& [lat, m] : load) {
            int target = 0;
            for (int w = 1; w < wave_count; ++w) {
                if ((int)split[w].size() >= G) continue;
                if ((int)split[target].size() >= G || totals[w] < totals[target]) target = w;
            }
            split[target].push_back(m);
            totals[target] += lat;
        }
        for (auto& wv : split) {
            std::sort(wv.begin(), wv.end());
            waves.push_back(std::move(wv));
        }
    }
    return waves;
}

// detail::distmm_wave, simulator.hpp:217-279.  The reference enumerates every composition
// (d_0..d_k-1) of at most G GPUs in ascending lexicographic order and keeps the first with
// the smallest wave time.  With every module exclusive on its own GPUs the wave time is
// max(0, max_i f_i(d_i)), f_i = exclusive_latency, so that first minimiser is closed-form:
// T* = the smallest threshold t for which the per-module minimal admissible degrees
// m_i(t) = min{d : degree_ok, f_i(d) <= t} fit in G GPUs, and the lexicographically first
// composition reaching T* is (m_0(T*), ..., m_k-1(T*)).  The k > 8 greedy is restated.
std::vector<Entry> Planner::distmm_wave(const std::vector<int>& wave) const {
    const int k = (int)wave.size(), G = P_.gpu_count, L = P_.quota_levels;
    const int max_d = P_.modules[wave[0]].surface.max_d();
    const double a = (double)L / L;
    auto degree_ok = [&](int m, int d) {
        const Surface& s = P_.modules[m].surface;
        if (d > s.max_d()) return false;
        return s.lookup(d, a).memory + P_.modules[m].memory_base <= P_.memory_capacity;
    };
    for (int i = 0; i < k; ++i)
        if (!degree_ok(wave[i], 1))
            throw Error(BASELINE_INFEASIBLE, "module " + P_.modules[wave[i]].id +
                                                 " does not fit one GPU at full quota");
    auto wave_time = [&](const std::vector<int>& deg) {
        double worst = 0.0;
        for (int i = 0; i < k; ++i) worst = std::max(worst, exclusive_latency(wave[i], deg[i]));
        return worst;
    };
    std::vector<int> degrees(k, 1);
    if (k <= 8) {
        const int dmax = std::min(max_d, G - (k - 1));
        std::vector<std::vector<double>> f(k, std::vector<double>(dmax + 1, 0.0));
        std::vector<std::vector<char>> ok(k, std::vector<char>(dmax + 1, 0));
        std::vector<double> cand{0.0};
        for (int i = 0; i < k; ++i)
            for (int d = 1; d <= dmax; ++d)
                if (degree_ok(wave[i], d)) {
                    ok[i][d] = 1;
                    f[i][d] = exclusive_latency(wave[i], d);
                    cand.push_back(f[i][d]);
                }
        auto minimal = [&](double t, std::vector<int>* out) {
            int used = 0;
            for (int i = 0; i < k; ++i) {
                int m = 0;
                for (int d = 1; d <= dmax && !m; ++d)
                    if (ok[i][d] && !(f[i][d] > t)) m = d;
                if (!m) return false;
                used += m;
                if (out) (*out)[i] = m;
            }
            return used <= G;
        };
        std::sort(cand.begin(), cand.end());
        cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
        // feasibility is monotone in t; thresholds below 0 collapse to 0 (wave_time's clamp)
        size_t lo = 0, hi = cand.size();
        while (lo < hi) {
            const size_t mid = (lo + hi) / 2;
            if (minimal(std::max(0.0, cand[mid]), nullptr)) hi = mid; else lo = mid + 1;
        }
        if (lo == cand.size()) throw Error(BASELINE_INFEASIBLE, "no DistMM composition fits");
        minimal(std::max(0.0, cand[lo]), &degrees);
    } else {
        int used = k;
        while (used < G) {
            const double cur_time = wave_time(degrees);
            std::vector<std::pair<double, int>> lat(k);
            for (int i = 0; i < k; ++i) lat[i] = {exclusive_latency(wave[i], degrees[i]), i};
            std::sort(lat.rbegin(), lat.rend());
            const int worst = lat[0].second;
            std::vector<int> trial = degrees;
            trial[worst]++;
            if (trial[worst] > max_d || !degree_ok(wave[worst], trial[worst])) break;
            if (wave_time(trial) >= cur_time) break;
            degrees = trial;
            ++used;
        }
    }
    std::vector<Entry> out;
    int next = 0;
    for (int i = 0; i < k; ++i) {
        Entry e{wave[i], degrees[i], L, {}};
        for (int g = 0; g < degrees[i]; ++g) e.gpus.push_back(next + g);
        next += degrees[i];
        out.push_back(std::move(e));
    }
    std::sort(out.begin(), out.end(), [](const Entry& x, const Entry& y) { return x.module < y.module; });
    return out;
}

PlanResult Planner::baseline_plan(int policy) {
    const int G = P_.gpu_count, L = P_.quota_levels;
    std::vector<std::vector<Entry>> stages;
    if (policy == 0) {  // Megatron: every module alone on all GPUs, topological order
        for (int m : topological_order(P_)) {
            const Surface& s = P_.modules[m].surface;
            if (G > s.max_d())
                throw Error(BASELINE_INFEASIBLE, "gpu_count exceeds profiled DP range");
            const double a = (double)L / L;
            if (s.lookup(G, a).memory + P_.modules[m].memory_base > P_.memory_capacity)
                throw Error(BASELINE_INFEASIBLE, "module " + P_.modules[m].id +
                                                     " exceeds GPU memory at forced degree");
            Entry e{m, G, L, {}};
            for (int g = 0; g < G; ++g) e.gpus.push_back(g);
            stages.push_back({e});
        }
    } else {
        for (const auto& wave : dependency_waves()) stages.push_back(distmm_wave(wave));
    }
    std::vector<double> st;
    std::vector<std::vector<double>> rect;
    stage_time(stages, st, rect);
    PlanResult pr;
    pr.status = OK;
    for (size_t i = 0; i < stages.size(); ++i) {
        StageResult r;
        r.status = OK;
        r.stage_time = st[i];
        r.entries = stages[i];
        uint64_t mask = 0;
        for (const auto& e : stages[i]) mask |= uint64_t(1) << e.module;
        pr.masks.push_back(mask);
        pr.stages.push_back(std::move(r));
        pr.iteration_time += st[i];
    }
    return pr;
}

void Planner::simulate(const std::vector<std::vector<Entry>>& stages, const mg::SimCfg& cfg,
                       const std::vector<uint64_t>& seeds, std::vector<double>& iter,
                       std::vector<double>& per_stage, std::vector<double>& busy,
                       std::vector<double>& mean_busy, std::vector<mg::SimInterval>* timeline) {
    if (cfg.iterations < 1) throw Error(INVALID_ARGUMENT, "iterations must be >= 1");
    if (cfg.pooled_overhead < 0 || cfg.on_demand_overhead < 0)
        throw Error(INVALID_ARGUMENT, "overheads must be >= 0");
    std::vector<double> st;
    std::vector<std::vector<double>> rect;
    stage_time(stages, st, rect);  // rectified latencies of every entry, on the device
    std::vector<mg::SimEntry> ents;
    std::vector<int> gpus, off{0};
    for (size_t s = 0; s < stages.size(); ++s) {
        for (size_t i = 0; i < stages[s].size(); ++i) {
            const Entry& e = stages[s][i];
            // rectified_latency(ctx, stage, e.module) looks the module up with find():
            // its first entry in the stage
            size_t first = i;
            for (size_t j = 0; j < i; ++j)
                if (stages[s][j].module == e.module) { first = j; break; }
            const double q = (double)e.units / (e.levels ? e.levels : P_.quota_levels);
            const Sample smp = P_.modules[e.module].surface.lookup(e.d, q);
            mg::SimEntry se{};
            se.dur0 = rect[s][first];
            se.quota = q;
            se.active_cap = smp.sm_active * smp.latency;
            se.module = e.module;
            se.gpu_off = (int)gpus.size();
            se.n_gpus = (int)e.gpus.size();
            ents.push_back(se);
            gpus.insert(gpus.end(), e.gpus.begin(), e.gpus.end());
        }
        off.push_back((int)ents.size());
    }
    mg::simulate_device(ents, gpus, off, P_.gpu_count, cfg, seeds, eng_->device(), iter,
                        per_stage, busy, mean_busy, timeline);
}

}  // namespace mosaic_b200
