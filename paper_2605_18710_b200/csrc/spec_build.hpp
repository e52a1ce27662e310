// spec_build.hpp — host side: turn one stage search request into the device Spec.
//
// The option rows of every module live in one device table in candidate_options
// order (stage_eval.hpp:68-93).  A level's list is a PREFIX of its module's rows:
// rows are sorted by base latency, and once base+e1 exceeds the threshold no later
// row can pass (stage_eval.hpp:122-127 filter / oracle.hpp:130-135 bound), so the
// prefix is all the device ever needs to scan.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "search_core.cuh"

namespace mg {

struct OptRow {
    int d, u;
    double base, B, fp, bound;
};

// Per module, the rows re-sorted by filter bound with prefix aggregates: with non-negative
// coefficients a row is usable at threshold t iff bound <= t, so the per-level summary
// build_spec needs (min quota demand, min solo bandwidth, all options full-width) is one
// binary search instead of a scan over the module's options.
struct BoundIndex {
    std::vector<double> bound;   // ascending
    std::vector<int> min_dem;    // prefix min of d*u
    std::vector<double> min_B;   // prefix min of B
    std::vector<int> not_full;   // prefix count of d != G
};

struct Model {
    int G = 1, L = 10;
    double cap = 80e9, e1 = 0, e2 = 0, e3 = 0;
    bool additive = false, include_self = true;
    bool nonneg() const { return e1 >= 0 && e2 >= 0 && (additive || e3 >= 0); }
    std::vector<std::vector<OptRow>> rows;  // per module, candidate_options order
    std::vector<int> row_off;               // per module offset into the flat table
    std::vector<BoundIndex> index;          // build_index(); empty: build_spec scans
};

inline void build_index(Model& M) {
    M.index.assign(M.rows.size(), {});
    for (size_t m = 0; m < M.rows.size(); ++m) {
        std::vector<const OptRow*> v;
        for (const auto& r : M.rows[m]) v.push_back(&r);
        std::stable_sort(v.begin(), v.end(),
                         [](const OptRow* a, const OptRow* b) { return a->bound < b->bound; });
        BoundIndex& ix = M.index[m];
        int dem = INT32_MAX, nf = 0;
        double bm = POS_INF;
        for (const OptRow* r : v) {
            dem = std::min(dem, r->d * r->u);
            bm = std::min(bm, r->B);
            nf += r->d != M.G;
            ix.bound.push_back(r->bound);
            ix.min_dem.push_back(dem);
            ix.min_B.push_back(bm);
            ix.not_full.push_back(nf);
        }
    }
}

// Filter bound exactly as FeasibilitySearch::run computes it (stage_eval.hpp:122-127).
inline double filter_bound(const Model& M, double base, double B) {
    double bound = base;
    if (M.nonneg()) {
        bound += M.e1;
        if (M.include_self) bound += M.e2 * B;
    }
    return bound;
}

struct SearchReq {
    int mode = MODE_FIRST;
    bool use_filter = false;
    double theta = POS_INF;  // FIRST acceptance threshold
    double ub = POS_INF;     // MIN: incumbent upper bound (an achieved value or +inf)
    std::vector<int> level_module;  // level -> module index (pi)
};

// Returns false if some level has no usable row (then no leaf can exist).
inline bool build_spec(const Model& M, const SearchReq& q, Spec& S) {
    const int k = (int)q.level_module.size();
    S = Spec{};
    S.k = k;
    S.G = M.G;
    S.L = M.L;
    S.mode = q.mode;
    S.nonneg = M.nonneg();
    S.include_self = M.include_self;
    S.additive = M.additive;
    S.use_filter = q.use_filter;
    S.shard_rank = 0;
    S.shard_world = 1;
    S.shard_level = 0;
    S.e1 = M.e1;
    S.e2 = M.e2;
    S.e3 = M.e3;
    S.cap_slack = M.cap * (1.0 + 1e-12);
    S.theta = q.theta;
    if (q.mode == MODE_MIN)
        S.thp = q.ub >= POS_INF ? POS_INF : q.ub * (1.0 - TIE_EPS);
    else
        S.thp = q.theta >= POS_INF ? POS_INF : q.theta * (1.0 + 1e-12);
    // module-index position -> level (no heap: this runs once per device search)
    std::pair<int, int> ml[MAXK];
    for (int l = 0; l < k; ++l) ml[l] = {q.level_module[l], l};
    std::sort(ml, ml + k);
    for (int p = 0; p < k; ++p) S.pos_lvl[p] = ml[p].second;

    double bmin[MAXK];
    int forced[MAXK], dmin[MAXK];
    for (int l = 0; l < k; ++l) {
        bmin[l] = 1.0;
        forced[l] = 1;
        dmin[l] = 0;
    }
    // fast path (non-negative coefficients, index built): the option list stops at the first
    // row with base + e1 above the threshold (rows are sorted by base latency); a row is usable
    // iff its bound (= base + e1 [+ e2 B]) is within the threshold — the scan below, exactly
    const bool fast = S.nonneg && !M.index.empty();
    const double t_stop = q.use_filter ? q.theta : S.thp;
    for (int l = 0; l < k && fast; ++l) {
        const int m = q.level_module[l];
        const auto& rows = M.rows[m];
        const BoundIndex& ix = M.index[m];
        S.lvl_off[l] = M.row_off[m];
        int lo = 0, hi = (int)rows.size();  // first row with base + e1 > t_stop
        while (lo < hi) {
            const int mid = (lo + hi) / 2;
            if (rows[mid].base + M.e1 > t_stop) hi = mid; else lo = mid + 1;
        }
        S.lvl_n[l] = lo;
        const int c = (int)(std::upper_bound(ix.bound.begin(), ix.bound.end(), t_stop) -
                            ix.bound.begin());
        if (c == 0) return false;
        dmin[l] = ix.min_dem[c - 1];
        bmin[l] = std::min(1.0, std::max(0.0, ix.min_B[c - 1]));
        forced[l] = ix.not_full[c - 1] == 0 ? 1 : 0;
    }
    for (int l = 0; l < k && !fast; ++l) {
        const int m = q.level_module[l];
        const auto& rows = M.rows[m];
        S.lvl_off[l] = M.row_off[m];
        int n = 0, best_dem = INT32_MAX;
        double bm = POS_INF;
        bool all_full = true;
        for (int i = 0; i < (int)rows.size(); ++i) {
            const OptRow& r = rows[i];
            // the same tests opt_test applies on the device, with the static threshold
            bool stop = false, skip = false;
            if (q.use_filter && r.bound > q.theta) {
                if (S.nonneg ? (r.base + M.e1 > q.theta) : (r.base > q.theta)) stop = true;
                skip = true;
            } else if (S.nonneg) {
                double be = r.base + M.e1;
                if (be > S.thp) stop = true;
                double lb = M.include_self ? be + M.e2 * r.B : be;
                if (lb > S.thp) skip = true;
            }
            if (stop) break;
            n = i + 1;
            if (skip) continue;
            best_dem = std::min(best_dem, r.d * r.u);
            bm = std::min(bm, r.B);
            if (r.d != M.G) all_full = false;
        }
        S.lvl_n[l] = n;
        if (best_dem == INT32_MAX) return false;
        dmin[l] = best_dem;
        bmin[l] = std::min(1.0, std::max(0.0, bm));
        forced[l] = all_full ? 1 : 0;
    }
    S.suffix_min[k] = 0;
    for (int l = k - 1; l >= 0; --l) S.suffix_min[l] = S.suffix_min[l + 1] + dmin[l];

    // Product-term envelope g_j(P) = min over subsets T of unplaced levels >= j that
    // contain every forced level of  e2*sum_T Bmin + e3*P*prod_T Bmin.  Lines dominated at
    // both ends of P in [0, 1] by another single line are dropped (ties: the lower index
    // stays).  Scratch vectors are reused across calls: this runs once per device search.
    const double e3 = S.additive ? 0.0 : M.e3;
    thread_local std::vector<double> la, lb;
    thread_local std::vector<int> kept;
    for (int j = 0; j <= k; ++j) {
        const int nf = k - j;
        la.clear();
        lb.clear();
        for (int T = 0; T < (1 << nf); ++T) {
            bool ok = true;
            double a = 0.0, b = e3;
            for (int i = 0; i < nf; ++i) {
                if (T >> i & 1) {
                    a += M.e2 * bmin[j + i];
                    b *= bmin[j + i];
                } else if (forced[j + i]) {
                    ok = false;
                }
            }
            if (ok) {
                la.push_back(a);
                lb.push_back(b);
            }
        }
        const int n = (int)la.size();
        kept.assign(n, 0);
        for (int i = 0; i < n; ++i) {
            bool dom = false;
            for (int h = 0; h < n && !dom; ++h) {
                if (h == i) continue;
                const bool le0 = la[h] <= la[i];
                const bool le1 = la[h] + lb[h] <= la[i] + lb[i];
                const bool strict = la[h] < la[i] || la[h] + lb[h] < la[i] + lb[i];
                if (le0 && le1 && (strict || h < i)) dom = true;
            }
            kept[i] = dom ? 0 : 1;
        }
        int nk = 0;
        for (int i = 0; i < n; ++i) nk += kept[i];
        if (nk > MAXENV) {
            // conservative: fall back to the weakest bound (min over all lines at P)
            double a = POS_INF;
            for (int i = 0; i < n; ++i)
                if (kept[i]) a = std::min(a, la[i]);
            S.env_n[j] = 1;
            S.env_a[j][0] = a * (1.0 - 1e-12);
            S.env_b[j][0] = 0.0;
        } else {
            // envelope is a lower bound: scale down by a hair so rounding cannot tighten it
            int c = 0;
            for (int i = 0; i < n; ++i)
                if (kept[i]) {
                    S.env_a[j][c] = la[i] * (1.0 - 1e-12);
                    S.env_b[j][c] = lb[i] * (1.0 - 1e-12);
                    ++c;
                }
            S.env_n[j] = c;
        }
        if (S.env_n[j] == 0) {
            S.env_n[j] = 1;
            S.env_a[j][0] = 0.0;
            S.env_b[j][0] = 0.0;
        }
    }
    return true;
}

}  // namespace mg
