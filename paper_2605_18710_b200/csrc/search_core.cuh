// search_core.cuh — per-thread canonical-placement branch-and-bound over one stage.
//
// What it searches (reference semantics, SURVEY.md §7 "Exact leaf order"):
//   levels j = 0..k-1 place module pi_j: choose an option (candidate_options order,
//   stage_eval.hpp:68-93) then a placement.  GPUs are kept as BLOCKS — maximal runs of
//   consecutive GPUs with identical resident sets, always contiguous — and a
//   placement takes a prefix of each eligible block (count vector x), visited in
//   descending lexicographic order of x.  That is exactly the set and order of leaves
//   FeasibilitySearch::place visits with its signature skip (stage_eval.hpp:204-214)
//   and, for ExactStageSolver (oracle.hpp:157-180), the order among canonical leaves,
//   which always contains its lexicographically-first argmin.
//
//   MODE_FIRST: first leaf in that DFS order whose stage_time <= theta
//               (FeasibilitySearch::run with theta = tau*(1+1e-12), filter
//               stage_eval.hpp:119-130; or the exact argmin with theta = T*).
//   MODE_MIN:   minimum stage_time over all leaves below an incumbent (T*).
//
// Leaf value is computed bit-exactly as stage_time (perf_model.hpp:442-479):
// residents summed in module-index order, (e1 + e2*sum) + e3*prod, base + worst,
// max starting at 0.0; the file is compiled with -fmad=false.  Because a block's
// contribution depends only on its resident set, the LAST level is resolved in
// closed form over blocks (per-block interval of admissible take counts) instead
// of enumerating its compositions.
//
// Pruning is sound and never reorders leaves: option filter/break, total quota
// demand (stage_eval.hpp:141-147,176-178), per-block capacity and memory
// (:208-210), an interference lower bound per block that adds a product-term
// envelope over the still-unplaced modules, and a one-step look-ahead that every
// unplaced module still has an option that fits.  All bound comparisons carry a
// 1e-12 relative slack so fp rounding can only weaken them.
#pragma once
#include <stdint.h>

#ifndef MG_HD
#define MG_HD __device__ __forceinline__
#endif
// Device code below is only compiled by nvcc (the host planner includes this header
// for the Spec/Node/Leaf layouts only; there is no host search path).
#if defined(__CUDACC__) || defined(MG_HOST_HARNESS)
#define MG_DEVICE_CODE 1
#endif

namespace mg {

constexpr int MAXK = 12;   // modules per stage
constexpr int MAXB = 128;  // blocks per level
constexpr int MAXENV = 16; // envelope lines per level
constexpr int FB = MAXB;   // blocks carried by a frontier node
constexpr double NEG_INF = -1.0e300;
constexpr double POS_INF = 1.0e300;
// MIN mode treats leaves within TIE_EPS (relative) of the incumbent as ties: it returns
// I* with T* in [I*(1 - TIE_EPS - rounding), I*].  Callers resolve a probe inside that
// band with an exact FIRST search (planner.cpp).
constexpr double TIE_EPS = 1e-14;

enum { MODE_MIN = 0, MODE_FIRST = 1 };

struct Spec {
    int k, G, L, mode;
    int nonneg, include_self, additive, use_filter;
    double e1, e2, e3, cap_slack;  // cap_slack = memory_capacity * (1 + 1e-12)
    double theta;                  // FIRST: accept iff stage_time <= theta
    double thp;                    // static prune threshold (theta or UB) * (1 + 1e-12)
    int lvl_n[MAXK];               // viable options per level (a prefix of the sorted list)
    int lvl_off[MAXK];             // row offset of each level's options
    int pos_lvl[MAXK];             // module-index position -> level
    int suffix_min[MAXK + 1];      // min quota demand d*u over levels >= j
    int shard_rank, shard_world;   // multi-GPU: this rank takes the option prefixes
    int shard_level;               //   (o_0..o_L) with shard_hash % world == rank, L = shard_level
    int env_n[MAXK + 1];           // product-term envelope over unplaced levels >= j
    double env_a[MAXK + 1][MAXENV];
    double env_b[MAXK + 1][MAXENV];
};

struct Rows {
    const double* base;
    const double* B;
    const double* fp;
    const double* bound;  // reference filter bound (stage_eval.hpp:122-127)
    const int* d;
    const int* u;
};

// Work item: a DFS cursor.  Levels < depth are placed; `ph` says how to continue at
// level `depth`: 0 = try the options after `oc`, 1 = try the compositions after `x` of
// option opt[depth] (within [lo, hi]).  The root is {depth 0, ph 0, oc -1}.  Items
// are ordered by `key`, which follows the reference DFS order.
struct alignas(16) Cont {
    unsigned long long key;
    uint16_t opt[MAXK];
    uint16_t depth, nb, ph;
    int16_t oc;
    int16_t oe;  // options at `depth` stop before oe (range split by work donation)
    int16_t pad16;
    int used;
    uint16_t bsz[MAXB];
    uint16_t bmk[MAXB];
    uint16_t x[MAXB];
    uint16_t lo[MAXB];
    uint16_t hi[MAXB];
};

// Position of a FIRST hit in the reference DFS order: (option, composition) per level.
struct HitPath {
    uint16_t opt[MAXK];
    uint16_t nb[MAXK];
    uint16_t x[MAXK][MAXB];
};

// Leaf: options of every level plus the final block list (sizes, level masks).
struct Leaf {
    double value;
    int nb;
    int pad;
    uint16_t opt[MAXK];
    uint16_t bsz[2 * MAXB];
    uint16_t bmk[2 * MAXB];
};

// Block storage offsets: level j holds at most min(2^j, MAXB) blocks.
#ifdef MG_DEVICE_CODE
MG_HD int lvl_cap(int j) { return j >= 7 ? MAXB : (1 << j); }
MG_HD int lvl_off(int j) {
    int off = 0;
    for (int i = 0; i < j; ++i) off += lvl_cap(i);
    return off;
}
#endif
constexpr int WALK_SLOTS = 255 + (MAXK + 1 - 8) * MAXB;  // sum_{j<=MAXK} lvl_cap(j)

struct Walk {
    uint16_t opt[MAXK];
    int16_t oc[MAXK];
    int16_t oe[MAXK];  // option range end per level (exclusive)
    uint8_t ph[MAXK];
    uint16_t nb[MAXK + 1];
    int used[MAXK + 1];
    uint16_t bsz[WALK_SLOTS];
    uint16_t bmk[WALK_SLOTS];
    uint16_t x[WALK_SLOTS];
    uint16_t lo[WALK_SLOTS];   // admissible take count per block: [lo, hi]
    uint16_t hi[WALK_SLOTS];
    // parent-block stats of level `ps_lvl` (recomputed when a deeper level overwrote them)
    int ps_lvl;
    int pu[MAXB];
    double pm[MAXB], psum[MAXB], pmb[MAXB], pP[MAXB], pmx[MAXB];
    // child-block stats (look-ahead) / last-level contributions
    int cu[MAXB];
    double cm[MAXB], cs[MAXB], cb[MAXB];
};

#ifdef MG_DEVICE_CODE
MG_HD double envelope(const Spec& S, int j, double P) {
    double g = POS_INF;
    for (int i = 0; i < S.env_n[j]; ++i) {
        double v = S.env_a[j][i] + S.env_b[j][i] * P;
        g = v < g ? v : g;
    }
    return S.env_n[j] ? g : 0.0;
}

// Exact contribution of one GPU block with resident levels `mask` (all k options set):
// max over residents m of base_m + delta(residents), module-index order sums.
MG_HD double contrib(const Spec& S, const Rows& R, const uint16_t* opt, unsigned mask) {
    if (!mask) return NEG_INF;
    if (S.include_self) {
        double s = 0.0, p = 1.0, mb = NEG_INF;
        for (int pos = 0; pos < S.k; ++pos) {
            int l = S.pos_lvl[pos];
            if (!(mask >> l & 1u)) continue;
            int r = S.lvl_off[l] + opt[l];
            double b = R.B[r];
            s = s + b;
            p = p * b;
            double ba = R.base[r];
            mb = ba > mb ? ba : mb;
        }
        double dl = S.e1 + S.e2 * s;
        dl = dl + (S.additive ? 0.0 : S.e3 * p);
        return mb + dl;
    }
    double best = NEG_INF;
    for (int pos = 0; pos < S.k; ++pos) {
        int l = S.pos_lvl[pos];
        if (!(mask >> l & 1u)) continue;
        double s = 0.0, p = 1.0;
        int n = 0;
        for (int pos2 = 0; pos2 < S.k; ++pos2) {
            int l2 = S.pos_lvl[pos2];
            if (l2 == l || !(mask >> l2 & 1u)) continue;
            double b = R.B[S.lvl_off[l2] + opt[l2]];
            s = s + b;
            p = p * b;
            ++n;
        }
        if (n == 0) p = 0.0;
        double dl = S.e1 + S.e2 * s;
        dl = dl + (S.additive ? 0.0 : S.e3 * p);
        double v = R.base[S.lvl_off[l] + opt[l]] + dl;
        best = v > best ? v : best;
    }
    return best;
}

// contrib() with the option of level `jl` replaced by `ol` (lanes evaluating different
// last-level options against the same shared walk).
MG_HD double contrib_o(const Spec& S, const Rows& R, const uint16_t* opt, unsigned mask, int jl,
                       int ol) {
    if (!mask) return NEG_INF;
    if (S.include_self) {
        double s = 0.0, p = 1.0, mb = NEG_INF;
        for (int pos = 0; pos < S.k; ++pos) {
            int l = S.pos_lvl[pos];
            if (!(mask >> l & 1u)) continue;
            int r = S.lvl_off[l] + (l == jl ? ol : opt[l]);
            double b = R.B[r];
            s = s + b;
            p = p * b;
            double ba = R.base[r];
            mb = ba > mb ? ba : mb;
        }
        double dl = S.e1 + S.e2 * s;
        dl = dl + (S.additive ? 0.0 : S.e3 * p);
        return mb + dl;
    }
    double best = NEG_INF;
    for (int pos = 0; pos < S.k; ++pos) {
        int l = S.pos_lvl[pos];
        if (!(mask >> l & 1u)) continue;
        double s = 0.0, p = 1.0;
        int n = 0;
        for (int pos2 = 0; pos2 < S.k; ++pos2) {
            int l2 = S.pos_lvl[pos2];
            if (l2 == l || !(mask >> l2 & 1u)) continue;
            double b = R.B[S.lvl_off[l2] + (l2 == jl ? ol : opt[l2])];
            s = s + b;
            p = p * b;
            ++n;
        }
        if (n == 0) p = 0.0;
        double dl = S.e1 + S.e2 * s;
        dl = dl + (S.additive ? 0.0 : S.e3 * p);
        double v = R.base[S.lvl_off[l] + (l == jl ? ol : opt[l])] + dl;
        best = v > best ? v : best;
    }
    return best;
}

// Owner rank of an option prefix (levels 0..j with level j's option o).
MG_HD unsigned shard_hash(const uint16_t* opt, int j, int o) {
    unsigned h = 2166136261u;
    for (int l = 0; l <= j; ++l) {
        h ^= (unsigned)(l == j ? o : opt[l]) + 0x9e37u * (unsigned)(l + 1);
        h *= 16777619u;
    }
    return h;
}

// 0 accept, 1 skip, 2 stop the option loop (all later options fail too).
MG_HD int opt_test(const Spec& S, const Rows& R, int r, double thr) {
    double base = R.base[r];
    if (S.use_filter && R.bound[r] > S.theta) {
        if (S.nonneg && base + S.e1 > S.theta) return 2;
        if (!S.nonneg && base > S.theta) return 2;
        return 1;
    }
    if (S.nonneg) {
        double be = base + S.e1;
        if (be > thr) return 2;
        double lb = S.include_self ? be + S.e2 * R.B[r] : be;
        if (lb > thr) return 1;
    }
    return 0;
}

// Stats of a block (levels < nlev in `mask`), accumulated in placement order like
// FeasibilitySearch::push_module (stage_eval.hpp:224-229).
MG_HD void block_stats(const Spec& S, const Rows& R, const uint16_t* opt, unsigned mask,
                       int nlev, int& units, double& mem, double& sum, double& mb,
                       double& P, double& mbx) {
    units = 0;
    mem = 0.0;
    sum = 0.0;
    mb = NEG_INF;
    P = 1.0;
    mbx = NEG_INF;  // max(base - e2*B): residents' own-excluded additive bound
    for (int l = 0; l < nlev; ++l) {
        if (!(mask >> l & 1u)) continue;
        int r = S.lvl_off[l] + opt[l];
        units += R.u[r];
        mem = mem + R.fp[r];
        sum = sum + R.B[r];
        P = P * R.B[r];
        double ba = R.base[r];
        mb = ba > mb ? ba : mb;
        double bx = ba - S.e2 * R.B[r];
        mbx = bx > mbx ? bx : mbx;
    }
}

MG_HD int hi_minus_x(const Walk& w, int i) { return (int)w.hi[i] - (int)w.x[i]; }

// First composition in descending lexicographic order with x_b in [lo_b, hi_b].
MG_HD bool first_comp(const uint16_t* lo, const uint16_t* hi, uint16_t* x, int nb, int d) {
    int R = d;
    for (int b = 0; b < nb; ++b) R -= lo[b];
    if (R < 0) return false;
    for (int b = 0; b < nb; ++b) {
        int room = hi[b] - lo[b];
        int e = room < R ? room : R;
        x[b] = (uint16_t)(lo[b] + e);
        R -= e;
    }
    return R == 0;
}

MG_HD bool next_comp(const uint16_t* lo, const uint16_t* hi, uint16_t* x, int nb) {
    if (nb < 2) return false;
    int slack = hi[nb - 1] - x[nb - 1];
    int extra = x[nb - 1] - lo[nb - 1];
    int i = nb - 2;
    for (; i >= 0; --i) {
        if (x[i] > lo[i] && slack >= 1) break;
        slack += hi[i] - x[i];
        extra += x[i] - lo[i];
    }
    if (i < 0) return false;
    x[i] -= 1;
    int R = extra + 1;
    for (int b = i + 1; b < nb; ++b) {
        int room = hi[b] - lo[b];
        int e = room < R ? room : R;
        x[b] = (uint16_t)(lo[b] + e);
        R -= e;
    }
    return true;
}

// Admissible take-count interval of every block at the last level for threshold t
// (le: contribution <= t, else < t).  Returns false if some block has none or the
// degree is unreachable.
MG_HD bool last_intervals(const Walk& w, int o0, int nb, int d, double t, bool le,
                          const double* rest, const double* take, int& sumlo, int& sumhi) {
    sumlo = 0;
    sumhi = 0;
    for (int b = 0; b < nb; ++b) {
        int s = w.bsz[o0 + b];
        bool rok = le ? rest[b] <= t : rest[b] < t;
        bool tok = w.hi[o0 + b] && (le ? take[b] <= t : take[b] < t);
        if (rok && tok) {
            sumhi += s;
        } else if (rok) {
        } else if (tok) {
            sumlo += s;
            sumhi += s;
        } else {
            return false;
        }
    }
    return sumlo <= d && d <= sumhi;
}

// Does level l (at ph 1: current composition x of option opt[l]) have untried work:
// another composition of this option, or a later option?
MG_HD bool level_has_rest(const Spec& S, const Rows& R, const Walk& w, int l) {
    if (w.opt[l] + 1 < S.lvl_n[l]) return true;
    const int o0 = lvl_off(l);
    const int nb = w.nb[l];
    // next_comp succeeds iff some x_i > lo_i has slack to its right
    int slack = hi_minus_x(w, o0 + nb - 1);
    for (int i = nb - 2; i >= 0; --i) {
        if (w.x[o0 + i] > w.lo[o0 + i] && slack >= 1) return true;
        slack += hi_minus_x(w, o0 + i);
    }
    return false;
}

// Stats of the blocks of level j into the parent scratch.
MG_HD void parent_stats(const Spec& S, const Rows& R, Walk& w, int j) {
    const int o0 = lvl_off(j);
    for (int b = 0; b < w.nb[j]; ++b)
        block_stats(S, R, w.opt, w.bmk[o0 + b], j, w.pu[b], w.pm[b], w.psum[b], w.pmb[b], w.pP[b],
                    w.pmx[b]);
    w.ps_lvl = j;
}

// The per-thread DFS from a loaded cursor at depth d0 (see Cont).  Returns 1 on a
// FIRST hit, 2 when abandoned (a better FIRST hit exists / MIN restart), 3 when the
// step budget ran out and the remaining work was handed back as cursors
// (h.split), 0 when the subtree is exhausted.
template <class H>
MG_HD int dfs(const Spec& S, const Rows& R, Walk& w, int d0, H& h) {
    const int k = S.k;
    const int GL = S.G * S.L;
    int j = d0;
    int floor_lvl = d0;  // levels below this were handed to other threads
    w.ps_lvl = -1;
    while (j >= floor_lvl) {
        const int o0 = lvl_off(j);
        const int nb = w.nb[j];
        if (w.ph[j] == 0) {
            h.level(j);
            int ab = h.abort();
            if (ab == 1) {
                h.split(w, floor_lvl, j);
                return 3;
            }
            if (ab == 2) return 2;
            if (ab == 3) {
                // hand the shallowest level that still has untried work to an idle thread
                while (floor_lvl < j && !level_has_rest(S, R, w, floor_lvl)) ++floor_lvl;
                if (floor_lvl < j && h.donate(w, floor_lvl)) ++floor_lvl;
            }
            const double thr = h.thr(S);
            const int n = S.lvl_n[j], off = S.lvl_off[j];
            int o = w.oc[j] + 1;
            bool got = false;
            for (; o < n; ++o) {
                int r = off + o;
                int t = opt_test(S, R, r, thr);
                if (t == 2) break;
                if (t == 1) continue;
                if (w.used[j] + R.d[r] * R.u[r] + S.suffix_min[j + 1] > GL) continue;
                got = true;
                break;
            }
            if (!got) {
                --j;
                continue;
            }
            w.oc[j] = (int16_t)o;
            w.opt[j] = (uint16_t)o;
            const int r = off + o;
            const int dd = R.d[r], uu = R.u[r];
            const double ff = R.fp[r], bo = R.B[r], ba = R.base[r];
            const bool last = j == k - 1;
            if (w.ps_lvl != j) {
                parent_stats(S, R, w, j);
                if (last) {
                    // approximate rest contributions (any summation order) for the fast filter
                    for (int b = 0; b < nb; ++b)
                        w.cm[b] = w.bmk[o0 + b] ? w.pmb[b] + S.e1 + S.e2 * w.psum[b] +
                                                      (S.additive ? 0.0 : S.e3 * w.pP[b])
                                                : NEG_INF;
                }
            }
            // per-block admissible take interval: capacity, memory, and (non-negative
            // models) the interference bound of the taken and the remaining part
            int sumlo = 0, sumhi = 0;
            bool dead = false;
            for (int b = 0; b < nb; ++b) {
                const int s = w.bsz[o0 + b];
                bool el = w.pu[b] + uu <= S.L && !(w.pm[b] + ff > S.cap_slack);
                bool tok = el, rok = true;
                if (!last && S.nonneg) {
                    if (el) {
                        double lbt;
                        if (S.include_self) {
                            double mb = w.pmb[b] > ba ? w.pmb[b] : ba;
                            lbt = mb + S.e1 + S.e2 * (w.psum[b] + bo) +
                                  envelope(S, j + 1, w.pP[b] * bo);
                        } else {
                            double bx = ba - S.e2 * bo;
                            double mx = w.pmx[b] > bx ? w.pmx[b] : bx;
                            lbt = mx + S.e1 + S.e2 * (w.psum[b] + bo) + envelope(S, j + 1, 0.0);
                        }
                        tok = !(lbt > thr);
                    }
                    if (w.bmk[o0 + b]) {
                        double lbr = S.include_self
                                         ? w.pmb[b] + S.e1 + S.e2 * w.psum[b] +
                                               envelope(S, j + 1, w.pP[b])
                                         : w.pmx[b] + S.e1 + S.e2 * w.psum[b] +
                                               envelope(S, j + 1, 0.0);
                        rok = !(lbr > thr);
                    }
                }
                int l, hgh;
                if (rok) {
                    l = 0;
                    hgh = tok ? s : 0;
                } else if (tok) {
                    l = s;
                    hgh = s;
                } else {
                    dead = true;
                    break;
                }
                w.lo[o0 + b] = (uint16_t)l;
                w.hi[o0 + b] = (uint16_t)hgh;
                sumlo += l;
                sumhi += hgh;
            }
            if (dead || sumlo > dd || sumhi < dd) continue;
            if (last) {
                // ---- last level: closed form over blocks ----
                h.count_leaf();
                if (S.include_self) {
                    // fast filter with approximate contributions and a 1e-12 slack: exact
                    // values differ by a few ulps, so a rejection here is always sound
                    // MIN rejects ties with the incumbent (and anything within TIE_EPS
                    // below it): the planner only ever needs T* to that precision.
                    const bool fm = S.mode == MODE_FIRST;
                    const double tx = fm ? S.theta * (1.0 + 1e-12) : h.incumbent() * (1.0 - TIE_EPS);
                    int flo = 0, fhi = 0;
                    bool fdead = false;
                    for (int b = 0; b < nb; ++b) {
                        const int s = w.bsz[o0 + b];
                        bool rok = fm ? w.cm[b] <= tx : w.cm[b] < tx;
                        bool tok = false;
                        if (w.hi[o0 + b]) {
                            double mb = w.pmb[b] > ba ? w.pmb[b] : ba;
                            double tv = mb + S.e1 + S.e2 * (w.psum[b] + bo) +
                                        (S.additive ? 0.0 : S.e3 * (w.pP[b] * bo));
                            tok = fm ? tv <= tx : tv < tx;
                        }
                        if (rok) {
                            fhi += tok ? s : 0;
                        } else if (tok) {
                            flo += s;
                            fhi += s;
                        } else {
                            fdead = true;
                            break;
                        }
                    }
                    if (fdead || flo > dd || fhi < dd) continue;
                }
                double* rest = w.cs;
                double* take = w.cb;
                for (int b = 0; b < nb; ++b) {
                    unsigned m = w.bmk[o0 + b];
                    rest[b] = contrib(S, R, w.opt, m);
                    take[b] = w.hi[o0 + b] ? contrib(S, R, w.opt, m | (1u << j)) : POS_INF;
                }
                if (S.mode == MODE_FIRST) {
                    int lo, hi;
                    if (!(0.0 <= S.theta)) continue;
                    if (!last_intervals(w, o0, nb, dd, S.theta, true, rest, take, lo, hi)) continue;
                    // greedy first composition (descending lexicographic)
                    int rem = dd - lo;
                    for (int b = 0; b < nb; ++b) {
                        int s = w.bsz[o0 + b];
                        bool rok = rest[b] <= S.theta;
                        bool tok = w.hi[o0 + b] && take[b] <= S.theta;
                        int l = (!rok) ? s : 0;
                        int hgh = tok ? s : 0;
                        int e = hgh - l < rem ? hgh - l : rem;
                        w.x[o0 + b] = (uint16_t)(l + e);
                        rem -= e;
                    }
                    double v = 0.0;
                    for (int b = 0; b < nb; ++b) {
                        int xb = w.x[o0 + b], s = w.bsz[o0 + b];
                        if (xb > 0 && take[b] > v) v = take[b];
                        if (xb < s && rest[b] > v) v = rest[b];
                    }
                    h.hit(w, j, v);
                    return 1;
                } else {
                    double I = h.incumbent();
                    double Ie = I * (1.0 - TIE_EPS);
                    int lo, hi;
                    if (!last_intervals(w, o0, nb, dd, Ie, false, rest, take, lo, hi)) continue;
                    double hiv = Ie;
                    while (true) {
                        double c = NEG_INF;
                        for (int b = 0; b < nb; ++b) {
                            if (rest[b] < hiv && rest[b] > c) c = rest[b];
                            if (w.hi[o0 + b] && take[b] < hiv && take[b] > c) c = take[b];
                        }
                        if (c <= NEG_INF) break;
                        if (last_intervals(w, o0, nb, dd, c, true, rest, take, lo, hi)) {
                            hiv = c;
                        } else {
                            break;
                        }
                    }
                    double v = hiv > 0.0 ? hiv : 0.0;
                    if (v < I) h.improve(v);
                }
                continue;
            }
            if (!first_comp(w.lo + o0, w.hi + o0, w.x + o0, nb, dd)) continue;
            w.ph[j] = 1;
        } else {
            if (!next_comp(w.lo + o0, w.hi + o0, w.x + o0, nb)) {
                w.ph[j] = 0;
                continue;
            }
        }
        // ---- build the child (level j+1 blocks + their stats) ----
        h.count_node();
        if (w.ps_lvl != j) parent_stats(S, R, w, j);
        const int o1 = lvl_off(j + 1);
        const int c1 = lvl_cap(j + 1);
        const int r = S.lvl_off[j] + w.opt[j];
        const int uu = R.u[r];
        const double ff = R.fp[r], bo = R.B[r], ba = R.base[r];
        int m = 0;
        bool overflow = false;
        for (int b = 0; b < nb; ++b) {
            int xb = w.x[o0 + b], s = w.bsz[o0 + b];
            unsigned mk = w.bmk[o0 + b];
            if (xb > 0) {
                if (m >= c1) { overflow = true; break; }
                w.bsz[o1 + m] = (uint16_t)xb;
                w.bmk[o1 + m] = (uint16_t)(mk | (1u << j));
                w.cu[m] = w.pu[b] + uu;
                w.cm[m] = w.pm[b] + ff;
                w.cs[m] = w.psum[b] + bo;
                w.cb[m] = w.pmb[b] > ba ? w.pmb[b] : ba;
                ++m;
            }
            if (xb < s) {
                if (m >= c1) { overflow = true; break; }
                w.bsz[o1 + m] = (uint16_t)(s - xb);
                w.bmk[o1 + m] = (uint16_t)mk;
                w.cu[m] = w.pu[b];
                w.cm[m] = w.pm[b];
                w.cs[m] = w.psum[b];
                w.cb[m] = w.pmb[b];
                ++m;
            }
        }
        if (overflow) {
            h.overflow();
            return 2;
        }
        w.nb[j + 1] = (uint16_t)m;
        w.used[j + 1] = w.used[j] + R.d[r] * R.u[r];
        const double thr = h.thr(S);
        bool prune = false;
        // look-ahead: every unplaced level keeps an option that fits somewhere
        for (int l = j + 1; l < k && !prune; ++l) {
            const int n = S.lvl_n[l], off = S.lvl_off[l];
            bool ok = false;
            for (int o = 0; o < n && !ok; ++o) {
                int rr = off + o;
                int t = opt_test(S, R, rr, thr);
                if (t == 2) break;
                if (t == 1) continue;
                const int dd = R.d[rr], u2 = R.u[rr];
                const double f2 = R.fp[rr], b2 = R.B[rr], a2 = R.base[rr];
                int cnt = 0;
                for (int b = 0; b < m; ++b) {
                    if (w.cu[b] + u2 > S.L) continue;
                    if (w.cm[b] + f2 > S.cap_slack) continue;
                    if (S.nonneg && S.include_self) {
                        double mb = w.cb[b] > a2 ? w.cb[b] : a2;
                        if (mb + S.e1 + S.e2 * (w.cs[b] + b2) > thr) continue;
                    }
                    cnt += w.bsz[o1 + b];
                    if (cnt >= dd) break;
                }
                ok = cnt >= dd;
            }
            if (!ok) prune = true;
        }
        if (prune) continue;
        ++j;
        w.ph[j] = 0;
        w.oc[j] = -1;
    }
    return 0;
}

// Load a cursor into a walk.
MG_HD void load_cont(const Cont& c, Walk& w) {
    const int dep = c.depth;
    for (int l = 0; l < dep; ++l) w.opt[l] = c.opt[l];
    const int o = lvl_off(dep);
    w.nb[dep] = c.nb;
    w.used[dep] = c.used;
    w.ph[dep] = (uint8_t)c.ph;
    w.oc[dep] = c.oc;
    if (c.ph) w.opt[dep] = (uint16_t)c.oc;
    for (int b = 0; b < c.nb; ++b) {
        w.bsz[o + b] = c.bsz[b];
        w.bmk[o + b] = c.bmk[b];
        if (c.ph) {
            w.x[o + b] = c.x[b];
            w.lo[o + b] = c.lo[b];
            w.hi[o + b] = c.hi[b];
        }
    }
    // Rebuild the blocks and compositions of every ancestor level: level l+1 lists each
    // parent block as (taken part, rest part), adjacent, with masks differing in bit l.
    for (int l = dep - 1; l >= 0; --l) {
        const int oc1 = lvl_off(l + 1), ol = lvl_off(l);
        const unsigned bit = 1u << l;
        int nbl = 0;
        for (int b = 0; b < w.nb[l + 1];) {
            const unsigned key = w.bmk[oc1 + b] & ~bit;
            int size = 0, taken = 0;
            while (b < w.nb[l + 1] && (w.bmk[oc1 + b] & ~bit) == key) {
                size += w.bsz[oc1 + b];
                if (w.bmk[oc1 + b] & bit) taken += w.bsz[oc1 + b];
                ++b;
            }
            w.bsz[ol + nbl] = (uint16_t)size;
            w.bmk[ol + nbl] = (uint16_t)key;
            w.x[ol + nbl] = (uint16_t)taken;
            ++nbl;
        }
        w.nb[l] = (uint16_t)nbl;
    }
}


// -1: path H precedes the walk's leaf path (levels 0..j), +1 follows it, 0 equal.
template <class HP>
MG_HD int path_cmp(const HP* H, const Walk& w, int j) {
    for (int l = 0; l <= j; ++l) {
        int ho = H->opt[l];
        if (ho != w.opt[l]) return ho < w.opt[l] ? -1 : 1;
        const int o0 = lvl_off(l);
        for (int b = 0; b < w.nb[l]; ++b) {
            int hx = H->x[l][b], wx = w.x[o0 + b];
            if (hx != wx) return hx > wx ? -1 : 1;  // larger count first
        }
    }
    return 0;
}

// Does H precede every leaf the walk can still reach?  Levels < j are fixed at their
// current (option, composition); at level j only the options after oc[j] remain.
template <class HP>
MG_HD bool path_precedes_rest(const HP* H, const Walk& w, int j) {
    for (int l = 0; l < j; ++l) {
        int ho = H->opt[l];
        if (ho != w.opt[l]) return ho < w.opt[l];
        const int o0 = lvl_off(l);
        for (int b = 0; b < w.nb[l]; ++b) {
            int hx = H->x[l][b], wx = w.x[o0 + b];
            if (hx != wx) return hx > wx;
        }
    }
    return (int)H->opt[j] <= w.oc[j];
}

template <class HP>
MG_HD void path_store(HP* H, const Walk& w, int j) {
    for (int l = 0; l <= j; ++l) {
        H->opt[l] = w.opt[l];
        H->nb[l] = w.nb[l];
        const int o0 = lvl_off(l);
        for (int b = 0; b < w.nb[l]; ++b) H->x[l][b] = w.x[o0 + b];
    }
}

// Cursor for "the rest of level l": options after oc[l] (ph 0) or compositions after
// the current x (ph 1).
MG_HD void store_cont(const Walk& w, int l, int ph, unsigned long long key, Cont& c) {
    c.key = key;
    for (int i = 0; i < MAXK; ++i) c.opt[i] = i < l ? w.opt[i] : 0;
    c.depth = (uint16_t)l;
    c.nb = w.nb[l];
    c.ph = (uint16_t)ph;
    c.oc = ph ? (int16_t)w.opt[l] : w.oc[l];
    c.used = w.used[l];
    const int o = lvl_off(l);
    for (int b = 0; b < c.nb; ++b) {
        c.bsz[b] = w.bsz[o + b];
        c.bmk[b] = w.bmk[o + b];
        if (ph) {
            c.x[b] = w.x[o + b];
            c.lo[b] = w.lo[o + b];
            c.hi[b] = w.hi[o + b];
        }
    }
}

// Write the FIRST leaf: options and the final block list after the last level.
MG_HD void store_leaf(const Walk& w, int j, double v, Leaf& lf) {
    lf.value = v;
    for (int l = 0; l <= j; ++l) lf.opt[l] = w.opt[l];
    int o0 = lvl_off(j);
    int m = 0;
    for (int b = 0; b < w.nb[j]; ++b) {
        int xb = w.x[o0 + b], s = w.bsz[o0 + b];
        unsigned mk = w.bmk[o0 + b];
        if (xb > 0) {
            lf.bsz[m] = (uint16_t)xb;
            lf.bmk[m] = (uint16_t)(mk | (1u << j));
            ++m;
        }
        if (xb < s) {
            lf.bsz[m] = (uint16_t)(s - xb);
            lf.bmk[m] = (uint16_t)mk;
            ++m;
        }
    }
    lf.nb = m;
}

#endif  // MG_DEVICE_CODE

}  // namespace mg
