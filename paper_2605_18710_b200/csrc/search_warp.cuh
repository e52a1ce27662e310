// search_warp.cuh — warp-cooperative version of the canonical-block DFS (sm_100a).
//
// One warp is one walker.  Its Walk lives in shared memory; the DFS control flow is
// warp-uniform (every lane runs the same scalar code on the same shared state, and
// every value read from global memory that steers control flow is read by lane 0 and
// broadcast).  The per-GPU-block work — block statistics, admissible take intervals,
// composition stepping (prefix scans), child construction, look-ahead counts and the
// closed-form last level — is spread over the 32 lanes, so irregular trees run
// without intra-warp divergence.  Semantics are exactly those of search_core.cuh.
#pragma once
#include "search_core.cuh"

namespace mg {

constexpr unsigned FULLW = 0xffffffffu;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int wsum(int v) { return __reduce_add_sync(FULLW, v); }
__device__ __forceinline__ int wmaxi(int v) { return __reduce_max_sync(FULLW, v); }
__device__ __forceinline__ bool wany(bool p) { return __any_sync(FULLW, p); }
__device__ __forceinline__ double wmaxd(double v) {
    for (int o = 16; o; o >>= 1) {
        double t = __shfl_xor_sync(FULLW, v, o);
        v = t > v ? t : v;
    }
    return v;
}
__device__ __forceinline__ int wscan_incl(int v) {
    const int lane = lane_id();
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(FULLW, v, o);
        if (lane >= o) v += y;
    }
    return v;
}


__device__ __forceinline__ void parent_stats_warp(const Spec& S, const Rows& R, Walk& w, int j) {
    double mbx_unused;  // the include_self kernels keep no own-excluded bound
    const int o0 = w.loff[j];
    #pragma unroll 1
    for (int b = lane_id(); b < w.nb[j]; b += 32)
        block_stats(S, w, w.bmk[o0 + b], j, w.pu[b], w.pm[b], w.psum[b], w.pmb[b], w.pP[b],
                    MG_SELF(S) ? mbx_unused : w.pmx[b]);
    __syncwarp();
}

// x_b = lo_b + min(room_b, max(0, R - sum_{t<b} room_t)),  R = d - sum lo
__device__ __forceinline__ bool first_comp_warp(Walk& w, int o0, int nb, int d) {
    const int lane = lane_id();
    int mylo = 0;
    #pragma unroll 1
    for (int b = lane; b < nb; b += 32) mylo += w.lo[o0 + b];
    const int R = d - wsum(mylo);
    if (R < 0) return false;
    int carry = 0;
    #pragma unroll 1
    for (int c = 0; c < nb; c += 32) {
        const int b = c + lane;
        const int room = b < nb ? (int)w.hi[o0 + b] - (int)w.lo[o0 + b] : 0;
        const int inc = wscan_incl(room);
        const int ex = carry + inc - room;
        if (b < nb) {
            int left = R - ex;
            left = left > 0 ? left : 0;
            w.x[o0 + b] = (uint16_t)(w.lo[o0 + b] + (room < left ? room : left));
        }
        carry += __shfl_sync(FULLW, inc, 31);
    }
    __syncwarp();
    return carry >= R;
}

// next composition in descending lexicographic order within [lo, hi]
__device__ __forceinline__ bool next_comp_warp(Walk& w, int o0, int nb) {
    if (nb < 2) return false;
    const int lane = lane_id();
    // inclusive prefix of slack_t = hi_t - x_t and extra_t = x_t - lo_t
    int cs = 0, ce = 0;
    #pragma unroll 1
    for (int c = 0; c < nb; c += 32) {
        const int b = c + lane;
        const int sl = b < nb ? (int)w.hi[o0 + b] - (int)w.x[o0 + b] : 0;
        const int ex = b < nb ? (int)w.x[o0 + b] - (int)w.lo[o0 + b] : 0;
        const int is = wscan_incl(sl), ie = wscan_incl(ex);
        if (b < nb) {
            w.sa[b] = cs + is;
            w.sb[b] = ce + ie;
        }
        cs += __shfl_sync(FULLW, is, 31);
        ce += __shfl_sync(FULLW, ie, 31);
    }
    __syncwarp();
    // rightmost i <= nb-2 with x_i > lo_i and slack to its right
    int best = -1;
    #pragma unroll 1
    for (int i = lane; i < nb - 1; i += 32)
        if (w.x[o0 + i] > w.lo[o0 + i] && cs - w.sa[i] >= 1) best = i;
    const int is = wmaxi(best);
    if (is < 0) return false;
    const int R = (ce - w.sb[is]) + 1;  // extra to the right of i*, plus the one unit
    __syncwarp();
    if (lane == 0) w.x[o0 + is] -= 1;
    int carry = 0;
    #pragma unroll 1
    for (int c = 0; c < nb; c += 32) {
        const int b = c + lane;
        const bool mine = b < nb && b > is;
        const int room = mine ? (int)w.hi[o0 + b] - (int)w.lo[o0 + b] : 0;
        const int inc = wscan_incl(room);
        const int ex = carry + inc - room;
        if (mine) {
            int left = R - ex;
            left = left > 0 ? left : 0;
            w.x[o0 + b] = (uint16_t)(w.lo[o0 + b] + (room < left ? room : left));
        }
        carry += __shfl_sync(FULLW, inc, 31);
    }
    __syncwarp();
    return true;
}

// Last level: admissible intervals at threshold t (le: <=, else <); feasibility of d.
__device__ __forceinline__ bool last_feasible_warp(const Walk& w, int o0, int nb, int d, double t,
                                                   bool le, const double* rest,
                                                   const double* take) {
    int lo = 0, hi = 0;
    bool dead = false;
    #pragma unroll 1
    for (int b = lane_id(); b < nb; b += 32) {
        const int s = w.bsz[o0 + b];
        const bool rok = le ? rest[b] <= t : rest[b] < t;
        const bool tok = w.hi[o0 + b] && (le ? take[b] <= t : take[b] < t);
        if (rok && tok) {
            hi += s;
        } else if (rok) {
        } else if (tok) {
            lo += s;
            hi += s;
        } else {
            dead = true;
        }
    }
    const int L = wsum(lo), H = wsum(hi);
    return !wany(dead) && L <= d && d <= H;
}

__device__ __forceinline__ bool level_has_rest_warp(const Spec& S, const Walk& w,
                                                    int l) {
    if (w.opt[l] + 1 < S.lvl_n[l]) return true;
    const int lane = lane_id();
    const int o0 = w.loff[l];
    const int nb = w.nb[l];
    int cs = 0;
    #pragma unroll 1
    for (int c = 0; c < nb; c += 32) {
        const int b = c + lane;
        const int sl = b < nb ? (int)w.hi[o0 + b] - (int)w.x[o0 + b] : 0;
        const int is = wscan_incl(sl);
        if (b < nb) w.sa[b] = cs + is;
        cs += __shfl_sync(FULLW, is, 31);
    }
    __syncwarp();
    bool any = false;
    #pragma unroll 1
    for (int i = lane; i < nb - 1; i += 32)
        if (w.x[o0 + i] > w.lo[o0 + i] && cs - w.sa[i] >= 1) any = true;
    const bool r = wany(any);
    __syncwarp();
    return r;
}

// Descending-lexicographic first composition whose present parts all have contribution
// <= t (rest/take per block); writes w.x at level j and returns the allocation's value.
__device__ __forceinline__ double greedy_fill_warp(Walk& w, int o0, int nb, int dd, double t,
                                                   const double* rest, const double* take) {
    const int lane = lane_id();
    int mylo = 0;
    #pragma unroll 1
    for (int b = lane; b < nb; b += 32) mylo += (rest[b] <= t) ? 0 : w.bsz[o0 + b];
    const int rem0 = dd - wsum(mylo);
    int carry = 0;
    double v = 0.0;
    #pragma unroll 1
    for (int c = 0; c < nb; c += 32) {
        const int b = c + lane;
        int l = 0, room = 0;
        if (b < nb) {
            const int s = w.bsz[o0 + b];
            const bool rok = rest[b] <= t;
            const bool tok = w.hi[o0 + b] && take[b] <= t;
            l = rok ? 0 : s;
            room = (tok ? s : 0) - l;
        }
        const int inc = wscan_incl(room);
        const int ex = carry + inc - room;
        if (b < nb) {
            int left = rem0 - ex;
            left = left > 0 ? left : 0;
            const int xb = l + (room < left ? room : left);
            w.x[o0 + b] = (uint16_t)xb;
            const int s = w.bsz[o0 + b];
            if (xb > 0 && take[b] > v) v = take[b];
            if (xb < s && rest[b] > v) v = rest[b];
        }
        carry += __shfl_sync(FULLW, inc, 31);
    }
    v = wmaxd(v);
    __syncwarp();
    return v;
}

// Per-lane exact check of last-level option `o` at threshold t (le: <=, else <).
__device__ __forceinline__ bool lane_last_feasible(const Spec& S, const Rows& R, const Walk& w,
                                                   int j, int o0, int nb, int o, int uu,
                                                   double ff, int dd, double t, bool le) {
    int lo = 0, hi = 0;
    #pragma unroll 1
    for (int b = 0; b < nb; ++b) {
        const int s = w.bsz[o0 + b];
        const double rv = w.cs[b];
        const bool rok = le ? rv <= t : rv < t;
        bool tok = false;
        if (w.pu[b] + uu <= S.L && !(w.pm[b] + ff > S.cap_slack)) {
            const double tv = contrib_o(S, R, w, w.bmk[o0 + b] | (1u << j), j, o);
            tok = le ? tv <= t : tv < t;
        }
        if (rok) {
            if (tok) hi += s;
        } else if (tok) {
            lo += s;
            hi += s;
        } else {
            return false;
        }
    }
    return lo <= dd && dd <= hi;
}

// The last level with lanes over OPTIONS: every lane screens its own candidate option
// against all blocks (no per-option warp reductions), then the winner — first feasible
// option (FIRST) or smallest value (MIN) — is materialised block-parallel.  Returns true
// when a FIRST hit was published.
template <class H>
__device__ bool last_level_batch(const Spec& S, const Rows& R, Walk& w, int j, int& ps_lvl, H& h) {
    const int lane = lane_id();
    const int o0 = w.loff[j], nb = w.nb[j];
    const int GL = S.G * S.L;
    if (ps_lvl != j) {
        parent_stats_warp(S, R, w, j);
        ps_lvl = j;
    }
    // per block: approximate rest contribution (fast filter); the exact one is computed
    // only once some option survives the filter (proof searches rarely need it)
    #pragma unroll 1
    for (int b = lane; b < nb; b += 32) {
        const unsigned m = w.bmk[o0 + b];
        w.cm[b] = m ? w.pmb[b] + S.e1 + S.e2 * w.psum[b] + (MG_ADD(S) ? 0.0 : S.e3 * w.pP[b])
                    : NEG_INF;
    }
    __syncwarp();
    bool rest_ready = !MG_SELF(S);
    if (rest_ready) {
        #pragma unroll 1
        for (int b = lane; b < nb; b += 32) w.cs[b] = contrib(S, w, w.bmk[o0 + b]);
        __syncwarp();
    }
    const bool fm = MG_MODE(S) == MODE_FIRST;
    const int n = S.lvl_n[j] < w.oe[j] ? S.lvl_n[j] : w.oe[j];
    const int off = S.lvl_off[j];
    const double thr = h.thr(S);
    #pragma unroll 1
    for (int start = w.oc[j] + 1; start < n; start += 32) {
        const int o = start + lane;
        const int t = o < n ? opt_test(S, R, off + o, thr) : 2;
        const unsigned brk = __ballot_sync(FULLW, t == 2);
        const int first_brk = brk ? __ffs(brk) - 1 : 32;
        bool valid = t == 0 && lane < first_brk;
        if (valid && j == S.shard_level && S.shard_world > 1 &&
            shard_hash(w.opt, j, o) % (unsigned)S.shard_world != (unsigned)S.shard_rank)
            valid = false;
        int dd = 0, uu = 0;
        double ff = 0.0, bo = 0.0, ba = 0.0;
        if (valid) {
            const int r = off + o;
            dd = R.d[r];
            uu = R.u[r];
            ff = R.fp[r];
            bo = R.B[r];
            ba = R.base[r];
            if (w.used[j] + dd * uu > GL) valid = false;
        }
        h.count_leaves(__popc(__ballot_sync(FULLW, valid)));
        const double I = fm ? 0.0 : h.incumbent();
        const double Ie = I * (1.0 - TIE_EPS);
        bool feas = false;
        double val = POS_INF;
        bool pass = false;
        if (valid) {
            // fast filter (approximate contributions, sound 1e-12 slack)
            pass = true;
            if (MG_SELF(S)) {
                const double tx = fm ? S.theta * (1.0 + 1e-12) : Ie;
                int lo = 0, hi = 0;
                #pragma unroll 1
                for (int b = 0; b < nb && pass; ++b) {
                    const int s = w.bsz[o0 + b];
                    const bool el = w.pu[b] + uu <= S.L && !(w.pm[b] + ff > S.cap_slack);
                    const bool rok = fm ? w.cm[b] <= tx : w.cm[b] < tx;
                    bool tok = false;
                    if (el) {
                        const double mb = w.pmb[b] > ba ? w.pmb[b] : ba;
                        const double tv = mb + S.e1 + S.e2 * (w.psum[b] + bo) +
                                          (MG_ADD(S) ? 0.0 : S.e3 * (w.pP[b] * bo));
                        tok = fm ? tv <= tx : tv < tx;
                    }
                    if (rok) {
                        if (tok) hi += s;
                    } else if (tok) {
                        lo += s;
                        hi += s;
                    } else {
                        pass = false;
                    }
                }
                pass = pass && lo <= dd && dd <= hi;
            }
        }
        if (!rest_ready && __any_sync(FULLW, valid && pass)) {
            #pragma unroll 1
            for (int b = lane; b < nb; b += 32) w.cs[b] = contrib(S, w, w.bmk[o0 + b]);
            __syncwarp();
            rest_ready = true;
        }
        if (valid) {
            if (pass) {
                if (fm) {
                    feas = 0.0 <= S.theta &&
                           lane_last_feasible(S, R, w, j, o0, nb, o, uu, ff, dd, S.theta, true);
                } else if (lane_last_feasible(S, R, w, j, o0, nb, o, uu, ff, dd, Ie, false)) {
                    // smallest feasible threshold: descend through candidate values
                    double hiv = Ie;
                    while (true) {
                        double c = NEG_INF;
                        #pragma unroll 1
                        for (int b = 0; b < nb; ++b) {
                            const double rv = w.cs[b];
                            if (rv < hiv && rv > c) c = rv;
                            if (w.pu[b] + uu <= S.L && !(w.pm[b] + ff > S.cap_slack)) {
                                const double tv =
                                    contrib_o(S, R, w, w.bmk[o0 + b] | (1u << j), j, o);
                                if (tv < hiv && tv > c) c = tv;
                            }
                        }
                        if (c <= NEG_INF) break;
                        if (lane_last_feasible(S, R, w, j, o0, nb, o, uu, ff, dd, c, true))
                            hiv = c;
                        else
                            break;
                    }
                    val = hiv > 0.0 ? hiv : 0.0;
                    feas = val < I;
                }
            }
        }
        const unsigned fb = __ballot_sync(FULLW, feas);
        if (fb) {
            int win;
            double v;
            if (fm) {
                win = __ffs(fb) - 1;
            } else {
                double mv = val;
                #pragma unroll 1
                for (int of = 16; of; of >>= 1) {
                    double x = __shfl_xor_sync(FULLW, mv, of);
                    mv = x < mv ? x : mv;
                }
                win = __ffs(__ballot_sync(FULLW, feas && val == mv)) - 1;
            }
            const int ow = start + win;
            const int r = off + ow;
            const int dd2 = R.d[r], uu2 = R.u[r];
            const double ff2 = R.fp[r];
            if (lane == 0) {
                sel_set(S, R, w, j, ow);
                w.oc[j] = (int16_t)ow;
            }
            __syncwarp();
            // block-parallel materialisation of the winner: take contributions + greedy fill
            #pragma unroll 1
            for (int b = lane; b < nb; b += 32) {
                const bool el = w.pu[b] + uu2 <= S.L && !(w.pm[b] + ff2 > S.cap_slack);
                w.hi[o0 + b] = el ? w.bsz[o0 + b] : 0;
                w.cb[b] = el ? contrib(S, w, w.bmk[o0 + b] | (1u << j)) : POS_INF;
            }
            __syncwarp();
            const double tfill = fm ? S.theta : __shfl_sync(FULLW, val, win);
            v = greedy_fill_warp(w, o0, nb, dd2, tfill, w.cs, w.cb);
            if (fm) {
                h.hit(w, j, v);
                return true;
            }
            h.improve_leaf(w, j, v);
        }
        if (first_brk < 32) break;
    }
    return false;
}

// Lane-parallel pre-screen of the options [start, start + 32) at a non-last level: each
// lane runs opt_test, the capacity test and the full admissible-interval test of its own
// option over all blocks (no warp reductions).  Only options whose intervals can reach d
// survive; they are then processed one by one with the block-parallel code.  The screen
// uses the current threshold, which only tightens later, so it never drops a leaf.
__device__ __forceinline__ void screen_options(const Spec& S, const Rows& R, Walk& w, int j,
                                               int start, int n, double thr) {
    const int lane = lane_id();
    const int o = start + lane;
    const int o0 = w.loff[j], nb = w.nb[j];
    const int off = S.lvl_off[j];
    // option-independent bound of the blocks the option would leave alone, once per block
    // (-inf where no module resides yet); lives in the composition scan scratch (sa|sb),
    // which is free between compositions
    double* lbrv = reinterpret_cast<double*>(w.sa);
    if (MG_NONNEG(S)) {
        #pragma unroll 1
        for (int b = lane; b < nb; b += 32)
            lbrv[b] = !w.bmk[o0 + b] ? NEG_INF
                      : MG_SELF(S)
                          ? w.pmb[b] + S.e1 + S.e2 * w.psum[b] + envelope(S, j + 1, w.pP[b])
                          : w.pmx[b] + S.e1 + S.e2 * w.psum[b] + envelope(S, j + 1, 0.0);
        __syncwarp();
    }
    const int t = o < n ? opt_test(S, R, off + o, thr) : 2;
    const unsigned brk = __ballot_sync(FULLW, t == 2);
    const int first_brk = brk ? __ffs(brk) - 1 : 32;
    bool viable = t == 0 && lane < first_brk;
    if (viable && j == S.shard_level && S.shard_world > 1 &&
        shard_hash(w.opt, j, o) % (unsigned)S.shard_world != (unsigned)S.shard_rank)
        viable = false;
    if (viable) {
        const int r = off + o;
        const int dd = R.d[r], uu = R.u[r];
        const double ff = R.fp[r], bo = R.B[r], ba = R.base[r];
        if (w.used[j] + dd * uu + S.suffix_min[j + 1] > S.G * S.L) {
            viable = false;
        } else {
            int lo = 0, hi = 0;
            #pragma unroll 1
            for (int b = 0; b < nb && viable; ++b) {
                const int s = w.bsz[o0 + b];
                const bool el = w.pu[b] + uu <= S.L && !(w.pm[b] + ff > S.cap_slack);
                bool tok = el, rok = true;
                if (MG_NONNEG(S)) {
                    if (el) {
                        double lbt;
                        if (MG_SELF(S)) {
                            const double mb = w.pmb[b] > ba ? w.pmb[b] : ba;
                            lbt = mb + S.e1 + S.e2 * (w.psum[b] + bo) +
                                  envelope(S, j + 1, w.pP[b] * bo);
                        } else {
                            const double bx = ba - S.e2 * bo;
                            const double mx = w.pmx[b] > bx ? w.pmx[b] : bx;
                            lbt = mx + S.e1 + S.e2 * (w.psum[b] + bo) + envelope(S, j + 1, 0.0);
                        }
                        tok = !(lbt > thr);
                    }
                    rok = !(lbrv[b] > thr);
                }
                if (rok) {
                    if (tok) hi += s;
                } else if (tok) {
                    lo += s;
                    hi += s;
                } else {
                    viable = false;
                }
            }
            viable = viable && lo <= dd && dd <= hi;
        }
    }
    const unsigned m = __ballot_sync(FULLW, viable);
    if (lane == 0) {
        w.vmask[j] = m;
        w.vbase[j] = (int16_t)start;
        w.vstop[j] = first_brk < 32 ? 1 : 0;
    }
    __syncwarp();
}

template <class H>
__device__ int dfs_warp(const Spec& S, const Rows& R, Walk& w, int d0, H& h) {
    const int lane = lane_id();
    const int k = S.k;
    const int GL = S.G * S.L;
    int j = d0;
    int floor_lvl = d0;
    int ps_lvl = -1;
    while (j >= floor_lvl) {
        const int o0 = w.loff[j];
        const int nb = w.nb[j];
        if (w.ph[j] == 0) {
            h.level(j);
            const int ab = h.abort();
            if (ab == 2) {
                h.note(S, 6);
                return 2;
            }
            if (ab == 5) {
                // a sibling of this CTA is idle: hand it the shallowest rest (any level above
                // the closed-form last one) through the CTA's shared-memory slot
                h.note(S, 7);
                while (floor_lvl < j && !level_has_rest_warp(S, w, floor_lvl)) ++floor_lvl;
                if (floor_lvl < j && floor_lvl <= k - 2) {
                    if (h.donate_local(w, floor_lvl, 1, -1)) {
                        ++floor_lvl;
                        h.note(S, 5);
                    }
                } else if (floor_lvl == j && j <= k - 2) {
                    const int a = w.oc[j] + 1, e = w.oe[j];
                    if (e - a >= 2) {
                        const int mid = a + (e - a) / 2;
                        if (h.donate_local(w, j, 0, mid)) {
                            if (lane == 0) w.oe[j] = (int16_t)mid;
                            h.note(S, 5);
                        }
                        __syncwarp();
                    }
                }
            }
            if (ab == 3 || ab == 4) {
                h.note(S, 7);
                // only shallow work is worth a hand-over (cursor traffic beats tiny
                // subtrees) — except in the tail, when most walkers are starving
                const int maxl = ab == 4 ? S.don_max_level_tail : S.don_max_level;
                while (floor_lvl < j && !level_has_rest_warp(S, w, floor_lvl)) ++floor_lvl;
                h.note(S, 8 + (j < 7 ? j : 7));
                // deeper than the shallow limit (tail rule only): hand over a level's rest only
                // if it still holds at least don_min_rest options (tiny pieces churn the ring)
                const bool big_enough = floor_lvl <= S.don_max_level || S.don_min_rest <= 0 ||
                                        (int)w.oe[floor_lvl] - (int)w.oc[floor_lvl] - 1 >= S.don_min_rest;
                if (floor_lvl < j && floor_lvl <= maxl && big_enough) {
                    if (h.donate(w, floor_lvl, 1, -1)) {
                        ++floor_lvl;
                        h.note(S, 5);
                    } else {
                        h.note(S, 0);
                    }
                } else if (floor_lvl == j && j <= maxl) {
                    // all that is left is this level's option range: hand over its upper half
                    const int a = w.oc[j] + 1, e = w.oe[j];
                    if (e - a >= 2) {
                        const int mid = a + (e - a) / 2;
                        if (h.donate(w, j, 0, mid)) {
                            if (lane == 0) w.oe[j] = (int16_t)mid;
                            h.note(S, 5);
                        }
                        __syncwarp();
                    } else {
                        h.note(S, 1);
                    }
                } else if (floor_lvl < j) {
                    h.note(S, 2);  // rest only below maxl
                } else {
                    h.note(S, 3);  // floor == j > maxl
                }
                if (ab == 4) h.note(S, 4);
            }
            if (j == k - 1 && MG_NONNEG(S)) {
                if (last_level_batch(S, R, w, j, ps_lvl, h)) return 1;
                --j;
                continue;
            }
            const double thr = h.thr(S);
            const int n = S.lvl_n[j] < w.oe[j] ? S.lvl_n[j] : w.oe[j], off = S.lvl_off[j];
            int o = w.oc[j] + 1;
            bool got = false;
            if (j < k - 1) {
                if (ps_lvl != j) {
                    parent_stats_warp(S, R, w, j);
                    ps_lvl = j;
                }
                while (o < n) {
                    if (w.vbase[j] < 0 || o < w.vbase[j] || o >= w.vbase[j] + 32)
                        screen_options(S, R, w, j, o, n, thr);
                    const unsigned mk = w.vmask[j] >> (o - w.vbase[j]);
                    if (mk) {
                        o += __ffs(mk) - 1;
                        if (!MG_NONNEG(S) && S.seq_cut && !(R.base[off + o] < h.incumbent())) {
                            ++o;  // the reference's `lb >= best_time_` skip (oracle.hpp:137)
                            continue;
                        }
                        got = true;
                        break;
                    }
                    if (w.vstop[j]) break;
                    o = w.vbase[j] + 32;
                }
            } else {
                #pragma unroll 1
                for (; o < n; ++o) {
                    const int r = off + o;
                    const int t = opt_test(S, R, r, thr);
                    if (t == 2) break;
                    if (t == 1) continue;
                    if (j == S.shard_level && S.shard_world > 1 &&
                        shard_hash(w.opt, j, o) % (unsigned)S.shard_world !=
                            (unsigned)S.shard_rank)
                        continue;
                    if (w.used[j] + R.d[r] * R.u[r] + S.suffix_min[j + 1] > GL) continue;
                    if (!MG_NONNEG(S) && S.seq_cut && !(R.base[r] < h.incumbent())) continue;
                    got = true;
                    break;
                }
            }
            __syncwarp();
            if (!got) {
                --j;
                continue;
            }
            if (lane == 0) {
                w.oc[j] = (int16_t)o;
                sel_set(S, R, w, j, o);
            }
            __syncwarp();
            const int r = off + o;
            const int dd = R.d[r], uu = R.u[r];
            const double ff = R.fp[r], bo = R.B[r], ba = R.base[r];
            const bool last = j == k - 1;
            if (ps_lvl != j) {
                parent_stats_warp(S, R, w, j);
                ps_lvl = j;
                if (last) {
                    #pragma unroll 1
                    for (int b = lane; b < nb; b += 32)
                        w.cm[b] = w.bmk[o0 + b] ? w.pmb[b] + S.e1 + S.e2 * w.psum[b] +
                                                      (MG_ADD(S) ? 0.0 : S.e3 * w.pP[b])
                                                : NEG_INF;
                    __syncwarp();
                }
            }
            // per-block admissible take interval
            int mylo = 0, myhi = 0;
            bool mydead = false;
            #pragma unroll 1
            for (int b = lane; b < nb; b += 32) {
                const int s = w.bsz[o0 + b];
                const bool el = w.pu[b] + uu <= S.L && !(w.pm[b] + ff > S.cap_slack);
                bool tok = el, rok = true;
                if (!last && MG_NONNEG(S)) {
                    if (el) {
                        double lbt;
                        if (MG_SELF(S)) {
                            const double mb = w.pmb[b] > ba ? w.pmb[b] : ba;
                            lbt = mb + S.e1 + S.e2 * (w.psum[b] + bo) +
                                  envelope(S, j + 1, w.pP[b] * bo);
                        } else {
                            const double bx = ba - S.e2 * bo;
                            const double mx = w.pmx[b] > bx ? w.pmx[b] : bx;
                            lbt = mx + S.e1 + S.e2 * (w.psum[b] + bo) + envelope(S, j + 1, 0.0);
                        }
                        tok = !(lbt > thr);
                    }
                    if (w.bmk[o0 + b]) {
                        const double lbr = MG_SELF(S)
                                               ? w.pmb[b] + S.e1 + S.e2 * w.psum[b] +
                                                     envelope(S, j + 1, w.pP[b])
                                               : w.pmx[b] + S.e1 + S.e2 * w.psum[b] +
                                                     envelope(S, j + 1, 0.0);
                        rok = !(lbr > thr);
                    }
                }
                int l, hg;
                if (rok) {
                    l = 0;
                    hg = tok ? s : 0;
                } else if (tok) {
                    l = s;
                    hg = s;
                } else {
                    l = 0;
                    hg = 0;
                    mydead = true;
                }
                w.lo[o0 + b] = (uint16_t)l;
                w.hi[o0 + b] = (uint16_t)hg;
                mylo += l;
                myhi += hg;
            }
            const int sumlo = wsum(mylo), sumhi = wsum(myhi);
            const bool dead = wany(mydead);
            __syncwarp();
            if (dead || sumlo > dd || sumhi < dd) continue;
            if (last) {
                h.count_leaf();
                const bool fm = MG_MODE(S) == MODE_FIRST;
                if (MG_SELF(S)) {
                    const double tx = fm ? S.theta * (1.0 + 1e-12) : h.incumbent() * (1.0 - TIE_EPS);
                    int flo = 0, fhi = 0;
                    bool fdead = false;
                    #pragma unroll 1
                    for (int b = lane; b < nb; b += 32) {
                        const int s = w.bsz[o0 + b];
                        const bool rok = fm ? w.cm[b] <= tx : w.cm[b] < tx;
                        bool tok = false;
                        if (w.hi[o0 + b]) {
                            const double mb = w.pmb[b] > ba ? w.pmb[b] : ba;
                            const double tv = mb + S.e1 + S.e2 * (w.psum[b] + bo) +
                                              (MG_ADD(S) ? 0.0 : S.e3 * (w.pP[b] * bo));
                            tok = fm ? tv <= tx : tv < tx;
                        }
                        if (rok) {
                            fhi += tok ? s : 0;
                        } else if (tok) {
                            flo += s;
                            fhi += s;
                        } else {
                            fdead = true;
                        }
                    }
                    const int FL = wsum(flo), FH = wsum(fhi);
                    if (wany(fdead) || FL > dd || FH < dd) continue;
                }
                double* rest = w.cs;
                double* take = w.cb;
                #pragma unroll 1
                for (int b = lane; b < nb; b += 32) {
                    const unsigned m = w.bmk[o0 + b];
                    rest[b] = contrib(S, w, m);
                    take[b] = w.hi[o0 + b] ? contrib(S, w, m | (1u << j)) : POS_INF;
                }
                __syncwarp();
                if (fm) {
                    if (!(0.0 <= S.theta)) continue;
                    if (!last_feasible_warp(w, o0, nb, dd, S.theta, true, rest, take)) continue;
                    int mylo2 = 0;
                    #pragma unroll 1
                    for (int b = lane; b < nb; b += 32)
                        mylo2 += (rest[b] <= S.theta) ? 0 : w.bsz[o0 + b];
                    const int rem0 = dd - wsum(mylo2);
                    int carry = 0;
                    double v = 0.0;
                    #pragma unroll 1
                    for (int c = 0; c < nb; c += 32) {
                        const int b = c + lane;
                        int l = 0, room = 0;
                        if (b < nb) {
                            const int s = w.bsz[o0 + b];
                            const bool rok = rest[b] <= S.theta;
                            const bool tok = w.hi[o0 + b] && take[b] <= S.theta;
                            l = rok ? 0 : s;
                            room = (tok ? s : 0) - l;
                        }
                        const int inc = wscan_incl(room);
                        const int ex = carry + inc - room;
                        if (b < nb) {
                            int left = rem0 - ex;
                            left = left > 0 ? left : 0;
                            const int xb = l + (room < left ? room : left);
                            w.x[o0 + b] = (uint16_t)xb;
                            const int s = w.bsz[o0 + b];
                            if (xb > 0 && take[b] > v) v = take[b];
                            if (xb < s && rest[b] > v) v = rest[b];
                        }
                        carry += __shfl_sync(FULLW, inc, 31);
                    }
                    v = wmaxd(v);
                    __syncwarp();
                    h.hit(w, j, v);
                    return 1;
                } else {
                    const double I = h.incumbent();
                    // sequential-cut replay: strict improvements only, no tie band
                    const double Ie = (!MG_NONNEG(S) && S.seq_cut) ? I : I * (1.0 - TIE_EPS);
                    if (!last_feasible_warp(w, o0, nb, dd, Ie, false, rest, take)) continue;
                    double hiv = Ie;
                    while (true) {
                        double c = NEG_INF;
                        #pragma unroll 1
                        for (int b = lane; b < nb; b += 32) {
                            if (rest[b] < hiv && rest[b] > c) c = rest[b];
                            if (w.hi[o0 + b] && take[b] < hiv && take[b] > c) c = take[b];
                        }
                        c = wmaxd(c);
                        if (c <= NEG_INF) break;
                        if (last_feasible_warp(w, o0, nb, dd, c, true, rest, take))
                            hiv = c;
                        else
                            break;
                    }
                    const double v = hiv > 0.0 ? hiv : 0.0;
                    if (v < I) {
                        // materialise one allocation reaching v (greedy fill at hiv) so the
                        // planner can seed later FIRST probes with the argmin
                        int mylo3 = 0;
                        #pragma unroll 1
                        for (int b = lane; b < nb; b += 32)
                            mylo3 += (rest[b] <= hiv) ? 0 : w.bsz[o0 + b];
                        const int rem0 = dd - wsum(mylo3);
                        int carry = 0;
                        #pragma unroll 1
                        for (int c = 0; c < nb; c += 32) {
                            const int b = c + lane;
                            int l = 0, room = 0;
                            if (b < nb) {
                                const int s = w.bsz[o0 + b];
                                const bool rok = rest[b] <= hiv;
                                const bool tok = w.hi[o0 + b] && take[b] <= hiv;
                                l = rok ? 0 : s;
                                room = (tok ? s : 0) - l;
                            }
                            const int inc = wscan_incl(room);
                            const int ex = carry + inc - room;
                            if (b < nb) {
                                int left = rem0 - ex;
                                left = left > 0 ? left : 0;
                                w.x[o0 + b] = (uint16_t)(l + (room < left ? room : left));
                            }
                            carry += __shfl_sync(FULLW, inc, 31);
                        }
                        __syncwarp();
                        h.improve_leaf(w, j, v);
                    }
                }
                continue;
            }
            if (!first_comp_warp(w, o0, nb, dd)) continue;
            __syncwarp();  // every lane has read ph[j] (loop head) before lane 0 rewrites it
            if (lane == 0) w.ph[j] = 1;
            __syncwarp();
        } else {
            if (!next_comp_warp(w, o0, nb)) {
                __syncwarp();
                if (lane == 0) w.ph[j] = 0;
                __syncwarp();
                continue;
            }
        }
        // ---- build the child (level j+1 blocks + their stats) ----
        h.count_node();
        if (ps_lvl != j) {
            parent_stats_warp(S, R, w, j);
            ps_lvl = j;
        }
        const int o1 = w.loff[j + 1];
        const int c1 = w.lcap[j + 1];
        const int uu = w.sU[j];
        const double ff = w.sFp[j], bo = w.sB[j], ba = w.sBase[j];
        int carry = 0;
        #pragma unroll 1
        for (int c = 0; c < nb; c += 32) {
            const int b = c + lane;
            int xb = 0, s = 0, cnt = 0;
            if (b < nb) {
                xb = w.x[o0 + b];
                s = w.bsz[o0 + b];
                cnt = (xb > 0) + (xb < s);
            }
            const int inc = wscan_incl(cnt);
            int pos = carry + inc - cnt;
            if (b < nb) {
                const unsigned mk = w.bmk[o0 + b];
                if (xb > 0 && pos < c1) {
                    w.bsz[o1 + pos] = (uint16_t)xb;
                    w.bmk[o1 + pos] = (uint16_t)(mk | (1u << j));
                    w.cu[pos] = w.pu[b] + uu;
                    w.cm[pos] = w.pm[b] + ff;
                    w.cs[pos] = w.psum[b] + bo;
                    w.cb[pos] = w.pmb[b] > ba ? w.pmb[b] : ba;
                    w.cP[pos] = w.pP[b] * bo;
                    const double bx = ba - S.e2 * bo;
                    if (!MG_SELF(S)) w.cmx[pos] = w.pmx[b] > bx ? w.pmx[b] : bx;
                    ++pos;
                } else if (xb > 0) {
                    ++pos;
                }
                if (xb < s && pos < c1) {
                    w.bsz[o1 + pos] = (uint16_t)(s - xb);
                    w.bmk[o1 + pos] = (uint16_t)mk;
                    w.cu[pos] = w.pu[b];
                    w.cm[pos] = w.pm[b];
                    w.cs[pos] = w.psum[b];
                    w.cb[pos] = w.pmb[b];
                    w.cP[pos] = w.pP[b];
                    if (!MG_SELF(S)) w.cmx[pos] = w.pmx[b];
                }
            }
            carry += __shfl_sync(FULLW, inc, 31);
        }
        const int m = carry;
        if (m > c1) {
            h.overflow();
            return 2;
        }
        if (lane == 0) {
            w.nb[j + 1] = (uint16_t)m;
            w.used[j + 1] = w.used[j] + w.sDU[j];
        }
        __syncwarp();
        const double thr = h.thr(S);
        bool prune = false;
        // (when only the closed-form last level remains, its batch screen subsumes this)
        #pragma unroll 1
        for (int l = j + 1; l < k && l <= j + S.lookahead && !prune &&
                            !(j + 1 == k - 1 && MG_NONNEG(S));
             ++l) {
            const int n = S.lvl_n[l], off = S.lvl_off[l];
            // lanes over options (32 at a time), each lane scanning the m child blocks:
            // "some option before the first stop (t == 2) passes opt_test and finds d2
            // GPUs with room" — the same predicate as testing the options one by one
            bool ok = false;
            #pragma unroll 1
            for (int c = 0; c < n && !ok; c += 32) {
                const int o = c + lane;
                const int t = o < n ? opt_test(S, R, off + o, thr) : 2;
                const unsigned stop = __ballot_sync(FULLW, t == 2);
                const int first_stop = stop ? __ffs(stop) - 1 : 32;
                bool mine = false;
                if (t == 0 && lane < first_stop) {
                    const int rr = off + o;
                    const int d2 = R.d[rr], u2 = R.u[rr];
                    const double f2 = R.fp[rr], b2 = R.B[rr], a2 = R.base[rr];
                    int cnt = 0;
                    #pragma unroll 1
                    for (int b = 0; b < m && cnt < d2; ++b) {
                        if (w.cu[b] + u2 > S.L) continue;
                        if (w.cm[b] + f2 > S.cap_slack) continue;
                        if (MG_NONNEG(S) && MG_SELF(S)) {
                            const double mb = w.cb[b] > a2 ? w.cb[b] : a2;
                            if (mb + S.e1 + S.e2 * (w.cs[b] + b2) > thr) continue;
                        }
                        cnt += w.bsz[o1 + b];
                    }
                    mine = cnt >= d2;
                }
                ok = wany(mine);
                if (stop) break;
            }
            if (!ok) prune = true;
        }
        if (prune) continue;
        ++j;
        if (lane == 0) {
            w.ph[j] = 0;
            w.oc[j] = -1;
            w.oe[j] = (int16_t)S.lvl_n[j];
            w.vbase[j] = -1;
            // the child stats are exactly the new level's parent stats (same summation
            // order as block_stats): swap the buffers instead of recomputing them
            int* ti = w.pu; w.pu = w.cu; w.cu = ti;
            double* t;
            t = w.pm; w.pm = w.cm; w.cm = t;
            t = w.psum; w.psum = w.cs; w.cs = t;
            t = w.pmb; w.pmb = w.cb; w.cb = t;
            t = w.pP; w.pP = w.cP; w.cP = t;
            t = w.pmx; w.pmx = w.cmx; w.cmx = t;
        }
        __syncwarp();
        ps_lvl = j;
    }
    return 0;
}

// ---- cursor load / store by a whole warp ----
template <class C>
__device__ __forceinline__ void load_cont_warp(const Spec& S, const Rows& R, const C& c, Walk& w,
                                               bool ancestors = true) {
    const int lane = lane_id();
    const int dep = c.depth;
    const int o = w.loff[dep];
    #pragma unroll 1
    for (int b = lane; b < c.nb; b += 32) {
        w.bsz[o + b] = c.bsz[b];
        w.bmk[o + b] = c.bmk[b];
        if (c.ph) {
            w.x[o + b] = c.x[b];
            w.lo[o + b] = c.lo[b];
            w.hi[o + b] = c.hi[b];
        }
    }
    __syncwarp();
    if (lane == 0) {
        #pragma unroll 1
        for (int l = 0; l < dep; ++l) sel_set(S, R, w, l, c.opt[l]);
        w.nb[dep] = c.nb;
        w.used[dep] = c.used;
        w.ph[dep] = (uint8_t)c.ph;
        w.oc[dep] = c.oc;
        w.oe[dep] = c.oe;
        w.vbase[dep] = -1;
        if (c.ph) sel_set(S, R, w, dep, c.oc);
        // only FIRST needs them (hit paths compare every level); MIN skips the rebuild
        #pragma unroll 1
        for (int l = ancestors ? dep - 1 : -1; l >= 0; --l) {
            const int oc1 = w.loff[l + 1], ol = w.loff[l];
            const unsigned bit = 1u << l;
            int nbl = 0;
            #pragma unroll 1
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
    __syncwarp();
}

// Cursor for the rest of level l: ph 1 = compositions after the current x of opt[l], then
// the options after it up to oe[l]; ph 0 = options oc_from+1 .. oe[l]-1 (range split).
template <class C>
__device__ __forceinline__ void store_cont_warp(const Walk& w, int l, int ph, C& c,
                                                int oc_from = -1) {
    const int lane = lane_id();
    const int o = w.loff[l];
    const int nb = w.nb[l];
    #pragma unroll 1
    for (int b = lane; b < nb; b += 32) {
        c.bsz[b] = w.bsz[o + b];
        c.bmk[b] = w.bmk[o + b];
        if (ph) {
            c.x[b] = w.x[o + b];
            c.lo[b] = w.lo[o + b];
            c.hi[b] = w.hi[o + b];
        }
    }
    if (lane == 0) {
        c.key = 0;
        #pragma unroll 1
        for (int i = 0; i < MAXK; ++i) c.opt[i] = i < l ? w.opt[i] : 0;
        c.depth = (uint16_t)l;
        c.nb = (uint16_t)nb;
        c.ph = (uint16_t)ph;
        c.oc = ph ? (int16_t)w.opt[l] : (int16_t)oc_from;
        c.oe = w.oe[l];
        c.used = w.used[l];
    }
    __syncwarp();
}

}  // namespace mg
