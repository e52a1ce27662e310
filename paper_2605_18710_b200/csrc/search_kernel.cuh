// search_kernel.cuh — the stage-search kernel (control block, walker hooks, k_search).
//
// Included by engine.cu (generic kernel `k_search`: every model flag read from the Spec)
// and by engine_fast.cu (`k_search_fast`: include_self, non-negative coefficients and the
// multiplicative term fixed at compile time through MG_SPECIALIZE — the configuration of
// every BASELINE config — so the kernel carries only the code that runs; the search is
// the same code either way).
#pragma once
#ifndef MG_KSEARCH_NAME
#define MG_KSEARCH_NAME k_search
#endif

namespace mg {

// Control block.  Fields that different threads write often live on their own 128-B
// lines so spinning workers do not serialize the busy ones.
struct Ctl {
    alignas(128) unsigned long long inc;  // MIN incumbent, fp64 bits (values are >= 0)
    double abort_below;
    int abort;
    int overflow;
    alignas(128) unsigned long long q_head;
    alignas(128) unsigned long long q_tail;
    unsigned long long q_cap;
    unsigned long long q_base;  // first ticket of this launch (q_head - q_base: pieces taken)
    alignas(128) unsigned long long outstanding;  // queued + in-flight cursors
    alignas(128) unsigned int idle;
    unsigned int walkers;  // resident walkers of this launch
    alignas(128) int lock;  // FIRST: best hit, published under a seqlock
    int ver;
    int has_hit;            // FIRST: a hit is published; MIN: an argmin leaf is stored
    double leaf_val;
    alignas(128) unsigned long long nodes, leaves;
    // trace >= 3 only: walker-ns inside pieces, pieces walked, hand-over request outcomes
    // (0 ring full, 1 range < 2, 2 rest only below the level limit, 3 floor above it, 4 deep,
    // 5 handed over, 6 pieces abandoned, 7 requests; 8 + l: requests at level l)
    unsigned long long busy, pieces;
    unsigned long long dbg[16];
};

// CTA-local hand-off: one cursor slot per CTA in shared memory that a busy walker fills for
// an idle sibling (no ring ticket, no L2 round trip, no contention with the grid).  The
// payload is packed into 32-bit words written and read with shared-memory atomics (the flag
// `state` orders them; atomics keep the two warps' accesses race-free by construction):
//   hdr[0] depth | nb << 16, hdr[1] ph | oc << 16, hdr[2] oe, hdr[3] used, hdr[4..9] opt pairs;
//   blk[b] = {bsz | bmk << 16, x | lo << 16, hi} for the LOCAL_CAP blocks at `depth`.
// state: 0 empty, 1 being written or read, 2 full.
constexpr int LOCAL_CAP = 32;  // blocks a local piece can carry (levels <= 5 always fit)
struct LocalSlot {
    int state;
    int idle;  // siblings of this CTA waiting for work
    unsigned hdr[10];
    unsigned blk[LOCAL_CAP][3];
};

// Hooks of one walker (a warp).  Everything that steers control flow is decided by
// lane 0 and broadcast, so the warp stays converged.
struct WarpHooks {
    Ctl* ctl;
    const Spec* sp;
    LocalSlot* ls;
    int mode;
    long long steps;
    double inc_cache;
    int refresh;
    Leaf* leaf_out;
    HitPath* best;
    Cont* q;
    int* ready;
    unsigned long long nodes, leaves;
    const Walk* w;
    int cur_level;
    int don_period;
    int may_donate;
    long long deep_after;
    int tail_idle;
    long long tail_after;
    // solo: the only walker of its search (no hand-overs): control state it alone writes is
    // kept in registers, so the DFS makes no L2 round trips for it
    int solo;
    int local_abort;
    int has_hit_local;
    double abort_below;

    __device__ bool hit_precedes() {  // lane 0 only
        int v0 = *(volatile int*)&ctl->ver;
        if (v0 & 1) return false;
        __threadfence();
        bool before = path_precedes_rest((const volatile HitPath*)best, *w, cur_level);
        __threadfence();
        int v1 = *(volatile int*)&ctl->ver;
        return v0 == v1 && before;
    }
    // 0 continue, 2 abandon (MIN restart, or a FIRST hit precedes all that is left),
    // 3 idle walkers are waiting: donate shallow work (4: deeper levels too)
    __device__ int abort() {
        ++steps;
        // global control state is read only every don_period steps: a per-step L2 round
        // trip (broadcast from lane 0) was the single hottest stall of the walker loop
        if ((steps & (unsigned)(don_period - 1)) != 0) return 0;
        if (solo) {
            int code = 0;
            if (lane_id() == 0) {
                if (local_abort)
                    code = 2;
                else if (mode == MODE_FIRST && has_hit_local &&
                         path_precedes_rest((const HitPath*)best, *w, cur_level))
                    code = 2;
            }
            return __shfl_sync(FULLW, code, 0);
        }
        int code = 0;
        if (lane_id() == 0) {
            if (*(volatile int*)&ctl->abort) {
                code = 2;
            } else {
                if (mode == MODE_FIRST && *(volatile int*)&ctl->has_hit && hit_precedes()) {
                    code = 2;
                } else if (may_donate && sp->local_don && *(volatile int*)&ls->idle > 0 &&
                           *(volatile int*)&ls->state == 0) {
                    code = 5;  // a sibling of this CTA waits and the local slot is free
                } else {
                    unsigned int idle = may_donate ? *(volatile unsigned int*)&ctl->idle : 0u;
                    if (idle) {
                        unsigned long long qn = *(volatile unsigned long long*)&ctl->q_tail -
                                                *(volatile unsigned long long*)&ctl->q_head;
                        if (qn == 0)  // queue drained and walkers waiting
                            // a walker that has been on its piece for long holds a big
                            // subtree: let it split deeper levels too
                        {
                            // tail phase (tail_idle > 0): the ramp-up is over (every walker
                            // has had a piece) and more than 1/tail_idle of them are idle
                            const unsigned wk = *(volatile unsigned int*)&ctl->walkers;
                            const bool tail =
                                tail_idle > 0 && (unsigned long long)idle * tail_idle > wk &&
                                *(volatile unsigned long long*)&ctl->q_head - ctl->q_base > wk;
                            code = steps > (tail ? tail_after : deep_after) ? 4 : 3;
                        }
                    }
                }
            }
        }
        return __shfl_sync(FULLW, code, 0);
    }
    __device__ void hit(const Walk& wk, int j, double v) {
        if (lane_id() == 0) {
            while (atomicCAS(&ctl->lock, 0, 1) != 0) __nanosleep(64);
            __threadfence();
            bool better = !*(volatile int*)&ctl->has_hit ||
                          path_cmp((const volatile HitPath*)best, wk, j) > 0;
            if (better) {
                atomicAdd(&ctl->ver, 1);
                __threadfence();
                path_store((volatile HitPath*)best, wk, j);
                store_leaf(wk, j, v, *leaf_out);
                ctl->has_hit = 1;
                __threadfence();
                atomicAdd(&ctl->ver, 1);
            }
            __threadfence();
            atomicExch(&ctl->lock, 0);
            // the other shards of this search: same seqlocked publication in their control
            // blocks (one lock held at a time), system-scope fences for peer GPUs
            if (better)
                for (int p = 0; p < sp->n_peer; ++p)
                    publish_peer(static_cast<Ctl*>(sp->peer_ctl[p]),
                                 static_cast<HitPath*>(sp->peer_best[p]),
                                 static_cast<Leaf*>(sp->peer_leaf[p]), wk, j, v);
        }
        __syncwarp();
    }
    __device__ static void publish_peer(Ctl* pc, HitPath* pb, Leaf* pl, const Walk& wk, int j,
                                        double v) {
        while (atomicCAS(&pc->lock, 0, 1) != 0) __nanosleep(64);
        __threadfence_system();
        const bool better = !*(volatile int*)&pc->has_hit ||
                            path_cmp((const volatile HitPath*)pb, wk, j) > 0;
        if (better) {
            atomicAdd(&pc->ver, 1);
            __threadfence_system();
            path_store((volatile HitPath*)pb, wk, j);
            store_leaf(wk, j, v, *pl);
            *(volatile int*)&pc->has_hit = 1;
            __threadfence_system();
            atomicAdd(&pc->ver, 1);
        }
        __threadfence_system();
        atomicExch(&pc->lock, 0);
    }
    // push the cursor "rest of level l" onto the ring queue (ticket t -> slot t % cap,
    // published by writing ready[slot] = t + 1)
    // ph 1: "rest of level l" (after the current composition); ph 0: options from mid on
    __device__ bool donate(const Walk& wk, int l, int ph, int mid) {
        long long slot = -1;
        unsigned long long t = 0;
        if (lane_id() == 0) {
            t = *(volatile unsigned long long*)&ctl->q_tail;
            while (true) {
                unsigned long long head = *(volatile unsigned long long*)&ctl->q_head;
                if (t + 1 - head > ctl->q_cap) break;  // ring full
                unsigned long long old = atomicCAS(&ctl->q_tail, t, t + 1);
                if (old == t) {
                    slot = (long long)(t % ctl->q_cap);
                    atomicAdd(&ctl->outstanding, 1ULL);
                    break;
                }
                t = old;
            }
        }
        slot = __shfl_sync(FULLW, slot, 0);
        if (slot < 0) return false;
        store_cont_warp(wk, l, ph, q[slot], mid - 1);
        __threadfence();  // every lane's part of the cursor is visible ...
        __syncwarp();
        if (lane_id() == 0) {
            __threadfence();
            atomicExch(&ready[slot], (int)(t + 1));  // ... before it is published
        }
        __syncwarp();
        return true;
    }
    // hand "rest of level l" (ph 1) or options mid.. (ph 0) to an idle sibling through the
    // CTA's shared-memory slot; counts in `outstanding` like a ring piece
    __device__ bool donate_local(const Walk& wk, int l, int ph, int mid) {
        const int nb = wk.nb[l];
        if (nb > LOCAL_CAP) return false;  // (warp-uniform: shared-memory walk state)
        int ok = 0;
        const int lane = lane_id();
        if (lane == 0 && atomicCAS(&ls->state, 0, 1) == 0) {
            atomicAdd(&ctl->outstanding, 1ULL);
            ok = 1;
        }
        ok = __shfl_sync(FULLW, ok, 0);
        if (!ok) return false;
        // the same cursor store_cont_warp writes: "rest of level l" (ph 1) or options
        // mid.. (ph 0), packed
        const int o = wk.loff[l];
        if (lane < nb) {
            const unsigned b0 = wk.bsz[o + lane], m0 = wk.bmk[o + lane];
            atomicExch(&ls->blk[lane][0], b0 | m0 << 16);
            if (ph) {
                atomicExch(&ls->blk[lane][1], (unsigned)wk.x[o + lane] | (unsigned)wk.lo[o + lane] << 16);
                atomicExch(&ls->blk[lane][2], (unsigned)wk.hi[o + lane]);
            }
        }
        if (lane < 6) {
            const unsigned a = 2 * lane < l ? wk.opt[2 * lane] : 0u;
            const unsigned b = 2 * lane + 1 < l ? wk.opt[2 * lane + 1] : 0u;
            atomicExch(&ls->hdr[4 + lane], a | b << 16);
        } else if (lane == 6) {
            atomicExch(&ls->hdr[0], (unsigned)l | (unsigned)nb << 16);
        } else if (lane == 7) {
            const int oc = ph ? (int)wk.opt[l] : mid - 1;
            atomicExch(&ls->hdr[1], (unsigned)ph | (unsigned)(uint16_t)(int16_t)oc << 16);
        } else if (lane == 8) {
            atomicExch(&ls->hdr[2], (unsigned)(uint16_t)wk.oe[l]);
        } else if (lane == 9) {
            atomicExch(&ls->hdr[3], (unsigned)wk.used[l]);
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            atomicExch(&ls->state, 2);
        }
        __syncwarp();
        return true;
    }
    __device__ double bcast_inc() {
        double I = 0.0;
        if (lane_id() == 0) I = __longlong_as_double(*(volatile long long*)&ctl->inc);
        return __shfl_sync(FULLW, I, 0);
    }
    __device__ double thr(const Spec& S) {
        if (mode != MODE_MIN) return S.thp;
        if (!solo && (refresh++ & 15) == 0) {
            double I = bcast_inc();
            inc_cache = I < inc_cache ? I : inc_cache;
        }
        double t = inc_cache >= POS_INF ? POS_INF : inc_cache * (1.0 - TIE_EPS);
        return t < S.thp ? t : S.thp;
    }
    __device__ double incumbent() {  // refreshed every 16 calls, like thr()
        if (!solo && (refresh++ & 15) == 0) {
            double I = bcast_inc();
            inc_cache = I < inc_cache ? I : inc_cache;
        }
        return inc_cache;
    }
    __device__ void improve(double v) {
        if (lane_id() == 0) {
            atomicMin(&ctl->inc, (unsigned long long)__double_as_longlong(v));
            if (v < abort_below) {
                atomicExch(&ctl->abort, 1);
                local_abort = 1;
            }
        }
        if (v < inc_cache) inc_cache = v;
        __syncwarp();
    }
    // MIN: lower the incumbent and keep the allocation that reached it
    __device__ void improve_leaf(const Walk& wk, int j, double v) {
        if (lane_id() == 0) {
            atomicMin(&ctl->inc, (unsigned long long)__double_as_longlong(v));
            if (v < abort_below) {
                atomicExch(&ctl->abort, 1);
                local_abort = 1;
            }
            // the other shards of this search prune with it at once (remote atomics over
            // NVLink for peer GPUs): no waiting for the end-of-launch merge
            for (int p = 0; p < sp->n_peer; ++p) {
                Ctl* pc = static_cast<Ctl*>(sp->peer_ctl[p]);
                atomicMin(&pc->inc, (unsigned long long)__double_as_longlong(v));
                if (v < abort_below) atomicExch(&pc->abort, 1);
            }
            while (atomicCAS(&ctl->lock, 0, 1) != 0) __nanosleep(64);
            __threadfence();
            if (!ctl->has_hit || v < ctl->leaf_val) {
                store_leaf(wk, j, v, *leaf_out);
                ctl->leaf_val = v;
                ctl->has_hit = 1;
            }
            __threadfence();
            atomicExch(&ctl->lock, 0);
        }
        if (v < inc_cache) inc_cache = v;
        __syncwarp();
    }
    __device__ void count_node() { ++nodes; }
    __device__ void count_leaf() { ++leaves; }
    __device__ void count_leaves(int n) { leaves += (unsigned long long)n; }
    __device__ void overflow() {
        if (lane_id() == 0) {
            atomicExch(&ctl->overflow, 1);
            atomicExch(&ctl->abort, 1);
        }
    }
    __device__ void level(int j) { cur_level = j; }
    __device__ void note(const Spec& S, int i) {
        if (S.timeline && lane_id() == 0) atomicAdd(&ctl->dbg[i], 1ull);
    }
};

constexpr int WPC = 4;  // walkers (warps) per CTA

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// trace timeline: spread one piece's busy interval [a, b) over the 0.25 ms bins
__device__ __noinline__ static void timeline_add(unsigned long long* tl, unsigned long long a, unsigned long long b) {
    unsigned long long t0 = *(volatile unsigned long long*)tl;
    if (t0 == 0) {
        atomicCAS(tl, 0ull, a);
        t0 = *(volatile unsigned long long*)tl;
    }
    if (a < t0) a = t0;
    if (b <= a) return;
    for (unsigned long long bin = (a - t0) / TL_BIN_NS; bin < (unsigned long long)TL_BINS; ++bin) {
        const unsigned long long lo = t0 + bin * TL_BIN_NS, hi = lo + TL_BIN_NS;
        const unsigned long long x = a > lo ? a : lo, y = b < hi ? b : hi;
        if (y <= x) break;
        atomicAdd(&tl[1 + bin], y - x);
    }
}

// trace >= 3: account one finished piece (busy time, timeline, log of long pieces)
__device__ __noinline__ static void trace_piece(const Spec& S, Ctl* ctl, unsigned long long g0, int d0,
                                                unsigned long long nodes) {
    unsigned long long* tl = S.timeline;
    const unsigned long long g1 = gtimer();
    atomicAdd(&ctl->busy, g1 - g0);
    atomicAdd(&ctl->pieces, 1ull);
    timeline_add(tl, g0, g1);
    if (g1 - g0 > 2000000ull) {  // pieces longer than 2 ms: start, end, depth, nodes
        unsigned long long* lg = tl + 1 + TL_BINS;
        const unsigned long long i = atomicAdd(lg, 1ull);
        if (i < (unsigned long long)TL_LOG) {
            lg[1 + 4 * i] = g0 - tl[0];
            lg[2 + 4 * i] = g1 - tl[0];
            lg[3 + 4 * i] = (unsigned long long)d0;
            lg[4 + 4 * i] = nodes;
        }
    }
}

// A launch runs up to MAXBATCH independent searches (one per module set of a GAHC round /
// probe wave): search s owns CTAs [cta_off[s], cta_off[s+1]), its own Spec, control block,
// hit path, leaf, root piece and a private slice of the cursor ring at q_off[s].
constexpr int MAXBATCH = 64;
struct BatchMap {
    int n;
    int cta_off[MAXBATCH + 1];
    long long q_off[MAXBATCH];
};

constexpr size_t SMEM_SPEC = (sizeof(Spec) + 15) & ~size_t(15);

// Per-search staging blob (host pinned and device mirror): Spec | Ctl | Leaf | root Cont,
// each 256-B aligned; searches of a batch are BLOB_STRIDE apart.
constexpr size_t blob_align(size_t x) { return (x + 255) & ~size_t(255); }
constexpr size_t BLOB_SPEC = 0;
constexpr size_t BLOB_CTL = BLOB_SPEC + blob_align(sizeof(Spec));
constexpr size_t BLOB_LEAF = BLOB_CTL + blob_align(sizeof(Ctl));
constexpr size_t BLOB_ROOT = BLOB_LEAF + blob_align(sizeof(Leaf));
constexpr size_t BLOB_STRIDE = BLOB_ROOT + blob_align(sizeof(Cont));

// dynamic shared memory of one CTA for a stage of k modules over G GPUs
static inline size_t smem_bytes(int G, int k, bool lean) {
    return SMEM_SPEC + WPC * walk_layout(G, k, lean).bytes + ((sizeof(LocalSlot) + 15) & ~size_t(15));
}

// One resident persistent grid per stage search.  Each warp is a walker: it pops a
// cursor from the shared ring queue and runs the warp-cooperative DFS on it; a busy
// walker that sees idle ones and a short queue donates its shallowest untried level.
// `outstanding` counts queued + in-flight cursors; every walker exits when it hits 0.
//   MIN:   shared incumbent (atomicMin on the fp64 bits), tie band TIE_EPS.
//   FIRST: hits are ordered by their reference-DFS path; the earliest is kept under a
//          seqlock, and work that lies after it is abandoned.
__global__ void __launch_bounds__(32 * WPC, MG_SPECIALIZE ? 7 : 6) MG_KSEARCH_NAME(const Spec* Sg, Rows R, Cont* Q, int* ready,
                                                     Ctl* ctl, HitPath* best, Leaf* leaf_out,
                                                     const Cont* root, const BatchMap map,
                                                     int ready0) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int sid_sh;
    if (threadIdx.x == 0) {
        int s = 0;
        while (s + 1 < map.n && (int)blockIdx.x >= map.cta_off[s + 1]) ++s;
        sid_sh = s;
    }
    __syncthreads();
    {
        // this CTA's search: its slice of every per-search array (blob stride = BLOB_STRIDE)
        const int sid = sid_sh;
        Sg = reinterpret_cast<const Spec*>(reinterpret_cast<const char*>(Sg) + sid * BLOB_STRIDE);
        ctl = reinterpret_cast<Ctl*>(reinterpret_cast<char*>(ctl) + sid * BLOB_STRIDE);
        leaf_out = reinterpret_cast<Leaf*>(reinterpret_cast<char*>(leaf_out) + sid * BLOB_STRIDE);
        root = reinterpret_cast<const Cont*>(reinterpret_cast<const char*>(root) + sid * BLOB_STRIDE);
        best += sid;
        Q += map.q_off[sid];
        ready += map.q_off[sid];
    }
    Spec& S = *reinterpret_cast<Spec*>(smem);
    {
        const int n = sizeof(Spec) / 4;
        const int* src = reinterpret_cast<const int*>(Sg);
        int* dst = reinterpret_cast<int*>(smem);
        for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
        if (threadIdx.x == 0) {
            LocalSlot* l0 = reinterpret_cast<LocalSlot*>(
                smem + SMEM_SPEC + WPC * walk_layout(Sg->G, Sg->k, MG_SPECIALIZE).bytes);
            atomicExch(&l0->state, 0);
            atomicExch(&l0->idle, 0);
        }
        __syncthreads();
    }
    const int wid = threadIdx.x >> 5;
    const int lane = lane_id();
    // no hand-overs (small trees): the first warp of the search's first CTA walks the whole
    // tree alone, everyone else leaves at once
    const bool solo = !S.donate;
    if (solo && ((int)blockIdx.x != map.cta_off[sid_sh] || wid != 0)) return;
    const size_t wbytes = walk_layout(S.G, S.k, MG_SPECIALIZE).bytes;
    unsigned char* wbase = smem + SMEM_SPEC + wid * wbytes;
    LocalSlot* ls = reinterpret_cast<LocalSlot*>(smem + SMEM_SPEC + WPC * wbytes);
    Walk& w = *reinterpret_cast<Walk*>(wbase);
    if (lane == 0) walk_carve(w, wbase, S.G, S.k, MG_SPECIALIZE);
    __syncwarp();
    unsigned long long nodes = 0, leaves = 0;
    if (solo) {
        load_cont_warp(S, R, *root, w, MG_MODE(S) == MODE_FIRST);
        WarpHooks h;
        h.ctl = ctl;
        h.sp = &S;
        h.ls = ls;
        h.mode = MG_MODE(S);
        h.steps = 0;
        h.refresh = 0;
        h.leaf_out = leaf_out;
        h.best = best;
        h.q = Q;
        h.ready = ready;
        h.nodes = 0;
        h.leaves = 0;
        h.w = &w;
        h.cur_level = 0;
        h.don_period = S.don_period;
        h.may_donate = 0;
        h.deep_after = S.deep_after;
        h.tail_idle = S.tail_idle;
        h.tail_after = S.tail_after;
        h.solo = 1;
        h.local_abort = 0;
        h.has_hit_local = ctl->has_hit;
        h.abort_below = ctl->abort_below;
        h.inc_cache = POS_INF;
        h.inc_cache = h.bcast_inc();
        dfs_warp(S, R, w, root->depth, h);
        __syncwarp();
        if (lane == 0) {
            ctl->outstanding = 0;
            atomicAdd(&ctl->nodes, h.nodes);
            atomicAdd(&ctl->leaves, h.leaves);
        }
        return;
    }
    while (true) {
        long long ticket = -1;
        if (lane == 0) {
            bool idle = false;
            unsigned backoff = 128;
            const unsigned backoff_cap = S.backoff_cap_ns;
            while (true) {
                if (*(volatile int*)&ctl->abort) break;
                // a sibling's piece in the CTA's slot first (shared memory, no contention)
                if (S.local_don && *(volatile int*)&ls->state == 2 &&
                    atomicCAS(&ls->state, 2, 1) == 2) {
                    ticket = -2;
                    break;
                }
                unsigned long long h = *(volatile unsigned long long*)&ctl->q_head;
                unsigned long long t = *(volatile unsigned long long*)&ctl->q_tail;
                if (h < t) {
                    if (atomicCAS(&ctl->q_head, h, h + 1) == h) {
                        ticket = (long long)h;
                        break;
                    }
                    continue;
                }
                if (*(volatile unsigned long long*)&ctl->outstanding == 0) break;
                if (!idle) {
                    atomicAdd(&ctl->idle, 1u);
                    if (S.local_don) atomicAdd(&ls->idle, 1);
                    idle = true;
                }
                __nanosleep(backoff);
                backoff = backoff < backoff_cap ? backoff * 2 : backoff_cap;
            }
            if (idle) {
                atomicSub(&ctl->idle, 1u);
                if (S.local_don) atomicSub(&ls->idle, 1);
            }
            // the root piece ships with the launch (`root`), every other piece is published
            // in the ring by its donor
            if (ticket >= 0 && ticket + 1 != ready0) {
                const long long slot = (long long)((unsigned long long)ticket % ctl->q_cap);
                while (*(volatile int*)&ready[slot] != (int)(ticket + 1)) __nanosleep(32);
                __threadfence();
            }
        }
        ticket = __shfl_sync(FULLW, ticket, 0);
        if (ticket == -1) break;
        int d0;
        if (ticket == -2) {
            // the sibling's piece: unpack it from the slot (atomic reads), free the slot,
            // then rebuild the walk from it exactly like a ring piece
            __threadfence_block();
            ContT<LOCAL_CAP> c;
            const unsigned h0 = atomicOr(&ls->hdr[0], 0u), h1 = atomicOr(&ls->hdr[1], 0u);
            c.depth = (uint16_t)(h0 & 0xffffu);
            c.nb = (uint16_t)(h0 >> 16);
            c.ph = (uint16_t)(h1 & 0xffffu);
            c.oc = (int16_t)(uint16_t)(h1 >> 16);
            c.oe = (int16_t)(uint16_t)(atomicOr(&ls->hdr[2], 0u) & 0xffffu);
            c.used = (int)atomicOr(&ls->hdr[3], 0u);
            c.key = 0;
            #pragma unroll
            for (int i = 0; i < 6; ++i) {
                const unsigned v = atomicOr(&ls->hdr[4 + i], 0u);
                c.opt[2 * i] = (uint16_t)(v & 0xffffu);
                c.opt[2 * i + 1] = (uint16_t)(v >> 16);
            }
            if (lane < c.nb) {
                const unsigned a = atomicOr(&ls->blk[lane][0], 0u);
                c.bsz[lane] = (uint16_t)(a & 0xffffu);
                c.bmk[lane] = (uint16_t)(a >> 16);
                if (c.ph) {
                    const unsigned b = atomicOr(&ls->blk[lane][1], 0u);
                    c.x[lane] = (uint16_t)(b & 0xffffu);
                    c.lo[lane] = (uint16_t)(b >> 16);
                    c.hi[lane] = (uint16_t)(atomicOr(&ls->blk[lane][2], 0u) & 0xffffu);
                }
            }
            __syncwarp();
            if (lane == 0) atomicExch(&ls->state, 0);
            d0 = c.depth;
            load_cont_warp(S, R, c, w, MG_MODE(S) == MODE_FIRST);
        } else {
            const long long slot = (long long)((unsigned long long)ticket % ctl->q_cap);
            __threadfence();
            const Cont& piece = ticket + 1 == ready0 ? *root : Q[slot];
            load_cont_warp(S, R, piece, w, MG_MODE(S) == MODE_FIRST);
            d0 = piece.depth;
        }
        WarpHooks h;
        h.ctl = ctl;
        h.sp = &S;
        h.ls = ls;
        h.mode = MG_MODE(S);
        h.steps = 0;
        h.refresh = 0;
        h.leaf_out = leaf_out;
        h.best = best;
        h.q = Q;
        h.ready = ready;
        h.nodes = 0;
        h.leaves = 0;
        h.w = &w;
        h.cur_level = 0;
        h.don_period = S.don_period;
        h.may_donate = S.donate;
        h.deep_after = S.deep_after;
        h.tail_idle = S.tail_idle;
        h.tail_after = S.tail_after;
        h.solo = 0;
        h.local_abort = 0;
        h.has_hit_local = 0;
        h.abort_below = ctl->abort_below;
        h.inc_cache = POS_INF;
        h.inc_cache = h.bcast_inc();
        if (S.timeline && lane == 0) w.t_start = gtimer();
        dfs_warp(S, R, w, d0, h);
        if (S.timeline && lane == 0) trace_piece(S, ctl, w.t_start, d0, h.nodes);
        nodes += h.nodes;
        leaves += h.leaves;
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicAdd(&ctl->outstanding, ~0ULL);  // -1
        }
    }
    if (lane == 0) {
        atomicAdd(&ctl->nodes, nodes);
        atomicAdd(&ctl->leaves, leaves);
    }
}

}  // namespace mg
