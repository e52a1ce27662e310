/* mosaic_oracle.c — plain-C restatement of the reference planner hot path.
 * TEST INFRASTRUCTURE ONLY (see mosaic_oracle.h).  Build: make -C oracle restatement
 * (gcc -O2 -ffp-contract=off).  Citations are /root/reference/proj/include/mosaic/.
 */
#include "mosaic_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXM 64
#define MAXD 16
#define MAXA 16
#define MAXG 1024
#define MAXK 16
#define TOL 1e-12 /* kAxisTolerance, perf_model.hpp:50 */

typedef struct {
    int d;
    double a, lat, bw, mem, sm;
} Pt;

typedef struct {
    char id[32];
    double membase;
    int nd, na;
    double dv[MAXD], av[MAXA];
    Pt grid[MAXD * MAXA];
} Surf;

typedef struct {
    int d, u;
    double base, bw, fp;
} Cand;

struct mo_problem {
    int n;
    Surf s[MAXM];
    int ne, eu[512], ev[512];
    int G;
    double cap, e1, e2, e3;
    int additive, self, L, prune, cache;
    double tol;
    int range_err[MAXM];
    Cand* opts[MAXM];
    int nopt[MAXM];
    mo_plan last;
    mo_stage* last_stages;
};

/* ------------------------------------------------------------------ mt19937_64 */
typedef struct {
    uint64_t mt[312];
    int i;
} MT;
static void mt_seed(MT* m, uint64_t s) {
    m->mt[0] = s;
    for (int i = 1; i < 312; ++i)
        m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
    m->i = 312;
}
static uint64_t mt_next(MT* m) {
    if (m->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            uint64_t x = (m->mt[k] & 0xFFFFFFFF80000000ULL) | (m->mt[(k + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
            m->mt[k] = m->mt[(k + 156) % 312] ^ xa;
        }
        m->i = 0;
    }
    uint64_t y = m->mt[m->i++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* std::normal_distribution<double>(0,1) over mt19937_64, libstdc++ (bits/random.tcc):
 * generate_canonical<double,53> = u / 2^64 (clamped below 1), polar method with the
 * second variate cached; result * stddev + mean. */
void mo_normals(uint64_t seed, int n, double* out) {
    MT m;
    mt_seed(&m, seed);
    int avail = 0;
    double saved = 0.0;
    for (int i = 0; i < n; ++i) {
        double ret;
        if (avail) {
            avail = 0;
            ret = saved;
        } else {
            double x, y, r2;
            do {
                double c1 = (double)mt_next(&m) / 18446744073709551616.0;
                if (c1 >= 1.0) c1 = 0x1.fffffffffffffp-1;
                x = 2.0 * c1 - 1.0;
                double c2 = (double)mt_next(&m) / 18446744073709551616.0;
                if (c2 >= 1.0) c2 = 0x1.fffffffffffffp-1;
                y = 2.0 * c2 - 1.0;
                r2 = x * x + y * y;
            } while (r2 > 1.0 || r2 == 0.0);
            const double mult = sqrt(-2.0 * log(r2) / r2);
            saved = x * mult;
            avail = 1;
            ret = y * mult;
        }
        out[i] = ret * 1.0 + 0.0;
    }
}

/* ------------------------------------------------------------------ profiler.hpp */
typedef struct {
    char id[32];
    double flops, bytes, grad, knee, act, mpq, fixed, dpp;
} Work;

/* detail::make_workload, profiler.hpp:185-199 */
static Work make_workload(const char* id, double tflops, double ci, double params_b, double knee,
                          double batch) {
    Work w;
    memset(&w, 0, sizeof w);
    snprintf(w.id, sizeof w.id, "%s", id);
    w.flops = tflops * 1e12 * batch;
    w.bytes = w.flops / ci;
    w.grad = params_b * 1e9 * 2.0;
    w.knee = knee;
    w.act = 1e9 + params_b * 1e9;
    w.mpq = 2e9 + 0.2e9 * tflops;
    w.fixed = 40e-3;
    w.dpp = 0.02;
    return w;
}

/* evaluate_workload, profiler.hpp:57-89 (ClusterSpec defaults, core.hpp:52-59) */
static Pt evaluate_workload(const Work* w, int d, double a) {
    const double peak_c = 500e12, peak_b = 3.35e12, alpha = 5e-6, beta = 2.2e-12;
    double eta = fmin(1.0, 0.85 + 0.15 * a / w->knee);
    double ct = (w->flops / d) / (a * peak_c * eta);
    double io = (w->bytes / d) / peak_b;
    double sync = 0.0;
    if (d > 1) sync = alpha * ceil(log2((double)d)) + beta * w->grad;
    Pt p;
    p.d = d;
    p.a = a;
    double dp = 1.0 + w->dpp * (d - 1);
    double mx = ct > io ? ct : io;
    p.lat = mx * dp + sync + w->fixed;
    p.sm = fmin(1.0, ct / p.lat);
    p.bw = fmin(1.0, io / mx * 1.0);
    p.mem = w->act + w->mpq * a + w->grad / d;
    return p;
}

/* ScalingSurface ctor (perf_model.hpp:57-79): axes sorted, tolerance-merged */
static void axis_insert(double* ax, int* n, double v) {
    for (int i = 0; i < *n; ++i)
        if (fabs(ax[i] - v) <= TOL) return;
    int pos = 0;
    while (pos < *n && ax[pos] < v) ++pos;
    for (int i = *n; i > pos; --i) ax[i] = ax[i - 1];
    ax[pos] = v;
    ++*n;
}
static int axis_index(const double* ax, int n, double v) {
    for (int i = 0; i < n; ++i)
        if (fabs(ax[i] - v) <= TOL) return i;
    return -1;
}
static void surface_build(Surf* s, const char* id, const Pt* pts, int np) {
    memset(s, 0, sizeof *s);
    snprintf(s->id, sizeof s->id, "%s", id);
    for (int i = 0; i < np; ++i) {
        axis_insert(s->dv, &s->nd, (double)pts[i].d);
        axis_insert(s->av, &s->na, pts[i].a);
    }
    for (int i = 0; i < np; ++i)
        s->grid[axis_index(s->dv, s->nd, pts[i].d) * s->na + axis_index(s->av, s->na, pts[i].a)] =
            pts[i];
}

/* generate_surface with default grids, profiler.hpp:44-54, 91-111 */
static void generate_surface(Surf* s, const Work* w, int G) {
    Pt pts[MAXD * MAXA];
    int np = 0;
    for (int d = 1; d <= G; d *= 2)
        for (int i = 1; i <= 10; ++i) pts[np++] = evaluate_workload(w, d, i / 10.0);
    surface_build(s, w->id, pts, np);
}

/* bracket, perf_model.hpp:174-192 */
static void bracket(const double* ax, int n, double v, int lg, int* lo, int* hi, double* w) {
    for (int i = 0; i < n; ++i)
        if (fabs(ax[i] - v) <= TOL * fmax(1.0, fabs(v))) {
            *lo = *hi = i;
            *w = 0.0;
            return;
        }
    int h = 0;
    while (h < n && !(v < ax[h])) ++h; /* upper_bound */
    int l = h - 1;
    double sv = lg ? log2(v) : v, sl = lg ? log2(ax[l]) : ax[l], sh = lg ? log2(ax[h]) : ax[h];
    *lo = l;
    *hi = h;
    *w = (sv - sl) / (sh - sl);
}

/* ScalingSurface::lookup, perf_model.hpp:124-147; returns 0, or -1 outside the hull */
static int lookup(const Surf* s, int d, double a, double out[4]) {
    if (d < (int)s->dv[0] || d > (int)s->dv[s->nd - 1]) return -1;
    if (a < s->av[0] - TOL || a > s->av[s->na - 1] + TOL) return -1;
    int dl, dh, al, ah;
    double wd, wa;
    bracket(s->dv, s->nd, (double)d, 1, &dl, &dh, &wd);
    bracket(s->av, s->na, a, 0, &al, &ah, &wa);
    const Pt *p00 = &s->grid[dl * s->na + al], *p01 = &s->grid[dl * s->na + ah];
    const Pt *p10 = &s->grid[dh * s->na + al], *p11 = &s->grid[dh * s->na + ah];
    if (dl == dh && al == ah) {
        out[0] = p00->lat;
        out[1] = p00->bw;
        out[2] = p00->mem;
        out[3] = p00->sm;
        return 0;
    }
#define BLEND(F)                                                  \
    do {                                                          \
        double lo_ = p00->F + (p01->F - p00->F) * wa;             \
        double hi_ = p10->F + (p11->F - p10->F) * wa;             \
        out[k_++] = lo_ + (hi_ - lo_) * wd;                       \
    } while (0)
    int k_ = 0;
    BLEND(lat);
    BLEND(bw);
    BLEND(mem);
    BLEND(sm);
#undef BLEND
    return 0;
}

/* ------------------------------------------------------------------ inputs */
static void add(mo_problem* p, Work* ws, int* nw, Work w) {
    ws[(*nw)++] = w;
    (void)p;
}
static int idx_of(Work* ws, int nw, const char* id) {
    for (int i = 0; i < nw; ++i)
        if (!strcmp(ws[i].id, id)) return i;
    return -1;
}
static void edge(mo_problem* p, Work* ws, int nw, const char* u, const char* v) {
    p->eu[p->ne] = idx_of(ws, nw, u);
    p->ev[p->ne] = idx_of(ws, nw, v);
    ++p->ne;
}

/* make_preset, profiler.hpp:229-285 */
static int preset(mo_problem* p, const char* name, int count, Work* ws, int* nw) {
#define W(id, t, c, pb, k) add(p, ws, nw, make_workload(id, t, c, pb, k, 64.0))
    if (!strcmp(name, "clip")) {
        W("vision", 4.17, 35.2, 0.30, 0.60);
        W("text", 1.04, 20.5, 0.12, 0.45);
        W("align", 0.40, 8.0, 0.02, 0.35);
        edge(p, ws, *nw, "vision", "align");
        edge(p, ws, *nw, "text", "align");
    } else if (!strcmp(name, "qwen3vl")) {
        W("vision", 2.58, 82.4, 0.60, 0.70);
        W("text", 0.15, 2.1, 0.05, 0.30);
        W("llm", 22.27, 145.2, 7.00, 0.80);
        edge(p, ws, *nw, "vision", "llm");
        edge(p, ws, *nw, "text", "llm");
    } else if (!strcmp(name, "unifiedio2")) {
        W("vision", 1.48, 24.6, 0.25, 0.55);
        W("audio", 1.06, 21.8, 0.20, 0.50);
        W("text", 0.10, 4.5, 0.04, 0.30);
        W("llm", 16.70, 110.5, 3.20, 0.80);
        edge(p, ws, *nw, "vision", "llm");
        edge(p, ws, *nw, "audio", "llm");
        edge(p, ws, *nw, "text", "llm");
    } else if (!strcmp(name, "imagebind")) {
        const double b = 160.0;
        add(p, ws, nw, make_workload("vision", 4.17, 35.2, 0.40, 0.60, b));
        add(p, ws, nw, make_workload("audio", 2.09, 22.8, 0.25, 0.50, b));
        add(p, ws, nw, make_workload("text", 1.04, 20.5, 0.15, 0.45, b));
        add(p, ws, nw, make_workload("depth", 0.90, 15.0, 0.10, 0.40, b));
        add(p, ws, nw, make_workload("thermal", 0.70, 12.0, 0.08, 0.40, b));
        add(p, ws, nw, make_workload("imu", 0.20, 3.5, 0.04, 0.30, b));
        add(p, ws, nw, make_workload("align", 0.50, 9.0, 0.03, 0.35, b));
        const char* e[] = {"vision", "audio", "text", "depth", "thermal", "imu"};
        for (int i = 0; i < 6; ++i) edge(p, ws, *nw, e[i], "align");
    } else if (!strcmp(name, "ofasys")) {
        Work pool[9] = {
            make_workload("vision", 1.35, 18.2, 0.30, 0.55, 64.0),
            make_workload("text", 0.72, 12.5, 0.15, 0.45, 64.0),
            make_workload("audio", 0.95, 14.8, 0.20, 0.50, 64.0),
            make_workload("video", 1.80, 22.0, 0.35, 0.60, 64.0),
            make_workload("depth", 0.60, 10.0, 0.12, 0.40, 64.0),
            make_workload("thermal", 0.50, 9.0, 0.10, 0.40, 64.0),
            make_workload("imu", 0.15, 2.5, 0.04, 0.30, 64.0),
            make_workload("box", 0.20, 5.0, 0.05, 0.35, 64.0),
            make_workload("action", 0.30, 6.5, 0.07, 0.35, 64.0),
        };
        int enc = count > 0 ? count - 1 : 9;
        if (enc < 1 || enc > 9) return -1;
        for (int i = 0; i < enc; ++i) add(p, ws, nw, pool[i]);
        W("backbone", 4.80, 41.6, 2.40, 0.70);
        for (int i = 0; i < enc; ++i) edge(p, ws, *nw, pool[i].id, "backbone");
    } else {
        return -1;
    }
#undef W
    return 0;
}

mo_problem* mo_synth(const char* spec, int levels) {
    mo_problem* p = (mo_problem*)calloc(1, sizeof(mo_problem));
    Work ws[MAXM];
    int nw = 0;
    p->L = 10;
    p->cap = 80e9;
    p->e1 = 0.4e-3; /* default_ground_truth, bench.hpp:31-37 */
    p->e2 = 1.2e-3;
    p->e3 = 0.8e-3;
    p->self = 1;
    p->tol = 1e-3;
    p->prune = p->cache = 1;
    unsigned long long seed;
    int n, g;
    char name[64];
#define W(id, t, c, pb, k) add(p, ws, &nw, make_workload(id, t, c, pb, k, 64.0))
    if (sscanf(spec, "random:%llu:%d:%d", &seed, &n, &g) == 3) {
        /* random_instance, profiler.hpp:304-338 */
        MT mt;
        mt_seed(&mt, seed);
#define UNIF(lo, hi) ((lo) + ((hi) - (lo)) * ((double)(mt_next(&mt) >> 11) / (double)(1ULL << 53)))
        int star = 0;
        if (n >= 2) star = UNIF(0.0, 1.0) < 0.7;
        for (int i = 0; i < n; ++i) {
            char id[16];
            snprintf(id, sizeof id, "m%02d", i);
            int bb = star && i == n - 1;
            double tf = bb ? exp(UNIF(log(2.0), log(20.0))) : exp(UNIF(log(0.2), log(4.0)));
            double ci = exp(UNIF(log(2.0), log(150.0)));
            double pr = tf * UNIF(0.05, 0.3);
            double kn = UNIF(0.3, 0.8);
            add(p, ws, &nw, make_workload(id, tf, ci, pr, kn, 64.0));
        }
        if (star) {
            for (int i = 0; i + 1 < n; ++i) {
                p->eu[p->ne] = i;
                p->ev[p->ne++] = n - 1;
            }
        } else {
            for (int i = 0; i < n; ++i)
                for (int j = i + 1; j < n; ++j)
                    if (UNIF(0.0, 1.0) < 0.4) {
                        p->eu[p->ne] = i;
                        p->ev[p->ne++] = j;
                    }
        }
#undef UNIF
        p->G = g;
    } else if (sscanf(spec, "preset:%63[^:]:%d:%d", name, &n, &g) == 3) {
        if (preset(p, name, n, ws, &nw)) {
            free(p);
            return NULL;
        }
        p->G = g;
    } else if (!strcmp(spec, "cfg1")) {
        W("vision", 4.17, 35.2, 0.30, 0.60);
        W("text", 1.04, 20.5, 0.12, 0.45);
        p->G = 8;
    } else if (!strcmp(spec, "cfg2")) {
        W("vit", 4.17, 35.2, 0.30, 0.60);
        W("proj", 0.05, 4.0, 0.02, 0.30);
        W("llm", 22.27, 145.2, 7.00, 0.80);
        edge(p, ws, nw, "vit", "proj");
        edge(p, ws, nw, "proj", "llm");
        p->G = 16;
        p->L = 8;
    } else if (!strcmp(spec, "cfg3")) {
        W("vision", 2.58, 82.4, 0.60, 0.70);
        W("text", 0.15, 2.1, 0.05, 0.30);
        W("deepstack", 0.30, 6.0, 0.05, 0.35);
        W("llm", 22.27, 145.2, 7.00, 0.80);
        edge(p, ws, nw, "vision", "deepstack");
        edge(p, ws, nw, "deepstack", "llm");
        edge(p, ws, nw, "text", "llm");
        p->G = 32;
    } else if (!strcmp(spec, "cfg4")) {
        W("image", 4.17, 35.2, 0.30, 0.60);
        W("video", 1.80, 22.0, 0.35, 0.60);
        W("audio", 2.09, 22.8, 0.25, 0.50);
        W("llm", 16.70, 110.5, 3.20, 0.80);
        W("speech_dec", 0.95, 14.8, 0.20, 0.50);
        W("image_dec", 1.48, 24.6, 0.25, 0.55);
        edge(p, ws, nw, "image", "llm");
        edge(p, ws, nw, "video", "llm");
        edge(p, ws, nw, "audio", "llm");
        edge(p, ws, nw, "llm", "speech_dec");
        edge(p, ws, nw, "llm", "image_dec");
        p->G = 64;
    } else if (!strcmp(spec, "cfg5")) {
        preset(p, "ofasys", 8, ws, &nw);
        p->G = 128;
        p->L = 32;
    } else {
        free(p);
        return NULL;
    }
#undef W
    if (levels > 0) p->L = levels;
    p->n = nw;
    for (int i = 0; i < nw; ++i) {
        generate_surface(&p->s[i], &ws[i], p->G);
        p->s[i].membase = ws[i].grad * 3.0; /* make_spec, profiler.hpp:201-207 */
    }
    for (int i = 0; i < nw; ++i) p->nopt[i] = -1;
    return p;
}

void mo_set_model(mo_problem* p, double e1, double e2, double e3, int self, int additive,
                  double cap) {
    if (!isnan(e1)) p->e1 = e1;
    if (!isnan(e2)) p->e2 = e2;
    if (!isnan(e3)) p->e3 = e3;
    if (self >= 0) p->self = self;
    if (additive >= 0) p->additive = additive;
    if (!isnan(cap) && cap > 0) p->cap = cap;
    for (int i = 0; i < p->n; ++i) {
        free(p->opts[i]);
        p->opts[i] = NULL;
        p->nopt[i] = -1;
    }
}
void mo_set_solve_flags(mo_problem* p, int prune, int cache) {
    p->prune = prune;
    p->cache = cache;
}

void mo_free(mo_problem* p) {
    if (!p) return;
    for (int i = 0; i < p->n; ++i) free(p->opts[i]);
    free(p->last_stages);
    free(p);
}
int mo_num_modules(const mo_problem* p) { return p->n; }

/* ------------------------------------------------------------------ perf model */
static int nonneg(const mo_problem* p) { return p->e1 >= 0 && p->e2 >= 0 && (p->additive || p->e3 >= 0); }
/* InterferenceModel::delta, perf_model.hpp:239-241 */
static double delta(const mo_problem* p, double s, double pr) {
    return p->e1 + p->e2 * s + (p->additive ? 0.0 : p->e3 * pr);
}

static int cand_cmp(const void* a, const void* b) {
    const Cand *x = (const Cand*)a, *y = (const Cand*)b;
    if (x->base != y->base) return x->base < y->base ? -1 : 1;
    if (x->d != y->d) return x->d < y->d ? -1 : 1;
    return x->u < y->u ? -1 : (x->u > y->u);
}

/* candidate_options, stage_eval.hpp:68-93 (stable tie order is total here) */
static int options(mo_problem* p, int m) {
    if (p->nopt[m] >= 0) return p->nopt[m];
    const Surf* s = &p->s[m];
    Cand* out = (Cand*)malloc(sizeof(Cand) * (MAXD * 256 + 1));
    int n = 0;
    for (int di = 0; di < s->nd; ++di) {
        int d = (int)s->dv[di];
        if (d > p->G) continue;
        for (int u = 1; u <= p->L; ++u) {
            double a = (double)u / p->L;
            if (a < s->av[0] - TOL || a > s->av[s->na - 1] + TOL) continue;
            double o[4], o1[4];
            if (lookup(s, d, a, o) || lookup(s, 1, a, o1)) {
                p->range_err[m] = 1;
                continue;
            }
            double fp = o[2] + s->membase;
            if (fp > p->cap) continue;
            out[n].d = d;
            out[n].u = u;
            out[n].base = o[0];
            out[n].bw = o1[1];
            out[n].fp = fp;
            ++n;
        }
    }
    qsort(out, n, sizeof(Cand), cand_cmp);
    p->opts[m] = out;
    p->nopt[m] = n;
    return n;
}

int mo_options(mo_problem* p, int m, int* d, int* u, double* base, double* bw, double* fp) {
    int n = options(p, m);
    for (int i = 0; i < n && d; ++i) {
        d[i] = p->opts[m][i].d;
        u[i] = p->opts[m][i].u;
        base[i] = p->opts[m][i].base;
        bw[i] = p->opts[m][i].bw;
        fp[i] = p->opts[m][i].fp;
    }
    return n;
}

/* An allocation: entries sorted by module, each with its gpu list. */
typedef struct {
    int n;
    int mod[MAXK], d[MAXK], u[MAXK], ng[MAXK];
    double base[MAXK], bw[MAXK];
    const int* g[MAXK];
} Alloc;

/* rectified_latency + stage_time, perf_model.hpp:442-479 */
static double rect(const mo_problem* p, const Alloc* A, int e) {
    double worst = -1e300;
    for (int gi = 0; gi < A->ng[e]; ++gi) {
        int r = A->g[e][gi];
        double sum = 0.0, prod = 1.0;
        int res = 0;
        for (int f = 0; f < A->n; ++f) {
            int on = 0;
            for (int t = 0; t < A->ng[f]; ++t)
                if (A->g[f][t] == r) {
                    on = 1;
                    break;
                }
            if (!on) continue;
            if (f == e && !p->self) continue;
            sum += A->bw[f];
            prod *= A->bw[f];
            ++res;
        }
        if (res == 0) prod = 0.0;
        double dl = delta(p, sum, prod);
        worst = worst > dl ? worst : dl;
    }
    return A->base[e] + worst;
}
static double stage_time_alloc(const mo_problem* p, const Alloc* A) {
    double worst = 0.0;
    for (int e = 0; e < A->n; ++e) {
        double r = rect(p, A, e);
        worst = worst > r ? worst : r;
    }
    return worst;
}

double mo_stage_time(mo_problem* p, int n, const int* ent, const int* gpus) {
    Alloc A;
    A.n = n;
    int off = 0;
    for (int e = 0; e < n; ++e) {
        A.mod[e] = ent[4 * e];
        A.d[e] = ent[4 * e + 1];
        A.u[e] = ent[4 * e + 2];
        A.ng[e] = ent[4 * e + 3];
        A.g[e] = gpus + off;
        off += A.ng[e];
        double a = (double)A.u[e] / p->L, o[4], o1[4];
        lookup(&p->s[A.mod[e]], A.d[e], a, o);
        lookup(&p->s[A.mod[e]], 1, a, o1);
        A.base[e] = o[0];
        A.bw[e] = o1[1];
    }
    return stage_time_alloc(p, &A);
}

/* ------------------------------------------------------------------ placement state */
typedef struct {
    mo_problem* p;
    int k;
    int mods[MAXK];
    double tau;
    int prune;
    /* per slot: filtered option list */
    const Cand* filt[MAXK][512];
    int nf[MAXK];
    int order[MAXK];
    int sufmin[MAXK + 1];
    int used[MAXG];
    double mem[MAXG], sumb[MAXG];
    int rslot[MAXG][MAXK], runits[MAXG][MAXK], nres[MAXG];
    const Cand* ch[MAXK];
    int chg[MAXK][MAXG], nchg[MAXK];
    long long nodes;
    /* ExactStageSolver */
    double best;
    int have;
    int bopt_d[MAXK], bopt_u[MAXK], bg[MAXK][MAXG], nbg[MAXK];
    double bbase[MAXK], bbw[MAXK];
} FS;

static void fill_alloc(const FS* f, Alloc* A) {
    /* entries sorted by module index (stage_eval.hpp:159-160) */
    int idx[MAXK];
    for (int i = 0; i < f->k; ++i) idx[i] = i;
    for (int i = 1; i < f->k; ++i)
        for (int j = i; j > 0 && f->mods[idx[j]] < f->mods[idx[j - 1]]; --j) {
            int t = idx[j];
            idx[j] = idx[j - 1];
            idx[j - 1] = t;
        }
    A->n = f->k;
    for (int e = 0; e < f->k; ++e) {
        int i = idx[e];
        A->mod[e] = f->mods[i];
        A->d[e] = f->ch[i]->d;
        A->u[e] = f->ch[i]->u;
        A->base[e] = f->ch[i]->base;
        A->bw[e] = f->ch[i]->bw;
        A->ng[e] = f->nchg[i];
        A->g[e] = f->chg[i];
    }
}

static void push(FS* f, int r, int slot, const Cand* c) {
    f->used[r] += c->u;
    f->mem[r] += c->fp;
    f->sumb[r] += c->bw;
    f->rslot[r][f->nres[r]] = slot;
    f->runits[r][f->nres[r]] = c->u;
    f->nres[r]++;
}
static void pop(FS* f, int r, const Cand* c) {
    f->used[r] -= c->u;
    f->mem[r] -= c->fp;
    f->sumb[r] -= c->bw;
    f->nres[r]--;
}
static int same_residents(const FS* f, int a, int b) {
    if (f->nres[a] != f->nres[b]) return 0;
    for (int i = 0; i < f->nres[a]; ++i)
        if (f->rslot[a][i] != f->rslot[b][i] || f->runits[a][i] != f->runits[b][i]) return 0;
    return 1;
}

/* FeasibilitySearch::admissible_after_placement, stage_eval.hpp:240-252 */
static int admissible_after(FS* f, int slot) {
    if (!f->prune) return 1;
    const mo_problem* p = f->p;
    for (int gi = 0; gi < f->nchg[slot]; ++gi) {
        int r = f->chg[slot][gi];
        for (int i = 0; i < f->nres[r]; ++i) {
            int s2 = f->rslot[r][i];
            double s = f->sumb[r];
            if (!p->self) s -= f->ch[s2]->bw;
            double lb = f->ch[s2]->base + p->e1 + p->e2 * s;
            if (lb > f->tau * (1.0 + 1e-12)) return 0;
        }
    }
    return 1;
}

/* FeasibilitySearch::verify_complete, stage_eval.hpp:254-265 */
static int verify_complete(FS* f) {
    Alloc A;
    fill_alloc(f, &A);
    for (int e = 0; e < A.n; ++e)
        if (rect(f->p, &A, e) > f->tau * (1.0 + 1e-12)) return 0;
    return 1;
}

static int fs_assign(FS* f, int pos);
/* FeasibilitySearch::place, stage_eval.hpp:192-222 */
static int fs_place(FS* f, int pos, int slot, const Cand* c, int from, int remaining) {
    const mo_problem* p = f->p;
    if (remaining == 0) {
        ++f->nodes;
        if (!admissible_after(f, slot)) return 0;
        return fs_assign(f, pos + 1);
    }
    if (p->G - from < remaining) return 0;
    int tried[MAXG], nt = 0;
    for (int r = from; r <= p->G - remaining; ++r) {
        if (f->used[r] + c->u > p->L) continue;
        if (f->mem[r] + c->fp > p->cap * (1.0 + 1e-12)) continue;
        int dup = 0;
        for (int t = 0; t < nt && !dup; ++t) dup = same_residents(f, tried[t], r);
        if (dup) continue;
        tried[nt++] = r;
        push(f, r, slot, c);
        f->chg[slot][f->nchg[slot]++] = r;
        if (fs_place(f, pos, slot, c, r + 1, remaining - 1)) return 1;
        f->nchg[slot]--;
        pop(f, r, c);
    }
    return 0;
}
/* FeasibilitySearch::assign, stage_eval.hpp:174-189 */
static int fs_assign(FS* f, int pos) {
    if (pos == f->k) return verify_complete(f);
    int free_units = 0;
    for (int r = 0; r < f->p->G; ++r) free_units += f->p->L - f->used[r];
    if (f->sufmin[pos] > free_units) return 0;
    int slot = f->order[pos];
    for (int i = 0; i < f->nf[slot]; ++i) {
        const Cand* c = f->filt[slot][i];
        f->ch[slot] = c;
        f->nchg[slot] = 0;
        if (fs_place(f, pos, slot, c, 0, c->d)) return 1;
    }
    return 0;
}

/* FeasibilitySearch::run, stage_eval.hpp:113-164 */
static int fs_run(FS* f, double tau) {
    mo_problem* p = f->p;
    f->tau = tau;
    int nn = nonneg(p);
    f->prune = nn;
    for (int i = 0; i < f->k; ++i) {
        int m = f->mods[i];
        int n = options(p, m);
        f->nf[i] = 0;
        for (int j = 0; j < n; ++j) {
            const Cand* c = &p->opts[m][j];
            double bound = c->base;
            if (nn) {
                bound += p->e1;
                if (p->self) bound += p->e2 * c->bw;
            }
            if (bound <= tau * (1.0 + 1e-12)) f->filt[i][f->nf[i]++] = c;
        }
        if (f->nf[i] == 0) return 0;
    }
    for (int i = 0; i < f->k; ++i) f->order[i] = i;
    for (int i = 1; i < f->k; ++i) /* stable insertion sort by (count, module) */
        for (int j = i; j > 0; --j) {
            int a = f->order[j - 1], b = f->order[j];
            if (f->nf[b] < f->nf[a] || (f->nf[b] == f->nf[a] && f->mods[b] < f->mods[a])) {
                f->order[j - 1] = b;
                f->order[j] = a;
            } else {
                break;
            }
        }
    f->sufmin[f->k] = 0;
    for (int i = f->k - 1; i >= 0; --i) {
        int best = 1 << 30;
        int s = f->order[i];
        for (int j = 0; j < f->nf[s]; ++j) {
            int dem = f->filt[s][j]->u * f->filt[s][j]->d;
            best = best < dem ? best : dem;
        }
        f->sufmin[i] = f->sufmin[i + 1] + best;
    }
    memset(f->used, 0, sizeof(int) * p->G);
    for (int r = 0; r < p->G; ++r) {
        f->mem[r] = 0.0;
        f->sumb[r] = 0.0;
        f->nres[r] = 0;
    }
    return fs_assign(f, 0);
}

static void export_stage(const FS* f, double t, mo_stage* out) {
    Alloc A;
    fill_alloc(f, &A);
    out->status = 0;
    out->stage_time = t;
    out->n_entries = A.n;
    int off = 0;
    for (int e = 0; e < A.n; ++e) {
        out->ent[4 * e] = A.mod[e];
        out->ent[4 * e + 1] = A.d[e];
        out->ent[4 * e + 2] = A.u[e];
        out->ent[4 * e + 3] = A.ng[e];
        for (int g = 0; g < A.ng[e]; ++g) out->gpus[off++] = A.g[e][g];
    }
}

static int mask_mods(uint64_t mask, int* mods) {
    int k = 0;
    for (int m = 0; m < 64; ++m)
        if (mask >> m & 1) mods[k++] = m;
    return k;
}

void mo_feasible(mo_problem* p, uint64_t mask, double tau, mo_stage* out) {
    FS* f = (FS*)calloc(1, sizeof(FS));
    f->p = p;
    f->k = mask_mods(mask, f->mods);
    out->probes = 1;
    if (fs_run(f, tau)) {
        Alloc A;
        fill_alloc(f, &A);
        export_stage(f, stage_time_alloc(p, &A), out);
    } else {
        out->status = 1;
    }
    free(f);
}

/* stage_eval, stage_eval.hpp:290-382 */
void mo_stage_eval(mo_problem* p, uint64_t mask, mo_stage* out) {
    FS* f = (FS*)calloc(1, sizeof(FS));
    f->p = p;
    f->k = mask_mods(mask, f->mods);
    memset(out, 0, sizeof(int) * 3);
    out->probes = 0;
    for (int i = 0; i < f->k; ++i)
        if (options(p, f->mods[i]) == 0) {
            out->status = 2;
            free(f);
            return;
        }
    int nn = nonneg(p);
    double tau_lo = 0.0, tau_hi = 0.0;
    for (int i = 0; i < f->k; ++i) {
        int m = f->mods[i];
        double lo = DBL_MAX, solo = DBL_MAX;
        for (int j = 0; j < p->nopt[m]; ++j) {
            const Cand* c = &p->opts[m][j];
            double bound = c->base;
            if (nn) {
                bound += p->e1;
                if (p->self) bound += p->e2 * c->bw;
            }
            lo = lo < bound ? lo : bound;
            double sr = c->base + (p->self ? delta(p, c->bw, c->bw) : delta(p, 0.0, 0.0));
            solo = solo < sr ? solo : sr;
        }
        if (nn) tau_lo = tau_lo > lo ? tau_lo : lo;
        tau_hi += solo;
    }
    mo_stage* cur = (mo_stage*)malloc(sizeof(mo_stage));
#define RUN(T) (++out->probes, fs_run(f, (T)))
    int ok = RUN(tau_hi);
    for (int a = 0; !ok && a < 60; ++a) {
        tau_hi *= 2.0;
        ok = RUN(tau_hi);
    }
    if (!ok) {
        out->status = 1;
        free(cur);
        free(f);
        return;
    }
    Alloc A;
    fill_alloc(f, &A);
    double tb = stage_time_alloc(p, &A);
    long long probes = out->probes;
    export_stage(f, tb, out);
    out->probes = probes;
    double lo = tau_lo < tb ? tau_lo : tb;
    while (tb - lo > p->tol * fabs(tb)) {
        double mid = 0.5 * (lo + tb);
        if (mid >= tb * (1.0 - 1e-12)) break;
        if (RUN(mid)) {
            fill_alloc(f, &A);
            tb = stage_time_alloc(p, &A);
            probes = out->probes;
            export_stage(f, tb, out);
            out->probes = probes;
        } else {
            lo = mid;
        }
    }
    for (int g = 0; g < 1000; ++g) {
        double pr = tb * (1.0 - 1e-9);
        if (pr <= lo) break;
        if (!RUN(pr)) break;
        fill_alloc(f, &A);
        tb = stage_time_alloc(p, &A);
        probes = out->probes;
        export_stage(f, tb, out);
        out->probes = probes;
    }
#undef RUN
    free(cur);
    free(f);
}

/* ------------------------------------------------------------------ ExactStageSolver */
static void ex_descend(FS* f, int i);
/* admissible(r), oracle.hpp:145-155 */
static int ex_admissible(FS* f, int r) {
    const mo_problem* p = f->p;
    if (!nonneg(p)) return 1;
    for (int t = 0; t < f->nres[r]; ++t) {
        int s = f->rslot[r][t];
        double sm = f->sumb[r];
        if (!p->self) sm -= f->ch[s]->bw;
        double lb = f->ch[s]->base + p->e1 + p->e2 * sm;
        if (lb >= f->best) return 0;
    }
    return 1;
}
/* place, oracle.hpp:157-180 */
static void ex_place(FS* f, int i, const Cand* c, int from, int remaining) {
    const mo_problem* p = f->p;
    if (remaining == 0) {
        for (int g = 0; g < f->nchg[i]; ++g)
            if (!ex_admissible(f, f->chg[i][g])) return;
        ex_descend(f, i + 1);
        return;
    }
    for (int r = from; r <= p->G - remaining; ++r) {
        if (f->used[r] + c->u > p->L) continue;
        if (f->mem[r] + c->fp > p->cap * (1.0 + 1e-12)) continue;
        push(f, r, i, c);
        f->chg[i][f->nchg[i]++] = r;
        ex_place(f, i, c, r + 1, remaining - 1);
        f->nchg[i]--;
        pop(f, r, c);
    }
}
/* descend, oracle.hpp:111-140 */
static void ex_descend(FS* f, int i) {
    mo_problem* p = f->p;
    if (i == f->k) {
        Alloc A;
        fill_alloc(f, &A);
        double t = stage_time_alloc(p, &A);
        if (t < f->best) {
            f->best = t;
            f->have = 1;
            for (int e = 0; e < A.n; ++e) {
                f->bopt_d[e] = A.d[e];
                f->bopt_u[e] = A.u[e];
                f->nbg[e] = A.ng[e];
                memcpy(f->bg[e], A.g[e], sizeof(int) * A.ng[e]);
            }
        }
        return;
    }
    int nn = nonneg(p);
    int m = f->mods[i];
    for (int j = 0; j < p->nopt[m]; ++j) {
        const Cand* c = &p->opts[m][j];
        double lb = c->base;
        if (nn) {
            lb += p->e1;
            if (p->self) lb += p->e2 * c->bw;
        }
        if (lb >= f->best) continue;
        f->ch[i] = c;
        f->nchg[i] = 0;
        ex_place(f, i, c, 0, c->d);
    }
}

void mo_exact(mo_problem* p, uint64_t mask, mo_stage* out) {
    FS* f = (FS*)calloc(1, sizeof(FS));
    f->p = p;
    f->k = mask_mods(mask, f->mods); /* ascending module order, oracle.hpp:89-90 */
    out->probes = 0;
    for (int i = 0; i < f->k; ++i)
        if (options(p, f->mods[i]) == 0) {
            out->status = 1;
            free(f);
            return;
        }
    f->best = DBL_MAX;
    ex_descend(f, 0);
    if (!f->have) {
        out->status = 1;
        free(f);
        return;
    }
    out->status = 0;
    out->stage_time = f->best;
    out->n_entries = f->k;
    int off = 0;
    for (int e = 0; e < f->k; ++e) {
        out->ent[4 * e] = f->mods[e];
        out->ent[4 * e + 1] = f->bopt_d[e];
        out->ent[4 * e + 2] = f->bopt_u[e];
        out->ent[4 * e + 3] = f->nbg[e];
        for (int g = 0; g < f->nbg[e]; ++g) out->gpus[off++] = f->bg[e][g];
    }
    free(f);
}

/* ------------------------------------------------------------------ GAHC + oracle */
static void topo_order(const mo_problem* p, int* order) {
    /* topological_order, core.hpp:211-238 (ready list kept sorted by id) */
    int indeg[MAXM] = {0}, ready[MAXM], nr = 0, no = 0;
    for (int e = 0; e < p->ne; ++e) indeg[p->ev[e]]++;
    for (int i = 0; i < p->n; ++i)
        if (!indeg[i]) ready[nr++] = i;
    for (int i = 1; i < nr; ++i)
        for (int j = i; j > 0 && strcmp(p->s[ready[j]].id, p->s[ready[j - 1]].id) < 0; --j) {
            int t = ready[j];
            ready[j] = ready[j - 1];
            ready[j - 1] = t;
        }
    while (nr) {
        int u = ready[0];
        memmove(ready, ready + 1, sizeof(int) * (nr - 1));
        --nr;
        order[no++] = u;
        for (int e = 0; e < p->ne; ++e) {
            if (p->eu[e] != u) continue;
            int v = p->ev[e];
            if (--indeg[v] == 0) {
                int pos = 0;
                while (pos < nr && strcmp(p->s[ready[pos]].id, p->s[v].id) < 0) ++pos;
                memmove(ready + pos + 1, ready + pos, sizeof(int) * (nr - pos));
                ready[pos] = v;
                ++nr;
            }
        }
    }
}
static void reach_masks(const mo_problem* p, uint64_t* reach) {
    int order[MAXM];
    topo_order(p, order);
    for (int i = 0; i < p->n; ++i) reach[i] = 0;
    for (int t = p->n - 1; t >= 0; --t) {
        int u = order[t];
        for (int e = 0; e < p->ne; ++e)
            if (p->eu[e] == u) reach[u] |= (1ULL << p->ev[e]) | reach[p->ev[e]];
    }
}

typedef struct {
    uint64_t mask;
    mo_stage* st;
} CacheEnt;

static int popc(uint64_t x) { return __builtin_popcountll(x); }

/* solve, solver.hpp:157-289 */
void mo_solve(mo_problem* p, mo_plan* out) {
    memset(out, 0, sizeof *out);
    CacheEnt* cache = (CacheEnt*)calloc(4096, sizeof(CacheEnt));
    int nc = 0;
    uint64_t reach[MAXM];
    reach_masks(p, reach);
    uint64_t masks[MAXM];
    mo_stage* res[MAXM];
    int ns = 0;
    int order[MAXM];
    topo_order(p, order);
#define EVAL(MASK, HIT, R)                                                   \
    do {                                                                     \
        (R) = NULL;                                                          \
        if (HIT) *(HIT) = 0;                                                 \
        if (p->cache)                                                        \
            for (int q_ = 0; q_ < nc; ++q_)                                  \
                if (cache[q_].mask == (MASK)) {                              \
                    (R) = cache[q_].st;                                      \
                    if (HIT) *(HIT) = 1;                                     \
                }                                                            \
        if (!(R)) {                                                          \
            mo_stage* s_ = (mo_stage*)malloc(sizeof(mo_stage));              \
            out->stage_eval_calls++;                                         \
            mo_stage_eval(p, (MASK), s_);                                    \
            if (s_->status == 2) {                                           \
                out->status = 2;                                             \
                free(s_);                                                    \
                goto done;                                                   \
            }                                                                \
            if (s_->status == 0) {                                           \
                out->feasibility_calls += s_->probes;                        \
                if (p->cache && nc < 4096) {                                 \
                    cache[nc].mask = (MASK);                                 \
                    cache[nc++].st = s_;                                     \
                }                                                            \
                (R) = s_;                                                    \
            } else {                                                         \
                free(s_);                                                    \
            }                                                                \
        }                                                                    \
    } while (0)
    for (int i = 0; i < p->n; ++i) {
        uint64_t mask = 1ULL << order[i];
        mo_stage* r;
        EVAL(mask, (int*)0, r);
        if (!r) {
            out->status = 2;
            goto done;
        }
        masks[ns] = mask;
        res[ns] = (mo_stage*)malloc(sizeof(mo_stage));
        memcpy(res[ns], r, sizeof(mo_stage));
        ++ns;
    }
    double minb[MAXM];
    for (int m = 0; m < p->n; ++m) {
        double b = DBL_MAX;
        int n = options(p, m);
        for (int j = 0; j < n; ++j) b = b < p->opts[m][j].base ? b : p->opts[m][j].base;
        minb[m] = b;
    }
    while (ns > 1) {
        int px[4096], py[4096], np = 0;
        for (int x = 0; x < ns; ++x)
            for (int y = x + 1; y < ns; ++y) {
                uint64_t up = masks[x];
                for (int z = x + 1; z < y; ++z) up |= masks[z];
                int legal = 1;
                for (int m = 0; m < 64 && legal; ++m)
                    if ((up >> m & 1) && (reach[m] & masks[y])) legal = 0;
                if (legal) {
                    px[np] = x;
                    py[np++] = y;
                }
            }
        for (int i = 1; i < np; ++i) /* candidate_order, solver.hpp:144-150 */
            for (int j = i; j > 0; --j) {
                uint64_t a = masks[px[j]] | masks[py[j]], b = masks[px[j - 1]] | masks[py[j - 1]];
                int lt = popc(a) != popc(b) ? popc(a) < popc(b)
                         : a != b           ? a < b
                                            : masks[px[j]] < masks[px[j - 1]];
                if (!lt) break;
                int t = px[j];
                px[j] = px[j - 1];
                px[j - 1] = t;
                t = py[j];
                py[j] = py[j - 1];
                py[j - 1] = t;
            }
        double dbest = 0.0;
        int bi = -1;
        mo_stage* bm = NULL;
        for (int i = 0; i < np; ++i) {
            int x = px[i], y = py[i];
            double tx = res[x]->stage_time, ty = res[y]->stage_time;
            if (p->prune) {
                double tlb = 0.0;
                uint64_t mm = masks[x] | masks[y];
                for (int m = 0; m < 64; ++m)
                    if (mm >> m & 1) tlb = tlb > minb[m] ? tlb : minb[m];
                if (tx + ty - tlb <= dbest) continue; /* early_prune, solver.hpp:95-97 */
            }
            mo_stage* mr;
            int hit;
            EVAL(masks[x] | masks[y], &hit, mr);
            if (!mr) continue;
            double gain = tx + ty - mr->stage_time;
            if (gain > dbest) {
                dbest = gain;
                bi = i;
                bm = mr;
            }
        }
        if (bi < 0) break;
        int x = px[bi], y = py[bi];
        masks[x] |= masks[y];
        memcpy(res[x], bm, sizeof(mo_stage));
        free(res[y]);
        for (int z = y; z + 1 < ns; ++z) {
            masks[z] = masks[z + 1];
            res[z] = res[z + 1];
        }
        --ns;
    }
    out->n_stages = ns;
    free(p->last_stages);
    p->last_stages = (mo_stage*)malloc(sizeof(mo_stage) * (ns ? ns : 1));
    for (int i = 0; i < ns; ++i) {
        out->masks[i] = masks[i];
        out->times[i] = res[i]->stage_time;
        out->iteration_time += res[i]->stage_time;
        memcpy(&p->last_stages[i], res[i], sizeof(mo_stage));
        free(res[i]);
    }
    ns = 0;
done:
    for (int i = 0; i < ns; ++i) free(res[i]);
    for (int i = 0; i < nc; ++i) free(cache[i].st);
    free(cache);
#undef EVAL
}

/* enumerate_partitions + brute_force_optimum, oracle.hpp:35-71, 206-255 */
typedef struct {
    mo_problem* p;
    uint64_t preds[MAXM], full;
    uint64_t cur[MAXM];
    int ncur;
    uint64_t memo_mask[1 << 12];
    mo_stage* memo[1 << 12];
    int nmemo;
    int have;
    double best;
    uint64_t best_masks[MAXM];
    int nbest;
    long long parts;
} BF;

static mo_stage* bf_stage(BF* b, uint64_t mask) {
    for (int i = 0; i < b->nmemo; ++i)
        if (b->memo_mask[i] == mask) return b->memo[i];
    mo_stage* s = (mo_stage*)malloc(sizeof(mo_stage));
    mo_exact(b->p, mask, s);
    b->memo_mask[b->nmemo] = mask;
    b->memo[b->nmemo++] = s;
    return s;
}
static void bf_rec(BF* b, uint64_t placed) {
    if (placed == b->full) {
        ++b->parts;
        double total = 0.0;
        int n = 0;
        for (int i = 0; i < b->ncur; ++i) {
            mo_stage* r = bf_stage(b, b->cur[i]);
            if (r->status != 0) return;
            total += r->stage_time;
            ++n;
            if (b->have && total >= b->best) return;
        }
        if (!b->have || total < b->best) {
            b->have = 1;
            b->best = total;
            b->nbest = b->ncur;
            memcpy(b->best_masks, b->cur, sizeof(uint64_t) * b->ncur);
        }
        return;
    }
    uint64_t avail = 0;
    for (int m = 0; m < b->p->n; ++m)
        if (!(placed >> m & 1) && (b->preds[m] & ~placed) == 0) avail |= 1ULL << m;
    for (uint64_t sub = avail; sub; sub = (sub - 1) & avail) {
        b->cur[b->ncur++] = sub;
        bf_rec(b, placed | sub);
        b->ncur--;
    }
}

void mo_brute_force(mo_problem* p, mo_plan* out) {
    memset(out, 0, sizeof *out);
    if (p->n > 8) {
        out->status = 4;
        return;
    }
    BF* b = (BF*)calloc(1, sizeof(BF));
    b->p = p;
    for (int e = 0; e < p->ne; ++e) b->preds[p->ev[e]] |= 1ULL << p->eu[e];
    b->full = (1ULL << p->n) - 1;
    bf_rec(b, 0);
    out->partitions = b->parts;
    if (!b->have) {
        out->status = 1;
    } else {
        out->n_stages = b->nbest;
        free(p->last_stages);
        p->last_stages = (mo_stage*)malloc(sizeof(mo_stage) * b->nbest);
        for (int i = 0; i < b->nbest; ++i) {
            mo_stage* r = bf_stage(b, b->best_masks[i]);
            out->masks[i] = b->best_masks[i];
            out->times[i] = r->stage_time;
            memcpy(&p->last_stages[i], r, sizeof(mo_stage));
        }
        out->iteration_time = b->best;
    }
    for (int i = 0; i < b->nmemo; ++i) free(b->memo[i]);
    free(b);
}

void mo_plan_stage(mo_problem* p, int s, mo_stage* out) {
    if (p->last_stages) memcpy(out, &p->last_stages[s], sizeof(mo_stage));
}
