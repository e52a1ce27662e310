// pack.cu — candidate-option tables built on the device.
//
// k_pack_options: one CTA per module.  Threads enumerate (d, units) over the profiled d
// axis and the quota lattice, evaluate the surface lookup (perf_model.hpp:124-147,
// bracket :174-192, restated operation for operation; -fmad=false), apply the hull and
// memory filters of candidate_options (stage_eval.hpp:68-85), then the CTA sorts the rows
// by (base latency, d, units) (stage_eval.hpp:87-91) with a bitonic sort in shared memory
// and writes the flat SoA table the search kernels read.  The host only ships the raw
// surface grids.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "pack.hpp"

namespace mg {

#define CKP(x)                                                                         \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                     " at " #x);                                       \
    } while (0)

constexpr int PK_THREADS = 256;
constexpr int PK_MAXROWS = 1024;  // d values x quota levels per module (32 KB of smem)
constexpr double PK_TOL = 1e-12;  // kAxisTolerance, perf_model.hpp:50

struct PackSurf {  // one module's grid, SoA, axes ascending
    int nd, na;
    int goff;      // offset of its grid in the flat arrays (nd*na points)
    double membase;
    double dv[PACK_MAXD], av[PACK_MAXA];
};

__device__ void bracket_dev(const double* ax, int n, double v, bool lg, int& lo, int& hi,
                            double& w) {
    for (int i = 0; i < n; ++i) {
        double av = fabs(v) > 1.0 ? fabs(v) : 1.0;
        if (fabs(ax[i] - v) <= PK_TOL * av) {
            lo = hi = i;
            w = 0.0;
            return;
        }
    }
    int h = 0;
    while (h < n && !(v < ax[h])) ++h;
    int l = h - 1;
    double sv = lg ? log2(v) : v, sl = lg ? log2(ax[l]) : ax[l], sh = lg ? log2(ax[h]) : ax[h];
    lo = l;
    hi = h;
    w = (sv - sl) / (sh - sl);
}

// ScalingSurface::lookup: field 0 latency, 1 bandwidth_util, 2 memory
__device__ double lookup_dev(const PackSurf& s, const double* g0, const double* g1,
                             const double* g2, int d, double a, int field) {
    int dl, dh, al, ah;
    double wd, wa;
    bracket_dev(s.dv, s.nd, (double)d, true, dl, dh, wd);
    bracket_dev(s.av, s.na, a, false, al, ah, wa);
    const double* g = field == 0 ? g0 : (field == 1 ? g1 : g2);
    g += s.goff;
    if (dl == dh && al == ah) return g[dl * s.na + al];
    double v00 = g[dl * s.na + al], v01 = g[dl * s.na + ah];
    double v10 = g[dh * s.na + al], v11 = g[dh * s.na + ah];
    double lo = v00 + (v01 - v00) * wa;
    double hi = v10 + (v11 - v10) * wa;
    return lo + (hi - lo) * wd;
}

struct PRow {
    double base, B, fp;
    int d, u;
};

__device__ bool row_less(const PRow& x, const PRow& y) {
    if (x.base != y.base) return x.base < y.base;
    if (x.d != y.d) return x.d < y.d;
    return x.u < y.u;
}

__global__ void __launch_bounds__(PK_THREADS)
    k_pack_options(const PackSurf* surfs, const double* glat, const double* gbw,
                   const double* gmem, int G, int L, double cap, int* counts, int* errs,
                   PRow* out) {
    __shared__ PRow rows[PK_MAXROWS];
    __shared__ int n;
    const PackSurf& s = surfs[blockIdx.x];
    if (threadIdx.x == 0) n = 0;
    __syncthreads();
    const double amin = s.av[0], amax = s.av[s.na - 1];
    const bool has_d1 = (int)s.dv[0] <= 1 && 1 <= (int)s.dv[s.nd - 1];
    for (int c = threadIdx.x; c < s.nd * L; c += blockDim.x) {
        const int di = c / L, units = c % L + 1;
        const int d = (int)s.dv[di];
        if (d > G) continue;
        const double a = (double)units / L;
        if (a < amin - PK_TOL || a > amax + PK_TOL) continue;
        if (!has_d1) {  // solo_bandwidth looks up d = 1 (perf_model.hpp:420-422)
            errs[blockIdx.x] = 1;
            continue;
        }
        const double fp = lookup_dev(s, glat, gbw, gmem, d, a, 2) + s.membase;
        if (fp > cap) continue;
        PRow r;
        r.base = lookup_dev(s, glat, gbw, gmem, d, a, 0);
        r.B = lookup_dev(s, glat, gbw, gmem, 1, a, 1);
        r.fp = fp;
        r.d = d;
        r.u = units;
        int slot = atomicAdd(&n, 1);
        if (slot < PK_MAXROWS) rows[slot] = r;
    }
    __syncthreads();
    const int cnt = n < PK_MAXROWS ? n : PK_MAXROWS;
    int pw = 1;
    while (pw < cnt) pw <<= 1;
    for (int i = cnt + threadIdx.x; i < pw; i += blockDim.x) {
        rows[i].base = 1e308;  // padding sorts last
        rows[i].d = 1 << 30;
        rows[i].u = 1 << 30;
    }
    __syncthreads();
    // bitonic sort by (base, d, units)
    for (int k = 2; k <= pw; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < pw; i += blockDim.x) {
                int p = i ^ j;
                if (p > i) {
                    bool up = (i & k) == 0;
                    PRow x = rows[i], y = rows[p];
                    if (up ? row_less(y, x) : row_less(x, y)) {
                        rows[i] = y;
                        rows[p] = x;
                    }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) out[blockIdx.x * PK_MAXROWS + i] = rows[i];
    if (threadIdx.x == 0) counts[blockIdx.x] = n > PK_MAXROWS ? -1 : n;
}

// evaluate_workload (profiler.hpp:65-89), operation for operation (-fmad=false; fp64 div /
// min / max are IEEE on the device).  ceil(log2(d)) is taken as the integer ceil-log2,
// which equals the host's std::ceil(std::log2(double(d))) for every d >= 1: log2 of a
// non-power of two is at least 1/(d ln 2) away from an integer, far above one ulp.
__global__ void k_gen_surfaces(const GenWorkload* ws, int nw, GenCluster c, const int* dset,
                               int nd, const double* aset, int na, double demand_scale,
                               GenPoint* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nw * nd * na) return;
    const int ai = i % na, di = (i / na) % nd, wi = i / (na * nd);
    const GenWorkload w = ws[wi];
    const int d = dset[di];
    const double a = aset[ai];
    const double eta0 = 0.85 + 0.15 * a / w.knee;
    const double eta = eta0 < 1.0 ? eta0 : 1.0;  // std::min(1.0, x)
    const double compute_time = (w.flops / d) / (a * c.peak_compute * eta);
    const double io_time = (w.bytes / d) / c.peak_bandwidth;
    double sync_time = 0.0;
    if (d > 1) {
        int e = 0;
        while ((1LL << e) < (long long)d) ++e;
        sync_time = c.alpha * (double)e + c.beta * w.grad;
    }
    GenPoint p;
    p.d = d;
    p.a = a;
    const double dp_eff = 1.0 + w.dp_penalty * (d - 1);
    const double mx = compute_time < io_time ? io_time : compute_time;  // std::max(ct, io)
    p.latency = mx * dp_eff + sync_time + w.fixed;
    const double sa = compute_time / p.latency;
    p.sm_active = sa < 1.0 ? sa : 1.0;
    const double bu = io_time / mx * demand_scale;
    p.bandwidth_util = bu < 1.0 ? bu : 1.0;
    p.memory = w.act_base + w.mem_per_quota * a + w.grad / d;
    out[i] = p;
}

std::vector<GenPoint> generate_surfaces_device(const std::vector<GenWorkload>& ws,
                                               const GenCluster& c, const std::vector<int>& d_set,
                                               const std::vector<double>& a_set,
                                               double demand_scale, int device) {
    CKP(cudaSetDevice(device));
    const size_t n = ws.size() * d_set.size() * a_set.size();
    std::vector<GenPoint> res(n);
    if (n == 0) return res;
    GenWorkload* dw;
    int* dd;
    double* da;
    GenPoint* dout;
    CKP(cudaMalloc(&dw, sizeof(GenWorkload) * ws.size()));
    CKP(cudaMalloc(&dd, sizeof(int) * d_set.size()));
    CKP(cudaMalloc(&da, sizeof(double) * a_set.size()));
    CKP(cudaMalloc(&dout, sizeof(GenPoint) * n));
    CKP(cudaMemcpy(dw, ws.data(), sizeof(GenWorkload) * ws.size(), cudaMemcpyHostToDevice));
    CKP(cudaMemcpy(dd, d_set.data(), sizeof(int) * d_set.size(), cudaMemcpyHostToDevice));
    CKP(cudaMemcpy(da, a_set.data(), sizeof(double) * a_set.size(), cudaMemcpyHostToDevice));
    const int T = 256;
    k_gen_surfaces<<<(int)((n + T - 1) / T), T>>>(dw, (int)ws.size(), c, dd, (int)d_set.size(),
                                                  da, (int)a_set.size(), demand_scale, dout);
    CKP(cudaGetLastError());
    CKP(cudaMemcpy(res.data(), dout, sizeof(GenPoint) * n, cudaMemcpyDeviceToHost));
    cudaFree(dw);
    cudaFree(dd);
    cudaFree(da);
    cudaFree(dout);
    return res;
}

namespace {
struct Arena {
    int device = -1;
    void *host = nullptr, *dev = nullptr, *stream = nullptr;
    size_t cap = 0;
};
size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }
std::mutex g_arena_mu;
std::vector<Arena*> g_arenas;

// The calling thread holds g_arena_mu while it uses the arena (pack_options_device).
Arena& arena(int device, size_t bytes) {
    Arena* a = nullptr;
    for (Arena* x : g_arenas)
        if (x->device == device) a = x;
    if (!a) {
        a = new Arena;
        a->device = device;
        cudaStream_t s;
        CKP(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        a->stream = s;
        g_arenas.push_back(a);
    }
    if (a->cap < bytes) {
        if (a->host) cudaFreeHost(a->host);
        if (a->dev) cudaFree(a->dev);
        a->host = a->dev = nullptr;
        a->cap = 0;
        const size_t c = std::max(bytes, (size_t)1 << 20);
        CKP(cudaMallocHost(&a->host, c));
        CKP(cudaMalloc(&a->dev, c));
        a->cap = c;
    }
    return *a;
}
}  // namespace

std::vector<std::vector<PackedRow>> pack_options_device(const std::vector<PackInput>& mods, int G,
                                                        int L, double cap, int device,
                                                        long long* h2d_bytes,
                                                        std::vector<int>* range_err) {
    CKP(cudaSetDevice(device));
    const int M = (int)mods.size();
    std::vector<std::vector<PackedRow>> res(M);
    if (M == 0) return res;
    std::lock_guard<std::mutex> lk(g_arena_mu);
    std::vector<PackSurf> hs(M);
    std::vector<double> lat, bw, mem;
    for (int m = 0; m < M; ++m) {
        const PackInput& in = mods[m];
        if ((int)in.dv.size() > PACK_MAXD || (int)in.av.size() > PACK_MAXA)
            throw std::runtime_error("surface grid too large for the packing kernel");
        PackSurf& s = hs[m];
        s.nd = (int)in.dv.size();
        s.na = (int)in.av.size();
        s.goff = (int)lat.size();
        s.membase = in.membase;
        for (int i = 0; i < s.nd; ++i) s.dv[i] = in.dv[i];
        for (int i = 0; i < s.na; ++i) s.av[i] = in.av[i];
        lat.insert(lat.end(), in.lat.begin(), in.lat.end());
        bw.insert(bw.end(), in.bw.begin(), in.bw.end());
        mem.insert(mem.end(), in.mem.begin(), in.mem.end());
    }
    for (const auto& in : mods)
        if ((long long)L * (long long)in.dv.size() > PK_MAXROWS)
            throw std::runtime_error("quota_levels x d values exceed the packing kernel");
    // one staging arena per device (pinned host + device, grow-only, reused by every context
    // created afterwards): one upload, one kernel, one read-back, one synchronisation
    const size_t npts = lat.size();
    const size_t o_surf = 0;
    const size_t o_lat = align_up(o_surf + sizeof(PackSurf) * M);
    const size_t o_bw = o_lat + 8 * npts;
    const size_t o_mem = o_bw + 8 * npts;
    const size_t in_bytes = align_up(o_mem + 8 * npts);
    const size_t o_cnt = in_bytes;
    const size_t o_err = o_cnt + sizeof(int) * M;
    const size_t o_rows = align_up(o_err + sizeof(int) * M);
    const size_t total = o_rows + sizeof(PRow) * PK_MAXROWS * M;
    Arena& ar = arena(device, total);
    char* h = static_cast<char*>(ar.host);
    char* d = static_cast<char*>(ar.dev);
    std::memcpy(h + o_surf, hs.data(), sizeof(PackSurf) * M);
    std::memcpy(h + o_lat, lat.data(), 8 * npts);
    std::memcpy(h + o_bw, bw.data(), 8 * npts);
    std::memcpy(h + o_mem, mem.data(), 8 * npts);
    cudaStream_t st = static_cast<cudaStream_t>(ar.stream);
    CKP(cudaMemcpyAsync(d, h, in_bytes, cudaMemcpyHostToDevice, st));
    CKP(cudaMemsetAsync(d + o_err, 0, sizeof(int) * M, st));
    if (h2d_bytes) *h2d_bytes += (long long)in_bytes;
    k_pack_options<<<M, PK_THREADS, 0, st>>>(
        reinterpret_cast<const PackSurf*>(d + o_surf), reinterpret_cast<const double*>(d + o_lat),
        reinterpret_cast<const double*>(d + o_bw), reinterpret_cast<const double*>(d + o_mem), G, L,
        cap, reinterpret_cast<int*>(d + o_cnt), reinterpret_cast<int*>(d + o_err),
        reinterpret_cast<PRow*>(d + o_rows));
    CKP(cudaGetLastError());
    CKP(cudaMemcpyAsync(h + o_cnt, d + o_cnt, total - o_cnt, cudaMemcpyDeviceToHost, st));
    CKP(cudaStreamSynchronize(st));
    std::vector<int> counts(M), errs(M);
    std::memcpy(counts.data(), h + o_cnt, sizeof(int) * M);
    std::memcpy(errs.data(), h + o_err, sizeof(int) * M);
    const PRow* rows = reinterpret_cast<const PRow*>(h + o_rows);
    if (range_err) range_err->assign(errs.begin(), errs.end());
    for (int m = 0; m < M; ++m) {
        if (counts[m] < 0) throw std::runtime_error("too many candidate options for one module");
        for (int i = 0; i < counts[m]; ++i) {
            const PRow& r = rows[(size_t)m * PK_MAXROWS + i];  // (arena: read before unlock)
            res[m].push_back(PackedRow{r.d, r.u, r.base, r.B, r.fp});
        }
    }
    return res;
}

}  // namespace mg
