// sim.cu — Monte-Carlo plan replay on the device.
//
// k_simulate restates simulate() (simulator.hpp:68-119) with one thread per seed: each
// thread owns a std::mt19937_64 stream (seeded exactly like the reference) and draws
// std::normal_distribution<double>(0, 1) the way libstdc++ does (Marsaglia polar method
// over generate_canonical<double, 53>, with the second variate cached), so a seed replays
// the same perturbation sequence as the reference.  Without perturbation the replay is
// bit-identical; with it, the only difference can come from the device's log/exp
// (≤ 1 ulp each, vs glibc), which the tests bound by a 1e-12 relative tolerance.
// Module durations start from the rectified latencies the batched evaluator k_eval
// produced for the plan's stages (bit-identical to perf_model.hpp:442-464).
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "sim.hpp"

namespace mg {

#define CKS(x)                                                                         \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                     " at " #x);                                       \
    } while (0)

struct Mt64 {  // std::mt19937_64: n = 312, m = 156, r = 31
    unsigned long long s[312];
    int i;
};

__device__ void mt_seed(Mt64& m, unsigned long long seed) {
    m.s[0] = seed;
#pragma unroll 1
    for (int i = 1; i < 312; ++i)
        m.s[i] = 6364136223846793005ULL * (m.s[i - 1] ^ (m.s[i - 1] >> 62)) +
                 (unsigned long long)i;
    m.i = 312;
}

__device__ unsigned long long mt_next(Mt64& m) {
    if (m.i >= 312) {
#pragma unroll 1
        for (int k = 0; k < 312; ++k) {
            const int k1 = k + 1 < 312 ? k + 1 : 0, km = k + 156 < 312 ? k + 156 : k - 156;
            const unsigned long long x =
                (m.s[k] & 0xFFFFFFFF80000000ULL) | (m.s[k1] & 0x7FFFFFFFULL);
            unsigned long long xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            m.s[k] = m.s[km] ^ xa;
        }
        m.i = 0;
    }
    unsigned long long y = m.s[m.i++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

// generate_canonical<double, 53>(mt19937_64): one draw, u / 2^64, clamped below 1
__device__ double canonical(Mt64& m) {
    const double r = __ull2double_rn(mt_next(m)) / 18446744073709551616.0;
    return r >= 1.0 ? 0x1.fffffffffffffp-1 : r;
}

struct Normal {  // std::normal_distribution<double>(0, 1), libstdc++ polar method
    double saved;
    bool avail;
};

__device__ double gauss(Normal& n, Mt64& m) {
    double ret;
    if (n.avail) {
        n.avail = false;
        ret = n.saved;
    } else {
        double x, y, r2;
        do {
            x = 2.0 * canonical(m) - 1.0;
            y = 2.0 * canonical(m) - 1.0;
            r2 = x * x + y * y;
        } while (r2 > 1.0 || r2 == 0.0);
        const double mult = sqrt(-2.0 * log(r2) / r2);
        n.saved = x * mult;
        n.avail = true;
        ret = y * mult;
    }
    return ret * 1.0 + 0.0;  // * stddev + mean
}

__global__ void __launch_bounds__(128)
    k_simulate(const SimEntry* ents, const int* gpus, const int* stage_off, int n_stages, int G,
               SimCfg cfg, const unsigned long long* seeds, int n_seeds, double* iter_out,
               double* stage_out, double* busy_out, double* mean_out, SimInterval* tl) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_seeds) return;
    Mt64 rng;
    mt_seed(rng, seeds[t]);
    Normal nd{0.0, false};
    double* busy = busy_out + (size_t)t * G;
    double* pst = stage_out + (size_t)t * n_stages;
#pragma unroll 1
    for (int r = 0; r < G; ++r) busy[r] = 0.0;
#pragma unroll 1
    for (int s = 0; s < n_stages; ++s) pst[s] = 0.0;
    double total = 0.0;
    int ntl = 0;
#pragma unroll 1
    for (int it = 0; it < cfg.iterations; ++it) {
        double tt = 0.0;
#pragma unroll 1
        for (int s = 0; s < n_stages; ++s) {
            double stage_dur = 0.0;
            int streams = 0;
#pragma unroll 1
            for (int e = stage_off[s]; e < stage_off[s + 1]; ++e) {
                const SimEntry E = ents[e];
                double dur = E.dur0;
                if (cfg.sigma > 0) dur *= exp(cfg.sigma * gauss(nd, rng));
                stage_dur = stage_dur < dur ? dur : stage_dur;         // std::max
                const double active = E.active_cap < dur ? E.active_cap : dur;  // std::min
                streams += E.n_gpus;
#pragma unroll 1
                for (int g = 0; g < E.n_gpus; ++g) {
                    const int r = gpus[E.gpu_off + g];
                    busy[r] += E.quota * active;
                    if (it == 0 && t == 0 && tl)
                        tl[ntl++] = SimInterval{r, E.module, tt, tt + dur, E.quota};
                }
            }
            const double overhead =
                cfg.on_demand ? cfg.on_demand_overhead * streams : cfg.pooled_overhead;
            pst[s] += stage_dur + overhead;
            tt += stage_dur + overhead;
        }
        total += tt;
    }
    iter_out[t] = total / cfg.iterations;
#pragma unroll 1
    for (int s = 0; s < n_stages; ++s) pst[s] /= cfg.iterations;
    double mean = 0.0;
#pragma unroll 1
    for (int r = 0; r < G; ++r) {
        busy[r] = total > 0 ? busy[r] / total : 0.0;
        mean += busy[r];
    }
    mean_out[t] = mean / G;
}

void simulate_device(const std::vector<SimEntry>& ents, const std::vector<int>& gpus,
                     const std::vector<int>& stage_off, int G, const SimCfg& cfg,
                     const std::vector<uint64_t>& seeds, int device, std::vector<double>& iter,
                     std::vector<double>& per_stage, std::vector<double>& busy,
                     std::vector<double>& mean_busy, std::vector<SimInterval>* timeline) {
    if (cfg.iterations < 1) throw std::invalid_argument("iterations must be >= 1");
    if (cfg.pooled_overhead < 0 || cfg.on_demand_overhead < 0)
        throw std::invalid_argument("overheads must be >= 0");
    CKS(cudaSetDevice(device));
    const int S = (int)stage_off.size() - 1, N = (int)seeds.size();
    iter.assign(N, 0.0);
    per_stage.assign((size_t)N * S, 0.0);
    busy.assign((size_t)N * G, 0.0);
    mean_busy.assign(N, 0.0);
    if (N == 0) return;
    const size_t ntl = gpus.size();
    SimEntry* de;
    int *dg, *doff;
    unsigned long long* dsd;
    double *di, *dst, *db, *dm;
    SimInterval* dtl = nullptr;
    CKS(cudaMalloc(&de, sizeof(SimEntry) * (ents.size() + 1)));
    CKS(cudaMalloc(&dg, sizeof(int) * (gpus.size() + 1)));
    CKS(cudaMalloc(&doff, sizeof(int) * stage_off.size()));
    CKS(cudaMalloc(&dsd, sizeof(unsigned long long) * N));
    CKS(cudaMalloc(&di, sizeof(double) * N));
    CKS(cudaMalloc(&dst, sizeof(double) * ((size_t)N * S + 1)));
    CKS(cudaMalloc(&db, sizeof(double) * ((size_t)N * G)));
    CKS(cudaMalloc(&dm, sizeof(double) * N));
    if (timeline) CKS(cudaMalloc(&dtl, sizeof(SimInterval) * (ntl + 1)));
    CKS(cudaMemcpy(de, ents.data(), sizeof(SimEntry) * ents.size(), cudaMemcpyHostToDevice));
    CKS(cudaMemcpy(dg, gpus.data(), sizeof(int) * gpus.size(), cudaMemcpyHostToDevice));
    CKS(cudaMemcpy(doff, stage_off.data(), sizeof(int) * stage_off.size(),
                   cudaMemcpyHostToDevice));
    CKS(cudaMemcpy(dsd, seeds.data(), sizeof(unsigned long long) * N, cudaMemcpyHostToDevice));
    k_simulate<<<(N + 127) / 128, 128>>>(de, dg, doff, S, G, cfg, dsd, N, di, dst, db, dm, dtl);
    CKS(cudaGetLastError());
    CKS(cudaMemcpy(iter.data(), di, sizeof(double) * N, cudaMemcpyDeviceToHost));
    CKS(cudaMemcpy(per_stage.data(), dst, sizeof(double) * (size_t)N * S, cudaMemcpyDeviceToHost));
    CKS(cudaMemcpy(busy.data(), db, sizeof(double) * (size_t)N * G, cudaMemcpyDeviceToHost));
    CKS(cudaMemcpy(mean_busy.data(), dm, sizeof(double) * N, cudaMemcpyDeviceToHost));
    if (timeline) {
        timeline->resize(ntl);
        CKS(cudaMemcpy(timeline->data(), dtl, sizeof(SimInterval) * ntl, cudaMemcpyDeviceToHost));
        cudaFree(dtl);
    }
    cudaFree(de);
    cudaFree(dg);
    cudaFree(doff);
    cudaFree(dsd);
    cudaFree(di);
    cudaFree(dst);
    cudaFree(db);
    cudaFree(dm);
}

}  // namespace mg
