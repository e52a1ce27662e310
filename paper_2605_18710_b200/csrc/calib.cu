// calib.cu — the on-chip roofline denominator of SURVEY.md §8(d): measured shared-memory
// load bandwidth of this B200 (MEASURED_PEAKS.json carries only HBM and bf16 peaks).
// Every warp streams conflict-free 16-B shared loads (512 B per warp instruction, one
// 128-B wavefront per bank cycle); the grid keeps every SM's shared pipe busy.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>

namespace mg {

constexpr int CB_THREADS = 512;
constexpr int CB_WORDS = 2048;  // int4 = 32 KB per CTA

__global__ void __launch_bounds__(CB_THREADS) k_smem_peak(unsigned* sink, int iters) {
    __shared__ int4 buf[CB_WORDS];
    for (int i = threadIdx.x; i < CB_WORDS; i += CB_THREADS) buf[i] = make_int4(i, 3 * i, 5 * i, 7 * i);
    __syncthreads();
    unsigned a = 0, b = 0, c = 0, d = 0;
    int idx = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
        #pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int4 v = buf[(idx + u * (CB_WORDS / 8)) & (CB_WORDS - 1)];  // 8 distinct rows
            a ^= (unsigned)v.x;
            b += (unsigned)v.y;
            c ^= (unsigned)v.z;
            d += (unsigned)v.w;
        }
        idx += 32;
    }
    if ((a ^ b ^ c ^ d) == 0x9e3779b9u) sink[threadIdx.x] = a + b + c + d;
}

// GB/s of shared-memory loads over the whole device (best of `reps` timed launches).
double smem_peak_gbs(int device, int reps) {
    auto ck = [](cudaError_t e, const char* w) {
        if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e) + " at " + w);
    };
    ck(cudaSetDevice(device), "cudaSetDevice");
    int sms = 0, per_sm = 0;
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attr");
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_smem_peak, CB_THREADS, 0), "occupancy");
    const int grid = sms * (per_sm > 0 ? per_sm : 1);
    const int iters = 4096;
    unsigned* sink = nullptr;
    ck(cudaMalloc(&sink, CB_THREADS * sizeof(unsigned)), "cudaMalloc");
    cudaEvent_t e0, e1;
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    double best = 0.0;
    for (int r = 0; r < reps + 1; ++r) {
        ck(cudaEventRecord(e0), "record");
        k_smem_peak<<<grid, CB_THREADS>>>(sink, iters);
        ck(cudaEventRecord(e1), "record");
        ck(cudaEventSynchronize(e1), "sync");
        float ms = 0;
        ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
        const double bytes = (double)grid * CB_THREADS * iters * 8 * 16;
        if (r > 0 && ms > 0) best = std::max(best, bytes / (ms * 1e-3) / 1e9);  // r = 0: warm-up
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    return best;
}

}  // namespace mg
