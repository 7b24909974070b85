// FP64 peak microbenchmarks (MEASURED_PEAKS.json carries no FP64 figure): DFMA (CUDA cores)
// and DMMA (mma.sync.aligned.m8n8k4 f64 tensor-core tiles, the only FP64 MMA on sm_100a —
// tcgen05 has no f64 kind). Used as the roofline denominator of the Legendre kernels and to
// decide DFMA vs DMMA (north star: "DMMA only if it measurably beats FP64 FMA").
#include "pswe_internal.h"

namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters, double a, double b) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;  // keep the work alive
}

__global__ void __launch_bounds__(128) dmma_peak_kernel(double* out, int iters) {
    // each warp issues independent m8n8k4 tiles: A 8x4 (1 reg), B 4x8 (1 reg), C/D 8x8 (2 regs)
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    double d[kChains][2];
#pragma unroll
    for (int c = 0; c < kChains; ++c) d[c][0] = d[c][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(d[c][0]), "+d"(d[c][1])
                         : "d"(a), "d"(b));
        }
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += d[c][0] + d[c][1];
    if (s == 12345.678) out[0] = s;
}

}  // namespace

extern "C" {

// Returns achieved TFLOP/s (DFMA if use_dmma == 0, DMMA otherwise); negative on error.
double pswe_fp64_peak(int use_dmma, int iters) {
    double tf = -1.0;
    pswe::guarded([&] {
        int dev = 0, sms = 0;
        PSWE_CUDA(cudaGetDevice(&dev));
        PSWE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        double* d_out;
        PSWE_CUDA(cudaMalloc(&d_out, sizeof(double)));
        cudaEvent_t e0, e1;
        PSWE_CUDA(cudaEventCreate(&e0));
        PSWE_CUDA(cudaEventCreate(&e1));
        const int blocks = sms * 8;
        double flops;
        for (int rep = 0; rep < 2; ++rep) {  // warm-up + timed
            PSWE_CUDA(cudaEventRecord(e0));
            if (!use_dmma) {
                dfma_peak_kernel<<<blocks, 256>>>(d_out, iters, 0.999999, 1e-7);
                flops = 2.0 * kChains * (double)iters * blocks * 256;
            } else {
                dmma_peak_kernel<<<blocks, 128>>>(d_out, iters);
                flops = 2.0 * 8 * 8 * 4 * kChains * (double)iters * blocks * (128 / 32);
            }
            PSWE_CUDA(cudaEventRecord(e1));
            PSWE_CUDA(cudaEventSynchronize(e1));
        }
        float ms = 0.f;
        PSWE_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        tf = flops / (ms * 1e-3) / 1e12;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(d_out);
    });
    return tf;
}

}  // extern "C"
