// DMMA (mma.sync m8n8k4 f64) throughput vs independent accumulator chains per warp (C) and
// warps per SM (W): tells how much ILP x TLP the Legendre kernels need to saturate the pipe.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void probe(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    double d[C][2];
    for (int c = 0; c < C; ++c) d[c][0] = d[c][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int c = 0; c < C; ++c) s += d[c][0] + d[c][1];
    if (s == 1.2345) out[0] = s;
}
template <int C>
void run(int warps_per_sm, int sms) {
    double* o; cudaMalloc(&o, 8);
    int iters = 4096 / C * 4;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int bw = warps_per_sm >= 4 ? 4 : warps_per_sm;  // warps per block
    const int blocks = sms * (warps_per_sm / bw);
    probe<C><<<blocks, 32 * bw>>>(o, iters);
    cudaEventRecord(e0);
    probe<C><<<blocks, 32 * bw>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 512.0 * C * iters * blocks * bw;
    printf("chains %2d warps/SM %2d : %6.1f TFLOP/s   (%.1f cyc/DMMA/SMSP @1.965GHz)\n", C, warps_per_sm,
           fl / (ms * 1e-3) / 1e12, (ms * 1e-3 * 1.965e9) / (C * (double)iters * (warps_per_sm / 4.0)));
    cudaFree(o);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {4, 8, 16, 32}) { run<1>(w, sms); run<2>(w, sms); run<4>(w, sms); run<8>(w, sms); run<16>(w, sms); }
    return 0;
}
