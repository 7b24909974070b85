// Microbenchmark (tuning only): the forward Legendre's inner k-step pattern on shared-memory
// operands, no bulk copies, no mbarriers - what DMMA rate can W warps per block x B blocks per SM
// reach when every k-step loads NG G values (+ NG/2 additions) and 2 SPW P values per warp and
// issues 2 SPW DMMAs?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/p tools/dmma_smem_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <int SPW, int PREF>
__global__ void probe(int iters, double* out) {
    extern __shared__ double sm[];  // 16 KB of operands per block
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = 1.0 + 1e-3 * i;
    __syncthreads();
    double acc[SPW][2][2] = {};
    const int r4 = lane >> 2, c4 = lane & 3;
    for (int it = 0; it < iters; ++it) {
        const int base = (it * 37 + warp * 64) & 1023;
        double be[SPW], bo[SPW];
#pragma unroll
        for (int u = 0; u < SPW; ++u) {
            if (PREF == 0) {  // conflict-free: 32 consecutive doubles per warp load
                be[u] = sm[(base + u * 64 + lane) & 2047];
                bo[u] = sm[(base + u * 64 + 32 + lane) & 2047];
            } else {  // register operands (no loads): the pipe's ceiling for this loop
                be[u] = 1.0 + u * 1e-3 + it * 1e-9;
                bo[u] = 2.0 + u * 1e-3;
            }
        }
        const double gn = PREF ? 0.5 + it * 1e-9 : sm[(base + 1024 + lane) & 2047];
        const double gs = PREF ? 0.25 : sm[(base + 1536 + lane) & 2047];
        const double ae = gn + gs, ao = gn - gs;
#pragma unroll
        for (int u = 0; u < SPW; ++u) {
            dmma(acc[u][0], ae, be[u]);
            dmma(acc[u][1], ao, bo[u]);
        }
    }
    double s = 0;
#pragma unroll
    for (int u = 0; u < SPW; ++u) s += acc[u][0][0] + acc[u][1][1];
    if (s == 12345.0) out[threadIdx.x] = s;
}

template <int SPW, int PREF>
void run(int warps, int blocks_per_sm) {
    int dev = 0, nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    cudaMalloc(&out, 4096 * 8);
    const int iters = 4096;
    const size_t smem = 16384;
    cudaFuncSetAttribute(probe<SPW, PREF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<SPW, PREF><<<nsm * blocks_per_sm, 32 * warps, smem>>>(64, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    probe<SPW, PREF><<<nsm * blocks_per_sm, 32 * warps, smem>>>(iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double dmmas = (double)nsm * blocks_per_sm * warps * iters * 2 * SPW;
    const double tf = dmmas * 512 / (ms * 1e-3) / 1e12;
    printf("%s SPW %d warps/block %2d blocks/SM %d : %6.1f TFLOP/s (%.0f%% of 36.9)\n", PREF ? "reg " : "smem", SPW, warps, blocks_per_sm, tf,
           100 * tf / 36.9);
    cudaFree(out);
}

int main() {
    for (int bps : {1, 2}) {
        run<8, 0>(7, bps);
        run<4, 0>(14, bps);
        run<2, 0>(8, bps);
        run<8, 1>(7, bps);
        run<4, 1>(14, bps);
    }
    return 0;
}
