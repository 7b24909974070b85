// Shared device helpers of the Legendre kernels (sm_100a, fp64).
#pragma once

#include "pswe_internal.h"

namespace pswe {
namespace legc {

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}

// -a^2/(s(s+1)) x_s (inverse Laplacian at degree s of order m; 0 outside m..R and at s = 0);
// with rtab (rtab[s] = 1/(s(s+1)), host-rounded) the division becomes one multiply
__device__ __forceinline__ double2 inv_lap_at(const double2* __restrict__ x, long bs, int m, int R, int t, double a2,
                                              const double* __restrict__ rtab = nullptr) {
    if (t < m || t > R || t == 0) return make_double2(0.0, 0.0);
    const double f = rtab ? -a2 * __ldg(rtab + t) : -a2 / (t * (t + 1.0));
    const double2 v = x[bs + t - m];
    return make_double2(v.x * f, v.y * f);
}

// H-sum coefficient at degree t rewritten as a P-sum over one extra degree:
// c_t = -(t-1) eps_t psi_{t-1} + (t+2) eps_{t+1} psi_{t+1}, psi = inverse Laplacian of x
__device__ __forceinline__ double2 hcoef(const double2* __restrict__ x, const double* __restrict__ eps, long bs,
                                         long bx, int m, int R, int t, double a2,
                                         const double* __restrict__ rtab = nullptr) {
    double2 c = make_double2(0.0, 0.0);
    if (t - 1 >= m) {
        const double2 pm = inv_lap_at(x, bs, m, R, t - 1, a2, rtab);
        const double f = -(double)(t - 1) * eps[bx + t - m];
        c.x += f * pm.x;
        c.y += f * pm.y;
    }
    if (t + 1 <= R) {
        const double2 pp = inv_lap_at(x, bs, m, R, t + 1, a2, rtab);
        const double f = (double)(t + 2) * eps[bx + t + 1 - m];
        c.x += f * pp.x;
        c.y += f * pp.y;
    }
    return c;
}

// 16-byte cp.async global -> shared with zero fill when !valid (src-size 0)
__device__ __forceinline__ void cp_async16z(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc), "r"(sz));
}

// Stage G_E = G_N + G_S and G_O = G_N - G_S of 4 NT complex columns (q0..) of Fourier rows
// four[q][m][i] for all Jp latitude pairs into shared memory: element (j, real col c) of the
// even plane at G[pos(j, c)], of the odd plane at G[odd + pos(j, c)]. Loads are issued in
// batches of B per thread before any store, so B loads per thread are in flight (the serial
// load -> store form leaves the SM idle for a full memory latency per element).
template <int NT, int B, class Pos>
__device__ __forceinline__ void stage_g(double* G, int odd, int Jp, int J, int nlat, int R, int m, int q0, int nq,
                                        const double2* __restrict__ four, Pos pos) {
    const int total = Jp * 4 * NT;
    for (int base = threadIdx.x; base < total; base += B * blockDim.x) {
        double2 gn[B], gs[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int idx = base + u * blockDim.x;
            gn[u] = gs[u] = make_double2(0.0, 0.0);
            if (idx < total) {
                const int ql = idx / Jp, jj = idx - ql * Jp;  // latitude fastest: coalesced rows
                const int q = q0 + ql;
                if (jj < J && q < nq) {
                    const double2* src = four + ((long)q * (R + 1) + m) * nlat;
                    const int iN = nlat - J + jj, iS = J - 1 - jj;
                    gn[u] = src[iN];
                    if (iN != iS) gs[u] = src[iS];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int idx = base + u * blockDim.x;
            if (idx < total) {
                const int ql = idx / Jp, jj = idx - ql * Jp;
                const int pe = pos(jj, 2 * ql), pi = pos(jj, 2 * ql + 1);
                G[pe] = gn[u].x + gs[u].x;
                G[pi] = gn[u].y + gs[u].y;
                G[odd + pe] = gn[u].x - gs[u].x;
                G[odd + pi] = gn[u].y - gs[u].y;
            }
        }
    }
}

}  // namespace legc
}  // namespace pswe
