// Shared device helpers of the Legendre kernels (sm_100a, fp64).
#pragma once

#include "pswe_internal.h"

namespace pswe {
namespace legc {

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
