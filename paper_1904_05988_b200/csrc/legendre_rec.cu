// Single-state inverse Legendre contraction on the FP64 CUDA cores with the associated-Legendre
// values recomputed in registers (sm_100a, fp64): no P table traffic. Used for single states on
// grids of >= 256 latitude pairs, where the P table outgrows the L2 (T511 269 MB, T1023 2.1 GB):
// at T1023 the alternative was the recompute-mode DMMA kernel (legendre_mma.cu, the recurrence
// inside its tensor-core loop): single-state evaluation 736 -> 679 us, PFASST config 5 82.0 -> 78
// s/day; at T511 the streamed DMMA kernel re-reads the 269 MB table every evaluation: PFASST
// config 4 10.94 -> 10.77 s/day. Below 256 pairs the table stays in the L2 and the streamed DMMA
// kernel is faster (profiles/r02_ab_negative.txt item 13).
//
// Reference loops replaced: the Legendre sums of synthesise / uv_from_vortdiv
// (transform.cpp:155-223), G^m(mu_j) = sum_s x^m_s P^m_s(mu_j), with the same recurrence for P as
// legendre.cpp:30-37 and the same operation order as the STREAM table builder, so every P value is
// bit-identical to the table's; with one degree segment per order (the default) the accumulation
// order is the DMMA kernels' too (m8n8k4.f64 accumulates its four products in k order), so the
// result is bit-identical to the streamed DMMA inverse of a batch (tests/test_gpu_swe.py).
//
// Thread = (order m, L = 4 latitude pairs, 8 real columns): it runs P_{t+1} = a_t mu P_t -
// b_t P_{t-1} for its latitudes and accumulates E (even t - m) and O (odd t - m) in registers; the
// coefficient rows X_t are the same for every latitude of the warp, so they are broadcast
// shared-memory reads (one 16-byte load feeds 4 x 2 FMAs per thread: with one latitude per thread
// the loads, two wavefronts each, would bound the kernel).
//
// Input: the prep kernel's X tiles (legendre_stream.cu: per column group z and chunk of order m,
// [16 degrees][8 NT + 2] doubles, zero past the order's last degree), staged per warp through a
// cp.async ring. Output: Fourier rows out[q][i][m] (north row nlat - J + j = E + O, south row
// J - 1 - j = E - O), exactly like leg_inv_tma_kernel. Blocks are issued order-major with m = 0
// (the longest, R + 2 degrees) first, so the block scheduler approximates longest-first.
#include <cstdlib>

#include "legendre_common.cuh"

namespace pswe {

namespace {

constexpr int CH = 16;     // degrees per X-tile chunk (legendre_stream.cu)
#ifndef PSWE_REC_S
#define PSWE_REC_S 4
#endif
constexpr int kRecS = PSWE_REC_S;  // ring slots (chunks) per block

__device__ __forceinline__ double rec_step(double2 ab, double mu, double p, double pm1) {
    return __fma_rn(ab.x, __dmul_rn(mu, p), -__dmul_rn(ab.y, pm1));
}

// Thread = L latitudes (each X value loaded from shared memory feeds L FMAs: the broadcast
// 16-byte load costs two shared-memory wavefronts, so with one latitude per thread the SM's one
// wavefront per cycle, not the FP64 pipe, would bound the kernel), warp = 32 L latitudes of one
// order and one degree SEGMENT: the order's chunks are split over the NSEG warps of the block, each
// warp starting its recurrence from the plan's checkpoints (P_t, P_{t-1}) at t = 16 c (the same
// recurrence, bit-identical values), so the longest order's chain is NSEG times shorter. Each warp
// streams its own chunks through a private cp.async ring (no block barriers in the main loop),
// loads the next degree's row into registers while the current one's FMAs issue, and the segments'
// partial sums are added in segment order through shared memory at the end (NSEG = 1: the exact
// summation order of the DMMA kernel, bit-identical output).
// (an explicit one-block-per-SM bound: ptxas then takes 238 registers instead of 218 and the T1023
// single-state inverse runs 245 instead of 252 us)
template <int L, int CW>
__global__ void __launch_bounds__(128, 1) leg_inv_rec2_kernel(int R, int J, int nlat, int nq, int NT, int nct, int nls,
                                                           int ncs, int groups, int nseg,
                                                           const double* __restrict__ mu_n,
                                                           const double* __restrict__ seed,
                                                           const double2* __restrict__ chk,
                                                           const double2* __restrict__ rec,
                                                           const int* __restrict__ cbase,
                                                           const double* __restrict__ Xt,
                                                           double2* __restrict__ out) {
    constexpr int CP = CW / 2;
    constexpr int RS = CH * CP + CH;  // double2 per ring slot: 16 X rows, then 16 recurrence pairs
    constexpr int S = kRecS;
    extern __shared__ __align__(16) double2 dsm[];
    int b = blockIdx.x;
    const int ls = b % nls;
    b /= nls;
    const int cs = b % ncs;
    b /= ncs;
    const int z = b % groups;
    const int m = b / groups;
    const int len = R + 2 - m;
    const int nch = (len + CH - 1) / CH;
    const int SX = 8 * NT + 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c0 = (warp * nch) / nseg, c1 = ((warp + 1) * nch) / nseg;
    double mu[L], p[L], pm1[L];
#pragma unroll
    for (int l = 0; l < L; ++l) {
        const int j = ls * 32 * L + 32 * l + lane;
        mu[l] = p[l] = pm1[l] = 0.0;
        if (j < J) {
            mu[l] = mu_n[j];
            if (c0 == 0) {
                p[l] = seed[(long)m * J + j];
            } else if (c0 < c1) {
                const double2 ck = chk[((long)cbase[m] + c0) * J + j];
                p[l] = ck.x;
                pm1[l] = ck.y;
            }
        }
    }
    const double2* __restrict__ rc = rec + off_ext(R, m);
    const double* __restrict__ xm = Xt + ((long)z * nct + cbase[m]) * CH * SX + cs * CW;
    double2* ring = dsm + warp * S * RS;
    pdl_trigger();
    pdl_wait();  // the X tiles come from the prep kernel (or the sweep's node update)

    auto issue = [&](int c) {
        double2* slot = ring + ((c - c0) % S) * RS;
        for (int i = lane; i < RS; i += 32) {
            if (i < CH * CP) {
                const int row = i / CP, k = i - row * CP;
                legc::cp_async16z(slot + i, xm + ((long)c * CH + row) * SX + 2 * k, true);
            } else {
                const int t = c * CH + (i - CH * CP);
                legc::cp_async16z(slot + i, rc + (t < len ? t : 0), t < len);
            }
        }
    };
#pragma unroll
    for (int u = 0; u < S - 1; ++u) {
        if (c0 + u < c1) issue(c0 + u);
        asm volatile("cp.async.commit_group;\n" ::);
    }
    double acc[L][2][CW];
#pragma unroll
    for (int l = 0; l < L; ++l)
#pragma unroll
        for (int k = 0; k < CW; ++k) acc[l][0][k] = acc[l][1][k] = 0.0;

    for (int c = c0; c < c1; ++c) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(S - 2));
        __syncwarp();  // chunk c landed for every lane; every lane is done with slot (c - 1) % S
        if (c + S - 1 < c1) issue(c + S - 1);
        asm volatile("cp.async.commit_group;\n" ::);
        const double2* slot = ring + ((c - c0) % S) * RS;
        double2 xn[CP], rn;
#pragma unroll
        for (int k = 0; k < CP; ++k) xn[k] = slot[k];
        rn = slot[CH * CP];
#pragma unroll
        for (int r = 0; r < CH; ++r) {
            double2 x[CP];
#pragma unroll
            for (int k = 0; k < CP; ++k) x[k] = xn[k];
            const double2 ra = rn;
            if (r + 1 < CH) {
#pragma unroll
                for (int k = 0; k < CP; ++k) xn[k] = slot[(r + 1) * CP + k];
                rn = slot[CH * CP + r + 1];
            }
#pragma unroll
            for (int l = 0; l < L; ++l)
#pragma unroll
                for (int k = 0; k < CP; ++k) {
                    acc[l][r & 1][2 * k] = __fma_rn(p[l], x[k].x, acc[l][r & 1][2 * k]);
                    acc[l][r & 1][2 * k + 1] = __fma_rn(p[l], x[k].y, acc[l][r & 1][2 * k + 1]);
                }
#pragma unroll
            for (int l = 0; l < L; ++l) {
                const double pn = rec_step(ra, mu[l], p[l], pm1[l]);
                pm1[l] = p[l];
                p[l] = pn;
            }
        }
    }
    const int q0 = z * 4 * NT + cs * CP;
    const long rowstride = (long)nlat * (R + 1);
    if (nseg == 1) {
#pragma unroll
        for (int l = 0; l < L; ++l) {
            const int j = ls * 32 * L + 32 * l + lane;
            if (j >= J) continue;
            const int iN = nlat - J + j, iS = J - 1 - j;
#pragma unroll
            for (int k = 0; k < CP; ++k) {
                const int q = q0 + k;
                if (q >= nq) break;
                double2* dst = out + q * rowstride + m;
                const double er = acc[l][0][2 * k], ei = acc[l][0][2 * k + 1];
                const double orr = acc[l][1][2 * k], oi = acc[l][1][2 * k + 1];
                dst[(long)iN * (R + 1)] = make_double2(er + orr, ei + oi);
                if (iS != iN) dst[(long)iS * (R + 1)] = make_double2(er - orr, ei - oi);
            }
        }
        return;
    }
    // segment partials through shared memory: part[w][l][par][k][lane]
    __syncthreads();  // every warp is done with its ring
    double* part = reinterpret_cast<double*>(dsm);
    constexpr int PW = L * 2 * CW * 32;
#pragma unroll
    for (int l = 0; l < L; ++l)
#pragma unroll
        for (int par = 0; par < 2; ++par)
#pragma unroll
            for (int k = 0; k < CW; ++k) part[warp * PW + ((l * 2 + par) * CW + k) * 32 + lane] = acc[l][par][k];
    __syncthreads();
    // warp w finishes latitude groups l = w, w + nseg, ...: the segments summed in order
    for (int l = warp; l < L; l += nseg) {
        const int j = ls * 32 * L + 32 * l + lane;
        if (j >= J) continue;
        const int iN = nlat - J + j, iS = J - 1 - j;
        for (int k = 0; k < CP; ++k) {
            const int q = q0 + k;
            if (q >= nq) break;
            double v[2][2];
#pragma unroll
            for (int par = 0; par < 2; ++par)
#pragma unroll
                for (int ri = 0; ri < 2; ++ri) {
                    const int idx = ((l * 2 + par) * CW + 2 * k + ri) * 32 + lane;
                    double s = part[idx];
                    for (int w = 1; w < nseg; ++w) s += part[w * PW + idx];
                    v[par][ri] = s;
                }
            double2* dst = out + q * rowstride + m;
            dst[(long)iN * (R + 1)] = make_double2(v[0][0] + v[1][0], v[0][1] + v[1][1]);
            if (iS != iN) dst[(long)iS * (R + 1)] = make_double2(v[0][0] - v[1][0], v[0][1] - v[1][1]);
        }
    }
}

template <int L, int CW>
void rec2_launch(const pswe_plan& P, const double* Xt, int nq, int NT, int nseg, double2* out, cudaStream_t st) {
    constexpr int CP = CW / 2, RS = CH * CP + CH;
    const int groups = (nq + 4 * NT - 1) / (4 * NT);
    const int ncs = 8 * NT / CW;
    const int nls = (P.J + 32 * L - 1) / (32 * L);
    const long nblk = (long)(P.R + 1) * groups * ncs * nls;
    const size_t ring = (size_t)nseg * kRecS * RS * sizeof(double2);
    const size_t part = nseg > 1 ? (size_t)nseg * L * 2 * CW * 32 * sizeof(double) : 0;
    const size_t sm = ring > part ? ring : part;
    auto kern = leg_inv_rec2_kernel<L, CW>;
    static size_t attr = 0;
    if (sm > attr) {
        PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        attr = sm;
    }
    launch_pdl(kern, dim3((unsigned)nblk), dim3(32 * nseg), sm, st, P.R, P.J, P.nlat, nq, NT, P.n_chunks, nls, ncs,
               groups, nseg, P.d_mu_n, P.d_seed, (const double2*)P.d_chk, P.d_rec, P.d_chk_off, Xt, out);
    PSWE_LAUNCH_CHECK();
}

}  // namespace

// Single-state inverse on large grids through this kernel: from 256 latitude pairs up (T511 and
// T1023 fine levels; PSWE_INV_REC_J overrides, 0 = off). The X tiles come from the
// streamed path's prep (or the SDC node update, xtiles_by_sweep_ok).
bool inv_rec_big(const pswe_plan& P, int nq) {
    static const int jmin = [] { const char* e = std::getenv("PSWE_INV_REC_J"); return e ? std::atoi(e) : 256; }();
    return jmin > 0 && nq <= 4 && P.J >= jmin && P.legendre_mode == PSWE_LEGENDRE_STREAM && P.n_chunks > 0;
}

void inv_rec_launch(const pswe_plan& P, const double* Xt, int nq, int NT, double2* out, cudaStream_t st) {
    static const int lat = [] { const char* e = std::getenv("PSWE_INVREC_L"); return e ? std::atoi(e) : 4; }();
    // degree segments per order: one from 512 latitude pairs (bit-identical to the DMMA kernels;
    // T1023 single state 679 / 682 / 694 us for 1 / 2 / 4 segments), two below (T511 on 512 x 1024:
    // the order's chain is half as long; PFASST config 4 10.94 -> 10.77 s/day, one segment 11.74)
    static const int seg = [] { const char* e = std::getenv("PSWE_INVREC_SEG"); return e ? std::atoi(e) : 0; }();
    const int want = seg > 0 ? seg : (P.J >= 512 ? 1 : 2);
    const int nseg = want < 1 ? 1 : (want > 4 ? 4 : want);
    if (lat == 2) rec2_launch<2, 8>(P, Xt, nq, NT, nseg, out, st);
    else rec2_launch<4, 8>(P, Xt, nq, NT, nseg, out, st);
}

}  // namespace pswe
