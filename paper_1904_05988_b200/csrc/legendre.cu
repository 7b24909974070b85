// Legendre contractions of the spherical-harmonic transform (sm_100a, fp64).
//
// Reference loops replaced (transform.cpp):
//   synthesise        :155-174  G^m_i = sum_s x^m_s P^m_s(mu_i)
//   uv_from_vortdiv   :176-223  U_m, V_m from psi/chi with P and H = (1-mu^2) dP/dmu
//   analyse           :136-153  x^m_s = sum_i w_i G^m_i P^m_s(mu_i)
//   vortdiv_from_uv   :225-270  (the P and H projections)
// Algorithmic changes (same mathematics):
//   * latitude folding: P^m_s(-mu) = (-1)^(s-m) P^m_s(mu) and the Gauss nodes are symmetric
//     (gauss.cpp:43-46), so each thread serves the latitude pair (mu_j, -mu_j);
//   * H-sums are rewritten as P-sums over s = m..R+1 of neighbour-combined coefficients
//     (H^m_s = -s eps^m_{s+1} P^m_{s+1} + (s+1) eps^m_s P^m_{s-1}, transform.cpp:69-73), so a
//     single P recurrence serves P and H terms and the reference's separate H table disappears;
//   * inverse direction: P^m_s(mu_j) is recomputed on the fly by the normalised recurrence
//     (legendre.cpp:30-37) from a seed table P^m_m(mu_j) — no table traffic at all;
//   * forward direction: either streams P from an HBM table laid out [m][j][s] (coalesced along
//     s; PSWE_LEGENDRE_STREAM) or recomputes P into shared-memory tiles (RECOMPUTE).
#include "pswe_internal.h"

namespace pswe {

namespace {

__device__ __forceinline__ void cfma(double2& acc, double2 a, double r) {
    acc.x = fma(a.x, r, acc.x);
    acc.y = fma(a.y, r, acc.y);
}

// psi_t = x_t * (-a^2/(t(t+1))), 0 at t = 0 and outside [m, R] (inv_laplacian, transform.cpp:282-290)
__device__ __forceinline__ double2 inv_lap_at(const double2* __restrict__ x, long bs, int m, int R, int t,
                                              double a2) {
    if (t < m || t > R || t == 0) return make_double2(0.0, 0.0);
    const double f = -a2 / (t * (t + 1.0));
    const double2 v = x[bs + t - m];
    return make_double2(v.x * f, v.y * f);
}

// H-part coefficient of P_t: c_t = -(t-1) eps_t psi_{t-1} + (t+2) eps_{t+1} psi_{t+1}
__device__ __forceinline__ double2 hcoef(const double2* __restrict__ x, const double* __restrict__ eps,
                                         long bs, long bx, int m, int R, int t, double a2) {
    double2 c = make_double2(0.0, 0.0);
    if (t - 1 >= m) {
        const double2 pm = inv_lap_at(x, bs, m, R, t - 1, a2);
        const double f = -(double)(t - 1) * eps[bx + t - m];
        c.x += f * pm.x;
        c.y += f * pm.y;
    }
    if (t + 1 <= R) {
        const double2 pp = inv_lap_at(x, bs, m, R, t + 1, a2);
        const double f = (double)(t + 2) * eps[bx + t + 1 - m];
        c.x += f * pp.x;
        c.y += f * pp.y;
    }
    return c;
}

// U_t = (i m chi_t - c^psi_t)/a ; V_t = (i m psi_t + c^chi_t)/a   (transform.cpp:204-206)
__device__ __forceinline__ void uv_coefs(const double2* __restrict__ vort, const double2* __restrict__ div,
                                         const double* __restrict__ eps, long bs, long bx, int m, int R,
                                         int t, double a2, double inv_a, double2& U, double2& V) {
    const double2 psi = inv_lap_at(vort, bs, m, R, t, a2);
    const double2 chi = inv_lap_at(div, bs, m, R, t, a2);
    const double2 cpsi = hcoef(vort, eps, bs, bx, m, R, t, a2);
    const double2 cchi = hcoef(div, eps, bs, bx, m, R, t, a2);
    U = make_double2(inv_a * (-m * chi.y - cpsi.x), inv_a * (m * chi.x - cpsi.y));
    V = make_double2(inv_a * (-m * psi.y + cchi.x), inv_a * (m * psi.x + cchi.y));
}

// ---- inverse: one thread per (m, latitude pair j); coefficients of this m staged in smem -----
// in: PLAIN  n fields [b][K];  UV  pairs [b][2][K] (vort, div);  EVAL states [b][3][K].
// out: Fourier rows [b][NF][m][i] (i = full latitude index, ascending mu).
template <int NF, int KIND>
__global__ void __launch_bounds__(64) leg_inv_kernel(int R, int J, int nlat, const double* __restrict__ mu_n,
                                                     const double* __restrict__ seed,
                                                     const double2* __restrict__ rec,
                                                     const double* __restrict__ eps,
                                                     const double2* __restrict__ in,
                                                     const double2* __restrict__ in2, double radius,
                                                     double2* __restrict__ out) {
    extern __shared__ double2 coef[];  // [NF][len]
    const int m = blockIdx.y;
    const int b = blockIdx.z;
    const int len = R + 2 - m;
    const long K = (long)(R + 1) * (R + 2) / 2;
    const long bs = off_std(R, m), bx = off_ext(R, m);
    const double a2 = radius * radius, inv_a = 1.0 / radius;

    if (KIND == INV_PLAIN) {
        const double2* x = in + (long)b * NF * K;
        for (int idx = threadIdx.x; idx < NF * len; idx += blockDim.x) {
            const int f = idx / len, t = idx - f * len;
            coef[idx] = (t < len - 1) ? x[(long)f * K + bs + t] : make_double2(0.0, 0.0);
        }
    } else if (KIND == INV_UV) {
        const double2* vort = in + (long)b * K;
        const double2* div = in2 + (long)b * K;
        for (int t = threadIdx.x; t < len; t += blockDim.x) {
            double2 U, V;
            uv_coefs(vort, div, eps, bs, bx, m, R, m + t, a2, inv_a, U, V);
            coef[t] = U;
            coef[len + t] = V;
        }
    } else {  // INV_EVAL: (Phi, zeta, U, V)
        const double2* phi = in + (long)b * 3 * K;
        const double2* vort = phi + K;
        const double2* div = phi + 2 * K;
        for (int t = threadIdx.x; t < len; t += blockDim.x) {
            const bool in_r = t < len - 1;
            coef[t] = in_r ? phi[bs + t] : make_double2(0.0, 0.0);
            coef[len + t] = in_r ? vort[bs + t] : make_double2(0.0, 0.0);
            double2 U, V;
            uv_coefs(vort, div, eps, bs, bx, m, R, m + t, a2, inv_a, U, V);
            coef[2 * len + t] = U;
            coef[3 * len + t] = V;
        }
    }
    __syncthreads();

    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= J) return;
    const double mu = mu_n[j];
    double p = seed[(long)m * J + j], pm1 = 0.0;
    const double2* __restrict__ rc = rec + bx;
    double2 aE[NF], aO[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) aE[f] = aO[f] = make_double2(0.0, 0.0);

    int t = 0;
    for (; t + 1 < len; t += 2) {
#pragma unroll
        for (int f = 0; f < NF; ++f) cfma(aE[f], coef[f * len + t], p);
        double2 ab = rc[t];
        double pn = ab.x * (mu * p) - ab.y * pm1;
        pm1 = p;
        p = pn;
#pragma unroll
        for (int f = 0; f < NF; ++f) cfma(aO[f], coef[f * len + t + 1], p);
        ab = rc[t + 1];
        pn = ab.x * (mu * p) - ab.y * pm1;
        pm1 = p;
        p = pn;
    }
    if (t < len) {
#pragma unroll
        for (int f = 0; f < NF; ++f) cfma(aE[f], coef[f * len + t], p);
    }
    const int iN = nlat - J + j, iS = J - 1 - j;  // iN == iS: equator (odd nlat)
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        double2* o = out + ((long)b * NF + f) * nlat * (R + 1) + m;  // rows [q][i][m]
        o[(long)iN * (R + 1)] = make_double2(aE[f].x + aO[f].x, aE[f].y + aO[f].y);
        o[(long)iS * (R + 1)] = make_double2(aE[f].x - aO[f].x, aE[f].y - aO[f].y);
    }
}

// ---- forward, table-streaming: one thread per (m, s); P^m_s(mu_j) read coalesced along s -----
// four: [b][nf][m][i]; the block stages gE = G_N + G_S and gO = G_N - G_S for its m.
template <int NF>
__global__ void __launch_bounds__(64) leg_fwd_stream_kernel(int R, int J, int nlat, int nf, int groups,
                                                            const double* __restrict__ ptab,
                                                            const double2* __restrict__ four,
                                                            double2* __restrict__ out, int ext) {
    extern __shared__ double2 g[];  // [NF][2][J]
    const int m = blockIdx.y;
    const int b = blockIdx.z / groups, f0 = (blockIdx.z % groups) * NF;
    const int len = R + 2 - m;
    for (int idx = threadIdx.x; idx < NF * J; idx += blockDim.x) {
        const int f = idx / J, j = idx - f * J;
        const double2* src = four + (((long)b * nf + f0 + f) * (R + 1) + m) * nlat;
        const int iN = nlat - J + j, iS = J - 1 - j;
        const double2 gn = src[iN], gs = (iN == iS) ? make_double2(0.0, 0.0) : src[iS];
        g[(2 * f) * J + j] = make_double2(gn.x + gs.x, gn.y + gs.y);
        g[(2 * f + 1) * J + j] = make_double2(gn.x - gs.x, gn.y - gs.y);
    }
    __syncthreads();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;  // s - m
    const int tmax = ext ? len : len - 1;
    if (t >= tmax) return;
    const int par = t & 1;
    const double* __restrict__ pt = ptab + off_ext(R, m) * J + t;
    double2 acc[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) acc[f] = make_double2(0.0, 0.0);
    int j = 0;
    for (; j + 4 <= J; j += 4) {
        double pv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) pv[u] = __ldg(pt + (long)(j + u) * len);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int f = 0; f < NF; ++f) cfma(acc[f], g[(2 * f + par) * J + j + u], pv[u]);
    }
    for (; j < J; ++j) {
        const double pv = __ldg(pt + (long)j * len);
#pragma unroll
        for (int f = 0; f < NF; ++f) cfma(acc[f], g[(2 * f + par) * J + j], pv);
    }
    if (ext) {
        const long Kx = (long)(R + 1) * (R + 4) / 2;
#pragma unroll
        for (int f = 0; f < NF; ++f) out[((long)b * nf + f0 + f) * Kx + off_ext(R, m) + t] = acc[f];
    } else {
        const long K = (long)(R + 1) * (R + 2) / 2;
#pragma unroll
        for (int f = 0; f < NF; ++f) out[((long)b * nf + f0 + f) * K + off_std(R, m) + t] = acc[f];
    }
}

// ---- forward, recompute: block per (m, field group); P tiles generated in shared memory ------
// Phase 1: threads walk the recurrence for their latitude pairs and write P[j][s] for an
//          s-chunk of SC degrees into smem.
// Phase 2: thread (s, jslice) accumulates sum_j P[j][s] g[f][j] over its slice for all NF
//          fields; partial sums over slices are reduced through smem at the end of the chunk.
template <int NF, int SC>
__global__ void __launch_bounds__(256) leg_fwd_rec_kernel(int R, int J, int nlat, int nf, int groups,
                                                          const double* __restrict__ mu_n,
                                                          const double* __restrict__ seed,
                                                          const double2* __restrict__ rec,
                                                          const double2* __restrict__ four,
                                                          double2* __restrict__ out, int ext) {
    extern __shared__ double2 smem[];
    constexpr int NT = 256;
    constexpr int JS = NT / SC;  // j slices
    double2* g = smem;                              // [NF][2][J]
    double* ptile = (double*)(g + 2 * NF * J);      // [SC][J+1] (padded: conflict-free both ways)
    double2* part = (double2*)(ptile + (long)(J + 1) * SC);  // [JS][SC][NF]

    const int m = blockIdx.x;
    const int b = blockIdx.y / groups, f0 = (blockIdx.y % groups) * NF;
    const int len = R + 2 - m;
    const int tmax = ext ? len : len - 1;
    const long bx = off_ext(R, m);
    for (int idx = threadIdx.x; idx < NF * J; idx += NT) {
        const int f = idx / J, j = idx - f * J;
        const double2* src = four + (((long)b * nf + f0 + f) * (R + 1) + m) * nlat;
        const int iN = nlat - J + j, iS = J - 1 - j;
        const double2 gn = src[iN], gs = (iN == iS) ? make_double2(0.0, 0.0) : src[iS];
        g[(2 * f) * J + j] = make_double2(gn.x + gs.x, gn.y + gs.y);
        g[(2 * f + 1) * J + j] = make_double2(gn.x - gs.x, gn.y - gs.y);
    }
    // recurrence state for up to 4 latitude pairs per thread (J <= 1024)
    constexpr int JPT = 4;
    double p[JPT], pm1[JPT], mu[JPT];
#pragma unroll
    for (int q = 0; q < JPT; ++q) {
        const int j = threadIdx.x + q * NT;
        mu[q] = j < J ? mu_n[j] : 0.0;
        p[q] = j < J ? seed[(long)m * J + j] : 0.0;
        pm1[q] = 0.0;
    }
    const int sl = threadIdx.x % SC;   // s within chunk
    const int js = threadIdx.x / SC;   // j slice
    const int jper = (J + JS - 1) / JS;
    const int j0 = js * jper, j1 = min(J, j0 + jper);
    for (int c0 = 0; c0 < tmax; c0 += SC) {
        __syncthreads();  // g ready / previous chunk consumed
        const int cn = min(SC, len - c0);
#pragma unroll
        for (int q = 0; q < JPT; ++q) {
            const int j = threadIdx.x + q * NT;
            if (j < J) {
                for (int u = 0; u < cn; ++u) {
                    ptile[(long)u * (J + 1) + j] = p[q];
                    const double2 ab = rec[bx + c0 + u];
                    const double pn = ab.x * (mu[q] * p[q]) - ab.y * pm1[q];
                    pm1[q] = p[q];
                    p[q] = pn;
                }
            }
        }
        __syncthreads();
        const int t = c0 + sl;
        const int par = t & 1;
        double2 acc[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) acc[f] = make_double2(0.0, 0.0);
        if (t < tmax) {
            for (int j = j0; j < j1; ++j) {
                const double pv = ptile[(long)sl * (J + 1) + j];
#pragma unroll
                for (int f = 0; f < NF; ++f) cfma(acc[f], g[(2 * f + par) * J + j], pv);
            }
        }
#pragma unroll
        for (int f = 0; f < NF; ++f) part[((long)js * SC + sl) * NF + f] = acc[f];
        __syncthreads();
        for (int idx = threadIdx.x; idx < SC * NF; idx += NT) {
            const int s2 = idx / NF, f = idx - s2 * NF;
            const int tt = c0 + s2;
            if (tt < tmax) {
                double2 sum = make_double2(0.0, 0.0);
                for (int q = 0; q < JS; ++q) {
                    const double2 v = part[((long)q * SC + s2) * NF + f];
                    sum.x += v.x;
                    sum.y += v.y;
                }
                if (ext) {
                    const long Kx = (long)(R + 1) * (R + 4) / 2;
                    out[((long)b * nf + f0 + f) * Kx + bx + tt] = sum;
                } else {
                    const long K = (long)(R + 1) * (R + 2) / 2;
                    out[((long)b * nf + f0 + f) * K + off_std(R, m) + tt] = sum;
                }
            }
        }
    }
}

}  // namespace

void legendre_inverse(const pswe_plan& P, int kind, const double2* in, const double2* in2, int n, double radius,
                      double2* out, cudaStream_t st) {
    if (n <= 0) return;
    if (!P.simt) {  // default: FP64 tensor cores (legendre_mma.cu)
        const int nq = n * (kind == INV_PLAIN ? 1 : kind == INV_UV ? 2 : 4);
        legendre_inverse_mma(P, kind, in, in2, nq, radius, out, st);
        return;
    }
    const int TJ = 64;
    const int len = P.R + 2;
    auto launch = [&](auto kern, int nf, int nz) {
        dim3 grid((P.J + TJ - 1) / TJ, P.R + 1, nz);
        const size_t sm = (size_t)nf * len * sizeof(double2);
        if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        kern<<<grid, TJ, sm, st>>>(P.R, P.J, P.nlat, P.d_mu_n, P.d_seed, P.d_rec, P.d_eps, in, in2, radius, out);
        PSWE_LAUNCH_CHECK();
    };
    switch (kind) {
        case INV_PLAIN:
            // group fields so one recurrence serves several fields
            if (n % 5 == 0) launch(leg_inv_kernel<5, INV_PLAIN>, 5, n / 5);
            else if (n % 3 == 0) launch(leg_inv_kernel<3, INV_PLAIN>, 3, n / 3);
            else if (n % 2 == 0) launch(leg_inv_kernel<2, INV_PLAIN>, 2, n / 2);
            else launch(leg_inv_kernel<1, INV_PLAIN>, 1, n);
            break;
        case INV_UV: launch(leg_inv_kernel<2, INV_UV>, 2, n); break;
        case INV_EVAL: launch(leg_inv_kernel<4, INV_EVAL>, 4, n); break;
        default: throw std::invalid_argument("legendre_inverse: bad kind");
    }
}

template <int NF>
static void fwd_stream(const pswe_plan& P, const double2* four, int nf, int n_batch, double2* out, bool ext,
                       cudaStream_t st) {
    const int TS = 64;
    const int groups = nf / NF;
    dim3 grid((P.R + 2 + TS - 1) / TS, P.R + 1, n_batch * groups);
    const size_t sm = (size_t)NF * 2 * P.J * sizeof(double2);
    auto kern = leg_fwd_stream_kernel<NF>;
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<grid, TS, sm, st>>>(P.R, P.J, P.nlat, nf, groups, P.d_ptab, four, out, ext ? 1 : 0);
    PSWE_LAUNCH_CHECK();
}

template <int NF, int SC>
static void fwd_rec(const pswe_plan& P, const double2* four, int nf, int n_batch, double2* out, bool ext,
                    cudaStream_t st) {
    const int groups = nf / NF;
    constexpr int JS = 256 / SC;
    dim3 grid(P.R + 1, n_batch * groups);
    const size_t sm = (size_t)NF * 2 * P.J * sizeof(double2) + (size_t)(P.J + 1) * SC * sizeof(double) +
                      (size_t)JS * SC * NF * sizeof(double2);
    auto kern = leg_fwd_rec_kernel<NF, SC>;
    if (sm > 227 * 1024) throw std::runtime_error("legendre_forward: shared memory tile too large");
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<grid, 256, sm, st>>>(P.R, P.J, P.nlat, nf, groups, P.d_mu_n, P.d_seed, P.d_rec, four, out,
                                ext ? 1 : 0);
    PSWE_LAUNCH_CHECK();
}

void legendre_forward(const pswe_plan& P, const double2* four, int nf, int n_batch, double2* out, bool ext,
                      cudaStream_t st) {
    if (n_batch <= 0) return;
    if (P.J > 1024) throw std::invalid_argument("legendre_forward: nlat > 2048 not supported");
    if (P.legendre_mode == PSWE_LEGENDRE_STREAM && !P.simt) {  // DMMA on the streamed table
        legendre_forward_stream(P, four, nf * n_batch, out, ext, st);
    } else if (P.legendre_mode == PSWE_LEGENDRE_STREAM) {
        if (nf % 5 == 0) fwd_stream<5>(P, four, nf, n_batch, out, ext, st);
        else if (nf % 2 == 0) fwd_stream<2>(P, four, nf, n_batch, out, ext, st);
        else fwd_stream<1>(P, four, nf, n_batch, out, ext, st);
    } else if (!P.simt) {  // default: FP64 tensor cores (legendre_mma.cu)
        legendre_forward_mma(P, four, nf * n_batch, out, ext, st);
    } else {
        // shared-memory budget: g = NF*2*J*16 B, tile = J*SC*8 B
        if (nf % 5 == 0 && P.J <= 384) fwd_rec<5, 32>(P, four, nf, n_batch, out, ext, st);
        else if (nf % 5 == 0) {
            // large grids: one field per block keeps g small
            fwd_rec<1, 16>(P, four, nf, n_batch, out, ext, st);
        } else if (nf % 2 == 0 && P.J <= 512) fwd_rec<2, 32>(P, four, nf, n_batch, out, ext, st);
        else fwd_rec<1, 16>(P, four, nf, n_batch, out, ext, st);
    }
}

}  // namespace pswe
