// Forward Legendre contraction on DMMA, v2 (sm_100a, fp64) — see legendre_mma.cu for the
// mathematics. Differences from leg_fwd_mma_kernel:
//   * a warp task covers CPW 16-degree chunks (16 CPW degrees): every B fragment (4 latitudes x
//     8 columns of G) feeds CPW degree tiles, which divides the dominant shared-memory traffic
//     (B-fragment wavefronts ~ DMMA time at CPW = 1) by CPW;
//   * the G tile has no padding: conflict-free B loads come from an XOR swizzle of the column
//     index (row stride 8 NT doubles), shrinking the tile by 20-33 % (occupancy).
#include <cstdlib>

#include "pswe_internal.h"

namespace pswe {

namespace {

constexpr int CH = 16;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ double rec_step(double2 ab, double mu, double p, double pm1) {
    return __fma_rn(ab.x, __dmul_rn(mu, p), -__dmul_rn(ab.y, pm1));
}

// swizzled position of (latitude j, real column c) in the G tile (row stride 8 NT)
template <int NT>
__device__ __forceinline__ int gpos(int j, int c) {
    if constexpr (NT == 1) return j * 8 + (c ^ (((j >> 1) & 1) << 2));
    else return j * (8 * NT) + (c ^ ((j & 3) << 2));
}

template <int NT, int CPW>
__global__ void __launch_bounds__(256) leg_fwd_mma2_kernel(int R, int J, int nlat, int nq,
                                                           const double* __restrict__ mu_n,
                                                           const double2* __restrict__ chk,
                                                           const int* __restrict__ chk_off,
                                                           const double2* __restrict__ rec,
                                                           const double2* __restrict__ four,
                                                           double2* __restrict__ out, int ext, int exp_mode) {
    constexpr int SP = 36;       // P tile stride (4 mod 8 doubles)
    constexpr int SG = 8 * NT;   // G tile stride (swizzled, no padding)
    constexpr int DEG = CH * CPW;
    extern __shared__ double smem[];
    const int W = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nsl = (J + 31) >> 5;
    const int Jp = nsl * 32;
    const int m = blockIdx.x;
    const int len = R + 2 - m;
    double* G = smem;                                           // [2][Jp][SG]
    double* mus = G + 2 * Jp * SG;                              // [Jp]
    double2* rcs = reinterpret_cast<double2*>(mus + Jp);        // [R+2]
    double* tile = mus + Jp + 2 * (R + 2) + warp * (DEG * SP);  // [DEG][SP] per warp

    const int q0 = blockIdx.y * 4 * NT;
    const int tmax = ext ? len : len - 1;
    const int ntask = (len + DEG - 1) / DEG;
    const long bx = off_ext(R, m);
    const long Kx = (long)(R + 1) * (R + 4) / 2, K = (long)(R + 1) * (R + 2) / 2;

    for (int idx = threadIdx.x; idx < Jp * 4 * NT; idx += blockDim.x) {
        const int ql = idx / Jp, jj = idx - ql * Jp;  // latitude fastest: coalesced rows
        const int q = q0 + ql;
        double2 e = make_double2(0.0, 0.0), o = e;
        if (jj < J && q < nq) {
            const double2* src = four + ((long)q * (R + 1) + m) * nlat;
            const int iN = nlat - J + jj, iS = J - 1 - jj;
            const double2 gn = src[iN];
            const double2 gs = (iN == iS) ? make_double2(0.0, 0.0) : src[iS];
            e = make_double2(gn.x + gs.x, gn.y + gs.y);
            o = make_double2(gn.x - gs.x, gn.y - gs.y);
        }
        G[gpos<NT>(jj, 2 * ql)] = e.x;
        G[gpos<NT>(jj, 2 * ql + 1)] = e.y;
        G[Jp * SG + gpos<NT>(jj, 2 * ql)] = o.x;
        G[Jp * SG + gpos<NT>(jj, 2 * ql + 1)] = o.y;
    }
    for (int jj = threadIdx.x; jj < Jp; jj += blockDim.x) mus[jj] = jj < J ? mu_n[jj] : 0.0;
    for (int t = threadIdx.x; t < len; t += blockDim.x) rcs[t] = rec[bx + t];
    __syncthreads();
    const double2* __restrict__ ck = chk + (long)chk_off[m] * J;
    const int r4 = lane >> 2, c4 = lane & 3;

    for (int task = warp; task < ntask; task += W) {
        const int t0 = task * DEG;
        const int c0 = task * CPW;  // checkpoint chunk index
        double acc[CPW][2][NT][2];
#pragma unroll
        for (int u = 0; u < CPW; ++u)
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < NT; ++b) acc[u][a][b][0] = acc[u][a][b][1] = 0.0;
        double2 nxt = lane < J ? ck[(long)c0 * J + lane] : make_double2(0.0, 0.0);
        for (int sl = 0; sl < nsl; ++sl) {
            const double2 cur = nxt;
            const int jn = (sl + 1) * 32 + lane;
            if (sl + 1 < nsl) nxt = jn < J ? ck[(long)c0 * J + jn] : make_double2(0.0, 0.0);
            double p = cur.x, pm1 = cur.y;
            const double mu = mus[sl * 32 + lane];
#pragma unroll
            for (int tl = 0; tl < DEG; ++tl) {
                const int t = t0 + tl;
                const bool v = t < len;
                tile[tl * SP + lane] = v ? p : 0.0;
                if (v && exp_mode != 1) {  // experiment 1: no recurrence
                    const double pn = rec_step(rcs[t], mu, p, pm1);
                    pm1 = p;
                    p = pn;
                }
            }
            __syncwarp();
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int jk = sl * 32 + 4 * ks + c4;
#pragma unroll
                for (int par = 0; par < 2; ++par) {
                    double af[CPW];
#pragma unroll
                    for (int u = 0; u < CPW; ++u) af[u] = tile[(CH * u + par + 2 * r4) * SP + 4 * ks + c4];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        const double bf = G[par * Jp * SG + gpos<NT>(jk, 8 * nt + r4)];
#pragma unroll
                        if (exp_mode != 2)  // experiment 2: no DMMA
                            for (int u = 0; u < CPW; ++u) dmma(acc[u][par][nt], af[u], bf);
                        else
                            for (int u = 0; u < CPW; ++u) acc[u][par][nt][0] += af[u] * bf;
                    }
                }
            }
            __syncwarp();
        }
#pragma unroll
        for (int u = 0; u < CPW; ++u)
#pragma unroll
            for (int par = 0; par < 2; ++par) {
                const int t = t0 + CH * u + par + 2 * r4;
                if (t >= tmax) continue;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const int q = q0 + 4 * nt + c4;
                    if (q >= nq) continue;
                    const double2 v = make_double2(acc[u][par][nt][0], acc[u][par][nt][1]);
                    if (ext) out[(long)q * Kx + bx + t] = v;
                    else out[(long)q * K + off_std(R, m) + t] = v;
                }
            }
    }
}

int exp_mode() {
    static const int e = std::getenv("PSWE_FWD_EXP") ? std::atoi(std::getenv("PSWE_FWD_EXP")) : 0;
    return e;
}

template <int NT, int CPW>
void launch2(const pswe_plan& P, const double2* four, int nq, double2* out, bool ext, int W, cudaStream_t st) {
    const int nsl = (P.J + 31) / 32;
    const int groups = (nq + 4 * NT - 1) / (4 * NT);
    const size_t sm = (size_t)(2 * nsl * 32 * 8 * NT + nsl * 32 + 2 * (P.R + 2) + W * CH * CPW * 36) * sizeof(double);
    if (sm > 227 * 1024) throw std::invalid_argument("legendre_forward: shared-memory tile too large");
    auto kern = leg_fwd_mma2_kernel<NT, CPW>;
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<dim3(P.R + 1, groups), 32 * W, sm, st>>>(P.R, P.J, P.nlat, nq, P.d_mu_n, P.d_chk, P.d_chk_off, P.d_rec,
                                                    four, out, ext ? 1 : 0, exp_mode());
    PSWE_LAUNCH_CHECK();
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

}  // namespace

// Returns false if the v2 kernel is disabled (PSWE_FWD_V=1 selects the v1 kernel).
bool legendre_forward_mma2(const pswe_plan& P, const double2* four, int nq, double2* out, bool ext, cudaStream_t st) {
    static const int ver = env_int("PSWE_FWD_V", 2);
    if (ver != 2) return false;
    static const int cpw = env_int("PSWE_FWD_CPW", 1);
    static const int W = env_int("PSWE_FWD_W", 8);
    const int nsl = (P.J + 31) / 32;
    const bool two = nq > 4 && nsl <= 24;
    if (cpw == 1) {
        if (two) launch2<2, 1>(P, four, nq, out, ext, W, st);
        else launch2<1, 1>(P, four, nq, out, ext, W, st);
    } else {
        if (two) launch2<2, 2>(P, four, nq, out, ext, W, st);
        else launch2<1, 2>(P, four, nq, out, ext, W, st);
    }
    return true;
}

}  // namespace pswe
