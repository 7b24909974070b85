// Legendre contractions on DMMA with the associated-Legendre values STREAMED from a per-plan
// table (PSWE_LEGENDRE_STREAM; sm_100a, fp64). Same mathematics as legendre_mma.cu; the P tiles
// arrive by cp.async instead of being recomputed, which removes the serial recurrence chains
// and the checkpoint loads from the contraction kernels.
//
// Table layout (built once per plan by the same recurrence, legendre.cpp:30-37): per m, per
// 32-latitude slice sl, per 16-degree chunk c, a 4 KB tile [32 rows][16] (ptile_off),
//   tile[row * 16 + (col ^ ((row & 3) << 2))] = P^m_{m + 16c + tl}(mu_{32 sl + row}),
//   col = (tl & 1) * 8 + (tl >> 1)
// i.e. the 8 even then the 8 odd degrees of a latitude, XOR-swizzled within the row. A tile is
// exactly its shared-memory image (one bulk copy; both fragment patterns below read it in two
// conflict-free wavefronts), and the chunks of one slice are contiguous, so a run of chunks is one
// copy. Degrees past R+1 are zero.
//
// forward  Y^T[col][t] = sum_j G_par^T[col][j] P[j][t]:  A = G^T (smem, swizzled), B = P tile
// inverse  E/O[j][col]  = sum_t P[j][t] X[t][col]:         A = P tile, B = X tile (smem)
// The inverse's X operand is written by its prep kernel directly as per-chunk shared-memory
// images ([16 degrees][8 NT + 2] doubles), so each pipeline stage is W + 1 bulk copies (TMA,
// cp.async.bulk) completing on one mbarrier; stages are released through a second mbarrier.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "legendre_common.cuh"
#include "xrow.cuh"

namespace pswe {

namespace {

constexpr int CH = 16;

using legc::dmma;

// swizzled column of degree-slot col (0..15) in latitude row j of a P tile
__host__ __device__ __forceinline__ int pswz(int j, int col) { return col ^ ((j & 3) << 2); }
// doubles offset of tile (chunk c, 32-latitude slice sl) of the order whose chunk base is cbm
// and chunk count nch; nsl slices per order
__host__ __device__ __forceinline__ long ptile_off(int cbm, int nch, int nsl, int c, int sl) {
    return ((long)cbm * nsl + (long)sl * nch + c) * 512;
}

__device__ __forceinline__ double rec_step(double2 ab, double mu, double p, double pm1) {
    return __fma_rn(ab.x, __dmul_rn(mu, p), -__dmul_rn(ab.y, pm1));
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// copy one (chunk, slice) tile (4 KB, already its smem image); 8 x 16 B per lane
__device__ __forceinline__ void load_tile(double* dst, const double* __restrict__ src, int lane) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int idx = u * 32 + lane;  // 256 16-byte pieces
        cp_async16(dst + 2 * idx, src + 2 * idx);
    }
}

// ---- mbarrier + bulk-copy (TMA) primitives ---------------------------------------------------
__device__ __forceinline__ unsigned sm_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sm_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sm_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(sm_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(sm_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            sm_addr(dst)),
        "l"(src), "r"(bytes), "r"(sm_addr(bar))
        : "memory");
}

// table builder: thread per (m, j)
__global__ void build_ptab2_kernel(int R, int J, int Jp, const double* __restrict__ mu_n, const double* __restrict__ seed,
                                   const double2* __restrict__ rec, const int* __restrict__ cbase,
                                   double* __restrict__ ptab) {
    const int m = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= Jp) return;
    const int len = R + 2 - m;
    const int nch = (len + CH - 1) / CH;
    const int nsl = Jp >> 5, row = j & 31;
    double* out = ptab + ptile_off(cbase[m], nch, nsl, 0, j >> 5) + row * 16;  // chunk c: + c * 512
    if (j >= J) {
        for (int c = 0; c < nch; ++c)
            for (int i = 0; i < 16; ++i) out[(long)c * 512 + i] = 0.0;
        return;
    }
    const double mu = mu_n[j];
    const double2* rc = rec + off_ext(R, m);
    double p = seed[(long)m * J + j], pm1 = 0.0;
    for (int t = 0; t < nch * CH; ++t) {
        const int c = t / CH, tl = t % CH;
        out[(long)c * 512 + pswz(row, (tl & 1) * 8 + (tl >> 1))] = t < len ? p : 0.0;
        if (t < len) {
            const double pn = rec_step(__ldg(rc + t), mu, p, pm1);
            pm1 = p;
            p = pn;
        }
    }
}

// Polar skip table: for order m and 32-latitude slice sl, the first 16-degree chunk whose P tile
// holds a value of magnitude >= kPolarEps. At high latitudes P^m_s starts from the seed
// P^m_m ~ (1 - mu^2)^(m/2) and grows with s, so the negligible tiles of a slice are a prefix of its
// chunks (T511: 17% of all tiles, T1023: 24%). The contractions start there: the skipped terms are
// < 1e-20 of the normalised P (orthonormal columns), below every double rounding of the sums
// they would enter (SHTns' "polar optimisation" with a threshold far under the 1e-12 parity bound).
constexpr double kPolarEps = 1e-20;
__global__ void build_polar_kernel(int R, int nsl, const int* __restrict__ cbase, const double* __restrict__ ptab,
                                   int* __restrict__ cstart) {
    const int sl = blockIdx.x, m = blockIdx.y, lane = threadIdx.x;
    const int nch = (R + 2 - m + CH - 1) / CH;
    int first = nch;
    for (int c = 0; c < nch; ++c) {
        const double* tile = ptab + ptile_off(cbase[m], nch, nsl, c, sl) + lane * 16;
        double mx = 0.0;
#pragma unroll
        for (int i = 0; i < 16; ++i) mx = fmax(mx, fabs(tile[i]));
        if (__any_sync(0xffffffffu, mx >= kPolarEps)) {
            first = c;
            break;
        }
    }
    if (lane == 0) cstart[m * nsl + sl] = first;
}

template <int NT>
__device__ __forceinline__ int gpos(int j, int c) {
    if constexpr (NT == 1) return j * 8 + (c ^ (((j >> 1) & 1) << 2));
    else return j * (8 * NT) + (c ^ ((j & 3) << 2));
}

// ---- forward ------------------------------------------------------------------------------
// grid (R+1, column groups); warp task = chunk c (16 degrees), loop over latitude slices with a
// double-buffered cp.async P tile.
template <int NT>
__global__ void __launch_bounds__(256) leg_fwd_stream_mma_kernel(int R, int J, int Jp, int nlat, int nq,
                                                                 const double* __restrict__ ptab,
                                                                 const int* __restrict__ cbase,
                                                                 const double2* __restrict__ four,
                                                                 double2* __restrict__ out, int ext) {
    constexpr int SG = 8 * NT;
    extern __shared__ double smem[];
    const int W = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nsl = Jp >> 5;
    const int m = blockIdx.x;
    const int len = R + 2 - m;
    const int nch = (len + CH - 1) / CH;
    double* G = smem;                                       // [2][Jp][SG] swizzled
    double* tiles = smem + 2 * Jp * SG + warp * (2 * 32 * 16);  // [2][32][16] per warp
    const int q0 = blockIdx.y * 4 * NT;
    const int tmax = ext ? len : len - 1;
    const long bx = off_ext(R, m);
    const long Kx = (long)(R + 1) * (R + 4) / 2, K = (long)(R + 1) * (R + 2) / 2;
    const double* __restrict__ pm = ptab + ptile_off(cbase[m], nch, nsl, 0, 0);  // + (sl nch + c) 512

    // first P tile of this warp's first chunk streams in while G is staged
    if (warp < nch) {
        load_tile(tiles, pm + (long)warp * 512, lane);
        cp_async_commit();
    }
#ifndef PSWE_FDIAG_NOSTAGE
    legc::stage_g<NT, 8>(G, Jp * SG, Jp, J, nlat, R, m, q0, nq, four,
                         [](int j, int col) { return gpos<NT>(j, col); });
#endif
    __syncthreads();
    const int r4 = lane >> 2, c4 = lane & 3;
    bool first = true;

    for (int c = warp; c < nch; c += W) {
        double acc[2][NT][2];  // [par][nt]: C[col 8nt + r4][deg-in-parity 2 c4 + v]
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < NT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        const double* src = pm + (long)c * 512;  // slice sl: + sl nch 512
#ifndef PSWE_FDIAG_NOTILE
        if (!first) {  // the first task's tile was issued before the G staging
            load_tile(tiles, src, lane);
            cp_async_commit();
        }
#endif
        first = false;
        for (int sl = 0; sl < nsl; ++sl) {
#ifndef PSWE_FDIAG_NOTILE
            if (sl + 1 < nsl) load_tile(tiles + ((sl + 1) & 1) * 32 * 16, src + (long)(sl + 1) * nch * 512, lane);
#endif
            cp_async_commit();
            cp_async_wait<1>();
            __syncwarp();
            const double* tl = tiles + (sl & 1) * 32 * 16;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int jk = sl * 32 + 4 * ks + c4;  // latitude of this lane's k
#pragma unroll
                for (int par = 0; par < 2; ++par) {
                    const double bf = tl[(4 * ks + c4) * 16 + pswz(c4, par * 8 + r4)];  // B[k=lat][n=degree]
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        const double af = G[par * Jp * SG + gpos<NT>(jk, 8 * nt + r4)];  // A[m=col][k=lat]
#ifdef PSWE_FDIAG_NODMMA
                        acc[par][nt][0] += af * bf;
#else
                        dmma(acc[par][nt], af, bf);
#endif
                    }
                }
            }
            __syncwarp();
        }
        cp_async_wait<0>();
        // lane holds real column 8 nt + r4, degrees t0 + par + 2 (2 c4 + v)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int col = 8 * nt + r4;
            const int q = q0 + (col >> 1);
            if (q >= nq) continue;
#pragma unroll
            for (int par = 0; par < 2; ++par)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int t = c * CH + par + 2 * (2 * c4 + v);
                    if (t >= tmax) continue;
                    double* dst = reinterpret_cast<double*>(ext ? out + (long)q * Kx + bx + t
                                                                : out + (long)q * K + off_std(R, m) + t);
                    dst[col & 1] = acc[par][nt][v];
                }
        }
    }
}

// ---- forward on G tiles ----------------------------------------------------------------------
// Task = a run of chunks of at most two orders m_a, m_b (plan task table, about kFwdPerSm per SM,
// equal work); column group z = blockIdx.y. Warp w owns CPW chunks of one order (2 CPW n-tiles:
// even and odd degrees) for all NTC column tiles. K (latitude) streams in 8-latitude stages: one
// bulk copy of the G tile of each order (both hemispheres, written in this layout by the grid
// stage) and one 1 KB copy per chunk of the P table, into an S-stage mbarrier ring.
// G_E = G_N + G_S and G_O = G_N - G_S are formed in registers and reused by the CPW chunks.
// register budget: the 8-warp and the narrow (one / two state, 32-latitude stage) configurations
// are held to 2 blocks per SM by shared memory anyway; saying so lets ptxas use 72-118 registers
// instead of its own 48-64 (+spills): single-state forward T255 -1.1 us, T511 -6 us. The 4-warp
// wide configurations keep ptxas' default (0 = unspecified; an explicit 1 or 2 grows the T511
// tiling to 188 registers and loses 6%).
// PROD: one extra warp only issues the ring refills (it waits for the compute warps' release of
// stage q and issues stage q + S), so no compute warp stalls on the slowest one before its next
// stage (T255 batch 98.3 -> 96.8 us, T511 batch 461 -> 443 us). PSWE_FWD_PROD=0: warp 0 refills.
// WTASK: forward tasks cut by polar-skip weight (build_legendre_table2); 0 = the earlier
// equal-chunk cut in pair order m, R-m. Bit-identical; T511 batch forward -3.7%, PFASST
// config 3 / 4 / 5 -0.7 / -0.9 / -1.5% (tools/ab_time.py on the B200).
#ifndef PSWE_FWD_WG
#define PSWE_FWD_WG 0  // per-stage G-tile cost of a task in chunk units (cut cost model)
#endif
#ifndef PSWE_FWD_WTASK
#define PSWE_FWD_WTASK 1
#endif
#ifndef PSWE_FWD_PROD
#define PSWE_FWD_PROD 1
#endif
template <int NTC, int W, int CPW, int S, int SUB, bool PROD = PSWE_FWD_PROD>
__global__ void __launch_bounds__(32 * (W + (PROD ? 1 : 0)), (W == 8 || SUB == 4) ? 2 : 0) leg_fwd_gt_kernel(int R, int Jp, int nq, GtLayout gl,
                                                           const double* __restrict__ ptab,
                                                           const int* __restrict__ cbase,
                                                           const int4* __restrict__ tasks_a,
                                                           const int2* __restrict__ tasks_b,
                                                           const double* __restrict__ gt,
                                                           double2* __restrict__ out,
                                                           const int* __restrict__ cstart) {
    constexpr int NS = W * CPW;  // chunk slots
    extern __shared__ __align__(128) double smem[];
    __shared__ long pbase[NS], pstride[NS];  // tile (chunk, slice 0) offset; per-slice stride
    __shared__ int pslot[NS], npc;
    const int sgc = gl.sgc;
    const int gsub = 2 * 8 * sgc;                // doubles of one 8-latitude sub-stage of G
    const int gstage = SUB * gsub;               // doubles of one order's G stage
    constexpr int PS = SUB * 128;                // doubles of one chunk's P stage
    double* sG = smem;                           // [S][2 orders][SUB][2][8][sgc]
    double* sP = sG + S * 2 * gstage;            // [S][NS][SUB * 8 * 16]
    unsigned long long* full = reinterpret_cast<unsigned long long*>(sP + S * NS * PS);
    unsigned long long* empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int4 ta = tasks_a[blockIdx.x];
    const int2 tb = tasks_b[blockIdx.x];
    const int na = ta.z, nb = tb.y;
    const int wa = (na + CPW - 1) / CPW;  // warps of order a
    const int z = blockIdx.y;
    const int ns8 = gl.ns8;
    __shared__ int nst_s;
    const bool ord_b = warp >= wa;
    const int my_m = ord_b ? ta.w : ta.x;
    const int my_c0 = ord_b ? tb.x + (warp - wa) * CPW : ta.y + warp * CPW;
    const int my_n = max(0, min(CPW, ord_b ? nb - (warp - wa) * CPW : na - warp * CPW));
    const bool mine = my_n > 0;
    const double* __restrict__ ga = gt + ((long)z * (R + 1) + ta.x) * ns8 * gsub;
    const double* __restrict__ gb = gt + ((long)z * (R + 1) + ta.w) * ns8 * gsub;
    const int r4 = lane >> 2, c4 = lane & 3;
    const unsigned GB = (unsigned)gstage * sizeof(double);

    if (threadIdx.x == 0) {
        int n = 0;  // valid chunk slots in warp order: slot (w, u) -> table tile
        for (int w = 0; w < W; ++w) {
            const bool b = w >= wa;
            const int m = b ? ta.w : ta.x;
            const int c0 = b ? tb.x + (w - wa) * CPW : ta.y + w * CPW;
            const int nn = max(0, min(CPW, b ? nb - (w - wa) * CPW : na - w * CPW));
            for (int u = 0; u < nn; ++u) {
                const int nchm = (R + 2 - m + CH - 1) / CH;
                pbase[n] = ptile_off(cbase[m], nchm, Jp >> 5, c0 + u, 0);
                pstride[n] = (long)nchm * 512;
                pslot[n] = w * CPW + u;
                ++n;
            }
        }
        npc = n;
        for (int k = 0; k < S; ++k) {
            mbar_init(full + k, 1);
            mbar_init(empty + k, W);
        }
        mbar_fence_init();
    }
    if (warp == 0) {
        // polar skip at block granularity: the stages (latitudes) past the last 32-latitude slice in
        // which any of the task's chunks reaches |P| >= 1e-20 are dropped (lane = slice; a task's
        // most significant chunk of each order is its last one)
        const int nsl = Jp >> 5;
        int nsl_eff = nsl;
        if (cstart) {
            const int ca = ta.y + na - 1, cb = tb.x + nb - 1;
            bool sig = false;
            if (lane < nsl) {
                sig = ca >= cstart[ta.x * nsl + lane];
                if (nb > 0) sig = sig || cb >= cstart[ta.w * nsl + lane];
            }
            const unsigned bm = __ballot_sync(0xffffffffu, sig);
            nsl_eff = 32 - __clz((int)bm);
        }
        if (lane == 0) nst_s = (nsl_eff * 4) / SUB;  // ns8 = 4 nsl
    }
    __syncthreads();
    pdl_trigger();
    const int np = npc;
    const int nst = nst_s;  // stages of 8 SUB latitudes
    // stage q: latitude rows 8 SUB q .. 8 SUB q + 8 SUB - 1; the P tiles (plan constants) and the G
    // tiles (the grid stage's output) complete on the same mbarrier
    auto issue_p = [&](int q) {
        const int k = q % S;
        constexpr unsigned PB = PS * sizeof(double);
        mbar_expect_tx(full + k, GB * (nb > 0 ? 2u : 1u) + np * PB);
        const int sub0 = q * SUB;  // first 8-latitude sub-slice: rows of slice sub0 / 4
        for (int u = 0; u < np; ++u)
            bulk_g2s(sP + (k * NS + pslot[u]) * PS, ptab + pbase[u] + (sub0 >> 2) * pstride[u] + (sub0 & 3) * 128,
                     PB, full + k);
    };
    auto issue_g = [&](int q) {
        const int k = q % S;
        bulk_g2s(sG + (k * 2) * gstage, ga + (long)q * gstage, GB, full + k);
        if (nb > 0) bulk_g2s(sG + (k * 2 + 1) * gstage, gb + (long)q * gstage, GB, full + k);
    };
    auto issue = [&](int q) {
        issue_p(q);
        issue_g(q);
    };
    // the first stages' P tiles stream in while the grid stage finishes (programmatic launch)
    if (threadIdx.x == 0)
        for (int q = 0; q < S && q < nst; ++q) issue_p(q);
    pdl_wait();  // G tiles come from the grid stage
    if (threadIdx.x == 0)
        for (int q = 0; q < S && q < nst; ++q) issue_g(q);

    if (PROD && warp == W) {  // producer warp: ring refills only
        if (lane == 0)
            for (int q = 0; q + S < nst; ++q) {
                mbar_wait(empty + q % S, (unsigned)(q / S) & 1u);
                issue(q + S);
            }
        return;
    }
    double acc[NTC][CPW][2][2];
#pragma unroll
    for (int a = 0; a < NTC; ++a)
#pragma unroll
        for (int b = 0; b < CPW; ++b) acc[a][b][0][0] = acc[a][b][0][1] = acc[a][b][1][0] = acc[a][b][1][1] = 0.0;

    for (int q = 0; q < nst; ++q) {
        const int k = q % S;
        const unsigned ph = (unsigned)(q / S) & 1u;
        mbar_wait(full + k, ph);
        __syncwarp();
        if (mine) {
#pragma unroll
            for (int sub = 0; sub < SUB; ++sub) {
            const double* g = sG + (k * 2 + (ord_b ? 1 : 0)) * gstage + sub * gsub;
            const double* pt = sP + (k * NS + warp * CPW) * PS + sub * 128;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                const int rr = 4 * ks + c4;  // latitude row of this lane's k
                double ae[NTC], ao[NTC], be[CPW], bo[CPW];
#pragma unroll
                for (int nt = 0; nt < NTC; ++nt) {
                    const int cs = (8 * nt + r4) ^ gt_swz(NTC, rr);
                    const double gn = g[rr * sgc + cs];
                    const double gs = g[(8 + rr) * sgc + cs];
                    ae[nt] = gn + gs;
                    ao[nt] = gn - gs;
                }
#pragma unroll
                for (int cc = 0; cc < CPW; ++cc) {
                    be[cc] = pt[cc * PS + rr * 16 + pswz(c4, r4)];
                    bo[cc] = pt[cc * PS + rr * 16 + pswz(c4, 8 + r4)];
                }
#pragma unroll
                for (int nt = 0; nt < NTC; ++nt)
#pragma unroll
                    for (int cc = 0; cc < CPW; ++cc) {
                        dmma(acc[nt][cc][0], ae[nt], be[cc]);
                        dmma(acc[nt][cc][1], ao[nt], bo[cc]);
                    }
            }
            }  // sub-stages
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + k);
        if (!PROD && threadIdx.x == 0 && q + S < nst) {
            mbar_wait(empty + k, ph);
            issue(q + S);
        }
    }
    if (!mine) return;
    // C[m = column 8 nt + r4][n = degree-in-parity 2 c4 + v]: t = 16 c + par + 2 (2 c4 + v)
    const long Kx = gl.plain ? (long)(R + 1) * (R + 2) / 2 : (long)(R + 1) * (R + 4) / 2;
    const long bx = gl.plain ? off_std(R, my_m) : off_ext(R, my_m);
    const int len = R + 2 - my_m - gl.plain;
    const int qz = z * gl.apg;
#pragma unroll
    for (int nt = 0; nt < NTC; ++nt) {
        const int col = 8 * nt + r4;
        const int q = qz + (col >> 1);
        if ((col >> 1) >= gl.apg || q >= nq) continue;
#pragma unroll
        for (int cc = 0; cc < CPW; ++cc) {
            if (cc >= my_n) continue;
#pragma unroll
            for (int par = 0; par < 2; ++par)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int t = (my_c0 + cc) * CH + par + 2 * (2 * c4 + v);
                    if (t >= len) continue;
                    reinterpret_cast<double*>(out + (long)q * Kx + bx + t)[col & 1] = acc[nt][cc][par][v];
                }
        }
    }
}

// PSWE_NO_POLAR=1 disables the polar skip (A/B and parity checks)
bool polar_on() {
    static const bool on = [] { const char* e = getenv("PSWE_NO_POLAR"); return !(e && atoi(e) != 0); }();
    return on;
}
template <int NTC, int W, int CPW, int S, int SUB = 1>
void fwd_gt_launch(const pswe_plan& P, const GtLayout& gl, int nq, double2* out, cudaStream_t st) {
    const int Jp = ((P.J + 31) / 32) * 32;
    const size_t sm = (size_t)S * SUB * (2 * 2 * 8 * gl.sgc + W * CPW * 128) * sizeof(double) +
                      2 * S * sizeof(unsigned long long);
    auto kern = leg_fwd_gt_kernel<NTC, W, CPW, S, SUB>;
    static int attr = 0;
    if ((int)sm > attr) {
        PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        attr = (int)sm;
    }
    launch_pdl(kern, dim3(P.n_fwd_tasks, gl.groups), dim3(32 * (W + (PSWE_FWD_PROD ? 1 : 0))), sm, st, P.R, Jp, nq, gl,
               P.d_ptab2, P.d_chk_off,
               P.d_fwd_ta, P.d_fwd_tb, P.d_gtile, out, (const int*)(polar_on() ? P.d_cstart : nullptr));
    PSWE_LAUNCH_CHECK();
}

// ---- forward, column-warp mapping ---------------------------------------------------------
// Same tasks (<= 8 chunk slots of <= 2 orders), the same producer warp / mbarrier ring of {G tiles,
// P tiles} stages and the same epilogue as leg_fwd_gt_kernel, but the work is split by COLUMN
// TILE instead of by chunk: compute warp w = (column tile w % NTC, slot group w / NTC) computes its
// 8 columns against every chunk slot of its group. Per k-step a warp forms G_E = G_N + G_S and
// G_O = G_N - G_S for ONE column tile per order (2 shared loads, 2 additions) and reuses them for
// 2 DMMA per slot: in leg_fwd_gt_kernel every warp re-formed all NTC tiles (NTC additions per
// 2 NTC DMMA, 1/8 of the FP64 pipe - the additions share the pipe with DMMA - and 25% of the
// instructions, profiles/r01_ncu_eval_kernels_r01l.txt). H slot groups: 8 / H chunk slots per
// warp (H = 1 for wide column groups, more warps for narrow ones).
#ifndef PSWE_FWD_CW
#define PSWE_FWD_CW 1
#endif
// one ring stage of leg_fwd_gt_cw_kernel: slots 0..NA-1 of this warp belong to the task's first
// order (G at g0), the others to its second (G at g0 + gstage)
template <int NTC, int SPW, int SUB, int NA>
__device__ __forceinline__ void cw_stage(double (&acc)[SPW][2][2], const double* g0, const double* pt, int gstage,
                                         int gsub, int sgc, int nt, int r4, int c4) {
    constexpr int PS = SUB * 128;
#pragma unroll
    for (int sub = 0; sub < SUB; ++sub) {
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            const int rr = 4 * ks + c4;
            const int cs = (8 * nt + r4) ^ gt_swz(NTC, rr);
            double be[SPW], bo[SPW];
#pragma unroll
            for (int u = 0; u < SPW; ++u) {
                be[u] = pt[u * PS + sub * 128 + rr * 16 + pswz(c4, r4)];
                bo[u] = pt[u * PS + sub * 128 + rr * 16 + pswz(c4, 8 + r4)];
            }
            double aea = 0.0, aoa = 0.0, aeb = 0.0, aob = 0.0;
            if constexpr (NA > 0) {
                const double* g = g0 + sub * gsub;
                const double gn = g[rr * sgc + cs], gs = g[(8 + rr) * sgc + cs];
                aea = gn + gs;
                aoa = gn - gs;
            }
            if constexpr (NA < SPW) {
                const double* g = g0 + gstage + sub * gsub;
                const double gn = g[rr * sgc + cs], gs = g[(8 + rr) * sgc + cs];
                aeb = gn + gs;
                aob = gn - gs;
            }
#pragma unroll
            for (int u = 0; u < SPW; ++u) {
                dmma(acc[u][0], u < NA ? aea : aeb, be[u]);
                dmma(acc[u][1], u < NA ? aoa : aob, bo[u]);
            }
        }
    }
}

template <int NTC, int H, int S, int SUB>
__global__ void __launch_bounds__(32 * (NTC * H + 1), (NTC * H + 1) <= 8 ? 2 : 1)
    leg_fwd_gt_cw_kernel(int R, int Jp, int nq, GtLayout gl, const double* __restrict__ ptab,
                         const int* __restrict__ cbase, const int4* __restrict__ tasks_a,
                         const int2* __restrict__ tasks_b, const double* __restrict__ gt,
                         double2* __restrict__ out, const int* __restrict__ cstart) {
    constexpr int NS = 8;       // chunk slots per task (task table: W x CPW = 8)
    constexpr int SPW = NS / H;  // slots per warp
    constexpr int WC = NTC * H;  // compute warps
    extern __shared__ __align__(128) double smem[];
    __shared__ long pbase[NS], pstride[NS];
    __shared__ int npc, nst_s;
    const int sgc = gl.sgc;
    const int gsub = 2 * 8 * sgc;
    const int gstage = SUB * gsub;
    constexpr int PS = SUB * 128;
    double* sG = smem;                // [S][2 orders][SUB][2][8][sgc]
    double* sP = sG + S * 2 * gstage;  // [S][NS][SUB * 8 * 16]
    unsigned long long* full = reinterpret_cast<unsigned long long*>(sP + S * NS * PS);
    unsigned long long* empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int4 ta = tasks_a[blockIdx.x];
    const int2 tb = tasks_b[blockIdx.x];
    const int na = ta.z, nb = tb.y;
    const int z = blockIdx.y;
    const int ns8 = gl.ns8;
    const double* __restrict__ ga = gt + ((long)z * (R + 1) + ta.x) * ns8 * gsub;
    const double* __restrict__ gb = gt + ((long)z * (R + 1) + ta.w) * ns8 * gsub;
    const int r4 = lane >> 2, c4 = lane & 3;
    const unsigned GB = (unsigned)gstage * sizeof(double);
    const int nt = warp % NTC, hg = warp / NTC;  // column tile, slot group
    const int u0 = hg * SPW;                      // first slot of this warp

    if (threadIdx.x == 0) {
        int n = 0;  // slots: order a's chunks, then order b's
        for (int i = 0; i < na + nb; ++i) {
            const bool b = i >= na;
            const int m = b ? ta.w : ta.x;
            const int c = b ? tb.x + (i - na) : ta.y + i;
            const int nchm = (R + 2 - m + CH - 1) / CH;
            pbase[n] = ptile_off(cbase[m], nchm, Jp >> 5, c, 0);
            pstride[n] = (long)nchm * 512;
            ++n;
        }
        npc = n;
        for (int k = 0; k < S; ++k) {
            mbar_init(full + k, 1);
            mbar_init(empty + k, WC);
        }
        mbar_fence_init();
    }
    if (warp == 0) {  // polar skip at block granularity (as leg_fwd_gt_kernel)
        const int nsl = Jp >> 5;
        int nsl_eff = nsl;
        if (cstart) {
            const int ca = ta.y + na - 1, cb = tb.x + nb - 1;
            bool sig = false;
            if (lane < nsl) {
                sig = ca >= cstart[ta.x * nsl + lane];
                if (nb > 0) sig = sig || cb >= cstart[ta.w * nsl + lane];
            }
            const unsigned bm = __ballot_sync(0xffffffffu, sig);
            nsl_eff = 32 - __clz((int)bm);
        }
        if (lane == 0) nst_s = (nsl_eff * 4) / SUB;
    }
    __syncthreads();
    pdl_trigger();
    const int np = npc;
    const int nst = nst_s;
    auto issue_p = [&](int q) {
        const int k = q % S;
        constexpr unsigned PB = PS * sizeof(double);
        mbar_expect_tx(full + k, GB * (nb > 0 ? 2u : 1u) + np * PB);
        const int sub0 = q * SUB;
        for (int u = 0; u < np; ++u)
            bulk_g2s(sP + (k * NS + u) * PS, ptab + pbase[u] + (sub0 >> 2) * pstride[u] + (sub0 & 3) * 128, PB,
                     full + k);
    };
    auto issue_g = [&](int q) {
        const int k = q % S;
        bulk_g2s(sG + (k * 2) * gstage, ga + (long)q * gstage, GB, full + k);
        if (nb > 0) bulk_g2s(sG + (k * 2 + 1) * gstage, gb + (long)q * gstage, GB, full + k);
    };
    if (threadIdx.x == 0)
        for (int q = 0; q < S && q < nst; ++q) issue_p(q);
    pdl_wait();  // G tiles come from the grid stage
    if (threadIdx.x == 0)
        for (int q = 0; q < S && q < nst; ++q) issue_g(q);

    if (warp == WC) {  // producer warp: ring refills only
        if (lane == 0)
            for (int q = 0; q + S < nst; ++q) {
                mbar_wait(empty + q % S, (unsigned)(q / S) & 1u);
                issue_p(q + S);
                issue_g(q + S);
            }
        return;
    }
    // slots of this warp: u0 .. u0 + SPW - 1; slot u is order a's chunk u (u < na) or order b's
    const int my_na = max(0, min(SPW, na - u0));           // order-a slots among mine
    const int my_n = max(0, min(SPW, na + nb - u0));       // live slots among mine
    double acc[SPW][2][2];
#pragma unroll
    for (int u = 0; u < SPW; ++u) acc[u][0][0] = acc[u][0][1] = acc[u][1][0] = acc[u][1][1] = 0.0;

    for (int q = 0; q < nst; ++q) {
        const int k = q % S;
        const unsigned ph = (unsigned)(q / S) & 1u;
        mbar_wait(full + k, ph);
        __syncwarp();
        if (my_n > 0) {
            const double* g0 = sG + (k * 2) * gstage;
            const double* pt = sP + (k * NS + u0) * PS;
            // the order split of this warp's slots as a compile-time constant: straight-line code,
            // every fragment loaded before the k-step's DMMAs (slots past my_n compute on stale
            // shared memory and are never stored)
            switch (my_na) {
#define PSWE_CW_CASE(NA) \
    case NA: if constexpr (NA <= SPW) cw_stage<NTC, SPW, SUB, NA>(acc, g0, pt, gstage, gsub, sgc, nt, r4, c4); break;
                PSWE_CW_CASE(0) PSWE_CW_CASE(1) PSWE_CW_CASE(2) PSWE_CW_CASE(3) PSWE_CW_CASE(4)
                PSWE_CW_CASE(5) PSWE_CW_CASE(6) PSWE_CW_CASE(7) PSWE_CW_CASE(8)
#undef PSWE_CW_CASE
                default: break;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + k);
    }
    if (my_n == 0) return;
    const long Kx = gl.plain ? (long)(R + 1) * (R + 2) / 2 : (long)(R + 1) * (R + 4) / 2;
    const int qz = z * gl.apg;
    const int col = 8 * nt + r4;
    const int q = qz + (col >> 1);
    if ((col >> 1) >= gl.apg || q >= nq) return;
#pragma unroll
    for (int u = 0; u < SPW; ++u) {
        if (u >= my_n) continue;
        const int slot = u0 + u;
        const bool b = slot >= na;
        const int m = b ? ta.w : ta.x;
        const int c = b ? tb.x + (slot - na) : ta.y + slot;
        const long bx = gl.plain ? off_std(R, m) : off_ext(R, m);
        const int len = R + 2 - m - gl.plain;
#pragma unroll
        for (int par = 0; par < 2; ++par)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int t = c * CH + par + 2 * (2 * c4 + v);
                if (t >= len) continue;
                reinterpret_cast<double*>(out + (long)q * Kx + bx + t)[col & 1] = acc[u][par][v];
            }
    }
}

template <int NTC, int H, int S, int SUB>
void fwd_cw_launch(const pswe_plan& P, const GtLayout& gl, int nq, double2* out, cudaStream_t st) {
    const int Jp = ((P.J + 31) / 32) * 32;
    const size_t sm = (size_t)S * SUB * (2 * 2 * 8 * gl.sgc + 8 * 128) * sizeof(double) +
                      2 * S * sizeof(unsigned long long);
    auto kern = leg_fwd_gt_cw_kernel<NTC, H, S, SUB>;
    static int attr = 0;
    if ((int)sm > attr) {
        PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        attr = (int)sm;
    }
    launch_pdl(kern, dim3(P.n_fwd_tasks, gl.groups), dim3(32 * (NTC * H + 1)), sm, st, P.R, Jp, nq, gl, P.d_ptab2,
               P.d_chk_off, P.d_fwd_ta, P.d_fwd_tb, P.d_gtile, out,
               (const int*)(polar_on() ? P.d_cstart : nullptr));
    PSWE_LAUNCH_CHECK();
}

// ---- forward, narrow column groups: P fragments straight from the table into registers --------
// PSWE_FWD_DIRECT (default): for one/two-state batches (NTC <= 3) on grids of up to NSL 32-latitude
// slices, every warp loads ALL the B fragments of its chunk (NSL x 8 k-steps x {even, odd} - one
// 8-byte value per lane each, 4 rows x 8 columns of a swizzled P tile per warp instruction: full
// sectors) into registers BEFORE the programmatic-launch wait, so the P table read (the kernel's
// dominant traffic, plan constants) overlaps the grid stage that precedes it; after the wait only
// the G tiles of the task's (at most two) orders arrive, as one bulk copy each into shared memory.
// Same task table, fragment maps, arithmetic order and epilogue as leg_fwd_gt_kernel<NTC, 8, 1>
// (bit-identical results).
#ifndef PSWE_FWD_DIRECT
#define PSWE_FWD_DIRECT 1
#endif
template <int NTC, int NSL>
__global__ void __launch_bounds__(256, 2) leg_fwd_gt_direct_kernel(int R, int Jp, int nq, GtLayout gl,
                                                                  const double* __restrict__ ptab,
                                                                  const int* __restrict__ cbase,
                                                                  const int4* __restrict__ tasks_a,
                                                                  const int2* __restrict__ tasks_b,
                                                                  const double* __restrict__ gt,
                                                                  double2* __restrict__ out) {
    constexpr int W = 8;
    extern __shared__ __align__(128) double smem[];
    const int sgc = gl.sgc;
    const int gsub = 2 * 8 * sgc;      // doubles of one 8-latitude slice of one order's G
    const int ns8 = gl.ns8;            // = 4 NSL
    double* sG = smem;                 // [2 orders][ns8][2][8][sgc]
    __shared__ unsigned long long full;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int4 ta = tasks_a[blockIdx.x];
    const int2 tb = tasks_b[blockIdx.x];
    const int na = ta.z, nb = tb.y;
    const int z = blockIdx.y;
    const bool ord_b = warp >= na;
    const int my_m = ord_b ? ta.w : ta.x;
    const int my_c = ord_b ? tb.x + (warp - na) : ta.y + warp;
    const bool mine = ord_b ? warp - na < nb : true;
    const int r4 = lane >> 2, c4 = lane & 3;
    if (threadIdx.x == 0) {
        mbar_init(&full, 1);
        mbar_fence_init();
    }
    // B fragments of this warp's chunk: a two-slice register window (slice sl in pb[sl & 1]), 8-latitude
    // sub-slice u, k-step ks, parity; slices 0 and 1 load before the wait, slice sl + 2 as soon as
    // slice sl has been consumed
    double pb[2][4][2][2];
    const double* pt = ptab;
    long pstride = 0;
    auto load_slice = [&](int sl) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                const double* row = pt + sl * pstride + (8 * u + 4 * ks + c4) * 16;
                pb[sl & 1][u][ks][0] = row[pswz(c4, r4)];
                pb[sl & 1][u][ks][1] = row[pswz(c4, 8 + r4)];
            }
    };
    if (mine) {
        const int nchm = (R + 2 - my_m + CH - 1) / CH;
        pt = ptab + ptile_off(cbase[my_m], nchm, Jp >> 5, my_c, 0);
        pstride = (long)nchm * 512;
        load_slice(0);
        if (NSL > 1) load_slice(1);
    }
    __syncthreads();
    pdl_trigger();
    pdl_wait();  // G tiles come from the grid stage
    if (threadIdx.x == 0) {
        const unsigned GB = (unsigned)(ns8 * gsub) * sizeof(double);
        mbar_expect_tx(&full, GB * (nb > 0 ? 2u : 1u));
        bulk_g2s(sG, gt + ((long)z * (R + 1) + ta.x) * ns8 * gsub, GB, &full);
        if (nb > 0) bulk_g2s(sG + ns8 * gsub, gt + ((long)z * (R + 1) + ta.w) * ns8 * gsub, GB, &full);
    }
    double acc[NTC][2][2];
#pragma unroll
    for (int a = 0; a < NTC; ++a) acc[a][0][0] = acc[a][0][1] = acc[a][1][0] = acc[a][1][1] = 0.0;
    mbar_wait(&full, 0u);
    if (!mine) return;
    const double* gbase = sG + (ord_b ? ns8 * gsub : 0);
#pragma unroll
    for (int sl = 0; sl < NSL; ++sl) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double* g = gbase + (4 * sl + u) * gsub;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                const int rr = 4 * ks + c4;
                double ae[NTC], ao[NTC];
#pragma unroll
                for (int nt = 0; nt < NTC; ++nt) {
                    const int cs = (8 * nt + r4) ^ gt_swz(NTC, rr);
                    const double gn = g[rr * sgc + cs];
                    const double gs = g[(8 + rr) * sgc + cs];
                    ae[nt] = gn + gs;
                    ao[nt] = gn - gs;
                }
#pragma unroll
                for (int nt = 0; nt < NTC; ++nt) {
                    dmma(acc[nt][0], ae[nt], pb[sl & 1][u][ks][0]);
                    dmma(acc[nt][1], ao[nt], pb[sl & 1][u][ks][1]);
                }
            }
        }
        if (sl + 2 < NSL) load_slice(sl + 2);
    }
    const long Kx = gl.plain ? (long)(R + 1) * (R + 2) / 2 : (long)(R + 1) * (R + 4) / 2;
    const long bx = gl.plain ? off_std(R, my_m) : off_ext(R, my_m);
    const int len = R + 2 - my_m - gl.plain;
    const int qz = z * gl.apg;
#pragma unroll
    for (int nt = 0; nt < NTC; ++nt) {
        const int col = 8 * nt + r4;
        const int q = qz + (col >> 1);
        if ((col >> 1) >= gl.apg || q >= nq) continue;
#pragma unroll
        for (int par = 0; par < 2; ++par)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int t = my_c * CH + par + 2 * (2 * c4 + v);
                if (t >= len) continue;
                reinterpret_cast<double*>(out + (long)q * Kx + bx + t)[col & 1] = acc[nt][par][v];
            }
    }
}

template <int NTC, int NSL>
void fwd_direct_launch(const pswe_plan& P, const GtLayout& gl, int nq, double2* out, cudaStream_t st) {
    const int Jp = ((P.J + 31) / 32) * 32;
    const size_t sm = (size_t)2 * gl.ns8 * 2 * 8 * gl.sgc * sizeof(double);
    auto kern = leg_fwd_gt_direct_kernel<NTC, NSL>;
    static int attr = 0;
    if ((int)sm > attr) {
        PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        attr = (int)sm;
    }
    launch_pdl(kern, dim3(P.n_fwd_tasks, gl.groups), dim3(256), sm, st, P.R, Jp, nq, gl, P.d_ptab2, P.d_chk_off,
               P.d_fwd_ta, P.d_fwd_tb, P.d_gtile, out);
    PSWE_LAUNCH_CHECK();
}

// ---- inverse ------------------------------------------------------------------------------
// X tiles: per column group z (4 NT complex columns from q0 = 4 NT z), per chunk (cbase(m) + c):
// [16 degrees tl][8 NT + 2] doubles, column 2 ql + {re, im}, two zero pad columns; degree
// t = 16 c + tl of order m (extended t = 0..R+1-m; standard t = 0..R-m), zero beyond.
// prep: block (chunk, item group), thread (item, degree tl) with the degree fastest (coalesced
// reads of the m-major coefficient rows) computes all PER columns of its item (transform.cpp:
// 204-206 with the H-sums as P-sums): EVAL item = state, columns {Phi, zeta, U, V}; UV item =
// pair, columns {U, V}; PLAIN item = field (standard layout, copied), and stores them into the
// tile of whichever column group they fall in. One block per chunk for every column tiling; the
// threads of item slot g < groups also zero tile g's pad columns and the columns past nq.
constexpr int kPrepItems = 32;  // items per block (blockIdx.y covers more)
template <int KIND>
__global__ void __launch_bounds__(CH * kPrepItems)
    xtile_prep_kernel(int R, int NQ, int SX, int nq, int nct, const int* __restrict__ chunk_desc,
                      const double* __restrict__ eps, const double* __restrict__ rtab,
                      const double2* __restrict__ in, const double2* __restrict__ in2, double radius,
                      double* __restrict__ Xt) {
    constexpr int PER = KIND == INV_EVAL ? 4 : (KIND == INV_UV ? 2 : 1);
    const int cg = blockIdx.x;
    const int tl = threadIdx.x & (CH - 1), il = threadIdx.x / CH;
    const int item = blockIdx.y * kPrepItems + il;
    const int nitems = (nq + PER - 1) / PER;
    const int groups = (nq + NQ - 1) / NQ;
    const int2 mc = reinterpret_cast<const int2*>(chunk_desc)[cg];  // (m, chunk within m)
    const int m = mc.x;
    const int t = mc.y * CH + tl;
    const int s = m + t;
    const long K = (long)(R + 1) * (R + 2) / 2;
    const long bs = off_std(R, m), bx = off_ext(R, m);
    double2 v[PER];
#pragma unroll
    for (int f = 0; f < PER; ++f) v[f] = make_double2(0.0, 0.0);
    pdl_trigger();
    pdl_wait();  // the states come from the preceding kernel
    if (item < nitems) {
        if (KIND == INV_PLAIN) {
            if (s <= R) v[0] = in[(long)item * K + bs + t];
        } else if (s <= R + 1) {
            const double a2 = radius * radius, inv_a = 1.0 / radius;
            const double2 *vort, *div;
            int o = 0;
            if (KIND == INV_EVAL) {
                const double2* st = in + (long)item * 3 * K;
                vort = st + K;
                div = st + 2 * K;
                if (s <= R) {
                    v[0] = st[bs + t];
                    v[1] = vort[bs + t];
                }
                o = 2;
            } else {
                vort = in + (long)item * K;
                div = in2 + (long)item * K;
            }
            // the same values as legc::inv_lap_at / hcoef, with every load issued up front (clamped
            // indices, range conditions applied afterwards) so they overlap in one memory round trip
            const int sm1 = max(s - 1, m), sp1 = min(s + 1, R), s0 = min(s, R);
            const double2 vm = vort[bs + sm1 - m], v0 = vort[bs + s0 - m], vp = vort[bs + sp1 - m];
            const double2 dm = div[bs + sm1 - m], d0 = div[bs + s0 - m], dp = div[bs + sp1 - m];
            const double rm = __ldg(rtab + max(s - 1, 0)), r0 = __ldg(rtab + s0), rp = __ldg(rtab + min(s + 1, R));
            const double em = eps[bx + t], ep = eps[bx + min(t + 1, R + 1 - m)];  // stay inside block m
            // inverse Laplacian factors -a^2/(s'(s'+1)) at s-1, s, s+1 (0 outside m..R and at 0)
            const double fm = (s - 1 >= m && s - 1 >= 1) ? -a2 * rm : 0.0;
            const double f0 = (s <= R && s >= 1) ? -a2 * r0 : 0.0;
            const double fp = (s + 1 <= R) ? -a2 * rp : 0.0;
            const double hm = (s - 1 >= m) ? -(double)(s - 1) * em : 0.0;  // H-sum weights
            const double hp = (s + 1 <= R) ? (double)(s + 2) * ep : 0.0;
            const double2 chi = make_double2(d0.x * f0, d0.y * f0);
            const double2 psi = make_double2(v0.x * f0, v0.y * f0);
            double2 cpsi = make_double2(0.0, 0.0), cchi = make_double2(0.0, 0.0);
            if (s - 1 >= m) {
                cpsi.x += hm * (vm.x * fm);
                cpsi.y += hm * (vm.y * fm);
                cchi.x += hm * (dm.x * fm);
                cchi.y += hm * (dm.y * fm);
            }
            if (s + 1 <= R) {
                cpsi.x += hp * (vp.x * fp);
                cpsi.y += hp * (vp.y * fp);
                cchi.x += hp * (dp.x * fp);
                cchi.y += hp * (dp.y * fp);
            }
            v[o] = make_double2(inv_a * (-m * chi.y - cpsi.x), inv_a * (m * chi.x - cpsi.y));
            v[o + 1] = make_double2(inv_a * (-m * psi.y + cchi.x), inv_a * (m * psi.x + cchi.y));
        }
        // NQ = 4 NT is a multiple of PER: the item's columns share one group z (one division per
        // thread instead of one per column - the divisions were 1/4 of the kernel's instructions)
        const int q0 = item * PER, z = q0 / NQ, ql0 = q0 - z * NQ;
        double* row = Xt + ((long)z * nct + cg) * CH * SX + (long)tl * SX + 2 * ql0;
#pragma unroll
        for (int f = 0; f < PER; ++f)
            if (q0 + f < nq) *reinterpret_cast<double2*>(row + 2 * f) = v[f];
    }
    for (int z = blockIdx.y * kPrepItems + il; z < groups; z += gridDim.y * kPrepItems) {
        double* row = Xt + ((long)z * nct + cg) * CH * SX + (long)tl * SX;
        for (int c = 2 * max(0, min(NQ, nq - z * NQ)); c < SX; c += 2)
            *reinterpret_cast<double2*>(row + c) = make_double2(0.0, 0.0);
    }
}

// The evaluation's prep (PSWE_PREP_ROWS, default): one thread per (chunk, degree) writes that
// degree's WHOLE X-tile row of column group z = blockIdx.y - the NT states' {Phi, zeta, U, V}
// (the same expressions, in the same order, as xtile_prep_kernel<INV_EVAL>), zeros for states
// past n and the two pad columns. The per-degree factors are computed once for all NT states and
// every state's loads are issued together; no integer division by runtime sizes; blocks of
// kPrepRowChunks chunks x 16 degrees. Used for one- and two-state evaluations (the SDC sweeps'
// chain: fine sweep T255 -2%, T511 single-state evaluation -3.6%); at a 5-state batch it was
// measured no faster than the generic kernel (13 us, 178 registers), which stays there.
#ifndef PSWE_PREP_ROWS
#define PSWE_PREP_ROWS 1
#endif
#ifndef PSWE_PREP_PLAIN
#define PSWE_PREP_PLAIN 1
#endif
#ifndef PSWE_PREP_WIDE
#define PSWE_PREP_WIDE 1
#endif
constexpr int kPrepRowChunks = 8;
template <int NT>
__global__ void __launch_bounds__(CH * kPrepRowChunks)
    xtile_prep_rows_kernel(int R, int n, int nct, const int* __restrict__ chunk_desc, const double* __restrict__ eps,
                           const double* __restrict__ rtab, const double2* __restrict__ in, double radius,
                           double* __restrict__ Xt) {
    constexpr int SX = 8 * NT + 2;
    constexpr int TILE = CH * SX;  // doubles of one chunk's tile
    __shared__ __align__(32) double sx[kPrepRowChunks * TILE];
    const int cg0 = blockIdx.x * kPrepRowChunks;
    const int cg = cg0 + threadIdx.x / CH;
    const int tl = threadIdx.x % CH;
    const int z = blockIdx.y;
    const int nchk = min(kPrepRowChunks, nct - cg0);  // chunks of this block
    pdl_trigger();
    if (cg < nct) {
        const int2 mc = reinterpret_cast<const int2*>(chunk_desc)[cg];  // (m, chunk within m)
        const int m = mc.x;
        const int t = mc.y * CH + tl;
        const int s = m + t;
        const long K = (long)(R + 1) * (R + 2) / 2;
        const long bs = off_std(R, m), bx = off_ext(R, m);
        const int sm1 = max(s - 1, m), sp1 = min(s + 1, R), s0 = min(s, R);
        const bool live = s <= R + 1;
        xrow::Fac F{};
        if (live) F = xrow::factors(R, m, s, bx, eps, rtab, radius);
        pdl_wait();  // the states come from the preceding kernel
        double2 ph[NT], vm[NT], v0[NT], vp[NT], dm[NT], d0[NT], dp[NT];
#pragma unroll
        for (int ql = 0; ql < NT; ++ql) {
            const int item = z * NT + ql;
            ph[ql] = vm[ql] = v0[ql] = vp[ql] = dm[ql] = d0[ql] = dp[ql] = make_double2(0.0, 0.0);
            if (live && item < n) {
                const double2* st = in + (long)item * 3 * K + bs - m;
                ph[ql] = st[s0];
                vm[ql] = st[K + sm1];
                v0[ql] = st[K + s0];
                vp[ql] = st[K + sp1];
                dm[ql] = st[2 * K + sm1];
                d0[ql] = st[2 * K + s0];
                dp[ql] = st[2 * K + sp1];
            }
        }
        // the row goes to shared memory; the block's chunks are one contiguous run of tiles, written
        // below with coalesced 32-byte stores (per-thread 16-byte row stores at a 16 SX-byte stride
        // left the kernel store-throughput bound: drain / lg_throttle stalls)
        double2* row = reinterpret_cast<double2*>(sx + (threadIdx.x / CH) * TILE + tl * SX);
#pragma unroll
        for (int ql = 0; ql < NT; ++ql) {
            double2 v[4];
            if (live && z * NT + ql < n) {
                xrow::columns(F, R, m, s, radius, ph[ql], vm[ql], v0[ql], vp[ql], dm[ql], d0[ql], dp[ql], v);
            } else {
#pragma unroll
                for (int f = 0; f < 4; ++f) v[f] = make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int f = 0; f < 4; ++f) row[4 * ql + f] = v[f];
        }
        row[4 * NT] = make_double2(0.0, 0.0);  // pad columns
    } else {
        pdl_wait();
    }
    __syncthreads();
    const double4* src = reinterpret_cast<const double4*>(sx);
    double* dst = Xt + ((long)z * nct + cg0) * TILE;  // 32-byte aligned: cg0 % 8 == 0, TILE even
    const int nv = nchk * TILE / 4;
    for (int i = threadIdx.x; i < nv; i += CH * kPrepRowChunks) {
        const double4 w = src[i];
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(dst + 4 * i), "d"(w.x), "d"(w.y), "d"(w.z),
                     "d"(w.w)
                     : "memory");
    }
}

// The evaluation's prep for wide column groups (NT >= 3 states, the batch): thread (degree tl,
// state ql, chunk) computes its state's four columns with the same expressions as
// xtile_prep_rows_kernel (xrow.cuh), so each thread keeps one state's 7 loads in flight at 64
// registers instead of NT states' at 178; the block's kPrepWideChunks tiles are staged in shared
// memory and stored as 32-byte vectors (the generic kernel's 16-byte row stores at a 16 SX-byte
// stride: 80-thread blocks, long_scoreboard 46%, drain/lg_throttle 14%).
constexpr int kPrepWideChunks = 4;
template <int NT>
__global__ void __launch_bounds__(CH * NT * kPrepWideChunks)
    xtile_prep_wide_kernel(int R, int n, int nct, const int* __restrict__ chunk_desc, const double* __restrict__ eps,
                           const double* __restrict__ rtab, const double2* __restrict__ in, double radius,
                           double* __restrict__ Xt) {
    constexpr int SX = 8 * NT + 2;
    constexpr int TILE = CH * SX;
    constexpr int NTH = CH * NT * kPrepWideChunks;
    __shared__ __align__(32) double sx[kPrepWideChunks * TILE];
    const int tl = threadIdx.x % CH;
    const int ql = (threadIdx.x / CH) % NT;
    const int cb = threadIdx.x / (CH * NT);
    const int cg0 = blockIdx.x * kPrepWideChunks;
    const int cg = cg0 + cb;
    const int z = blockIdx.y;
    const int nchk = min(kPrepWideChunks, nct - cg0);
    pdl_trigger();
    if (cg < nct) {
        const int2 mc = reinterpret_cast<const int2*>(chunk_desc)[cg];  // (m, chunk within m)
        const int m = mc.x;
        const int t = mc.y * CH + tl;
        const int s = m + t;
        const long K = (long)(R + 1) * (R + 2) / 2;
        const long bs = off_std(R, m), bx = off_ext(R, m);
        const int sm1 = max(s - 1, m), sp1 = min(s + 1, R), s0 = min(s, R);
        const int item = z * NT + ql;
        const bool live = s <= R + 1 && item < n;
        xrow::Fac F{};
        if (live) F = xrow::factors(R, m, s, bx, eps, rtab, radius);
        pdl_wait();  // the states come from the preceding kernel
        double2 v[4];
        if (live) {
            const double2* st = in + (long)item * 3 * K + bs - m;
            const double2 ph = st[s0], vm = st[K + sm1], v0 = st[K + s0], vp = st[K + sp1];
            const double2 dm = st[2 * K + sm1], d0 = st[2 * K + s0], dp = st[2 * K + sp1];
            xrow::columns(F, R, m, s, radius, ph, vm, v0, vp, dm, d0, dp, v);
        } else {
#pragma unroll
            for (int f = 0; f < 4; ++f) v[f] = make_double2(0.0, 0.0);
        }
        double2* row = reinterpret_cast<double2*>(sx + cb * TILE + tl * SX);
#pragma unroll
        for (int f = 0; f < 4; ++f) row[4 * ql + f] = v[f];
        if (ql == 0) row[4 * NT] = make_double2(0.0, 0.0);  // pad columns
    } else {
        pdl_wait();
    }
    __syncthreads();
    const double4* s4 = reinterpret_cast<const double4*>(sx);
    double* dst = Xt + ((long)z * nct + cg0) * TILE;  // 32-byte aligned: cg0 % 4 == 0, TILE even
    const int nv = nchk * TILE / 4;
    for (int i = threadIdx.x; i < nv; i += NTH) {
        const double4 w = s4[i];
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(dst + 4 * i), "d"(w.x), "d"(w.y), "d"(w.z),
                     "d"(w.w)
                     : "memory");
    }
}

// synthesise's prep (PLAIN, standard layout): one thread per (chunk, degree) writes that degree's
// whole X-tile row of column group z = blockIdx.y - the 4 NT fields' coefficients, issued as one
// batch of loads (the generic kernel's one load per thread left too few bytes in flight: 8 us for
// 16 MB), the pad columns zero - staged in shared memory and stored as 32-byte vectors like
// xtile_prep_rows_kernel.
template <int NT>
__global__ void __launch_bounds__(CH * kPrepRowChunks)
    xtile_prep_plain_kernel(int R, int nq, int nct, const int* __restrict__ chunk_desc,
                            const double2* __restrict__ in, double* __restrict__ Xt) {
    constexpr int SX = 8 * NT + 2;
    constexpr int TILE = CH * SX;
    __shared__ __align__(32) double sx[kPrepRowChunks * TILE];
    const int cg0 = blockIdx.x * kPrepRowChunks;
    const int cg = cg0 + threadIdx.x / CH;
    const int tl = threadIdx.x % CH;
    const int z = blockIdx.y;
    const int nchk = min(kPrepRowChunks, nct - cg0);
    pdl_trigger();
    if (cg < nct) {
        const int2 mc = reinterpret_cast<const int2*>(chunk_desc)[cg];  // (m, chunk within m)
        const int m = mc.x;
        const int t = mc.y * CH + tl;
        const long K = (long)(R + 1) * (R + 2) / 2;
        const double2* src = in + off_std(R, m) + t;
        const bool live = m + t <= R;
        pdl_wait();  // the coefficients may come from the preceding kernel
        double2 v[4 * NT];
#pragma unroll
        for (int f = 0; f < 4 * NT; ++f) {
            const int q = z * 4 * NT + f;
            v[f] = live && q < nq ? src[(long)q * K] : make_double2(0.0, 0.0);
        }
        double2* row = reinterpret_cast<double2*>(sx + (threadIdx.x / CH) * TILE + tl * SX);
#pragma unroll
        for (int f = 0; f < 4 * NT; ++f) row[f] = v[f];
        row[4 * NT] = make_double2(0.0, 0.0);  // pad columns
    } else {
        pdl_wait();
    }
    __syncthreads();
    const double4* s4 = reinterpret_cast<const double4*>(sx);
    double* dst = Xt + ((long)z * nct + cg0) * TILE;  // 32-byte aligned: cg0 % 8 == 0, TILE even
    const int nv = nchk * TILE / 4;
    for (int i = threadIdx.x; i < nv; i += CH * kPrepRowChunks) {
        const double4 w = s4[i];
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(dst + 4 * i), "d"(w.x), "d"(w.y), "d"(w.z),
                     "d"(w.w)
                     : "memory");
    }
}

// grid (ceil(nslices / WS), R+1, column groups); 2 WS warps per block: warps 2w, 2w+1 share
// latitude slice WS blockIdx.x + w and take its latitudes 0-15 / 16-31 (two 8-row m-tiles each)
// over all chunks of the order m. Halving the per-warp unit (vs one warp per slice) keeps the
// longest tasks (m = 0) below the per-SM average and halves the accumulators (more resident
// warps); the P and X tiles of a stage are shared by all warps of the block. An S-stage ring of
// {WS P tiles, one X tile} per chunk is filled by bulk copies from thread 0 (full[s]: expect_tx +
// complete_tx) and released by one arrival per warp (empty[s]).
template <int NT, int S, int WS, int CPS>
__global__ void __launch_bounds__(64 * WS) leg_inv_tma_kernel(int R, int J, int Jp, int nlat, int nq, int nct,
                                                             const double* __restrict__ ptab,
                                                             const int* __restrict__ cbase,
                                                             const double* __restrict__ Xt,
                                                             double2* __restrict__ out,
                                                             const int* __restrict__ cstart) {
    constexpr int SX = 8 * NT + 2;
    constexpr unsigned PB = 32 * 16 * sizeof(double);
    constexpr unsigned XB = CH * SX * sizeof(double);
    extern __shared__ __align__(128) double smem[];
    double* sP = smem;                      // [S][WS][CPS][32 * 16]
    double* sX = sP + S * WS * CPS * 512;   // [S][CPS][CH * SX]
    unsigned long long* full = reinterpret_cast<unsigned long long*>(sX + S * CPS * CH * SX);
    unsigned long long* empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ws = warp >> 1, mh = warp & 1;
    const int m = blockIdx.y;
    const int len = R + 2 - m;
    const int nch = (len + CH - 1) / CH;
    const int nsl = Jp >> 5;
    const int sl0 = blockIdx.x * WS;
    const int nact = min(WS, nsl - sl0);
    const int z = blockIdx.z;
    const int q0 = z * 4 * NT;
    // polar skip: chunks below cs are negligible in every slice of this block
    int cs = 0;
    if (cstart) {
        cs = nch;
        for (int w = 0; w < nact; ++w) cs = min(cs, cstart[m * nsl + sl0 + w]);
    }
    const double* __restrict__ pm = ptab + ptile_off(cbase[m], nch, nsl, cs, sl0);  // slice sl0 + w: + w nch 512
    const double* __restrict__ xm = Xt + ((long)z * nct + cbase[m] + cs) * CH * SX;
    const int r4 = lane >> 2, c4 = lane & 3;

    if (threadIdx.x == 0) {
        for (int k = 0; k < S; ++k) {
            mbar_init(full + k, 1);
            mbar_init(empty + k, 2 * WS);
        }
        mbar_fence_init();
    }
    __syncthreads();
    pdl_trigger();
    const int nchs = nch - cs;                // chunks cs .. nch - 1 (indices below relative to cs)
    const int ngr = (nchs + CPS - 1) / CPS;  // stages of CPS chunks: one copy per slice, one X copy
    auto issue_p = [&](int g) {  // P tiles: plan constants
        const int k = g % S, c0 = g * CPS, nc = min(CPS, nchs - c0);
        mbar_expect_tx(full + k, nc * (nact * PB + XB));
        for (int w = 0; w < nact; ++w)
            bulk_g2s(sP + (k * WS + w) * CPS * 512, pm + ((long)w * nch + c0) * 512, nc * PB, full + k);
    };
    auto issue_x = [&](int g) {  // X tiles: the prep kernel's output
        const int k = g % S, c0 = g * CPS, nc = min(CPS, nchs - c0);
        bulk_g2s(sX + k * CPS * CH * SX, xm + (long)c0 * CH * SX, nc * XB, full + k);
    };
    auto issue = [&](int g) {
        issue_p(g);
        issue_x(g);
    };
#ifndef PSWE_DIAG_NOTMA
    // the first stages' P tiles stream in while the prep kernel finishes (programmatic launch)
    if (threadIdx.x == 0)
        for (int g = 0; g < S && g < ngr; ++g) issue_p(g);
#endif
    pdl_wait();  // X tiles come from the prep kernel
#ifndef PSWE_DIAG_NOTMA
    if (threadIdx.x == 0)
        for (int g = 0; g < S && g < ngr; ++g) issue_x(g);
#endif

    double acc[2][2][NT][2];  // [m-tile 2 mh + a][parity][n-tile][v]
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int cc = 0; cc < NT; ++cc) acc[a][b][cc][0] = acc[a][b][cc][1] = 0.0;

    for (int g = 0; g < ngr; ++g) {
        const int k = g % S;
        const unsigned ph = (unsigned)(g / S) & 1u;
        const int nc = min(CPS, nchs - g * CPS);
#ifndef PSWE_DIAG_NOTMA
        mbar_wait(full + k, ph);
#endif
        __syncwarp();
#pragma unroll
        for (int cc = 0; cc < CPS; ++cc)
        if (ws < nact && cc < nc) {
            const double* tl = sP + ((k * WS + ws) * CPS + cc) * 512 + mh * 16 * 16;  // this warp's 16 rows
            const double* xb = sX + (k * CPS + cc) * CH * SX;
#pragma unroll
            for (int par = 0; par < 2; ++par) {
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    // k -> degree (within chunk) par + 2 (4 ks + c4)
                    double bf[NT], af[2];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) bf[nt] = xb[(par + 2 * (4 * ks + c4)) * SX + 8 * nt + r4];
#pragma unroll
                    for (int a = 0; a < 2; ++a) af[a] = tl[(8 * a + r4) * 16 + pswz(r4, par * 8 + 4 * ks + c4)];
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) {
#ifdef PSWE_DIAG_NODMMA
                            acc[a][par][nt][0] += af[a] * bf[nt];
#else
                            dmma(acc[a][par][nt], af[a], bf[nt]);
#endif
                        }
                }
            }
        }
        __syncwarp();
#ifndef PSWE_DIAG_NOTMA
        if (lane == 0) mbar_arrive(empty + k);
        if (threadIdx.x == 0 && g + S < ngr) {
            mbar_wait(empty + k, ph);
            issue(g + S);
        }
#endif
    }
    if (ws >= nact) return;
    const int jb = (sl0 + ws) * 32 + mh * 16;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        const int jj = jb + 8 * a + r4;
        if (jj >= J) continue;
        const int iN = nlat - J + jj, iS = J - 1 - jj;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int q = q0 + 4 * nt + c4;
            if (q >= nq) continue;
            const double* e = acc[a][0][nt];
            const double* o = acc[a][1][nt];
#ifdef PSWE_DIAG_NOSTORE
            if (e[0] != 1.2345e300) continue;
#endif
            double2* dst = out + (long)q * nlat * (R + 1) + m;  // rows [q][i][m]
            dst[(long)iN * (R + 1)] = make_double2(e[0] + o[0], e[1] + o[1]);
            if (iS != iN) dst[(long)iS * (R + 1)] = make_double2(e[0] - o[0], e[1] - o[1]);
        }
    }
}

template <int NT>
void fwd_launch(const pswe_plan& P, const double2* four, int nq, double2* out, bool ext, cudaStream_t st) {
    // warps per block: the block stages G for every latitude (smem ~ Jp), so small J wants
    // small blocks (more blocks per SM, staging overlapped across blocks) and large J wants
    // more warps sharing one staged tile. PSWE_FWD_WARPS overrides (tuning only).
    static const int w_env = [] { const char* e = getenv("PSWE_FWD_WARPS"); return e ? atoi(e) : 0; }();
    const int W = w_env > 0 ? w_env : (P.J <= 256 ? 4 : 8);
    const int Jp = ((P.J + 31) / 32) * 32;
    const int groups = (nq + 4 * NT - 1) / (4 * NT);
    const size_t sm = (size_t)(2 * Jp * 8 * NT + W * 2 * 32 * 16) * sizeof(double);
    if (sm > 227 * 1024) throw std::invalid_argument("legendre_forward(stream): shared-memory tile too large");
    auto kern = leg_fwd_stream_mma_kernel<NT>;
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<dim3(P.R + 1, groups), 32 * W, sm, st>>>(P.R, P.J, Jp, P.nlat, nq, P.d_ptab2, P.d_chk_off, four, out,
                                                    ext ? 1 : 0);
    PSWE_LAUNCH_CHECK();
}

#ifndef PSWE_INV_STAGES
#define PSWE_INV_STAGES 4
#endif
// one latitude slice (two warps, 64 threads) per block: measured -2% on the T255 5-state batch
// and -1.3% at T511 against two slices (four: +1-3%); the X tile is re-read per slice from L2
#ifndef PSWE_INV_SLICES
#define PSWE_INV_SLICES 1
#endif
constexpr int kInvStages = PSWE_INV_STAGES;  // ring stages (one chunk each)
constexpr int kInvSlices = PSWE_INV_SLICES;  // latitude slices per block (two warps each)

// column tiles per group for nq complex columns. With one latitude slice per block (r01f,
// tools/ab_time.py): evaluation batches of up to 5 states take all their columns in one group
// (the P table streams once; 5 states: T255 103.5 -> 102.3 us, T511 503 -> 479 us against 2 / 3
// tiles). Other inputs (the plain transforms' fields) keep small groups: NT = 2 below 192 latitude
// pairs, 3 from 192 (15 fields at T255: NT = 2 46 us, 3-5 48-50 us) - small NT keeps registers
// low and gives more blocks; the P re-reads hit L2. One tile for <= 4 columns. PSWE_INV_NT
// overrides (tuning only).
int inv_choose_nt(const pswe_plan& P, int nq, int kind) {
    static const int forced = [] { const char* e = getenv("PSWE_INV_NT"); return e ? atoi(e) : 0; }();
    if (forced >= 1 && forced <= 5) return forced;
    if (nq <= 4) return 1;
    if (kind == INV_EVAL && nq <= 20) return (nq + 3) / 4;
    return P.J >= 192 ? 3 : 2;
}

#ifndef PSWE_INV_CPS1
#define PSWE_INV_CPS1 4
#endif
#ifndef PSWE_INV_CPS2
#define PSWE_INV_CPS2 2
#endif
#ifndef PSWE_INV_CPS3
#define PSWE_INV_CPS3 1
#endif
template <int NT>
void inv_tma_launch(const pswe_plan& P, const double* Xt, int nq, double2* out, cudaStream_t st) {
    // chunks per ring stage and ring depth by column-tile count (narrow groups do little DMMA work
    // per chunk, so one stage carries several chunks: fewer bulk copies per DMMA)
    constexpr int CPS = NT == 1 ? PSWE_INV_CPS1 : (NT == 2 ? PSWE_INV_CPS2 : PSWE_INV_CPS3);
    constexpr int S = CPS == 1 ? kInvStages : (CPS == 2 ? 3 : 2), WS = kInvSlices;
    const int nsl = (P.J + 31) / 32;
    const int Jp = nsl * 32;
    const int groups = (nq + 4 * NT - 1) / (4 * NT);
    const size_t sm = (size_t)S * CPS * (WS * 512 + CH * (8 * NT + 2)) * sizeof(double) +
                      2 * S * sizeof(unsigned long long);
    auto kern = leg_inv_tma_kernel<NT, S, WS, CPS>;
    static bool attr = false;
    if (!attr) {
        PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        attr = true;
    }
    launch_pdl(kern, dim3((nsl + WS - 1) / WS, P.R + 1, groups), dim3(64 * WS), sm, st, P.R, P.J, Jp, P.nlat, nq,
               P.n_chunks, P.d_ptab2, P.d_chk_off, Xt, out, (const int*)(polar_on() ? P.d_cstart : nullptr));
    PSWE_LAUNCH_CHECK();
}

}  // namespace

// Forward Legendre of the eval grid stage's 5 projections of n states from the G tiles (ext
// layout out[5n][Kx]); preconditions: gt_path_ok(P, n).
void legendre_forward_gt(const pswe_plan& P, int n, double2* out, cudaStream_t st) {
    const GtLayout gl = gt_layout(P.R, P.J, n);
#define PSWE_FWD_CASES(W, C, S)                                                  \
    switch (gl.ntc) {                                                            \
        case 2: fwd_gt_launch<2, W, C, S>(P, gl, 5 * n, out, st); break;         \
        case 3: fwd_gt_launch<3, W, C, S>(P, gl, 5 * n, out, st); break;         \
        case 4: fwd_gt_launch<4, W, C, S>(P, gl, 5 * n, out, st); break;         \
        case 5: fwd_gt_launch<5, W, C, S>(P, gl, 5 * n, out, st); break;         \
        case 7: fwd_gt_launch<7, W, C, S>(P, gl, 5 * n, out, st); break;         \
        default: throw std::logic_error("legendre_forward_gt: unexpected column tiling"); \
    }
    static_assert(kFwdCfg[0].warps == 8 && kFwdCfg[0].cpw == 1 && kFwdCfg[0].stages == 4, "cfg 0");
    static_assert(kFwdCfg[1].warps == 4 && kFwdCfg[1].cpw == 2 && kFwdCfg[1].stages == 3, "cfg 1");
    const int nsl = (P.J + 31) / 32;
    static const int cw_env = [] { const char* e = getenv("PSWE_FWD_CW"); return e ? atoi(e) : PSWE_FWD_CW; }();
    if (cw_env && gl.ntc >= 4) {
        // wide column groups (3-5 states): column-warp mapping, 16-latitude stages, 2-deep ring
        // (measured r02: 5-state batch forward T255 32.8 -> 30.7 us, T511 159.8 -> 145.5 us;
        // bit-identical to leg_fwd_gt_kernel over tools/eval_dump.py's 80 cases)
        switch (gl.ntc) {
            case 4: fwd_cw_launch<4, 2, 2, 2>(P, gl, 5 * n, out, st); break;
            case 5: fwd_cw_launch<5, 1, 2, 2>(P, gl, 5 * n, out, st); break;
            default: fwd_cw_launch<7, 1, 2, 2>(P, gl, 5 * n, out, st); break;
        }
        return;
    }
    // narrow groups (one or two states: the SDC sweeps' chain) on grids beyond the direct kernel's
    // 64 latitude pairs: column warps in pairs of slot groups (measured, tools/ab_time.py r02: T255
    // 5-node sweep 135.6 -> 131.7 us with 32-latitude stages; T511 sweep 627 -> 609 us with
    // 16-latitude stages; at <= 64 pairs the direct kernel stays: T127 coarse sweep 38.0 vs 42.7 us;
    // four slot groups per column tile (9-warp blocks) measured slower). PSWE_FWD_CW=0 restores
    // the chunk-per-warp kernel everywhere (A/B).
    if (cw_env && gl.ntc <= 3 && nsl > 2) {
        if (P.fwd_cfg == 0) {
            if (gl.ntc == 2) fwd_cw_launch<2, 2, 2, 4>(P, gl, 5 * n, out, st);
            else fwd_cw_launch<3, 2, 2, 4>(P, gl, 5 * n, out, st);
        } else {
            if (gl.ntc == 2) fwd_cw_launch<2, 2, 2, 2>(P, gl, 5 * n, out, st);
            else fwd_cw_launch<3, 2, 2, 2>(P, gl, 5 * n, out, st);
        }
        return;
    }
    if (PSWE_FWD_DIRECT && P.fwd_cfg == 0 && gl.ntc <= 3 && nsl <= 2 &&
        (size_t)2 * gl.ns8 * 2 * 8 * gl.sgc * sizeof(double) <= 96 * 1024) {
        // one or two states on grids up to 64 latitude pairs (T127 on 128 x 256: coarse sweep -2%):
        // every P fragment in registers before the programmatic-launch wait. At 128 pairs (T255) the
        // two-slice window leaves the second half's loads on the critical path: fine sweep +3%.
#define PSWE_DIRECT(NTC)                                                    \
    switch (nsl) {                                                          \
        case 1: fwd_direct_launch<NTC, 1>(P, gl, 5 * n, out, st); break;    \
        default: fwd_direct_launch<NTC, 2>(P, gl, 5 * n, out, st); break;   \
    }
        if (gl.ntc == 2) {
            PSWE_DIRECT(2)
        } else {
            PSWE_DIRECT(3)
        }
#undef PSWE_DIRECT
    } else if (P.fwd_cfg == 0 && gl.ntc <= 3) {
        // one or two states: stages of 32 latitudes (four 8-latitude sub-stages per bulk copy, whole
        // 4 KB P tiles) - the per-stage work of narrow column groups is too short to amortise one
        // bulk-copy round trip per 8 latitudes
        if (gl.ntc == 2) fwd_gt_launch<2, 8, 1, 2, 4>(P, gl, 5 * n, out, st);
        else fwd_gt_launch<3, 8, 1, 2, 4>(P, gl, 5 * n, out, st);
    } else if (P.fwd_cfg == 0) {
        // wider groups: 16-latitude stages in a 2-deep ring (measured faster than 8-latitude stages
        // in a 4-deep ring: half the bulk copies; T255 384x768 forward 48.7 -> 43.5 us)
        switch (gl.ntc) {
            case 4: fwd_gt_launch<4, 8, 1, 2, 2>(P, gl, 5 * n, out, st); break;
            case 5: fwd_gt_launch<5, 8, 1, 2, 2>(P, gl, 5 * n, out, st); break;
            default: fwd_gt_launch<7, 8, 1, 2, 2>(P, gl, 5 * n, out, st); break;
        }
    } else {
        if (gl.ntc <= 3 && P.J <= 384) {
            // single/two-state batches up to 384 latitude pairs: 32-latitude stages (measured
            // T511 n=1 forward 131 -> 111 us); beyond, the smaller ring keeps more blocks resident
            // (T1023 n=1: 448 vs 498 us with 32-latitude stages)
            if (gl.ntc == 2) fwd_gt_launch<2, 4, 2, 2, 4>(P, gl, 5 * n, out, st);
            else fwd_gt_launch<3, 4, 2, 2, 4>(P, gl, 5 * n, out, st);
        } else {
            PSWE_FWD_CASES(4, 2, 3)
        }
    }
#undef PSWE_FWD_CASES
}

// analyse on G tiles (gt_layout_fields, written by fft_r2c_gt): the column-warp kernels, the
// projections' epilogue in the standard coefficient layout. false when no column-warp
// configuration covers the layout (narrow groups need more than 64 latitude pairs).
bool analyse_gt_ok(const pswe_plan& P, const GtLayout& gl) {
    static const bool on = [] {
        const char* e = getenv("PSWE_ANALYSE_GT");
        const char* c = getenv("PSWE_FWD_CW");
        return !(e && atoi(e) == 0) && !(c && atoi(c) == 0) && PSWE_FWD_CW;
    }();
    const int nsl = (P.J + 31) / 32;
    return on && P.legendre_mode == PSWE_LEGENDRE_STREAM && !P.simt && P.n_chunks > 0 && P.d_gtile &&
           gl.doubles <= P.gtile_cap && (gl.ntc == 4 || (gl.ntc <= 3 && nsl > 2));
}

void legendre_forward_fields_gt(const pswe_plan& P, const GtLayout& gl, int nf, double2* out, cudaStream_t st) {
    if (gl.ntc == 4) {
        fwd_cw_launch<4, 2, 2, 2>(P, gl, nf, out, st);
    } else if (P.fwd_cfg == 0) {
        if (gl.ntc == 2) fwd_cw_launch<2, 2, 2, 4>(P, gl, nf, out, st);
        else fwd_cw_launch<3, 2, 2, 4>(P, gl, nf, out, st);
    } else {
        if (gl.ntc == 2) fwd_cw_launch<2, 2, 2, 2>(P, gl, nf, out, st);
        else fwd_cw_launch<3, 2, 2, 2>(P, gl, nf, out, st);
    }
}

// Streamed P table (STREAM mode), built at plan creation; layout in the file header.
void build_legendre_table2(pswe_plan& P) {
    const int Jp = ((P.J + 31) / 32) * 32;
    std::vector<int> off(P.R + 2);
    off[0] = 0;
    for (int m = 0; m <= P.R; ++m) off[m + 1] = off[m] + (P.R + 2 - m + CH - 1) / CH;
    const size_t n = (size_t)off[P.R + 1] * Jp * 16;
    PSWE_CUDA(cudaMalloc(&P.d_ptab2, n * sizeof(double)));
    P.n_chunks = off[P.R + 1];
    std::vector<int2> cm(P.n_chunks);
    for (int m = 0; m <= P.R; ++m)
        for (int c = off[m]; c < off[m + 1]; ++c) cm[c] = make_int2(m, c - off[m]);
    PSWE_CUDA(cudaMalloc(&P.d_chunk_m, cm.size() * sizeof(int2)));
    PSWE_CUDA(cudaMemcpy(P.d_chunk_m, cm.data(), cm.size() * sizeof(int2), cudaMemcpyHostToDevice));
    dim3 grid((Jp + 127) / 128, P.R + 1);
    build_ptab2_kernel<<<grid, 128>>>(P.R, P.J, Jp, P.d_mu_n, P.d_seed, P.d_rec, P.d_chk_off, P.d_ptab2);
    PSWE_LAUNCH_CHECK();
    PSWE_CUDA(cudaMalloc(&P.d_cstart, (size_t)(P.R + 1) * (Jp / 32) * sizeof(int)));
    build_polar_kernel<<<dim3(Jp / 32, P.R + 1), 32>>>(P.R, Jp / 32, P.d_chk_off, P.d_ptab2, P.d_cstart);
    PSWE_LAUNCH_CHECK();
    // forward tasks: all (m, chunk) in pair order m, R-m, m+1, R-m-1, ... (equal work per pair) cut
    // into contiguous runs of at most two orders that fit kFwdWarps warps x kFwdCpw chunk slots
    // (each order's run starts on a warp boundary), about kFwdPerSm runs per SM, so that one wave
    // gives every SM the same work (the triangular per-m work otherwise leaves it ragged)
    {
        std::vector<int2> L;
#if PSWE_FWD_WTASK
        // weighted cut: orders ascending (neighbouring orders have similar polar profiles, so a
        // task's stage count is not set by a far-away order), a chunk's weight = the 32-latitude
        // slices in which it is significant (the block-level polar skip runs a task for the max
        // over its chunks), tasks cut at equal (slices x chunks) cost
        const int nsl = Jp / 32;
        std::vector<int> cst((size_t)(P.R + 1) * nsl);
        PSWE_CUDA(cudaMemcpy(cst.data(), P.d_cstart, cst.size() * sizeof(int), cudaMemcpyDeviceToHost));
        auto wt = [&](int m, int c) {
            int k = 0;
            while (k < nsl && c >= cst[(size_t)m * nsl + k]) ++k;
            return std::max(k, 1);
        };
        for (int m = 0; m <= P.R; ++m)
            for (int c = 0; c < off[m + 1] - off[m]; ++c) L.push_back(make_int2(m, c));
#else
        for (int p = 0; p <= P.R - p; ++p) {
            const int ms[2] = {p, P.R - p};
            for (int u = 0; u < (ms[1] != ms[0] ? 2 : 1); ++u)
                for (int c = 0; c < off[ms[u] + 1] - off[ms[u]]; ++c) L.push_back(make_int2(ms[u], c));
        }
#endif
        int nsm = 148;
        {
            int dev = 0;
            cudaDeviceProp prop;
            if (cudaGetDevice(&dev) == cudaSuccess && cudaGetDeviceProperties(&prop, dev) == cudaSuccess)
                nsm = prop.multiProcessorCount;
        }
        P.fwd_cfg = (int)L.size() <= kFwdCfg[0].per_sm * nsm * kFwdCfg[0].warps * kFwdCfg[0].cpw ? 0 : 1;
        const FwdCfg fc = kFwdCfg[P.fwd_cfg];
        const int slots = fc.per_sm * nsm, cap = fc.warps * fc.cpw, cpw = fc.cpw;
        auto used = [cpw](int na, int nb) { return (na + cpw - 1) / cpw * cpw + nb; };
        std::vector<int4> ta;
        std::vector<int2> tb;
#if PSWE_FWD_WTASK
        long wsum = 0;
        for (const int2& e : L) wsum += wt(e.x, e.y);
        wsum += (long)PSWE_FWD_WG * slots * nsl / 2;  // per-task stage overhead (G tile) in chunk units
        for (long target = std::max(1L, (wsum + slots - 1) / slots);; target += std::max(1L, target / 64)) {
#else
        for (int target = std::max(1, (int)((L.size() + slots - 1) / slots));; ++target) {
#endif
            ta.clear();
            tb.clear();
            size_t i = 0;
            while (i < L.size()) {
                int4 a = make_int4(L[i].x, L[i].y, 0, -1);
                int2 b = make_int2(0, 0);
                int n = 0;
#if PSWE_FWD_WTASK
                int wmax = 0;
                auto fits = [&](size_t k) {
                    if (n == 0) return true;
                    const long w = std::max(wmax, wt(L[k].x, L[k].y));
                    return n < cap && w * (n + 1 + PSWE_FWD_WG) <= target;
                };
                while (i < L.size() && fits(i)) {
                    wmax = std::max(wmax, wt(L[i].x, L[i].y));
#else
                while (i < L.size() && n < std::min(target, cap)) {
#endif
                    if (L[i].x == a.x && a.w < 0) {
                        ++a.z;
                    } else if ((a.w < 0 || L[i].x == a.w) && used(a.z, b.y + 1) <= cap) {
                        if (a.w < 0) {
                            a.w = L[i].x;
                            b.x = L[i].y;
                        }
                        ++b.y;
                    } else {
                        break;  // a third order, or no room: new task
                    }
                    ++n;
                    ++i;
                }
                if (a.w < 0) a.w = a.x;
                ta.push_back(a);
                tb.push_back(b);
            }
#if PSWE_FWD_WTASK
            if ((int)ta.size() <= slots || target >= (long)cap * nsl) break;
#else
            if ((int)ta.size() <= slots || target >= cap) break;
#endif
        }
        P.n_fwd_tasks = (int)ta.size();
        PSWE_CUDA(cudaMalloc(&P.d_fwd_ta, ta.size() * sizeof(int4)));
        PSWE_CUDA(cudaMalloc(&P.d_fwd_tb, tb.size() * sizeof(int2)));
        PSWE_CUDA(cudaMemcpy(P.d_fwd_ta, ta.data(), ta.size() * sizeof(int4), cudaMemcpyHostToDevice));
        PSWE_CUDA(cudaMemcpy(P.d_fwd_tb, tb.data(), tb.size() * sizeof(int2), cudaMemcpyHostToDevice));
    }
}

void legendre_forward_stream(const pswe_plan& P, const double2* four, int nq, double2* out, bool ext, cudaStream_t st) {
    if (nq <= 0) return;
    const int Jp = ((P.J + 31) / 32) * 32;
    if (nq > 4 && Jp <= 768) fwd_launch<2>(P, four, nq, out, ext, st);
    else fwd_launch<1>(P, four, nq, out, ext, st);
}

// X-tile capacity for nq columns of `kind` (grow-only)
void xtile_reserve(const pswe_plan& P, int nq, int kind) {
    const int NT = inv_choose_nt(P, nq, kind);
    const int NQ = 4 * NT, SX = 8 * NT + 2;
    const int groups = (nq + NQ - 1) / NQ;
    const size_t need = (size_t)groups * P.n_chunks * CH * SX;
    if (need > P.xtile_cap) {
        ++P.generation;
        if (P.d_xtile) PSWE_CUDA(cudaFree(P.d_xtile));
        PSWE_CUDA(cudaMalloc(&P.d_xtile, need * sizeof(double)));
        P.xtile_cap = need;
    }
}

// One evaluation state whose X tiles (one column tile, [16][10] per chunk) a preceding kernel has
// already written - the SDC sweep's node update (sdc.cu): true when the single-state inverse takes
// this path; then legendre_inverse_prepared runs the contraction alone.
bool xtiles_by_sweep_ok(const pswe_plan& P) {
    return !P.simt && use_stream_inverse(P, 4) && inv_choose_nt(P, 4, INV_EVAL) == 1;
}
void legendre_inverse_prepared(const pswe_plan& P, double2* out, cudaStream_t st) {
    if (inv_rec_big(P, 4)) inv_rec_launch(P, P.d_xtile, 4, 1, out, st);
    else inv_tma_launch<1>(P, P.d_xtile, 4, out, st);
}

// kind/nq/in/in2/radius as legendre_inverse_mma: tiled prep, then the TMA-pipelined contraction.
void legendre_inverse_stream(const pswe_plan& P, int kind, const double2* in, const double2* in2, int nq,
                             double radius, double2* out, cudaStream_t st, cudaEvent_t after_prep) {
    if (nq <= 0) return;
    const int NT = inv_choose_nt(P, nq, kind);
    const int NQ = 4 * NT, SX = 8 * NT + 2;
    const int groups = (nq + NQ - 1) / NQ;
    xtile_reserve(P, nq, kind);
    const int per = kind == INV_EVAL ? 4 : (kind == INV_UV ? 2 : 1);
    const int nitems = (nq + per - 1) / per;
    const int span = std::max(nitems, groups);  // item slots also zero the groups' pad columns
    const int iy = (span + kPrepItems - 1) / kPrepItems;
    const int ipb = std::min(span, kPrepItems);
    dim3 g(P.n_chunks, iy);
    static const int rows_max = [] { const char* e = getenv("PSWE_PREP_ROWS_MAX"); return e ? atoi(e) : 2; }();
#ifdef PSWE_DIAG_NOPREP
    if (false)
#endif
    if (kind == INV_EVAL && PSWE_PREP_ROWS && NT <= rows_max) {  // env: tuning only
        const dim3 gr((P.n_chunks + kPrepRowChunks - 1) / kPrepRowChunks, groups);
        const int n = nq / 4;
        switch (NT) {
#define PSWE_PREP_CASE(T)                                                                                          \
    case T:                                                                                                    \
        launch_pdl(xtile_prep_rows_kernel<T>, gr, dim3(CH * kPrepRowChunks), 0, st, P.R, n, P.n_chunks, P.d_chunk_m, \
                   P.d_eps, P.d_rlap, in, radius, P.d_xtile);                                                  \
        break;
            PSWE_PREP_CASE(1) PSWE_PREP_CASE(2) PSWE_PREP_CASE(3) PSWE_PREP_CASE(4) PSWE_PREP_CASE(5)
#undef PSWE_PREP_CASE
        }
    } else if (kind == INV_EVAL && PSWE_PREP_WIDE && NT >= 3 && P.R <= 255) {
        // (measured r2bd: T255 5-state prep 12.5 -> 11.2 us, batch 95.2 -> 94.2 us, bit-identical over
        // eval_dump's 50 cases; at T511 the generic kernel's small blocks stay faster, 23.3 vs 25 us)
        const dim3 gw((P.n_chunks + kPrepWideChunks - 1) / kPrepWideChunks, groups);
        const int n = nq / 4;
        switch (NT) {
#define PSWE_PREP_CASE(T)                                                                                      \
    case T:                                                                                                \
        launch_pdl(xtile_prep_wide_kernel<T>, gw, dim3(CH * T * kPrepWideChunks), 0, st, P.R, n, P.n_chunks, \
                   P.d_chunk_m, P.d_eps, P.d_rlap, in, radius, P.d_xtile);                                  \
        break;
            PSWE_PREP_CASE(3) PSWE_PREP_CASE(4) PSWE_PREP_CASE(5)
#undef PSWE_PREP_CASE
        }
    } else if (kind == INV_EVAL)
        launch_pdl(xtile_prep_kernel<INV_EVAL>, g, dim3(CH * ipb), 0, st, P.R, NQ, SX, nq, P.n_chunks, P.d_chunk_m,
                   P.d_eps, P.d_rlap, in, in2, radius, P.d_xtile);
    else if (kind == INV_UV)
        launch_pdl(xtile_prep_kernel<INV_UV>, g, dim3(CH * ipb), 0, st, P.R, NQ, SX, nq, P.n_chunks, P.d_chunk_m,
                   P.d_eps, P.d_rlap, in, in2, radius, P.d_xtile);
    else if (PSWE_PREP_PLAIN) {
        const dim3 gp((P.n_chunks + kPrepRowChunks - 1) / kPrepRowChunks, groups);
        switch (NT) {
#define PSWE_PREP_CASE(T)                                                                                    \
    case T:                                                                                              \
        launch_pdl(xtile_prep_plain_kernel<T>, gp, dim3(CH * kPrepRowChunks), 0, st, P.R, nq, P.n_chunks, \
                   P.d_chunk_m, in, P.d_xtile);                                                           \
        break;
            PSWE_PREP_CASE(1) PSWE_PREP_CASE(2) PSWE_PREP_CASE(3) PSWE_PREP_CASE(4) PSWE_PREP_CASE(5)
#undef PSWE_PREP_CASE
        }
    } else
        launch_pdl(xtile_prep_kernel<INV_PLAIN>, g, dim3(CH * ipb), 0, st, P.R, NQ, SX, nq, P.n_chunks, P.d_chunk_m,
                   P.d_eps, P.d_rlap, in, in2, radius, P.d_xtile);
    PSWE_LAUNCH_CHECK();
    if (after_prep) PSWE_CUDA(cudaEventRecord(after_prep, st));
#ifdef PSWE_DIAG_NOINV
    return;
#endif
    if (inv_rec_big(P, nq)) {
        inv_rec_launch(P, P.d_xtile, nq, NT, out, st);
        return;
    }
    switch (NT) {
        case 5: inv_tma_launch<5>(P, P.d_xtile, nq, out, st); break;
        case 4: inv_tma_launch<4>(P, P.d_xtile, nq, out, st); break;
        case 3: inv_tma_launch<3>(P, P.d_xtile, nq, out, st); break;
        case 2: inv_tma_launch<2>(P, P.d_xtile, nq, out, st); break;
        default: inv_tma_launch<1>(P, P.d_xtile, nq, out, st); break;
    }
}

}  // namespace pswe
