// Legendre contractions on DMMA with the associated-Legendre values STREAMED from a per-plan
// table (PSWE_LEGENDRE_STREAM; sm_100a, fp64). Same mathematics as legendre_mma.cu; the P tiles
// arrive by cp.async instead of being recomputed, which removes the serial recurrence chains
// and the checkpoint loads from the contraction kernels.
//
// Table layout (built once per plan by the same recurrence, legendre.cpp:30-37):
//   ptab[(cbase(m) + c) * J * 16 + j * 16 + par * 8 + i] = P^m_{m + 16c + par + 2i}(mu_j)
// i.e. per m, per 16-degree chunk c, per latitude j: the 8 even then the 8 odd degrees. A
// (chunk, 32-latitude slice) tile is one contiguous 4 KB block. Degrees past R+1 are zero.
//
// forward  Y^T[col][t] = sum_j G_par^T[col][j] P[j][t]:  A = G^T (smem, swizzled), B = P tile
// inverse  E/O[j][col]  = sum_t P[j][t] X[t][col]:         A = P tile, B = X (smem)
// P tile in smem: [32 latitudes][20] (8 even, 8 odd, 4 pad): both fragment patterns hit two
// conflict-free wavefronts (row stride = 4 mod 16 doubles).
#include <cmath>
#include <cstdlib>

#include "legendre_common.cuh"

namespace pswe {

namespace {

constexpr int CH = 16;
constexpr int ST = 20;  // smem P-tile row stride (doubles)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
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

// copy one (chunk, slice) tile: 32 rows x 128 B -> smem [32][ST]; 8 x 16 B per lane
__device__ __forceinline__ void load_tile(double* dst, const double* __restrict__ src, int lane) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int idx = u * 32 + lane;  // 256 16-byte pieces
        const int row = idx >> 3, piece = idx & 7;
        cp_async16(dst + row * ST + 2 * piece, src + row * 16 + 2 * piece);
    }
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
    double* out = ptab + (long)cbase[m] * Jp * 16 + (long)j * 16;
    if (j >= J) {
        for (int c = 0; c < nch; ++c)
            for (int i = 0; i < 16; ++i) out[(long)c * Jp * 16 + i] = 0.0;
        return;
    }
    const double mu = mu_n[j];
    const double2* rc = rec + off_ext(R, m);
    double p = seed[(long)m * J + j], pm1 = 0.0;
    for (int t = 0; t < nch * CH; ++t) {
        const int c = t / CH, tl = t % CH;
        out[(long)c * Jp * 16 + (tl & 1) * 8 + (tl >> 1)] = t < len ? p : 0.0;
        if (t < len) {
            const double pn = rec_step(__ldg(rc + t), mu, p, pm1);
            pm1 = p;
            p = pn;
        }
    }
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
    double* tiles = smem + 2 * Jp * SG + warp * (2 * 32 * ST);  // [2][32][ST] per warp
    const int q0 = blockIdx.y * 4 * NT;
    const int tmax = ext ? len : len - 1;
    const long bx = off_ext(R, m);
    const long Kx = (long)(R + 1) * (R + 4) / 2, K = (long)(R + 1) * (R + 2) / 2;
    const double* __restrict__ pm = ptab + (long)cbase[m] * Jp * 16;

    // first P tile of this warp's first chunk streams in while G is staged
    if (warp < nch) {
        load_tile(tiles, pm + (long)warp * Jp * 16, lane);
        cp_async_commit();
    }
    legc::stage_g<NT, 8>(G, Jp * SG, Jp, J, nlat, R, m, q0, nq, four,
                         [](int j, int col) { return gpos<NT>(j, col); });
    __syncthreads();
    const int r4 = lane >> 2, c4 = lane & 3;
    bool first = true;

    for (int c = warp; c < nch; c += W) {
        double acc[2][NT][2];  // [par][nt]: C[col 8nt + r4][deg-in-parity 2 c4 + v]
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < NT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        const double* src = pm + (long)c * Jp * 16;
        if (!first) {  // the first task's tile was issued before the G staging
            load_tile(tiles, src, lane);
            cp_async_commit();
        }
        first = false;
        for (int sl = 0; sl < nsl; ++sl) {
            if (sl + 1 < nsl) load_tile(tiles + ((sl + 1) & 1) * 32 * ST, src + (long)(sl + 1) * 32 * 16, lane);
            cp_async_commit();
            cp_async_wait<1>();
            __syncwarp();
            const double* tl = tiles + (sl & 1) * 32 * ST;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int jk = sl * 32 + 4 * ks + c4;  // latitude of this lane's k
#pragma unroll
                for (int par = 0; par < 2; ++par) {
                    const double bf = tl[(4 * ks + c4) * ST + par * 8 + r4];  // B[k=lat][n=degree]
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        const double af = G[par * Jp * SG + gpos<NT>(jk, 8 * nt + r4)];  // A[m=col][k=lat]
                        dmma(acc[par][nt], af, bf);
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

// ---- inverse ------------------------------------------------------------------------------
// grid (ceil(nslices / W), R+1, column groups); warp = 32-latitude slice walking all chunks;
// X (prep output / input fields) staged per chunk by each warp; P tiles by cp.async.
template <bool EXT, int NT>
__global__ void __launch_bounds__(256) leg_inv_stream_mma_kernel(int R, int J, int Jp, int nlat, int nq,
                                                                 const double* __restrict__ ptab,
                                                                 const int* __restrict__ cbase,
                                                                 const double2* __restrict__ X,
                                                                 double2* __restrict__ out) {
    constexpr int SX = 8 * NT + 2;  // X tile stride (2 SX = 4 mod 16)
    constexpr int NQ = 4 * NT;
    extern __shared__ double smem[];
    const int W = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = blockIdx.y;
    const int len = R + 2 - m;
    const int nch = (len + CH - 1) / CH;
    const int sl = blockIdx.x * W + warp;
    double* tiles = smem + warp * (2 * 32 * ST + 2 * CH * SX);  // [2][32][ST] then [2][CH][SX]
    double* xs = tiles + 2 * 32 * ST;
    const int q0 = blockIdx.z * NQ;
    const long Kq = EXT ? (long)(R + 1) * (R + 4) / 2 : (long)(R + 1) * (R + 2) / 2;
    const long base = EXT ? off_ext(R, m) : off_std(R, m);
    const int tlim = EXT ? len : len - 1;
    if (sl * 32 >= Jp) return;
    const double* __restrict__ pm = ptab + (long)cbase[m] * Jp * 16 + (long)sl * 32 * 16;
    const int r4 = lane >> 2, c4 = lane & 3;

    // X chunk: 16 degrees x NQ complex columns -> xs[tl][2 ql + v], zero beyond tlim / nq
    // asynchronous (cp.async, zero-filled) so it overlaps the DMMAs of the previous chunk
    auto stage_x = [&](double* dst, int t0) {
        for (int idx = lane; idx < CH * NQ; idx += 32) {
            const int ql = idx / CH, tl = idx - ql * CH;  // degree fastest
            const int t = t0 + tl, q = q0 + ql;
            const bool v = t < tlim && q < nq;
            legc::cp_async16z(dst + tl * SX + 2 * ql, v ? (const void*)(X + (long)q * Kq + base + t) : (const void*)X, v);
        }
    };

    double acc[4][2][NT][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int cc = 0; cc < NT; ++cc) acc[a][b][cc][0] = acc[a][b][cc][1] = 0.0;

    load_tile(tiles, pm, lane);
    stage_x(xs, 0);
    cp_async_commit();
    for (int c = 0; c < nch; ++c) {
        const int b = c & 1;
        if (c + 1 < nch) {
            load_tile(tiles + (b ^ 1) * 32 * ST, pm + (long)(c + 1) * Jp * 16, lane);
            stage_x(xs + (b ^ 1) * CH * SX, (c + 1) * CH);
        }
        cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        const double* tl = tiles + b * 32 * ST;
        const double* xb = xs + b * CH * SX;
#pragma unroll
        for (int par = 0; par < 2; ++par) {
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                // k -> degree (within chunk) par + 2 (4 ks + c4)
                double bf[NT], af[4];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) bf[nt] = xb[(par + 2 * (4 * ks + c4)) * SX + 8 * nt + r4];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) af[mt] = tl[(8 * mt + r4) * ST + par * 8 + 4 * ks + c4];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][par][nt], af[mt], bf[nt]);
            }
        }
        __syncwarp();
    }
    cp_async_wait<0>();
    const int jb = sl * 32;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
        const int jj = jb + 8 * mt + r4;
        if (jj >= J) continue;
        const int iN = nlat - J + jj, iS = J - 1 - jj;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int q = q0 + 4 * nt + c4;
            if (q >= nq) continue;
            const double* e = acc[mt][0][nt];
            const double* o = acc[mt][1][nt];
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
    const size_t sm = (size_t)(2 * Jp * 8 * NT + W * 2 * 32 * ST) * sizeof(double);
    if (sm > 227 * 1024) throw std::invalid_argument("legendre_forward(stream): shared-memory tile too large");
    auto kern = leg_fwd_stream_mma_kernel<NT>;
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<dim3(P.R + 1, groups), 32 * W, sm, st>>>(P.R, P.J, Jp, P.nlat, nq, P.d_ptab2, P.d_chk_off, four, out,
                                                    ext ? 1 : 0);
    PSWE_LAUNCH_CHECK();
}

template <bool EXT, int NT>
void inv_launch(const pswe_plan& P, const double2* X, int nq, double2* out, cudaStream_t st) {
    const int nsl = (P.J + 31) / 32;
    const int Jp = nsl * 32;
    const int W = nsl < 4 ? nsl : 4;
    const int groups = (nq + 4 * NT - 1) / (4 * NT);
    const size_t sm = (size_t)W * (2 * 32 * ST + 2 * CH * (8 * NT + 2)) * sizeof(double);
    auto kern = leg_inv_stream_mma_kernel<EXT, NT>;
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<dim3((nsl + W - 1) / W, P.R + 1, groups), 32 * W, sm, st>>>(P.R, P.J, Jp, P.nlat, nq, P.d_ptab2,
                                                                       P.d_chk_off, X, out);
    PSWE_LAUNCH_CHECK();
}

template <bool EXT>
void inv_dispatch(const pswe_plan& P, const double2* X, int nq, double2* out, cudaStream_t st) {
    // cost per (chunk, slice) in shared-memory wavefronts + DMMA issue: a block of NT n-tiles
    // issues 16 NT DMMA (x16 cycles) against 16 P-fragment + 4 NT X-fragment loads (2 wavefronts
    // each, shared by the SM's 4 SMSPs), plus one P tile (32 wavefronts) per column group.
    // Measured (tools/stage_times.py): NT = 5 (one group of 20 columns: 0.45 fragment loads per
    // DMMA, 252 registers) wins for a 5-state batch once there are >= 192 latitude pairs to fill
    // the machine; otherwise the fewest padded n-tiles, then the fewest groups.
    int best = 1;
    if (nq >= 20 && nq % 20 == 0 && P.J >= 192) {
        best = 5;
    } else {
        int best_cost = 1 << 30;
        for (int nt = 4; nt >= 1; --nt) {
            const int groups = (nq + 4 * nt - 1) / (4 * nt);
            const int cost = groups * nt * 8 + groups;
            if (cost < best_cost) {
                best_cost = cost;
                best = nt;
            }
        }
    }
    switch (best) {
        case 5: inv_launch<EXT, 5>(P, X, nq, out, st); break;
        case 4: inv_launch<EXT, 4>(P, X, nq, out, st); break;
        case 3: inv_launch<EXT, 3>(P, X, nq, out, st); break;
        case 2: inv_launch<EXT, 2>(P, X, nq, out, st); break;
        default: inv_launch<EXT, 1>(P, X, nq, out, st); break;
    }
}

}  // namespace

// Streamed P table (STREAM mode), built at plan creation; layout in the file header.
void build_legendre_table2(pswe_plan& P) {
    const int Jp = ((P.J + 31) / 32) * 32;
    std::vector<int> off(P.R + 2);
    off[0] = 0;
    for (int m = 0; m <= P.R; ++m) off[m + 1] = off[m] + (P.R + 2 - m + CH - 1) / CH;
    const size_t n = (size_t)off[P.R + 1] * Jp * 16;
    PSWE_CUDA(cudaMalloc(&P.d_ptab2, n * sizeof(double)));
    dim3 grid((Jp + 127) / 128, P.R + 1);
    build_ptab2_kernel<<<grid, 128>>>(P.R, P.J, Jp, P.d_mu_n, P.d_seed, P.d_rec, P.d_chk_off, P.d_ptab2);
    PSWE_LAUNCH_CHECK();
}

void legendre_forward_stream(const pswe_plan& P, const double2* four, int nq, double2* out, bool ext, cudaStream_t st) {
    if (nq <= 0) return;
    const int Jp = ((P.J + 31) / 32) * 32;
    if (nq > 4 && Jp <= 768) fwd_launch<2>(P, four, nq, out, ext, st);
    else fwd_launch<1>(P, four, nq, out, ext, st);
}

// kind/nq as legendre_inverse_mma; X = prep output (UV/EVAL, ext layout) or input fields (PLAIN)
void legendre_inverse_stream(const pswe_plan& P, bool ext_layout, const double2* X, int nq, double2* out,
                             cudaStream_t st) {
    if (nq <= 0) return;
    if (ext_layout) inv_dispatch<true>(P, X, nq, out, st);
    else inv_dispatch<false>(P, X, nq, out, st);
}

}  // namespace pswe
