// Legendre contractions on the FP64 tensor cores (DMMA, mma.sync.aligned.m8n8k4 .f64) with
// associated-Legendre values recomputed on the fly (sm_100a; tcgen05 has no f64 kind).
//
// Both directions are, per zonal wavenumber m, small dense GEMMs over the columns of a batch
// (columns = fields x states x {re, im}; P is real, so complex coefficients split into two real
// columns and every state of the batch shares one P tile):
//   inverse  (synthesise / uv_from_vortdiv, transform.cpp:155-223):
//       E[j][c] = sum_{t even} P[j][t] X[t][c],   O[j][c] = sum_{t odd} P[j][t] X[t][c],
//       G(mu_j) = E + O, G(-mu_j) = E - O          (M = latitudes, K = degrees)
//   forward  (analyse / vortdiv_from_uv, transform.cpp:136-153,225-270):
//       Y[t][c] = sum_j P[j][t] (G_N[j][c] +- G_S[j][c]),  + for t even, - for t odd
//                                                  (M = degrees, K = latitudes)
// with t = s - m. P tiles: a warp owns 32 latitudes (lane = latitude) and advances their
// normalised 3-term recurrences (legendre.cpp:30-37) 16 degrees at a time into a padded shared
// tile from which the m8n8k4 A fragments are read. Inverse: a warp walks all degrees of its
// latitude slice. Forward: a warp owns 16-degree chunks and restarts the recurrence for every
// latitude slice from a per-plan checkpoint table (P_t, P_{t-1} at t = 16c), so chunks are
// independent and no cross-warp reduction is needed.
// Fragment layouts (CuTe SM80_8x4 / SM80_8x8_Row): A[m = lane>>2][k = lane&3],
// B[k = lane&3][n = lane>>2], C[m = lane>>2][n = 2(lane&3) + v]. Tile strides make every
// fragment load two conflict-free shared-memory wavefronts.
#include "legendre_common.cuh"

#include <cstdlib>

namespace pswe {

namespace {

constexpr int CH = 16;  // degrees per chunk
constexpr int XC = 64;  // inverse: degrees per staged coefficient super-chunk

using legc::dmma;
using legc::hcoef;
using legc::inv_lap_at;

// (m, t) of extended index kx (t = s - m, s = m..R+1)
__device__ __forceinline__ void decode_ext(int R, long kx, int& m, int& t) {
    const double b = 2.0 * R + 5.0;
    int mm = (int)floor((b - sqrt(b * b - 8.0 * (double)kx)) * 0.5);
    if (mm < 0) mm = 0;
    if (mm > R) mm = R;
    while (mm > 0 && off_ext(R, mm) > kx) --mm;
    while (mm < R && off_ext(R, mm + 1) <= kx) ++mm;
    m = mm;
    t = (int)(kx - off_ext(R, mm));
}

// Prep: inverse coefficients in the extended layout X[q][Kx], q = 4*state + {Phi, zeta, U, V}
// (EVAL) or 2*pair + {U, V} (UV); U_t = (i m chi_t - c^psi_t)/a, V_t = (i m psi_t + c^chi_t)/a
// (transform.cpp:204-206 with the H-sums rewritten as P-sums).
template <int KIND>
__global__ void inv_prep_kernel(int R, const double* __restrict__ eps, const double2* __restrict__ in,
                                const double2* __restrict__ in2, double radius, double2* __restrict__ X) {
    const long K = (long)(R + 1) * (R + 2) / 2, Kx = (long)(R + 1) * (R + 4) / 2;
    const long kx = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (kx >= Kx) return;
    int m, t;
    decode_ext(R, kx, m, t);
    const int s = m + t;
    const long bs = off_std(R, m), bx = off_ext(R, m);
    const double a2 = radius * radius, inv_a = 1.0 / radius;
    const double2 *vort, *div;
    double2* out;
    if (KIND == INV_EVAL) {
        const double2* st = in + (long)b * 3 * K;
        vort = st + K;
        div = st + 2 * K;
        out = X + (long)b * 4 * Kx;
        out[kx] = (s <= R) ? st[bs + t] : make_double2(0.0, 0.0);
        out[Kx + kx] = (s <= R) ? vort[bs + t] : make_double2(0.0, 0.0);
        out += 2 * Kx;
    } else {
        vort = in + (long)b * K;
        div = in2 + (long)b * K;
        out = X + (long)b * 2 * Kx;
    }
    const double2 chi = inv_lap_at(div, bs, m, R, s, a2);
    const double2 cpsi = hcoef(vort, eps, bs, bx, m, R, s, a2);
    const double2 psi = inv_lap_at(vort, bs, m, R, s, a2);
    const double2 cchi = hcoef(div, eps, bs, bx, m, R, s, a2);
    out[kx] = make_double2(inv_a * (-m * chi.y - cpsi.x), inv_a * (m * chi.x - cpsi.y));
    out[Kx + kx] = make_double2(inv_a * (-m * psi.y + cchi.x), inv_a * (m * psi.x + cchi.y));
}

// one recurrence step with explicit rounding (bit-identical in every kernel and the checkpoint
// builder): P_{t+1} = (1/eps_{t+1}) (mu P_t) - (eps_t/eps_{t+1}) P_{t-1}
__device__ __forceinline__ double rec_step(double2 ab, double mu, double p, double pm1) {
    return __fma_rn(ab.x, __dmul_rn(mu, p), -__dmul_rn(ab.y, pm1));
}

// Advance this lane's recurrence over one chunk, writing P_{t0..t0+CH-1} to tile[tl*S + lane].
template <int S>
__device__ __forceinline__ void ptile_chunk(double* __restrict__ tile, int lane, double mu, double& p, double& pm1,
                                            const double2* rc, int t0, int len) {
#pragma unroll
    for (int tl = 0; tl < CH; ++tl) {
        const int t = t0 + tl;
        const bool v = t < len;
        tile[tl * S + lane] = v ? p : 0.0;
        if (v) {
            const double pn = rec_step(rc[t], mu, p, pm1);
            pm1 = p;
            p = pn;
        }
    }
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    const int sz = valid ? 16 : 0;  // src-size 0 -> zero fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// ---- inverse -----------------------------------------------------------------------------------
// grid (ceil(nslices / W), R+1, column groups); block 32 W threads; warp = 32-latitude slice.
// X: PLAIN -> the std-layout input fields [q][K]; otherwise the prep output [q][Kx].
// NT n-tiles = 4 NT complex columns per block. Coefficients are staged 64 degrees at a time
// with cp.async into a double buffer (the next super-chunk streams in during the MMAs).
// out: Fourier rows [q][m][i].
template <bool EXT, int NT>
__global__ void __launch_bounds__(256) leg_inv_mma_kernel(int R, int J, int nlat, int nq,
                                                          const double* __restrict__ mu_n,
                                                          const double* __restrict__ seed,
                                                          const double2* __restrict__ rec,
                                                          const double2* __restrict__ X,
                                                          double2* __restrict__ out) {
    constexpr int SP = 34;          // P tile row stride (2 SP = 4 mod 16 doubles)
    constexpr int SX = 8 * NT + 2;  // coefficient tile row stride (2 SX = 4 mod 16; 16-B rows)
    constexpr int NQ = 4 * NT;
    extern __shared__ double smem[];
    const int W = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = blockIdx.y;
    const int len = R + 2 - m;
    double* xs = smem;                                            // [2][XC][SX]
    double2* rcs = reinterpret_cast<double2*>(smem + 2 * XC * SX);  // [len] recurrence coefs
    double* tile = smem + 2 * XC * SX + 2 * (R + 2) + warp * (CH * SP);  // [CH][SP] per warp

    const int q0 = blockIdx.z * NQ;
    const long Kq = EXT ? (long)(R + 1) * (R + 4) / 2 : (long)(R + 1) * (R + 2) / 2;
    const long base = EXT ? off_ext(R, m) : off_std(R, m);
    const int tlim = EXT ? len : len - 1;  // degrees present in X

    auto stage = [&](int buf, int t0) {
        double* dst = xs + buf * XC * SX;
        for (int idx = threadIdx.x; idx < XC * NQ; idx += blockDim.x) {
            const int ql = idx / XC, tl = idx - ql * XC;  // degree fastest: coalesced
            const int t = t0 + tl, q = q0 + ql;
            const bool v = t < tlim && q < nq;
            cp_async16(dst + tl * SX + 2 * ql, v ? (const void*)(X + (long)q * Kq + base + t) : (const void*)X, v);
        }
        cp_async_commit();
    };
    stage(0, 0);
    for (int t = threadIdx.x; t < len; t += blockDim.x) rcs[t] = rec[off_ext(R, m) + t];

    const int j = (blockIdx.x * W + warp) * 32 + lane;
    const bool jv = j < J;
    const double mu = jv ? mu_n[j] : 0.0;
    double p = jv ? seed[(long)m * J + j] : 0.0, pm1 = 0.0;

    double acc[4][2][NT][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int c = 0; c < NT; ++c) acc[a][b][c][0] = acc[a][b][c][1] = 0.0;

    const int r4 = lane >> 2, c4 = lane & 3;
    cp_async_wait_all();
    __syncthreads();
    int buf = 0;
    for (int s0 = 0; s0 < len; s0 += XC) {
        if (s0 + XC < len) stage(buf ^ 1, s0 + XC);  // streams in during this super-chunk's MMAs
        const double* xb = xs + buf * XC * SX;
        const int cend = min(XC, len - s0);
        for (int c0 = 0; c0 < cend; c0 += CH) {
            ptile_chunk<SP>(tile, lane, mu, p, pm1, rcs, s0 + c0, len);
            __syncwarp();
#pragma unroll
            for (int par = 0; par < 2; ++par) {
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const int tk = par + 2 * c4 + 8 * ks;
                    double bf[NT], af[4];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) bf[nt] = xb[(c0 + tk) * SX + 8 * nt + r4];
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) af[mt] = tile[tk * SP + 8 * mt + r4];
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][par][nt], af[mt], bf[nt]);
                }
            }
            __syncwarp();
        }
        cp_async_wait_all();
        __syncthreads();
        buf ^= 1;
    }
    // epilogue: lane holds latitude 8 mt + r4, complex column 4 nt + c4 (re, im)
    const int jb = (blockIdx.x * W + warp) * 32;
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
            // latitude-major rows [q][i][m]: the FFT stage then reads contiguous rows
            double2* dst = out + (long)q * nlat * (R + 1) + m;
            dst[(long)iN * (R + 1)] = make_double2(e[0] + o[0], e[1] + o[1]);
            if (iS != iN) dst[(long)iS * (R + 1)] = make_double2(e[0] - o[0], e[1] - o[1]);
        }
    }
}

// ---- forward -----------------------------------------------------------------------------------
// grid (R+1, column groups); block 32 W threads; warp w handles 16-degree chunks w, w+W, ...
// over all latitude slices, restarting the recurrence from the checkpoint table chk (the next
// slice's seeds are prefetched while the current slice's MMAs run).
// four: rows [q][m][i]; out: [q][Kx] (ext, s = m..R+1) or [q][K] (std, s = m..R).
template <int NT>
__global__ void __launch_bounds__(256) leg_fwd_mma_kernel(int R, int J, int nlat, int nq,
                                                          const double* __restrict__ mu_n,
                                                          const double2* __restrict__ chk,
                                                          const int* __restrict__ chk_off,
                                                          const double2* __restrict__ rec,
                                                          const double2* __restrict__ four,
                                                          double2* __restrict__ out, int ext) {
    constexpr int SP = 36;                   // P tile stride (4 mod 8 doubles)
    constexpr int SG = NT == 1 ? 12 : 20;    // G tile stride (4 mod 8)
    extern __shared__ double smem[];
    const int W = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nsl = (J + 31) >> 5;
    const int Jp = nsl * 32;
    const int m = blockIdx.x;
    const int len = R + 2 - m;
    double* G = smem;                                              // [2][Jp][SG]
    double* mus = G + 2 * Jp * SG;                                 // [Jp]
    double2* rcs = reinterpret_cast<double2*>(mus + Jp);           // [len]
    double* tile = mus + Jp + 2 * (R + 2) + warp * (CH * SP);      // [CH][SP] per warp

    const int q0 = blockIdx.y * 4 * NT;
    const int tmax = ext ? len : len - 1;
    const int nch = (len + CH - 1) / CH;
    const long bx = off_ext(R, m);
    const long Kx = (long)(R + 1) * (R + 4) / 2, K = (long)(R + 1) * (R + 2) / 2;

    // stage G_E = G_N + G_S and G_O = G_N - G_S (Gauss weights folded in by the FFT stage)
    legc::stage_g<NT, 8>(G, Jp * SG, Jp, J, nlat, R, m, q0, nq, four,
                         [](int j, int col) { return j * SG + col; });
    for (int jj = threadIdx.x; jj < Jp; jj += blockDim.x) mus[jj] = jj < J ? mu_n[jj] : 0.0;
    for (int t = threadIdx.x; t < len; t += blockDim.x) rcs[t] = rec[bx + t];
    __syncthreads();
    const double2* __restrict__ ck = chk + (long)chk_off[m] * J;
    const int r4 = lane >> 2, c4 = lane & 3;

    for (int c = warp; c < nch; c += W) {
        const int t0 = c * CH;
        double acc[2][NT][2];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < NT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        double2 nxt = lane < J ? ck[(long)c * J + lane] : make_double2(0.0, 0.0);
        for (int sl = 0; sl < nsl; ++sl) {
            const double2 cur = nxt;
            const int jn = (sl + 1) * 32 + lane;
            if (sl + 1 < nsl) nxt = jn < J ? ck[(long)c * J + jn] : make_double2(0.0, 0.0);
            double p = cur.x, pm1 = cur.y;
            ptile_chunk<SP>(tile, lane, mus[sl * 32 + lane], p, pm1, rcs, t0, len);
            __syncwarp();
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int jk = sl * 32 + 4 * ks + c4;
#pragma unroll
                for (int par = 0; par < 2; ++par) {
                    const double af = tile[(par + 2 * r4) * SP + 4 * ks + c4];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        const double bf = G[(par * Jp + jk) * SG + 8 * nt + r4];
                        dmma(acc[par][nt], af, bf);
                    }
                }
            }
            __syncwarp();
        }
        // lane holds degree t0 + par + 2 r4, complex column 4 nt + c4 (re, im)
#pragma unroll
        for (int par = 0; par < 2; ++par) {
            const int t = t0 + par + 2 * r4;
            if (t >= tmax) continue;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int q = q0 + 4 * nt + c4;
                if (q >= nq) continue;
                const double2 v = make_double2(acc[par][nt][0], acc[par][nt][1]);
                if (ext) out[(long)q * Kx + bx + t] = v;
                else out[(long)q * K + off_std(R, m) + t] = v;
            }
        }
    }
}

template <bool EXT, int NT>
void launch_inv(const pswe_plan& P, const double2* X, int nq, double2* out, cudaStream_t st) {
    const int nsl = (P.J + 31) / 32;
    const int W = nsl < 8 ? nsl : 8;
    const int groups = (nq + 4 * NT - 1) / (4 * NT);
    dim3 grid((nsl + W - 1) / W, P.R + 1, groups);
    const size_t sm = (size_t)(2 * XC * (8 * NT + 2) + 2 * (P.R + 2) + W * CH * 34) * sizeof(double);
    auto kern = leg_inv_mma_kernel<EXT, NT>;
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<grid, 32 * W, sm, st>>>(P.R, P.J, P.nlat, nq, P.d_mu_n, P.d_seed, P.d_rec, X, out);
    PSWE_LAUNCH_CHECK();
}

template <bool EXT>
void dispatch_inv(const pswe_plan& P, const double2* X, int nq, double2* out, cudaStream_t st) {
    // n-tiles per block (4 complex columns each): fewest padded tiles, then fewest groups
    int best = 1, best_cost = 1 << 30;
    for (int nt = 4; nt >= 1; --nt) {
        const int groups = (nq + 4 * nt - 1) / (4 * nt);
        const int cost = groups * nt * 4 + groups;  // padded tiles dominate, recurrences break ties
        if (cost < best_cost) {
            best_cost = cost;
            best = nt;
        }
    }
    switch (best) {
        case 4: launch_inv<EXT, 4>(P, X, nq, out, st); break;
        case 3: launch_inv<EXT, 3>(P, X, nq, out, st); break;
        case 2: launch_inv<EXT, 2>(P, X, nq, out, st); break;
        default: launch_inv<EXT, 1>(P, X, nq, out, st); break;
    }
}

template <int NT>
void launch_fwd(const pswe_plan& P, const double2* four, int nq, double2* out, bool ext, cudaStream_t st) {
    const int W = 8;
    const int nsl = (P.J + 31) / 32;
    const int groups = (nq + 4 * NT - 1) / (4 * NT);
    const int SG = NT == 1 ? 12 : 20;
    const size_t sm = (size_t)(2 * nsl * 32 * SG + nsl * 32 + 2 * (P.R + 2) + W * CH * 36) * sizeof(double);
    if (sm > 227 * 1024) throw std::invalid_argument("legendre_forward: shared-memory tile too large");
    auto kern = leg_fwd_mma_kernel<NT>;
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<dim3(P.R + 1, groups), 32 * W, sm, st>>>(P.R, P.J, P.nlat, nq, P.d_mu_n, P.d_chk, P.d_chk_off, P.d_rec,
                                                    four, out, ext ? 1 : 0);
    PSWE_LAUNCH_CHECK();
}

// checkpoint builder: (P_t, P_{t-1}) at t = 16 c for every (m, c, j)
__global__ void build_chk_kernel(int R, int J, const double* __restrict__ mu_n, const double* __restrict__ seed,
                                 const double2* __restrict__ rec, const int* __restrict__ chk_off,
                                 double2* __restrict__ chk) {
    const int m = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= J) return;
    const double mu = mu_n[j];
    const int len = R + 2 - m;
    const double2* rc = rec + off_ext(R, m);
    double2* out = chk + (long)chk_off[m] * J + j;
    double p = seed[(long)m * J + j], pm1 = 0.0;
    for (int t = 0; t < len; ++t) {
        if (t % CH == 0) out[(long)(t / CH) * J] = make_double2(p, pm1);
        const double pn = rec_step(__ldg(rc + t), mu, p, pm1);
        pm1 = p;
        p = pn;
    }
}

}  // namespace

// Checkpoint table of the forward DMMA kernel (called at plan creation).
void build_legendre_checkpoints(pswe_plan& P) {
    std::vector<int> off(P.R + 2);
    off[0] = 0;
    for (int m = 0; m <= P.R; ++m) off[m + 1] = off[m] + (P.R + 2 - m + CH - 1) / CH;
    PSWE_CUDA(cudaMalloc(&P.d_chk_off, off.size() * sizeof(int)));
    PSWE_CUDA(cudaMemcpy(P.d_chk_off, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice));
    PSWE_CUDA(cudaMalloc(&P.d_chk, (size_t)off[P.R + 1] * P.J * sizeof(double2)));
    dim3 grid((P.J + 127) / 128, P.R + 1);
    build_chk_kernel<<<grid, 128>>>(P.R, P.J, P.d_mu_n, P.d_seed, P.d_rec, P.d_chk_off, P.d_chk);
    PSWE_LAUNCH_CHECK();
}

// Streamed (TMA) inverse or the recurrence inverse. Measured (tools/stage_times.py): streamed wins
// for every batch up to 384 latitude pairs and for batched columns (nq > 4) at every size
// (T1023 n=5: 1029 vs 1580 us); the recurrence only for single states on the largest grids (T1023
// n=1: 330 vs 383 us). PSWE_STREAM_INV_MAX_J overrides the size threshold (tuning only).
bool use_stream_inverse(const pswe_plan& P, int nq) {
    static const int maxj = [] { const char* e = std::getenv("PSWE_STREAM_INV_MAX_J"); return e ? std::atoi(e) : 384; }();
    return P.legendre_mode == PSWE_LEGENDRE_STREAM && (P.J <= maxj || nq > 4 || inv_rec_big(P, nq));
}

// Inverse Legendre on DMMA. nq complex columns: PLAIN = fields, UV = 2 per pair, EVAL = 4 per state.
void legendre_inverse_mma(const pswe_plan& P, int kind, const double2* in, const double2* in2, int nq, double radius,
                          double2* out, cudaStream_t st) {
    if (nq <= 0) return;
    if (kind == INV_PLAIN) {
        if (use_stream_inverse(P, nq))
            legendre_inverse_stream(P, kind, in, in2, nq, radius, out, st);
        else
            dispatch_inv<false>(P, in, nq, out, st);
        return;
    }
    if (use_stream_inverse(P, nq)) {
        legendre_inverse_stream(P, kind, in, in2, nq, radius, out, st);
        return;
    }
    const long Kx = P.Kx;
    const int per = kind == INV_EVAL ? 4 : 2;
    const int nitems = nq / per;
    dim3 g((unsigned)((Kx + 127) / 128), nitems);
    if (kind == INV_EVAL) inv_prep_kernel<INV_EVAL><<<g, 128, 0, st>>>(P.R, P.d_eps, in, in2, radius, P.d_xcoef);
    else inv_prep_kernel<INV_UV><<<g, 128, 0, st>>>(P.R, P.d_eps, in, in2, radius, P.d_xcoef);
    PSWE_LAUNCH_CHECK();
    dispatch_inv<true>(P, P.d_xcoef, nq, out, st);
}

// Forward Legendre on DMMA over nq complex columns.
void legendre_forward_mma(const pswe_plan& P, const double2* four, int nq, double2* out, bool ext,
                          cudaStream_t st) {
    if (nq <= 0) return;
    const int nsl = (P.J + 31) / 32;
    if (nq > 4 && nsl <= 16) launch_fwd<2>(P, four, nq, out, ext, st);
    else launch_fwd<1>(P, four, nq, out, ext, st);
}

}  // namespace pswe
