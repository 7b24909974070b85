// In-place longitude FFT stage of eval_nonlinear (sm_100a, fp64).
//
// Replaces the ping-pong Stockham kernels of fft.cu (kept for lengths without an in-place plan) for the fused grid stage (swe.cpp:41-54 with
// the FFT halves of uv_from_vortdiv / synthesise / vortdiv_from_uv / analyse, transform.cpp:
// 101-190). One block per (latitude row, state) holds the 5 complex rows of length N = nlon/2 in
// shared memory ONCE (no scratch copy):
//
//   load + c2r pre-pass   X_k (k <= R) of Phi, zeta, U, V -> Z_k, natural order (pair k, N-k
//                         owned by one thread, straight from global memory)
//   inverse DIF passes    in place; the grid leaves in mixed-radix digit-reversed order
//   grid-point products   pointwise, so the permuted order does not matter (4 -> 5 rows)
//   forward DIT passes    in place, the exact transpose of the DIF: digit-reversed in, natural out
//   r2c post-pass         X_k = 1/2 (Z_k + conj Z_{N-k}) - i/2 W^k (Z_k - conj Z_{N-k}), k <= R,
//                         Gauss weight / cos^2 scaling folded, rows [q][m][i] to global
//
// Radix plans end with a radix-8 pass and the shared layout pads one slot per 8 (ipad), which
// makes every pass's 16-byte accesses conflict-free for j-fastest thread mapping (checked with a
// bank model for all instantiated N). Half the shared memory of the ping-pong form, no copy-back
// passes and no separate pre-pass phase: 8 barriers per block instead of 12.
#include <cmath>
#include <cstdlib>

#include "fft_t.cuh"

namespace pswe {

using namespace fftt;

namespace {

constexpr int kIpThreads = 256;



// radix of pass s (0 = first) of the in-place plan for length N; 0 past the last pass.
// Plans: head(N/8) then a final radix-8 pass.
// Plan pl = 1 (narrow evaluations and the plain row transforms): N = 256 as two radix-16 passes
// (fewer shared-memory round trips; 128 registers, so the 5-state grid stage keeps plan 0 and
// 3 blocks/SM: measured single-state eval -1.5 us, transform round trip -4 us, 5-state batch
// +6 us with plan 1). Other N: plan 1 = plan 0.
__host__ __device__ constexpr int ip_radix(int N, int s, int pl = 0) {
    if (N % 8 != 0) return 0;  // every plan ends in a radix-8 pass (N = 25 once matched h = 3)
    if (pl == 1 && N == 256) return s < 2 ? 16 : 0;
    const int h = N / 8;
    int h0 = 0, h1 = 0;
    switch (h) {
        case 3: h0 = 3; break;
        case 4: h0 = 4; break;
        case 6: h0 = 6; break;
        case 8: h0 = 8; break;
        case 12: h0 = 12; break;
        case 16: h0 = 16; break;
        case 24: h0 = 8; h1 = 3; break;
        case 32: h0 = 4; h1 = 8; break;
        case 48: h0 = 8; h1 = 6; break;
        case 64: h0 = 8; h1 = 8; break;
        case 96: h0 = 12; h1 = 8; break;
        case 128: h0 = 16; h1 = 8; break;
        case 192: h0 = 12; h1 = 16; break;
        default: return 0;
    }
    if (s == 0) return h0;
    if (h1) return s == 1 ? h1 : (s == 2 ? 8 : 0);
    return s == 1 ? 8 : 0;
}
__host__ __device__ constexpr int ip_npass(int N, int pl = 0) {
    int s = 0;
    while (ip_radix(N, s, pl)) ++s;
    return s;
}
__host__ __device__ constexpr int ip_len(int N, int s, int pl = 0) {  // sub-transform length entering pass s
    int n = N;
    for (int r = 0; r < s; ++r) n /= ip_radix(N, r, pl);
    return n;
}
__host__ __device__ constexpr int ip_off(int N, int s, int pl = 0) {  // twiddle table offset of pass s
    int o = 0;
    for (int r = 0; r < s; ++r) o += (ip_radix(N, r, pl) - 1) * (ip_len(N, r, pl) / ip_radix(N, r, pl));
    return o;
}

// blocks per SM the register budget is sized for: 4 (64 registers) when every radix is <= 8,
// fewer for the radix-12/16 plans (their butterflies alone hold 24-32 doubles). N = 256 (T255 on
// 256 x 512): 3 (78 registers) - the single-state evaluation of an SDC sweep has one block per
// latitude (256 < 3 x 148), so fewer instructions per block win (eval 36.3 -> 34.0 us, fine sweep
// 177 -> 166 us; the 5-state batch is unchanged); at N = 512 the same change costs 2 us.
__host__ __device__ constexpr int ip_minblocks(int N, int pl = 0) {
    int mx = 0;
    for (int s = 0; ip_radix(N, s, pl); ++s) mx = ip_radix(N, s, pl) > mx ? ip_radix(N, s, pl) : mx;
    if (mx <= 8 && N == 256) return 3;
    if (mx <= 8) return N <= 512 ? 4 : 2;
    return N <= 1024 ? 2 : 1;
}

__host__ __device__ constexpr int ip_ntw(int N, int pl = 0) { return ip_off(N, ip_npass(N, pl), pl); }  // twiddle entries

__device__ __forceinline__ int ipad(int i) { return i + (i >> 3); }
__host__ __device__ constexpr int ipadded(int n) { return n + (n >> 3); }

// w[k] = w1^k, k = 1..P-1, from the one root w1 = w_n^j read from the table: squares for even k,
// one more factor w1 for odd k (product depth <= log2(k) + 1; a few ulp). Trades P-2 shared-memory
// twiddle reads per butterfly (the FFT stage is shared-memory-bandwidth bound) for FP64 work.
template <int P>
__device__ __forceinline__ void pass_roots(double2 (&w)[P], double2 w1) {
    w[0] = make_double2(1.0, 0.0);
    if constexpr (P > 1) w[1] = w1;
#pragma unroll
    for (int k = 2; k < P; ++k) w[k] = (k & 1) ? cmul(w[k - 1], w1) : cmul(w[k >> 1], w[k >> 1]);
}

// DIF pass s on G rows of A: sub-blocks of length n, butterflies over t (stride M), then the
// twiddle w_n^(j k) on output k; outputs back to the same slots.
template <int N, int s, int G, bool INV, int PL = 0>
__device__ __forceinline__ void dif_pass(double2* A, const double2* TW) {
    constexpr int P = ip_radix(N, s, PL), n = ip_len(N, s, PL), M = n / P, OFF = ip_off(N, s, PL);
    constexpr int T = G * N / P;
    for (int it = threadIdx.x; it < T; it += kIpThreads) {
        const int j = it % M;
        const int base = (it - j) * P + j;  // (it / M) n + j
        double2 v[P];
#pragma unroll
        for (int t = 0; t < P; ++t) v[t] = A[ipad(base + t * M)];
        double2 w[P];
        if constexpr (M > 1) pass_roots<P>(w, TW[OFF + j]);
        dft<P, INV>(v);
        A[ipad(base)] = v[0];
#pragma unroll
        for (int k = 1; k < P; ++k) {
            double2 o = v[k];
            if constexpr (M > 1) o = cmul(o, INV ? cconj(w[k]) : w[k]);
            A[ipad(base + k * M)] = o;
        }
    }
}

// DIT pass s (transpose of dif_pass): twiddle w_n^(j t) on input t, then the butterfly.
template <int N, int s, int G, bool INV, int PL = 0>
__device__ __forceinline__ void dit_pass(double2* A, const double2* TW) {
    constexpr int P = ip_radix(N, s, PL), n = ip_len(N, s, PL), M = n / P, OFF = ip_off(N, s, PL);
    constexpr int T = G * N / P;
    for (int it = threadIdx.x; it < T; it += kIpThreads) {
        const int j = it % M;
        const int base = (it - j) * P + j;
        double2 v[P];
#pragma unroll
        for (int t = 0; t < P; ++t) v[t] = A[ipad(base + t * M)];
        if constexpr (M > 1) {
            double2 w[P];
            pass_roots<P>(w, TW[OFF + j]);
#pragma unroll
            for (int t = 1; t < P; ++t) v[t] = cmul(v[t], INV ? cconj(w[t]) : w[t]);
        }
        dft<P, INV>(v);
#pragma unroll
        for (int k = 0; k < P; ++k) A[ipad(base + k * M)] = v[k];
    }
}

template <int N, int s, int G, bool INV, int PL = 0>
struct DifGuard {
    __device__ static void run(double2* A, const double2* TW) {
        if constexpr (s < ip_npass(N, PL)) {
            dif_pass<N, s, G, INV, PL>(A, TW);
            __syncthreads();
            DifGuard<N, s + 1, G, INV, PL>::run(A, TW);
        }
    }
};
template <int N, int s, int G, bool INV, int PL = 0>
struct DitGuard {  // passes s, s-1, ..., 0
    __device__ static void run(double2* A, const double2* TW) {
        if constexpr (s >= 0) {
            dit_pass<N, s, G, INV, PL>(A, TW);
            __syncthreads();
            DitGuard<N, s - 1, G, INV, PL>::run(A, TW);
        }
    }
};

// Z_k of the half-length c2r trick from X_k and X_{N-k}
__device__ __forceinline__ double2 c2r_z(double2 a, double2 bb, double2 w) {
    const double2 b = cconj(bb);
    const double2 e = cadd(a, b);
    const double2 o = cmul(csub(a, b), cconj(w));
    return make_double2(e.x - o.y, e.y + o.x);
}

// Latitude rows J .. 8 ns8 - 1 of a G tile are padding (the P table is zero there). The buffer is
// shared by every batch size, each with its own layout, so those rows may hold another layout's
// values; NaN/Inf there would survive the multiplication by zero. The producer of
// row J - 1 of hemisphere h (one block per hemisphere) zeroes the padding rows of its ncol columns.
__device__ void gt_zero_pad(double* __restrict__ gtile, const GtLayout& gl, int R, int J, int z, int h, int gcol,
                            int ncol, int nthreads) {
    const int npad = 8 * gl.ns8 - J;
#ifdef PSWE_DIAG_NOGTPAD
    return;
#endif
    if (npad <= 0) return;
    const int per_m = npad * ncol;
    for (int it = threadIdx.x; it < (R + 1) * per_m; it += nthreads) {
        const int k = it / per_m, rem = it - k * per_m;
        const int pr = J + rem / ncol, c = gcol + rem % ncol;
        const long row = ((((long)z * (R + 1) + k) * gl.ns8 + (pr >> 3)) * 2 + h) * 8 + (pr & 7);
        gtile[row * gl.sgc + (c ^ gt_swz(gl.ntc, pr & 7))] = 0.0;
    }
}

// GT: write the products as forward-Legendre G tiles (GtLayout, pswe_internal.h) instead of
// Fourier rows [q][m][i]: for each m the block's 5 fields are one 80-byte run.
template <int N, bool GT, int PL = 0>
__global__ void __launch_bounds__(kIpThreads, ip_minblocks(N, PL))
    fft_eval_ip_kernel(int R, int nlat, const double2* __restrict__ TW, const double2* __restrict__ post,
                       const double2* __restrict__ four_in, double2* __restrict__ four_out,
                       const double* __restrict__ rowc, const double* __restrict__ roww,
                       const double* __restrict__ rowmu, double phi_bar, double omega, double inv_a,
                       GtLayout gl) {
    extern __shared__ double2 A[];  // [5][N], ipad layout; then the twiddles [ip_ntw(N)]
    double2* sTW = A + 5 * ipadded(N);
    // GT: the states of one latitude row are consecutive blocks (grid (n, nlat)), so the G-tile
    // sectors two states share are written close together in time (merged in L2 instead of
    // read-modify-written in DRAM when the tiles outgrow it: T1023 with several states)
    const int i = GT ? blockIdx.y : blockIdx.x, b = GT ? blockIdx.x : blockIdx.y;
    // twiddles to shared memory (cp.async, overlapped with the row loads; waited before the
    // first barrier)
    for (int t = threadIdx.x; t < ip_ntw(N, PL); t += kIpThreads) {
        const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(sTW + t));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(TW + t));
    }
    asm volatile("cp.async.commit_group;\n" ::);
    pdl_trigger();
    pdl_wait();  // the Fourier rows come from the inverse Legendre kernel
    const long rowsz = (long)(R + 1) * nlat;
    const double2* in = four_in + ((long)b * 4 * nlat + i) * (R + 1);  // rows [q][i][m]

    // load + pre-pass: task (f, k), k = 0..N/2, owns Z_k and Z_{N-k}; all loads issued first
    constexpr int H = N / 2 + 1;
    constexpr int HS = (H + 7) & ~7;  // task stride per field: 8-aligned k runs (no bank conflicts)
    constexpr int U = (4 * HS + kIpThreads - 1) / kIpThreads;
    double2 xa[U], xb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int it = threadIdx.x + u * kIpThreads;
        xa[u] = xb[u] = make_double2(0.0, 0.0);
        const int f = it / HS, k = it - f * HS;
        if (f < 4 && k < H) {
#ifdef PSWE_FDIAG_NOLOAD
            xa[u] = make_double2(1.0 + k, 0.5 * f);
            xb[u] = make_double2(0.25 * k, 1.0);
#else
            if (k <= R) xa[u] = in[f * rowsz + k];
            if (k > 0 && N - k <= R) xb[u] = in[f * rowsz + N - k];
#endif
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int it = threadIdx.x + u * kIpThreads;
        const int f = it / HS, k = it - f * HS;
        if (f < 4 && k < H) {
            double2 a = xa[u];
            if (k == 0) a.y = 0.0;  // Im G_0 := 0
            A[ipad(f * N + k)] = c2r_z(a, xb[u], __ldg(post + k));
            if (k > 0 && k < N / 2) A[ipad(f * N + N - k)] = c2r_z(xb[u], xa[u], __ldg(post + N - k));
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
#ifndef PSWE_FDIAG_NOFFT
    DifGuard<N, 0, 4, true, PL>::run(A, sTW);
#endif

    // grid-point products (swe.cpp:41-54), two grid points per complex slot, slot order permuted
    const double c = rowc[i];
    const double ic = 1.0 / c;
    const double fc = 2.0 * omega * rowmu[i];
    for (int k = threadIdx.x; k < N; k += kIpThreads) {
        const int p = ipad(k);
        constexpr int RS = ipadded(N);
        const double2 ph = A[p], ze = A[RS + p], U2 = A[2 * RS + p], V2 = A[3 * RS + p];
        double o[5][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double Uh = h ? U2.y : U2.x, Vh = h ? V2.y : V2.x;
            const double uu = Uh * ic, vv = Vh * ic;
            const double phip = (h ? ph.y : ph.x) - phi_bar;
            const double absv = (h ? ze.y : ze.x) + fc;
            o[0][h] = (phip * uu) * c;
            o[1][h] = (phip * vv) * c;
            o[2][h] = (absv * uu) * c;
            o[3][h] = (absv * vv) * c;
            o[4][h] = 0.5 * (uu * uu + vv * vv);
        }
#pragma unroll
        for (int q = 0; q < 5; ++q) A[q * RS + p] = make_double2(o[q][0], o[q][1]);
    }
    __syncthreads();
#ifndef PSWE_FDIAG_NOFFT
    DitGuard<N, ip_npass(N, PL) - 1, 5, false, PL>::run(A, sTW);
#endif

    const double nl = 2.0 * N;
    const double sflux = (1.0 / nl) * (inv_a * roww[i] / (c * c));
    const double ske = (1.0 / nl) * roww[i];
    double2* out = four_out + (long)b * 5 * rowsz + i;
    double* gt = nullptr;
    long gstep = 0;
    int swz = 0, gcol = 0;
    bool equator = false, last_state = false;
    if constexpr (GT) {
        const int J = (nlat + 1) / 2;
        const bool north = i >= nlat - J;
        const int j = north ? i - (nlat - J) : J - 1 - i;
        const int z = b / gl.spg, bl = b - z * gl.spg;
        equator = north && (J - 1 - j == i);  // odd nlat: the equator row is its own mirror
        const long row = (((long)z * (R + 1) * gl.ns8 + (j >> 3)) * 2 + (north ? 0 : 1)) * 8 + (j & 7);
        gt = reinterpret_cast<double*>(four_out) + row * gl.sgc;
        gstep = (long)gl.ns8 * 2 * 8 * gl.sgc;  // doubles between consecutive m
        swz = gt_swz(gl.ntc, j & 7);
        gcol = 10 * bl;
        last_state = bl == min(gl.spg, (int)gridDim.x - z * gl.spg) - 1;
    }
    for (int k = threadIdx.x; k <= R; k += kIpThreads) {
        const double2 w = __ldg(post + k);
        double v[10];  // the 5 scaled X_k, (re, im) each
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const double2 zk = A[ipad(q * N + k)];
            const double2 zc = cconj(A[ipad(q * N + (k == 0 ? 0 : N - k))]);
            const double2 e = make_double2(0.5 * (zk.x + zc.x), 0.5 * (zk.y + zc.y));
            const double2 d = csub(zk, zc);
            const double2 o = make_double2(0.5 * d.y, -0.5 * d.x);
            const double2 x = cadd(e, cmul(w, o));
            const double sc = q < 4 ? sflux : ske;
            v[2 * q] = x.x * sc;
            v[2 * q + 1] = x.y * sc;
        }
#ifdef PSWE_FDIAG_NOSTORE
        if (v[0] == 1.2345e300) gt[0] = v[1];
        continue;
#endif
        if constexpr (GT) {
            // the state's 10 columns gcol.. of this row: the XOR swizzle (a multiple of 4) maps
            // 4-aligned column groups onto 4-aligned groups, so they go out as two 32-byte stores
            // and one 16-byte store (gcol = 10 b is 0 or 2 mod 4)
            double* row = gt + k * gstep;
            auto st4 = [&](int c, double a0, double a1, double a2, double a3) {
                double* p4 = row + (c ^ swz);
                asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p4), "d"(a0), "d"(a1), "d"(a2),
                             "d"(a3)
                             : "memory");
                if (equator)  // G_S := 0
                    asm volatile("st.global.v4.f64 [%0], {%1, %1, %1, %1};\n" ::"l"(p4 + 8 * gl.sgc), "d"(0.0)
                                 : "memory");
            };
            auto st2 = [&](int c, double a0, double a1) {
                double* p2 = row + (c ^ swz);
                *reinterpret_cast<double2*>(p2) = make_double2(a0, a1);
                if (equator) *reinterpret_cast<double2*>(p2 + 8 * gl.sgc) = make_double2(0.0, 0.0);
            };
            if ((gcol & 3) == 0) {
                st4(gcol, v[0], v[1], v[2], v[3]);
                st4(gcol + 4, v[4], v[5], v[6], v[7]);
                // the group's last state ends mid-sector: its padding half (two columns the forward
                // multiplies but never stores) is written with zeros, so every 32-byte sector of the
                // tile row is written whole (a partially written sector costs a DRAM read-modify-
                // write once the tiles outgrow the L2: T1023 single state, 134 MB of tiles)
                if (last_state && gcol + 12 <= gl.sgc) st4(gcol + 8, v[8], v[9], 0.0, 0.0);
                else st2(gcol + 8, v[8], v[9]);
            } else {
                st2(gcol, v[0], v[1]);
                st4(gcol + 2, v[2], v[3], v[4], v[5]);
                st4(gcol + 6, v[6], v[7], v[8], v[9]);
            }
        } else {
#pragma unroll
            for (int q = 0; q < 5; ++q) out[q * rowsz + (long)k * nlat] = make_double2(v[2 * q], v[2 * q + 1]);
        }
    }
    if constexpr (GT) {
        const int J = (nlat + 1) / 2;
        const bool north = i >= nlat - J;
        if ((north ? i - (nlat - J) : J - 1 - i) == J - 1)
            gt_zero_pad(reinterpret_cast<double*>(four_out), gl, R, J, b / gl.spg, north ? 0 : 1,
                        10 * (b % gl.spg), 10, kIpThreads);
    }
}

template <int N, bool GT = false, int PL = 0>
bool eval_ip(const pswe_plan& P, const pswe_params& prm, const double2* fin, double2* fout, int n, cudaStream_t st,
             GtLayout gl = GtLayout()) {
    const size_t sm = (size_t)(5 * ipadded(N) + ip_ntw(N, PL)) * sizeof(double2);
    auto kern = fft_eval_ip_kernel<N, GT, PL>;
    static bool attr = false;  // once per instantiation
    if (!attr) {
        if (sm > 48 * 1024)
            PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        // several blocks per SM only fit with the whole unified L1 given to shared memory
        PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       (int)cudaSharedmemCarveoutMaxShared));
        attr = true;
    }
    launch_pdl(kern, GT ? dim3(n, P.nlat) : dim3(P.nlat, n), dim3(kIpThreads), sm, st, P.R, P.nlat,
               PL ? P.d_fft_iptw1 : P.d_fft_iptw,
               P.d_fft_post, fin, fout,
               P.d_rowc, P.d_roww, P.d_rowmu, prm.phi_bar, prm.omega, 1.0 / prm.radius, gl);
    PSWE_LAUNCH_CHECK();
    return true;
}

// slot of frequency k after the DIF passes (k = d0 + P0 d1 + P0 P1 d2 -> d0 M0 + d1 M1 + d2 M2):
// the mixed-radix digit reversal of the in-place plan
template <int N, int PL = 0>
__device__ __forceinline__ int ip_slot(int k) {
    int p = 0;
#pragma unroll
    for (int s = 0; s < ip_npass(N, PL); ++s) {
        const int P = ip_radix(N, s, PL), M = ip_len(N, s, PL) / P;
        p += (k % P) * M;
        k /= P;
    }
    return p;
}

// rows of one field per block: 8 consecutive latitudes up to N = 512 (so the [q][m][i] Fourier
// writes of r2c are 128-byte runs), fewer beyond (shared memory)
__host__ __device__ constexpr int ip_rows(int N) { return N <= 512 ? 8 : (N <= 1024 ? 4 : 2); }

// Plain longitude transforms of ROWS consecutive latitude rows of one field (synthesise / analyse /
// uv_from_vortdiv / vortdiv_from_uv, transform.cpp:101-190), in place in shared memory.
// C2R: Fourier rows [q][i][m] (q = b in_stride + in_off) -> c2r pre-pass written straight to the
//      digit-reversed slots -> inverse DIT passes -> natural-order grid rows (optionally / cos).
// R2C: grid rows (optionally * cos) -> forward DIF passes -> r2c post-pass gathered from the
//      digit-reversed slots, scaled (scale_mode 0: w / nlon, 1: w / (a cos^2 nlon)), staged
//      [m][row] in shared memory -> Fourier rows [q][m][i] (q = b out_stride + out_off).
// (c2r at N = 256 takes 96 registers, two blocks per SM; capping it at three blocks spills and
// measured no faster, r2aw)
template <int N, bool C2R, int ROWS>
__global__ void __launch_bounds__(kIpThreads)
    fft_rows_ip_kernel(int R, int nlat, const double2* __restrict__ TW, const double2* __restrict__ post,
                       const double2* __restrict__ four_in, const double* __restrict__ grid_in, double2* __restrict__ four_out,
                       double* __restrict__ grid_out, int stride, int off, const double* __restrict__ rowc,
                       const double* __restrict__ roww, int cos_flag, int scale_mode, double inv_a) {
    constexpr int RS = ipadded(N);
    extern __shared__ double2 A[];  // [ROWS][N] ipad layout (R2C: then the [R+1][ROWS] staging); twiddles
    double2* sTW = A + ROWS * RS;
    const int i0 = blockIdx.x * ROWS, b = blockIdx.y;
    const int nrow = min(ROWS, nlat - i0);
    for (int t = threadIdx.x; t < ip_ntw(N, 1); t += kIpThreads) {
        const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(sTW + t));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(TW + t));
    }
    asm volatile("cp.async.commit_group;\n" ::);
    if constexpr (C2R) {
        const double2* in = four_in + (((long)b * stride + off) * nlat + i0) * (R + 1);  // row r: + r (R + 1)
        constexpr int H = N / 2 + 1;
        constexpr int HS = (H + 7) & ~7;
        constexpr int U = (ROWS * HS + kIpThreads - 1) / kIpThreads;
        double2 xa[U], xb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int it = threadIdx.x + u * kIpThreads;
            const int r = it / HS, k = it - r * HS;
            xa[u] = xb[u] = make_double2(0.0, 0.0);
            if (r < nrow && k < H) {
                if (k <= R) xa[u] = in[(long)r * (R + 1) + k];
                if (k > 0 && N - k <= R) xb[u] = in[(long)r * (R + 1) + N - k];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int it = threadIdx.x + u * kIpThreads;
            const int r = it / HS, k = it - r * HS;
            if (r < ROWS && k < H) {
                double2 a = xa[u];
                if (k == 0) a.y = 0.0;
                A[ipad(r * N + ip_slot<N, 1>(k))] = c2r_z(a, xb[u], __ldg(post + k));
                if (k > 0 && k < N / 2) A[ipad(r * N + ip_slot<N, 1>(N - k))] = c2r_z(xb[u], xa[u], __ldg(post + N - k));
            }
        }
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();
        DitGuard<N, ip_npass(N, 1) - 1, ROWS, true, 1>::run(A, sTW);
        for (int it = threadIdx.x; it < ROWS * N; it += kIpThreads) {
            const int r = it / N, k = it - r * N;
            if (r >= nrow) break;
            double2 v = A[ipad(it)];
            if (cos_flag) {
                const double cc = 1.0 / rowc[i0 + r];
                v = make_double2(v.x * cc, v.y * cc);
            }
            reinterpret_cast<double2*>(grid_out + ((long)b * nlat + i0 + r) * 2 * N)[k] = v;
        }
    } else {
        const double2* in = reinterpret_cast<const double2*>(grid_in + ((long)b * nlat + i0) * 2 * N);
        constexpr int UL = (ROWS * N + kIpThreads - 1) / kIpThreads;
        double2 v[UL];
#pragma unroll
        for (int u = 0; u < UL; ++u) {
            const int it = threadIdx.x + u * kIpThreads;
            v[u] = (it < ROWS * N && it / N < nrow) ? in[it] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < UL; ++u) {
            const int it = threadIdx.x + u * kIpThreads;
            if (it >= ROWS * N) break;
            if (cos_flag && it / N < nrow) {
                const double c = rowc[i0 + it / N];
                v[u] = make_double2(v[u].x * c, v[u].y * c);
            }
            A[ipad(it)] = v[u];
        }
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();
        DifGuard<N, 0, ROWS, false, 1>::run(A, sTW);
        // post-pass into registers, then staged [m][row] over the rows (row index XOR-swizzled
        // with m: conflict-free for both the m-fastest writes and the row-fastest reads)
        constexpr int UP = (ROWS * N + kIpThreads - 1) / kIpThreads;  // >= ROWS (R + 1) / 256
        double2 xr[UP];
#pragma unroll
        for (int u = 0; u < UP; ++u) {
            const int it = threadIdx.x + u * kIpThreads;
            const int r = it / (R + 1), k = it - r * (R + 1);
            if (r < ROWS) {
                const double2 zk = A[ipad(r * N + ip_slot<N, 1>(k))];
                const double2 zc = cconj(A[ipad(r * N + ip_slot<N, 1>(k == 0 ? 0 : N - k))]);
                const double2 e = make_double2(0.5 * (zk.x + zc.x), 0.5 * (zk.y + zc.y));
                const double2 d = csub(zk, zc);
                const double2 o = make_double2(0.5 * d.y, -0.5 * d.x);
                xr[u] = cadd(e, cmul(__ldg(post + k), o));
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < UP; ++u) {
            const int it = threadIdx.x + u * kIpThreads;
            const int r = it / (R + 1), k = it - r * (R + 1);
            if (r < ROWS) A[k * ROWS + (r ^ (k & (ROWS - 1)))] = xr[u];
        }
        __syncthreads();
        const double nl = 2.0 * N;
        double2* out = four_out + ((long)b * stride + off) * (R + 1) * nlat + i0;
        for (int it = threadIdx.x; it < ROWS * (R + 1); it += kIpThreads) {
            const int k = it / ROWS, r = it - k * ROWS;
            if (r >= nrow) continue;
            const int i = i0 + r;
            const double c = rowc[i];
            const double sc = scale_mode == 0 ? (1.0 / nl) * roww[i] : (1.0 / nl) * (inv_a * roww[i] / (c * c));
            const double2 x = A[k * ROWS + (r ^ (k & (ROWS - 1)))];
            out[(long)k * nlat + r] = make_double2(x.x * sc, x.y * sc);
        }
    }
}

template <int N, bool C2R, int ROWS>
bool rows_ip_r(const pswe_plan& P, const double2* four_in, const double* grid_in, double2* four_out, double* grid_out,
               int stride, int off, int n, int cos_flag, int scale_mode, double inv_a, cudaStream_t st) {
    const size_t sm = (size_t)(ROWS * ipadded(N) + ip_ntw(N, 1)) * sizeof(double2);  // plan 1
    if (sm > 227 * 1024) return false;
    auto kern = fft_rows_ip_kernel<N, C2R, ROWS>;
    static bool attr = false;  // once per instantiation (the cap, not the size of this launch)
    if (!attr) {
        PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr = true;
    }
    kern<<<dim3((P.nlat + ROWS - 1) / ROWS, n), kIpThreads, sm, st>>>(
        P.R, P.nlat, P.d_fft_iptw1, P.d_fft_post, four_in, grid_in, four_out, grid_out, stride, off, P.d_rowc,
        P.d_roww, cos_flag, scale_mode, inv_a);
    PSWE_LAUNCH_CHECK();
    return true;
}

template <int N, bool C2R>
bool rows_ip(const pswe_plan& P, const double2* four_in, const double* grid_in, double2* four_out, double* grid_out,
             int stride, int off, int n, int cos_flag, int scale_mode, double inv_a, cudaStream_t st) {
    // (4 or 2 latitude rows per block measured slower at N = 256, r2au: c2r 13.5 -> 14.5 / 18.7 us)
    return rows_ip_r<N, C2R, ip_rows(N)>(P, four_in, grid_in, four_out, grid_out, stride, off, n, cos_flag, scale_mode,
                                         inv_a, st);
}

// analyse's longitude transforms on the forward-Legendre G tiles (transform.cpp:163-174 with the
// Fourier coefficients written where the streamed forward reads them, gt_layout_fields): block =
// (latitude row i, 8 fields f0..f0+7), the rows of fft_rows_ip_kernel<N, false> being 8 FIELDS
// of one latitude instead of 8 latitudes of one field, so each order m's (re, im) pairs of the
// block's fields are one 128-byte run of a G-tile row (the column swizzle moves 32-byte groups).
// Same passes, post-pass and scaling (w_i / nlon) as the row kernel.
template <int N>
__global__ void __launch_bounds__(kIpThreads)
    fft_r2c_gt_kernel(int R, int nlat, int nf, const double2* __restrict__ TW, const double2* __restrict__ post,
                      const double* __restrict__ grid_in, double* __restrict__ gtile, const double* __restrict__ roww,
                      GtLayout gl) {
    constexpr int ROWS = 8, RS = ipadded(N);
    extern __shared__ double2 A[];  // [ROWS][N] ipad layout, then the [R+1][ROWS] staging; twiddles
    double2* sTW = A + ROWS * RS;
    const int i = blockIdx.x, f0 = blockIdx.y * ROWS;
    const int nrow = min(ROWS, nf - f0);
    pdl_trigger();  // the forward's P-tile prologue overlaps this kernel (it waits before the G reads)
    for (int t = threadIdx.x; t < ip_ntw(N, 1); t += kIpThreads) {
        const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(sTW + t));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(TW + t));
    }
    asm volatile("cp.async.commit_group;\n" ::);
    constexpr int UL = (ROWS * N + kIpThreads - 1) / kIpThreads;
    double2 v[UL];
#pragma unroll
    for (int u = 0; u < UL; ++u) {
        const int it = threadIdx.x + u * kIpThreads;
        const int r = it / N, e = it - r * N;
        v[u] = r < nrow && it < ROWS * N ? reinterpret_cast<const double2*>(grid_in + ((long)(f0 + r) * nlat + i) * 2 * N)[e]
                        : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < UL; ++u)
        if (threadIdx.x + u * kIpThreads < ROWS * N) A[ipad(threadIdx.x + u * kIpThreads)] = v[u];
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    DifGuard<N, 0, ROWS, false, 1>::run(A, sTW);
    constexpr int UP = (ROWS * N + kIpThreads - 1) / kIpThreads;
    double2 xr[UP];
#pragma unroll
    for (int u = 0; u < UP; ++u) {
        const int it = threadIdx.x + u * kIpThreads;
        const int r = it / (R + 1), k = it - r * (R + 1);
        if (r < ROWS) {
            const double2 zk = A[ipad(r * N + ip_slot<N, 1>(k))];
            const double2 zc = cconj(A[ipad(r * N + ip_slot<N, 1>(k == 0 ? 0 : N - k))]);
            const double2 e = make_double2(0.5 * (zk.x + zc.x), 0.5 * (zk.y + zc.y));
            const double2 d = csub(zk, zc);
            const double2 o = make_double2(0.5 * d.y, -0.5 * d.x);
            xr[u] = cadd(e, cmul(__ldg(post + k), o));
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < UP; ++u) {
        const int it = threadIdx.x + u * kIpThreads;
        const int r = it / (R + 1), k = it - r * (R + 1);
        if (r < ROWS) A[k * ROWS + (r ^ (k & (ROWS - 1)))] = xr[u];
    }
    __syncthreads();
    const int J = (nlat + 1) / 2;
    const bool north = i >= nlat - J;
    const int j = north ? i - (nlat - J) : J - 1 - i;
    const int h = north ? 0 : 1;
    const bool equator = north && (J - 1 - j == i);  // odd nlat: G_S := 0 on the equator row
    const int swz = gt_swz(gl.ntc, j & 7);
    const long gstep = (long)gl.ns8 * 2 * 8 * gl.sgc;  // doubles between consecutive m
    const long row0 = (((long)(j >> 3)) * 2 + h) * 8 + (j & 7);
    const double sc = (1.0 / (2.0 * N)) * roww[i];
    for (int it = threadIdx.x; it < ROWS * (R + 1); it += kIpThreads) {
        const int k = it / ROWS, r = it - k * ROWS;
        if (r >= nrow) continue;
        const int f = f0 + r, z = f / gl.apg, fl = f - z * gl.apg;
        const double2 x = A[k * ROWS + (r ^ (k & (ROWS - 1)))];
        double* p = gtile + ((long)z * (R + 1) + k) * gstep + row0 * gl.sgc + ((2 * fl) ^ swz);
        *reinterpret_cast<double2*>(p) = make_double2(x.x * sc, x.y * sc);
        if (equator) *reinterpret_cast<double2*>(p + 8 * gl.sgc) = make_double2(0.0, 0.0);
    }
    if (j == J - 1)
        for (int r = 0; r < nrow; ++r) {
            const int f = f0 + r, z = f / gl.apg;
            gt_zero_pad(gtile, gl, R, J, z, h, 2 * (f - z * gl.apg), 2, kIpThreads);
        }
}

}  // namespace

// analyse's row transforms into the G tiles of gt_layout_fields(nf) (P.d_gtile); false when
// nlon/2 has no in-place plan or the tiles do not fit the plan's reservation
bool fft_r2c_gt(const pswe_plan& P, const double* grid, const GtLayout& gl, int nf, cudaStream_t st) {
    static const bool off_env = [] { const char* e = getenv("PSWE_FFT_STOCKHAM"); return e && atoi(e) != 0; }();
    if (off_env || !P.d_gtile || gl.doubles > P.gtile_cap || ip_radix(P.N, 0) == 0) return false;
    switch (P.N) {
#define PSWE_CASE(NN)                                                                                     \
    case NN: {                                                                                            \
        const size_t sm = (size_t)(8 * ipadded(NN) + ip_ntw(NN, 1)) * sizeof(double2);                  \
        if (sm > 227 * 1024) return false;                                                                \
        static bool attr = false;                                                                         \
        if (!attr) {                                                                                      \
            PSWE_CUDA(cudaFuncSetAttribute(fft_r2c_gt_kernel<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                           227 * 1024));                                                  \
            attr = true;                                                                                  \
        }                                                                                                 \
        fft_r2c_gt_kernel<NN><<<dim3(P.nlat, (nf + 7) / 8), kIpThreads, sm, st>>>(                        \
            P.R, P.nlat, nf, P.d_fft_iptw1, P.d_fft_post, grid, P.d_gtile, P.d_roww, gl);                 \
        PSWE_LAUNCH_CHECK();                                                                              \
        return true;                                                                                      \
    }
        PSWE_CASE(24) PSWE_CASE(32) PSWE_CASE(48) PSWE_CASE(64) PSWE_CASE(96) PSWE_CASE(128) PSWE_CASE(192)
        PSWE_CASE(256) PSWE_CASE(384) PSWE_CASE(512) PSWE_CASE(768) PSWE_CASE(1024)
#undef PSWE_CASE
        default: return false;
    }
}

bool fft_rows_ip(const pswe_plan& P, bool c2r, const double2* four_in, const double* grid_in, double2* four_out,
                 double* grid_out, int stride, int off, int n, bool cos_flag, int scale_mode, double radius,
                 cudaStream_t st) {
    static const bool off_env = [] { const char* e = getenv("PSWE_FFT_STOCKHAM"); return e && atoi(e) != 0; }();
    if (off_env) return false;
    const int cf = cos_flag ? 1 : 0;
    const double ia = 1.0 / radius;
    switch (P.N) {
#define PSWE_CASE(NN)                                                                                        \
    case NN:                                                                                                 \
        return c2r ? rows_ip<NN, true>(P, four_in, grid_in, four_out, grid_out, stride, off, n, cf, scale_mode, ia, st) \
                   : rows_ip<NN, false>(P, four_in, grid_in, four_out, grid_out, stride, off, n, cf, scale_mode, ia, st);
        PSWE_CASE(24) PSWE_CASE(32) PSWE_CASE(48) PSWE_CASE(64) PSWE_CASE(96) PSWE_CASE(128) PSWE_CASE(192)
        PSWE_CASE(256) PSWE_CASE(384) PSWE_CASE(512) PSWE_CASE(768) PSWE_CASE(1024) PSWE_CASE(1536)
#undef PSWE_CASE
        default: return false;
    }
}

// Twiddles of the in-place plan: pass s (P, M, n = P M): entries OFF_s + (k-1) M + j =
// exp(-2 pi i j k / n), k = 1..P-1, j = 0..M-1. Empty (one dummy entry) if N has no plan.
std::vector<double2> fft_ip_twiddles(int N, int pl) {
    std::vector<double2> tw;
    for (int s = 0; ip_radix(N, s, pl); ++s) {
        const int P = ip_radix(N, s, pl), n = ip_len(N, s, pl), M = n / P;
        for (int k = 1; k < P; ++k)
            for (int j = 0; j < M; ++j) {
                const long double a = -2.0L * 3.141592653589793238462643383279502884L * ((long)j * k % n) / n;
                tw.push_back(make_double2((double)std::cos(a), (double)std::sin(a)));
            }
    }
    if (tw.empty()) tw.push_back(make_double2(1.0, 0.0));
    return tw;
}

bool fft_eval_products_ip(const pswe_plan& P, const pswe_params& prm, const double2* fin, double2* fout, int n,
                          cudaStream_t st) {
    static const bool off = [] { const char* e = getenv("PSWE_FFT_STOCKHAM"); return e && atoi(e) != 0; }();
    if (off) return false;
    switch (P.N) {
#define PSWE_CASE(NN) \
    case NN: return eval_ip<NN>(P, prm, fin, fout, n, st);
        PSWE_CASE(24) PSWE_CASE(32) PSWE_CASE(48) PSWE_CASE(64) PSWE_CASE(96) PSWE_CASE(128) PSWE_CASE(192)
        PSWE_CASE(256) PSWE_CASE(384) PSWE_CASE(512) PSWE_CASE(768) PSWE_CASE(1024) PSWE_CASE(1536)
#undef PSWE_CASE
        default: return false;
    }
}

bool gt_path_ok(const pswe_plan& P, int n) {
    static const bool off = [] { const char* e = getenv("PSWE_FFT_STOCKHAM"); return e && atoi(e) != 0; }();
    static const bool gt_off = [] { const char* e = getenv("PSWE_NO_GTILE"); return e && atoi(e) != 0; }();
    return !off && !gt_off && P.legendre_mode == PSWE_LEGENDRE_STREAM && !P.simt && P.n_chunks > 0 &&
           ip_radix(P.N, 0) != 0 && P.d_gtile != nullptr && gt_layout(P.R, P.J, n).doubles <= P.gtile_cap;
}

void fft_eval_products_gt(const pswe_plan& P, const pswe_params& prm, const double2* fin, int n, cudaStream_t st) {
    const GtLayout gl = gt_layout(P.R, P.J, n);
    double2* g = reinterpret_cast<double2*>(P.d_gtile);
    switch (P.N) {
#define PSWE_CASE(NN) \
    case NN:                                                                                  \
        if (n <= 2) eval_ip<NN, true, 1>(P, prm, fin, g, n, st, gl);                          \
        else eval_ip<NN, true, 0>(P, prm, fin, g, n, st, gl);                                 \
        return;
        PSWE_CASE(24) PSWE_CASE(32) PSWE_CASE(48) PSWE_CASE(64) PSWE_CASE(96) PSWE_CASE(128) PSWE_CASE(192)
        PSWE_CASE(256) PSWE_CASE(384) PSWE_CASE(512) PSWE_CASE(768) PSWE_CASE(1024) PSWE_CASE(1536)
#undef PSWE_CASE
        default: throw std::logic_error("fft_eval_products_gt: no in-place plan for this grid");
    }
}

}  // namespace pswe
