// Compile-time-sized longitude FFT kernels (sm_100a, fp64) — see fft.cu for the algorithm and
// the reference loops they replace; this file instantiates them for the grid sizes in use
// (nlon/2 in {24, 32, 48, 64, 96, 128, 192, 256, 384, 512, 768, 1024, 1536}); other 5-smooth
// sizes use the runtime-generic kernels of fft.cu. Shared buffers use padded indexing
// (fftt::pidx) and all loop bounds are compile-time (no runtime integer division).
#include <cmath>

#include "fft_t.cuh"

namespace pswe {

using namespace fftt;

namespace {

// c2r pre-pass from staged X (xs[k], k <= R): Z_k = (X_k + conj X_{N-k}) + i conj(W2^k)(X_k - conj X_{N-k})
template <int N>
__device__ __forceinline__ double2 c2r_pre_s(const double2* xs, int k, int R, const double2* __restrict__ post) {
    double2 a = (k <= R) ? xs[k] : make_double2(0.0, 0.0);
    const int kk = N - k;
    const double2 bb = (k > 0 && kk <= R) ? xs[kk] : make_double2(0.0, 0.0);
    if (k == 0) a.y = 0.0;
    const double2 b = cconj(bb);
    const double2 e = cadd(a, b);
    const double2 o = cmul(csub(a, b), cconj(__ldg(post + k)));
    return make_double2(e.x - o.y, e.y + o.x);
}

// r2c post-pass on a padded sequence starting at element base:
// X_k = 1/2 (Z_k + conj Z_{N-k}) - i/2 W2^k (Z_k - conj Z_{N-k}), k <= R < N
template <int N>
__device__ __forceinline__ double2 r2c_post_s(const double2* z, int base, int k, const double2* __restrict__ post) {
    const double2 zk = z[pidx(base + k)];
    const double2 zc = cconj(z[pidx(base + (k == 0 ? 0 : N - k))]);
    const double2 e = make_double2(0.5 * (zk.x + zc.x), 0.5 * (zk.y + zc.y));
    const double2 d = csub(zk, zc);
    const double2 o = make_double2(0.5 * d.y, -0.5 * d.x);
    return cadd(e, cmul(__ldg(post + k), o));
}

// complex FFT of G padded sequences in data with scratch tmp; result back in data
template <int N, int G, bool INV>
__device__ __forceinline__ void fft_fields(double2* data, double2* tmp, const double2* TW) {
    double2* res = fft<N, G, INV>(data, tmp, TW);
    if (res != data) {
        for (int i = threadIdx.x; i < padded(G * N); i += blockDim.x) data[i] = res[i];
        __syncthreads();
    }
}

// Fused grid stage of eval_nonlinear (see fft.cu fft_eval_kernel). BIG: transforms one field
// at a time with a single scratch row (large N); otherwise all fields per pass.
template <int N, bool BIG>
__global__ void __launch_bounds__(256) fft_eval_t_kernel(int R, int nlat, const double2* __restrict__ TW,
                                                         const double2* __restrict__ post,
                                                         const double2* __restrict__ four_in,
                                                         double2* __restrict__ four_out,
                                                         const double* __restrict__ rowc,
                                                         const double* __restrict__ roww,
                                                         const double* __restrict__ rowmu, double phi_bar,
                                                         double omega, double inv_a) {
    constexpr int NT = 256;
    constexpr int KU = (N + NT - 1) / NT;  // row elements per thread (R + 1 <= N)
    constexpr int SEQ = padded(N);         // BIG: stride between separately padded sequences
    extern __shared__ double2 sm[];
    double2* data = sm;                                   // BIG: 5 x padded(N); else padded(5N)
    double2* tmp = sm + (BIG ? 5 * SEQ : padded(5 * N));  // scratch; also the X staging area
    const int i = blockIdx.x, b = blockIdx.y;
    const long rowsz = (long)(R + 1) * nlat;
    const double2* in = four_in + ((long)b * 4 * nlat + i) * (R + 1);  // rows [q][i][m]
    if (BIG) {
        double2* xs = data + 4 * SEQ;  // field 4 of data is free until the products
        for (int f = 0; f < 4; ++f) {
            double2 v[KU];
#pragma unroll
            for (int u = 0; u < KU; ++u) {
                const int k = threadIdx.x + u * NT;
                if (k <= R) v[u] = in[f * rowsz + k];
            }
#pragma unroll
            for (int u = 0; u < KU; ++u) {
                const int k = threadIdx.x + u * NT;
                if (k <= R) xs[k] = v[u];
            }
            __syncthreads();
            for (int k = threadIdx.x; k < N; k += NT) data[f * SEQ + pidx(k)] = c2r_pre_s<N>(xs, k, R, post);
            __syncthreads();
        }
        for (int f = 0; f < 4; ++f) fft_fields<N, 1, true>(data + f * SEQ, tmp, TW);
    } else {
        // stage X_k (k <= R) of the 4 input fields: every load issued before any store
        double2* xs = tmp;
        double2 v[4][KU];
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int u = 0; u < KU; ++u) {
                const int k = threadIdx.x + u * NT;
                if (k <= R) v[f][u] = in[f * rowsz + k];
            }
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int u = 0; u < KU; ++u) {
                const int k = threadIdx.x + u * NT;
                if (k <= R) xs[f * N + k] = v[f][u];
            }
        __syncthreads();
#pragma unroll
        for (int f = 0; f < 4; ++f)
            for (int k = threadIdx.x; k < N; k += NT) data[pidx(f * N + k)] = c2r_pre_s<N>(xs + f * N, k, R, post);
        __syncthreads();
        fft_fields<N, 4, true>(data, tmp, TW);
    }
    // grid-point products (swe.cpp:41-54), two grid points per complex slot, in place
    auto at = [&](int f, int k) -> double2& { return BIG ? data[f * SEQ + pidx(k)] : data[pidx(f * N + k)]; };
    const double c = rowc[i];
    const double ic = 1.0 / c;
    const double fc = 2.0 * omega * rowmu[i];
    for (int k = threadIdx.x; k < N; k += NT) {
        const double2 ph = at(0, k), ze = at(1, k), U = at(2, k), V = at(3, k);
        double o[5][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double Uh = h ? U.y : U.x, Vh = h ? V.y : V.x;
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
        for (int q = 0; q < 5; ++q) at(q, k) = make_double2(o[q][0], o[q][1]);
    }
    __syncthreads();
    if (BIG) {
        for (int q = 0; q < 5; ++q) fft_fields<N, 1, false>(data + q * SEQ, tmp, TW);
    } else {
        fft_fields<N, 5, false>(data, tmp, TW);
    }
    const double nl = 2.0 * N;
    const double sflux = (1.0 / nl) * (inv_a * roww[i] / (c * c));
    const double ske = (1.0 / nl) * roww[i];
    double2* out = four_out + (long)b * 5 * rowsz + i;
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const double2* zq = BIG ? data + q * SEQ : data;
        const int base = BIG ? 0 : q * N;
        const double sc = q < 4 ? sflux : ske;
        for (int k = threadIdx.x; k <= R; k += NT) {
            const double2 x = r2c_post_s<N>(zq, base, k, post);
            out[q * rowsz + (long)k * nlat] = make_double2(x.x * sc, x.y * sc);
        }
    }
}

template <int N>
__global__ void __launch_bounds__(128) fft_c2r_t_kernel(int R, int nlat, const double2* __restrict__ TW,
                                                        const double2* __restrict__ post,
                                                        const double2* __restrict__ four, int in_stride, int in_off,
                                                        double* __restrict__ grid, const double* __restrict__ rowc,
                                                        int div_cos) {
    extern __shared__ double2 sm[];
    double2* buf = sm;
    double2* tmp = sm + padded(N);
    const int i = blockIdx.x, b = blockIdx.y;
    const double2* row = four + (((long)b * in_stride + in_off) * nlat + i) * (R + 1);
    for (int k = threadIdx.x; k <= R; k += blockDim.x) tmp[k] = row[k];
    __syncthreads();
    for (int k = threadIdx.x; k < N; k += blockDim.x) buf[pidx(k)] = c2r_pre_s<N>(tmp, k, R, post);
    __syncthreads();
    double2* res = fft<N, 1, true>(buf, tmp, TW);
    const double cc = div_cos ? 1.0 / rowc[i] : 1.0;
    double2* out = (double2*)(grid + ((long)b * nlat + i) * 2 * N);
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        double2 v = res[pidx(k)];
        if (div_cos) v = make_double2(v.x * cc, v.y * cc);
        out[k] = v;
    }
}

template <int N>
__global__ void __launch_bounds__(128) fft_r2c_t_kernel(int R, int nlat, const double2* __restrict__ TW,
                                                        const double2* __restrict__ post,
                                                        const double* __restrict__ grid, double2* __restrict__ four,
                                                        int out_stride, int out_off, const double* __restrict__ rowc,
                                                        const double* __restrict__ roww, int pre_cos, int scale_mode,
                                                        double inv_a) {
    extern __shared__ double2 sm[];
    double2* buf = sm;
    double2* tmp = sm + padded(N);
    const int i = blockIdx.x, b = blockIdx.y;
    const double2* in = (const double2*)(grid + ((long)b * nlat + i) * 2 * N);
    const double c = rowc[i];
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        double2 v = in[k];
        if (pre_cos) v = make_double2(v.x * c, v.y * c);
        buf[pidx(k)] = v;
    }
    __syncthreads();
    double2* res = fft<N, 1, false>(buf, tmp, TW);
    const double nl = 2.0 * N;
    const double sc = scale_mode == 0 ? (1.0 / nl) * roww[i] : (1.0 / nl) * (inv_a * roww[i] / (c * c));
    double2* out = four + ((long)b * out_stride + out_off) * (R + 1) * nlat + i;
    for (int k = threadIdx.x; k <= R; k += blockDim.x) {
        const double2 x = r2c_post_s<N>(res, 0, k, post);
        out[(long)k * nlat] = make_double2(x.x * sc, x.y * sc);
    }
}

template <int N>
bool eval_t(const pswe_plan& P, const pswe_params& prm, const double2* fin, double2* fout, int n, cudaStream_t st) {
    constexpr bool BIG = N >= 1024;
    const size_t sm = (size_t)(BIG ? 6 * padded(N) : 2 * padded(5 * N)) * sizeof(double2);
    auto kern = fft_eval_t_kernel<N, BIG>;
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<dim3(P.nlat, n), 256, sm, st>>>(P.R, P.nlat, P.d_fft_ptw, P.d_fft_post, fin, fout, P.d_rowc, P.d_roww,
                                           P.d_rowmu, prm.phi_bar, prm.omega, 1.0 / prm.radius);
    PSWE_LAUNCH_CHECK();
    return true;
}

template <int N>
bool c2r_t(const pswe_plan& P, const double2* four, int in_stride, int in_off, double* grid, int n, bool div_cos,
           cudaStream_t st) {
    const size_t sm = 2 * (size_t)padded(N) * sizeof(double2);
    auto kern = fft_c2r_t_kernel<N>;
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<dim3(P.nlat, n), 128, sm, st>>>(P.R, P.nlat, P.d_fft_ptw, P.d_fft_post, four, in_stride, in_off, grid,
                                           P.d_rowc, div_cos ? 1 : 0);
    PSWE_LAUNCH_CHECK();
    return true;
}

template <int N>
bool r2c_t(const pswe_plan& P, const double* grid, double2* four, int out_stride, int out_off, int n, bool pre_cos,
           int scale_mode, double radius, cudaStream_t st) {
    const size_t sm = 2 * (size_t)padded(N) * sizeof(double2);
    auto kern = fft_r2c_t_kernel<N>;
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<dim3(P.nlat, n), 128, sm, st>>>(P.R, P.nlat, P.d_fft_ptw, P.d_fft_post, grid, four, out_stride, out_off,
                                           P.d_rowc, P.d_roww, pre_cos ? 1 : 0, scale_mode, 1.0 / radius);
    PSWE_LAUNCH_CHECK();
    return true;
}

#define PSWE_FFT_SIZES(X) X(24) X(32) X(48) X(64) X(96) X(128) X(192) X(256) X(384) X(512) X(768) X(1024) X(1536)

}  // namespace

// Per-pass twiddle tables of the compile-time Stockham (same radix sequence as fftt::radix_of):
// pass (P, M): entries (t-1) M + j = exp(-2 pi i j t / (P M)), t = 1..P-1, j = 0..M-1.
std::vector<double2> fft_pass_twiddles(int N) {
    std::vector<double2> tw;
    int n = N;
    while (n > 1) {
        const int P = radix_of(n), M = n / P;
        for (int t = 1; t < P; ++t)
            for (int j = 0; j < M; ++j) {
                const long double a = -2.0L * 3.141592653589793238462643383279502884L * ((long)j * t % n) / n;
                tw.push_back(make_double2((double)std::cos(a), (double)std::sin(a)));
            }
        n = M;
    }
    if (tw.empty()) tw.push_back(make_double2(1.0, 0.0));
    return tw;
}

// Compile-time-sized dispatch; return false when nlon/2 is not an instantiated size (the caller
// then uses the runtime-generic kernels of fft.cu).
bool fft_eval_products_t(const pswe_plan& P, const pswe_params& prm, const double2* fin, double2* fout, int n,
                         cudaStream_t st) {
    switch (P.N) {
#define PSWE_CASE(NN) \
    case NN: return eval_t<NN>(P, prm, fin, fout, n, st);
        PSWE_FFT_SIZES(PSWE_CASE)
#undef PSWE_CASE
        default: return false;
    }
}

bool fft_rows_c2r_t(const pswe_plan& P, const double2* four, int in_stride, int in_off, double* grid, int n,
                    bool div_cos, cudaStream_t st) {
    switch (P.N) {
#define PSWE_CASE(NN) \
    case NN: return c2r_t<NN>(P, four, in_stride, in_off, grid, n, div_cos, st);
        PSWE_FFT_SIZES(PSWE_CASE)
#undef PSWE_CASE
        default: return false;
    }
}

bool fft_rows_r2c_t(const pswe_plan& P, const double* grid, double2* four, int out_stride, int out_off, int n,
                    bool pre_cos, int scale_mode, double radius, cudaStream_t st) {
    switch (P.N) {
#define PSWE_CASE(NN) \
    case NN: return r2c_t<NN>(P, grid, four, out_stride, out_off, n, pre_cos, scale_mode, radius, st);
        PSWE_FFT_SIZES(PSWE_CASE)
#undef PSWE_CASE
        default: return false;
    }
}

}  // namespace pswe
