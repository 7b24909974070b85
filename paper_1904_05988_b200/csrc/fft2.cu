// Compile-time-sized longitude FFT kernels (sm_100a, fp64) — see fft.cu for the algorithm and
// the reference loops they replace; this file instantiates them for the grid sizes in use
// (nlon/2 in {24, 32, 48, 64, 96, 128, 192, 256, 384, 512, 768, 1024, 1536}); other 5-smooth
// sizes use the runtime-generic kernels of fft.cu.
#include "fft_t.cuh"

namespace pswe {

using namespace fftt;

namespace {

// stage the N roots exp(-2 pi i k/N) into shared memory
template <int N>
__device__ __forceinline__ void load_roots(double2* W, const double2* __restrict__ roots) {
    for (int k = threadIdx.x; k < N; k += blockDim.x) W[k] = roots[k];
}

// c2r pre-pass from staged X (xs[k], k <= R): Z_k = (X_k + conj X_{N-k}) + i conj(W2^k)(X_k - conj X_{N-k})
template <int N>
__device__ __forceinline__ double2 c2r_pre_s(const double2* xs, int k, int R, const double2* __restrict__ post) {
    double2 a = (k <= R) ? xs[k] : make_double2(0.0, 0.0);
    const int kk = N - k;
    const double2 bb = (k > 0 && kk <= R) ? xs[kk] : make_double2(0.0, 0.0);
    if (k == 0) a.y = 0.0;
    const double2 b = cconj(bb);
    const double2 e = cadd(a, b);
    const double2 o = cmul(csub(a, b), cconj(post[k]));
    return make_double2(e.x - o.y, e.y + o.x);
}

// r2c post-pass: X_k = 1/2 (Z_k + conj Z_{N-k}) - i/2 W2^k (Z_k - conj Z_{N-k}), k <= R < N
template <int N>
__device__ __forceinline__ double2 r2c_post_s(const double2* z, int k, const double2* __restrict__ post) {
    const double2 zk = z[k];
    const double2 zc = cconj(z[k == 0 ? 0 : N - k]);
    const double2 e = make_double2(0.5 * (zk.x + zc.x), 0.5 * (zk.y + zc.y));
    const double2 d = csub(zk, zc);
    const double2 o = make_double2(0.5 * d.y, -0.5 * d.x);
    return cadd(e, cmul(post[k], o));
}

// complex FFT of fields [f0, f0+nf) of data (length N each) with scratch; result back in data
template <int N, int G, bool INV>
__device__ __forceinline__ void fft_fields(double2* data, double2* tmp, const double2* W) {
    double2* res = fft<N, G, INV>(data, tmp, W);
    if (res != data) {
        for (int i = threadIdx.x; i < G * N; i += blockDim.x) data[i] = res[i];
        __syncthreads();
    }
}

// Fused grid stage of eval_nonlinear (see fft.cu fft_eval_kernel). BIG: transforms one field
// at a time with a single scratch row (large N); otherwise all fields per pass.
template <int N, bool BIG>
__global__ void __launch_bounds__(256) fft_eval_t_kernel(int R, int nlat, const double2* __restrict__ roots,
                                                         const double2* __restrict__ post,
                                                         const double2* __restrict__ four_in,
                                                         double2* __restrict__ four_out,
                                                         const double* __restrict__ rowc,
                                                         const double* __restrict__ roww,
                                                         const double* __restrict__ rowmu, double phi_bar,
                                                         double omega, double inv_a) {
    extern __shared__ double2 sm[];
    double2* W = sm;              // [N]
    double2* ps = sm + N;         // [N+1] exp(-2 pi i k/nlon)
    double2* data = sm + 2 * N + 2;  // [5][N]
    double2* tmp = data + 5 * N;  // [BIG ? 1 : 5][N]
    const int i = blockIdx.x, b = blockIdx.y;
    const long rowsz = (long)(R + 1) * nlat;
    const double2* in = four_in + ((long)b * 4 * nlat + i) * (R + 1);  // rows [q][i][m]
    load_roots<N>(W, roots);
    for (int k = threadIdx.x; k <= N; k += blockDim.x) ps[k] = post[k];
    // stage X_k (k <= R) of the 4 input fields, then the c2r pre-pass into data
    double2* xs = BIG ? data + 4 * N : tmp;  // BIG: data[4] is free until the products
    if (BIG) {
        for (int f = 0; f < 4; ++f) {
            for (int k = threadIdx.x; k <= R; k += blockDim.x) xs[k] = in[f * rowsz + k];
            __syncthreads();
            for (int k = threadIdx.x; k < N; k += blockDim.x) data[f * N + k] = c2r_pre_s<N>(xs, k, R, ps);
            __syncthreads();
        }
        for (int f = 0; f < 4; ++f) fft_fields<N, 1, true>(data + f * N, tmp, W);
    } else {
        // strided row gather: issue every load of this thread before any store (memory-level
        // parallelism; the rows [q][m][i] are latitude-contiguous for the Legendre kernels)
        constexpr int MAXU = (4 * N + 255) / 256;
        double2 v[MAXU];
        const int tot = 4 * (R + 1);
#pragma unroll
        for (int u = 0; u < MAXU; ++u) {
            const int idx = threadIdx.x + u * blockDim.x;
            if (idx < tot) {
                const int ff = idx / (R + 1), k = idx - ff * (R + 1);
                v[u] = in[ff * rowsz + k];
            }
        }
#pragma unroll
        for (int u = 0; u < MAXU; ++u) {
            const int idx = threadIdx.x + u * blockDim.x;
            if (idx < tot) {
                const int ff = idx / (R + 1), k = idx - ff * (R + 1);
                xs[ff * N + k] = v[u];
            }
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < 4 * N; idx += blockDim.x) {
            const int f = idx / N, k = idx - f * N;
            data[idx] = c2r_pre_s<N>(xs + f * N, k, R, ps);
        }
        __syncthreads();
        fft_fields<N, 4, true>(data, tmp, W);
    }
    // grid-point products (swe.cpp:41-54), two grid points per complex slot, in place
    const double c = rowc[i];
    const double ic = 1.0 / c;
    const double f = 2.0 * omega * rowmu[i];
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        const double2 ph = data[k], ze = data[N + k], U = data[2 * N + k], V = data[3 * N + k];
        double o[5][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double Uh = h ? U.y : U.x, Vh = h ? V.y : V.x;
            const double uu = Uh * ic, vv = Vh * ic;
            const double phip = (h ? ph.y : ph.x) - phi_bar;
            const double absv = (h ? ze.y : ze.x) + f;
            o[0][h] = (phip * uu) * c;
            o[1][h] = (phip * vv) * c;
            o[2][h] = (absv * uu) * c;
            o[3][h] = (absv * vv) * c;
            o[4][h] = 0.5 * (uu * uu + vv * vv);
        }
#pragma unroll
        for (int q = 0; q < 5; ++q) data[q * N + k] = make_double2(o[q][0], o[q][1]);
    }
    __syncthreads();
    if (BIG) {
        for (int q = 0; q < 5; ++q) fft_fields<N, 1, false>(data + q * N, tmp, W);
    } else {
        fft_fields<N, 5, false>(data, tmp, W);
    }
    const double nl = 2.0 * N;
    const double sflux = (1.0 / nl) * (inv_a * roww[i] / (c * c));
    const double ske = (1.0 / nl) * roww[i];
    double2* out = four_out + (long)b * 5 * rowsz + i;
    for (int idx = threadIdx.x; idx < 5 * (R + 1); idx += blockDim.x) {
        const int q = idx / (R + 1), k = idx - q * (R + 1);
        const double2 x = r2c_post_s<N>(data + q * N, k, ps);
        const double sc = q < 4 ? sflux : ske;
        out[q * rowsz + (long)k * nlat] = make_double2(x.x * sc, x.y * sc);
    }
}

template <int N>
__global__ void __launch_bounds__(128) fft_c2r_t_kernel(int R, int nlat, const double2* __restrict__ roots,
                                                        const double2* __restrict__ post,
                                                        const double2* __restrict__ four, int in_stride, int in_off,
                                                        double* __restrict__ grid, const double* __restrict__ rowc,
                                                        int div_cos) {
    extern __shared__ double2 sm[];
    double2* W = sm;
    double2* buf = sm + N;
    double2* tmp = buf + N;
    const int i = blockIdx.x, b = blockIdx.y;
    load_roots<N>(W, roots);
    const double2* row = four + (((long)b * in_stride + in_off) * nlat + i) * (R + 1);
    for (int k = threadIdx.x; k <= R; k += blockDim.x) tmp[k] = row[k];
    __syncthreads();
    for (int k = threadIdx.x; k < N; k += blockDim.x) buf[k] = c2r_pre_s<N>(tmp, k, R, post);
    __syncthreads();
    double2* res = fft<N, 1, true>(buf, tmp, W);
    const double cc = div_cos ? 1.0 / rowc[i] : 1.0;
    double2* out = (double2*)(grid + ((long)b * nlat + i) * 2 * N);
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        double2 v = res[k];
        if (div_cos) v = make_double2(v.x * cc, v.y * cc);
        out[k] = v;
    }
}

template <int N>
__global__ void __launch_bounds__(128) fft_r2c_t_kernel(int R, int nlat, const double2* __restrict__ roots,
                                                        const double2* __restrict__ post,
                                                        const double* __restrict__ grid, double2* __restrict__ four,
                                                        int out_stride, int out_off, const double* __restrict__ rowc,
                                                        const double* __restrict__ roww, int pre_cos, int scale_mode,
                                                        double inv_a) {
    extern __shared__ double2 sm[];
    double2* W = sm;
    double2* buf = sm + N;
    double2* tmp = buf + N;
    const int i = blockIdx.x, b = blockIdx.y;
    load_roots<N>(W, roots);
    const double2* in = (const double2*)(grid + ((long)b * nlat + i) * 2 * N);
    const double c = rowc[i];
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        double2 v = in[k];
        if (pre_cos) v = make_double2(v.x * c, v.y * c);
        buf[k] = v;
    }
    __syncthreads();
    double2* res = fft<N, 1, false>(buf, tmp, W);
    const double nl = 2.0 * N;
    const double sc = scale_mode == 0 ? (1.0 / nl) * roww[i] : (1.0 / nl) * (inv_a * roww[i] / (c * c));
    double2* out = four + ((long)b * out_stride + out_off) * (R + 1) * nlat + i;
    for (int k = threadIdx.x; k <= R; k += blockDim.x) {
        const double2 x = r2c_post_s<N>(res, k, post);
        out[(long)k * nlat] = make_double2(x.x * sc, x.y * sc);
    }
}

template <int N>
bool eval_t(const pswe_plan& P, const pswe_params& prm, const double2* fin, double2* fout, int n, cudaStream_t st) {
    constexpr bool BIG = N >= 1024;
    const size_t sm = (size_t)(2 * N + 2 + 5 * N + (BIG ? 1 : 5) * N) * sizeof(double2);
    auto kern = fft_eval_t_kernel<N, BIG>;
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<dim3(P.nlat, n), 256, sm, st>>>(P.R, P.nlat, P.d_fft_roots, P.d_fft_post, fin, fout, P.d_rowc, P.d_roww,
                                           P.d_rowmu, prm.phi_bar, prm.omega, 1.0 / prm.radius);
    PSWE_LAUNCH_CHECK();
    return true;
}

template <int N>
bool c2r_t(const pswe_plan& P, const double2* four, int in_stride, int in_off, double* grid, int n, bool div_cos,
           cudaStream_t st) {
    const size_t sm = 3 * (size_t)N * sizeof(double2);
    auto kern = fft_c2r_t_kernel<N>;
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<dim3(P.nlat, n), 128, sm, st>>>(P.R, P.nlat, P.d_fft_roots, P.d_fft_post, four, in_stride, in_off, grid,
                                           P.d_rowc, div_cos ? 1 : 0);
    PSWE_LAUNCH_CHECK();
    return true;
}

template <int N>
bool r2c_t(const pswe_plan& P, const double* grid, double2* four, int out_stride, int out_off, int n, bool pre_cos,
           int scale_mode, double radius, cudaStream_t st) {
    const size_t sm = 3 * (size_t)N * sizeof(double2);
    auto kern = fft_r2c_t_kernel<N>;
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<dim3(P.nlat, n), 128, sm, st>>>(P.R, P.nlat, P.d_fft_roots, P.d_fft_post, grid, four, out_stride, out_off,
                                           P.d_rowc, P.d_roww, pre_cos ? 1 : 0, scale_mode, 1.0 / radius);
    PSWE_LAUNCH_CHECK();
    return true;
}

#define PSWE_FFT_SIZES(X) X(24) X(32) X(48) X(64) X(96) X(128) X(192) X(256) X(384) X(512) X(768) X(1024) X(1536)

}  // namespace

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
