// Longitude FFTs of the spherical-harmonic transform, staged in shared memory (sm_100a, fp64).
//
// Reference: fourier_rows / inverse_rows (transform.cpp:97-134) call FFTW r2c/c2r per latitude
// row. Here a real row of length nlon is packed as nlon/2 complex values (even/odd samples),
// transformed by a self-sorting Stockham DIF complex FFT (radices 4, 2, 3, 5, precomputed
// twiddles) and split/merged with the exp(-2 pi i k/nlon) twiddle pass. One CTA per latitude
// row (per batch item); all stages stay in shared memory.
//
// fft_eval_products fuses the whole grid-point stage of eval_nonlinear (swe.cpp:41-54): the
// c2r of the Fourier rows of Phi, zeta, U = u cos(phi), V = v cos(phi) (uv_from_vortdiv's
// inverse_rows + ÷cos(phi), synthesise's inverse_rows), the five products, and the r2c of
// Phi'U, Phi'V, (zeta+f)U, (zeta+f)V, ke with the Gauss weights of analyse /
// vortdiv_from_uv folded in (transform.cpp:111,147,255). Grid fields never touch HBM.
#include "pswe_internal.h"

namespace pswe {

namespace {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 rot(double2 a) {
    return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}
template <bool INV>
__device__ __forceinline__ double2 twid(const double2* __restrict__ tw, int idx) {
    const double2 w = __ldg(tw + idx);
    return INV ? cconj(w) : w;
}

// One radix-p Stockham DIF stage on G sequences of length N: src -> dst.
template <bool INV>
__device__ void fft_stage(const double2* __restrict__ src, double2* __restrict__ dst, const FftStage st, int N,
                          int G, const double2* __restrict__ tw) {
    const int p = st.p, m = st.m, s = st.s;
    const int per = N / p;
    const double2* __restrict__ tws = tw + st.tw_off;
    for (int it = threadIdx.x; it < G * per; it += blockDim.x) {
        const int g = it / per;
        const int r = it - g * per;
        const int j = r / s;
        const int q = r - j * s;
        const double2* x = src + (long)g * N + q + s * j;
        double2* y = dst + (long)g * N + q + s * p * j;
        if (p == 4) {
            const double2 a0 = x[0], a1 = x[s * m], a2 = x[2 * s * m], a3 = x[3 * s * m];
            const double2 b0 = cadd(a0, a2), b1 = csub(a0, a2), b2 = cadd(a1, a3);
            const double2 b3 = rot<INV>(csub(a1, a3));
            y[0] = cadd(b0, b2);
            y[s] = cmul(cadd(b1, b3), twid<INV>(tws, j * 4 + 1));
            y[2 * s] = cmul(csub(b0, b2), twid<INV>(tws, j * 4 + 2));
            y[3 * s] = cmul(csub(b1, b3), twid<INV>(tws, j * 4 + 3));
        } else if (p == 2) {
            const double2 a0 = x[0], a1 = x[s * m];
            y[0] = cadd(a0, a1);
            y[s] = cmul(csub(a0, a1), twid<INV>(tws, j * 2 + 1));
        } else if (p == 3) {
            const double c1 = -0.5, s1 = 0.86602540378443864676372317075294;  // cos/sin(2pi/3)
            const double2 a0 = x[0], a1 = x[s * m], a2 = x[2 * s * m];
            const double2 t1 = cadd(a1, a2);
            const double2 t2 = make_double2(a0.x + c1 * t1.x, a0.y + c1 * t1.y);
            const double2 d = csub(a1, a2);
            const double2 t3 = rot<INV>(make_double2(s1 * d.x, s1 * d.y));  // -i s1 d (fwd)
            y[0] = cadd(a0, t1);
            y[s] = cmul(cadd(t2, t3), twid<INV>(tws, j * 3 + 1));
            y[2 * s] = cmul(csub(t2, t3), twid<INV>(tws, j * 3 + 2));
        } else {  // p == 5
            const double c1 = 0.30901699437494742410229341718282, c2 = -0.80901699437494742410229341718282;
            const double s1 = 0.95105651629515357211643933337938, s2 = 0.58778525229247312916870595463907;
            const double2 a0 = x[0], a1 = x[s * m], a2 = x[2 * s * m], a3 = x[3 * s * m], a4 = x[4 * s * m];
            const double2 b1 = cadd(a1, a4), b2 = cadd(a2, a3), d1 = csub(a1, a4), d2 = csub(a2, a3);
            const double2 e1 = make_double2(a0.x + c1 * b1.x + c2 * b2.x, a0.y + c1 * b1.y + c2 * b2.y);
            const double2 e2 = make_double2(a0.x + c2 * b1.x + c1 * b2.x, a0.y + c2 * b1.y + c1 * b2.y);
            const double2 f1 = rot<INV>(make_double2(s1 * d1.x + s2 * d2.x, s1 * d1.y + s2 * d2.y));
            const double2 f2 = rot<INV>(make_double2(s2 * d1.x - s1 * d2.x, s2 * d1.y - s1 * d2.y));
            y[0] = cadd(a0, cadd(b1, b2));
            y[s] = cmul(cadd(e1, f1), twid<INV>(tws, j * 5 + 1));
            y[4 * s] = cmul(csub(e1, f1), twid<INV>(tws, j * 5 + 4));
            y[2 * s] = cmul(cadd(e2, f2), twid<INV>(tws, j * 5 + 2));
            y[3 * s] = cmul(csub(e2, f2), twid<INV>(tws, j * 5 + 3));
        }
    }
}

// Full complex FFT of G sequences (buf, length N each), scratch tmp (>= G*N); result in buf.
// Caller must __syncthreads() before (inputs ready); returns after a barrier.
template <bool INV>
__device__ void fft_cplx(double2* buf, double2* tmp, int G, const FftDesc& fd, const double2* __restrict__ tw) {
    double2* src = buf;
    double2* dst = tmp;
    for (int k = 0; k < fd.nst; ++k) {
        fft_stage<INV>(src, dst, fd.st[k], fd.N, G, tw);
        __syncthreads();
        double2* t = src;
        src = dst;
        dst = t;
    }
    if (src != buf) {
        for (int i = threadIdx.x; i < G * fd.N; i += blockDim.x) buf[i] = src[i];
        __syncthreads();
    }
}

// c2r pre-pass: Z_k = (X_k + conj X_{N-k}) + i conj(W^k) (X_k - conj X_{N-k}), X_k = 0 for k > R,
// Im X_0 := 0 (transform.cpp:126). row: X_k at row[k * stride] for k <= R.
__device__ __forceinline__ double2 c2r_pre(const double2* __restrict__ row, long stride, int k, int N, int R,
                                           const double2* __restrict__ post) {
    double2 a = (k <= R) ? row[(long)k * stride] : make_double2(0.0, 0.0);
    const int kk = N - k;  // k = 0 -> X_N = 0 since R < N
    double2 bb = (k > 0 && kk <= R) ? row[(long)kk * stride] : make_double2(0.0, 0.0);
    if (k == 0) a.y = 0.0;
    if (kk == 0) bb.y = 0.0;
    const double2 b = cconj(bb);
    const double2 e = cadd(a, b);
    const double2 o = cmul(csub(a, b), cconj(__ldg(post + k)));
    return make_double2(e.x - o.y, e.y + o.x);  // e + i*o
}

// r2c post-pass: X_k = 1/2 (Z_k + conj Z_{N-k}) - i/2 W^k (Z_k - conj Z_{N-k})
__device__ __forceinline__ double2 r2c_post(const double2* __restrict__ z, int k, int N,
                                            const double2* __restrict__ post) {
    const double2 zk = z[k % N];
    const double2 zc = cconj(z[(N - k) % N]);
    const double2 e = make_double2(0.5 * (zk.x + zc.x), 0.5 * (zk.y + zc.y));
    const double2 d = csub(zk, zc);
    const double2 o = make_double2(0.5 * d.y, -0.5 * d.x);  // -i/2 d
    return cadd(e, cmul(__ldg(post + k), o));
}

__global__ void __launch_bounds__(256) fft_c2r_kernel(FftDesc fd, int R, int nlat, const double2* __restrict__ tw,
                                                      const double2* __restrict__ post,
                                                      const double2* __restrict__ four, int in_stride, int in_off,
                                                      double* __restrict__ grid,
                                                      const double* __restrict__ rowc, int div_cos) {
    extern __shared__ double2 sm[];
    const int N = fd.N;
    double2* buf = sm;
    double2* tmp = sm + N;
    const int i = blockIdx.x, b = blockIdx.y;
    const double2* row = four + (((long)b * in_stride + in_off) * nlat + i) * (R + 1);
    for (int k = threadIdx.x; k < N; k += blockDim.x) buf[k] = c2r_pre(row, 1, k, N, R, post);
    __syncthreads();
    fft_cplx<true>(buf, tmp, 1, fd, tw);
    const double c = div_cos ? 1.0 / rowc[i] : 1.0;
    double2* out = (double2*)(grid + ((long)b * nlat + i) * 2 * N);
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        double2 v = buf[k];
        if (div_cos) v = make_double2(v.x * c, v.y * c);
        out[k] = v;
    }
}

__global__ void __launch_bounds__(256) fft_r2c_kernel(FftDesc fd, int R, int nlat, const double2* __restrict__ tw,
                                                      const double2* __restrict__ post,
                                                      const double* __restrict__ grid, double2* __restrict__ four,
                                                      int out_stride, int out_off,
                                                      const double* __restrict__ rowc,
                                                      const double* __restrict__ roww, int pre_cos,
                                                      int scale_mode, double inv_a) {
    extern __shared__ double2 sm[];
    const int N = fd.N;
    double2* buf = sm;
    double2* tmp = sm + N;
    const int i = blockIdx.x, b = blockIdx.y;
    const double2* in = (const double2*)(grid + ((long)b * nlat + i) * 2 * N);
    const double c = rowc[i];
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        double2 v = in[k];
        if (pre_cos) v = make_double2(v.x * c, v.y * c);
        buf[k] = v;
    }
    __syncthreads();
    fft_cplx<false>(buf, tmp, 1, fd, tw);
    const double nl = 2.0 * N;
    const double sc = scale_mode == 0 ? (1.0 / nl) * roww[i] : (1.0 / nl) * (inv_a * roww[i] / (c * c));
    double2* out = four + ((long)b * out_stride + out_off) * (R + 1) * nlat + i;
    for (int k = threadIdx.x; k <= R; k += blockDim.x) {
        const double2 x = r2c_post(buf, k, N, post);
        out[(long)k * nlat] = make_double2(x.x * sc, x.y * sc);
    }
}

// Fused grid stage of eval_nonlinear. four_in [b][4][m][i]: Phi, zeta, U, V Fourier rows.
// four_out [b][5][m][i]: Phi'U, Phi'V, (zeta+f)U, (zeta+f)V (x w/(a cos^2 nlon)), ke (x w/nlon).
__global__ void __launch_bounds__(256) fft_eval_kernel(FftDesc fd, int R, int nlat, int G,
                                                       const double2* __restrict__ tw,
                                                       const double2* __restrict__ post,
                                                       const double2* __restrict__ four_in,
                                                       double2* __restrict__ four_out,
                                                       const double* __restrict__ rowc,
                                                       const double* __restrict__ roww,
                                                       const double* __restrict__ rowmu, double phi_bar,
                                                       double omega, double inv_a) {
    extern __shared__ double2 sm[];
    const int N = fd.N;
    double2* data = sm;            // [5][N]
    double2* tmp = sm + 5 * N;     // [G][N]
    const int i = blockIdx.x, b = blockIdx.y;
    const long rowsz = (long)(R + 1) * nlat;
    const double2* in = four_in + ((long)b * 4 * nlat + i) * (R + 1);
    for (int idx = threadIdx.x; idx < 4 * N; idx += blockDim.x) {
        const int f = idx / N, k = idx - f * N;
        data[idx] = c2r_pre(in + f * rowsz, 1, k, N, R, post);
    }
    __syncthreads();
    for (int f0 = 0; f0 < 4; f0 += G) fft_cplx<true>(data + (long)f0 * N, tmp, min(G, 4 - f0), fd, tw);

    // grid-point products (swe.cpp:41-54), two grid points per complex slot
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
    for (int f0 = 0; f0 < 5; f0 += G) fft_cplx<false>(data + (long)f0 * N, tmp, min(G, 5 - f0), fd, tw);

    const double nl = 2.0 * N;
    const double sflux = (1.0 / nl) * (inv_a * roww[i] / (c * c));
    const double ske = (1.0 / nl) * roww[i];
    double2* out = four_out + (long)b * 5 * rowsz + i;
    for (int idx = threadIdx.x; idx < 5 * (R + 1); idx += blockDim.x) {
        const int q = idx / (R + 1), k = idx - q * (R + 1);
        const double2 x = r2c_post(data + (long)q * N, k, N, post);
        const double sc = q < 4 ? sflux : ske;
        out[q * rowsz + (long)k * nlat] = make_double2(x.x * sc, x.y * sc);
    }
}

}  // namespace

void fft_rows_c2r(const pswe_plan& P, const double2* four, int in_stride, int in_off, double* grid, int n,
                  bool div_cos, cudaStream_t st) {
    if (n <= 0) return;
    if (fft_rows_ip(P, true, four, nullptr, nullptr, grid, in_stride, in_off, n, div_cos, 0, 1.0, st)) return;
    const size_t sm = 2 * (size_t)P.N * sizeof(double2);
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(fft_c2r_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    fft_c2r_kernel<<<dim3(P.nlat, n), 256, sm, st>>>(P.fft, P.R, P.nlat, P.d_fft_tw, P.d_fft_post, four, in_stride,
                                                     in_off, grid, P.d_rowc, div_cos ? 1 : 0);
    PSWE_LAUNCH_CHECK();
}

void fft_rows_r2c(const pswe_plan& P, const double* grid, double2* four, int out_stride, int out_off, int n,
                  bool pre_cos, int scale_mode, double radius, cudaStream_t st) {
    if (n <= 0) return;
    if (fft_rows_ip(P, false, nullptr, grid, four, nullptr, out_stride, out_off, n, pre_cos, scale_mode, radius, st))
        return;
    const size_t sm = 2 * (size_t)P.N * sizeof(double2);
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(fft_r2c_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    fft_r2c_kernel<<<dim3(P.nlat, n), 256, sm, st>>>(P.fft, P.R, P.nlat, P.d_fft_tw, P.d_fft_post, grid, four,
                                                     out_stride, out_off, P.d_rowc, P.d_roww, pre_cos ? 1 : 0, scale_mode,
                                                     1.0 / radius);
    PSWE_LAUNCH_CHECK();
}

void fft_eval_products(const pswe_plan& P, const pswe_params& prm, const double2* four_in, double2* four_out,
                       int n_batch, cudaStream_t st) {
    if (n_batch <= 0) return;
    if (fft_eval_products_ip(P, prm, four_in, four_out, n_batch, st)) return;
    int G = 5;
    size_t sm = (size_t)(5 + G) * P.N * sizeof(double2);
    if (sm > 200 * 1024) {
        G = 1;
        sm = (size_t)(5 + G) * P.N * sizeof(double2);
    }
    if (sm > 48 * 1024) PSWE_CUDA(cudaFuncSetAttribute(fft_eval_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    fft_eval_kernel<<<dim3(P.nlat, n_batch), 256, sm, st>>>(P.fft, P.R, P.nlat, G, P.d_fft_tw, P.d_fft_post,
                                                            four_in, four_out, P.d_rowc, P.d_roww, P.d_rowmu,
                                                            prm.phi_bar, prm.omega, 1.0 / prm.radius);
    PSWE_LAUNCH_CHECK();
}

}  // namespace pswe
