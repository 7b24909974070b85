// Spectral-space elementwise / banded kernels (sm_100a, fp64): the tails of eval_nonlinear and
// vortdiv_from_uv, eval_linear, solve_implicit, laplacian.
#include "pswe_internal.h"
#include "tail.cuh"

namespace pswe {

namespace {

__device__ __forceinline__ double2 cz() { return make_double2(0.0, 0.0); }

using tailc::decode_rs;
using tailc::hcomb;

// eval_nonlinear assembly (swe.cpp:61-67) plus eval_linear (swe.cpp:9-25) of the same state, one
// thread per coefficient doing the three fields (tail.cuh: tail_field)
__global__ void eval_tail_kernel(int R, const double* __restrict__ eps, const double2* __restrict__ proj,
                                 const double2* __restrict__ state, double2* __restrict__ f_imp,
                                 double2* __restrict__ f_exp, double inv_a2, double phi_bar, double nu) {
    const long K = (long)(R + 1) * (R + 2) / 2;
    const long Kx = (long)(R + 1) * (R + 4) / 2;
    const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    pdl_trigger();
    // plan constants first: they overlap the forward kernel's tail
    int m = 0, s = 0;
    double eu = 0.0, el = 0.0;
    if (k < K) {
        decode_rs(R, k, m, s);
        eu = eps[off_ext(R, m) + s - m + 1];
        el = eps[off_ext(R, m) + s - m];
    }
    pdl_wait();  // the projections come from the forward Legendre kernel
    if (k >= K) return;
    const long bx = off_ext(R, m);
    const double2* A = proj + (long)b * 5 * Kx;
    const double lam = -s * (s + 1.0) * inv_a2;
    const double2* st = state + (long)b * 3 * K;
    double2* fe = f_exp + (long)b * 3 * K;
    double2* fi = f_imp ? f_imp + (long)b * 3 * K : nullptr;
    double2 e[3], i[3];  // every load before any store
#pragma unroll
    for (int f = 0; f < 3; ++f)
        tailc::tail_field(f, eu, el, A, Kx, bx, m, s, lam, st, K, k, phi_bar, nu, fi != nullptr, e[f], i[f]);
#pragma unroll
    for (int f = 0; f < 3; ++f) {
        fe[f * K + k] = e[f];
        if (fi) fi[f * K + k] = i[f];
    }
}

// vortdiv_from_uv assembly (transform.cpp:263-266): zeta = i m A_V + H[A_U], delta = i m A_U - H[A_V]
__global__ void vortdiv_tail_kernel(int R, const double* __restrict__ eps, const double2* __restrict__ proj,
                                    double2* __restrict__ vort, double2* __restrict__ div) {
    const long K = (long)(R + 1) * (R + 2) / 2;
    const long Kx = (long)(R + 1) * (R + 4) / 2;
    const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (k >= K) return;
    int m, s;
    decode_rs(R, k, m, s);
    const long bx = off_ext(R, m);
    const double2* AU = proj + (long)b * 2 * Kx;
    const double2* AV = AU + Kx;
    const double2 au = AU[bx + s - m], av = AV[bx + s - m];
    const double2 hu = hcomb(AU, eps, bx, m, s), hv = hcomb(AV, eps, bx, m, s);
    vort[(long)b * K + k] = make_double2(-m * av.y + hu.x, m * av.x + hu.y);
    div[(long)b * K + k] = make_double2(-m * au.y - hv.x, m * au.x - hv.y);
}

__global__ void eval_linear_kernel(int R, const double2* __restrict__ state, double2* __restrict__ out,
                                   double inv_a2, double phi_bar, double nu) {
    const long K = (long)(R + 1) * (R + 2) / 2;
    const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (k >= K) return;
    int m, s;
    decode_rs(R, k, m, s);
    const double lam = -s * (s + 1.0) * inv_a2;
    const double2* st = state + (long)b * 3 * K;
    const double2 ph = st[k], vo = st[K + k], dv = st[2 * K + k];
    double2* o = out + (long)b * 3 * K;
    o[k] = make_double2(-phi_bar * dv.x + nu * lam * ph.x, -phi_bar * dv.y + nu * lam * ph.y);
    o[K + k] = make_double2(nu * lam * vo.x, nu * lam * vo.y);
    o[2 * K + k] = make_double2(-lam * ph.x + nu * lam * dv.x, -lam * ph.y + nu * lam * dv.y);
}

// solve_implicit (swe.cpp:77-98): diffusion rescaling then the analytic 2x2 gravity-wave solve
__global__ void solve_implicit_kernel(int R, const double2* __restrict__ bin, double c, double2* __restrict__ out,
                                      double inv_a2, double phi_bar, double nu) {
    const long K = (long)(R + 1) * (R + 2) / 2;
    const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (k >= K) return;
    int m, s;
    decode_rs(R, k, m, s);
    const double lam = -s * (s + 1.0) * inv_a2;
    const double diff = 1.0 - c * nu * lam;
    const double2* bb = bin + (long)b * 3 * K;
    const double2 bp = make_double2(bb[k].x / diff, bb[k].y / diff);
    const double2 bz = make_double2(bb[K + k].x / diff, bb[K + k].y / diff);
    const double2 bd = make_double2(bb[2 * K + k].x / diff, bb[2 * K + k].y / diff);
    const double ce = c / diff;
    const double det = 1.0 - ce * ce * phi_bar * lam;
    double2* o = out + (long)b * 3 * K;
    o[k] = make_double2((bp.x - ce * phi_bar * bd.x) / det, (bp.y - ce * phi_bar * bd.y) / det);
    o[2 * K + k] = make_double2((bd.x - ce * lam * bp.x) / det, (bd.y - ce * lam * bp.y) / det);
    o[K + k] = bz;
}

__global__ void laplacian_kernel(int R, const double2* __restrict__ x, double radius, double2* __restrict__ y,
                                 int inverse) {
    const long K = (long)(R + 1) * (R + 2) / 2;
    const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (k >= K) return;
    int m, s;
    decode_rs(R, k, m, s);
    const double2 v = x[(long)b * K + k];
    double2 r;
    if (!inverse) {
        const double f = -s * (s + 1.0) * (1.0 / (radius * radius));
        r = make_double2(f * v.x, f * v.y);
    } else if (s == 0) {
        r = cz();
    } else {
        const double f = -(radius * radius) / (s * (s + 1.0));
        r = make_double2(v.x * f, v.y * f);
    }
    y[(long)b * K + k] = r;
}

}  // namespace

static dim3 grid_k(int R, int n, int bs) {
    const long K = num_coeffs(R);
    return dim3((unsigned)((K + bs - 1) / bs), n);
}

void eval_tail(const pswe_plan& P, const pswe_params& prm, const double2* proj, const double2* state,
               double2* f_imp, double2* f_exp, int n_batch, cudaStream_t st) {
    if (n_batch <= 0) return;
    launch_pdl(eval_tail_kernel, grid_k(P.R, n_batch, 128), dim3(128), 0, st, P.R, P.d_eps, proj, state, f_imp, f_exp,
                                                                1.0 / (prm.radius * prm.radius), prm.phi_bar,
                                                                prm.nu);
    PSWE_LAUNCH_CHECK();
}

void vortdiv_tail(const pswe_plan& P, const double2* proj, double2* vort, double2* div, int n_pairs,
                  cudaStream_t st) {
    if (n_pairs <= 0) return;
    vortdiv_tail_kernel<<<grid_k(P.R, n_pairs, 128), 128, 0, st>>>(P.R, P.d_eps, proj, vort, div);
    PSWE_LAUNCH_CHECK();
}

void eval_linear(int R, const pswe_params& prm, const double2* state, double2* out, int n, cudaStream_t st) {
    if (n <= 0) return;
    eval_linear_kernel<<<grid_k(R, n, 128), 128, 0, st>>>(R, state, out, 1.0 / (prm.radius * prm.radius),
                                                          prm.phi_bar, prm.nu);
    PSWE_LAUNCH_CHECK();
}

void solve_implicit(int R, const pswe_params& prm, const double2* b, double c, double2* out, int n,
                    cudaStream_t st) {
    if (n <= 0) return;
    solve_implicit_kernel<<<grid_k(R, n, 128), 128, 0, st>>>(R, b, c, out, 1.0 / (prm.radius * prm.radius),
                                                             prm.phi_bar, prm.nu);
    PSWE_LAUNCH_CHECK();
}

void laplacian(int R, const double2* x, double radius, double2* y, int n, bool inverse, cudaStream_t st) {
    if (n <= 0) return;
    laplacian_kernel<<<grid_k(R, n, 128), 128, 0, st>>>(R, x, radius, y, inverse ? 1 : 0);
    PSWE_LAUNCH_CHECK();
}

}  // namespace pswe
