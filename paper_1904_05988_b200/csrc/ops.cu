// Spectral-space elementwise / banded kernels (sm_100a, fp64): the tails of eval_nonlinear and
// vortdiv_from_uv, eval_linear, solve_implicit, laplacian.
#include "pswe_internal.h"

namespace pswe {

namespace {

__device__ __forceinline__ double2 cz() { return make_double2(0.0, 0.0); }

// (r, s) of r-major index k (field.hpp:29-32)
__device__ __forceinline__ void decode_rs(int R, long k, int& m, int& s) {
    const double b = 2.0 * R + 3.0;
    int mm = (int)floor((b - sqrt(b * b - 8.0 * (double)k)) * 0.5);
    if (mm < 0) mm = 0;
    if (mm > R) mm = R;
    while (mm > 0 && off_std(R, mm) > k) --mm;
    while (mm < R && off_std(R, mm + 1) <= k) ++mm;
    m = mm;
    s = mm + (int)(k - off_std(R, mm));
}

// H-combination of a projection A (extended layout, block m): H_s = -s eps_{s+1} A_{s+1} + (s+1) eps_s A_{s-1}
// (the lower neighbour's load is clamped rather than branched, so all loads issue together)
__device__ __forceinline__ double2 hcomb(const double2* __restrict__ A, const double* __restrict__ eps, long bx,
                                         int m, int s) {
    const int t = s - m;
    const double fu = -(double)s * eps[bx + t + 1];
    const double2 up = A[bx + t + 1];
    const double el = eps[bx + t];
    const double2 lo = A[bx + (t > 0 ? t - 1 : 0)];
    double2 h = make_double2(fu * up.x, fu * up.y);
    if (t > 0) {
        const double fl = (s + 1.0) * el;
        h.x += fl * lo.x;
        h.y += fl * lo.y;
    }
    return h;
}

// eval_nonlinear assembly (swe.cpp:61-67) from the five projections A1..A5 (extended layout,
// s = m..R+1) plus eval_linear (swe.cpp:9-25) of the same state:
//   Phi_t  = -(i m A1 - H[A2])          (-flux_div)
//   zeta_t = -(i m A3 - H[A4])          (-q_div)
//   div_t  = (i m A4 + H[A3]) - lap(A5) (q_curl - lap ke)
__global__ void eval_tail_kernel(int R, const double* __restrict__ eps, const double2* __restrict__ proj,
                                 const double2* __restrict__ state, double2* __restrict__ f_imp,
                                 double2* __restrict__ f_exp, double inv_a2, double phi_bar, double nu) {
    const long K = (long)(R + 1) * (R + 2) / 2;
    const long Kx = (long)(R + 1) * (R + 4) / 2;
    const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    pdl_trigger();
    pdl_wait();  // the projections come from the forward Legendre kernel
    if (k >= K) return;
    int m, s;
    decode_rs(R, k, m, s);
    const long bx = off_ext(R, m);
    const double2* A = proj + (long)b * 5 * Kx;
    const double2 a1 = A[bx + s - m], a3 = A[2 * Kx + bx + s - m], a4 = A[3 * Kx + bx + s - m];
    const double2 a5 = A[4 * Kx + bx + s - m];
    const double2 h2 = hcomb(A + Kx, eps, bx, m, s), h3 = hcomb(A + 2 * Kx, eps, bx, m, s);
    const double2 h4 = hcomb(A + 3 * Kx, eps, bx, m, s);
    const double lam = -s * (s + 1.0) * inv_a2;
    // flux_div = i m a1 - h2
    const double2 fdiv = make_double2(-m * a1.y - h2.x, m * a1.x - h2.y);
    const double2 qdiv = make_double2(-m * a3.y - h4.x, m * a3.x - h4.y);
    const double2 qcurl = make_double2(-m * a4.y + h3.x, m * a4.x + h3.y);
    const double2 kel = make_double2(lam * a5.x, lam * a5.y);
    double2* fe = f_exp + (long)b * 3 * K;
    fe[k] = make_double2(-fdiv.x, -fdiv.y);
    fe[K + k] = make_double2(-qdiv.x, -qdiv.y);
    fe[2 * K + k] = make_double2(qcurl.x - kel.x, qcurl.y - kel.y);
    if (f_imp) {
        const double2* st = state + (long)b * 3 * K;
        const double2 ph = st[k], vo = st[K + k], dv = st[2 * K + k];
        double2* fi = f_imp + (long)b * 3 * K;
        fi[k] = make_double2(-phi_bar * dv.x + nu * lam * ph.x, -phi_bar * dv.y + nu * lam * ph.y);
        fi[K + k] = make_double2(nu * lam * vo.x, nu * lam * vo.y);
        fi[2 * K + k] = make_double2(-lam * ph.x + nu * lam * dv.x, -lam * ph.y + nu * lam * dv.y);
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
