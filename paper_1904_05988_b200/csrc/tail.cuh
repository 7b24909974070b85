// Per-coefficient tail of the RHS evaluation (sm_100a, fp64), shared by eval_tail_kernel (ops.cu)
// and the fused tail + node-update kernel of the SDC sweep (sdc.cu): one definition of the
// F_E / F_I expressions.
#pragma once

#include "pswe_internal.h"

namespace pswe {
namespace tailc {

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
// (the lower neighbour's load is clamped rather than branched, so all loads issue together);
// eu = eps_{s+1}, el = eps_s (plan constants: loaded before the programmatic-launch wait)
__device__ __forceinline__ double2 hcomb(const double2* __restrict__ A, double eu, double el, long bx, int m,
                                         int s) {
    const int t = s - m;
    const double fu = -(double)s * eu;
    const double2 up = A[bx + t + 1];
    const double2 lo = A[bx + (t > 0 ? t - 1 : 0)];
    double2 h = make_double2(fu * up.x, fu * up.y);
    if (t > 0) {
        const double fl = (s + 1.0) * el;
        h.x += fl * lo.x;
        h.y += fl * lo.y;
    }
    return h;
}
__device__ __forceinline__ double2 hcomb(const double2* __restrict__ A, const double* __restrict__ eps, long bx,
                                         int m, int s) {
    return hcomb(A, eps[bx + s - m + 1], eps[bx + s - m], bx, m, s);
}

// Field f (0 Phi, 1 zeta, 2 delta) of the eval_nonlinear assembly (swe.cpp:61-67) from the five
// projections A1..A5 (A = proj of this state, extended layout, s = m..R+1; eu, el as hcomb) and of eval_linear
// (swe.cpp:9-25, only if need_fi) of the state st (3K) at coefficient k = (m, s), lam = -s(s+1)/a^2:
//   Phi_t  = -(i m A1 - H[A2])          (-flux_div)
//   zeta_t = -(i m A3 - H[A4])          (-q_div)
//   div_t  = (i m A4 + H[A3]) - lap(A5) (q_curl - lap ke)
__device__ __forceinline__ void tail_field(int f, double eu, double el, const double2* __restrict__ A,
                                           long Kx, long bx, int m, int s, double lam,
                                           const double2* __restrict__ st, long K, long k, double phi_bar,
                                           double nu, bool need_fi, double2& fe, double2& fi) {
    const long o = bx + s - m;
    if (f == 0) {
        const double2 a1 = A[o];
        const double2 h2 = hcomb(A + Kx, eu, el, bx, m, s);
        const double2 fdiv = make_double2(-m * a1.y - h2.x, m * a1.x - h2.y);
        fe = make_double2(-fdiv.x, -fdiv.y);
        if (!need_fi) return;
        const double2 ph = st[k], dv = st[2 * K + k];
        fi = make_double2(-phi_bar * dv.x + nu * lam * ph.x, -phi_bar * dv.y + nu * lam * ph.y);
    } else if (f == 1) {
        const double2 a3 = A[2 * Kx + o];
        const double2 h4 = hcomb(A + 3 * Kx, eu, el, bx, m, s);
        const double2 qdiv = make_double2(-m * a3.y - h4.x, m * a3.x - h4.y);
        fe = make_double2(-qdiv.x, -qdiv.y);
        if (!need_fi) return;
        const double2 vo = st[K + k];
        fi = make_double2(nu * lam * vo.x, nu * lam * vo.y);
    } else {
        const double2 a4 = A[3 * Kx + o], a5 = A[4 * Kx + o];
        const double2 h3 = hcomb(A + 2 * Kx, eu, el, bx, m, s);
        const double2 qcurl = make_double2(-m * a4.y + h3.x, m * a4.x + h3.y);
        const double2 kel = make_double2(lam * a5.x, lam * a5.y);
        fe = make_double2(qcurl.x - kel.x, qcurl.y - kel.y);
        if (!need_fi) return;
        const double2 ph = st[k], dv = st[2 * K + k];
        fi = make_double2(-lam * ph.x + nu * lam * dv.x, -lam * ph.y + nu * lam * dv.y);
    }
}

}  // namespace tailc
}  // namespace pswe
