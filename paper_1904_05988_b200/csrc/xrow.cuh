// One degree's inverse-Legendre coefficient columns {Phi, zeta, U, V} of one state (the evaluation's
// X-tile row entries), transform.cpp:176-223 with the H-sums rewritten as P-sums over the
// neighbouring degrees: U = u cos(phi), V = v cos(phi) from psi = inv_laplacian(zeta),
// chi = inv_laplacian(delta). Shared by the prep kernel of one/two-state evaluations
// (legendre_stream.cu) and the SDC sweep kernel that emits the next node's X tiles (sdc.cu), so
// both produce the same bits. Degree s of order m (t = s - m), s = m..R+1; values past R are zero.
#pragma once

#include "pswe_internal.h"

namespace pswe {
namespace xrow {

struct Fac {
    double fm, f0, fp, hm, hp;  // inverse Laplacian factors at s-1, s, s+1; H-sum weights
};

// eps: extended-layout epsilon table, rtab[s] = 1/(s(s+1)); bx = off_ext(R, m)
__device__ __forceinline__ Fac factors(int R, int m, int s, long bx, const double* __restrict__ eps,
                                       const double* __restrict__ rtab, double radius) {
    const double a2 = radius * radius;
    const int t = s - m, s0 = min(s, R);
    const double rm = __ldg(rtab + max(s - 1, 0)), r0 = __ldg(rtab + s0), rp = __ldg(rtab + min(s + 1, R));
    const double em = eps[bx + t], ep = eps[bx + min(t + 1, R + 1 - m)];
    Fac F;
    F.fm = (s - 1 >= m && s - 1 >= 1) ? -a2 * rm : 0.0;
    F.f0 = (s <= R && s >= 1) ? -a2 * r0 : 0.0;
    F.fp = (s + 1 <= R) ? -a2 * rp : 0.0;
    F.hm = (s - 1 >= m) ? -(double)(s - 1) * em : 0.0;
    F.hp = (s + 1 <= R) ? (double)(s + 2) * ep : 0.0;
    return F;
}

// ph = Phi(s), v* = zeta and d* = delta at (s-1, s, s+1) clamped into m..R (values at clamped
// positions are not used)
__device__ __forceinline__ void columns(const Fac& F, int R, int m, int s, double radius, double2 ph, double2 vm,
                                        double2 v0, double2 vp, double2 dm, double2 d0, double2 dp,
                                        double2 (&v)[4]) {
    const double inv_a = 1.0 / radius;
    v[0] = v[1] = make_double2(0.0, 0.0);
    if (s <= R) {
        v[0] = ph;
        v[1] = v0;
    }
    const double2 chi = make_double2(d0.x * F.f0, d0.y * F.f0);
    const double2 psi = make_double2(v0.x * F.f0, v0.y * F.f0);
    double2 cpsi = make_double2(0.0, 0.0), cchi = make_double2(0.0, 0.0);
    if (s - 1 >= m) {
        cpsi.x += F.hm * (vm.x * F.fm);
        cpsi.y += F.hm * (vm.y * F.fm);
        cchi.x += F.hm * (dm.x * F.fm);
        cchi.y += F.hm * (dm.y * F.fm);
    }
    if (s + 1 <= R) {
        cpsi.x += F.hp * (vp.x * F.fp);
        cpsi.y += F.hp * (vp.y * F.fp);
        cchi.x += F.hp * (dp.x * F.fp);
        cchi.y += F.hp * (dp.y * F.fp);
    }
    v[2] = make_double2(inv_a * (-m * chi.y - cpsi.x), inv_a * (m * chi.x - cpsi.y));
    v[3] = make_double2(inv_a * (-m * psi.y + cchi.x), inv_a * (m * psi.x + cchi.y));
}

}  // namespace xrow
}  // namespace pswe
