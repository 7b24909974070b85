"""Extended-precision (x87 80-bit long double, eps 1.1e-19) restatement of eval_nonlinear.

TEST INFRASTRUCTURE ONLY (like oracle/pswe_oracle.py). It answers "which implementation drifts":
the same discrete operator as the reference (swe.cpp:27-69 over transform.cpp:136-270 — the
Gauss nodes and weights are the double-precision ones of gauss.cpp:24-50, i.e. exactly the grid
every implementation uses), evaluated with 11 more bits, so its result is the exact value of that
operator to ~1e-17 relative. The GPU path, the reference build (oracle/_ref) and the numpy
restatement are each measured against it (tools/precision_check.py, profiles/r02_precision_*.json).
"""
from __future__ import annotations

import numpy as np

from . import pswe_oracle as O

LD = np.longdouble
CLD = np.clongdouble


def _eps(r, s):
    s = np.asarray(s, dtype=LD)
    r = LD(r)
    out = np.sqrt(np.maximum(s * s - r * r, LD(0)) / (LD(4) * s * s - LD(1)))
    return np.where(s <= r, LD(0), out)


class PrecisePlan:
    """TransformPlan (transform.cpp:45-89) with long-double P / H tables."""

    def __init__(self, R: int, nlat: int, nlon: int):
        self.R, self.nlat, self.nlon = R, nlat, nlon
        mu, w = O.gauss_latitudes(nlat)  # the double nodes of the discrete operator
        self.mu, self.w = mu.astype(LD), w.astype(LD)
        self.cos_phi = np.sqrt(LD(1) - self.mu * self.mu)
        self.offsets = [O.index(R, r, r) for r in range(R + 1)]
        self.p_tab, self.h_tab = [], []
        log_half = np.log(LD(0.5))
        acc = LD(0.5) * log_half  # sectoral_log_amplitude (legendre.cpp:16-20)
        cos2 = LD(1) - self.mu * self.mu
        for r in range(R + 1):
            if r > 0:
                acc += LD(0.5) * np.log(LD(2 * r + 1) / LD(2 * r))
            p = np.zeros((nlat, R + 2 - r), dtype=LD)
            p[:, 0] = np.exp(acc + LD(0.5) * LD(r) * np.log(cos2))
            prev = np.zeros(nlat, dtype=LD)
            for s in range(r, R + 1):  # legendre.cpp:30-37
                p[:, s + 1 - r] = (self.mu * p[:, s - r] - _eps(r, s) * prev) / _eps(r, s + 1)
                prev = p[:, s - r]
            s = np.arange(r, R + 1, dtype=LD)
            upper = -s * _eps(r, s + 1) * p[:, 1:]
            lower = np.zeros_like(upper)
            if R > r:
                lower[:, 1:] = (s[1:] + LD(1)) * _eps(r, s[1:]) * p[:, :-2]
            self.p_tab.append(p)
            self.h_tab.append(upper + lower)

    def fourier_rows(self, g):
        return np.fft.rfft(g, axis=1)[:, : self.R + 1] / LD(self.nlon)

    def inverse_rows(self, rows):
        full = np.zeros((self.nlat, self.nlon // 2 + 1), dtype=CLD)
        full[:, : self.R + 1] = rows
        full[:, 0] = full[:, 0].real
        return np.fft.irfft(full, n=self.nlon, axis=1) * LD(self.nlon)

    def _seg(self, x, r):
        o = self.offsets[r]
        return x[o: o + self.R + 1 - r]

    def synthesise(self, x):
        rows = np.zeros((self.nlat, self.R + 1), dtype=CLD)
        for r in range(self.R + 1):
            rows[:, r] = self.p_tab[r][:, : self.R + 1 - r] @ self._seg(x, r)
        return self.inverse_rows(rows)

    def analyse(self, g):
        rows = self.fourier_rows(g)
        x = np.zeros(O.num_coeffs(self.R), dtype=CLD)
        for r in range(self.R + 1):
            x[self.offsets[r]: self.offsets[r] + self.R + 1 - r] = (self.w * rows[:, r]) @ self.p_tab[r][:, : self.R + 1 - r]
        return x

    def uv_from_vortdiv(self, vort, div, radius):
        psi, chi = _inv_lap(self.R, vort, radius), _inv_lap(self.R, div, radius)
        ur = np.zeros((self.nlat, self.R + 1), dtype=CLD)
        vr = np.zeros_like(ur)
        inv_a = LD(1) / LD(radius)
        for r in range(self.R + 1):
            p, h = self.p_tab[r][:, : self.R + 1 - r], self.h_tab[r]
            ps, ch = self._seg(psi, r), self._seg(chi, r)
            ur[:, r] = inv_a * (1j * LD(r) * (p @ ch) - h @ ps)
            vr[:, r] = inv_a * (1j * LD(r) * (p @ ps) + h @ ch)
        return self.inverse_rows(ur) / self.cos_phi[:, None], self.inverse_rows(vr) / self.cos_phi[:, None]

    def vortdiv_from_uv(self, u, v, radius):
        urows = self.fourier_rows(u * self.cos_phi[:, None])
        vrows = self.fourier_rows(v * self.cos_phi[:, None])
        K = O.num_coeffs(self.R)
        vort, div = np.zeros(K, dtype=CLD), np.zeros(K, dtype=CLD)
        wfac = (LD(1) / LD(radius)) * self.w / (self.cos_phi * self.cos_phi)
        for r in range(self.R + 1):
            ur, vr = wfac * urows[:, r], wfac * vrows[:, r]
            p, h = self.p_tab[r][:, : self.R + 1 - r], self.h_tab[r]
            o, n = self.offsets[r], self.R + 1 - r
            vort[o: o + n] = (1j * LD(r) * vr) @ p + ur @ h
            div[o: o + n] = (1j * LD(r) * ur) @ p - vr @ h
        return vort, div


def _degree(R):
    _, s = O.degree_order(R)
    return s.astype(LD)


def _inv_lap(R, x, radius):
    s = _degree(R)
    with np.errstate(divide="ignore", invalid="ignore"):
        y = np.asarray(x, dtype=CLD) * (-(LD(radius) ** 2) / (s * (s + LD(1))))
    y[s == 0] = 0
    return y


def eval_nonlinear(st, p, plan: PrecisePlan):
    """eval_nonlinear (swe.cpp:27-69) in long double; st is a double (3, K) state."""
    st = np.asarray(st).astype(CLD)
    u, v = plan.uv_from_vortdiv(st[1], st[2], p.radius)
    phi, vort = plan.synthesise(st[0]), plan.synthesise(st[1])
    f = LD(2) * LD(p.omega) * plan.mu[:, None]
    phip, absv = phi - LD(p.phi_bar), vort + f
    ke = LD(0.5) * (u * u + v * v)
    _, flux_div = plan.vortdiv_from_uv(phip * u, phip * v, p.radius)
    q_curl, q_div = plan.vortdiv_from_uv(absv * u, absv * v, p.radius)
    s = _degree(plan.R)
    ke_lap = plan.analyse(ke) * (-s * (s + LD(1)) / LD(p.radius) ** 2)
    return np.stack([-flux_div, -q_div, q_curl - ke_lap])
