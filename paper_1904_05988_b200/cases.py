"""Seeded initial conditions of BASELINE.json's configs (the reference ships none for these;
its analytic cases live in proj/src/cases.cpp:43-167 and are not used by BASELINE).

* ``balanced_random_state``: vorticity with random complex coefficients for 1 <= n <= R and an
  n^-3 kinetic-energy spectrum, scaled to a target rms velocity; divergence 0; geopotential from
  linear balance  lap(Phi') = div(f grad psi), f = 2 Omega mu;  Phi(0,0) = phi_bar sqrt(2)
  (P^0_0 = 1/sqrt(2), test_transform.cpp:60-61).
* ``add_gaussian_bump``: + g * A exp(-(d/r)^2) at a seeded centre (config 3).
* ``add_zonal_jet``: + u = u0 sin^2(2 phi) in the northern hemisphere (config 4), vorticity and
  divergence by the GPU vortdiv_from_uv, geopotential in gradient-wind balance
  dPhi/dphi = -a u (2 Omega sin phi + u tan phi / a), integrated in latitude with the global mean
  removed (the mean geopotential stays phi_bar).

Host numpy does only coefficient set-up (random draws, spectral scalings) and 1-D latitude
profiles; the grid operations (the bump's and the jet's analysis) run on the GPU through
TransformPlan.

Conventions:
* the rms velocity is the spectral (continuous) one, mean |V|^2 = 1/2 sum' s(s+1)/a^2 |psi_rs|^2
  with weight 1 for r = 0 and 2 for r > 0 (Parseval of test_transform.cpp:133-150);
* linear balance uses the exact spectral form of mu*X and (1-mu^2) dX/dmu of the normalised
  Legendre functions (the recurrences of legendre.cpp / transform.cpp:69-73), truncated at R.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from .transform import TransformPlan, num_coeffs


def _degree_order(R):
    rs = np.concatenate([np.full(R + 1 - r, r) for r in range(R + 1)])
    ss = np.concatenate([np.arange(r, R + 1) for r in range(R + 1)])
    return rs, ss


def _eps(rs, ss):
    s = ss.astype(np.float64)
    r = rs.astype(np.float64)
    with np.errstate(invalid="ignore"):
        e = np.sqrt(np.maximum(s * s - r * r, 0.0) / (4.0 * s * s - 1.0))
    return np.where(ss <= rs, 0.0, e)


def _shift(x, R, rs, ss, d):
    """coefficient at (r, s+d) for every slot (0 outside the triangle)."""
    out = np.zeros_like(x)
    t = ss + d
    ok = (t >= rs) & (t <= R)
    idx = rs * (2 * R + 3 - rs) // 2 + (t - rs)
    out[ok] = x[idx[ok]]
    return out


def balanced_random_state(R: int, rms_wind: float, seed: int, radius: float = 6.37122e6, omega: float = 7.292e-5,
                          phi_bar: float = 9.80616 * 1e4) -> np.ndarray:
    rs, ss = _degree_order(R)
    K = num_coeffs(R)
    rng = np.random.default_rng(seed)
    re = rng.uniform(-1.0, 1.0, K)
    im = rng.uniform(-1.0, 1.0, K)
    im[rs == 0] = 0.0
    n = ss.astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        amp = np.sqrt(n ** -3.0 * n * (n + 1.0) / (2.0 * n + 1.0))
    amp[ss == 0] = 0.0
    zeta = (re + 1j * im) * amp
    a2 = radius * radius
    with np.errstate(divide="ignore", invalid="ignore"):
        psi = np.where(ss > 0, -a2 * zeta / (n * (n + 1.0)), 0.0)
    wgt = np.where(rs == 0, 1.0, 2.0)
    ms = 0.5 * float(np.sum(wgt * n * (n + 1.0) / a2 * np.abs(psi) ** 2))
    scale = rms_wind / math.sqrt(ms)
    zeta *= scale
    psi *= scale
    # linear balance: lap Phi' = 2 Omega [ mu zeta + (1/a^2) (1-mu^2) dpsi/dmu ]
    eps_s = _eps(rs, ss)          # eps^r_s
    eps_s1 = _eps(rs, ss + 1)     # eps^r_{s+1}
    mu_zeta = eps_s * _shift(zeta, R, rs, ss, -1) + eps_s1 * _shift(zeta, R, rs, ss, +1)
    h_psi = -(n - 1.0) * eps_s * _shift(psi, R, rs, ss, -1) + (n + 2.0) * eps_s1 * _shift(psi, R, rs, ss, +1)
    rhs = 2.0 * omega * (mu_zeta + h_psi / a2)
    with np.errstate(divide="ignore", invalid="ignore"):
        phi = np.where(ss > 0, -a2 * rhs / (n * (n + 1.0)), 0.0)
    phi = phi.astype(np.complex128)
    phi[0] = phi_bar * math.sqrt(2.0)
    return np.stack([phi, zeta.astype(np.complex128), np.zeros(K, dtype=np.complex128)])


def add_gaussian_bump(state: np.ndarray, plan: TransformPlan, amplitude_m: float, radius_m: float, seed: int,
                      gravity: float = 9.80616, earth_radius: float = 6.37122e6) -> np.ndarray:
    rng = np.random.default_rng(seed)
    lam_c = rng.uniform(0.0, 2.0 * math.pi)
    phi_c = math.asin(rng.uniform(-0.8, 0.8))
    lat = np.arcsin(plan.mu)
    lam = 2.0 * math.pi * np.arange(plan.nlon) / plan.nlon
    cosd = (np.sin(lat)[:, None] * math.sin(phi_c)
            + np.cos(lat)[:, None] * math.cos(phi_c) * np.cos(lam[None, :] - lam_c))
    d = earth_radius * np.arccos(np.clip(cosd, -1.0, 1.0))
    h = amplitude_m * np.exp(-((d / radius_m) ** 2))
    coef = plan.analyse(torch.as_tensor(gravity * h).cuda()).cpu().numpy()
    out = state.copy()
    out[0] += coef
    return out


def add_zonal_jet(state: np.ndarray, plan: TransformPlan, u0: float = 60.0, radius: float = 6.37122e6,
                  omega: float = 7.292e-5) -> np.ndarray:
    lat = np.arcsin(plan.mu)

    def u_of(phi):
        return np.where(phi > 0.0, u0 * np.sin(2.0 * phi) ** 2, 0.0)

    # gradient-wind balance integrated on a fine latitude grid (u = 0 south of the equator)
    fine = np.linspace(0.0, 0.5 * math.pi, 20001)
    uf = u_of(fine)
    with np.errstate(invalid="ignore"):
        dphi = -radius * uf * (2.0 * omega * np.sin(fine) + uf * np.tan(fine) / radius)
    dphi[-1] = 0.0  # u = 0 at the pole
    prof = np.concatenate([[0.0], np.cumsum(0.5 * (dphi[1:] + dphi[:-1]) * np.diff(fine))])
    geo = np.interp(np.maximum(lat, 0.0), fine, prof)
    geo -= 0.5 * float(np.sum(plan.weight * geo))  # zero global mean (Gauss weights sum to 2)
    ug = np.repeat(u_of(lat)[:, None], plan.nlon, axis=1)
    u = torch.as_tensor(ug).cuda()
    zeta, delta = plan.vortdiv_from_uv(u, torch.zeros_like(u), radius)
    phi_c = plan.analyse(torch.as_tensor(np.repeat(geo[:, None], plan.nlon, axis=1)).cuda())
    out = state.copy()
    out[0] += phi_c.cpu().numpy()
    out[1] += zeta.cpu().numpy()
    out[2] += delta.cpu().numpy()
    return out


def config_state(config: int, plan: TransformPlan | None = None, seed: int = 1904_05988) -> np.ndarray:
    """BASELINE.json configs: 1 (T63, 20 m/s), 3 (T255, 40 m/s + bump), 4 (T511, 20 m/s + zonal
    jet; the rms wind of config 4's random field is not stated, 20 m/s as config 1), 5 (T1023,
    30 m/s)."""
    phi_bar = 9.80616 * 1e4
    if config == 1:
        return balanced_random_state(63, 20.0, seed, phi_bar=phi_bar)
    if config == 3:
        s = balanced_random_state(255 if plan is None else plan.R, 40.0, seed, phi_bar=phi_bar)
        if plan is not None:
            s = add_gaussian_bump(s, plan, 120.0, 5.0e5, seed + 1)
        return s
    if config == 4:
        s = balanced_random_state(511 if plan is None else plan.R, 20.0, seed, phi_bar=phi_bar)
        if plan is not None:
            s = add_zonal_jet(s, plan)
        return s
    if config == 5:
        return balanced_random_state(1023, 30.0, seed, phi_bar=phi_bar)
    raise ValueError("config must be 1, 3, 4 or 5")
