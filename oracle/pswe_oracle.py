"""CPU restatement (numpy) of the reference PFASST-SH hot path.

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` leg may import this module, and only as the checker. The product path
(``paper_1904_05988_b200``) never imports it and fails loudly without its CUDA library.

Parity of this restatement is pinned against the reference itself: ``oracle/_ref`` (the
reference C++ compiled from /root/reference/proj/src by ``oracle/build_ref.sh``) generated the
fixtures in ``tests/golden/`` (script: ``oracle/make_golden.py``) and
``tests/test_oracle_golden.py`` checks every function below against them.

Layout conventions (reference ``proj/include/pintswe/field.hpp:14-111``, ``grid.hpp:14-37``):
* a spectral field is a complex128 vector of K = (R+1)(R+2)/2 coefficients, r-major,
  ``index(r, s) = r(2R+3-r)/2 + (s-r)`` (field.hpp:29-32);
* a state is an array (3, K): (Phi, zeta, delta);
* a grid is (nlat, nlon) real, rows south -> north at the Gauss nodes, lambda_j = 2 pi j/nlon.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------------------------
# indexing


def num_coeffs(R: int) -> int:
    """SpectralField::size (field.hpp:21-23)."""
    return (R + 1) * (R + 2) // 2


def index(R: int, r: int, s: int) -> int:
    """SpectralField::index (field.hpp:29-32)."""
    return r * (2 * R + 3 - r) // 2 + (s - r)


def degree_order(R: int):
    """Arrays (r, s) of each r-major slot."""
    rs = np.concatenate([np.full(R + 1 - r, r) for r in range(R + 1)])
    ss = np.concatenate([np.arange(r, R + 1) for r in range(R + 1)])
    return rs, ss


# ----------------------------------------------------------------------------------------------
# numerical setup


def _legendre_pn(n, x):
    """legendre_pn (gauss.cpp:11-20), vectorised over x with the same operation order."""
    p0 = np.ones_like(x)
    p1 = x.copy()
    for k in range(2, n + 1):
        p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k
        p0, p1 = p1, p2
    dp = n * (x * p1 - p0) / (x * x - 1.0)
    return p1, dp


def gauss_latitudes(n: int):
    """gauss_latitudes (gauss.cpp:24-50): Newton on P_n from cos(pi(i+3/4)/(n+1/2)), |dx| < 1e-15,
    w = 2/((1-x^2) P_n'^2), stored ascending and symmetric."""
    if n < 1:
        raise ValueError("gauss_latitudes: need n >= 1")
    half = (n + 1) // 2
    i = np.arange(half, dtype=np.float64)
    x = np.cos(math.pi * (i + 0.75) / (n + 0.5))
    active = np.ones(half, dtype=bool)
    for _ in range(100):
        if not active.any():
            break
        p, dp = _legendre_pn(n, x[active])
        dx = p / dp
        xa = x[active] - dx
        x[active] = xa
        idx = np.nonzero(active)[0]
        active[idx[np.abs(dx) < 1e-15]] = False
    p, dp = _legendre_pn(n, x)
    w = 2.0 / ((1.0 - x * x) * dp * dp)
    mu = np.zeros(n)
    wt = np.zeros(n)
    mu[n - 1 - np.arange(half)] = x
    mu[np.arange(half)] = -x
    wt[n - 1 - np.arange(half)] = w
    wt[np.arange(half)] = w
    if n % 2 == 1:
        mu[n // 2] = 0.0
    return mu, wt


def legendre_eps(r: int, s):
    """legendre_eps (legendre.cpp:7-11): sqrt((s^2-r^2)/(4s^2-1)), 0 for s <= r."""
    s = np.asarray(s, dtype=np.float64)
    out = np.sqrt(np.maximum(s * s - r * r, 0.0) / (4.0 * s * s - 1.0))
    return np.where(s <= r, 0.0, out)


def sectoral_log_amplitude(r: int) -> float:
    """sectoral_log_amplitude (legendre.cpp:16-20)."""
    acc = 0.5 * math.log(0.5)
    for k in range(1, r + 1):
        acc += 0.5 * math.log((2.0 * k + 1.0) / (2.0 * k))
    return acc


def legendre_columns(r: int, smax: int, mu: np.ndarray) -> np.ndarray:
    """legendre_column (legendre.cpp:24-38) for all mu at once: returns (len(mu), smax-r+1),
    P^r_s(mu) for s = r..smax. Log-space sectoral seed, then the normalised 3-term recurrence."""
    mu = np.asarray(mu, dtype=np.float64)
    cos2 = 1.0 - mu * mu
    log_seed = sectoral_log_amplitude(r) + 0.5 * r * np.log(cos2)
    out = np.zeros((mu.size, smax - r + 1))
    pmm = np.exp(log_seed)
    out[:, 0] = pmm
    prev = np.zeros_like(mu)
    curr = pmm
    for s in range(r, smax):
        nxt = (mu * curr - float(legendre_eps(r, s)) * prev) / float(legendre_eps(r, s + 1))
        out[:, s + 1 - r] = nxt
        prev, curr = curr, nxt
    return out


def dealiased_nlon(R: int) -> int:
    """dealiased_nlon (transform.cpp:38-43): smallest even 5-smooth n >= 3R+1."""
    def smooth(n):
        for p in (2, 3, 5):
            while n % p == 0:
                n //= p
        return n == 1
    n = 3 * R + 1
    if n % 2:
        n += 1
    while not smooth(n):
        n += 2
    return n


# ----------------------------------------------------------------------------------------------
# transform plan (transform.cpp:45-290)


class TransformPlan:
    """Restatement of TransformPlan (transform.hpp:27-96, transform.cpp:45-290). An explicit grid
    may be given (the reference always uses the dealiased grid of transform.cpp:45-48)."""

    def __init__(self, R: int, nlat: int | None = None, nlon: int | None = None):
        if R < 1:
            raise ValueError("TransformPlan: truncation must be >= 1")
        self.R = R
        self.nlon = nlon if nlon else dealiased_nlon(R)
        self.nlat = nlat if nlat else self.nlon // 2
        self.mu, self.w = gauss_latitudes(self.nlat)
        self.cos_phi = np.sqrt(1.0 - self.mu * self.mu)
        self.p_tab = []  # [r] -> (nlat, R+2-r)
        self.h_tab = []  # [r] -> (nlat, R+1-r)
        for r in range(R + 1):
            p = legendre_columns(r, R + 1, self.mu)
            s = np.arange(r, R + 1, dtype=np.float64)
            upper = -s * legendre_eps(r, s + 1) * p[:, 1:]
            lower = np.zeros_like(upper)
            if R > r:
                lower[:, 1:] = (s[1:] + 1.0) * legendre_eps(r, s[1:]) * p[:, :-2]
            self.p_tab.append(p)
            self.h_tab.append(upper + lower)
        self.offsets = [index(R, r, r) for r in range(R + 1)]

    # fourier_rows (transform.cpp:97-115): r2c per row, x 1/nlon, keep r <= R
    def fourier_rows(self, g):
        return np.fft.rfft(np.asarray(g, dtype=np.float64), axis=1)[:, : self.R + 1] / self.nlon

    # inverse_rows (transform.cpp:117-134): c2r with Im G_0 := 0, r > R := 0 (unnormalised)
    def inverse_rows(self, rows):
        full = np.zeros((self.nlat, self.nlon // 2 + 1), dtype=np.complex128)
        full[:, : self.R + 1] = rows
        full[:, 0] = full[:, 0].real
        return np.fft.irfft(full, n=self.nlon, axis=1) * self.nlon

    def _seg(self, x, r):
        o = self.offsets[r]
        return x[o : o + self.R + 1 - r]

    def analyse(self, g):
        """analyse (transform.cpp:136-153): x^r_s = sum_i w_i G^r_i P^r_s(mu_i)."""
        rows = self.fourier_rows(g)
        x = np.zeros(num_coeffs(self.R), dtype=np.complex128)
        for r in range(self.R + 1):
            gw = self.w * rows[:, r]
            x[self.offsets[r] : self.offsets[r] + self.R + 1 - r] = gw @ self.p_tab[r][:, : self.R + 1 - r]
        return x

    def synthesise(self, x):
        """synthesise (transform.cpp:155-174): G^r_i = sum_s x^r_s P^r_s(mu_i), then c2r."""
        rows = np.zeros((self.nlat, self.R + 1), dtype=np.complex128)
        for r in range(self.R + 1):
            rows[:, r] = self.p_tab[r][:, : self.R + 1 - r] @ self._seg(x, r)
        return self.inverse_rows(rows)

    def uv_from_vortdiv(self, vort, div, radius):
        """uv_from_vortdiv (transform.cpp:176-223)."""
        psi = inv_laplacian(self.R, vort, radius)
        chi = inv_laplacian(self.R, div, radius)
        ur = np.zeros((self.nlat, self.R + 1), dtype=np.complex128)
        vr = np.zeros_like(ur)
        inv_a = 1.0 / radius
        for r in range(self.R + 1):
            p = self.p_tab[r][:, : self.R + 1 - r]
            h = self.h_tab[r]
            ps, ch = self._seg(psi, r), self._seg(chi, r)
            psi_p, chi_p, psi_h, chi_h = p @ ps, p @ ch, h @ ps, h @ ch
            ur[:, r] = inv_a * (1j * r * chi_p - psi_h)
            vr[:, r] = inv_a * (1j * r * psi_p + chi_h)
        u = self.inverse_rows(ur) / self.cos_phi[:, None]
        v = self.inverse_rows(vr) / self.cos_phi[:, None]
        return u, v

    def vortdiv_from_uv(self, u, v, radius):
        """vortdiv_from_uv (transform.cpp:225-270)."""
        uc = np.asarray(u) * self.cos_phi[:, None]
        vc = np.asarray(v) * self.cos_phi[:, None]
        urows, vrows = self.fourier_rows(uc), self.fourier_rows(vc)
        K = num_coeffs(self.R)
        vort = np.zeros(K, dtype=np.complex128)
        div = np.zeros(K, dtype=np.complex128)
        wfac = (1.0 / radius) * self.w / (self.cos_phi * self.cos_phi)
        for r in range(self.R + 1):
            ur = wfac * urows[:, r]
            vr = wfac * vrows[:, r]
            p = self.p_tab[r][:, : self.R + 1 - r]
            h = self.h_tab[r]
            o = self.offsets[r]
            n = self.R + 1 - r
            vort[o : o + n] = (1j * r * vr) @ p + ur @ h
            div[o : o + n] = (1j * r * ur) @ p - vr @ h
        return vort, div


def laplacian(R, x, radius):
    """laplacian (transform.cpp:272-280): x (-s(s+1)/a^2)."""
    _, s = degree_order(R)
    return -s * (s + 1.0) * (1.0 / (radius * radius)) * np.asarray(x)


def inv_laplacian(R, x, radius):
    """inv_laplacian (transform.cpp:282-290): x (-a^2/(s(s+1))), (0,0) := 0."""
    _, s = degree_order(R)
    a2 = radius * radius
    with np.errstate(divide="ignore", invalid="ignore"):
        y = np.asarray(x) * (-a2 / (s * (s + 1.0)))
    y[s == 0] = 0.0
    return y


# ----------------------------------------------------------------------------------------------
# direct-sum transforms (reference.cpp:15-108), arbitrary latitude sets


def direct_synthesise(R, x, mu, nlon):
    """reference::synthesise (reference.cpp:28-44)."""
    mu = np.asarray(mu)
    lam = 2.0 * math.pi * np.arange(nlon) / nlon
    out = np.zeros((mu.size, nlon))
    for r in range(R + 1):
        p = legendre_columns(r, R, mu)  # (nlat, R+1-r)
        g = p @ x[index(R, r, r) : index(R, r, r) + R + 1 - r]
        if r == 0:
            out += g.real[:, None]
        else:
            out += 2.0 * (np.outer(g.real, np.cos(r * lam)) - np.outer(g.imag, np.sin(r * lam)))
    return out


# ----------------------------------------------------------------------------------------------
# SWE right-hand side (swe.hpp:13-79, swe.cpp:9-98)


@dataclass
class ModelParams:
    """ModelParams (swe.hpp:13-19)."""
    radius: float = 6.37122e6
    omega: float = 7.292e-5
    gravity: float = 9.80616
    phi_bar: float = 9.80616 * 29400.0
    nu: float = 0.0


def eval_linear(R, st, p: ModelParams):
    """eval_linear (swe.cpp:9-25)."""
    _, s = degree_order(R)
    lam = -s * (s + 1.0) * (1.0 / (p.radius * p.radius))
    phi, vor, div = st
    out = np.empty_like(st)
    out[0] = -p.phi_bar * div + p.nu * lam * phi
    out[1] = p.nu * lam * vor
    out[2] = -lam * phi + p.nu * lam * div
    return out


def eval_nonlinear(st, p: ModelParams, plan: TransformPlan):
    """eval_nonlinear (swe.cpp:27-69)."""
    u, v = plan.uv_from_vortdiv(st[1], st[2], p.radius)
    phi = plan.synthesise(st[0])
    vort = plan.synthesise(st[1])
    f = 2.0 * p.omega * plan.mu[:, None]
    phip = phi - p.phi_bar
    absv = vort + f
    fu, fv = phip * u, phip * v
    qu, qv = absv * u, absv * v
    ke = 0.5 * (u * u + v * v)
    _, flux_div = plan.vortdiv_from_uv(fu, fv, p.radius)
    q_curl, q_div = plan.vortdiv_from_uv(qu, qv, p.radius)
    ke_lap = laplacian(plan.R, plan.analyse(ke), p.radius)
    return np.stack([-flux_div, -q_div, q_curl - ke_lap])


def solve_implicit(R, b, c, p: ModelParams):
    """solve_implicit (swe.cpp:77-98): diffusion rescaling, then the analytic 2x2 solve."""
    _, s = degree_order(R)
    lam = -s * (s + 1.0) * (1.0 / (p.radius * p.radius))
    diff = 1.0 - c * p.nu * lam
    bp, bz, bd = b[0] / diff, b[1] / diff, b[2] / diff
    ce = c / diff
    det = 1.0 - ce * ce * p.phi_bar * lam
    out = np.empty_like(b)
    out[0] = (bp - ce * p.phi_bar * bd) / det
    out[2] = (bd - ce * lam * bp) / det
    out[1] = bz
    return out


class SweOde:
    """SweOde (swe.hpp:57-79), the ImexOde implementation."""

    def __init__(self, plan: TransformPlan, params: ModelParams):
        self.plan, self.params = plan, params

    def truncation(self):
        return self.plan.R

    def eval_implicit(self, st):
        return eval_linear(self.plan.R, st, self.params)

    def eval_explicit(self, st):
        return eval_nonlinear(st, self.params, self.plan)

    def solve_implicit(self, b, c):
        return solve_implicit(self.plan.R, b, c, self.params)


# ----------------------------------------------------------------------------------------------
# quadrature (quadrature.cpp:8-106)


def lobatto_nodes(n):
    """lobatto_nodes (quadrature.cpp:57-70)."""
    if n == 2:
        return [0.0, 1.0]
    if n == 3:
        return [0.0, 0.5, 1.0]
    if n == 5:
        c = math.sqrt(3.0 / 7.0)
        return [0.0, 0.5 * (1.0 - c), 0.5, 0.5 * (1.0 + c), 1.0]
    raise ValueError("build_tables: supported node counts are 2, 3, 5")


def lagrange_basis(nodes, j, x):
    """lagrange_basis (quadrature.cpp:19-26)."""
    acc = 1.0
    for i in range(len(nodes)):
        if i == j:
            continue
        acc *= (x - nodes[i]) / (nodes[j] - nodes[i])
    return acc


def _lagrange_monomial(nodes, j):
    c = [1.0]
    denom = 1.0
    for i in range(len(nodes)):
        if i == j:
            continue
        denom *= nodes[j] - nodes[i]
        nxt = [0.0] * (len(c) + 1)
        for k in range(len(c)):
            nxt[k] -= nodes[i] * c[k]
            nxt[k + 1] += c[k]
        c = nxt
    return [v / denom for v in c]


def _integrate_monomial(c, upper):
    acc, xp = 0.0, upper
    for k in range(len(c)):
        acc += c[k] * xp / float(k + 1)
        xp *= upper
    return acc


@dataclass
class QuadratureTables:
    num_nodes: int
    nodes: list
    q: np.ndarray
    q_exp: np.ndarray
    q_imp: np.ndarray


def build_tables(n) -> QuadratureTables:
    """build_tables (quadrature.cpp:74-106): Q, forward-Euler Q_E, LU-rule Q_I."""
    nodes = lobatto_nodes(n)
    q = np.zeros((n, n))
    for j in range(n):
        c = _lagrange_monomial(nodes, j)
        for m in range(n):
            q[m, j] = _integrate_monomial(c, nodes[m])
    qe = np.zeros((n, n))
    for m in range(1, n):
        for j in range(m):
            qe[m, j] = nodes[j + 1] - nodes[j]
    mm = n - 1
    qt = np.zeros((mm, mm))
    for i in range(mm):
        for j in range(mm):
            qt[i, j] = q[1 + j, 1 + i]
    for k in range(mm):
        for i in range(k + 1, mm):
            l_ = qt[i, k] / qt[k, k]
            for j in range(k, mm):
                qt[i, j] -= l_ * qt[k, j]
    qi = np.zeros((n, n))
    for i in range(mm):
        for j in range(i + 1):
            qi[1 + i, 1 + j] = qt[j, i]
    return QuadratureTables(n, nodes, q, qe, qi)


# ----------------------------------------------------------------------------------------------
# SDC (sdc.cpp:7-72)


@dataclass
class SpaceTimeState:
    """SpaceTimeState (sdc.hpp:14-20)."""
    state: list = field(default_factory=list)
    f_imp: list = field(default_factory=list)
    f_exp: list = field(default_factory=list)

    def num_nodes(self):
        return len(self.state)

    def copy(self):
        return SpaceTimeState([s.copy() for s in self.state], [s.copy() for s in self.f_imp],
                              [s.copy() for s in self.f_exp])


def spread(theta0, n, ode) -> SpaceTimeState:
    """spread (sdc.cpp:7-13)."""
    fi = ode.eval_implicit(theta0)
    fe = ode.eval_explicit(theta0)
    return SpaceTimeState([theta0.copy() for _ in range(n)], [fi.copy() for _ in range(n)],
                          [fe.copy() for _ in range(n)])


def refresh_node(sts, node, ode):
    """refresh_node (sdc.cpp:15-18)."""
    sts.f_imp[node] = ode.eval_implicit(sts.state[node])
    sts.f_exp[node] = ode.eval_explicit(sts.state[node])


def sweep(sts, dt, t: QuadratureTables, ode, fas=None):
    """sweep (sdc.cpp:20-49), same axpy order."""
    M = sts.num_nodes() - 1
    theta_n = sts.state[0]
    fi_old = [x.copy() for x in sts.f_imp]
    fe_old = [x.copy() for x in sts.f_exp]
    for m in range(M):
        rhs = theta_n.copy()
        for j in range(1, m + 1):
            rhs += (dt * t.q_exp[m + 1, j]) * sts.f_exp[j]
            rhs += (-dt * t.q_exp[m + 1, j]) * fe_old[j]
            rhs += (dt * t.q_imp[m + 1, j]) * sts.f_imp[j]
            rhs += (-dt * t.q_imp[m + 1, j]) * fi_old[j]
        rhs += (-dt * t.q_imp[m + 1, m + 1]) * fi_old[m + 1]
        for j in range(M + 1):
            rhs += (dt * t.q[m + 1, j]) * fi_old[j]
            rhs += (dt * t.q[m + 1, j]) * fe_old[j]
        if fas is not None:
            rhs += fas[m + 1]
        sts.state[m + 1] = ode.solve_implicit(rhs, dt * t.q_imp[m + 1, m + 1])
        refresh_node(sts, m + 1, ode)


def max_abs(st):
    return float(np.abs(st).max()) if st.size else 0.0


def collocation_residual(sts, dt, t: QuadratureTables):
    """collocation_residual (sdc.cpp:51-64): absolute max over nodes and all 3 fields."""
    M = sts.num_nodes() - 1
    res = 0.0
    for m in range(M + 1):
        acc = sts.state[m] - sts.state[0]
        for j in range(M + 1):
            acc += (-dt * t.q[m, j]) * sts.f_imp[j]
            acc += (-dt * t.q[m, j]) * sts.f_exp[j]
        res = max(res, max_abs(acc))
    return res


def sdc_step(theta0, dt, t, n_sweeps, ode):
    """sdc_step (sdc.cpp:66-72); returns (last-node state, final residual)."""
    sts = spread(theta0, t.num_nodes, ode)
    for _ in range(n_sweeps):
        sweep(sts, dt, t, ode)
    return sts.state[t.num_nodes - 1].copy(), collocation_residual(sts, dt, t)


# ----------------------------------------------------------------------------------------------
# multilevel (multilevel.cpp:9-158)


def lagrange_matrix(from_nodes, to_nodes):
    """lagrange_matrix (multilevel.cpp:9-15)."""
    pi = np.zeros((len(to_nodes), len(from_nodes)))
    for i in range(len(to_nodes)):
        for j in range(len(from_nodes)):
            pi[i, j] = lagrange_basis(from_nodes, j, to_nodes[i])
    return pi


@dataclass
class LevelSpec:
    truncation: int
    tables: QuadratureTables
    ode: object

    def num_nodes(self):
        return self.tables.num_nodes


@dataclass
class TransferPair:
    fine: LevelSpec
    coarse: LevelSpec
    time_restrict: np.ndarray
    time_interp: np.ndarray
    qf_time_restricted: np.ndarray


def make_transfer_pair(fine: LevelSpec, coarse: LevelSpec) -> TransferPair:
    """make_transfer_pair (multilevel.cpp:37-51)."""
    if coarse.truncation > fine.truncation:
        raise ValueError("make_transfer_pair: coarse truncation exceeds fine")
    if coarse.truncation < 1:
        raise ValueError("make_transfer_pair: coarse truncation must be >= 1")
    nf, nc = fine.num_nodes(), coarse.num_nodes()
    if not (nf == nc or (nf, nc) in ((3, 2), (5, 3))):
        raise ValueError("make_transfer_pair: unsupported node pair")
    tr = lagrange_matrix(fine.tables.nodes, coarse.tables.nodes)
    ti = lagrange_matrix(coarse.tables.nodes, fine.tables.nodes)
    # matmul (quadrature.cpp:8-17): i, k, j loop order
    qfr = np.zeros((tr.shape[0], fine.tables.q.shape[1]))
    for i in range(tr.shape[0]):
        for k in range(tr.shape[1]):
            for j in range(qfr.shape[1]):
                qfr[i, j] += tr[i, k] * fine.tables.q[k, j]
    return TransferPair(fine, coarse, tr, ti, qfr)


def restrict_space(x, Rf, Rc):
    """restrict_space (multilevel.cpp:53-58) on a (..., Kf) array."""
    idx = np.concatenate([index(Rf, r, r) + np.arange(Rc + 1 - r) for r in range(Rc + 1)])
    return np.asarray(x)[..., idx]


def interpolate_space(x, Rc, Rf):
    """interpolate_space (multilevel.cpp:60-66): zero-pad."""
    idx = np.concatenate([index(Rf, r, r) + np.arange(Rc + 1 - r) for r in range(Rc + 1)])
    x = np.asarray(x)
    out = np.zeros(x.shape[:-1] + (num_coeffs(Rf),), dtype=x.dtype)
    out[..., idx] = x
    return out


def apply_time_matrix(pi, xs):
    """apply_time_matrix (multilevel.cpp:22-33): skips zero weights, same axpy order."""
    out = []
    for i in range(pi.shape[0]):
        acc = np.zeros_like(xs[0])
        for j in range(pi.shape[1]):
            if pi[i, j] != 0.0:
                acc += pi[i, j] * xs[j]
        out.append(acc)
    return out


def restrict_states(fine_states, pair: TransferPair):
    """restrict_states (multilevel.cpp:100-107)."""
    comb = apply_time_matrix(pair.time_restrict, fine_states)
    return [restrict_space(s, pair.fine.truncation, pair.coarse.truncation) for s in comb]


def fas_correction(fine_sts, coarse_sts, dt, pair: TransferPair):
    """fas_correction (multilevel.cpp:109-137)."""
    mc, mf = pair.coarse.num_nodes(), pair.fine.num_nodes()
    tau = []
    for i in range(mc):
        acc_f = np.zeros_like(fine_sts.state[0])
        for j in range(mf):
            w = pair.qf_time_restricted[i, j]
            if w == 0.0:
                continue
            acc_f += w * fine_sts.f_imp[j]
            acc_f += w * fine_sts.f_exp[j]
        t = restrict_space(acc_f, pair.fine.truncation, pair.coarse.truncation)
        for j in range(mc):
            w = pair.coarse.tables.q[i, j]
            if w == 0.0:
                continue
            t += (-w) * coarse_sts.f_imp[j]
            t += (-w) * coarse_sts.f_exp[j]
        tau.append(t * dt)
    return tau


def interpolate_increment(coarse_new, coarse_saved, pair: TransferPair):
    """interpolate_increment (multilevel.cpp:139-150)."""
    delta = [interpolate_space(a - b, pair.coarse.truncation, pair.fine.truncation)
             for a, b in zip(coarse_new, coarse_saved)]
    return apply_time_matrix(pair.time_interp, delta)


def interpolate_states(coarse_states, pair: TransferPair):
    """interpolate_states (multilevel.cpp:152-158)."""
    padded = [interpolate_space(s, pair.coarse.truncation, pair.fine.truncation) for s in coarse_states]
    return apply_time_matrix(pair.time_interp, padded)


# ----------------------------------------------------------------------------------------------
# PFASST, serial emulation (pfasst.cpp:78-251)


def run_block(pair: TransferPair, theta0, n_ts, dt, n_iter):
    """run_block in serial-emulation order (pfasst.cpp:194-251, 212-216): workers run to
    completion in index order. Returns (step_final list, residuals[w][k], message log)."""
    mf, mc = pair.fine.num_nodes(), pair.coarse.num_nodes()
    fo, co = pair.fine.ode, pair.coarse.ode
    fine_ch = {w: [] for w in range(n_ts)}
    coarse_ch = {w: [] for w in range(n_ts)}
    finals, residuals, log = [], [], []

    def expect(ch, phase, it, level):
        m = ch.pop(0)
        if (m[1], m[2], m[3]) != (phase, it, level):
            raise RuntimeError("pfasst: message tag mismatch")
        return m[0]

    for w in range(n_ts):
        res = [0.0] * (n_iter + 1)
        # worker_predict (pfasst.cpp:78-120)
        if w == 0:
            for r in range(1, n_ts):
                log.append((0, 0, "B", 0, r, 0, 0))
        th0c = restrict_space(theta0, pair.fine.truncation, pair.coarse.truncation)
        coarse = spread(th0c, mc, co)
        for q in range(w + 1):
            if q >= 1:
                coarse.state[0] = expect(coarse_ch[w], 0, q - 1, 1)
                refresh_node(coarse, 0, co)
            sweep(coarse, dt, pair.coarse.tables, co)
            if w < n_ts - 1:
                coarse_ch[w + 1].append((coarse.state[mc - 1].copy(), 0, q, 1))
                log.append((0, q, "P", w, w + 1, 1, mc - 1))
        fine = SpaceTimeState(interpolate_states(coarse.state, pair), [None] * mf, [None] * mf)
        for m in range(mf):
            refresh_node(fine, m, fo)
        res[0] = collocation_residual(fine, dt, pair.fine.tables)
        # worker_iterate (pfasst.cpp:122-176)
        for k in range(1, n_iter + 1):
            sweep(fine, dt, pair.fine.tables, fo)
            res[k] = collocation_residual(fine, dt, pair.fine.tables)
            if k == n_iter:
                break
            if w < n_ts - 1:
                fine_ch[w + 1].append((fine.state[mf - 1].copy(), 1, k, 0))
                log.append((1, k, "A", w, w + 1, 0, mf - 1))
            coarse.state = restrict_states(fine.state, pair)
            for m in range(mc):
                refresh_node(coarse, m, co)
            saved = coarse.copy()
            tau = fas_correction(fine, coarse, dt, pair)
            if w > 0:
                coarse.state[0] = expect(coarse_ch[w], 1, k, 1)
            refresh_node(coarse, 0, co)
            sweep(coarse, dt, pair.coarse.tables, co, tau)
            if w < n_ts - 1:
                coarse_ch[w + 1].append((coarse.state[mc - 1].copy(), 1, k, 1))
                log.append((1, k, "C", w, w + 1, 1, mc - 1))
            dstate = interpolate_increment(coarse.state, saved.state, pair)
            dfi = interpolate_increment(coarse.f_imp, saved.f_imp, pair)
            dfe = interpolate_increment(coarse.f_exp, saved.f_exp, pair)
            for m in range(mf):
                fine.state[m] = fine.state[m] + dstate[m]
                fine.f_imp[m] = fine.f_imp[m] + dfi[m]
                fine.f_exp[m] = fine.f_exp[m] + dfe[m]
            if w > 0:
                fine.state[0] = expect(fine_ch[w], 1, k, 0) + dstate[0]
            refresh_node(fine, 0, fo)
        finals.append(fine.state[mf - 1].copy())
        residuals.append(res)
    rank = {"B": 0, "P": 1, "A": 2, "C": 3}
    log.sort(key=lambda m: (m[0], m[1], m[3], rank[m[2]]))
    return finals, residuals, log
