"""ctypes binding of oracle/_ref/libpintswe_ref.so (the REFERENCE C++ compiled by build_ref.sh).

TEST INFRASTRUCTURE ONLY: used by tests/, oracle/make_golden.py and bench.py's reference arm /
cpu_baseline leg. States are numpy complex128 arrays (3, K); grids (nlat, nlon) float64.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libpintswe_ref.so")

_c_int, _c_double, _vp = ctypes.c_int, ctypes.c_double, ctypes.c_void_p


class Params(ctypes.Structure):
    _fields_ = [("radius", _c_double), ("omega", _c_double), ("gravity", _c_double),
                ("phi_bar", _c_double), ("nu", _c_double)]


def available() -> bool:
    return os.path.exists(LIB_PATH)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference library missing: {LIB_PATH} (run oracle/build_ref.sh)")
        L = ctypes.CDLL(LIB_PATH)
        sig = {
            "ref_last_error": (ctypes.c_char_p, []),
            "ref_set_threads": (None, [_c_int]),
            "ref_max_threads": (_c_int, []),
            "ref_dealiased_nlon": (_c_int, [_c_int]),
            "ref_gauss": (_c_int, [_c_int, _vp, _vp]),
            "ref_legendre_column": (_c_int, [_c_int, _c_int, _c_double, _vp]),
            "ref_plan_create": (_vp, [_c_int, _c_int, _c_int]),
            "ref_plan_destroy": (None, [_vp]),
            "ref_plan_nlat": (_c_int, [_vp]),
            "ref_plan_nlon": (_c_int, [_vp]),
            "ref_plan_latitudes": (_c_int, [_vp, _vp, _vp]),
            "ref_synthesise": (_c_int, [_vp, _vp, _vp]),
            "ref_analyse": (_c_int, [_vp, _vp, _vp]),
            "ref_uv_from_vortdiv": (_c_int, [_vp, _vp, _vp, _c_double, _vp, _vp]),
            "ref_vortdiv_from_uv": (_c_int, [_vp, _vp, _vp, _c_double, _vp, _vp]),
            "ref_direct_synthesise": (_c_int, [_c_int, _vp, _c_int, _c_int, _vp, _vp]),
            "ref_direct_analyse": (_c_int, [_c_int, _vp, _vp, _c_int, _c_int, _vp, _vp]),
            "ref_direct_uv": (_c_int, [_c_int, _vp, _vp, _c_double, _vp, _c_int, _c_int, _vp, _vp]),
            "ref_laplacian": (_c_int, [_c_int, _vp, _c_double, _vp]),
            "ref_inv_laplacian": (_c_int, [_c_int, _vp, _c_double, _vp]),
            "ref_eval_linear": (_c_int, [_c_int, _vp, _vp, _vp]),
            "ref_eval_nonlinear": (_c_int, [_vp, _vp, _vp, _vp]),
            "ref_solve_implicit": (_c_int, [_c_int, _vp, _vp, _c_double, _vp]),
            "ref_time_eval": (_c_double, [_vp, _vp, _vp, _c_int]),
            "ref_time_roundtrip": (_c_double, [_vp, _vp, _c_int, _c_int]),
            "ref_build_tables": (_c_int, [_c_int, _vp, _vp, _vp, _vp]),
            "ref_transfer_matrices": (_c_int, [_c_int, _c_int, _vp, _vp, _vp]),
            "ref_sdc_run": (_c_int, [_vp, _vp, _c_int, _c_int, _c_double, _c_int, _vp, _vp, _vp]),
            "ref_sdc_sweep": (_c_int, [_vp, _vp, _c_int, _c_double, _vp, _vp]),
            "ref_collocation_residual": (_c_double, [_c_int, _c_int, _c_double, _vp]),
            "ref_pfasst_run": (_c_int, [_c_int] * 6 + [_vp, _c_int, _c_int, _c_int, _c_double,
                                        _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _c_int, _vp]),
            "ref_mlsdc_run": (_c_int, [_c_int] * 6 + [_vp, _c_int, _c_int, _c_double, _c_int,
                                       _c_int, _vp, _vp, _vp]),
            "ref_last_wall": (_c_double, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_vp) if a is not None else None


def _check(rc):
    if rc != 0:
        raise RuntimeError("reference error: " + lib().ref_last_error().decode())


def num_coeffs(R):
    return (R + 1) * (R + 2) // 2


def params_struct(p) -> Params:
    return Params(p.radius, p.omega, p.gravity, p.phi_bar, p.nu)


def _cvec(x):
    return np.ascontiguousarray(x, dtype=np.complex128)


class RefPlan:
    """The reference TransformPlan (transform.hpp:27-96); nlat = nlon = 0 gives the dealiased grid."""

    def __init__(self, R, nlat=0, nlon=0):
        self.R = R
        self.h = lib().ref_plan_create(R, nlat, nlon)
        if not self.h:
            _check(1)
        self.nlat = lib().ref_plan_nlat(self.h)
        self.nlon = lib().ref_plan_nlon(self.h)
        self.mu = np.zeros(self.nlat)
        self.w = np.zeros(self.nlat)
        lib().ref_plan_latitudes(self.h, _p(self.mu), _p(self.w))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_plan_destroy(self.h)
            self.h = None

    def synthesise(self, x):
        g = np.zeros((self.nlat, self.nlon))
        _check(lib().ref_synthesise(self.h, _p(_cvec(x)), _p(g)))
        return g

    def analyse(self, g):
        x = np.zeros(num_coeffs(self.R), dtype=np.complex128)
        _check(lib().ref_analyse(self.h, _p(np.ascontiguousarray(g, dtype=np.float64)), _p(x)))
        return x

    def uv_from_vortdiv(self, vort, div, radius):
        u = np.zeros((self.nlat, self.nlon))
        v = np.zeros_like(u)
        _check(lib().ref_uv_from_vortdiv(self.h, _p(_cvec(vort)), _p(_cvec(div)), radius, _p(u), _p(v)))
        return u, v

    def vortdiv_from_uv(self, u, v, radius):
        K = num_coeffs(self.R)
        z = np.zeros(K, dtype=np.complex128)
        d = np.zeros(K, dtype=np.complex128)
        _check(lib().ref_vortdiv_from_uv(self.h, _p(np.ascontiguousarray(u, dtype=np.float64)),
                                         _p(np.ascontiguousarray(v, dtype=np.float64)), radius, _p(z), _p(d)))
        return z, d

    def eval_nonlinear(self, st, params):
        out = np.zeros((3, num_coeffs(self.R)), dtype=np.complex128)
        ps = params_struct(params)
        _check(lib().ref_eval_nonlinear(self.h, ctypes.byref(ps), _p(_cvec(st)), _p(out)))
        return out

    def time_eval(self, st, params, reps):
        ps = params_struct(params)
        return lib().ref_time_eval(self.h, ctypes.byref(ps), _p(_cvec(st)), reps)

    def time_roundtrip(self, xs, reps):
        xs = _cvec(xs)
        return lib().ref_time_roundtrip(self.h, _p(xs), xs.shape[0], reps)


def gauss(n):
    mu, w = np.zeros(n), np.zeros(n)
    _check(lib().ref_gauss(n, _p(mu), _p(w)))
    return mu, w


def legendre_column(r, smax, mu):
    out = np.zeros(smax - r + 1)
    _check(lib().ref_legendre_column(r, smax, float(mu), _p(out)))
    return out


def direct_synthesise(R, x, mu, nlon):
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    g = np.zeros((mu.size, nlon))
    _check(lib().ref_direct_synthesise(R, _p(mu), mu.size, nlon, _p(_cvec(x)), _p(g)))
    return g


def direct_analyse(R, g, mu, w):
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    x = np.zeros(num_coeffs(R), dtype=np.complex128)
    _check(lib().ref_direct_analyse(R, _p(mu), _p(w), mu.size, g.shape[1], _p(g), _p(x)))
    return x


def direct_uv(R, vort, div, radius, mu, nlon):
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    u = np.zeros((mu.size, nlon))
    v = np.zeros_like(u)
    _check(lib().ref_direct_uv(R, _p(_cvec(vort)), _p(_cvec(div)), radius, _p(mu), mu.size, nlon, _p(u), _p(v)))
    return u, v


def eval_linear(R, st, params):
    out = np.zeros((3, num_coeffs(R)), dtype=np.complex128)
    ps = params_struct(params)
    _check(lib().ref_eval_linear(R, ctypes.byref(ps), _p(_cvec(st)), _p(out)))
    return out


def solve_implicit(R, b, c, params):
    out = np.zeros((3, num_coeffs(R)), dtype=np.complex128)
    ps = params_struct(params)
    _check(lib().ref_solve_implicit(R, ctypes.byref(ps), _p(_cvec(b)), float(c), _p(out)))
    return out


def laplacian(R, x, radius):
    y = np.zeros(num_coeffs(R), dtype=np.complex128)
    _check(lib().ref_laplacian(R, _p(_cvec(x)), radius, _p(y)))
    return y


def inv_laplacian(R, x, radius):
    y = np.zeros(num_coeffs(R), dtype=np.complex128)
    _check(lib().ref_inv_laplacian(R, _p(_cvec(x)), radius, _p(y)))
    return y


def build_tables(n):
    nodes = np.zeros(n)
    q, qe, qi = (np.zeros((n, n)) for _ in range(3))
    _check(lib().ref_build_tables(n, _p(nodes), _p(q), _p(qe), _p(qi)))
    return nodes, q, qe, qi


def transfer_matrices(nf, nc):
    tr, ti, qfr = np.zeros((nc, nf)), np.zeros((nf, nc)), np.zeros((nc, nf))
    _check(lib().ref_transfer_matrices(nf, nc, _p(tr), _p(ti), _p(qfr)))
    return tr, ti, qfr


def sdc_run(plan: RefPlan, params, nodes, n_sweeps, dt, n_steps, theta0):
    fin = np.zeros((3, num_coeffs(plan.R)), dtype=np.complex128)
    res = np.zeros(n_steps)
    ps = params_struct(params)
    _check(lib().ref_sdc_run(plan.h, ctypes.byref(ps), nodes, n_sweeps, dt, n_steps,
                             _p(_cvec(theta0)), _p(fin), _p(res)))
    return fin, res, lib().ref_last_wall()


def sdc_sweep(plan: RefPlan, params, nodes, dt, sts, tau=None):
    """sts: complex array (3, nodes, 3, K) = (state | f_imp | f_exp) x node; updated copy returned."""
    s = _cvec(sts).copy()
    ps = params_struct(params)
    _check(lib().ref_sdc_sweep(plan.h, ctypes.byref(ps), nodes, dt, _p(s),
                               _p(_cvec(tau)) if tau is not None else None))
    return s


def collocation_residual(R, nodes, dt, sts):
    return lib().ref_collocation_residual(R, nodes, dt, _p(_cvec(sts)))


@dataclass
class PfasstResult:
    final: np.ndarray
    residuals: np.ndarray  # (n_blocks, n_ts, n_iter+1)
    messages: list
    wall: float


def pfasst_run(Rf, grid_f, Rc, grid_c, params, nodes_f, nodes_c, n_ts, dt, n_iter, n_blocks,
               theta0, serial=True, max_msgs=4096):
    fin = np.zeros((3, num_coeffs(Rf)), dtype=np.complex128)
    res = np.zeros((n_blocks, n_ts, n_iter + 1))
    msgs = np.zeros((max_msgs, 7), dtype=np.int32)
    nm = ctypes.c_int(0)
    ps = params_struct(params)
    _check(lib().ref_pfasst_run(Rf, grid_f[0], grid_f[1], Rc, grid_c[0], grid_c[1], ctypes.byref(ps),
                                nodes_f, nodes_c, n_ts, dt, n_iter, n_blocks, 1 if serial else 0,
                                _p(_cvec(theta0)), _p(fin), _p(res), _p(msgs), max_msgs, ctypes.byref(nm)))
    log = [(int(m[0]), int(m[1]), chr(m[2]), int(m[3]), int(m[4]), int(m[5]), int(m[6]))
           for m in msgs[: nm.value]]
    return PfasstResult(fin, res, log, lib().ref_last_wall())


def mlsdc_run(Rf, grid_f, Rc, grid_c, params, nodes_f, nodes_c, dt, n_iter, n_steps, theta0):
    fin = np.zeros((3, num_coeffs(Rf)), dtype=np.complex128)
    res = np.zeros(n_steps)
    ps = params_struct(params)
    _check(lib().ref_mlsdc_run(Rf, grid_f[0], grid_f[1], Rc, grid_c[0], grid_c[1], ctypes.byref(ps),
                               nodes_f, nodes_c, dt, n_iter, n_steps, _p(_cvec(theta0)), _p(fin), _p(res)))
    return fin, res
