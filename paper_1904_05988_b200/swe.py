"""Shallow-water right-hand side on a B200 — ImexOde / SweOde (swe.hpp:13-79) over libpswe.

States are complex128 CUDA tensors (..., 3, K): (Phi, zeta, delta), r-major per field.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .transform import TransformPlan, _dev, _stream, num_coeffs


@dataclass
class ModelParams:
    """ModelParams (swe.hpp:13-19): Williamson standard constants."""
    radius: float = 6.37122e6
    omega: float = 7.292e-5
    gravity: float = 9.80616
    phi_bar: float = 9.80616 * 29400.0
    nu: float = 0.0

    def c(self) -> _lib.Params:
        return _lib.Params(self.radius, self.omega, self.gravity, self.phi_bar, self.nu)


def _states(st, R):
    st = _dev(st, torch.complex128)
    if st.shape[-2:] != (3, num_coeffs(R)):
        raise _lib.PsweError("state shape must be (..., 3, K) for the plan's truncation")
    n = int(np.prod(st.shape[:-2])) if st.dim() > 2 else 1
    return st, n


def eval_linear(R: int, state, p: ModelParams):
    """eval_linear (swe.cpp:9-25)."""
    st, n = _states(state, R)
    out = torch.empty_like(st)
    prm = p.c()
    _lib.check(_lib.lib().pswe_eval_implicit(R, ctypes.byref(prm), st.data_ptr(), out.data_ptr(), n, _stream()))
    return out


def eval_nonlinear(state, p: ModelParams, plan: TransformPlan):
    """eval_nonlinear (swe.cpp:27-69)."""
    st, n = _states(state, plan.R)
    out = torch.empty_like(st)
    prm = p.c()
    _lib.check(_lib.lib().pswe_eval_explicit(plan.handle, ctypes.byref(prm), st.data_ptr(), out.data_ptr(), n,
                                             _stream()))
    return out


def imex_split(state, p: ModelParams, plan: TransformPlan):
    """imex_split (swe.cpp:71-75): (F_I, F_E) in one fused pass."""
    st, n = _states(state, plan.R)
    fi = torch.empty_like(st)
    fe = torch.empty_like(st)
    prm = p.c()
    _lib.check(_lib.lib().pswe_eval_imex(plan.handle, ctypes.byref(prm), st.data_ptr(), fi.data_ptr(),
                                         fe.data_ptr(), n, _stream()))
    return fi, fe


def solve_implicit(R: int, b, c: float, p: ModelParams):
    """solve_implicit (swe.cpp:77-98): Theta - c F_I(Theta) = b per mode."""
    st, n = _states(b, R)
    out = torch.empty_like(st)
    prm = p.c()
    _lib.check(_lib.lib().pswe_solve_implicit(R, ctypes.byref(prm), st.data_ptr(), float(c), out.data_ptr(), n,
                                              _stream()))
    return out


class SweOde:
    """SweOde (swe.hpp:57-79), the ImexOde implementation bound to one plan."""

    def __init__(self, plan: TransformPlan, params: ModelParams):
        self.plan = plan
        self.params = params

    def truncation(self):
        return self.plan.R

    def eval_implicit(self, state):
        return eval_linear(self.plan.R, state, self.params)

    def eval_explicit(self, state):
        return eval_nonlinear(state, self.params, self.plan)

    def solve_implicit(self, b, c):
        return solve_implicit(self.plan.R, b, c, self.params)
