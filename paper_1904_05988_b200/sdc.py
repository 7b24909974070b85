"""SDC on a B200 — QuadratureTables / SpaceTimeState / sweep (quadrature.hpp, sdc.hpp) over libpswe.

A ``Level`` is the reference's LevelSpec (multilevel.hpp:16-23) plus its SpaceTimeState
(sdc.hpp:14-20) resident on the device: (M+1) nodes x {state, F_I, F_E}.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .swe import ModelParams
from .transform import TransformPlan, _dev, _stream, num_coeffs


@dataclass
class QuadratureTables:
    """QuadratureTables (quadrature.hpp:16-22)."""
    num_nodes: int
    nodes: np.ndarray
    q: np.ndarray
    q_exp: np.ndarray
    q_imp: np.ndarray


def build_tables(n: int) -> QuadratureTables:
    """build_tables (quadrature.cpp:74-106), computed by libpswe's host code."""
    nodes = np.zeros(n)
    q, qe, qi = (np.zeros((n, n)) for _ in range(3))
    _lib.check(_lib.lib().pswe_quadrature_tables(n, nodes.ctypes.data, q.ctypes.data, qe.ctypes.data,
                                                 qi.ctypes.data))
    return QuadratureTables(n, nodes, q, qe, qi)


class _DevView:
    """__cuda_array_interface__ wrapper: zero-copy torch view of library-owned device memory."""

    def __init__(self, ptr, shape, typestr="<c16"):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None}


def device_view(ptr, shape, dtype=torch.complex128):
    typestr = {torch.complex128: "<c16", torch.float64: "<f8"}[dtype]
    return torch.as_tensor(_DevView(ptr, shape, typestr), device="cuda")


class Level:
    """LevelSpec + device SpaceTimeState."""

    def __init__(self, plan: TransformPlan, params: ModelParams, num_nodes: int):
        h = ctypes.c_void_p()
        self._prm = params.c()
        _lib.check(_lib.lib().pswe_level_create(plan.handle, ctypes.byref(self._prm), num_nodes, ctypes.byref(h)))
        self._h = h
        self.plan, self.params = plan, params
        self.truncation = plan.R
        self.K = num_coeffs(plan.R)
        self.tables = build_tables(num_nodes)
        self._res = torch.zeros(1, dtype=torch.float64, device="cuda")

    @property
    def handle(self):
        return self._h

    def num_nodes(self):
        return self.tables.num_nodes

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.lib().pswe_level_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # views of node arrays (which: 0 state, 1 f_imp, 2 f_exp)
    def _ptr(self, which, node):
        p = _lib.lib().pswe_level_ptr(self._h, which, node)
        if not p:
            raise _lib.PsweError("level_ptr: bad node")
        return p

    def state(self, node):
        return device_view(self._ptr(0, node), (3, self.K))

    def f_imp(self, node):
        return device_view(self._ptr(1, node), (3, self.K))

    def f_exp(self, node):
        return device_view(self._ptr(2, node), (3, self.K))

    def states(self):
        return device_view(self._ptr(0, 0), (self.num_nodes(), 3, self.K))

    # sdc.hpp operations
    def spread(self, theta0):
        """spread (sdc.cpp:7-13)."""
        th = _dev(theta0, torch.complex128)
        _lib.check(_lib.lib().pswe_spread(self._h, th.data_ptr(), _stream()))

    def refresh_nodes(self, first=0, count=None):
        """refresh_node (sdc.cpp:15-18) for a contiguous node range, batched in one pass."""
        count = self.num_nodes() - first if count is None else count
        _lib.check(_lib.lib().pswe_refresh_nodes(self._h, first, count, _stream()))

    def sweep(self, dt: float, tau=None):
        """sweep (sdc.cpp:20-49); tau: (num_nodes, 3, K) FAS correction or None."""
        tp = None
        if tau is not None:
            tau = _dev(tau, torch.complex128)
            tp = tau.data_ptr()
        _lib.check(_lib.lib().pswe_sweep(self._h, float(dt), tp, _stream()))

    def collocation_residual(self, dt: float, out: torch.Tensor | None = None) -> torch.Tensor:
        """collocation_residual (sdc.cpp:51-64); device scalar (no host sync)."""
        out = self._res if out is None else out
        _lib.check(_lib.lib().pswe_collocation_residual(self._h, float(dt), out.data_ptr(), _stream()))
        return out

    def sdc_step(self, theta0, dt: float, n_sweeps: int, residual: torch.Tensor | None = None):
        """sdc_step (sdc.cpp:66-72): returns a view of the last-node state."""
        th = _dev(theta0, torch.complex128)
        rp = residual.data_ptr() if residual is not None else None
        _lib.check(_lib.lib().pswe_sdc_step(self._h, th.data_ptr(), float(dt), int(n_sweeps), rp, _stream()))
        return self.state(self.num_nodes() - 1)


def sdc_run(level: Level, theta0, dt: float, n_sweeps: int, n_steps: int):
    """runner.cpp:114-122: n_steps serial SDC steps; returns (final state, residual per step)."""
    s = _dev(theta0, torch.complex128).clone()
    res = torch.zeros(n_steps, dtype=torch.float64, device="cuda")
    for n in range(n_steps):
        last = level.sdc_step(s, dt, n_sweeps, res[n:n + 1])
        s.copy_(last)
    return s, res
