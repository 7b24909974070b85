"""Two-level transfers on a B200 — TransferPair and the FAS machinery (multilevel.hpp:29-80)."""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .sdc import Level
from .transform import _dev, _stream, num_coeffs


def restrict_space(x, rf: int, rc: int):
    """restrict_space (multilevel.cpp:53-58, 68-74) on states (..., 3, Kf)."""
    x = _dev(x, torch.complex128)
    n = int(np.prod(x.shape[:-2])) if x.dim() > 2 else 1
    y = torch.empty(x.shape[:-1] + (num_coeffs(rc),), dtype=torch.complex128, device=x.device)
    _lib.check(_lib.lib().pswe_restrict_space(rf, rc, x.data_ptr(), y.data_ptr(), n, _stream()))
    return y


def interpolate_space(x, rc: int, rf: int):
    """interpolate_space (multilevel.cpp:60-66, 76-82): zero-pad, on states (..., 3, Kc)."""
    x = _dev(x, torch.complex128)
    n = int(np.prod(x.shape[:-2])) if x.dim() > 2 else 1
    y = torch.empty(x.shape[:-1] + (num_coeffs(rf),), dtype=torch.complex128, device=x.device)
    _lib.check(_lib.lib().pswe_interpolate_space(rc, rf, x.data_ptr(), y.data_ptr(), n, _stream()))
    return y


class TransferPair:
    """TransferPair (multilevel.hpp:29-35) between two device levels."""

    def __init__(self, fine: Level, coarse: Level):
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().pswe_pair_create(fine.handle, coarse.handle, ctypes.byref(h)))
        self._h = h
        self.fine, self.coarse = fine, coarse
        self.tau = torch.zeros((coarse.num_nodes(), 3, coarse.K), dtype=torch.complex128, device="cuda")
        self.dstate0 = torch.zeros((3, fine.K), dtype=torch.complex128, device="cuda")

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.lib().pswe_pair_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def restrict_states(self):
        """coarse.state := restrict_states(fine.state) (multilevel.cpp:100-107)."""
        _lib.check(_lib.lib().pswe_restrict_states(self._h, _stream()))

    def fas_correction(self, dt: float, tau_fine=None):
        """tau := fas_correction(fine, coarse, dt) (multilevel.cpp:109-137); with tau_fine (the fine
        level's own FAS term, fine num_nodes states) the multi-level form of Eq. 19
        (PAPER.md:576-581): tau += R tau_fine."""
        if tau_fine is None:
            _lib.check(_lib.lib().pswe_fas_correction(self._h, float(dt), self.tau.data_ptr(), _stream()))
        else:
            _lib.check(_lib.lib().pswe_fas_correction_ml(self._h, float(dt), tau_fine.data_ptr(),
                                                         self.tau.data_ptr(), _stream()))
        return self.tau

    def save_coarse(self):
        _lib.check(_lib.lib().pswe_save_coarse(self._h, _stream()))

    def interpolate_increment_add(self):
        """fine += interpolate_increment(coarse - saved) for state, F_I, F_E (multilevel.cpp:139-150)."""
        _lib.check(_lib.lib().pswe_interpolate_increment_add(self._h, self.dstate0.data_ptr(), _stream()))
        return self.dstate0

    def interpolate_states(self):
        """fine.state := interpolate_states(coarse.state) (multilevel.cpp:152-158)."""
        _lib.check(_lib.lib().pswe_interpolate_states(self._h, _stream()))


def mlsdc_step(pair: TransferPair, theta0, dt: float, n_iter: int, residual=None):
    """mlsdc_step (multilevel.cpp:160-194) composed from the device operations."""
    fine, coarse = pair.fine, pair.coarse
    fine.spread(theta0)
    for k in range(n_iter):
        fine.sweep(dt)
        pair.restrict_states()
        # node 0 never changes in the serial scheme; refresh 1..mc-1 (k > 0) / all (k == 0)
        if k == 0:
            coarse.refresh_nodes(0)
        else:
            coarse.refresh_nodes(1)
        pair.save_coarse()
        tau = pair.fas_correction(dt)
        coarse.sweep(dt, tau)
        pair.interpolate_increment_add()
    if residual is not None:
        fine.collocation_residual(dt, residual)
    return fine.state(fine.num_nodes() - 1)
