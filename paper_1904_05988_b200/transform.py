"""TransformPlan on a B200 — the reference's operator API (transform.hpp:19-96) over libpswe.

Arrays are torch CUDA tensors (torch is the device-memory/stream plumbing only; every transform
runs in the sm_100a kernels of libpswe.so): spectral fields complex128 (..., K) r-major,
grids float64 (..., nlat, nlon). Leading dimensions are batched into one launch sequence.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

LEGENDRE_RECOMPUTE = 0
LEGENDRE_STREAM = 1


def num_coeffs(R: int) -> int:
    """SpectralField::size (field.hpp:21-23)."""
    return (R + 1) * (R + 2) // 2


def dealiased_nlon(R: int) -> int:
    """dealiased_nlon (transform.cpp:38-43)."""
    return _lib.lib().pswe_dealiased_nlon(R)


def gauss_latitudes(n: int):
    """gauss_latitudes (gauss.cpp:24-50), host setup."""
    mu, w = np.zeros(n), np.zeros(n)
    _lib.check(_lib.lib().pswe_gauss_latitudes(n, mu.ctypes.data, w.ctypes.data))
    return mu, w


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(t: torch.Tensor, dtype) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(t)
    if t.device.type != "cuda":
        raise _lib.PsweError("libpswe operates on CUDA tensors (no CPU path)")
    return t.to(dtype).contiguous()


class TransformPlan:
    """TransformPlan(R) (transform.hpp:27-96). ``nlat``/``nlon`` default to the reference's
    dealiased grid; an explicit Gaussian grid may be given (BASELINE's linear grids)."""

    def __init__(self, truncation: int, nlat: int = 0, nlon: int = 0,
                 legendre_mode: int = LEGENDRE_STREAM):
        if not torch.cuda.is_available():
            raise _lib.PsweError("TransformPlan needs a CUDA device (libpswe has no CPU path)")
        torch.cuda.init()
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().pswe_plan_create(truncation, nlat, nlon, legendre_mode, ctypes.byref(h)))
        self._h = h
        R, la, lo, md = (ctypes.c_int() for _ in range(4))
        _lib.check(_lib.lib().pswe_plan_info(h, ctypes.byref(R), ctypes.byref(la), ctypes.byref(lo), ctypes.byref(md)))
        self.R, self.nlat, self.nlon, self.legendre_mode = R.value, la.value, lo.value, md.value
        self.K = num_coeffs(self.R)
        self.mu = np.zeros(self.nlat)
        self.weight = np.zeros(self.nlat)
        _lib.check(_lib.lib().pswe_plan_latitudes(h, self.mu.ctypes.data, self.weight.ctypes.data))

    @property
    def handle(self):
        return self._h

    def truncation(self):
        return self.R

    def reserve(self, max_batch: int):
        _lib.check(_lib.lib().pswe_plan_reserve(self._h, max_batch))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.lib().pswe_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- transforms ---------------------------------------------------------------------------
    def synthesise(self, x: torch.Tensor) -> torch.Tensor:
        """Spectral -> grid (transform.cpp:155-174)."""
        x = _dev(x, torch.complex128)
        if x.shape[-1] != self.K:
            raise _lib.PsweError("synthesise: field truncation does not match the plan")
        lead = x.shape[:-1]
        n = int(np.prod(lead)) if lead else 1
        g = torch.empty(lead + (self.nlat, self.nlon), dtype=torch.float64, device=x.device)
        _lib.check(_lib.lib().pswe_synthesise(self._h, x.data_ptr(), g.data_ptr(), n, _stream()))
        return g

    def analyse(self, g: torch.Tensor) -> torch.Tensor:
        """Grid -> spectral (transform.cpp:136-153)."""
        g = _dev(g, torch.float64)
        if tuple(g.shape[-2:]) != (self.nlat, self.nlon):
            raise _lib.PsweError("analyse: grid dimensions do not match the plan")
        lead = g.shape[:-2]
        n = int(np.prod(lead)) if lead else 1
        x = torch.empty(lead + (self.K,), dtype=torch.complex128, device=g.device)
        _lib.check(_lib.lib().pswe_analyse(self._h, g.data_ptr(), x.data_ptr(), n, _stream()))
        return x

    def uv_from_vortdiv(self, vort, div, radius: float):
        """(u, v) grids from spectral vorticity/divergence (transform.cpp:176-223)."""
        vort = _dev(vort, torch.complex128)
        div = _dev(div, torch.complex128)
        if vort.shape[-1] != self.K or div.shape != vort.shape:
            raise _lib.PsweError("uv_from_vortdiv: truncation mismatch")
        lead = vort.shape[:-1]
        n = int(np.prod(lead)) if lead else 1
        u = torch.empty(lead + (self.nlat, self.nlon), dtype=torch.float64, device=vort.device)
        v = torch.empty_like(u)
        _lib.check(_lib.lib().pswe_uv_from_vortdiv(self._h, vort.data_ptr(), div.data_ptr(), float(radius),
                                                    u.data_ptr(), v.data_ptr(), n, _stream()))
        return u, v

    def vortdiv_from_uv(self, u, v, radius: float):
        """Spectral vorticity/divergence of a grid vector field (transform.cpp:225-270)."""
        u = _dev(u, torch.float64)
        v = _dev(v, torch.float64)
        if tuple(u.shape[-2:]) != (self.nlat, self.nlon) or v.shape != u.shape:
            raise _lib.PsweError("vortdiv_from_uv: grid dimensions do not match the plan")
        lead = u.shape[:-2]
        n = int(np.prod(lead)) if lead else 1
        z = torch.empty(lead + (self.K,), dtype=torch.complex128, device=u.device)
        d = torch.empty_like(z)
        _lib.check(_lib.lib().pswe_vortdiv_from_uv(self._h, u.data_ptr(), v.data_ptr(), float(radius),
                                                    z.data_ptr(), d.data_ptr(), n, _stream()))
        return z, d


def _lap(R, x, radius, inverse):
    x = _dev(x, torch.complex128)
    if x.shape[-1] != num_coeffs(R):
        raise _lib.PsweError("laplacian: truncation mismatch")
    n = int(np.prod(x.shape[:-1])) if x.dim() > 1 else 1
    y = torch.empty_like(x)
    _lib.check(_lib.lib().pswe_laplacian(R, x.data_ptr(), float(radius), y.data_ptr(), n, 1 if inverse else 0,
                                         _stream()))
    return y


def laplacian(R: int, x, radius: float):
    """laplacian (transform.cpp:272-280)."""
    return _lap(R, x, radius, False)


def inv_laplacian(R: int, x, radius: float):
    """inv_laplacian (transform.cpp:282-290)."""
    return _lap(R, x, radius, True)
