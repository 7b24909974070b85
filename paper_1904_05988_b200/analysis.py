"""Error diagnostics of the reference (analysis.cpp:8-46) on device tensors: the E_Rnorm semi-norm
 used in the paper's accuracy studies, and the max-amplitude spectrum.
States are (3, K) complex tensors (torch, on the GPU) or numpy arrays."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def _degrees(R: int):
    rs = np.concatenate([np.full(R + 1 - r, r) for r in range(R + 1)])
    ss = np.concatenate([np.arange(r, R + 1) for r in range(R + 1)])
    return rs, ss


def _abs(x):
    return x.abs() if hasattr(x, "abs") and not isinstance(x, np.ndarray) else np.abs(x)


def _trunc_of(K: int) -> int:
    return int(round((-3 + np.sqrt(1 + 8 * K)) / 2))


def _mask(R, cap, like):
    rs, ss = _degrees(R)
    m = (rs <= cap) & (ss <= cap)
    if hasattr(like, "device") and not isinstance(like, np.ndarray):
        import torch
        return torch.as_tensor(m, device=like.device)
    return m


def seminorm(x, r_norm: int) -> float:
    """seminorm (analysis.cpp:8-14): max |x_rs| over r <= s <= min(r_norm, R)."""
    R = _trunc_of(x.shape[-1])
    cap = min(r_norm, R)
    a = _abs(x)[..., _mask(R, cap, x)]
    n = a.numel() if hasattr(a, "numel") else a.size
    return float(a.max()) if n else 0.0


@dataclass
class ErrorReport:
    """ErrorReport (analysis.hpp:11-16)."""
    r_norm: int
    e_phi: float
    e_vort: float
    e_div: float


def spectral_error(x, ref, r_norm: int) -> ErrorReport:
    """spectral_error (analysis.cpp:31-38): per-field relative max error on modes s <= r_norm."""
    errs = []
    for f in range(3):
        Rx, Rr = _trunc_of(x[f].shape[-1]), _trunc_of(ref[f].shape[-1])
        cap = min(r_norm, Rx, Rr)
        denom = seminorm(ref[f], r_norm)
        if denom == 0.0:
            raise ValueError("spectral_error: reference norm vanishes on the retained modes")
        d = x[f][..., _mask(Rx, cap, x[f])] - ref[f][..., _mask(Rr, cap, ref[f])]
        errs.append(float(_abs(d).max()) / denom)
    return ErrorReport(r_norm, *errs)


def max_spectrum(x) -> np.ndarray:
    """max_spectrum (analysis.cpp:40-46): spec[s] = max_r |x_rs|."""
    xa = x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)
    R = _trunc_of(xa.shape[-1])
    _, ss = _degrees(R)
    spec = np.zeros(R + 1)
    np.maximum.at(spec, ss, np.abs(xa))
    return spec
