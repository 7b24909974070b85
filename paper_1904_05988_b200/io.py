"""Spectral checkpoints in the reference's JSON format (io.cpp:15-67, io.hpp:12-13) — the wire format
used to exchange initial conditions / final states with the reference.

    {"time": t, "Phi": F, "zeta": F, "delta": F},  F = {"R": R, "order": "r-major",
                                                        "coeffs": [[re, im], ...]}

Host-side I/O only (not on the hot path). Values round-trip losslessly (repr of float64)."""
from __future__ import annotations

import json

import numpy as np


def _field_json(x: np.ndarray, R: int) -> dict:
    x = np.asarray(x, dtype=np.complex128)
    return {"R": int(R), "order": "r-major", "coeffs": [[float(c.real), float(c.imag)] for c in x]}


def _field_from(j: dict) -> np.ndarray:
    """field_from (io.cpp:22-32)."""
    if j.get("order") != "r-major":
        raise ValueError("spectral dump: unsupported coefficient order")
    R = int(j["R"])
    coeffs = j["coeffs"]
    if len(coeffs) != (R + 1) * (R + 2) // 2:
        raise ValueError("spectral dump: coefficient count does not match R")
    a = np.asarray(coeffs, dtype=np.float64)
    return a[:, 0] + 1j * a[:, 1]


def save_checkpoint(path: str, state, time: float = 0.0) -> None:
    """save_checkpoint (io.cpp:48-54). state: (3, K) complex (numpy or torch)."""
    st = state.detach().cpu().numpy() if hasattr(state, "detach") else np.asarray(state)
    K = st.shape[-1]
    R = int(round((-3 + np.sqrt(1 + 8 * K)) / 2))
    doc = {"time": float(time), "Phi": _field_json(st[0], R), "zeta": _field_json(st[1], R),
           "delta": _field_json(st[2], R)}
    with open(path, "w") as f:
        f.write(json.dumps(doc) + "\n")


def load_checkpoint(path: str):
    """load_checkpoint (io.cpp:56-67): returns (state (3, K) complex128, time)."""
    with open(path) as f:
        j = json.load(f)
    st = np.stack([_field_from(j["Phi"]), _field_from(j["zeta"]), _field_from(j["delta"])])
    return st, float(j["time"])
