"""Seeded test inputs shared by the golden generator and the tests (TEST INFRASTRUCTURE ONLY).

Mirrors the reference's test fixtures (proj/tests/support.hpp:11-31 random_field/random_state,
proj/tests/test_swe.cpp:287-300 smooth_state). numpy's PCG64 replaces std::mt19937_64 +
normal_distribution (the latter is implementation-defined); inputs are generated once and
passed to both the reference and the implementation under test, so the generator choice does
not affect parity.
"""
from __future__ import annotations

import math

import numpy as np


def num_coeffs(R):
    return (R + 1) * (R + 2) // 2


def degree_order(R):
    rs = np.concatenate([np.full(R + 1 - r, r) for r in range(R + 1)])
    ss = np.concatenate([np.arange(r, R + 1) for r in range(R + 1)])
    return rs, ss


def random_field(R, seed):
    """random_field (support.hpp:11-19): unit normal re/im, r = 0 kept real."""
    rng = np.random.default_rng(seed)
    K = num_coeffs(R)
    re = rng.standard_normal(K)
    im = rng.standard_normal(K)
    rs, _ = degree_order(R)
    im[rs == 0] = 0.0
    return re + 1j * im


def random_state(R, seed, scale_phi=1.0, scale_wind=1.0):
    """random_state (support.hpp:21-31)."""
    return np.stack([random_field(R, seed) * scale_phi,
                     random_field(R, seed + 1000003) * scale_wind,
                     random_field(R, seed + 2000003) * scale_wind])


def smooth_state(R, phi_bar, seed):
    """smooth_state (test_swe.cpp:287-300): Gaussian spectral decay exp(-(s/3)^2)."""
    s = random_state(R, seed)
    _, ss = degree_order(R)
    decay = np.exp(-((ss / 3.0) ** 2))
    s[0] *= 1.0e4 * decay
    s[1] *= 1.0e-5 * decay
    s[2] *= 1.0e-6 * decay
    s[1, 0] = 0.0
    s[2, 0] = 0.0
    s[0, 0] = phi_bar * math.sqrt(2.0)
    return s


def micro_bench_fields(R, n_fields, seed):
    """BASELINE config 2 input: uniform[-1,1] complex x (n+1)^-1.5, r = 0 real."""
    rng = np.random.default_rng(seed)
    K = num_coeffs(R)
    rs, ss = degree_order(R)
    x = rng.uniform(-1, 1, (n_fields, K)) + 1j * rng.uniform(-1, 1, (n_fields, K))
    x *= (ss + 1.0) ** -1.5
    x[:, rs == 0] = x[:, rs == 0].real
    return x
