import numpy as np


def rel_diff(a, b):
    """rel_diff (proj/tests/support.hpp:33-38): max|a-b| / max(max|a|, max|b|)."""
    a = np.asarray(a)
    b = np.asarray(b)
    scale = max(np.abs(a).max(initial=0.0), np.abs(b).max(initial=0.0))
    d = np.abs(a - b).max(initial=0.0)
    return d if scale == 0.0 else d / scale


def rel_diff_fields(a, b):
    """Per-prognostic-variable relative L-inf: max over the 3 fields."""
    return max(rel_diff(a[..., i, :], b[..., i, :]) for i in range(3))
