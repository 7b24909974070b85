"""analysis.cpp:8-46 diagnostics (semi-norm error, max spectrum) on known inputs."""
import numpy as np

from oracle import fixtures as fx


def test_spectral_error_and_spectrum():
    from paper_1904_05988_b200 import analysis as A
    R = 10
    a = fx.random_state(R, 1)
    b = a.copy()
    b[0, 3] += 0.5  # (r=0, s=3)
    rep = A.spectral_error(b, a, 5)
    rs, ss = fx.degree_order(R)
    keep = (rs <= 5) & (ss <= 5)
    assert abs(rep.e_phi - 0.5 / np.abs(a[0][keep]).max()) < 1e-15
    assert rep.e_vort == 0.0 and rep.e_div == 0.0
    # modes above r_norm are ignored
    c = a.copy()
    c[1, -1] += 1.0  # (r=R, s=R)
    assert A.spectral_error(c, a, R - 1).e_vort == 0.0
    spec = A.max_spectrum(a[2])
    assert spec.shape == (R + 1,)
    rs, ss = fx.degree_order(R)
    for s in range(R + 1):
        assert spec[s] == np.abs(a[2][ss == s]).max()
