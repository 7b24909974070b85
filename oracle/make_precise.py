"""Generates tests/golden/precise_t{255,511}.npz: the EXACT value (long double, oracle/precise.py)
of eval_nonlinear (swe.cpp:27-69) for one seeded state on BASELINE grids, stored as complex128,
with the distance of the reference build (oracle/_ref) and of the numpy restatement from it.

TEST INFRASTRUCTURE ONLY. Run here (needs oracle/_ref built): python oracle/make_precise.py
T255 256x512: bench.py's first headline state; T511 512x1024: the seed-7 random state of
tests/test_gpu_swe.py::test_large_grid_eval_vs_reference.
"""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import fixtures as fx  # noqa: E402
from oracle import precise as PR  # noqa: E402
from oracle import pswe_oracle as O  # noqa: E402
from oracle import ref_lib as ref  # noqa: E402


def t511_state():
    po = O.ModelParams(phi_bar=9.80616e4)
    _, ss = fx.degree_order(511)
    st = fx.random_state(511, 7, 1e3, 1e-5) * (ss + 1.0) ** -1.5
    st[0, 0] = po.phi_bar * math.sqrt(2.0)
    st[1:, 0] = 0
    return st


def t255_state():
    from paper_1904_05988_b200.cases import balanced_random_state
    return balanced_random_state(255, 40.0, 20261019)  # == bench.bench_states()[0]


def rel(a, b):
    return [float(np.abs(a[i] - b[i]).max() / np.abs(b[i]).max()) for i in range(3)]


def main():
    po = O.ModelParams(phi_bar=9.80616e4)
    for R, nlat, nlon, make in ((255, 256, 512, t255_state), (511, 512, 1024, t511_state)):
        st = make()
        exact = PR.eval_nonlinear(st, po, PR.PrecisePlan(R, nlat, nlon)).astype(np.complex128)
        r = ref.RefPlan(R, nlat, nlon).eval_nonlinear(st, po)
        o = O.eval_nonlinear(st, po, O.TransformPlan(R, nlat, nlon))
        out = os.path.join(ROOT, "tests", "golden", f"precise_t{R}.npz")
        np.savez(out, state=st, exact=exact, grid=np.array([nlat, nlon]), ref_err=np.array(rel(r, exact)),
                 numpy_err=np.array(rel(o, exact)))
        print(out, "ref vs exact", rel(r, exact), "numpy vs exact", rel(o, exact))


if __name__ == "__main__":
    main()
