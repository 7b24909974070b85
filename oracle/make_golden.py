"""Generates tests/golden/golden_ref.npz by running the REFERENCE (oracle/_ref, compiled from
/root/reference/proj/src by oracle/build_ref.sh) on seeded inputs.

Run here (the reference is only present in this container):
    ./oracle/build_ref.sh && python oracle/make_golden.py
The fixtures pin both oracle/pswe_oracle.py (tests/test_oracle_golden.py) and the CUDA path
(tests/test_gpu_*.py), so GPU parity does not need /root/reference at run time.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import fixtures as fx  # noqa: E402
from oracle import ref_lib as ref  # noqa: E402
from oracle.pswe_oracle import ModelParams  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "golden_ref.npz")


def main():
    g = {}
    for n in (8, 24, 48, 96):
        g[f"gauss_{n}_mu"], g[f"gauss_{n}_w"] = ref.gauss(n)
    for r, smax, mu in ((0, 16, 0.3), (5, 31, -0.7), (40, 64, 0.999), (200, 256, 0.995)):
        g[f"leg_{r}_{smax}"] = ref.legendre_column(r, smax, mu)
    g["dealiased"] = np.array([[R, ref.lib().ref_dealiased_nlon(R)] for R in (15, 31, 42, 63, 85, 127, 128, 255, 511, 1023)])

    radius = 6.37122e6
    # transforms: dealiased T15 (24x48) and T31 (48x96), linear-grid override T31 (32x64)
    for tag, (R, nlat, nlon) in {"t15": (15, 0, 0), "t31": (31, 0, 0), "t31lin": (31, 32, 64)}.items():
        plan = ref.RefPlan(R, nlat, nlon)
        x = fx.random_field(R, 33)
        vort, div = fx.random_field(R, 34), fx.random_field(R, 35)
        g[f"{tag}_grid"] = np.array([plan.nlat, plan.nlon])
        g[f"{tag}_x"] = x
        g[f"{tag}_synth"] = plan.synthesise(x)
        g[f"{tag}_analyse"] = plan.analyse(g[f"{tag}_synth"])
        g[f"{tag}_vort"], g[f"{tag}_div"] = vort, div
        u, v = plan.uv_from_vortdiv(vort, div, radius)
        g[f"{tag}_u"], g[f"{tag}_v"] = u, v
        # vortdiv of a generic (non-band-limited) grid pair
        rng = np.random.default_rng(36)
        gu, gv = rng.standard_normal((plan.nlat, plan.nlon)), rng.standard_normal((plan.nlat, plan.nlon))
        g[f"{tag}_gu"], g[f"{tag}_gv"] = gu, gv
        g[f"{tag}_vd_vort"], g[f"{tag}_vd_div"] = plan.vortdiv_from_uv(gu, gv, radius)
        g[f"{tag}_direct_synth"] = ref.direct_synthesise(R, x, plan.mu, plan.nlon)

    # SWE operators
    for tag, (R, nlat, nlon) in {"t15": (15, 0, 0), "t31": (31, 0, 0), "t31lin": (31, 32, 64)}.items():
        plan = ref.RefPlan(R, nlat, nlon)
        p = ModelParams(nu=1e5)
        st = fx.smooth_state(R, p.phi_bar, 99)
        g[f"swe_{tag}_state"] = st
        g[f"swe_{tag}_lin"] = ref.eval_linear(R, st, p)
        g[f"swe_{tag}_nonlin"] = plan.eval_nonlinear(st, p)
        g[f"swe_{tag}_solve"] = ref.solve_implicit(R, st, 50.0, p)
        # a rough (unit-normal) state exercises every mode of the nonlinear products
        rough = fx.random_state(R, 7, 1e3, 1e-5)
        rough[0, 0] += p.phi_bar * np.sqrt(2.0)
        g[f"swe_{tag}_rough"] = rough
        g[f"swe_{tag}_rough_nonlin"] = plan.eval_nonlinear(rough, p)

    # quadrature + transfer tables
    for n in (2, 3, 5):
        nodes, q, qe, qi = ref.build_tables(n)
        g[f"tab{n}_nodes"], g[f"tab{n}_q"], g[f"tab{n}_qe"], g[f"tab{n}_qi"] = nodes, q, qe, qi
    for nf, nc in ((5, 3), (3, 2), (3, 3)):
        g[f"tp{nf}{nc}_restrict"], g[f"tp{nf}{nc}_interp"], g[f"tp{nf}{nc}_qfr"] = ref.transfer_matrices(nf, nc)

    # serial SDC (config-1 shape, reduced size): T15 dealiased, 3 nodes, 4 sweeps, dt=120, 3 steps
    p0 = ModelParams(phi_bar=9.80616 * 10000.0, nu=0.0)
    plan15 = ref.RefPlan(15)
    th = fx.smooth_state(15, p0.phi_bar, 5)
    g["sdc_theta0"] = th
    g["sdc_final"], g["sdc_res"], _ = ref.sdc_run(plan15, p0, 3, 4, 120.0, 3, th)

    # PFASST: T31/T15 dealiased grids, 5/3 nodes, dt = 60, 3 iterations
    th31 = fx.smooth_state(31, p0.phi_bar, 8)
    g["pf_theta0"] = th31
    for n_ts, n_blocks in ((1, 1), (2, 2), (4, 1)):
        r = ref.pfasst_run(31, (0, 0), 15, (0, 0), p0, 5, 3, n_ts, 60.0, 3, n_blocks, th31, serial=True)
        g[f"pf_nts{n_ts}_final"] = r.final
        g[f"pf_nts{n_ts}_res"] = r.residuals
        g[f"pf_nts{n_ts}_msgs"] = np.array([[m[0], m[1], ord(m[2]), m[3], m[4], m[5], m[6]] for m in r.messages],
                                          dtype=np.int32).reshape(-1, 7)
    # MLSDC T31/T15, 2 steps, 3 iterations
    g["ml_final"], g["ml_res"] = ref.mlsdc_run(31, (0, 0), 15, (0, 0), p0, 5, 3, 60.0, 3, 2, th31)

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
