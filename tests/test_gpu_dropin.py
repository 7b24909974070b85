"""Drop-in and end-to-end parity on the B200.

1. The reference's UNMODIFIED sdc::sdc_step and pf::run_block (compiled from /root/reference into
   oracle/_ref/libpintswe_gpu.so) driven through GpuImexOde — the reference's ImexOde plugin
   interface implemented over include/pswe.h (oracle/ref_build/gpu_imexode.cpp) — reproduce the
   reference's CPU results.
2. BASELINE configs on the native device-resident path (pswe_level / pswe_pfasst) against the
   reference CPU run on the same seeded inputs: config 1 (T63 SDC, 10 steps) and the config-3
   shape (T255/T127 PFASST, 5/3 nodes, dt 60 s, 4 iterations, 8 time steps in serial emulation).
Tolerances (BASELINE north star): final coefficients 1e-10 relative L-inf per field; residual
histories per iteration |r - r_ref| <= 1e-6 r_ref + 64 eps max|Phi|.
"""
import ctypes
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from _util import rel_diff_fields  # noqa: E402
from oracle import ref_lib as ref  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GPU_REF = os.path.join(ROOT, "oracle", "_ref", "libpintswe_gpu.so")
PHI_BAR = 9.80616 * 10000.0


def res_ok(mine, refv, state):
    floor = 64 * 2.0**-52 * np.abs(state[0]).max()
    return np.all(np.abs(np.asarray(mine) - np.asarray(refv)) <= 1e-6 * np.abs(refv) + floor)


@pytest.fixture(scope="module")
def P():
    import paper_1904_05988_b200 as P
    return P


@pytest.fixture(scope="module")
def gref():
    if not os.path.exists(GPU_REF):
        pytest.skip("oracle/_ref/libpintswe_gpu.so not built (needs /root/reference at build time)")
    L = ctypes.CDLL(GPU_REF)
    vp, ci, cd = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
    L.gpuref_last_error.restype = ctypes.c_char_p
    L.gpuref_sdc_run.argtypes = [ci, ci, ci, vp, ci, ci, cd, ci, vp, vp, vp]
    L.gpuref_pfasst_run.argtypes = [ci] * 6 + [vp, ci, ci, ci, cd, ci, ci, vp, vp, vp]
    L.gpuref_pfasst_run_mode.argtypes = [ci] * 6 + [vp, ci, ci, ci, cd, ci, ci, vp, vp, vp, ci]
    return L


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def test_reference_sdc_on_gpu_rhs(gref, golden):
    th = np.ascontiguousarray(golden["sdc_theta0"])
    fin = np.zeros_like(th)
    res = np.zeros(3)
    prm = ref.Params(6.37122e6, 7.292e-5, 9.80616, PHI_BAR, 0.0)
    rc = gref.gpuref_sdc_run(15, 0, 0, ctypes.byref(prm), 3, 4, 120.0, 3, _p(th), _p(fin), _p(res))
    assert rc == 0, gref.gpuref_last_error()
    assert rel_diff_fields(fin, golden["sdc_final"]) < 1e-10
    assert res_ok(res, golden["sdc_res"], fin)


def test_reference_pfasst_on_gpu_rhs(gref, golden):
    th = np.ascontiguousarray(golden["pf_theta0"])
    fin = np.zeros_like(th)
    res = np.zeros((1, 4, 4))
    prm = ref.Params(6.37122e6, 7.292e-5, 9.80616, PHI_BAR, 0.0)
    rc = gref.gpuref_pfasst_run(31, 0, 0, 15, 0, 0, ctypes.byref(prm), 5, 3, 4, 60.0, 3, 1, _p(th), _p(fin),
                                _p(res))
    assert rc == 0, gref.gpuref_last_error()
    assert rel_diff_fields(fin, golden["pf_nts4_final"]) < 1e-10
    assert res_ok(res, golden["pf_nts4_res"], fin)


def test_reference_pfasst_threaded_on_gpu_rhs(gref, golden):
    """The reference's Mode::threaded (one std::thread per worker, pfasst.cpp:219-234) sharing ONE
    GpuImexOde between the 4 workers (runner.cpp:143-144): the adapter serialises its calls, and
    the block reproduces the serial reference result."""
    th = np.ascontiguousarray(golden["pf_theta0"])
    fin = np.zeros_like(th)
    res = np.zeros((1, 4, 4))
    prm = ref.Params(6.37122e6, 7.292e-5, 9.80616, PHI_BAR, 0.0)
    rc = gref.gpuref_pfasst_run_mode(31, 0, 0, 15, 0, 0, ctypes.byref(prm), 5, 3, 4, 60.0, 3, 1, _p(th), _p(fin),
                                     _p(res), 1)
    assert rc == 0, gref.gpuref_last_error()
    assert rel_diff_fields(fin, golden["pf_nts4_final"]) < 1e-10
    assert res_ok(res, golden["pf_nts4_res"], fin)


def test_config1_sdc_t63(P):
    """BASELINE config 1: T63 (96x192), 3 Lobatto nodes, 4 sweeps, dt 120 s, 10 steps."""
    if not ref.available():
        pytest.skip("reference library not built")
    from paper_1904_05988_b200.cases import config_state
    th = config_state(1)
    p = P.ModelParams(phi_bar=PHI_BAR)
    plan = P.TransformPlan(63)
    assert (plan.nlat, plan.nlon) == (96, 192)
    lvl = P.Level(plan, p, 3)
    fin, res = P.sdc_run(lvl, torch.as_tensor(th).cuda(), 120.0, 4, 10)
    fin = fin.cpu().numpy()
    rfin, rres, _ = ref.sdc_run(ref.RefPlan(63), p, 3, 4, 120.0, 10, th)
    assert rel_diff_fields(fin, rfin) < 1e-10
    assert res_ok(res.cpu().numpy(), rres, fin)


def test_config3_shape_pfasst_t255(P):
    """Config-3 shape on the reference grids: T255 (384x768) / T127 (192x384), 5/3 nodes,
    dt 60 s, 4 iterations, one block of 8 time steps (serial emulation on one GPU)."""
    if not ref.available():
        pytest.skip("reference library not built")
    from paper_1904_05988_b200.cases import config_state
    p = P.ModelParams(phi_bar=PHI_BAR)
    pf_plan, pc_plan = P.TransformPlan(255), P.TransformPlan(127)
    th = config_state(3, pf_plan)
    pair = P.TransferPair(P.Level(pf_plan, p, 5), P.Level(pc_plan, p, 3))
    pf = P.Pfasst(pair, P.BlockConfig(8, 60.0, 4))
    fin, hist = P.run_blocks(pf, torch.as_tensor(th).cuda(), 1)
    fin = fin.cpu().numpy()
    r = ref.pfasst_run(255, (0, 0), 127, (0, 0), p, 5, 3, 8, 60.0, 4, 1, th, serial=True)
    assert rel_diff_fields(fin, r.final) < 1e-10
    assert res_ok(hist, r.residuals, fin)
    mine = sorted((m[0], m[1], ord(m[2]), m[3], m[4], m[5], m[6]) for m in pf.messages())
    assert mine == sorted((m[0], m[1], ord(m[2]), m[3], m[4], m[5], m[6]) for m in r.messages)
