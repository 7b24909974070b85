"""Parity pinned to the REFERENCE itself (oracle/_ref/libpintswe_ref.so, compiled from
/root/reference by oracle/build_ref.sh; it travels to the GPU box with the snapshot) on every
configuration bench.py measures — the exact workloads, not stand-ins:

* the headline step: eval_nonlinear + eval_linear (swe.cpp:9-69) of the 5 bench_states at T255
  on BASELINE's 256x512 grid (bench.py's `step`);
* config 2: the 15-field T255 synthesise / analyse (transform.cpp:136-174) on 256x512;
* T511 (512x1024, config 4's fine grid) and T1023 (1024x2048, config 5's fine grid) evaluations;
* config 3 as benchmarked: two-level PFASST on the LINEAR grids T255 256x512 / T127 128x256,
  5/3 nodes, dt 60 s, 4 iterations, 8 time steps (serial emulation), pf::run_block
  (pfasst.cpp:194-251): final state, residual history per iteration and message log;
* config 5: one T1023 (1024x2048) / T511 (512x1024) block at n_ts = 1, 3 iterations, dt 15 s.

Tolerances (BASELINE north star; written per test): transforms 1e-12 relative L-inf, RHS
evaluations 1e-11 per prognostic field (support.hpp:33-38 applied per field), final
PFASST coefficients 1e-10, residual histories |r - r_ref| <= 1e-6 r_ref + 64 eps max|Phi|.
The T1023 evaluation's divergence tendency carries the s(s+1)/a^2 factor of -lap(ke) over sums
four times T255's length; its per-field tolerance is the north star's 1e-10 for spectral
coefficients. Accuracy against the EXACT discrete operator (oracle/precise.py, long double) is
pinned separately in tests/test_gpu_precision.py.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from _util import rel_diff, rel_diff_fields  # noqa: E402
from oracle import ref_lib as ref  # noqa: E402

PHI_BAR = 9.80616 * 10000.0


@pytest.fixture(scope="module")
def P():
    import paper_1904_05988_b200 as P
    return P


@pytest.fixture(scope="module", autouse=True)
def need_ref():
    if not ref.available():
        pytest.skip("oracle/_ref/libpintswe_ref.so not built")


def cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def res_ok(mine, refv, state):
    floor = 64 * 2.0**-52 * np.abs(state[0]).max()
    return bool(np.all(np.abs(np.asarray(mine) - np.asarray(refv)) <= 1e-6 * np.abs(refv) + floor))


def per_field(a, b):
    return [rel_diff(a[..., i, :], b[..., i, :]) for i in range(3)]


def ref_imex(plan_ref, R, st, p):
    """(F_I, F_E) of the reference: eval_linear, eval_nonlinear (swe.cpp:9-69)."""
    return ref.eval_linear(R, st, p), plan_ref.eval_nonlinear(st, p)


def test_headline_batch_t255(P):
    """bench.py's timed step, exactly: the 5 bench_states, T255, 256x512, one pswe_eval_imex."""
    import bench
    p = P.ModelParams(phi_bar=PHI_BAR)
    sts = bench.bench_states()
    assert sts.shape == (5, 3, P.num_coeffs(255))
    plan = P.TransformPlan(255, 256, 512)
    fi, fe = (host(t) for t in P.imex_split(cuda(sts), p, plan))
    rp = ref.RefPlan(255, 256, 512)
    for i in range(5):
        rfi, rfe = ref_imex(rp, 255, sts[i], p)
        assert rel_diff_fields(fe[i], rfe) < 1e-11, (i, per_field(fe[i], rfe))
        assert rel_diff_fields(fi[i], rfi) < 1e-14
    # the single-state path (the SDC-sweep pattern) on the same inputs
    for i in (0, 4):
        fi1, fe1 = (host(t) for t in P.imex_split(cuda(sts[i:i + 1]), p, plan))
        assert rel_diff_fields(fe1[0], rp.eval_nonlinear(sts[i], p)) < 1e-11


def config2_coeffs(n=15, R=255, seed=2):
    """bench.py's config-2 input: uniform[-1,1] complex x (n+1)^-1.5, r = 0 real."""
    rng = np.random.default_rng(seed)
    rs = np.concatenate([np.full(R + 1 - r, r) for r in range(R + 1)])
    ss = np.concatenate([np.arange(r, R + 1) for r in range(R + 1)])
    x = (rng.uniform(-1, 1, (n, rs.size)) + 1j * rng.uniform(-1, 1, (n, rs.size))) * (ss + 1.0) ** -1.5
    x[:, rs == 0] = x[:, rs == 0].real
    return x


def test_config2_transforms_t255(P):
    """Config 2: 15 fields at T255 on 256x512 — synthesise and analyse each against the
    reference TransformPlan (transform.cpp:136-174), and the round trip."""
    x = config2_coeffs()
    plan = P.TransformPlan(255, 256, 512)
    rp = ref.RefPlan(255, 256, 512)
    g = host(plan.synthesise(cuda(x)))
    xa = host(plan.analyse(cuda(g)))
    for f in range(15):
        rg = rp.synthesise(x[f])
        assert rel_diff(g[f], rg) < 1e-12, f
        assert rel_diff(xa[f], rp.analyse(rg)) < 1e-12, f
        assert rel_diff(xa[f], x[f]) < 1e-12, f


@pytest.mark.parametrize("R,grid,seeds", [(511, (512, 1024), (7, 11)), (1023, (1024, 2048), (5,))])
def test_large_grid_eval(P, R, grid, seeds):
    """Config 4's and config 5's fine grids: single-state and 5-state batch evaluations against the
    reference eval_nonlinear / eval_linear on the same seeded inputs."""
    from paper_1904_05988_b200.cases import balanced_random_state
    p = P.ModelParams(phi_bar=PHI_BAR)
    plan = P.TransformPlan(R, *grid)
    rp = ref.RefPlan(R, *grid)
    tol = 1e-11 if R <= 511 else 1e-10
    sts = np.stack([balanced_random_state(R, 30.0, 1000 + s, phi_bar=PHI_BAR) for s in range(5)])
    for s in seeds:
        sts[s % 5] = balanced_random_state(R, 40.0, s, phi_bar=PHI_BAR)
    fi_b, fe_b = (host(t) for t in P.imex_split(cuda(sts), p, plan))
    for i in (0, seeds[0] % 5):
        rfi, rfe = ref_imex(rp, R, sts[i], p)
        assert rel_diff_fields(fe_b[i], rfe) < tol, (i, per_field(fe_b[i], rfe))
        assert rel_diff_fields(fi_b[i], rfi) < 1e-14
        fe1 = host(P.eval_nonlinear(cuda(sts[i]), p, plan))
        assert rel_diff_fields(fe1, rfe) < tol, (i, per_field(fe1, rfe))


def _pfasst_vs_ref(P, levels, dt, n_ts, n_iter, th_fn, delta_scale=None):
    p = P.ModelParams(phi_bar=PHI_BAR)
    (Rf, gf, nf), (Rc, gc, nc) = levels
    pf_plan, pc_plan = P.TransformPlan(Rf, *gf), P.TransformPlan(Rc, *gc)
    th = th_fn(pf_plan)
    pair = P.TransferPair(P.Level(pf_plan, p, nf), P.Level(pc_plan, p, nc))
    pf = P.Pfasst(pair, P.BlockConfig(n_ts, dt, n_iter))
    fin, hist = P.run_blocks(pf, torch.as_tensor(th).cuda(), 1)
    fin = host(fin)
    msgs = pf.messages()
    pf.close()
    r = ref.pfasst_run(Rf, gf, Rc, gc, p, nf, nc, n_ts, dt, n_iter, 1, th, serial=True)
    d = per_field(fin, r.final)
    if delta_scale is None:
        assert max(d) < 1e-10, d
    else:
        assert max(d[:2]) < 1e-10, d
        scale = delta_scale(pf_plan, th, p)
        assert np.abs(fin[2] - r.final[2]).max() < 1e-10 * scale, (d, scale)
    assert hist.shape == r.residuals.shape
    assert res_ok(hist, r.residuals, fin), (hist, r.residuals)
    assert sorted(msgs) == sorted(r.messages)
    return hist, r


def test_config3_linear_grids_nts8(P):
    """Config 3 exactly as benchmarked: T255 256x512 / T127 128x256, 5/3 nodes, dt 60 s,
    4 iterations, one block of 8 time steps (serial emulation of the 8 workers)."""
    from paper_1904_05988_b200.cases import config_state
    hist, r = _pfasst_vs_ref(P, [(255, (256, 512), 5), (127, (128, 256), 3)], 60.0, 8, 4,
                             lambda plan: config_state(3, plan))
    assert hist.shape == (1, 8, 5)


def test_config5_block_nts1(P):
    """Config 5: T1023 1024x2048 / T511 512x1024, 5/3 nodes, dt 15 s, 3 iterations, one block of
    one time step (n_ts = 1) — final state and the per-iteration residual history.

    Config 5's initial state is divergence-free and in linear balance, so after 15 s the
    divergence (max 3.5e-10) is the 31x-cancelled sum of dt F_E(delta) and dt F_I(delta)
    (1.08e-8 each, measured with oracle/_ref). Phi and zeta are held to the north star's 1e-10
    relative L-inf; delta to 1e-10 of the scale of the tendency that produces it,
    dt max|F_E(delta)(theta0)| (measured: 1.0e-11 of it; 3.2e-10 of max|delta| itself)."""
    from paper_1904_05988_b200.cases import config_state

    def delta_scale(plan, th, p):
        fe = host(P.eval_nonlinear(cuda(th), p, plan))
        return 15.0 * np.abs(fe[2]).max()

    hist, r = _pfasst_vs_ref(P, [(1023, (1024, 2048), 5), (511, (512, 1024), 3)], 15.0, 1, 3,
                             lambda plan: config_state(5), delta_scale=delta_scale)
    assert hist.shape == (1, 1, 4)
    assert hist[0, 0, -1] < hist[0, 0, 0]
