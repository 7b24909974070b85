"""GPU parity of SDC (sdc.cpp), MLSDC (multilevel.cpp) and serial-emulation PFASST
(pfasst.cpp) against the reference's own runs (tests/golden): final spectral coefficients to
1e-10 relative L-inf per field, residual histories per iteration to
|r - r_ref| <= 1e-6 r_ref + 64 eps max|Phi|, message logs identical."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from _util import rel_diff_fields  # noqa: E402
from oracle import fixtures as fx  # noqa: E402
from oracle import pswe_oracle as O  # noqa: E402

PHI_BAR = 9.80616 * 10000.0


@pytest.fixture(scope="module")
def P():
    import paper_1904_05988_b200 as P
    return P


def cuda(a):
    return torch.as_tensor(np.asarray(a)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def res_ok(mine, ref, state):
    floor = 64 * 2.0**-52 * np.abs(state[0]).max()
    return np.all(np.abs(np.asarray(mine) - np.asarray(ref)) <= 1e-6 * np.abs(ref) + floor)


def test_quadrature_tables(P, golden):
    for n in (2, 3, 5):
        t = P.build_tables(n)
        for k, a in (("nodes", t.nodes), ("q", t.q), ("qe", t.q_exp), ("qi", t.q_imp)):
            np.testing.assert_allclose(a, golden[f"tab{n}_{k}"], rtol=1e-14, atol=4e-15)


@pytest.mark.parametrize("mode", [0, 1])
def test_sdc_steps(P, golden, mode):
    plan = P.TransformPlan(15, 0, 0, mode)
    lvl = P.Level(plan, P.ModelParams(phi_bar=PHI_BAR), 3)
    fin, res = P.sdc_run(lvl, cuda(golden["sdc_theta0"]), 120.0, 4, 3)
    fin = host(fin)
    assert rel_diff_fields(fin, golden["sdc_final"]) < 1e-10
    assert res_ok(host(res), golden["sdc_res"], fin)


def test_sweep_matches_oracle_sweep(P):
    """One sweep with a FAS term from an arbitrary space-time state, node by node."""
    R = 15
    p = P.ModelParams(phi_bar=PHI_BAR, nu=1e5)
    plan = P.TransformPlan(R)
    lvl = P.Level(plan, p, 5)
    ode = O.SweOde(O.TransformPlan(R), O.ModelParams(phi_bar=PHI_BAR, nu=1e5))
    th = fx.smooth_state(R, PHI_BAR, 3)
    lvl.spread(cuda(th))
    sts = O.spread(th, 5, ode)
    tau = [fx.smooth_state(R, 0.0, 10 + m) * 1e-3 for m in range(5)]
    lvl.sweep(60.0, cuda(np.stack(tau)))
    O.sweep(sts, 60.0, O.build_tables(5), ode, tau)
    for m in range(5):
        assert rel_diff_fields(host(lvl.state(m)), sts.state[m]) < 1e-11
        assert rel_diff_fields(host(lvl.f_exp(m)), sts.f_exp[m]) < 1e-10
    r = float(host(lvl.collocation_residual(60.0))[0])
    rr = O.collocation_residual(sts, 60.0, O.build_tables(5))
    assert abs(r - rr) <= 1e-6 * rr + 64 * 2**-52 * np.abs(th[0]).max()


@pytest.mark.parametrize("nodes,R", [(2, 15), (3, 31), (5, 63)])
def test_fused_tail_residual_bit_identical(P, nodes, R):
    """sdc_step's last sweep ends in one kernel that finishes the last node's evaluation and
    computes the collocation residual (tail_residual_kernel); the separate residual kernel over the
    stored right-hand sides must give the same bits, and the stored F[M] must be the separate
    tail's (a second step from the same state reproduces every node bit for bit)."""
    prm = P.ModelParams(phi_bar=PHI_BAR, nu=1e5)
    lvl = P.Level(P.TransformPlan(R), prm, nodes)
    th = cuda(fx.smooth_state(R, PHI_BAR, 5))
    r_fused = torch.zeros(1, dtype=torch.float64, device="cuda")
    lvl.sdc_step(th, 90.0, 2, r_fused)
    r_sep = lvl.collocation_residual(90.0)
    torch.cuda.synchronize()
    assert host(r_fused)[0] == host(r_sep)[0] and host(r_sep)[0] > 0
    first = [host(lvl.f_exp(m)).copy() for m in range(nodes)] + [host(lvl.f_imp(m)).copy() for m in range(nodes)]
    lvl.sdc_step(th, 90.0, 2, None)  # the last sweep's tail by the separate kernel
    again = [host(lvl.f_exp(m)) for m in range(nodes)] + [host(lvl.f_imp(m)) for m in range(nodes)]
    for a, b in zip(first, again):
        assert np.array_equal(a, b)


def _pair(P, mode=0):
    p = P.ModelParams(phi_bar=PHI_BAR)
    pf, pc = P.TransformPlan(31, 0, 0, mode), P.TransformPlan(15, 0, 0, mode)
    fine, coarse = P.Level(pf, p, 5), P.Level(pc, p, 3)
    return P.TransferPair(fine, coarse), (pf, pc)


def test_transfers(P):
    x = np.stack([fx.smooth_state(31, PHI_BAR, s) for s in range(2)])
    y = host(P.restrict_space(cuda(x), 31, 15))
    np.testing.assert_array_equal(y, O.restrict_space(x, 31, 15))
    z = host(P.interpolate_space(cuda(y), 15, 31))
    np.testing.assert_array_equal(z, O.interpolate_space(y, 15, 31))


def test_mlsdc(P, golden):
    pair, _ = _pair(P)
    s = cuda(golden["pf_theta0"])
    res = torch.zeros(2, dtype=torch.float64, device="cuda")
    for n in range(2):
        last = P.mlsdc_step(pair, s, 60.0, 3, res[n:n + 1])
        s = last.clone()
    fin = host(s)
    assert rel_diff_fields(fin, golden["ml_final"]) < 1e-10
    assert res_ok(host(res), golden["ml_res"], fin)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("n_ts,n_blocks", [(1, 1), (2, 2), (4, 1)])
def test_pfasst_serial_emulation(P, golden, n_ts, n_blocks, mode):
    pair, _ = _pair(P, mode)
    pf = P.Pfasst(pair, P.BlockConfig(n_ts, 60.0, 3))
    fin, hist = P.run_blocks(pf, cuda(golden["pf_theta0"]), n_blocks)
    fin = host(fin)
    assert rel_diff_fields(fin, golden[f"pf_nts{n_ts}_final"]) < 1e-10
    assert res_ok(hist, golden[f"pf_nts{n_ts}_res"], fin)
    ref_log = sorted(tuple(int(v) for v in m) for m in golden[f"pf_nts{n_ts}_msgs"])
    mine = sorted((m[0], m[1], ord(m[2]), m[3], m[4], m[5], m[6]) for m in pf.messages())
    assert mine == ref_log


@pytest.mark.parametrize("n_ts", [1, 2])
def test_run_blocks_matches_block_by_block(P, golden, n_ts):
    """pswe_pfasst_run_blocks (runner.cpp:145-151, no host synchronisation between blocks) against
    the same blocks run one call at a time with the host read-back: bit-identical final state and
    residual history; n_blocks = 0 leaves theta0 as the result."""
    th = cuda(golden["pf_theta0"])
    pair, _ = _pair(P)
    pf = P.Pfasst(pair, P.BlockConfig(n_ts, 60.0, 3))
    fin, hist = P.run_blocks(pf, th, 3)
    s, rows = th.clone(), []
    for _ in range(3):
        f1, r1 = pf.run_block(s)
        s.copy_(f1)
        rows.append(r1)
    np.testing.assert_array_equal(host(fin), host(s))
    np.testing.assert_array_equal(hist, np.array(rows))
    fin0, hist0 = P.run_blocks(pf, th, 0)
    np.testing.assert_array_equal(host(fin0), host(th))
    assert hist0.shape == (0, n_ts, 4)
    pf.close()


def test_pfasst_nccl_executor_single_rank(P, golden):
    """The NCCL executor on one GPU (world = 1): communicator set-up, the final-state broadcast and
    the residual all-gather; the result must equal the serial-emulation / reference run."""
    pytest.importorskip("torch")
    pair, _ = _pair(P)
    try:
        uid = P.pfasst.nccl_unique_id()
    except Exception as e:  # NCCL not loadable on this machine
        pytest.skip(f"NCCL unavailable: {e}")
    pf = P.Pfasst(pair, P.BlockConfig(1, 60.0, 3), rank=0, world=1, nccl_id=uid)
    fin, hist = P.run_blocks(pf, cuda(golden["pf_theta0"]), 1)
    fin = host(fin)
    assert rel_diff_fields(fin, golden["pf_nts1_final"]) < 1e-10
    assert res_ok(hist, golden["pf_nts1_res"], fin)
    pf.close()


def test_level_rejects_unsupported_node_counts(P):
    """Gauss-Lobatto tables exist for 2, 3, 5 nodes (sdc.cpp; the kernels size their node arrays
    for at most 5): other counts are an error, not an out-of-bounds launch."""
    plan = P.TransformPlan(15)
    for nn in (1, 4, 6):
        with pytest.raises(P._lib.PsweError):
            P.Level(plan, P.ModelParams(), nn)


def test_sweep_emitted_xtiles_bit_identical(tmp_path):
    """The SDC node update writes the next evaluation's X tiles itself (the prep launch skipped);
    the sweeps must give the same bits as with the separate prep kernel (PSWE_NO_SWEEP_PREP=1),
    at T255 / 5 nodes, T127 / 3 nodes (fused) and T63 / 2 nodes."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ("0", "1"):
        out = tmp_path / f"sw{env}.npz"
        subprocess.run([sys.executable, os.path.join(root, "tools", "sweep_dump.py"), str(out)], check=True,
                       env={**os.environ, "PSWE_NO_SWEEP_PREP": env}, timeout=300)
        outs.append(np.load(out))
    assert sorted(outs[0].files) == sorted(outs[1].files)
    for k in outs[0].files:
        np.testing.assert_array_equal(outs[0][k], outs[1][k])


def test_worker0_refresh_elision_bit_identical(tmp_path):
    """The executor skips worker 0's node-0 re-evaluations after Steps C/D (its node-0 states never
    change: pfasst.cpp:152, :175 recompute the same F); results must be bit-identical to running
    them (PSWE_PFASST_NO_ELIDE=1) - two and three levels, n_ts 1, 2, 4, eager and graph blocks."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ("0", "1"):
        out = tmp_path / f"pf{env}.npz"
        subprocess.run([sys.executable, os.path.join(root, "tools", "pfasst_dump.py"), str(out)], check=True,
                       env={**os.environ, "PSWE_PFASST_NO_ELIDE": env}, timeout=600)
        outs.append(np.load(out))
    assert sorted(outs[0].files) == sorted(outs[1].files)
    for k in outs[0].files:
        np.testing.assert_array_equal(outs[0][k], outs[1][k])
