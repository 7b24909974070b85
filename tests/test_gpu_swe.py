"""GPU parity of the SWE right-hand side (swe.cpp) against the reference's outputs
(tests/golden) and the numpy oracle, plus the reference's property tests (test_swe.cpp)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from _util import rel_diff_fields  # noqa: E402
from oracle import fixtures as fx  # noqa: E402
from oracle import pswe_oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def P():
    import paper_1904_05988_b200 as P
    return P


def cuda(a):
    return torch.as_tensor(np.asarray(a)).cuda()


def host(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("tag,R", [("t15", 15), ("t31", 31), ("t31lin", 31)])
def test_operators_vs_reference(P, golden, tag, R, mode):
    nlat, nlon = (int(v) for v in golden[f"{tag}_grid"])
    plan = P.TransformPlan(R, nlat, nlon, mode)
    p = P.ModelParams(nu=1e5)
    st = cuda(golden[f"swe_{tag}_state"])
    assert rel_diff_fields(host(P.eval_linear(R, st, p)), golden[f"swe_{tag}_lin"]) < 1e-14
    assert rel_diff_fields(host(P.solve_implicit(R, st, 50.0, p)), golden[f"swe_{tag}_solve"]) < 1e-14
    assert rel_diff_fields(host(P.eval_nonlinear(st, p, plan)), golden[f"swe_{tag}_nonlin"]) < 1e-11
    rough = cuda(golden[f"swe_{tag}_rough"])
    assert rel_diff_fields(host(P.eval_nonlinear(rough, p, plan)), golden[f"swe_{tag}_rough_nonlin"]) < 1e-11
    fi, fe = P.imex_split(st, p, plan)
    assert rel_diff_fields(host(fi), golden[f"swe_{tag}_lin"]) < 1e-14
    assert rel_diff_fields(host(fe), golden[f"swe_{tag}_nonlin"]) < 1e-11


@pytest.mark.parametrize("R,grid", [(63, (96, 192)), (255, (256, 512))])
def test_eval_vs_numpy_oracle(P, R, grid):
    """eval_nonlinear at T63 (reference grid) and T255 on BASELINE's 256x512 grid."""
    plan = P.TransformPlan(R, grid[0], grid[1])
    ref = O.TransformPlan(R, grid[0], grid[1])
    p = P.ModelParams(phi_bar=9.80616 * 1e4)
    st = fx.random_state(R, 5, 1e3, 1e-5)
    _, ss = fx.degree_order(R)
    st *= (ss + 1.0) ** -1.5
    st[0, 0] = p.phi_bar * math.sqrt(2.0)
    st[1:, 0] = 0
    po = O.ModelParams(phi_bar=p.phi_bar)
    mine = host(P.eval_nonlinear(cuda(st), p, plan))
    assert rel_diff_fields(mine, O.eval_nonlinear(st, po, ref)) < 1e-11


@pytest.mark.parametrize("R,grid", [(511, (512, 1024))])
def test_large_grid_eval_vs_reference(P, R, grid):
    """T511 on BASELINE config 4's 512x1024 grid: the large-grid forward configuration (4-warp
    tasks, 2 chunks per warp, cut by polar-skip weight) and the single-state one, both against the
    REFERENCE (oracle/_ref) - the batch-vs-single test alone would not see a chunk the shared task
    table dropped. Tolerance 2e-11 per field = the two implementations' distances from the EXACT
    operator added: the GPU is held to 1e-11 of it (tests/test_gpu_precision.py), and the
    reference build itself sits up to 8.6e-12 from it on these states (seed 11: Phi 5.6e-12,
    delta 8.6e-12; seed 7: 2.8e-12; oracle/precise.py, long double)."""
    from oracle import ref_lib as ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    plan = P.TransformPlan(R, grid[0], grid[1])
    rp = ref.RefPlan(R, grid[0], grid[1])
    p = P.ModelParams(phi_bar=9.80616 * 1e4)
    _, ss = fx.degree_order(R)
    sts = []
    for seed in (7, 8, 9, 10, 11):
        st = fx.random_state(R, seed, 1e3, 1e-5) * (ss + 1.0) ** -1.5
        st[0, 0] = p.phi_bar * math.sqrt(2.0)
        st[1:, 0] = 0
        sts.append(st)
    sts = np.stack(sts)
    batch = host(P.imex_split(cuda(sts), p, plan)[1])
    for i in (0, 4):
        want = rp.eval_nonlinear(sts[i], p)
        assert rel_diff_fields(batch[i], want) < 2e-11
        assert rel_diff_fields(host(P.eval_nonlinear(cuda(sts[i]), p, plan)), want) < 2e-11


def test_batched_equals_single(P):
    R = 31
    plan = P.TransformPlan(R)
    p = P.ModelParams(nu=1e5)
    sts = np.stack([fx.smooth_state(R, p.phi_bar, s) for s in range(5)])
    batch = host(P.imex_split(cuda(sts), p, plan)[1])
    for i in range(5):
        single = host(P.eval_nonlinear(cuda(sts[i]), p, plan))
        np.testing.assert_array_equal(batch[i], single)


@pytest.mark.parametrize("n", [6, 7, 11])
@pytest.mark.parametrize("R,grid", [(63, (96, 192)), (255, (256, 512))])
def test_large_batches_equal_single(P, R, grid, n):
    """Batches above 5 states split into several column groups (G tiles of <= 5 states, inverse
    X tiles of 4 NT columns): every state must match its own single-state evaluation (to rounding:
    on the 256 x 512 grid single states take the two-pass radix-16 FFT plan, batches the
    three-pass one)."""
    from paper_1904_05988_b200.cases import balanced_random_state
    plan = P.TransformPlan(R, grid[0], grid[1])
    p = P.ModelParams(phi_bar=9.80616 * 1e4)
    sts = np.stack([balanced_random_state(R, 40.0, 100 + s, phi_bar=p.phi_bar) for s in range(n)])
    fi_b, fe_b = (host(t) for t in P.imex_split(cuda(sts), p, plan))
    for i in range(n):
        fi, fe = (host(t) for t in P.imex_split(cuda(sts[i:i + 1]), p, plan))
        assert rel_diff_fields(fe_b[i], fe[0]) < 1e-12
        assert rel_diff_fields(fi_b[i], fi[0]) < 1e-15


@pytest.mark.parametrize("R,grid", [(511, (768, 1536)), (1023, (1024, 2048))])
def test_large_grid_batch_equals_single(P, R, grid):
    """T511 / T1023: a 5-state batch (streamed TMA inverse, large-grid forward configuration) must
    match single-state evaluations (T1023: recurrence inverse) - two independent implementations
    of the inverse Legendre contraction checked against each other."""
    from paper_1904_05988_b200.cases import balanced_random_state
    plan = P.TransformPlan(R, grid[0], grid[1])
    p = P.ModelParams(phi_bar=9.80616 * 1e4)
    sts = np.stack([balanced_random_state(R, 30.0, 300 + s, phi_bar=p.phi_bar) for s in range(5)])
    fi_b, fe_b = (host(t) for t in P.imex_split(cuda(sts), p, plan))
    for i in (0, 4):
        fi, fe = (host(t) for t in P.imex_split(cuda(sts[i:i + 1]), p, plan))
        assert rel_diff_fields(fe_b[i], fe[0]) < 1e-12
        assert rel_diff_fields(fi_b[i], fi[0]) < 1e-15


def test_nonlinear_properties(P):
    """test_swe.cpp:75-129."""
    R = 15
    plan = P.TransformPlan(R)
    p = P.ModelParams(nu=1e5)
    s = np.zeros((3, P.num_coeffs(R)), dtype=np.complex128)
    s[0] = fx.random_field(R, 5) * 1e3
    s[0, 0] += p.phi_bar * math.sqrt(2)
    out = host(P.eval_nonlinear(cuda(s), p, plan))
    assert np.abs(out).max() < 1e-12 * np.abs(s[0]).max()
    sm = fx.smooth_state(R, p.phi_bar, 17)
    nl = host(P.eval_nonlinear(cuda(sm), p, plan))
    li = host(P.eval_linear(R, cuda(sm), p))
    assert nl[0, 0] == 0 and nl[2, 0] == 0 and li[0, 0] == 0 and li[2, 0] == 0
    s = np.stack([fx.random_field(R, 31), fx.random_field(R, 32), fx.random_field(R, 33)])
    _, ss = fx.degree_order(R)
    decay = np.exp(-((ss / 3.0) ** 2))
    s[0] *= decay
    s[1] *= 1e-6 * decay
    s[2] *= 1e-6 * decay
    s[1, 0] = s[2, 0] = 0
    # test_swe.cpp:370-377 keeps the default phi_bar, so Phi' = Phi - phi_bar is dominated by
    # -phi_bar and the flux is LINEAR in the winds: the reference's own code gives ratio 2.0000005
    # there (checked with oracle/_ref), i.e. that reference test cannot pass as written. We check
    # the reference's value, and the intended quadratic property with phi_bar = 0.
    q = P.ModelParams(omega=0.0, nu=0.0)
    n1 = np.abs(host(P.eval_nonlinear(cuda(s), q, plan))[0]).max()
    n2 = np.abs(host(P.eval_nonlinear(cuda(0.5 * s), q, plan))[0]).max()
    assert abs(n1 / n2 - 2.0000004845649686) < 1e-9
    q = P.ModelParams(omega=0.0, nu=0.0, phi_bar=0.0)
    n1 = np.abs(host(P.eval_nonlinear(cuda(s), q, plan))[0]).max()
    n2 = np.abs(host(P.eval_nonlinear(cuda(0.5 * s), q, plan))[0]).max()
    assert abs(n1 / n2 - 4.0) < 1e-9


def test_implicit_solve_residual(P):
    """test_swe.cpp:131-170."""
    R = 10
    for nu in (0.0, 1.0):
        p = P.ModelParams(radius=1.0, omega=1.0, gravity=1.0, phi_bar=1.0, nu=nu)
        for c in (1e-3, 0.3, 1.0, 1e3):
            b = cuda(fx.random_state(R, 7 + int(c * 10)))
            x = P.solve_implicit(R, b, c, p)
            res = host(x - c * P.eval_linear(R, x, p) - b)
            assert np.abs(res).max() < 1e-12 * np.abs(host(b)).max()
    p = P.ModelParams(radius=1.0, omega=1.0, gravity=1.0, phi_bar=1.0, nu=1.0)
    b = np.zeros((3, P.num_coeffs(R)), dtype=np.complex128)
    b[1, O.index(R, 0, 2)] = 1.0
    x = host(P.solve_implicit(R, cuda(b), 1.0, p))
    assert abs(x[1, O.index(R, 0, 2)].real - 1.0 / 7.0) < 1e-15


def test_zonal_jet_is_balanced(P):
    """config 4's jet (cases.add_zonal_jet): a zonal flow in gradient-wind balance is a steady
    state of the nonlinear SWE, so its tendencies are small next to the same jet without the
    balancing geopotential."""
    from paper_1904_05988_b200.cases import add_zonal_jet
    R = 85
    plan = P.TransformPlan(R, 128, 256)
    p = P.ModelParams(phi_bar=9.80616 * 1e4)
    base = np.zeros((3, P.num_coeffs(R)), dtype=np.complex128)
    base[0, 0] = p.phi_bar * math.sqrt(2.0)
    jet = add_zonal_jet(base, plan)
    unbal = jet.copy()
    unbal[0] = base[0]
    def tendency(st):  # F_I + F_E: the balance is a cancellation between the two parts
        fi, fe = P.imex_split(cuda(st), p, plan)
        return np.abs(host(fi) + host(fe)).max(axis=1)

    t_bal, t_unb = tendency(jet), tendency(unbal)
    # Phi and zeta tendencies vanish for any zonal flow; the divergence tendency is the balance
    assert t_bal[2] < 3e-2 * t_unb[2]
    assert t_bal[0] < 1e-6 * p.phi_bar and t_bal[1] < 1e-12


@pytest.mark.parametrize("R,grid,n", [(21, (45, 96), 1), (21, (45, 96), 3), (31, (49, 96), 5)])
def test_eval_odd_latitudes_vs_oracle(P, R, grid, n):
    """Odd latitude counts: the equator row is its own mirror (its G tile takes G_S := 0 in the
    fused grid stage) and the last 32-latitude P/G slices are partly padding; single states and
    batches against the numpy oracle's eval_nonlinear / eval_linear."""
    from paper_1904_05988_b200.cases import balanced_random_state
    plan = P.TransformPlan(R, grid[0], grid[1])
    ref = O.TransformPlan(R, grid[0], grid[1])
    p = P.ModelParams(phi_bar=9.80616 * 1e4, nu=1e5)
    po = O.ModelParams(phi_bar=p.phi_bar, nu=1e5)
    sts = np.stack([balanced_random_state(R, 30.0, 500 + s, phi_bar=p.phi_bar) for s in range(n)])
    fi, fe = (host(t) for t in P.imex_split(cuda(sts), p, plan))
    for i in range(n):
        assert rel_diff_fields(fe[i], O.eval_nonlinear(sts[i], po, ref)) < 1e-11
        assert rel_diff_fields(fi[i], O.eval_linear(R, sts[i], po)) < 1e-14


def test_empty_batches(P):
    """A batch of zero states / fields is a no-op (the reference's loops simply do not run): every
    operator returns an empty result without launching or failing."""
    R = 31
    plan = P.TransformPlan(R)
    p = P.ModelParams()
    K = P.num_coeffs(R)
    empty = torch.empty((0, 3, K), dtype=torch.complex128, device="cuda")
    fi, fe = P.imex_split(empty, p, plan)
    assert fi.shape == (0, 3, K) and fe.shape == (0, 3, K)
    assert P.eval_nonlinear(empty, p, plan).shape == (0, 3, K)
    assert P.eval_linear(R, empty, p).shape == (0, 3, K)
    assert P.solve_implicit(R, empty, 60.0, p).shape == (0, 3, K)
    g = plan.synthesise(torch.empty((0, K), dtype=torch.complex128, device="cuda"))
    assert g.shape[0] == 0
    assert plan.analyse(g).shape[0] == 0
    torch.cuda.synchronize()


def test_tile_padding_not_poisoned(P):
    """The forward G tiles are one buffer per plan, laid out per batch size: a
    NaN state evaluated in one layout must not leak into later evaluations / analyses in another
    through the padding latitude rows (T63 on 96 x 192: 48 latitude pairs, 16 padding rows per
    32-latitude slice set)."""
    from paper_1904_05988_b200.cases import balanced_random_state
    R = 63
    plan = P.TransformPlan(R, 96, 192)
    ref = O.TransformPlan(R, 96, 192)
    p = P.ModelParams(phi_bar=9.80616 * 1e4)
    po = O.ModelParams(phi_bar=p.phi_bar)
    good = np.stack([balanced_random_state(R, 20.0, 900 + s, phi_bar=p.phi_bar) for s in range(5)])
    bad = good.copy()
    bad[:, 1, 5] = np.nan
    P.imex_split(cuda(bad), p, plan)  # 5-state layout, NaN everywhere downstream
    P.imex_split(cuda(bad[:2]), p, plan)  # 2-state layout
    fe1 = host(P.eval_nonlinear(cuda(good[3]), p, plan))
    assert np.isfinite(fe1).all()
    assert rel_diff_fields(fe1, O.eval_nonlinear(good[3], po, ref)) < 1e-11
    x = fx.micro_bench_fields(R, 7, 3)
    g = ref.synthesise(x[0])
    gb = np.stack([ref.synthesise(f) for f in x])
    P.imex_split(cuda(bad), p, plan)
    back = host(plan.analyse(cuda(gb)))
    assert np.isfinite(back).all()
    assert np.abs(back[0] - ref.analyse(g)).max() < 1e-12 * np.abs(x[0]).max()
    fe5 = host(P.imex_split(cuda(good), p, plan)[1])
    for i in range(5):
        assert rel_diff_fields(fe5[i], O.eval_nonlinear(good[i], po, ref)) < 1e-11


def test_polar_skip_bit_identical(tmp_path):
    """The inverse contraction starts each (order, 32-latitude slice) at the first chunk whose P
    values reach 1e-20 (polar skip); the evaluations must give the same bits as without it
    (PSWE_NO_POLAR=1) at T63 ... T511 for batches of 1, 2, 3, 5 and 7 states."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ("0", "1"):
        out = tmp_path / f"ev{env}.npz"
        subprocess.run([sys.executable, os.path.join(root, "tools", "eval_dump.py"), str(out)], check=True,
                       env={**os.environ, "PSWE_NO_POLAR": env}, timeout=600)
        outs.append(np.load(out))
    for k in outs[0].files:
        np.testing.assert_array_equal(outs[0][k], outs[1][k])
