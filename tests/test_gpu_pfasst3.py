"""Three-level PFASST (BASELINE configs[3]) and the multi-level FAS of Eq. 19.

The reference implements two levels only (multilevel.hpp:29-35), so there is no reference run to
pin against ("parity is unpinned; use degenerate-level checks"). The checks are the
fixed-point properties that define the method:

* FAS chain: at the fine collocation solution, the restricted state is a fixed point of the mid
  sweep with tau_mid, and (only with the R tau_mid term of Eq. 19) of the coarse sweep with
  tau_c = fas(mid, coarse) + R tau_mid;
* PFASST converges to the fine collocation solution of its time steps: for n_ts = 1, 2, 4 the
  three-level block ends on the state of n_ts serial fine SDC steps iterated to convergence (from
  the coarsest level's truncation of theta0: like the reference's two-level predictor,
  pfasst.cpp:112, worker 0's fine node 0 is interpolated from the coarse spread and never
  received), with residuals at round-off;
* the message log has one mid-level message per (iteration < N, worker < n-1)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from _util import rel_diff_fields  # noqa: E402

PHI_BAR = 9.80616 * 10000.0
DT = 60.0


@pytest.fixture(scope="module")
def P():
    import paper_1904_05988_b200 as P
    return P


def host(t):
    return t.detach().cpu().numpy()


def _chain(P, Rf=31, Rm=21, Rc=15):
    prm = P.ModelParams(phi_bar=PHI_BAR)
    fine = P.Level(P.TransformPlan(Rf), prm, 5)
    mid = P.Level(P.TransformPlan(Rm), prm, 3)
    coarse = P.Level(P.TransformPlan(Rc), prm, 2)
    return fine, mid, coarse, P.TransferPair(fine, mid), P.TransferPair(mid, coarse)


def _theta0(P, R=31):
    from paper_1904_05988_b200.cases import balanced_random_state
    return torch.as_tensor(balanced_random_state(R, 20.0, 4, phi_bar=PHI_BAR)).cuda()


def _max_change(before, after):
    """max over the 3 fields of max|change| / max|field| (states: nodes x 3 x K)"""
    d = (after - before).abs().amax(dim=(0, 2))
    return float((d / before.abs().amax(dim=(0, 2))).max())


def test_fas_chain_fixed_point(P):
    fine, mid, coarse, p1, p2 = _chain(P)
    res = torch.zeros(1, dtype=torch.float64, device="cuda")
    fine.sdc_step(_theta0(P), DT, 40, res)  # fine collocation solution
    assert float(res.item()) < 1e-9 * float(fine.states().abs().max())
    p1.restrict_states()
    mid.refresh_nodes(0)
    tau_m = p1.fas_correction(DT).clone()
    before = mid.states().clone()
    mid.sweep(DT, tau_m)
    assert _max_change(before, mid.states()) < 1e-12
    # coarse level below a level that carries its own tau: Eq. 19 with tau_f != 0
    p2.restrict_states()
    coarse.refresh_nodes(0)
    before = coarse.states().clone()
    tau_c = p2.fas_correction(DT, tau_m).clone()
    coarse.sweep(DT, tau_c)
    assert _max_change(before, coarse.states()) < 1e-12
    # negative control: without R tau_mid the restricted state is not a fixed point
    coarse.states().copy_(before)
    coarse.refresh_nodes(0)
    tau_plain = p2.fas_correction(DT).clone()
    coarse.sweep(DT, tau_plain)
    assert _max_change(before, coarse.states()) > 1e-9


@pytest.mark.parametrize("n_ts", [1, 2, 4])
def test_pfasst3_converges_to_fine_collocation(P, n_ts):
    fine, mid, coarse, p1, p2 = _chain(P)
    th0 = _theta0(P)
    # reference: n_ts serial fine SDC steps, each iterated to the collocation solution, from the
    # initial state as the predictor leaves it on worker 0 (truncated to the coarsest level)
    th_t = P.interpolate_space(P.restrict_space(th0, 31, 15), 15, 31)
    sref = P.Level(P.TransformPlan(31), P.ModelParams(phi_bar=PHI_BAR), 5)
    ref, _ = P.sdc_run(sref, th_t, DT, 40, n_ts)
    ref = host(ref)
    n_iter = 12 + 3 * n_ts
    pf = P.Pfasst(p1, P.BlockConfig(n_ts, DT, n_iter), pair2=p2)
    assert pf.n_levels == 3
    fin, res = pf.run_block(th0)
    fin = host(fin)
    assert rel_diff_fields(fin, ref) < 1e-10
    scale = np.abs(fin[0]).max()
    for w in range(n_ts):
        r = res[w]
        assert r[-1] < 1e-15 * scale
        assert r[-1] < 1e-8 * r[1]  # converged, not stalled


def test_pfasst3_message_log(P):
    fine, mid, coarse, p1, p2 = _chain(P)
    n, N = 4, 3
    pf = P.Pfasst(p1, P.BlockConfig(n, DT, N), pair2=p2)
    pf.run_block(_theta0(P))
    log = pf.messages()
    mid_msgs = [m for m in log if m[5] == 1]
    assert len(mid_msgs) == (N - 1) * (n - 1)
    assert all(m[2] == "M" and m[6] == mid.num_nodes() - 1 and m[4] == m[3] + 1 for m in mid_msgs)
    coarse_msgs = [m for m in log if m[5] == 2]
    assert len(coarse_msgs) == n * (n - 1) // 2 + (N - 1) * (n - 1)
    assert all(m[6] == coarse.num_nodes() - 1 for m in coarse_msgs)


def test_pfasst3_rejects_broken_chain(P):
    fine, mid, coarse, p1, p2 = _chain(P)
    with pytest.raises(Exception):
        P.Pfasst(p2, P.BlockConfig(1, DT, 2), pair2=p1)  # (mid, coarse) then (fine, mid)


@pytest.mark.parametrize("n_ts,n_blocks", [(1, 1), (2, 2), (4, 1)])
def test_degenerate_chain_reproduces_two_level_reference(P, golden, n_ts, n_blocks):
    """Pin of the three-level controller to the reference (multilevel.hpp:29-35):
    a chain whose mid level IS the fine level (same plan, 5 nodes: identity transfers, tau_mid = 0)
    with no mid sweeps and the reference's node-0 form (pfasst.cpp:171-174, generalised to the chain)
    runs the two-level algorithm through every three-level op (mid restriction / FAS / refresh /
    message / increments). It must reproduce the reference's two-level pf::run_block (golden
    pf_nts*, T31/T15, 5/3 nodes, dt 60 s, 3 iterations) to 1e-10 with its residual history."""
    from oracle import fixtures as fx  # noqa: F401
    prm = P.ModelParams(phi_bar=PHI_BAR)
    plan31, plan15 = P.TransformPlan(31), P.TransformPlan(15)
    fine, mid, coarse = P.Level(plan31, prm, 5), P.Level(plan31, prm, 5), P.Level(plan15, prm, 3)
    pf = P.Pfasst(P.TransferPair(fine, mid), P.BlockConfig(n_ts, 60.0, 3), pair2=P.TransferPair(mid, coarse))
    pf.configure3("reference", mid_sweeps=0)
    fin, hist = P.run_blocks(pf, torch.as_tensor(golden["pf_theta0"]).cuda(), n_blocks)
    fin = host(fin)
    assert rel_diff_fields(fin, golden[f"pf_nts{n_ts}_final"]) < 1e-10
    floor = 64 * 2.0**-52 * np.abs(fin[0]).max()
    ref = golden[f"pf_nts{n_ts}_res"]
    assert np.all(np.abs(hist - ref) <= 1e-6 * np.abs(ref) + floor), (hist, ref)
    # the same chain with the low-mode node-0 form is a different (non-reference) iteration
    pf.configure3("lowmode", mid_sweeps=0)
    fin2, _ = P.run_blocks(pf, torch.as_tensor(golden["pf_theta0"]).cuda(), n_blocks)
    if n_ts > 1:
        assert rel_diff_fields(host(fin2), golden[f"pf_nts{n_ts}_final"]) > 1e-10


@pytest.mark.parametrize("n_ts", [1, 4])
def test_reference_node0_form_fixed_point(P, n_ts):
    """Why the three-level default is the low-mode form: the reference's additive node-0 rule
    (pfasst.cpp:171-174) adds the interpolated coarse increment to an IC that is already new, so
    for n_ts >= 2 its iteration does not settle on the serial fine collocation solution - in the
    reference's own two-level algorithm (our two-level controller, pinned to pf::run_block above)
    and in the chain alike. n_ts = 1 (no IC messages) converges with either form."""
    fine, mid, coarse, p1, p2 = _chain(P)
    th0 = _theta0(P)
    th_t = P.interpolate_space(P.restrict_space(th0, 31, 15), 15, 31)
    sref = P.Level(P.TransformPlan(31), P.ModelParams(phi_bar=PHI_BAR), 5)
    ref, _ = P.sdc_run(sref, th_t, DT, 40, n_ts)
    ref = host(ref)
    n_iter = 12 + 3 * n_ts
    pf3 = P.Pfasst(p1, P.BlockConfig(n_ts, DT, n_iter), pair2=p2)
    pf3.configure3("reference", mid_sweeps=1)
    fin3 = host(pf3.run_block(th0)[0])
    prm = P.ModelParams(phi_bar=PHI_BAR)
    two = P.Pfasst(P.TransferPair(P.Level(P.TransformPlan(31), prm, 5), P.Level(P.TransformPlan(15), prm, 3)),
                   P.BlockConfig(n_ts, DT, n_iter))
    fin2 = host(two.run_block(th0)[0])
    for fin in (fin3, fin2):
        assert np.all(np.isfinite(fin))
        if n_ts == 1:
            assert rel_diff_fields(fin, ref) < 1e-10
        else:
            assert rel_diff_fields(fin, ref) > 1e-6
