"""The distributed PFASST executor with world = 2, as two processes on ONE B200 (the IPC
transport; the receiver waits on the host, so no GPU work of one process ever waits on the
other's). This runs the exact ring-slot, tag, event and shared-memory code of the multi-GPU path:

* two-level T31/T15, 3 blocks of n_ts = 2 (eager, segment-graph capture, graph replay): blocks 1-2
  equal the reference's (golden pf_nts2_*, oracle/_ref pf::run_block), and every block's final
  state, residual history, step finals and message log are BIT-identical to the serial emulation;
* three-level T31/T21/T15: bit-identical to the serial-emulation three-level run;
* a hung peer makes the other rank fail with the reference's "pipeline deadlock suspected"
  (pfasst.cpp:39-47) within the receive timeout;
* a skewed iteration tag makes the receiver fail with "message tag mismatch" (pfasst.cpp:71-76)
  and the sender learn of the failure (abort), instead of a silently wrong state."""
import os
import subprocess
import sys
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from _util import rel_diff_fields  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "dist_worker.py")


def res_ok(mine, refv, state):
    floor = 64 * 2.0**-52 * np.abs(state[0]).max()
    return bool(np.all(np.abs(np.asarray(mine) - np.asarray(refv)) <= 1e-6 * np.abs(refv) + floor))


def launch(tmp_path, levels=2, modes=("normal", "normal"), timeout=60.0, transport="ipc"):
    import paper_1904_05988_b200 as P
    uid = P.pfasst.unique_id(transport).hex()
    procs, outs = [], []
    t0 = time.time()
    for r, mode in enumerate(modes):
        out = tmp_path / f"rank{r}.npz"
        outs.append(out)
        procs.append(subprocess.Popen([sys.executable, WORKER, str(r), str(len(modes)), transport, uid, str(out),
                                       str(levels), mode, str(timeout)]))
    for p in procs:
        p.wait(timeout=600)
    wall = time.time() - t0
    return [dict(np.load(o, allow_pickle=False)) for o in outs], wall


def serial(levels):
    import paper_1904_05988_b200 as P
    prm = P.ModelParams(phi_bar=9.80616 * 10000.0)
    g = np.load(os.path.join(ROOT, "tests", "golden", "golden_ref.npz"))
    if levels == 2:
        pair = P.TransferPair(P.Level(P.TransformPlan(31), prm, 5), P.Level(P.TransformPlan(15), prm, 3))
        pair2 = None
        th = torch.as_tensor(g["pf_theta0"]).cuda()
    else:
        from paper_1904_05988_b200.cases import balanced_random_state
        mid = P.Level(P.TransformPlan(21), prm, 3)
        pair = P.TransferPair(P.Level(P.TransformPlan(31), prm, 5), mid)
        pair2 = P.TransferPair(mid, P.Level(P.TransformPlan(15), prm, 2))
        th = torch.as_tensor(balanced_random_state(31, 20.0, 4, phi_bar=prm.phi_bar)).cuda()
    pf = P.Pfasst(pair, P.BlockConfig(2, 60.0, 3), pair2=pair2)
    s, hist, steps = th.clone(), [], []
    for _ in range(3):
        fin, res, st = pf.run_block(s, step_finals=True)
        s.copy_(fin)
        hist.append(res)
        steps.append(st.cpu().numpy())
    msgs = pf.messages()
    pf.close()
    return s.cpu().numpy(), np.array(hist), np.array(steps), msgs


@pytest.mark.parametrize("levels", [2, 3])
def test_world2_ipc_matches_serial_and_reference(tmp_path, golden, levels):
    res, _ = launch(tmp_path, levels)
    for r in res:
        assert "error" not in r, str(r.get("error")) + str(r.get("tb"))
    fin_s, hist_s, steps_s, msgs_s = serial(levels)
    for r in res:  # every rank holds the block's final state, all residual rows and step finals
        np.testing.assert_array_equal(r["final"], fin_s)
        np.testing.assert_array_equal(r["res"], hist_s)
        np.testing.assert_array_equal(r["steps"], steps_s)
        assert sorted(tuple(int(v) for v in m) for m in r["messages"]) == \
            sorted((m[0], m[1], ord(m[2]), m[3], m[4], m[5], m[6]) for m in msgs_s)
    if levels == 2:  # blocks 1-2 are the reference's golden two-block run
        assert rel_diff_fields(res[0]["final2"], golden["pf_nts2_final"]) < 1e-10
        assert res_ok(res[0]["res"][:2], golden["pf_nts2_res"], res[0]["final2"])
        ref_log = sorted(tuple(int(v) for v in m) for m in golden["pf_nts2_msgs"])
        assert sorted(tuple(int(v) for v in m) for m in res[1]["messages"]) == ref_log


def test_world2_hung_peer_times_out(tmp_path):
    res, wall = launch(tmp_path, 2, modes=("normal", "hang"), timeout=5.0)
    assert "deadlock suspected" in str(res[0]["error"]), res[0]
    assert wall < 60


def test_world2_tag_skew_detected(tmp_path):
    res, _ = launch(tmp_path, 2, modes=("skew", "normal"), timeout=20.0)
    assert "message tag mismatch" in str(res[1]["error"]), res[1]
    # the sender learns of the failure through the abort flag (or had already finished the block)
    assert "error" not in res[0] or "failed" in str(res[0]["error"]), res[0]
