"""One PFASST time rank as its own process (used by tests/test_gpu_pfasst_dist.py; not a test
module). All ranks may share one GPU with the IPC transport.

python tests/dist_worker.py RANK WORLD TRANSPORT UID_HEX OUT.npz LEVELS MODE TIMEOUT
  LEVELS 2: T31/T15 (5/3 nodes), the golden pf_nts2 case (dt 60 s, 3 iterations), 3 blocks (the
            first two are the golden case; eager, segment-graph capture, replay);
  LEVELS 3: T31/T21/T15 (5/3/2 nodes), 3 blocks;
  MODE normal | hang (this rank never runs a block) | skew (this rank's first iteration message
  carries the wrong iteration tag, PSWE_PFASST_FAULT=1).
Writes final / residual history / step finals, or the error text."""
import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank, world, transport, uid_hex, out, levels, mode, timeout = sys.argv[1:9]
    rank, world, levels, timeout = int(rank), int(world), int(levels), float(timeout)
    if mode == "skew":
        os.environ["PSWE_PFASST_FAULT"] = "1"
    import torch

    import paper_1904_05988_b200 as P
    torch.cuda.set_device(0)
    prm = P.ModelParams(phi_bar=9.80616 * 10000.0)
    g = np.load(os.path.join(ROOT, "tests", "golden", "golden_ref.npz"))
    try:
        if levels == 2:
            fine = P.Level(P.TransformPlan(31), prm, 5)
            coarse = P.Level(P.TransformPlan(15), prm, 3)
            pair, pair2 = P.TransferPair(fine, coarse), None
            th = torch.as_tensor(g["pf_theta0"]).cuda()
        else:
            from paper_1904_05988_b200.cases import balanced_random_state
            fine = P.Level(P.TransformPlan(31), prm, 5)
            mid = P.Level(P.TransformPlan(21), prm, 3)
            coarse = P.Level(P.TransformPlan(15), prm, 2)
            pair, pair2 = P.TransferPair(fine, mid), P.TransferPair(mid, coarse)
            th = torch.as_tensor(balanced_random_state(31, 20.0, 4, phi_bar=prm.phi_bar)).cuda()
        pf = P.Pfasst(pair, P.BlockConfig(world, 60.0, 3), rank=rank, world=world, pair2=pair2,
                      transport=transport, uid=bytes.fromhex(uid_hex), recv_timeout=timeout)
        if mode == "hang":
            time.sleep(timeout * 3)
            np.savez(out, error="hung on purpose")
            return
        s = th.clone()
        hist, steps = [], []
        t0 = time.time()
        final2 = None
        for b in range(3):  # eager block, segment-graph capture block, replay block
            fin, res, st = pf.run_block(s, step_finals=True)
            s.copy_(fin)
            hist.append(res)
            steps.append(st.cpu().numpy())
            if b == 1:
                final2 = s.cpu().numpy()
        np.savez(out, final=s.cpu().numpy(), final2=final2, res=np.array(hist), steps=np.array(steps),
                 wall=time.time() - t0,
                 messages=np.array([[m[0], m[1], ord(m[2]), m[3], m[4], m[5], m[6]] for m in pf.messages()]))
        pf.close()
    except Exception as e:  # reported to the parent test
        np.savez(out, error=f"{type(e).__name__}: {e}", tb=traceback.format_exc())


if __name__ == "__main__":
    main()
