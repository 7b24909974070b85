"""Dump PFASST block results (final state, residual rows) for bit-equality A/B checks between
settings (e.g. PSWE_PFASST_NO_ELIDE=1). Usage: python tools/pfasst_dump.py out.npz"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05988_b200 as P  # noqa: E402
from paper_1904_05988_b200.cases import balanced_random_state  # noqa: E402

prm = P.ModelParams(phi_bar=9.80616e4)
out = {}
for n_ts in (1, 2, 4):
    pair = P.TransferPair(P.Level(P.TransformPlan(31), prm, 5), P.Level(P.TransformPlan(15), prm, 3))
    pf = P.Pfasst(pair, P.BlockConfig(n_ts, 60.0, 3))
    fin, hist = P.run_blocks(pf, torch.as_tensor(balanced_random_state(31, 40.0, 3)).cuda(), 3)
    out[f"two_{n_ts}_final"], out[f"two_{n_ts}_res"] = fin.cpu().numpy(), hist
    pf.close()
    mid = P.Level(P.TransformPlan(21), prm, 3)
    pf3 = P.Pfasst(P.TransferPair(P.Level(P.TransformPlan(31), prm, 5), mid), P.BlockConfig(n_ts, 60.0, 3),
                   pair2=P.TransferPair(mid, P.Level(P.TransformPlan(15), prm, 2)))
    fin, hist = P.run_blocks(pf3, torch.as_tensor(balanced_random_state(31, 20.0, 4)).cuda(), 2)
    out[f"three_{n_ts}_final"], out[f"three_{n_ts}_res"] = fin.cpu().numpy(), hist
    pf3.close()
np.savez(sys.argv[1], **out)
print("dumped", len(out))
