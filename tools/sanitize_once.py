"""Small end-to-end run for compute-sanitizer (racecheck / memcheck / synccheck), one tool per call:
T31 (48 x 96) evaluation batches of 1 and 5 (TMA/mbarrier rings, PDL chain), the same on the
T24 26 x 50 grid (generic FFT), one 5-node sweep with the fused node update / X-tile emission,
the collocation residual (last-block reduction) and a two-level PFASST block of 2 steps (serial
emulation; eager and graph replay). Usage: compute-sanitizer --tool racecheck python tools/sanitize_once.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05988_b200 as P  # noqa: E402
from paper_1904_05988_b200.cases import balanced_random_state  # noqa: E402

p = P.ModelParams(phi_bar=9.80616e4)
for R, nlat, nlon in ((31, 48, 96), (24, 26, 50)):
    plan = P.TransformPlan(R, nlat, nlon)
    for n in (1, 5):
        st = torch.as_tensor(np.stack([balanced_random_state(R, 40.0, 3 + i) for i in range(n)])).cuda()
        P.imex_split(st, p, plan)
fine = P.Level(P.TransformPlan(31), p, 5)
coarse = P.Level(P.TransformPlan(15), p, 3)
th = torch.as_tensor(balanced_random_state(31, 40.0, 9)).cuda()
fine.spread(th)
fine.sweep(60.0)
res = torch.zeros(1, dtype=torch.float64, device="cuda")
fine.collocation_residual(60.0, res)
pf = P.Pfasst(P.TransferPair(fine, coarse), P.BlockConfig(2, 60.0, 2))
P.run_blocks(pf, th, 3)  # eager, capture, replay
torch.cuda.synchronize()
print("sanitize_once ok")
