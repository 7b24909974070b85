"""A few SDC sweeps at T255 (256x512, 5 nodes) and T127 (3 nodes); node states and right-hand sides
to an npz - for bit-equality A/B of sweep-kernel variants (PSWE_NO_SWEEP_PREP=1 vs default).
Usage: python tools/sweep_dump.py out.npz"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05988_b200 as P  # noqa: E402
from paper_1904_05988_b200.cases import balanced_random_state  # noqa: E402

prm = P.ModelParams(phi_bar=9.80616e4, nu=1e5)
out = {}
for R, nlat, nlon, nn in ((255, 256, 512, 5), (127, 128, 256, 3), (63, 96, 192, 2)):
    lvl = P.Level(P.TransformPlan(R, nlat, nlon), prm, nn)
    lvl.spread(torch.as_tensor(balanced_random_state(R, 40.0, 11)).cuda())
    for _ in range(3):
        lvl.sweep(60.0)
    for m in range(nn):
        out[f"T{R}_state{m}"] = lvl.state(m).cpu().numpy()
torch.cuda.synchronize()
np.savez(sys.argv[1], **out)
print("ok", len(out))
