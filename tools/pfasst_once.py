"""One config-3 PFASST block at n_ts = 1 (T255 256x512 / T127 128x256): a small ncu target.
Usage: python tools/pfasst_once.py [config]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05988_b200 as P  # noqa: E402
from paper_1904_05988_b200.cases import config_state  # noqa: E402

os.environ.setdefault("PSWE_NO_GRAPH", "1")  # eager launches so every kernel is visible
prm = P.ModelParams(phi_bar=9.80616e4)
fp, cp = P.TransformPlan(255, 256, 512), P.TransformPlan(127, 128, 256)
pair = P.TransferPair(P.Level(fp, prm, 5), P.Level(cp, prm, 3))
pf = P.Pfasst(pair, P.BlockConfig(1, 60.0, 4))
th = torch.as_tensor(config_state(3, fp)).cuda()
P.run_blocks(pf, th, 2)
torch.cuda.synchronize()
print("ok")
