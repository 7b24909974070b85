"""Config-2 transform round trip (15 fields T255 256x512: synthesise + analyse) a few times: a small
ncu target and a quick timer. Usage: python tools/transform_once.py [reps] [fields]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05988_b200 as P  # noqa: E402
from paper_1904_05988_b200 import _lib  # noqa: E402
from paper_1904_05988_b200.transform import _stream  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
nf = int(sys.argv[2]) if len(sys.argv) > 2 else 15
L = _lib.lib()
plan = P.TransformPlan(255, 256, 512)
plan.reserve(3)
rng = np.random.default_rng(2)
K = P.num_coeffs(255)
x = torch.as_tensor(rng.uniform(-1, 1, (nf, K)) + 1j * rng.uniform(-1, 1, (nf, K))).cuda()
g = torch.empty((nf, 256, 512), dtype=torch.float64, device="cuda")
xb = torch.empty_like(x)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
ts = {"syn": [], "ana": []}
for it in range(reps):
    flush.zero_()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    _lib.check(L.pswe_synthesise(plan.handle, x.data_ptr(), g.data_ptr(), nf, _stream()))
    e[1].record()
    _lib.check(L.pswe_analyse(plan.handle, g.data_ptr(), xb.data_ptr(), nf, _stream()))
    e[2].record()
    torch.cuda.synchronize()
    if it >= reps // 2:
        ts["syn"].append(e[0].elapsed_time(e[1]) * 1e3)
        ts["ana"].append(e[1].elapsed_time(e[2]) * 1e3)
print({k: round(float(np.median(v)), 1) for k, v in ts.items()})
