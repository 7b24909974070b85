"""Run pswe_eval_imex a few times for one (R, nlat, nlon, n) — a small target for ncu captures.
Usage: python tools/eval_once.py R nlat nlon n [reps]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05988_b200 as P  # noqa: E402
from paper_1904_05988_b200 import _lib  # noqa: E402
from paper_1904_05988_b200.cases import balanced_random_state  # noqa: E402
from paper_1904_05988_b200.transform import _stream  # noqa: E402

R, nlat, nlon, n = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 4
L = _lib.lib()
prm = P.ModelParams(phi_bar=9.80616e4)
cp = prm.c()
plan = P.TransformPlan(R, nlat, nlon)
plan.reserve(n)
st = torch.as_tensor(np.stack([balanced_random_state(R, 40.0, 7 + i) for i in range(n)])).cuda()
fi, fe = torch.empty_like(st), torch.empty_like(st)
for _ in range(reps):
    _lib.check(L.pswe_eval_imex(plan.handle, ctypes.byref(cp), st.data_ptr(), fi.data_ptr(), fe.data_ptr(), n,
                                _stream()))
torch.cuda.synchronize()
print("ok")
