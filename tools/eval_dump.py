"""Dump eval_imex outputs for a few (R, grid, n) to an .npz (A/B bit-equality checks between builds).
Usage: PSWE_LIB_VARIANT=x python tools/eval_dump.py out.npz"""
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

L = _lib.lib()
prm = P.ModelParams(phi_bar=9.80616e4)
cp = prm.c()
out = {}
SIZES = ((63, 96, 192), (127, 128, 256), (255, 256, 512), (511, 512, 1024), (21, 45, 96))
if os.environ.get("EVAL_DUMP_LARGE"):
    SIZES = ((511, 512, 1024), (511, 768, 1536), (1023, 1024, 2048))
for R, nlat, nlon in SIZES:
    plan = P.TransformPlan(R, nlat, nlon)
    for n in (1, 2, 3, 5, 7):
        st = torch.as_tensor(np.stack([balanced_random_state(R, 40.0, 11 + i) for i in range(n)])).cuda()
        fi, fe = torch.empty_like(st), torch.empty_like(st)
        _lib.check(L.pswe_eval_imex(plan.handle, ctypes.byref(cp), st.data_ptr(), fi.data_ptr(), fe.data_ptr(), n,
                                    _stream()))
        torch.cuda.synchronize()
        out[f"T{R}_{nlat}_n{n}_fi"] = fi.cpu().numpy()
        out[f"T{R}_{nlat}_n{n}_fe"] = fe.cpu().numpy()
np.savez(sys.argv[1], **out)
print("dumped", len(out))
