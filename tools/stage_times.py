"""Per-kernel device times of one eval_imex call (CUDA events between the launches) for a few
truncations and batch sizes. Usage: python tools/stage_times.py [R:nlat:nlon ...] (nlat 0 = default
grid); with sizes given only those run, at batch 5 (STAGE_BATCHES=1,5 to change)."""
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
SIZES = ((63, 0, 0), (127, 0, 0), (255, 0, 0), (255, 256, 512), (511, 0, 0), (1023, 1024, 2048))
BATCHES = (1, 5)
if len(sys.argv) > 1:
    SIZES = [tuple(int(x) for x in a.split(':')) for a in sys.argv[1:]]
    BATCHES = tuple(int(b) for b in os.environ.get("STAGE_BATCHES", "5").split(","))
for R, nlat, nlon in SIZES:
    plan = P.TransformPlan(R, nlat, nlon, int(os.environ.get('LEGENDRE_MODE', '0')))
    for n in BATCHES:
        plan.reserve(n)
        st = torch.as_tensor(np.stack([balanced_random_state(R, 40.0, 7 + i) for i in range(n)])).cuda()
        fi, fe = torch.empty_like(st), torch.empty_like(st)
        ms = (ctypes.c_float * 4)()
        acc = np.zeros(4)
        for it in range(6):
            _lib.check(L.pswe_eval_imex_timed(plan.handle, ctypes.byref(cp), st.data_ptr(), fi.data_ptr(),
                                              fe.data_ptr(), n, _stream(), ms))
            if it >= 2:
                acc += np.array(list(ms))
        acc /= 4
        print(f"T{R} {plan.nlat}x{plan.nlon} n={n}: inv {acc[0]*1e3:7.1f}  fft {acc[1]*1e3:7.1f}  "
              f"fwd {acc[2]*1e3:7.1f}  tail {acc[3]*1e3:6.1f}  total {acc.sum()*1e3:7.1f} us  "
              f"({acc.sum()*1e3/n:6.1f} us/state)", flush=True)
