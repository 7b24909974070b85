"""A/B timing of the single-state evaluation chain and PFASST configs (tuning only; the bench is
the measurement of record). Usage: PSWE_LIB_VARIANT=x python tools/ab_time.py [configs, e.g. 3,4]"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1904_05988_b200 as P  # noqa: E402
from paper_1904_05988_b200 import _lib  # noqa: E402
from paper_1904_05988_b200.cases import balanced_random_state  # noqa: E402
from paper_1904_05988_b200.transform import _stream  # noqa: E402

configs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "3").split(",") if c]
L = _lib.lib()
prm = P.ModelParams(phi_bar=9.80616e4)
cp = prm.c()
out = {"variant": os.environ.get("PSWE_LIB_VARIANT", "default")}
for R, nlat, nlon in ((255, 256, 512), (511, 512, 1024)):
    plan = P.TransformPlan(R, nlat, nlon)
    plan.reserve(1)
    st = torch.as_tensor(balanced_random_state(R, 40.0, 7)[None]).cuda()
    fi, fe = torch.empty_like(st), torch.empty_like(st)

    def ev():
        _lib.check(L.pswe_eval_imex(plan.handle, ctypes.byref(cp), st.data_ptr(), fi.data_ptr(), fe.data_ptr(),
                                    1, _stream()))

    for _ in range(10):
        ev()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 200
    a.record()
    for _ in range(n):
        ev()
    b.record()
    torch.cuda.synchronize()
    out[f"seq_us_T{R}"] = round(a.elapsed_time(b) * 1e3 / n, 2)
    ms = (ctypes.c_float * 5)()
    ks = []
    for _ in range(50):
        _lib.check(L.pswe_eval_imex_kernel_times(plan.handle, ctypes.byref(cp), st.data_ptr(), fi.data_ptr(),
                                                 fe.data_ptr(), 1, _stream(), ms))
        ks.append(list(ms))
    out[f"stages_us_T{R}"] = dict(zip(("prep", "inverse", "fft", "forward", "tail"),
                                      (round(float(v) * 1e3, 1) for v in np.median(np.array(ks), axis=0))))
    # 5-state batch (the bench's step), L2 flushed before each timed call
    plan.reserve(5)
    st5 = torch.as_tensor(np.stack([balanced_random_state(R, 40.0, 7 + i) for i in range(5)])).cuda()
    fi5, fe5 = torch.empty_like(st5), torch.empty_like(st5)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    tt = []
    for it in range(25):
        flush.zero_()
        a.record()
        _lib.check(L.pswe_eval_imex(plan.handle, ctypes.byref(cp), st5.data_ptr(), fi5.data_ptr(), fe5.data_ptr(),
                                    5, _stream()))
        b.record()
        torch.cuda.synchronize()
        if it >= 5:
            tt.append(a.elapsed_time(b) * 1e3)
    out[f"batch5_us_T{R}"] = round(float(np.median(tt)), 1)
    ks = []
    for _ in range(30):
        _lib.check(L.pswe_eval_imex_kernel_times(plan.handle, ctypes.byref(cp), st5.data_ptr(), fi5.data_ptr(),
                                                 fe5.data_ptr(), 5, _stream(), ms))
        ks.append(list(ms))
    out[f"stages5_us_T{R}"] = dict(zip(("prep", "inverse", "fft", "forward", "tail"),
                                       (round(float(v) * 1e3, 1) for v in np.median(np.array(ks), axis=0))))
    del plan
# one fine SDC sweep (5 nodes: 4 single-state evaluations + node updates) and one coarse sweep
for R, nlat, nlon, nn in ((255, 256, 512, 5), (127, 128, 256, 3), (511, 512, 1024, 5), (255, 256, 512, 3)):
    lvl = P.Level(P.TransformPlan(R, nlat, nlon), prm, nn)
    lvl.spread(torch.as_tensor(balanced_random_state(R, 40.0, 3)).cuda())
    for _ in range(5):
        lvl.sweep(60.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        lvl.sweep(60.0)
    b.record()
    torch.cuda.synchronize()
    out[f"sweep_us_T{R}_{nn}"] = round(a.elapsed_time(b) * 1e3 / 50, 1)
dev = torch.device("cuda:0")
for c in configs:
    v = sorted(bench.run_pfasst(P, prm, 1, 0, dev, config=c)["wall_s_per_sim_day"] for _ in range(3))
    out[f"pf{c}_s_per_day"] = round(v[1], 3)  # median of 3 runs
    out[f"pf{c}_min"] = round(v[0], 3)
print(json.dumps(out))
