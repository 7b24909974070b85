"""Single-state evaluation chain (the SDC-sweep pattern): eager launches from Python vs the same
chain captured once into a CUDA graph (as the PFASST controller replays its blocks) - separates the
device time of the chain from host launch overhead. Usage: python tools/seq_graph.py [R nlat nlon]"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05988_b200 as P  # noqa: E402
from paper_1904_05988_b200 import _lib  # noqa: E402
from paper_1904_05988_b200.cases import balanced_random_state  # noqa: E402

R, nlat, nlon = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (255, 256, 512)
L = _lib.lib()
prm = P.ModelParams(phi_bar=9.80616e4)
cp = prm.c()
plan = P.TransformPlan(R, nlat, nlon)
plan.reserve(1)
st = torch.as_tensor(balanced_random_state(R, 40.0, 7)[None]).cuda()
fi, fe = torch.empty_like(st), torch.empty_like(st)
s = torch.cuda.Stream()


def chain(k):
    for _ in range(k):
        _lib.check(L.pswe_eval_imex(plan.handle, ctypes.byref(cp), st.data_ptr(), fi.data_ptr(), fe.data_ptr(), 1,
                                    ctypes.c_void_p(s.cuda_stream)))


out = {"R": R}
with torch.cuda.stream(s):
    chain(20)
torch.cuda.synchronize()
n = 200
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
chain(n)
b.record(s)
torch.cuda.synchronize()
out["eager_us_per_eval"] = round(a.elapsed_time(b) * 1e3 / n, 2)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    chain(20)
with torch.cuda.stream(s):
    g.replay()
torch.cuda.synchronize()
a.record(s)
with torch.cuda.stream(s):
    for _ in range(10):
        g.replay()
b.record(s)
torch.cuda.synchronize()
out["graph_us_per_eval"] = round(a.elapsed_time(b) * 1e3 / 200, 2)
print(json.dumps(out))
