"""Evaluate saved states on the GPU (measurement aid): python tools/eval_state.py R nlat nlon in.npy out.npz
in.npy: (n, 3, K) or (3, K) complex states; out.npz: fe_batch, fe_single (F_E of eval_nonlinear)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05988_b200 as P  # noqa: E402

R, nlat, nlon = (int(a) for a in sys.argv[1:4])
st = np.load(sys.argv[4])
if st.ndim == 2:
    st = st[None]
p = P.ModelParams(phi_bar=9.80616e4)
plan = P.TransformPlan(R, nlat, nlon)
d = torch.as_tensor(st).cuda()
fe_b = P.imex_split(d, p, plan)[1].cpu().numpy()
fe_s = np.stack([P.eval_nonlinear(d[i], p, plan).cpu().numpy() for i in range(st.shape[0])])
np.savez(sys.argv[5], fe_batch=fe_b, fe_single=fe_s)
print("saved", sys.argv[5])
