import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_05988_b200 as P
from paper_1904_05988_b200 import _lib
from paper_1904_05988_b200.cases import balanced_random_state
from paper_1904_05988_b200.transform import _stream
R, nlat, nlon, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
plan = P.TransformPlan(R, nlat, nlon); plan.reserve(n)
p = P.ModelParams(phi_bar=9.80616e4); cp = p.c()
st = torch.as_tensor(np.stack([balanced_random_state(R, 40.0, 7 + i) for i in range(n)])).cuda()
fi, fe = torch.empty_like(st), torch.empty_like(st)
for _ in range(3):
    _lib.check(_lib.lib().pswe_eval_imex(plan.handle, ctypes.byref(cp), st.data_ptr(), fi.data_ptr(), fe.data_ptr(), n, _stream()))
torch.cuda.synchronize(); print("ok")
