"""Which kernel generation each grid reaches (the dispatch is by grid, batch and plan mode; env
switches exist only for A/B measurements). Every test names the configuration that reaches a
path, asserts from the CUDA profiler's kernel list that the path actually ran, and checks the
result against the numpy oracle (oracle/pswe_oracle.py) - no kernel generation is dead code.

| path                                   | reached by                                          |
|----------------------------------------|-----------------------------------------------------|
| in-place fused grid stage (fft_ip.cu)  | nlon/2 in {24, 32, ..., 1536} (every BASELINE grid) |
| generic Stockham (fft.cu)              | other 5-smooth nlon/2, e.g. T24 on 26 x 50 (N = 25) |
| streamed-P DMMA Legendre, bulk-copy    | STREAM plans (default)                              |
|   ring (legendre_stream.cu)            |                                                     |
| recurrence DMMA Legendre               | RECOMPUTE plans (GpuImexOde)                        |
|   (legendre_mma.cu)                    |                                                     |
| DFMA recurrence inverse, P in registers| the single-state inverse from 256 latitude pairs    |
|   (legendre_rec.cu)                    | (T511 / T1023: configs 4 and 5; one degree segment  |
|                                        | per order from 512 pairs, two below)                |
| DFMA (CUDA-core) Legendre (legendre.cu)| PSWE_LEGENDRE_SIMT=1: the measured FP64-FMA         |
|                                        | alternative the north star compares DMMA against    |
"""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RUN = r"""
import sys, json
sys.path.insert(0, %r)
import numpy as np, torch
import paper_1904_05988_b200 as P
from oracle import pswe_oracle as O
from paper_1904_05988_b200.cases import balanced_random_state
R, nlat, nlon, n, mode = %d, %d, %d, %d, %d
plan = P.TransformPlan(R, nlat, nlon, mode)
p = P.ModelParams(phi_bar=9.80616e4)
st = np.stack([balanced_random_state(R, 40.0, 5 + i, phi_bar=p.phi_bar) for i in range(n)])
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    fe = P.imex_split(torch.as_tensor(st).cuda(), p, plan)[1].cpu().numpy()
names = sorted({e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA})
po = O.ModelParams(phi_bar=p.phi_bar)
op = O.TransformPlan(R, nlat, nlon)
err = 0.0
for i in (0, n - 1):
    want = O.eval_nonlinear(st[i], po, op)
    err = max(err, max(float(np.abs(fe[i][f] - want[f]).max() / np.abs(want[f]).max()) for f in range(3)))
print(json.dumps({"kernels": names, "err": err}))
"""


def run(R, nlat, nlon, n, mode=1, env=None):
    out = subprocess.run([sys.executable, "-c", RUN % (ROOT, R, nlat, nlon, n, mode)], capture_output=True, text=True,
                         env={**os.environ, **(env or {})}, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    import json
    return json.loads(out.stdout.strip().splitlines()[-1])


def has(names, sub):
    return any(sub in k for k in names)


def test_inplace_grid_stage_and_streamed_legendre():
    r = run(63, 96, 192, 2)
    assert has(r["kernels"], "fft_eval_ip_kernel") and has(r["kernels"], "leg_inv_tma_kernel")
    assert has(r["kernels"], "leg_fwd_gt_direct_kernel")  # one/two states, <= 64 latitude pairs
    assert r["err"] < 1e-11


def test_column_warp_forward():
    r = run(255, 256, 512, 5)
    assert has(r["kernels"], "leg_fwd_gt_cw_kernel<7"), r["kernels"]
    assert r["err"] < 1e-11
    r = run(255, 256, 512, 1)
    assert has(r["kernels"], "leg_fwd_gt_cw_kernel<2"), r["kernels"]
    assert r["err"] < 1e-11


def test_generic_stockham_grid():
    """N = nlon/2 = 25 has no in-place plan: the generic Stockham kernels of fft.cu run."""
    r = run(24, 26, 50, 3)
    assert has(r["kernels"], "fft_eval_kernel"), r["kernels"]
    assert not has(r["kernels"], "fft_eval_ip_kernel")
    assert r["err"] < 1e-11


def test_recompute_mode_legendre():
    r = run(31, 48, 96, 3, mode=0)
    assert has(r["kernels"], "leg_inv_mma_kernel") and has(r["kernels"], "leg_fwd_mma_kernel"), r["kernels"]
    assert r["err"] < 1e-11


def test_dfma_legendre_alternative():
    r = run(31, 48, 96, 3, mode=0, env={"PSWE_LEGENDRE_SIMT": "1"})
    assert has(r["kernels"], "leg_inv_kernel") and not has(r["kernels"], "mma_kernel"), r["kernels"]
    assert r["err"] < 1e-11


def test_register_recurrence_inverse_large_grid():
    """A single state on a grid of >= 256 latitude pairs takes the CUDA-core recurrence inverse
    (here T255 on 1024 x 512 and 512 x 512 - one and two degree segments - the oracle's cost kept
    small); a batch keeps the streamed DMMA one."""
    r = run(255, 1024, 512, 1)
    assert has(r["kernels"], "leg_inv_rec2_kernel") and not has(r["kernels"], "leg_inv_tma_kernel"), r["kernels"]
    assert r["err"] < 1e-11
    r = run(255, 1024, 512, 3)
    assert has(r["kernels"], "leg_inv_tma_kernel") and not has(r["kernels"], "leg_inv_rec2_kernel"), r["kernels"]
    assert r["err"] < 1e-11
    r = run(255, 512, 512, 1)
    assert has(r["kernels"], "leg_inv_rec2_kernel"), r["kernels"]
    assert r["err"] < 1e-11
