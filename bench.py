#!/usr/bin/env python
"""Benchmark of the PFASST-SH hot path on B200.

Headline metric (BASELINE.json): SWE RHS evals/s (fp64 SH fwd+inv) at T255.
  step  = one explicit+implicit right-hand-side evaluation (eval_nonlinear + eval_linear,
          swe.cpp:9-69) of B = 5 T255 states (the 5 fine SDC nodes of config 3; refresh of all
          nodes after prediction/restriction) on BASELINE's T255 grid 256 x 512 (configs[1] and
          the fine level of configs[2]); the reference's dealiased grid 384 x 768 is reported
          beside it (dealiased_grid).
  value = evals/s over the whole job (all ranks; each rank evaluates its own states: weak).
  L2    = flushed (256 MiB write) between timed steps, outside the event-timed span.
Side results on the same JSON line:
  e2e            same metric through the public C ABI (pswe_eval_imex) with pinned HOST buffers,
                 every step's H2D + D2H inside the timed region (double-buffered on copy streams);
  roofline       dominant (longest) kernel's algorithmic work / its event-timed duration: FP64
                 flops vs the FP64 DMMA peak measured in-run for the two Legendre contractions
                 (MEASURED_PEAKS.json has no FP64 figure), bytes vs MEASURED_PEAKS.json hbm_gbs
                 for the coefficient prep, the grid stage and the tail; all five kernels are
                 listed under roofline.kernels;
  cpu_baseline   the reference (oracle/_ref, compiled from /root/reference) timed on the host
                 cores, rank 0 at N=1 only;
  pfasst         config-3 PFASST block (T255 256x512 / T127 128x256, 5/3 nodes, dt 60 s, 8 steps, 4 its),
                 n_ts = N time ranks (NCCL) — wall s per simulated day; pfasst_configs adds
                 config 4 (three-level T511/T255/T127) and config 5 (T1023/T511);
  transform      config-2 micro-bench: 15-field round trip at T255 on 256 x 512.
--impl reference times the reference's CPU path (oracle/_ref) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SWE RHS evals/s (fp64 SH fwd+inv) at T255"
R_BENCH, NLAT, NLON, BATCH = 255, 256, 512, 5
NLAT_DEALIASED, NLON_DEALIASED = 384, 768


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-pfasst", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sizes", action="store_true", help="skip the T511/T1023 Legendre roofline lines")
    ap.add_argument("--legendre", type=int, default=1, help="0 recompute, 1 stream (default, measured faster)")
    ap.add_argument("--ref-worker", default=None, help=argparse.SUPPRESS)
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def bench_states(R=R_BENCH, n=BATCH, seed=20261019):
    from paper_1904_05988_b200.cases import balanced_random_state
    return np.stack([balanced_random_state(R, 40.0, seed + i) for i in range(n)])


# ----------------------------------------------------------------------------------------------
# reference arm / CPU baseline (oracle/_ref = the reference C++ compiled from its own sources)


# the workload both arms print (identical dicts: the driver compares them)
CONFIG = {"workload": f"rhs_eval T{R_BENCH} {NLAT}x{NLON} x{BATCH} states", "R": R_BENCH, "nlat": NLAT,
          "nlon": NLON, "batch_states": BATCH}


def use_all_host_cores(ref):
    """The reference's OpenMP team on every core this process may run on (torchrun exports
    OMP_NUM_THREADS=1 to its workers; the reference arm must use all host threads it can)."""
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    ref.lib().ref_set_threads(n)


REF_WARM_S = 6.0
# The reference's OpenMP team runs with active waiting and bound threads (its best standard setting
# on this box: on 8 / 16 host cores +15-25% over the default; measured), in a subprocess of its own
# that never imports torch (torch's OpenMP pool would compete for the bound cores), so the arm
# (--impl reference) and the cpu_baseline legs time the same code under the same conditions.
REF_OMP_ENV = {"OMP_WAIT_POLICY": "active", "OMP_PROC_BIND": "true"}


def _ref_steps(states, steps: int, warmup: int, budget_s: float | None):
    from oracle import ref_lib as ref
    from oracle.pswe_oracle import ModelParams
    use_all_host_cores(ref)
    plan = ref.RefPlan(R_BENCH, NLAT, NLON)
    p = ModelParams(phi_bar=9.80616 * 1e4)
    cores = ref.lib().ref_max_threads()

    def step():
        for st in states:
            plan.time_eval(st, p, 1)

    # warm-up: the requested steps, and at least REF_WARM_S seconds (first touch of the plan's
    # tables, the OpenMP team, clocks)
    w0 = time.perf_counter()
    k = 0
    while k < warmup or time.perf_counter() - w0 < REF_WARM_S:
        step()
        k += 1
    times, t_start = [], time.perf_counter()
    while len(times) < steps:
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
        if budget_s is not None and time.perf_counter() - t_start >= budget_s:
            break
    return times, cores


def _ref_pfasst(n_ts: int, th, config: int):
    from oracle import ref_lib as ref
    from oracle.pswe_oracle import ModelParams
    lv, dt, _, n_iter = PF_CONFIGS[config]
    (Rf, nf_lat, nf_lon, nn_f), (Rc, nc_lat, nc_lon, nn_c) = lv
    p = ModelParams(phi_bar=9.80616 * 1e4)
    use_all_host_cores(ref)
    r = ref.pfasst_run(Rf, (nf_lat, nf_lon), Rc, (nc_lat, nc_lon), p, nn_f, nn_c, n_ts, dt, n_iter, 1, th,
                       serial=(n_ts == 1))
    cores = ref.lib().ref_max_threads()
    return {"config": config, "n_ts": n_ts, "wall_s_per_sim_day": r.wall / (n_ts * dt) * 86400,
            "wall_s": r.wall, "blocks": 1, "cores": cores if n_ts == 1 else n_ts, "kind": "reference",
            "mode": "serial emulation, OpenMP" if n_ts == 1 else "threaded (one core per worker)",
            "omp": dict(REF_OMP_ENV),
            "sample": f"one block of {n_ts} step(s), {n_iter} iterations (oracle/_ref pf::run_block)"}


def ref_worker_main(spec_json: str):
    """bench.py --ref-worker SPEC: one reference measurement in a clean process (no torch)."""
    spec = json.loads(spec_json)
    if spec["kind"] == "steps":
        times, cores = _ref_steps(np.load(spec["states"]), spec["steps"], spec["warmup"], spec.get("budget"))
        print(json.dumps({"times": times, "cores": cores}))
    else:
        print(json.dumps(_ref_pfasst(spec["n_ts"], np.load(spec["theta"]), spec["config"])))


def _run_ref_worker(spec: dict, arrays: dict):
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        for name, arr in arrays.items():
            path = os.path.join(d, name + ".npy")
            np.save(path, arr)
            spec[name] = path
        env = dict(os.environ)
        for k, v in REF_OMP_ENV.items():
            env.setdefault(k, v)
        out = subprocess.run([sys.executable, os.path.abspath(__file__), "--ref-worker", json.dumps(spec)], env=env,
                             capture_output=True, text=True, timeout=1800)
        if out.returncode != 0:
            raise RuntimeError(f"reference worker failed: {out.stderr[-500:]}")
        return json.loads(out.stdout.strip().splitlines()[-1])


def reference_step_times(steps: int, warmup: int, budget_s: float | None = None):
    """The reference's eval_nonlinear + eval_linear (oracle/_ref, swe.cpp:9-69) on bench.py's step:
    the 5 bench_states at T255 256x512, one state after the other, OpenMP on every host core
    (REF_OMP_ENV, its own process). Returns (per-step wall times, cores). With budget_s the run
    stops once that much time is spent (at least one timed step) - the cpu_baseline leg's bounded
    sample; the reference arm times exactly `steps`. Both legs time the same thing the same way."""
    r = _run_ref_worker({"kind": "steps", "steps": steps, "warmup": warmup, "budget": budget_s},
                        {"states": bench_states()})
    return r["times"], r["cores"]


def reference_pfasst(n_ts: int, theta0=None, config: int = 3):
    """The reference's own pf::run_block (oracle/_ref, pfasst.cpp:194-251) on a BASELINE PFASST
    config at n_ts time steps per block, ONE block timed (its steady_clock around run_block):
    serial emulation with OpenMP on every host core at n_ts = 1, the reference's threaded mode
    (one core per worker, pfasst.cpp:224) beyond — SURVEY §8d(4). Wall s per simulated day =
    wall / (n_ts dt) * 86400. Two-level configs only (config 5's T1023 plan needs ~13 GB of host
    memory and minutes per block; config 4 has no reference implementation)."""
    if theta0 is None:
        from paper_1904_05988_b200.cases import config_state
        theta0 = config_state(config)
    return _run_ref_worker({"kind": "pfasst", "n_ts": n_ts, "config": config}, {"theta": np.asarray(theta0)})


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import ref_lib as ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libpintswe_ref.so not built"}))
        return
    times, cores = reference_step_times(args.steps, args.warmup)
    total = sum(times)
    value = BATCH * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded balanced n^-3 random states, 40 m/s rms)",
        "config": dict(CONFIG),
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} steps x {BATCH} evals, reference eval_nonlinear+eval_linear "
                                   f"(OpenMP {cores} threads, active wait, bound; own process; "
                                   f"FFTW-API shim)"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_pfasst:
        try:  # the metric's second half: PFASST-SH wall s per simulated day (IC without the bump:
            # the reference arm never touches the GPU; run time does not depend on the values)
            line["pfasst"] = reference_pfasst(world)
        except Exception as e:
            line["pfasst"] = {"error": f"{type(e).__name__}: {e}"}
    print(json.dumps(line))


# ----------------------------------------------------------------------------------------------
# clocks sampler


class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(dev)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
                pw.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        busy = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(pw) if pw else None}


# ----------------------------------------------------------------------------------------------
# our arm


def max_over_ranks(v: float, dev) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cpu" if dist.get_backend() == "gloo" else dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args):
    import ctypes

    import torch
    import torch.distributed as dist

    import paper_1904_05988_b200 as P
    from paper_1904_05988_b200 import _lib
    from paper_1904_05988_b200.transform import _stream

    rank, world, local = dist_env()
    # PSWE_BENCH_SHARED_GPU=1: every rank on cuda:0 with a gloo process group - a functional dry run
    # of the N > 1 code path (transport set-up, PFASST ranks, max-over-ranks) on a one-GPU box; its
    # timings are not scaling numbers (the ranks share one GPU)
    shared = os.environ.get("PSWE_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    L = _lib.lib()

    prm = P.ModelParams(phi_bar=9.80616 * 1e4)
    cprm = prm.c()
    plan = P.TransformPlan(R_BENCH, NLAT, NLON, args.legendre)
    plan.reserve(BATCH)
    states = torch.as_tensor(bench_states()).to(dev)
    fi = torch.empty_like(states)
    fe = torch.empty_like(states)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    def step():
        _lib.check(L.pswe_eval_imex(plan.handle, ctypes.byref(cprm), states.data_ptr(), fi.data_ptr(),
                                    fe.data_ptr(), BATCH, _stream()))

    clocks = Clocks(local)
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for k in range(args.steps):
        flush.zero_()
        ev0[k].record()
        step()
        ev1[k].record()
    torch.cuda.synchronize()
    total_ms = sum(a.elapsed_time(b) for a, b in zip(ev0, ev1))
    if world > 1:
        total_ms = max_over_ranks(total_ms, dev)
        dist.barrier()
    torch.cuda.synchronize()
    value = world * BATCH * args.steps / (total_ms * 1e-3)
    gpu_launches = 5 * args.steps  # prep, inverse Legendre, FFT+products, forward Legendre, tail

    # sequential single-state evaluations (the pattern inside an SDC sweep: node m+1 needs node m),
    # captured once into a CUDA graph and replayed - as the PFASST controller replays its blocks -
    # so the number is the device time of the chain, not Python/ctypes launch overhead (eager
    # launches from Python are reported beside it); L2 flushed before each group of 5
    seq_stream = torch.cuda.Stream()

    def seq_chain():
        for s in range(BATCH):
            _lib.check(L.pswe_eval_imex(plan.handle, ctypes.byref(cprm), states[s].data_ptr(), fi[s].data_ptr(),
                                        fe[s].data_ptr(), 1, ctypes.c_void_p(seq_stream.cuda_stream)))

    with torch.cuda.stream(seq_stream):
        seq_chain()
    torch.cuda.synchronize()
    seq_graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(seq_graph, stream=seq_stream):
        seq_chain()
    seq, seq_eager = [], []
    for k in range(args.steps):
        for mode in ("graph", "eager"):
            flush.zero_()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(seq_stream)
            with torch.cuda.stream(seq_stream):
                if mode == "graph":
                    seq_graph.replay()
                else:
                    seq_chain()
            b.record(seq_stream)
            torch.cuda.synchronize()
            (seq if mode == "graph" else seq_eager).append(a.elapsed_time(b))
    seq_ms = sum(seq)
    sequential = {"value": BATCH * args.steps / (seq_ms * 1e-3), "unit": "evals/s",
                  "us_per_eval": 1e3 * seq_ms / (BATCH * args.steps),
                  "us_per_eval_eager": 1e3 * sum(seq_eager) / (BATCH * args.steps),
                  "note": "one state per call, 5 back to back (as inside an SDC sweep), CUDA-graph replay; "
                          "us_per_eval_eager: the same launched eagerly from Python"}
    del seq_graph

    # the same batch on the reference's dealiased T255 grid 384 x 768 (side result)
    dplan = P.TransformPlan(R_BENCH, NLAT_DEALIASED, NLON_DEALIASED, args.legendre)
    dplan.reserve(BATCH)
    for _ in range(3):
        _lib.check(L.pswe_eval_imex(dplan.handle, ctypes.byref(cprm), states.data_ptr(), fi.data_ptr(),
                                    fe.data_ptr(), BATCH, _stream()))
    dms = 0.0
    for k in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(L.pswe_eval_imex(dplan.handle, ctypes.byref(cprm), states.data_ptr(), fi.data_ptr(),
                                    fe.data_ptr(), BATCH, _stream()))
        b.record()
        torch.cuda.synchronize()
        dms += a.elapsed_time(b)
    dealiased = {"grid": f"{NLAT_DEALIASED}x{NLON_DEALIASED}", "value": BATCH * args.steps / (dms * 1e-3),
                 "unit": "evals/s", "ms_per_step": dms / args.steps}
    del dplan

    # per-kernel durations (same workload, L2 flushed) for the roofline
    stage = np.zeros(5)
    ms5 = (ctypes.c_float * 5)()
    for k in range(args.steps):
        flush.zero_()
        _lib.check(L.pswe_eval_imex_kernel_times(plan.handle, ctypes.byref(cprm), states.data_ptr(), fi.data_ptr(),
                                                 fe.data_ptr(), BATCH, _stream(), ms5))
        stage += np.array(list(ms5))
    stage /= args.steps
    F_L = NLAT * (R_BENCH + 1) * (R_BENCH + 2)  # flops per complex field per direction
    rowb = (R_BENCH + 1) * NLAT * 16               # bytes of one field's Fourier rows (m <= R)
    Kb = P.num_coeffs(R_BENCH) * 16                # bytes of one spectral field
    Kxb = (R_BENCH + 1) * (R_BENCH + 4) // 2 * 16  # bytes of one extended-triangle column
    # per-kernel algorithmic work: the Legendre contractions are FP64-
    # tensor bound (flops), the prep, the grid stage and the tail stream bytes (HBM)
    work = {
        "prep": ("hbm", BATCH * (3 * Kb + 4 * Kxb)),               # state in, 4 inverse columns out
        "legendre_inverse": ("tensor", 4 * BATCH * F_L),           # Phi, zeta, U, V
        "fft_products": ("hbm", (4 + 5) * BATCH * rowb),            # 4 fields in, 5 products out
        "legendre_forward": ("tensor", 5 * BATCH * F_L),           # Phi'U, Phi'V, qU, qV, ke
        "tail": ("hbm", BATCH * (5 + 3 + 6) * Kb),                 # 5 projections + state in, 2 x 3 out
    }
    names = list(work)
    peak_dfma = float(L.pswe_fp64_peak(0, 4096))
    peak_dmma = float(L.pswe_fp64_peak(1, 2048))
    peak_fp64 = max(peak_dfma, peak_dmma)
    peak = peak_fp64
    hbm_peak, hbm_src = 6650.0, "of fallback (B200_PROFILING.md: 6.65 TB/s)"
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm_peak, hbm_src = float(mp["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (burst copy)"
    except Exception:
        pass
    try:  # per-launch DRAM traffic of each kernel from the committed ncu --set full capture
        traffic_tab = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))["stages"]
    except Exception:
        traffic_tab = {}
    stages = {}
    for n, v in zip(names, stage):
        kind, amount = work[n]
        sec = v * 1e-3
        if kind == "tensor":
            ach, pk, unit = amount / sec / 1e12, peak_fp64, "TFLOP/s"
        else:
            ach, pk, unit = amount / sec / 1e9, hbm_peak, "GB/s"
        stages[n] = {"bound": kind, "ms": float(v), "achieved": ach, "peak": pk, "unit": unit, "frac": ach / pk,
                     "algorithmic": amount, "traffic": traffic_tab.get(n)}
    dom = names[int(np.argmax(stage))]
    d = stages[dom]
    roofline = {
        "bound": d["bound"], "kernel": dom, "achieved": d["achieved"], "peak": d["peak"], "unit": d["unit"],
        "frac": d["frac"], "traffic": d["traffic"],
        "algorithmic_per_launch": d["algorithmic"],
        "peak_source": (f"measured in-run FP64 microbenchmarks (DFMA {peak_dfma:.1f}, DMMA m8n8k4 {peak_dmma:.1f} "
                        f"TFLOP/s; MEASURED_PEAKS.json has no FP64 figure)" if d["bound"] == "tensor"
                        else hbm_src),
        "traffic_source": "profiles/ncu_traffic.json (dram__bytes_read.sum + dram__bytes_write.sum per launch, "
                          "ncu --set full, cache flushed)",
        "kernels": stages,
    }

    # the same kernels on the larger BASELINE grids (configs 4/5): the Legendre contractions'
    # fraction of the FP64 peak once the problem fills the GPU (one wave at T255, several beyond)
    by_size = {}
    if not args.no_sizes:
        for Rs, nls, nlo in ((511, 512, 1024), (1023, 1024, 2048)):
            try:
                splan = P.TransformPlan(Rs, nls, nlo, args.legendre)
                splan.reserve(BATCH)
                sst = torch.as_tensor(bench_states(Rs)).to(dev)
                sfi, sfe = torch.empty_like(sst), torch.empty_like(sst)
                acc5, reps = np.zeros(5), 5
                for k in range(reps + 1):
                    flush.zero_()
                    _lib.check(L.pswe_eval_imex_kernel_times(splan.handle, ctypes.byref(cprm), sst.data_ptr(),
                                                             sfi.data_ptr(), sfe.data_ptr(), BATCH, _stream(), ms5))
                    if k:
                        acc5 += np.array(list(ms5))
                acc5 /= reps
                FLs = nls * (Rs + 1) * (Rs + 2)
                ent = {"workload": f"rhs_eval T{Rs} {nls}x{nlo} x{BATCH} states", "stage_ms": dict(zip(names, acc5.tolist()))}
                for n, nf, col in (("legendre_inverse", 4, 1), ("legendre_forward", 5, 3)):
                    tf = nf * BATCH * FLs / (acc5[col] * 1e-3) / 1e12
                    ent[n] = {"ms": float(acc5[col]), "achieved": tf, "peak": peak_fp64, "unit": "TFLOP/s",
                              "frac": tf / peak_fp64}
                by_size[f"T{Rs}"] = ent
                del splan, sst, sfi, sfe
            except Exception as e:  # reported, never hides the headline
                by_size[f"T{Rs}"] = {"error": f"{type(e).__name__}: {e}"}
        torch.cuda.empty_cache()
    roofline["by_size"] = by_size

    # e2e through the public C ABI (pswe_eval_imex, the drop-in boundary) with pinned host
    # buffers: every step copies its 5 input states host -> device, evaluates, and copies both
    # results (F_I, F_E) device -> host. Double-buffered pipeline: the copies of steps k+1 / k-1
    # run on their own streams while step k evaluates (evals stay ordered on one compute stream, the
    # plan's scratch being single-stream); every step's transfers are inside the timed region.
    nbuf = 2
    h_in = [torch.as_tensor(bench_states()).pin_memory() for _ in range(nbuf)]
    # F_I and F_E of a step side by side in one buffer: one device->host copy per step
    h_out = [torch.empty((2,) + tuple(h_in[0].shape), dtype=h_in[0].dtype).pin_memory() for _ in range(nbuf)]
    d_in = [torch.empty_like(states) for _ in range(nbuf)]
    d_out = [torch.empty((2,) + tuple(states.shape), dtype=states.dtype, device=states.device) for _ in range(nbuf)]
    d_fi = [d[0] for d in d_out]
    d_fe = [d[1] for d in d_out]
    h_fe = [h[1] for h in h_out]
    s_h2d, s_cmp, s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev_h2d = [torch.cuda.Event() for _ in range(nbuf)]
    ev_cmp = [torch.cuda.Event() for _ in range(nbuf)]
    ev_d2h = [torch.cuda.Event() for _ in range(nbuf)]
    for e in ev_cmp + ev_d2h:
        e.record(s_cmp)

    def e2e_run(nsteps):
        for k in range(nsteps):
            j = k % nbuf
            s_h2d.wait_event(ev_cmp[j])  # eval k-2 has read d_in[j]
            with torch.cuda.stream(s_h2d):
                d_in[j].copy_(h_in[j], non_blocking=True)
            ev_h2d[j].record(s_h2d)
            s_cmp.wait_event(ev_h2d[j])
            s_cmp.wait_event(ev_d2h[j])  # the copies of step k-2 have read d_fi[j], d_fe[j]
            _lib.check(L.pswe_eval_imex(plan.handle, ctypes.byref(cprm), d_in[j].data_ptr(), d_fi[j].data_ptr(),
                                        d_fe[j].data_ptr(), BATCH, ctypes.c_void_p(s_cmp.cuda_stream)))
            ev_cmp[j].record(s_cmp)
            s_d2h.wait_event(ev_cmp[j])
            with torch.cuda.stream(s_d2h):
                h_out[j].copy_(d_out[j], non_blocking=True)
            ev_d2h[j].record(s_d2h)

    e2e_run(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_h2d)
    e2e_run(args.steps)
    s_d2h.wait_event(ev_cmp[(args.steps - 1) % nbuf])
    e1.record(s_d2h)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        e2e_ms = max_over_ranks(e2e_ms, dev)
    st_bytes = BATCH * 3 * P.num_coeffs(R_BENCH) * 16
    e2e = {"value": world * BATCH * args.steps / (e2e_ms * 1e-3), "unit": "evals/s",
           "h2d_bytes_per_step": st_bytes, "d2h_bytes_per_step": 2 * st_bytes,
           "api": "pswe_eval_imex (C ABI) with pinned host buffers, copies double-buffered on their own streams; "
                  "F_I and F_E of a step adjacent (one device->host copy)"}
    # correctness of the pipelined results (last step) against the device-resident evaluation
    np.testing.assert_allclose(h_fe[(args.steps - 1) % nbuf].numpy(), fe.cpu().numpy(), rtol=0, atol=0)

    # config-2 transform micro-bench (15 fields, T255, 256x512)
    tplan = P.TransformPlan(255, 256, 512, args.legendre)
    tplan.reserve(3)
    rng = np.random.default_rng(2)
    rs = np.concatenate([np.full(256 - r, r) for r in range(256)])
    ss = np.concatenate([np.arange(r, 256) for r in range(256)])
    x = (rng.uniform(-1, 1, (15, rs.size)) + 1j * rng.uniform(-1, 1, (15, rs.size))) * (ss + 1.0) ** -1.5
    x[:, rs == 0] = x[:, rs == 0].real
    xd = torch.as_tensor(x).to(dev)
    g = torch.empty((15, 256, 512), dtype=torch.float64, device=dev)
    xb = torch.empty_like(xd)

    def rt():
        _lib.check(L.pswe_synthesise(tplan.handle, xd.data_ptr(), g.data_ptr(), 15, _stream()))
        _lib.check(L.pswe_analyse(tplan.handle, g.data_ptr(), xb.data_ptr(), 15, _stream()))

    for _ in range(3):
        rt()
    tms = 0.0
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rt()
        b.record()
        torch.cuda.synchronize()
        tms += a.elapsed_time(b)
    tms /= args.steps
    rt_err = float((xb - xd).abs().max() / xd.abs().max())
    F_L2 = 256 * 256 * 257
    rt_flops = 2 * 15 * F_L2 + 2 * 15 * 2.5 * 256 * 512 * 9
    transform = {"workload": "config 2: 15 fields T255 256x512 synthesise+analyse", "us_per_roundtrip": 1e3 * tms,
                 "roundtrip_rel_err": rt_err, "tflops": rt_flops / (tms * 1e-3) / 1e12,
                 "frac_of_fp64_peak": rt_flops / (tms * 1e-3) / 1e12 / peak}

    # PFASST (config-3 shape) at n_ts = world
    pf_res, pf_all = None, {}
    if not args.no_pfasst:
        for c in (3, 4, 5):
            try:
                pf_all[str(c)] = run_pfasst(P, prm, world, rank, dev, clocks_dev=local, config=c)
            except Exception as e:  # reported, never hides the headline
                pf_all[str(c)] = {"error": f"{type(e).__name__}: {e}"}
        pf_res = pf_all.get("3")
        if rank == 0 and not args.no_cpu_baseline and pf_res is not None and "error" not in pf_res:
            try:  # the reference's PFASST on the host cores, same IC and n_ts (outside the timed spans)
                th = pf_res.pop("_theta0", None)
                pf_res["cpu_reference"] = reference_pfasst(world, th)
            except Exception as e:
                pf_res["cpu_reference"] = {"error": f"{type(e).__name__}: {e}"}
        for v in pf_all.values():
            v.pop("_theta0", None)

    clk = clocks.stop()

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:  # rank 0 only, after every timed region (also at N > 1)
        try:
            times, cores = reference_step_times(1000, 1, budget_s=10.0 if world == 1 else 5.0)
            cpu = {"value": BATCH * len(times) / sum(times), "unit": "evals/s", "cores": cores, "kind": "reference",
                   "sample": f"{len(times)} steps x {BATCH} evals (bench step: T{R_BENCH} {NLAT}x{NLON}, the 5 "
                             f"bench_states), reference eval_nonlinear+eval_linear, OpenMP {cores} threads, "
                             f"timed like --impl reference (own process, OpenMP active wait, bound) ({sum(times):.1f} s)"}
        except Exception as e:
            cpu = {"value": None, "unit": "evals/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded balanced n^-3 random states, 40 m/s rms; BASELINE config shapes)",
            "config": dict(CONFIG),
            "run": {"shared_gpu_dry_run": shared,"legendre": "recompute" if args.legendre == 0 else "stream",
                    "l2": "flushed between timed steps (256 MiB write, outside the timed span)",
                    "parallelism": f"{world} rank(s), {BATCH} independent states per rank per step"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "gpu_launches": gpu_launches,
            "transform": transform, "pfasst": pf_res, "sequential_single_state": sequential,
            "dealiased_grid": dealiased, "pfasst_configs": pf_all,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


PF_CONFIGS = {
    # BASELINE configs[2..4]: (levels (R, nlat, nlon, nodes) fine -> coarse, dt, steps, iterations)
    3: ([(255, 256, 512, 5), (127, 128, 256, 3)], 60.0, 8, 4),
    4: ([(511, 512, 1024, 5), (255, 256, 512, 3), (127, 128, 256, 2)], 30.0, 16, 4),
    5: ([(1023, 1024, 2048, 5), (511, 512, 1024, 3)], 15.0, 8, 3),
}


def run_pfasst(P, prm, world, rank, dev, clocks_dev=0, config=3):
    """PFASST blocks of a BASELINE config at n_ts = world time ranks (one per GPU, NCCL; serial
    emulation of the one worker at world = 1): wall s per simulated day. Config 4 is three-level
    (the reference has no three-level implementation; grids for the coarse levels: the linear
    (R+1) x 2(R+1) grid, BASELINE states only the fine grid); config 4's iteration count is not
    stated (4, as config 3)."""
    import torch
    import torch.distributed as dist

    from paper_1904_05988_b200.cases import config_state
    lv, dt, steps, n_iter = PF_CONFIGS[config]
    if steps % world:
        return {"skipped": f"{steps} steps not divisible by {world} ranks"}
    n_blocks = steps // world
    plans = [P.TransformPlan(R, nlat, nlon) for R, nlat, nlon, _ in lv]
    levels = [P.Level(pl, prm, nn) for pl, (_, _, _, nn) in zip(plans, lv)]
    pair = P.TransferPair(levels[0], levels[1])
    pair2 = P.TransferPair(levels[1], levels[2]) if len(levels) == 3 else None
    cfg = P.BlockConfig(world, dt, n_iter)
    if world == 1:
        pf = P.Pfasst(pair, cfg, pair2=pair2)
    else:
        transport = os.environ.get("PSWE_TRANSPORT", "ipc")  # CUDA IPC over NVLink (default) or "nccl"
        uid = [P.pfasst.unique_id(transport) if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        pf = P.Pfasst(pair, cfg, rank=rank, world=world, uid=uid[0], pair2=pair2, transport=transport)
    theta0 = torch.as_tensor(config_state(config, plans[0])).to(dev)
    # warm-up: an eager block, then the block whose launches are captured into CUDA graphs (serial
    # emulation: the whole block; distributed: segment graphs) - neither inside the timed region
    P.run_blocks(pf, theta0, 2)
    torch.cuda.synchronize()
    runs = []
    for _ in range(3):  # the whole config (all its steps) three times; the median is reported
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fin, hist = P.run_blocks(pf, theta0, n_blocks)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        if world > 1:
            ms = max_over_ranks(ms, dev)
        runs.append(ms)
    ms = sorted(runs)[1]
    wall = ms * 1e-3
    desc = "/".join(f"T{R}({nlat}x{nlon})" for R, nlat, nlon, _ in lv)
    nodes = "/".join(str(nn) for *_, nn in lv)
    pf.close()
    return {"config": f"config {config}: {desc}, {nodes} nodes, dt {dt:g} s, {steps} steps, {n_iter} iterations",
            "levels": len(lv), "n_ts": world, "blocks": n_blocks, "wall_s": wall,
            "wall_s_per_sim_day": wall / (steps * dt) * 86400,
            "timing": "median of 3 runs of all steps, after an eager and a graph-capture warm-up block",
            "final_residuals": [float(r) for r in hist[-1][:, -1]],
            "_theta0": theta0.cpu().numpy() if config == 3 else None}


def main():
    args = parse()
    if args.ref_worker is not None:
        ref_worker_main(args.ref_worker)
        return
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
