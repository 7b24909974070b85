"""The PFASST controller's per-worker schedule (csrc/pfasst.cpp build_schedule, exported as
pswe_pfasst_schedule) checked on CPU:

* its message log equals the reference's (pfasst.cpp:78-251 via tests/golden);
* executed by 2 real processes over torch.distributed/gloo — one worker per rank, SEND/RECV as
  point-to-point messages on two channels like the NCCL executor — with the numpy oracle as the
  numerical checker, it reproduces the reference's serial-emulation results (final state and
  residual history) for n_ts = 2 over 2 chained blocks.
The schedule is the same data the GPU executors (serial emulation and NCCL) run."""
import os
import socket

import numpy as np
import pytest

from _util import rel_diff_fields

PHI_BAR = 9.80616 * 10000.0


def _log_from_schedule(P, n, n_iter, mf, mc):
    log = [(0, 0, ord("B"), 0, r, 0, 0) for r in range(1, n)]
    for w in range(n):
        for op, phase, it, arg in P.schedule(w, n, n_iter):
            if op == "SEND_COARSE":
                log.append((phase, it, arg, w, w + 1, 1, mc - 1))
            if op == "SEND_FINE":
                log.append((phase, it, arg, w, w + 1, 0, mf - 1))
    return sorted(log)


@pytest.mark.parametrize("n_ts", [1, 2, 4])
def test_schedule_message_log_matches_reference(golden, n_ts):
    import paper_1904_05988_b200 as P
    ref = sorted(tuple(int(v) for v in m) for m in golden[f"pf_nts{n_ts}_msgs"])
    assert _log_from_schedule(P, n_ts, 3, 5, 3) == ref


_LEVEL = {"SEND_FINE": 0, "RECV_FINE_IC": 0, "SEND_MID": 1, "RECV_MID_IC": 1}


@pytest.mark.parametrize("n_levels", [2, 3])
@pytest.mark.parametrize("n,n_iter", [(1, 1), (2, 3), (4, 3), (8, 4)])
def test_schedule_queues_consistent(n_levels, n, n_iter):
    """Replay every worker's schedule in worker order (the serial executor's order) through FIFO
    queues per (receiver, level): each receive must find the message its sender tagged with the
    same (phase, iteration) - the check the C++ executors make - and no message may be left over.
    Covers the three-level V-cycle schedule (BASELINE config 4), which has no reference log."""
    import collections

    import paper_1904_05988_b200 as P
    lc = n_levels - 1
    level = dict(_LEVEL, SEND_COARSE=lc, RECV_COARSE_IC=lc)
    q = collections.defaultdict(collections.deque)
    counts = collections.Counter()
    for w in range(n):
        for op, phase, it, _ in P.schedule(w, n, n_iter, n_levels):
            if op.startswith("SEND_"):
                q[(w + 1, level[op])].append((phase, it))
                counts[level[op]] += 1
            elif op.startswith("RECV_"):
                assert q[(w, level[op])], f"w={w} {op} on an empty channel"
                assert q[(w, level[op])].popleft() == (phase, it), f"w={w} {op} tag mismatch"
    assert all(len(v) == 0 for v in q.values())
    # coarse: n(n-1)/2 predictor + (N-1)(n-1) iteration messages; fine and mid: (N-1)(n-1)
    assert counts[lc] == n * (n - 1) // 2 + (n_iter - 1) * (n - 1)
    assert counts[0] == (n_iter - 1) * (n - 1)
    if n_levels == 3:
        assert counts[1] == (n_iter - 1) * (n - 1)


def test_schedule_counts():
    """coarse messages n(n-1)/2 + (N-1)(n-1), fine (N-1)(n-1)."""
    import paper_1904_05988_b200 as P
    for n in (2, 4, 8):
        for N in (2, 4):
            ops = [o for w in range(n) for o in P.schedule(w, n, N)]
            coarse = sum(o[0] == "SEND_COARSE" for o in ops)
            fine = sum(o[0] == "SEND_FINE" for o in ops)
            assert coarse == n * (n - 1) // 2 + (N - 1) * (n - 1)
            assert fine == (N - 1) * (n - 1)
            assert coarse == sum(o[0] == "RECV_COARSE_IC" for o in ops)
            assert fine == sum(o[0] == "RECV_FINE_IC" for o in ops)


def _execute(rank, world, port, theta0, n_blocks, out):
    """One worker per process: run the C++ schedule with oracle operations and gloo messages."""
    import torch
    import torch.distributed as dist

    import paper_1904_05988_b200 as P
    from oracle import pswe_oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p0 = O.ModelParams(phi_bar=PHI_BAR)
    fine = O.LevelSpec(31, O.build_tables(5), O.SweOde(O.TransformPlan(31), p0))
    coarse = O.LevelSpec(15, O.build_tables(3), O.SweOde(O.TransformPlan(15), p0))
    pair = O.make_transfer_pair(fine, coarse)
    mf, mc, dt, N = 5, 3, 60.0, 3
    th = theta0.copy()
    hist = []

    # Like the NCCL executor: one channel per level (tag = level) and sends that never block the
    # worker (the reference's Channel::send, pfasst.cpp:31-37). A single blocking channel would
    # deadlock: worker w sends fine (Step A) before coarse (Step C), worker w+1 receives coarse
    # (Step C) before fine (Step D).
    pending = []

    def send(x, level):
        t = torch.from_numpy(np.ascontiguousarray(x).view(np.float64).copy())
        pending.append((dist.isend(t, dst=rank + 1, tag=level), t))

    def recv(shape, level):
        t = torch.empty(int(np.prod(shape)) * 2, dtype=torch.float64)
        dist.recv(t, src=rank - 1, tag=level)
        return t.numpy().view(np.complex128).reshape(shape)

    for _ in range(n_blocks):
        res = [0.0] * (N + 1)
        st = {}
        for op, phase, it, arg in P.schedule(rank, world, N):
            if op == "PREDICT_INIT":
                st["c"] = O.spread(O.restrict_space(th, 31, 15), mc, coarse.ode)
            elif op == "RECV_COARSE_IC":
                st["c"].state[0] = recv(th[:, :O.num_coeffs(15)].shape, 1)
            elif op == "REFRESH_COARSE0":
                O.refresh_node(st["c"], 0, coarse.ode)
            elif op == "SWEEP_COARSE":
                O.sweep(st["c"], dt, coarse.tables, coarse.ode, st.get("tau") if arg else None)
            elif op == "SEND_COARSE":
                send(st["c"].state[mc - 1], 1)
            elif op == "INTERP_STATES":
                st["f"] = O.SpaceTimeState(O.interpolate_states(st["c"].state, pair), [None] * mf, [None] * mf)
            elif op == "REFRESH_FINE_ALL":
                for m in range(mf):
                    O.refresh_node(st["f"], m, fine.ode)
            elif op == "RESIDUAL":
                res[arg] = O.collocation_residual(st["f"], dt, fine.tables)
            elif op == "SWEEP_FINE":
                O.sweep(st["f"], dt, fine.tables, fine.ode)
            elif op == "SEND_FINE":
                send(st["f"].state[mf - 1], 0)
            elif op == "RESTRICT":
                st["c"].state = O.restrict_states(st["f"].state, pair)
            elif op == "REFRESH_COARSE_ALL":
                for m in range(mc):
                    O.refresh_node(st["c"], m, coarse.ode)
            elif op == "SAVE":
                st["saved"] = st["c"].copy()
            elif op == "FAS":
                st["tau"] = O.fas_correction(st["f"], st["c"], dt, pair)
            elif op == "INTERP_INC":
                sv = st["saved"]
                ds = O.interpolate_increment(st["c"].state, sv.state, pair)
                di = O.interpolate_increment(st["c"].f_imp, sv.f_imp, pair)
                de = O.interpolate_increment(st["c"].f_exp, sv.f_exp, pair)
                for m in range(mf):
                    st["f"].state[m] = st["f"].state[m] + ds[m]
                    st["f"].f_imp[m] = st["f"].f_imp[m] + di[m]
                    st["f"].f_exp[m] = st["f"].f_exp[m] + de[m]
                st["d0"] = ds[0]
            elif op == "RECV_FINE_IC":
                st["f"].state[0] = recv(th.shape, 0) + st["d0"]
            elif op == "REFRESH_FINE0":
                O.refresh_node(st["f"], 0, fine.ode)
            else:
                raise AssertionError(op)
        for wk, _ in pending:
            wk.wait()
        pending.clear()
        # block chaining (runner.cpp:145-147): the last rank's final state to everyone
        fin = torch.from_numpy(np.ascontiguousarray(st["f"].state[mf - 1]).view(np.float64).copy())
        dist.broadcast(fin, src=world - 1)
        th = fin.numpy().view(np.complex128).reshape(th.shape)
        gathered = [torch.zeros(N + 1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, torch.tensor(res, dtype=torch.float64))
        hist.append([g.numpy() for g in gathered])
    if rank == 0:
        out.put((th, np.array(hist)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_execution_matches_reference(golden):
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_execute, args=(r, 2, port, golden["pf_theta0"], 2, q)) for r in range(2)]
    for p in procs:
        p.start()
    th, hist = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert rel_diff_fields(th, golden["pf_nts2_final"]) < 1e-10
    ref = golden["pf_nts2_res"]
    floor = 64 * 2.0**-52 * np.abs(th[0]).max()
    assert np.all(np.abs(hist - ref) <= 1e-6 * np.abs(ref) + floor)
