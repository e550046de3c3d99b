"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 paths.

1. bench.py under torchrun: the reference arm runs on rank 0 only, prints
   exactly one JSON line, every rank exits 0 (the contract's launch mode).
2. Dispatch routing across ranks: each rank takes its FIFO from the planner
   C-ABI (tasks with gpu == rank, reference dispatcher) and derives its
   outgoing hand-offs (slot boundary -> worker of (round, slot+1)) and its
   incoming ones; an all_gather over gloo checks that every send has exactly
   one matching receive on the addressed rank and that per-rank FIFOs
   partition the dispatch list.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_reference_arm_two_ranks():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
           "--warmup", "3", "--model", "tiny", "--seq", "256", "--micro-batches", "4"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["value"] > 0 and j["n_gpus"] == 2
    assert j["cpu_baseline"]["kind"] == "port" and j["e2e"]["h2d_bytes_per_step"] == 0


def _routing_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    from paper_2604_27085_b200.planner import COST_DTYPE, Planner
    pl = Planner()
    c = np.zeros(5, dtype=COST_DTYPE)
    c["t_fwd_ns"], c["t_bwd_ns"], c["param_bytes"] = 1000, 3000, 1
    plan = pl.optimal_partition(c, world, 2 * world, mem_limit_bytes=8)  # forces S > 1
    durs = pl.slot_durations(plan, c)
    S = len(durs)
    sched = pl.synthesize("roundpipe", world, 2 * world, 0, 3, durs)
    mine = sched.tasks[sched.tasks["gpu"] == rank]
    sends, recvs = [], []
    for t in mine:
        r, s, mb = int(t["round"]), int(t["slot"]), int(t["mb"])
        if s + 1 < S:
            sends.append((r, s + 1, mb, (r * S + s + 1) % world))
        if s > 0:
            recvs.append((r, s, mb, (r * S + s - 1) % world))
    gathered = [None] * world
    dist.all_gather_object(gathered, {"rank": rank, "sends": sends, "n_tasks": len(mine)})
    expected = sorted((r, s, mb) for g in gathered for (r, s, mb, dst) in g["sends"]
                      if dst == rank)
    got = sorted((r, s, mb) for (r, s, mb, _) in recvs)
    ok_pairing = expected == got
    # each receive's producer is the rank that actually ran (round, slot-1, mb)
    owner = {(int(t["round"]), int(t["slot"]), int(t["mb"])): int(t["gpu"]) for t in sched.tasks}
    ok_src = all(owner[(r, s - 1, mb)] == src for (r, s, mb, src) in recvs)
    total = sum(g["n_tasks"] for g in gathered)
    dist.barrier()
    dist.destroy_process_group()
    out[rank] = (ok_pairing, ok_src, total == len(sched.tasks), S)


def test_dispatch_handoff_routing_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_routing_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        ok_pairing, ok_src, ok_partition, S = res[rank]
        assert ok_pairing and ok_src and ok_partition, (rank, res[rank])
    assert res[0][3] > 1  # the plan really has several slots to hand off between
