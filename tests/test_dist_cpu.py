"""Multi-GPU host logic on CPU: the exact range planner against the oracle,
and a world-size-2 gloo run of the sharded path's host exchanges."""
import os

import numpy as np
import pytest

import oracle
from tests import dist_workers


def test_planner_matches_oracle_ancestors():
    import paper_2112_00364_b200 as smc
    rng = np.random.default_rng(7)
    for case in range(60):
        world = int(rng.integers(1, 9))
        n_per = int(rng.integers(1, 300))
        lw = float(rng.choice([0.5, 3.0, 20.0])) * rng.standard_normal(world * n_per)
        lw[rng.random(lw.size) < 0.3] = -np.inf
        if case % 7 == 0:                      # a whole shard with zero weight
            g = int(rng.integers(0, world))
            lw[g * n_per:(g + 1) * n_per] = -np.inf
        if not np.isfinite(lw).any():
            lw[0] = 0.0
        q = oracle.quantize(lw)
        z = int(rng.integers(0, 2 ** 53))
        totals = [sum(int(x) for x in q[g * n_per:(g + 1) * n_per]) for g in range(world)]
        plan = smc.plan_ranges(totals, n_per, z)
        anc = oracle.systematic(q, z).astype(np.int64)
        ref = [int(np.searchsorted(anc, g * n_per)) for g in range(world)] + [world * n_per]
        assert plan == ref
        # migrated slots: outputs a shard produces outside its own slot range
        for g in range(world):
            lo, hi = plan[g], plan[g + 1]
            own = set(range(g * n_per, (g + 1) * n_per))
            assert all(anc[j] // n_per == g for j in range(lo, hi))
            assert len(own) == n_per


def test_gloo_world2_host_exchanges(tmp_path):
    import torch.multiprocessing as mp
    port = dist_workers.free_port()
    mp.spawn(dist_workers.cpu_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "r0.npy", allow_pickle=True)
    r1 = np.load(tmp_path / "r1.npy", allow_pickle=True)
    assert r0[0] == r1[0] and len(r0[0]) == 2          # same gathered totals, rank order
    assert r0[1] == r1[1]                              # identical plans on every rank
    import paper_2112_00364_b200 as smc
    assert r0[1] == smc.plan_ranges(r0[0], 1000, 0x1234567890ABC)
    assert r0[3] == 0 and r1[3] == 0
    assert r0[2] == [1] * 16 + [2] * 16 == r1[2]       # callback concatenates in rank order
    assert r0[4] == r1[4]                              # broadcast NCCL id (or the same error)


def test_reference_arm_under_torchrun_world2():
    """bench.py --impl reference launched like the driver's N=2 run: rank 0 alone
    times the oracle and prints ONE JSON line; rank 1 exits 0 without work."""
    import json
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "1", "--warmup", "0", "--cpu-budget", "1"]
    p = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
