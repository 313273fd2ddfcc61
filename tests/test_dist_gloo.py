"""World-size-2 gloo tests of the multi-process host logic (CPU only):
region-descriptor exchange/validation as connect_process_group uses it,
layout agreement across ranks from all-gathered count rows, and the
max-over-ranks timing reduction bench.py uses."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_27656_b200 import moe
from paper_2510_27656_b200.engine import NvlinkFabric, RegionDesc
from paper_2510_27656_b200.errors import RegionError


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank: int, world: int, port: int, case: str, q) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fab = NvlinkFabric(group=dist.group.WORLD)
        spec = moe.RoutingSpec(world, 8, 16, 2, hidden=64, elem_size=4, scales=0)
        key = tuple(vars(spec).values())
        if case == "ok":
            d = RegionDesc(rank, "hostA", rank, bytes([rank]) * 64, 4096, key)
            got = fab.exchange(d)
            q.put((rank, [x.rank for x in got], [x.handle[0] for x in got]))
        elif case == "spec_mismatch":
            k = key if rank == 0 else key[:-1] + (99,)
            try:
                fab.exchange(RegionDesc(rank, "hostA", rank, b"\0" * 64, 4096, k))
                q.put((rank, "no error"))
            except RegionError as e:
                q.put((rank, "RegionError:" + str(e)[:40]))
        elif case == "same_gpu":
            try:
                fab.exchange(RegionDesc(rank, "hostA", 0, b"\0" * 64, 4096, key))
                q.put((rank, "no error"))
            except RegionError as e:
                q.put((rank, "RegionError:" + str(e)[:20]))
        elif case == "layout":
            rng = np.random.default_rng(10 + rank)
            routes = np.stack([rng.choice(8, 2, replace=False) for _ in range(16)])
            row = np.bincount(routes.ravel(), minlength=8)
            rows = fab.all_gather(row)
            lay = moe.compute_layout(spec, np.stack(rows))
            q.put((rank, lay.recv_start.tolist(), lay.send_start.tolist(), int(lay.recv_total.sum())))
        elif case == "max":
            t = torch.tensor([1.0 + rank, 5.0 - rank, 3.0])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            q.put((rank, t.tolist()))
    finally:
        dist.destroy_process_group()


def _run(case: str, world: int = 2) -> list:
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    return sorted(out, key=lambda x: x[0])


def test_exchange_sorted_by_rank():
    out = _run("ok")
    for rank, ranks, first_bytes in out:
        assert ranks == [0, 1] and first_bytes == [0, 1]


def test_exchange_rejects_spec_mismatch():
    out = _run("spec_mismatch")
    assert all(msg.startswith("RegionError") for _, msg in out)


def test_exchange_rejects_two_ranks_on_one_gpu():
    out = _run("same_gpu")
    assert all(msg.startswith("RegionError") for _, msg in out)


def test_layout_agrees_across_ranks():
    out = _run("layout")
    assert out[0][1:] == out[1][1:]
    assert out[0][3] == 2 * 16 * 2


def test_max_over_ranks():
    out = _run("max")
    assert out[0][1] == out[1][1] == [2.0, 5.0, 3.0]


def test_reference_arm_under_torchrun_world2():
    """The driver launches `bench.py --impl reference` the same way as the
    B200 arm (torchrun, one process per GPU).  Rank 0 alone times the
    reference's EP=2 step on the host and prints one JSON line; rank 1 exits
    cleanly.  Runs on CPU (no GPU is touched on this path)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--cpu-seconds", "1", "--tokens", "16"]
    p = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [x for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["config"]["ep"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and "EP=2" in d["cpu_baseline"]["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0
