"""Multi-GPU parity: one rank per GPU in one process (threads, peer access)
and one rank per process (torchrun, CUDA IPC).  Skipped with fewer GPUs
than ranks; run with `gpurun --gpus N`."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from golden_io import load_moe
from oracle import moe_oracle as mo

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0

if NGPU:
    from moe_driver import check_device_round, close_mesh, device_round, ospec_of, run_moe_round
    from paper_2510_27656_b200.errors import ProtocolError
    from paper_2510_27656_b200 import moe
    from paper_2510_27656_b200.engine import local_engines


def _np(x):
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


@pytest.mark.parametrize("name", ["cfg1_full", "cfg1_rand", "check_moe", "n4_e16_t9_r4", "n4_e8_t5_r1",
                                  "n8_e16_t7_r3", "fp8_n4_h64_s1", "fp8_dsv3ish", "empty"])
def test_golden_one_rank_per_gpu(name):
    case = load_moe(name)
    spec = moe.RoutingSpec(**case.spec_args)
    if NGPU < spec.ranks:
        pytest.skip(f"needs {spec.ranks} GPUs")
    mesh = moe.build_mesh(local_engines(list(range(spec.ranks))), spec, timeout=20.0)
    assert not mesh[0].host_gated
    try:
        for st in case.steps:
            res = run_moe_round(mesh, spec, st.routes, st.values, st.weights, timeout=20.0)
            for q in range(spec.ranks):
                g, comb, pos = res[q]
                assert np.array_equal(pos, st.pos[q])
                assert np.array_equal(_np(g.rows), st.rows[q])
                assert np.array_equal(_np(g.sources), st.sources[q])
                assert np.array_equal(_np(g.data), st.data[q])
                assert np.array_equal(comb, st.combined[q])
    finally:
        close_mesh(mesh)


@pytest.mark.parametrize("shape", ["dsv3", "kimi"])
@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_dsv3_decode_device_mode(ranks, shape):
    """DeepSeek-V3 decode shape (256 experts, uniform routes) or Kimi-K2 shape
    (384 experts, bench.py's skewed routes), EP=ranks over NVLink, fused fp8
    encode in the dispatch kernel, bf16 combine rows; several steps back to
    back."""
    if NGPU < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    import threading
    import bench
    E = 256 if shape == "dsv3" else 384
    spec = moe.RoutingSpec(ranks=ranks, experts=E, max_tokens=128, topk=8, hidden=7168,
                           elem_size=1, scales=56, comb_elem_size=2, comb_scales=0)
    os_ = ospec_of(spec)
    cs = mo.Spec(ranks, E, 128, 8, hidden=7168, elem_size=2, scales=0)
    mesh = moe.build_mesh(local_engines(list(range(ranks))), spec, timeout=20.0)
    try:
        for step in range(3):
            rng = np.random.default_rng(200 + step)
            routes, values, weights = mo.random_step(os_, rng, tokens=128)
            if shape == "kimi":
                routes = [bench.routes_for(bench.WORKLOADS["kimi"], rng, 128) for _ in range(ranks)]
            xb = [torch.from_numpy(v).to(torch.bfloat16) for v in values]
            ref = mo.dispatch(os_, routes, [mo.encode_tokens(os_, x.float().numpy()) for x in xb])
            got = [None] * ranks
            outs_np = [None] * ranks
            errs = []

            def worker(r):
                try:
                    torch.cuda.set_device(r)
                    rk = mesh[r]
                    rk.dispatch_send(xb[r].cuda(r), torch.from_numpy(routes[r]).cuda(r))
                    g = rk.dispatch_recv()
                    dec = moe.decode_tokens(spec, g.data)
                    y = (dec * 0.5).to(torch.bfloat16)
                    outs_np[r] = (g.data.cpu().numpy(), y.float().cpu().numpy())
                    rk.combine_send(y)
                    got[r] = rk.combine_recv(torch.from_numpy(weights[r]).cuda(r), out_dtype=torch.bfloat16)
                    torch.cuda.synchronize(r)
                except Exception as e:  # noqa: BLE001
                    errs.append(e)

            th = [threading.Thread(target=worker, args=(r,)) for r in range(ranks)]
            for t in th:
                t.start()
            for t in th:
                t.join(120)
            if errs:
                raise errs[0]
            for r in range(ranks):
                assert np.array_equal(outs_np[r][0], ref.ranks[r].grouped.data)
            outs = [mo.bf16_encode(outs_np[r][1]).view(np.uint8).reshape(outs_np[r][1].shape[0], -1)
                    for r in range(ranks)]
            comb = mo.combine(os_, ref, outs, weights, comb_spec=cs)
            for r in range(ranks):
                want = mo.bf16_encode(comb[r])
                assert np.array_equal(got[r].view(torch.int16).cpu().numpy().view(np.uint16), want)
    finally:
        close_mesh(mesh)


@pytest.mark.parametrize("config", ["decode", "kimi"])
@pytest.mark.parametrize("ranks", [2, 4])
def test_torchrun_ipc_bench_smoke(ranks, config, tmp_path):
    """One rank per process over CUDA IPC (connect_process_group): a bench
    run under torchrun (graph replays, L2 flush, device barrier, e2e from
    pinned host memory; ~200 steps in all) must finish and print one JSON
    line.  The Kimi-shape case is the one that exposed an intermittent fault
    no thread-mesh test showed."""
    if NGPU < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(29531 + ranks + (10 if config == "kimi" else 0)),
           str(ROOT / "bench.py"), "--config", config,
           "--gpus", str(ranks), "--steps", "60", "--warmup", "3", "--no-cpu-baseline"]
    env = dict(os.environ)
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert "txb check failed" not in p.stdout, p.stdout[:4000]
    assert p.returncode == 0, p.stderr[-4000:]
    import json
    line = [x for x in p.stdout.splitlines() if x.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == ranks and d["value"] > 0


CHECKED_LIB = ROOT / "paper_2510_27656_b200" / "libtxb200_checked.so"


@pytest.mark.parametrize("ranks", [2, 4])
def test_torchrun_bench_checked_build(ranks):
    """The bench under torchrun on the bounds-checked library, three times:
    no device-side check may fire.  This is the run that caught the
    receive-table race of round 2 (recv_tables_body read rowbase[0] while
    thread 0 rewrote it; a warp's return slots then ran past comb_rows):
    one torchrun bench in four tripped it at EP=2, none in twelve after the
    fix (profiles/r02/README.md)."""
    if NGPU < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    if not CHECKED_LIB.exists():
        pytest.skip("libtxb200_checked.so not built (make checked)")
    env = dict(os.environ, TXB200_LIB=str(CHECKED_LIB))
    for rep in range(3):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
               "--master-addr", "127.0.0.1", "--master-port", str(29571 + 4 * rep + ranks),
               str(ROOT / "bench.py"), "--config", "decode",
               "--gpus", str(ranks), "--steps", "60", "--warmup", "3", "--no-cpu-baseline"]
        p = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
        assert "txb check failed" not in p.stdout, f"run {rep}: " + p.stdout[:4000]
        assert p.returncode == 0, f"run {rep}: " + p.stderr[-4000:]


@pytest.mark.parametrize("ranks", [2, 4])
def test_prefill_size_generic_path_multi_gpu(ranks):
    """Large batch (generic fused kernel, grid barrier) across GPUs: grouped
    payloads bit-exact vs the oracle, bf16 combine exact in bf16 bits."""
    if NGPU < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    import threading
    T = 512
    spec = moe.RoutingSpec(ranks=ranks, experts=64, max_tokens=T, topk=8, hidden=512,
                           elem_size=2, scales=0, comb_elem_size=2, comb_scales=0)
    os_ = ospec_of(spec)
    rng = np.random.default_rng(7)
    routes, values, weights = mo.random_step(os_, rng, tokens=T)
    xb = [torch.from_numpy(v).to(torch.bfloat16) for v in values]
    ref = mo.dispatch(os_, routes, [mo.encode_tokens(os_, x.float().numpy()) for x in xb])
    mesh = moe.build_mesh(local_engines(list(range(ranks))), spec, timeout=20.0)
    got, errs = [None] * ranks, []

    def worker(r):
        try:
            torch.cuda.set_device(r)
            rk = mesh[r]
            rk.dispatch_send(xb[r].cuda(r), torch.from_numpy(routes[r]).cuda(r))
            g = rk.dispatch_recv()
            y = g.data.view(torch.bfloat16).reshape(g.data.shape[0], -1).clone()
            rk.combine_send(y)
            out = rk.combine_recv(torch.from_numpy(weights[r]).cuda(r), out_dtype=torch.bfloat16)
            got[r] = (g.data.cpu().numpy(), out.view(torch.int16).cpu().numpy().view(np.uint16))
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(ranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(120)
    try:
        if errs:
            raise errs[0]
        outs = []
        for r in range(ranks):
            assert np.array_equal(got[r][0], ref.ranks[r].grouped.data)
            outs.append(ref.ranks[r].grouped.data)
        comb = mo.combine(os_, ref, outs, weights, comb_spec=os_)
        for r in range(ranks):
            assert np.array_equal(got[r][1], mo.bf16_encode(comb[r]))
    finally:
        close_mesh(mesh)


@pytest.mark.parametrize("ranks", [2, 4])
def test_per_token_completion_mixed_batches(ranks):
    """max_tokens above the per-token threshold: large steps use per-token
    combine completion (whole-row returns, per-origin-token counters), small
    steps the decode kernels and the global counter, empty steps neither.
    The counters must stay consistent across any sequence of them; every
    step is checked bit-exactly (grouped data, bf16 combine bits)."""
    if NGPU < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    import threading
    T = 600
    spec = moe.RoutingSpec(ranks=ranks, experts=32, max_tokens=T, topk=4, hidden=256,
                           elem_size=2, scales=0, comb_elem_size=2, comb_scales=0)
    os_ = ospec_of(spec)
    mesh = moe.build_mesh(local_engines(list(range(ranks))), spec, timeout=20.0)
    try:
        for step, n in enumerate([600, 90, 0, 333, 17, 600]):
            rng = np.random.default_rng(900 + step)
            routes, values, weights = mo.random_step(os_, rng, tokens=n)
            xb = [torch.from_numpy(v).to(torch.bfloat16) for v in values]
            ref = mo.dispatch(os_, routes, [mo.encode_tokens(os_, x.float().numpy()) for x in xb])
            got, errs = [None] * ranks, []

            def worker(r):
                try:
                    torch.cuda.set_device(r)
                    rk = mesh[r]
                    rk.dispatch_send(xb[r].cuda(r), torch.from_numpy(routes[r]).cuda(r))
                    g = rk.dispatch_recv()
                    y = g.data.view(torch.bfloat16).reshape(g.data.shape[0], spec.hidden).clone()
                    rk.combine_send(y)
                    out = rk.combine_recv(torch.from_numpy(weights[r]).cuda(r), out_dtype=torch.bfloat16)
                    got[r] = (g.data.cpu().numpy(), out.view(torch.int16).cpu().numpy().view(np.uint16))
                except Exception as e:  # noqa: BLE001
                    errs.append(e)

            th = [threading.Thread(target=worker, args=(r,)) for r in range(ranks)]
            for t in th:
                t.start()
            for t in th:
                t.join(120)
            if errs:
                raise errs[0]
            outs = []
            for r in range(ranks):
                assert np.array_equal(got[r][0], ref.ranks[r].grouped.data), (step, r)
                outs.append(ref.ranks[r].grouped.data)
            comb = mo.combine(os_, ref, outs, weights, comb_spec=os_)
            for r in range(ranks):
                assert np.array_equal(got[r][1], mo.bf16_encode(comb[r])), (step, r)
    finally:
        close_mesh(mesh)


@pytest.mark.parametrize("ptok", [0, 4, 32, 128])
@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_private_round_one_rank_per_gpu(ranks, ptok):
    """DeepSeek-V3 decode shape over NVLink with the speculative private
    round at P in {0, 4, 32, T}: the decode kernel stores each copy whose
    slab slot is below P into the owner's private slab before the route
    exchange completes; the owner moves it to its grouped row.  Payloads,
    indices and the bf16 combine bit-exact vs the oracle, three steps."""
    if NGPU < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    spec = moe.RoutingSpec(ranks=ranks, experts=256, max_tokens=128, topk=8, hidden=7168,
                           elem_size=1, scales=56, comb_elem_size=2, comb_scales=0)
    mesh = moe.build_mesh(local_engines(list(range(ranks))), spec, private=moe.PrivateBufferConfig(ptok),
                          timeout=20.0)
    assert not mesh[0].host_gated
    try:
        for step in range(3):
            rng = np.random.default_rng(500 + 10 * ptok + step)
            routes, values, weights = mo.random_step(ospec_of(spec), rng, tokens=128 - 37 * (step == 1))
            xb, got = device_round(mesh, spec, routes, values, weights, timeout=20.0)
            check_device_round(spec, routes, xb, weights, got, f"P={ptok} step {step}")
        _, c = mesh[0].status()
        assert c["priv_ctr"][0] == c["priv_target"][0] and c["priv_ctr"][1] == c["priv_target"][1]
    finally:
        close_mesh(mesh)


def test_route_timeout_fused_names_the_silent_rank():
    """Fused path across two GPUs: rank 1 never sends, rank 0's dispatch
    kernel gives up at its device deadline and dispatch_recv raises the
    reference-shaped ProtocolError naming rank 1 (moe.py:869-899)."""
    if NGPU < 2:
        pytest.skip("needs 2 GPUs")
    spec = moe.RoutingSpec(ranks=2, experts=16, max_tokens=32, topk=4, hidden=512, elem_size=1, scales=4)
    mesh = moe.build_mesh(local_engines([0, 1]), spec, timeout=1.5)
    try:
        rng = np.random.default_rng(4)
        routes, values, _ = mo.random_step(ospec_of(spec), rng, tokens=32)
        torch.cuda.set_device(0)
        mesh[0].dispatch_send(torch.from_numpy(values[0]).cuda(0), torch.from_numpy(routes[0]).cuda(0))
        with pytest.raises(ProtocolError, match=r"rank 0 step 0 timed out waiting for route counts; "
                                                r"missing: \{'route': \[1\]\}"):
            mesh[0].dispatch_recv(1.5)
    finally:
        close_mesh(mesh)


def test_combine_timeout_fused_names_the_silent_rank():
    """Both ranks dispatch, rank 1 never returns its expert outputs: rank
    0's combine gives up and names rank 1 in the combine lane."""
    if NGPU < 2:
        pytest.skip("needs 2 GPUs")
    import threading
    spec = moe.RoutingSpec(ranks=2, experts=16, max_tokens=32, topk=4, hidden=512, elem_size=1, scales=4)
    mesh = moe.build_mesh(local_engines([0, 1]), spec, timeout=1.5)
    try:
        rng = np.random.default_rng(5)
        routes, values, weights = mo.random_step(ospec_of(spec), rng, tokens=32)
        gs = [None, None]

        def disp(r):
            torch.cuda.set_device(r)
            mesh[r].dispatch_send(torch.from_numpy(values[r]).cuda(r), torch.from_numpy(routes[r]).cuda(r))
            gs[r] = mesh[r].dispatch_recv(10.0)

        th = [threading.Thread(target=disp, args=(r,)) for r in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join(60)
        assert gs[0] is not None and gs[1] is not None
        torch.cuda.set_device(0)
        mesh[0].combine_send(gs[0].data)
        with pytest.raises(ProtocolError, match=r"rank 0 step 0 timed out waiting for combine writes; "
                                                r"missing: \{'combine': \[1\]\}"):
            mesh[0].combine_recv(torch.from_numpy(weights[0]).cuda(0), 1.5)
    finally:
        close_mesh(mesh)


@pytest.mark.parametrize("ranks", [2, 4])
def test_per_token_mode_odd_rows_alternating_paths(ranks):
    """max_tokens above the per-token threshold, fp8 rows of 132 bytes (not
    16-byte vectorisable), and steps that alternate between
    the fused kernels and the split kernels on every rank: per-token
    counters (tokc / tokt) must stay in step across paths -- every step
    bit-exact, and the counters balanced at the end."""
    if NGPU < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    spec = moe.RoutingSpec(ranks=ranks, experts=16, max_tokens=300, topk=4, hidden=100, elem_size=1, scales=8)
    mesh = moe.build_mesh(local_engines(list(range(ranks))), spec, private=moe.PrivateBufferConfig(16),
                          timeout=20.0)
    try:
        for step, (n, fused) in enumerate([(300, True), (300, False), (57, True), (300, True), (0, False),
                                           (211, False), (300, True)]):
            for rk in mesh:
                rk.fused = fused
            rng = np.random.default_rng(300 + step)
            routes, values, weights = mo.random_step(ospec_of(spec), rng, tokens=n)
            xb, got = device_round(mesh, spec, routes, values, weights, timeout=20.0, out_dtype=torch.float32)
            check_device_round(spec, routes, xb, weights, got, f"step {step} fused={fused}")
        for q, rk in enumerate(mesh):
            _, c = rk.status()
            assert c["tok_ctr"] == c["tok_target"], q
            assert c["comb_ctr"] == c["comb_target"], q
    finally:
        close_mesh(mesh)


@pytest.mark.parametrize("ranks", [2, 4])
def test_dsv3_prefill_full_size_multi_gpu(ranks):
    """DeepSeek-V3 prefill at full size (4096 tokens per rank, hidden 7168,
    256 experts, top-8, bf16 both ways) at EP=2/4 over NVLink: the
    large-batch path with per-token combine completion, bit-exact."""
    if NGPU < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    spec = moe.RoutingSpec(ranks=ranks, experts=256, max_tokens=4096, topk=8, hidden=7168, elem_size=2,
                           scales=0, comb_elem_size=2, comb_scales=0)
    mesh = moe.build_mesh(local_engines(list(range(ranks))), spec, timeout=60.0)
    try:
        rng = np.random.default_rng(44)
        routes, values, weights = mo.random_step(ospec_of(spec), rng, tokens=4096)
        xb, got = device_round(mesh, spec, routes, values, weights, timeout=60.0)
        check_device_round(spec, routes, xb, weights, got)
    finally:
        close_mesh(mesh)


@pytest.mark.parametrize("n,e,t,r", [(2, 4, 9, 2), (2, 16, 16, 4), (4, 8, 5, 1), (4, 16, 13, 4), (4, 4, 16, 2),
                                     (8, 8, 7, 4), (8, 16, 16, 2), (8, 16, 3, 1)])
def test_acceptance_grid_one_rank_per_gpu(n, e, t, r):
    """SPEC.md criterion 6 grid points on real peers (fused cooperative
    kernels, one GPU per rank): bit-exact against the oracle over three
    seeded steps."""
    if NGPU < n:
        pytest.skip(f"needs {n} GPUs")
    spec = moe.RoutingSpec(ranks=n, experts=e, max_tokens=t, topk=r, hidden=64, elem_size=1, scales=8)
    os_ = ospec_of(spec)
    mesh = moe.build_mesh(local_engines(list(range(n))), spec, timeout=20.0)
    try:
        for seed in range(3):
            rng = np.random.default_rng(77 + seed)
            routes, values, weights = mo.random_step(os_, rng)
            res = run_moe_round(mesh, spec, routes, values, weights, timeout=20.0)
            ref = mo.dispatch(os_, routes, [mo.encode_tokens(os_, v) for v in values])
            comb = mo.combine(os_, ref, mo.apply_experts(os_, ref), weights)
            for q in range(n):
                g, c, pos = res[q]
                assert np.array_equal(_np(g.data), ref.ranks[q].grouped.data), (seed, q)
                assert np.array_equal(_np(g.rows), ref.ranks[q].grouped.rows), (seed, q)
                assert np.array_equal(c, comb[q]), (seed, q)
    finally:
        close_mesh(mesh)
