"""Benchmark: MoE dispatch+combine p50 latency on B200 (BASELINE.json metric).

Default workload (BASELINE.json configs[1], DeepSeek-V3 decode): 128 tokens
per rank, hidden 7168, 256 experts, top-8; dispatch carries fp8 e4m3 rows
with per-token f32 scales (7168 + 56*4 = 7392 B, encoded inside the
dispatch kernel from bf16 activations), combine carries bf16 rows
(14336 B) and produces bf16 outputs.  EP = number of GPUs (1 = loopback
through HBM).  --config prefill (configs[2]: 4096 tok/rank, bf16 both
ways) and --config kimi (configs[3]: 384 experts, skewed routing) run the
other BASELINE configurations with the same methodology.

A step = dispatch_send -> dispatch_recv -> combine_send -> combine_recv
through the public MoeRank API (launch-only, sync=False).  The K timed
steps run back to back in CUDA graphs of B steps each, every step on its
own input set from a pool whose touched bytes are twice the L2 (no flush
between steps); each graph replay follows a device-side all-rank barrier
(N > 1) and is timed with CUDA events on the rank's stream.
value = p50 over the K/B blocks of (max over ranks of the block span) / B.
The flushed single step (L2 flushed by a 512 MiB write + read, CUDA event
nodes inside its graph), the eager step and the %globaltimer kernel span
are reported beside it.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]
        torchrun --nproc-per-node N bench.py --gpus N ...
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    "decode": dict(tokens=128, experts=256, topk=8, hidden=7168, elem=1, scales=56, routing="uniform",
                   name="DeepSeek-V3 decode dispatch+combine",
                   metric="dispatch+combine p50 us (decode, DeepSeek-V3 shape)"),
    "prefill": dict(tokens=4096, experts=256, topk=8, hidden=7168, elem=2, scales=0, routing="uniform",
                    name="DeepSeek-V3 prefill dispatch+combine (bf16)",
                    metric="dispatch+combine p50 us (prefill, DeepSeek-V3 shape, bf16)"),
    "kimi": dict(tokens=128, experts=384, topk=8, hidden=7168, elem=1, scales=56, routing="skewed",
                 name="Kimi-K2-shape decode dispatch+combine, skewed routing",
                 metric="dispatch+combine p50 us (decode, Kimi-K2 shape, skewed)"),
}


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="decode", choices=sorted(WORKLOADS))
    ap.add_argument("--tokens", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--flush", default="write+read", choices=["write+read", "write"])
    ap.add_argument("--private", type=int, default=0,
                    help="PrivateBufferConfig.tokens (0: no speculative private round, the tuned "
                         "choice on NVLink, DESIGN.md §10; the API default is min(32, tokens))")
    return ap.parse_args()


def workload_config(wl: dict, tokens: int, ep: int, private: int | None) -> dict:
    """The `config` object both arms print (identical keys and values, so
    the driver can match the GPU arm's line with the reference arm's)."""
    P = wl["hidden"] * wl["elem"] + 4 * wl["scales"]
    return {"workload": wl["name"], "tokens_per_rank": tokens, "hidden": wl["hidden"],
            "experts": wl["experts"], "topk": wl["topk"], "ep": ep, "dispatch_row_bytes": P,
            "combine_row_bytes": 2 * wl["hidden"], "routing": f"{wl['routing']} top-{wl['topk']}",
            "parallelism": f"ep{ep}",
            "private_tokens": private if private is not None else min(32, tokens)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def routes_for(wl: dict, rng: np.random.Generator, tokens: int) -> np.ndarray:
    """Uniform top-R, or skewed: Gumbel-top-R over logits
    -log(1 + rank_e) on a seeded expert permutation (Zipf-like hot experts)."""
    E, R = wl["experts"], wl["topk"]
    if wl["routing"] == "uniform":
        return np.argsort(rng.random((tokens, E)), axis=1)[:, :R].astype(np.int64)
    perm = np.random.default_rng(1234).permutation(E)
    logits = -np.log1p(np.arange(E, dtype=np.float64))[np.argsort(perm)]
    g = -np.log(-np.log(rng.random((tokens, E))))
    return np.argsort(-(logits[None, :] + g), axis=1)[:, :R].astype(np.int64)


def _inputs(wl: dict, rank: int, tokens: int, seed: int = 0):
    rng = np.random.default_rng((seed << 8) + rank)
    x = rng.standard_normal((tokens, wl["hidden"])).astype(np.float32)
    routes = routes_for(wl, rng, tokens)
    w = rng.random((tokens, wl["topk"])).astype(np.float32)
    return x, routes, w


# ------------------------------------------------------------ CPU baseline


def cpu_port_step(ospec, cspec, xbs, routes, ws, outs, mo, pool=None, nthr: int = 1):
    """One step of the reference algorithm on the host (oracle port) for all
    ospec.ranks ranks, the same work the GPU step times: encode the bf16
    values to fp8 rows -> dispatch regroup -> return the (given) expert output
    rows to their origins -> fp32 weighted sum -> bf16 out.  The per-token
    parts (encode, decode + sum, bf16 rounding) run in `nthr` row chunks on a
    thread pool (numpy drops the GIL inside its array kernels); the regroup
    and the returns are vectorised gathers / scatters."""
    N = len(xbs)
    run = (lambda f, xs: list(pool.map(f, xs))) if pool is not None else (lambda f, xs: [f(c) for c in xs])
    jobs = [(r, c) for r in range(N) for c in np.array_split(np.arange(xbs[r].shape[0]), nthr) if c.size]
    enc = run(lambda rc: mo.encode_tokens(ospec, xbs[rc[0]][rc[1]]), jobs)
    pays = [np.concatenate([e for (r, _), e in zip(jobs, enc) if r == q] or
                           [np.zeros((0, ospec.payload_bytes), np.uint8)]) for q in range(N)]
    res = mo.dispatch(ospec, routes, pays)
    send = [np.zeros((max(1, res.ranks[q].pos.size), cspec.payload_bytes), np.uint8) for q in range(N)]
    for d in range(N):
        rr = res.ranks[d]
        valid = np.nonzero(rr.grouped.rows >= 0)[0]
        srcs = rr.grouped.sources[valid]
        for q in range(N):
            m = valid[srcs == q]
            send[q][rr.src_slot[m]] = outs[d][m]
    R = ospec.topk

    def reduce(rc):
        r, c = rc
        y = mo.decode_tokens(cspec, send[r][res.ranks[r].pos[c].ravel()])
        return mo.bf16_encode(mo.weighted_combine(y, np.arange(c.size * R).reshape(c.size, R), ws[r][c]))

    red = run(reduce, jobs)
    return [np.concatenate([o for (r, _), o in zip(jobs, red) if r == q] or
                           [np.zeros((0, ospec.hidden), np.uint16)]) for q in range(N)]


def _host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def cpu_baseline(wl: dict, tokens: int, seconds: float, ranks: int = 1) -> dict:
    """The oracle port timed on the host with every host thread (row chunks
    on a thread pool), for `ranks` ranks (the reference runs every rank of an
    EP=N step in one host process over its SimFabric), on a bounded sample:
    the full step when it is short, else a 512-token slice per rank scaled
    linearly to the step's token count (stated in `sample`).  The result is
    checked against the serial oracle once before timing."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import moe_oracle as mo
    sample = min(tokens, 512)
    E, R, H = wl["experts"], wl["topk"], wl["hidden"]
    N = ranks
    ospec = mo.Spec(N, E, sample, R, hidden=H, elem_size=wl["elem"], scales=wl["scales"])
    cspec = mo.Spec(N, E, sample, R, hidden=H, elem_size=2, scales=0)
    ins = [_inputs(wl, r, sample) for r in range(N)]
    xbs = [mo.bf16_decode(mo.bf16_encode(x)) for x, _, _ in ins]
    routes = [rt for _, rt, _ in ins]
    ws = [w for _, _, w in ins]
    res = mo.dispatch(ospec, routes, [mo.encode_tokens(ospec, xb) for xb in xbs])
    # synthetic expert outputs (bf16 rows), like the GPU step's
    outs = []
    for d in range(N):
        rows = res.ranks[d].grouped.rows.size
        o = mo.bf16_encode(np.random.default_rng(5 + d).standard_normal((rows, H)).astype(np.float32))
        outs.append(o.view(np.uint8).reshape(rows, -1))
    host = _host_threads()
    want = [mo.bf16_encode(c) for c in mo.combine(ospec, res, outs, ws, comb_spec=cspec)]
    # thread count: the fastest of 1, 2, 4, ... host threads on a short trial
    # (tiny per-thread chunks lose to Python overhead on many-core hosts)
    cands = sorted({min(host, 1 << k) for k in range(0, 8)})
    best = None
    for nthr in cands:
        with ThreadPoolExecutor(nthr) as pool:
            got = cpu_port_step(ospec, cspec, xbs, routes, ws, outs, mo, pool, nthr)
            assert all(np.array_equal(g, wv) for g, wv in zip(got, want)), \
                "threaded port differs from the serial oracle"
            trial = []
            t_end = time.perf_counter() + min(0.5, seconds / (2 * len(cands)))
            while time.perf_counter() < t_end or len(trial) < 2:
                t0 = time.perf_counter()
                cpu_port_step(ospec, cspec, xbs, routes, ws, outs, mo, pool, nthr)
                trial.append(time.perf_counter() - t0)
        if best is None or statistics.median(trial) < best[1]:
            best = (nthr, statistics.median(trial))
    nthr = best[0]
    with ThreadPoolExecutor(nthr) as pool:
        times = []
        t_end = time.perf_counter() + seconds
        while time.perf_counter() < t_end or len(times) < 3:
            t0 = time.perf_counter()
            cpu_port_step(ospec, cspec, xbs, routes, ws, outs, mo, pool, nthr)
            times.append((time.perf_counter() - t0) * 1e6)
    v = statistics.median(times) * tokens / sample
    what = (f"{len(times)} full EP={N} steps ({N} ranks on the host)" if sample == tokens else
            f"{len(times)} EP={N} steps on a {sample}-token slice per rank, scaled x{tokens / sample:g} "
            f"to {tokens} tokens")
    return {"value": round(v, 1), "unit": "us", "cores": nthr, "kind": "port",
            "sample": f"{what} ({wl['name']}, H={H}, E={E}, top-{R}); numpy oracle port "
                      f"(oracle/moe_oracle.py): fp8 encode, regroup, return of given bf16 expert rows, "
                      f"fp32 weighted sum, bf16 out; row chunks on {nthr} threads (fastest of "
                      f"{cands} on {host} host threads), p50"}


# ------------------------------------------------------------ clocks


class Clocks:
    def __init__(self, device: int) -> None:
        self.p = None
        self.path = Path(f"/tmp/txb_clocks_{os.getpid()}.csv")
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(device), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap,clocks.mem", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        sm, mx, mem, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
            try:
                mem.append(float(parts[8]))
            except (IndexError, ValueError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "mem_mhz": statistics.median(mem) if mem else None, "samples": len(sm)}


# ------------------------------------------------------------ GPU arm


def expected_rows(wl: dict, rank: int, n: int, tokens: int) -> dict:
    """Row counts of this rank for the synthetic inputs (for the bytes)."""
    E = wl["experts"]
    L = E // n
    all_routes = [_inputs(wl, q, tokens)[1] for q in range(n)]
    dest = all_routes[rank] // L
    counts = np.zeros(L, np.int64)
    for r in all_routes:
        e = r.ravel()
        counts += np.bincount(e[e // L == rank] - rank * L, minlength=L)
    return {"out_rows": int((dest != rank).sum()), "self_rows": int((dest == rank).sum()),
            "in_rows": int(sum(((r // L) == rank).sum() for q, r in enumerate(all_routes) if q != rank)),
            "valid_rows": int(counts.sum()), "pad_rows": int(((-counts) % 8).sum())}


def _max_over_ranks(arr, world: int):
    if world == 1:
        return np.asarray(arr)
    import torch
    import torch.distributed as dist
    t = torch.tensor(np.asarray(arr, dtype=np.float64))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.numpy()


def run_b200(a) -> None:
    import torch
    wl = dict(WORKLOADS[a.config])
    world, rank, local = _dist()
    n_gpu = world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2510_27656_b200 import moe
    from paper_2510_27656_b200.engine import NvlinkFabric, TransferEngine

    tokens = a.tokens or wl["tokens"]
    E, R, H = wl["experts"], wl["topk"], wl["hidden"]
    spec = moe.RoutingSpec(ranks=n_gpu, experts=E, max_tokens=tokens, topk=R, hidden=H,
                           elem_size=wl["elem"], scales=wl["scales"], comb_elem_size=2, comb_scales=0)
    priv = moe.PrivateBufferConfig(a.private) if a.private is not None else None
    if world > 1:
        import torch.distributed as dist
        # setup-only plumbing (IPC-handle exchange, barriers, max-over-ranks
        # of the timings); the data path is the txb kernels over NVLink
        dist.init_process_group("gloo")
        eng = TransferEngine(NvlinkFabric(group=dist.group.WORLD), device=local)
        rk = moe.connect_process_group(eng, spec, private=priv)
    else:
        eng = TransferEngine(NvlinkFabric(), device=local)
        rk = moe.build_mesh([eng], spec, private=priv)[0]
    rk.record_stats = False
    x, routes, w = _inputs(wl, rank, tokens)
    xd = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    rd = torch.from_numpy(routes).to(dev)
    wd = torch.from_numpy(w).to(dev)
    G = int(rk._shape.grouped_rows)
    y = torch.randn(G, H, device=dev).to(torch.bfloat16)     # synthetic expert outputs
    flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    class _Flush:
        """L2 flush between timed steps: write a 512 MiB buffer (4x the L2),
        then (default) read it back, so the step starts with a cold L2 that
        holds no dirty lines: what a GEMM between MoE layers leaves behind
        (it streams weights in).  --flush write keeps the
        write-only flush, whose dirty lines the step then pays to write
        back; both numbers are reported."""

        def __init__(self, mode: str) -> None:
            self.mode = mode

        def fill_(self, v: int) -> None:
            flush_buf.fill_(v)
            if self.mode == "write+read":
                flush_buf.view(torch.int32).amax()

    flush = _Flush(a.flush)

    def mark(name: str) -> None:
        """TXB_BENCH_TRACE=1: sync and name the phase (device printf of a
        checked build lands between the marks)."""
        if os.environ.get("TXB_BENCH_TRACE"):
            torch.cuda.synchronize()
            print(f"[mark] rank {rank} {name} err={rk.status()[0]:#x}", flush=True)

    stream = torch.cuda.Stream(dev)          # graphs capture on a non-default stream
    torch.cuda.set_stream(stream)

    def step():
        rk.dispatch_send(xd, rd, sync=False)
        rk.dispatch_recv(sync=False)
        rk.combine_send(y)
        return rk.combine_recv(wd, out_dtype=torch.bfloat16, sync=False)

    for _ in range(max(3, a.warmup)):
        step()
    torch.cuda.synchronize()
    err, _ = rk.status()
    assert err == 0, f"device error word {err:#x} during warm-up"
    mark("warm-up")

    # The step is launch-only and keeps all per-step state on the device
    # (step counter, counter targets), so it is captured once into a CUDA
    # graph and replayed.  CUDA events recorded INSIDE the graph (external
    # event nodes) bracket the step on the device: the span is the step's
    # device time, as it is when the step is a node of a model's graph,
    # without the ~5 us a graph launch adds at its head.  Events around the
    # replay (launch included) are reported beside it.  Three event nodes
    # split the span into the two kernels.
    ein = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(3)]
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        ein[0].record(stream)
        step()
        ein[2].record(stream)
    # the per-kernel split comes from a second graph with an event node
    # between the kernels (an event node there delays the combine's launch,
    # so the headline graph has none)
    graph_k = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph_k, stream=stream):
        ein[0].record(stream)
        rk.dispatch_send(xd, rd, sync=False)
        rk.dispatch_recv(sync=False)
        ein[1].record(stream)
        rk.combine_send(y)
        rk.combine_recv(wd, out_dtype=torch.bfloat16, sync=False)
        ein[2].record(stream)
    for _ in range(max(3, a.warmup)):
        graph.replay()
        graph_k.replay()
    torch.cuda.synchronize()
    mark("graph warm-up")

    # -------- timed: L2 flush + barrier outside the span, one step at a time
    K = a.steps
    eo = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    clocks = Clocks(local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()

    def run(n_steps: int, flushed: bool, g) -> tuple:
        tin, tout, kd, kc = [], [], [], []
        for k in range(n_steps):
            if flushed:
                flush.fill_(k & 0xFF)
            if world > 1:
                rk.barrier()
            eo[0].record(stream)
            g.replay()
            eo[1].record(stream)
            torch.cuda.synchronize()
            tin.append(ein[0].elapsed_time(ein[2]) * 1e3)
            tout.append(eo[0].elapsed_time(eo[1]) * 1e3)
            if g is graph_k:
                kd.append(ein[0].elapsed_time(ein[1]) * 1e3)
                kc.append(ein[1].elapsed_time(ein[2]) * 1e3)
        return tuple(_max_over_ranks(v, world) for v in (tin, tout, kd, kc))

    tot, tot_launch = run(K, True, graph)[:2]
    other = "write" if a.flush == "write+read" else "write+read"
    flush.mode = other
    mark("flushed")
    tot_other = run(max(20, K // 2), True, graph)[0]
    flush.mode = a.flush
    mark("flushed other")

    # the same step launched eagerly (no graph): the L2 flush keeps the GPU
    # busy while the host enqueues the step, so the event span is device
    # time with stream launch latencies instead of graph-node latencies
    def run_eager(n_steps: int) -> np.ndarray:
        t = []
        for k in range(n_steps + 3):
            flush.fill_(k & 0xFF)
            if world > 1:
                rk.barrier()
            eo[0].record(stream)
            step()
            eo[1].record(stream)
            torch.cuda.synchronize()
            if k >= 3:
                t.append(eo[0].elapsed_time(eo[1]) * 1e3)
        return _max_over_ranks(t, world)

    eager = run_eager(max(20, K // 2))
    mark("eager")


    # back-to-back steps: B steps per graph, step i on input set i % S of a
    # pool whose touched bytes (activations + expert rows) are twice the L2,
    # so every step starts on cold inputs with no flush between steps
    # (contract: "use inputs larger than L2"); events around each replay
    # (host ahead of the GPU), per-step time = span / B, max over ranks
    per_set = tokens * H * 2 + tokens * R * H * 2
    S = int(min(16, max(2, -(-2 * (126 << 20) // per_set))))
    B = max(d for d in range(1, 26) if K % d == 0)
    pool = []
    for si in range(S):
        xs, rs, ws = _inputs(wl, rank, tokens, seed=1 + si)
        pool.append((torch.from_numpy(xs).to(dev).to(torch.bfloat16), torch.from_numpy(rs).to(dev),
                     torch.from_numpy(ws).to(dev), torch.randn(G, H, device=dev).to(torch.bfloat16)))

    def pool_step(i: int):
        xs, rs, ws, ys = pool[i % S]
        rk.dispatch_send(xs, rs, sync=False)
        rk.dispatch_recv(sync=False)
        rk.combine_send(ys)
        return rk.combine_recv(ws, out_dtype=torch.bfloat16, sync=False)

    for i in range(S):
        pool_step(i)
    torch.cuda.synchronize()
    mark("pool eager")
    graph_b = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph_b, stream=stream):
        for i in range(B):
            pool_step(i)
    graph_b.replay()
    torch.cuda.synchronize()
    blocks = []
    for rep in range(K // B):
        if world > 1:
            rk.barrier()
        torch.cuda._sleep(40000)                 # the host enqueues the replay meanwhile
        eo[0].record(stream)
        graph_b.replay()
        eo[1].record(stream)
        torch.cuda.synchronize()
        blocks.append(eo[0].elapsed_time(eo[1]) * 1e3 / B)
    block = _max_over_ranks(blocks, world)
    mark("back to back")

    # kernel span on the device clock: first dispatch CTA start -> last
    # combine CTA end (%globaltimer phase stamps, one graph with stamps on)
    from paper_2510_27656_b200 import _lib as _l
    prof = torch.zeros(_l.TXB_MAX_CTAS * 32, dtype=torch.int64, device=dev)
    rk._bufs.prof = prof.data_ptr()
    graph_p = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph_p, stream=stream):
        step()
    rk._bufs.prof = 0
    spans, kd_span, kc_span = [], [], []
    for k in range(max(20, K // 2) + 3):
        flush.fill_(k & 0xFF)
        if world > 1:
            rk.barrier()
        prof.zero_()
        graph_p.replay()
        torch.cuda.synchronize()
        if k >= 3:
            pv = prof.view(-1, 32).cpu().numpy()
            st0 = pv[:, 0][pv[:, 0] > 0]
            en = pv[:, 13][pv[:, 13] > 0]
            spans.append((en.max() - st0.min()) / 1e3 if st0.size and en.size else float("nan"))
            d_end, c0 = pv[:, 8][pv[:, 8] > 0], pv[:, 9][pv[:, 9] > 0]
            kd_span.append((d_end.max() - st0.min()) / 1e3 if st0.size and d_end.size else float("nan"))
            kc_span.append((en.max() - c0.min()) / 1e3 if c0.size and en.size else float("nan"))
    kspan = _max_over_ranks(spans, world)
    kd_span = _max_over_ranks(kd_span, world)
    kc_span = _max_over_ranks(kc_span, world)
    mark("stamped")
    # L2-warm steps (no flush between; SURVEY.md §8d asks for both numbers)
    b2b = run(max(20, K // 2), False, graph)[0]
    mark("b2b")
    kdisp = run(max(20, K // 2), True, graph_k)[2]
    mark("split")
    clk = clocks.stop()
    err, _ = rk.status()
    assert err == 0, f"device error word {err:#x}"
    names = ["dispatch", "combine"]
    # dispatch: event node -> dispatch kernel -> event node (its launch inside
    # the graph included); combine: the rest of the step (the event node
    # between the kernels would delay the combine's launch and inflate it)
    kt = {"dispatch": float(np.median(kdisp))}
    kt["combine"] = max(0.0, float(np.median(tot)) - kt["dispatch"])

    # -------- e2e through the public API with pinned host buffers
    e2e = e2e_times(rk, x, routes, w, stream, flush, dev, K, world)
    mark("e2e")

    # -------- bytes / roofline
    ex = expected_rows(wl, rank, n_gpu, tokens)
    P, Pc = spec.payload_bytes, spec.comb_payload_bytes
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    nvl_peak = 770.0
    # algorithmic bytes per launch: EP=1 moves everything
    # through HBM; EP>1 is bounded by the larger of NVLink egress/ingress
    if n_gpu == 1:
        # dispatch reads n*H*in_elem and writes n*R*P;
        # combine reads n*R*Pc and writes n*H*out_elem (padding rows are
        # not algorithmic: they are re-zeroed only when dirty)
        bytes_k = {"dispatch": tokens * H * 2 + tokens * R * P,
                   "combine": tokens * R * Pc + tokens * H * 2}
        bound = "hbm"
    else:
        bytes_k = {"dispatch": max(ex["out_rows"], ex["in_rows"]) * P,
                   "combine": max(ex["valid_rows"] - ex["self_rows"], ex["out_rows"]) * Pc}
        bound = "nvlink"
    dom = max(names, key=lambda k: kt[k])
    kname = {"dispatch": "k_dispatch_roles" if tokens <= 148 and wl["elem"] == 1 else "k_dispatch_fused",
             "combine": "k_combine_fused"}
    # DRAM bytes per launch of that kernel from the committed ncu capture
    # (EP=1 decode only; profiles/r01_ncu_traffic.json)
    traffic = None
    tf = ROOT / "profiles" / "r02" / "ncu_traffic.json"
    if n_gpu == 1 and a.config in ("decode", "prefill") and tf.exists():
        tj = json.loads(tf.read_text())
        t = (tj if a.config == "decode" else tj.get(a.config, {})).get(kname[dom])
        if t:
            traffic = int(t["dram_read"] + t["dram_write"])
    traffic_src = "ncu dram__bytes_read.sum + dram__bytes_write.sum (profiles/r02/ncu_traffic.json)"
    nf = ROOT / "profiles" / "r01_nvlink" / "summary.json"
    if n_gpu == 2 and nf.exists():
        # NVLink bytes on the wire per launch at EP=2, from the ncu capture of
        # the host-gated split kernels that move the same rows
        t = json.loads(nf.read_text()).get(a.config, {}).get(dom)
        if t:
            traffic = int(t["nvltx_wire"])
            traffic_src = (f"ncu nvltx__bytes.sum (wire) of {t['kernel']} at EP=2 (profiles/r01_nvlink); "
                           f"user data {t['nvltx_user']} B")
    peak = hbm_peak if bound == "hbm" else nvl_peak
    achieved = bytes_k[dom] / (kt[dom] * 1e-6) / 1e9
    span_k = {"dispatch": float(np.nanmedian(kd_span)), "combine": float(np.nanmedian(kc_span))}
    roofline = {"bound": bound, "kernel": kname[dom],
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "traffic_source": traffic_src if traffic is not None else None,
                "peak_source": ("MEASURED_PEAKS.json hbm_gbs (burst copy)" if bound == "hbm"
                                else "B200_PROFILING.md measured peer copy 770 GB/s (fallback)"),
                "algorithmic_bytes": int(bytes_k[dom]), "kernel_us": round(kt[dom], 2),
                # the same kernel's duration on the device clock (first CTA start -> last CTA end,
                # %globaltimer phase stamps), free of the event node between the two kernels
                "kernel_span_us": round(span_k[dom], 2),
                "frac_on_span": round(bytes_k[dom] / (span_k[dom] * 1e-6) / 1e9 / peak, 4),
                "all_kernels": {k: {"bytes": int(bytes_k[k]), "us": round(kt[k], 2),
                                    "gbs": round(bytes_k[k] / (kt[k] * 1e-6) / 1e9, 1)} for k in names}}
    if bound == "hbm" and dom == "dispatch":
        # the dispatch writes R rows per row it reads: its ceiling is the
        # HBM's write bandwidth, measured here (512 MiB fill, best of 5)
        wts = []
        for _ in range(7):
            w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            w0.record(stream)
            flush_buf.fill_(3)
            w1.record(stream)
            torch.cuda.synchronize()
            wts.append(w0.elapsed_time(w1))
        wpeak = flush_buf.numel() / (min(wts[2:]) * 1e-3) / 1e9
        wbytes = tokens * R * P
        roofline["write_share"] = round(wbytes / bytes_k[dom], 3)
        roofline["write_fill_gbs"] = round(wpeak, 1)
        roofline["frac_of_write_fill"] = round(achieved / wpeak, 4)
        roofline["frac_of_write_fill_on_span"] = round(bytes_k[dom] / (span_k[dom] * 1e-6) / 1e9 / wpeak, 4)
        roofline["write_fill_note"] = ("write-only HBM stream measured in this run (512 MiB fill_, best of 5): "
                                       "the nearest ceiling for a kernel whose bytes are mostly row writes "
                                       "(a mix with some reads can exceed it slightly); frac stays against "
                                       "the copy peak")
    # headline: K back-to-back steps timed in blocks of B with inputs cycled
    # through a pool twice the L2 (the contract's "inputs larger than L2"),
    # so no per-step event node or flush artefact sits inside the number;
    # the flushed single-step p50 is reported beside it
    p50 = float(np.median(block))
    res = {
        "metric": wl["metric"], "value": round(p50, 2), "unit": "us",
        "n_gpus": n_gpu, "steps": K, "warmup": a.warmup, "ms_per_step": round(p50 / 1e3, 5),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": ("fp8-e4m3" if wl["elem"] == 1 else "bf16") + " dispatch / bf16 combine (fp32 accumulate)",
        "data": "synthetic",
        "config": workload_config(wl, tokens, n_gpu, rk.private_tokens),
        "l2": (f"inputs larger than L2: {S} input sets (activations, routes, weights, expert rows) of "
               f"{per_set / 1e6:.1f} MB touched per step, cycled step by step (no flush between the "
               f"timed steps); the flushed single-step numbers flush with a 512 MiB "
               + ("write then read" if a.flush == "write+read" else "write")),
        "timing": f"public-API steps captured as CUDA graphs of {B} back-to-back steps; CUDA events "
                  f"around each replay on the step stream (host ahead of the GPU), per-step time = span / "
                  f"{B}; device barrier + synchronize before each block; p50 over the {K // B} blocks of "
                  f"the max over ranks",
        "p50_flushed_step_us": round(float(np.median(tot)), 2),
        "flushed_step_timing": "one step per graph replay after the L2 flush (+ device barrier for N>1), CUDA "
                               "event nodes inside the graph around the step; p50 over steps of the max over ranks",
        f"p50_flushed_step_{other.replace('+', '_')}_flush_us": round(float(np.median(tot_other)), 2),
        "p90_flushed_step_us": round(float(np.percentile(tot, 90)), 2),
        "p99_flushed_step_us": round(float(np.percentile(tot, 99)), 2),
        "p50_l2_warm_us": round(float(np.median(b2b)), 2),
        "p50_with_graph_launch_us": round(float(np.median(tot_launch)), 2),
        "p50_eager_us": round(float(np.median(eager)), 2),
        "back_to_back": {"steps_per_graph": B, "input_sets": S, "bytes_per_set": per_set,
                         "timed_steps": B * (K // B),
                         "p90_us": round(float(np.percentile(block, 90)), 2)},
        "p50_kernel_span_us": round(float(np.nanmedian(kspan)), 2),
        "span_note": "p50_eager_us: events around one eager flushed step with the host ahead of the GPU; "
                     "p50_kernel_span_us: %globaltimer from the first dispatch CTA's start to the last combine "
                     "CTA's end of one flushed step (max over ranks)",
        "tokens_per_s": round(n_gpu * tokens / (p50 * 1e-6), 1),
        "kernel_us": {k: round(v, 2) for k, v in kt.items()},
        "kernel_us_note": "the flushed graph step split by a CUDA event node between the two kernels (the "
                          "node's own cost lands in the dispatch); roofline.kernel_span_us gives the same "
                          "kernel on the device clock",
        "roofline": roofline,
        "e2e": e2e,
        "gpu_launches": 2 * K,
        "clocks": clk,
    }
    if rank == 0 and n_gpu == 1 and not a.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(wl, tokens, a.cpu_seconds)
    if rank == 0:
        print(json.dumps(res), flush=True)
    rk.close()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def e2e_times(rk, x, routes, w, stream, flush, dev, K: int, world: int) -> dict:
    """The step end to end through the public API from page-locked HOST
    buffers: activations (bf16), routes (i64) and weights (f32) come from
    pinned host memory and the combined bf16 rows land in pinned host
    memory inside the timed span.  Three ways a caller can drive it:
      copies  -- eager calls with explicit H2D / D2H copies around them;
      zcopy   -- eager calls on the pinned tensors themselves: the dispatch
                 kernel reads the activations and the combine kernel reads
                 the weights / writes the result over PCIe in place;
      graph   -- the zcopy calls captured once into a CUDA graph and
                 replayed (how a decode loop runs them).
    `value` is the graph variant; all three are reported."""
    import torch
    xh = torch.from_numpy(x).to(torch.bfloat16).pin_memory()
    rh = torch.from_numpy(routes).pin_memory()
    wh = torch.from_numpy(w).pin_memory()
    oh = torch.empty((x.shape[0], x.shape[1]), dtype=torch.bfloat16).pin_memory()
    G = int(rk._shape.grouped_rows)
    y = torch.randn(G, x.shape[1], device=dev).to(torch.bfloat16)

    def step_copies():
        xd = xh.to(dev, non_blocking=True)
        rd = rh.to(dev, non_blocking=True)
        wd = wh.to(dev, non_blocking=True)
        rk.dispatch_send(xd, rd, sync=False)
        rk.dispatch_recv(sync=False)
        rk.combine_send(y)
        out = rk.combine_recv(wd, out_dtype=torch.bfloat16, sync=False)
        oh.copy_(out, non_blocking=True)

    def step_zcopy():
        rk.dispatch_send(xh, rh, sync=False)
        rk.dispatch_recv(sync=False)
        rk.combine_send(y)
        rk.combine_recv(wh, out_dtype=torch.bfloat16, sync=False, out=oh)

    def timed(fn, reps):
        times = []
        for k in range(reps + 5):
            flush.fill_(2)
            if world > 1:
                rk.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            if k >= 5:
                times.append(e0.elapsed_time(e1) * 1e3)
        return float(np.median(_max_over_ranks(times, world)))

    res = {"copies": timed(step_copies, K), "zcopy": timed(step_zcopy, K)}
    want = oh.clone()
    graph = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(graph, stream=stream):
        step_zcopy()
    oh.zero_()
    res["graph"] = timed(graph.replay, K)
    assert torch.equal(oh, want), "graph replay result differs from the eager step"
    err, _ = rk.status()
    assert err == 0, f"device error word {err:#x} in the e2e runs"
    bi = x.shape[0] * x.shape[1] * 2 + routes.size * 8 + w.size * 4
    return {"value": round(res["graph"], 2), "unit": "us",
            "h2d_bytes_per_step": int(bi), "d2h_bytes_per_step": int(x.shape[0] * x.shape[1] * 2),
            "path": "public MoeRank API on pinned host tensors (kernels read inputs / write the result "
                    "over PCIe in place), captured once as a CUDA graph and replayed; events around "
                    "each replay, L2 flushed between steps",
            "variants_us": {k: round(v, 2) for k, v in res.items()}}


# ------------------------------------------------------------ reference arm


def reference_live(wl: dict, tokens: int, steps: int = 3, ranks: int = 1, private: int | None = None) -> dict:
    """The unmodified reference (railtx, installed into baseline/_ref with
    pip --no-deps; pure Python + numpy + numba) run through its own public
    API on the host: per rank encode_tokens -> MoeRank.dispatch_send ->
    dispatch_recv -> combine_send (identity expert) -> combine_recv, all
    `ranks` ranks in one process over a SimFabric with one thread per rank
    (its test harness's model, moe.py:470-833, _invariants.py:254-292).
    Its payloads are fp8 or f32 (elem_size 2 does not exist there), so a
    bf16 workload runs as f32.  Bounded sample: at most 512 tokens per rank,
    scaled linearly to the step."""
    import threading
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "railtx").is_dir():
        return {"unavailable": "baseline/_ref/railtx not installed (see DESIGN.md section 9)"}
    sys.path.insert(0, str(ref))
    try:
        from railtx import FaultConfig, SimFabric, TransferEngine
        from railtx import moe as rmoe
    except Exception as exc:  # numba or numpy missing on this host
        return {"unavailable": f"railtx import failed: {exc!r}"[:200]}
    sample = min(tokens, 512)
    elem, scales = (1, wl["scales"]) if wl["elem"] == 1 else (4, 0)
    N = ranks
    spec = rmoe.RoutingSpec(ranks=N, experts=wl["experts"], max_tokens=sample, topk=wl["topk"],
                            hidden=wl["hidden"], elem_size=elem, scales=scales)
    fab = SimFabric(FaultConfig(mtu=1 << 20))
    engs = [TransferEngine(fab, rails=1, name=f"ref{r}") for r in range(N)]
    pv = None if private is None else rmoe.PrivateBufferConfig(min(private, sample))
    mesh = rmoe.build_mesh(engs, spec, private=pv, ranks_per_node=N)
    ins = [_inputs(wl, r, sample) for r in range(N)]
    errs: list = []

    def rank_step(r: int) -> None:
        try:
            x, routes, w = ins[r]
            rk = mesh[r]
            rk.dispatch_send(rmoe.encode_tokens(spec, x), routes)
            g = rk.dispatch_recv(300.0)
            rk.combine_send(g.data)
            rk.combine_recv(w, 300.0)
        except Exception as exc:  # surfaced below
            errs.append(exc)

    times = []
    try:
        for i in range(steps + 2):  # two warm-up steps (numba JIT)
            t0 = time.perf_counter()
            th = [threading.Thread(target=rank_step, args=(r,)) for r in range(N)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            if errs:
                return {"unavailable": f"railtx step failed: {errs[0]!r}"[:200]}
            if i >= 2:
                times.append((time.perf_counter() - t0) * 1e6)
    finally:
        for rk in mesh:
            rk.close()
        for e in engs:
            e.close()
    v = statistics.median(times) * tokens / sample
    return {"value": round(v, 1), "unit": "us", "cores": N, "kind": "reference",
            "sample": f"{len(times)} steps of the unmodified railtx MoeRank API (baseline/_ref), EP={N} "
                      f"({N} rank threads over SimFabric), {sample} tokens per rank"
                      + (f" scaled x{tokens / sample:g}" if sample < tokens else "")
                      + f", {'fp8' if elem == 1 else 'f32'} payloads, identity expert, p50 after 2 warm-up steps"}


def run_reference(a) -> None:
    """The reference's algorithm on the host cores, on this arm's config.
    `value` is the oracle port of it with every host thread (the faster,
    conservative CPU baseline); the unmodified reference from
    baseline/_ref, run through its own API, is timed beside it
    (`reference_live`).  Rank 0 only; other ranks exit without work."""
    world, rank, _ = _dist()
    if rank != 0:
        return
    wl = WORKLOADS[a.config]
    tokens = a.tokens or wl["tokens"]
    N = max(world, a.gpus)  # the reference runs all N ranks of an EP=N step on the host
    cb = cpu_baseline(wl, tokens, max(2.0, min(a.cpu_seconds, 30.0)), ranks=N)
    res = {"impl": "reference", "metric": wl["metric"], "value": cb["value"], "unit": "us",
           "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "higher_is_better": False,
           "scaling": "weak", "vs_baseline": None,
           "dtype": ("fp8-e4m3" if wl["elem"] == 1 else "bf16") + " dispatch / bf16 combine (fp32 accumulate)",
           "data": "synthetic",
           "config": workload_config(wl, tokens, N, a.private),
           "cpu_baseline": cb,
           "e2e": {"value": cb["value"], "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "reference_live": reference_live(wl, tokens, ranks=N, private=a.private),
           "note": "value: the threaded oracle port of railtx's algorithm (oracle/moe_oracle.py) on the host "
                   "cores; reference_live: the unmodified railtx API from baseline/_ref, one thread per rank"}
    print(json.dumps(res), flush=True)


def main() -> None:
    a = _args()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_b200(a)


if __name__ == "__main__":
    main()
