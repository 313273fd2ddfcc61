"""Round drivers for the GPU parity tests.

`run_moe_round` mirrors the reference harness (tests/_invariants.py:254-292):
one Python thread per rank, numpy in and out, expert outputs formed by
decode -> expert_fn -> encode per local expert.  The codecs come from the
CPU oracle here (the checker), so the only thing under test is the device
path between the numpy inputs and the numpy outputs.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from oracle import moe_oracle as mo
from paper_2510_27656_b200 import moe
from paper_2510_27656_b200.engine import local_engines


def ospec_of(spec: moe.RoutingSpec) -> mo.Spec:
    return mo.Spec(spec.ranks, spec.experts, spec.max_tokens, spec.topk, spec.hidden,
                   spec.elem_size, spec.scales)


def devices_for(n: int) -> list[int]:
    """Distinct GPUs when the box has enough, else every rank on cuda:0
    (host-gated single-device emulation)."""
    count = torch.cuda.device_count()
    return list(range(n)) if count >= n else [0] * n


def make_mesh(spec: moe.RoutingSpec, private: int | None = None, timeout: float = 30.0, trace: bool = False):
    engines = local_engines(devices_for(spec.ranks), trace=trace)
    pv = None if private is None else moe.PrivateBufferConfig(private)
    return moe.build_mesh(engines, spec, private=pv, timeout=timeout)


def run_moe_round(mesh, spec: moe.RoutingSpec, routes, values, weights, timeout: float = 30.0):
    os_ = ospec_of(spec)
    results: list = [None] * spec.ranks
    errors: list = []

    def worker(r: int) -> None:
        try:
            torch.cuda.set_device(mesh[r].device)
            rank = mesh[r]
            rank.dispatch_send(mo.encode_tokens(os_, values[r]), routes[r])
            grouped = rank.dispatch_recv(timeout)
            pos = rank.pos.cpu().numpy()
            out = np.zeros_like(grouped.data)
            for le in range(spec.local_experts):
                s = int(grouped.group_starts[le])
                cnt = int(grouped.group_sizes[le])
                if cnt:
                    xs = mo.decode_tokens(os_, grouped.data[s:s + cnt])
                    ys = mo.expert_fn(r * spec.local_experts + le, xs)
                    out[s:s + cnt] = mo.encode_tokens(os_, ys)
            rank.combine_send(out)
            results[r] = (grouped, rank.combine_recv(weights[r], timeout), pos)
        except Exception as exc:  # surfaced below, like the reference driver
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(spec.ranks)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout + 30.0)
    if errors:
        raise errors[0]
    assert all(r is not None for r in results), "a rank never finished"
    return results


def close_mesh(mesh) -> None:
    for m in mesh:
        m.close()


def device_round(mesh, spec: moe.RoutingSpec, routes, values, weights, timeout: float = 30.0,
                 out_dtype=torch.bfloat16):
    """One device-mode step on every rank (one thread per rank): bf16 values
    encoded inside the dispatch kernel; expert = 0.5 * decoded rows in the
    combine wire format (bf16 rows when comb_elem_size is 2, else the
    dispatch rows themselves).  Returns per rank (grouped data, rows,
    sources, pos, expert rows as wire bytes, combined output) as numpy."""
    ranks = spec.ranks
    xb = [torch.from_numpy(np.ascontiguousarray(v)).to(torch.bfloat16) for v in values]
    got: list = [None] * ranks
    errs: list = []
    ce, _ = spec.comb_format

    def worker(r: int) -> None:
        try:
            rk = mesh[r]
            dev = torch.device("cuda", rk.device)
            torch.cuda.set_device(dev)
            rk.dispatch_send(xb[r].to(dev), torch.from_numpy(np.ascontiguousarray(routes[r])).to(dev))
            g = rk.dispatch_recv(timeout)
            pos = rk.pos.cpu().numpy()
            if ce == 2:
                y = (moe.decode_tokens(spec, g.data) * 0.5).to(torch.bfloat16)
                ywire = y.view(torch.uint8).reshape(y.shape[0], -1)
            else:
                y = g.data.clone()
                ywire = y
            rk.combine_send(y)
            out = rk.combine_recv(torch.from_numpy(np.ascontiguousarray(weights[r])).to(dev), timeout,
                                  out_dtype=out_dtype)
            got[r] = (g.data.cpu().numpy(), g.rows.cpu().numpy(), g.sources.cpu().numpy(), pos,
                      ywire.cpu().numpy(), out.cpu())
        except Exception as exc:  # surfaced below
            errs.append(exc)

    threads = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(ranks)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout + 60.0)
    if errs:
        raise errs[0]
    assert all(g is not None for g in got), "a rank never finished"
    return xb, got


def check_device_round(spec: moe.RoutingSpec, routes, xb, weights, got, what: str = "") -> None:
    """Bit-exact check of a device_round against the CPU oracle: grouped
    payloads (incl. zero padding), rows, sources, pos, and the combine (fp32
    bits, or bf16 bits of the fp32 oracle sum rounded RNE)."""
    os_ = ospec_of(spec)
    ce, cs = spec.comb_format
    comb_spec = mo.Spec(spec.ranks, spec.experts, spec.max_tokens, spec.topk, spec.hidden, ce, cs)
    ref = mo.dispatch(os_, [np.asarray(r) for r in routes],
                      [mo.encode_tokens(os_, x.float().numpy()) for x in xb])
    for r in range(spec.ranks):
        data, rows, srcs, pos, _, _ = got[r]
        want = ref.ranks[r].grouped
        assert np.array_equal(data, want.data), f"{what} rank {r}: grouped data"
        assert np.array_equal(rows, want.rows), f"{what} rank {r}: rows"
        assert np.array_equal(srcs, want.sources), f"{what} rank {r}: sources"
        assert np.array_equal(pos.reshape(-1), ref.ranks[r].pos.reshape(-1)), f"{what} rank {r}: pos"
    outs = [got[r][4] for r in range(spec.ranks)]
    comb = mo.combine(os_, ref, outs, [np.asarray(w, np.float32) for w in weights], comb_spec=comb_spec)
    for r in range(spec.ranks):
        out = got[r][5]
        if out.dtype == torch.bfloat16:
            assert np.array_equal(out.view(torch.int16).numpy().view(np.uint16), mo.bf16_encode(comb[r])), \
                f"{what} rank {r}: combine (bf16 bits)"
        else:
            assert np.array_equal(out.numpy(), comb[r]), f"{what} rank {r}: combine (fp32 bits)"
