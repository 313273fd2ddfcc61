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
