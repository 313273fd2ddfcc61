"""Load the committed reference golden vectors (tests/golden/*.npz)."""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@dataclass
class GoldenStep:
    routes: list
    values: list
    weights: list
    payload: list
    pos: list
    data: list
    group_sizes: list
    group_starts: list
    rows: list
    sources: list
    outputs: list
    combined: list
    counts: np.ndarray | None


@dataclass
class GoldenCase:
    name: str
    spec_args: dict
    steps: list


def moe_cases() -> list[str]:
    return sorted(p.stem[len("moe_"):] for p in GOLDEN.glob("moe_*.npz"))


def load_moe(name: str) -> GoldenCase:
    z = np.load(GOLDEN / f"moe_{name}.npz")
    n, e, t, r, h, el, sc = (int(v) for v in z["spec"])
    args = dict(ranks=n, experts=e, max_tokens=t, topk=r, hidden=h, elem_size=el, scales=sc)
    steps = []
    for k in range(int(z["steps"])):
        def per(key):
            return [z[f"s{k}_r{q}_{key}"] for q in range(n)]
        steps.append(GoldenStep(
            routes=per("routes"), values=per("values"), weights=per("weights"),
            payload=per("payload"), pos=per("pos"), data=per("data"),
            group_sizes=per("group_sizes"), group_starts=per("group_starts"),
            rows=per("rows"), sources=per("sources"), outputs=per("outputs"),
            combined=per("combined"),
            counts=z[f"s{k}_counts"] if f"s{k}_counts" in z else None))
    return GoldenCase(name, args, steps)


def load_codecs() -> dict:
    z = np.load(GOLDEN / "codecs.npz")
    return {k: z[k] for k in z.files}
