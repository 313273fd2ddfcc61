"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [--ref /root/reference]

It imports railtx from <ref>/pkg/src and the reference's own test helpers
from <ref>/pkg/tests (random_step, run_moe_round, expert_fn), drives whole
dispatch/combine rounds over the reference SimFabric, and stores inputs and
outputs as small .npz fixtures next to this script.  The GPU box never reads
/root/reference: tests there use only the committed fixtures.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

# (name, RoutingSpec kwargs, steps, seed, fixed token count or None, fabric mode, private)
MOE_CASES = [
    ("cfg1_full", dict(ranks=2, experts=8, max_tokens=16, topk=2, hidden=1024,
                       elem_size=4, scales=0), 1, 7, 16, "inorder", None),
    ("cfg1_rand", dict(ranks=2, experts=8, max_tokens=16, topk=2, hidden=1024,
                       elem_size=4, scales=0), 1, 11, None, "reverse", None),
    ("check_moe", dict(ranks=2, experts=4, max_tokens=4, topk=2, hidden=8,
                       elem_size=4, scales=0), 3, 105, None, "window", 2),
    ("n4_e16_t9_r4", dict(ranks=4, experts=16, max_tokens=9, topk=4, hidden=16,
                          elem_size=4, scales=0), 2, 21, None, "reverse", 0),
    ("n4_e8_t5_r1", dict(ranks=4, experts=8, max_tokens=5, topk=1, hidden=16,
                         elem_size=4, scales=0), 2, 22, None, "inorder", 5),
    ("n8_e16_t7_r3", dict(ranks=8, experts=16, max_tokens=7, topk=3, hidden=16,
                          elem_size=4, scales=0), 2, 23, None, "mtu4k", 2),
    ("n3_e12_t11_r4", dict(ranks=3, experts=12, max_tokens=11, topk=4, hidden=16,
                           elem_size=4, scales=0), 2, 24, None, "window", 3),
    ("n1_e8_t16_r4", dict(ranks=1, experts=8, max_tokens=16, topk=4, hidden=64,
                          elem_size=4, scales=0), 2, 25, None, "inorder", None),
    ("fp8_n2_h256", dict(ranks=2, experts=8, max_tokens=16, topk=2, hidden=256,
                         elem_size=1, scales=8), 2, 31, None, "reverse", None),
    ("fp8_n4_h64_s1", dict(ranks=4, experts=16, max_tokens=8, topk=4, hidden=64,
                           elem_size=1, scales=1), 2, 32, None, "inorder", 4),
    ("fp8_n2_h33_odd", dict(ranks=2, experts=4, max_tokens=6, topk=2, hidden=33,
                            elem_size=1, scales=1), 2, 33, None, "window", 3),
    ("fp8_dsv3ish", dict(ranks=8, experts=256, max_tokens=8, topk=8, hidden=128,
                         elem_size=1, scales=56), 1, 34, 8, "inorder", None),
    ("empty", dict(ranks=2, experts=8, max_tokens=4, topk=2, hidden=16,
                   elem_size=4, scales=0), 1, 35, 0, "inorder", None),
]


def _import_ref(ref: Path):
    sys.path.insert(0, str(ref / "pkg" / "src"))
    sys.path.insert(0, str(ref / "pkg" / "tests"))
    import railtx  # noqa: F401
    from railtx import kernels, moe
    import _fabric
    import _invariants
    return moe, kernels, _fabric, _invariants


def make_moe(ref: Path) -> None:
    moe, kernels, fab, inv = _import_ref(ref)
    for name, kw, steps, seed, tokens, mode, priv in MOE_CASES:
        spec = moe.RoutingSpec(**kw)
        cfg = fab.mode_config(mode, 1)
        rng = np.random.default_rng(seed)
        blob: dict[str, np.ndarray] = {
            "spec": np.array([spec.ranks, spec.experts, spec.max_tokens, spec.topk,
                              spec.hidden, spec.elem_size, spec.scales], np.int64),
            "steps": np.array(steps),
        }
        with fab.engines(cfg, spec.ranks, rails=2, prefix="g") as es:
            private = None if priv is None else moe.PrivateBufferConfig(priv)
            mesh = moe.build_mesh(es, spec, private=private, ranks_per_node=1)
            cap_pos: dict[int, np.ndarray] = {}
            cap_out: dict[int, np.ndarray] = {}
            for rk in mesh:
                orig_stage = rk._stage
                orig_cs = rk.combine_send

                def _stage(st, p, r, rk=rk, orig=orig_stage):
                    orig(st, p, r)
                    cap_pos[rk.rank] = st.pos.copy()

                def _cs(outputs, rk=rk, orig=orig_cs):
                    cap_out[rk.rank] = np.array(outputs, dtype=np.uint8, copy=True)
                    return orig(outputs)
                rk._stage = _stage
                rk.combine_send = _cs
            try:
                for k in range(steps):
                    routes, values, weights = inv.random_step(spec, rng, tokens)
                    results = inv.run_moe_round(mesh, spec, routes, values, weights)
                    if spec.elem_size == 4:
                        inv.verify_moe_round(spec, results, routes, values, weights)
                    for r in range(spec.ranks):
                        pre = f"s{k}_r{r}_"
                        g, comb = results[r]
                        lay = mesh[r].last_layout
                        blob[pre + "routes"] = routes[r]
                        blob[pre + "values"] = values[r]
                        blob[pre + "weights"] = weights[r]
                        blob[pre + "payload"] = moe.encode_tokens(spec, values[r])
                        blob[pre + "pos"] = cap_pos[r]
                        blob[pre + "data"] = g.data
                        blob[pre + "group_sizes"] = g.group_sizes
                        blob[pre + "group_starts"] = g.group_starts
                        blob[pre + "rows"] = g.rows
                        blob[pre + "sources"] = g.sources
                        blob[pre + "outputs"] = cap_out[r]
                        blob[pre + "combined"] = comb
                        if lay is not None:
                            blob[f"s{k}_counts"] = lay.counts
                            blob[f"s{k}_assigned"] = lay.assigned
                            blob[f"s{k}_recv_start"] = lay.recv_start
                            blob[f"s{k}_recv_total"] = lay.recv_total
                            blob[f"s{k}_send_start"] = lay.send_start
            finally:
                for rk in mesh:
                    rk.close()
        np.savez_compressed(HERE / f"moe_{name}.npz", **blob)
        print(f"moe_{name}.npz", sum(v.nbytes for v in blob.values()), "bytes raw")


def make_codecs(ref: Path) -> None:
    moe, kernels, _, _ = _import_ref(ref)
    rng = np.random.default_rng(1234)
    mags = np.concatenate([kernels._FP8_MAGS, kernels._FP8_MIDS,
                           np.nextafter(kernels._FP8_MIDS, 0), np.nextafter(kernels._FP8_MIDS, 1e9)])
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, -np.nan, 448.0, 449.0, 464.0,
                        465.0, 480.0, 1e30, -1e30, 2.0 ** -9, 2.0 ** -10, 2.0 ** -11,
                        3 * 2.0 ** -11, 1e-45, -1e-45], np.float64)
    x = np.concatenate([mags, -mags, special, rng.standard_normal(20000) * 50,
                        rng.standard_normal(5000) * 1e-3]).astype(np.float32)
    fp8 = kernels.fp8_encode_nb(x.astype(np.float64))
    assert np.array_equal(fp8, kernels.fp8_encode_np(x.astype(np.float64)))
    bf_in = np.concatenate([x, np.array([np.float32(1.0) + np.float32(2 ** -8)], np.float32),
                            np.frombuffer(np.array([0x7F800001, 0xFF800001, 0x7FFFFFFF,
                                                    0x3F808000, 0x3F818000, 0x7F7FFFFF],
                                                   np.uint32).tobytes(), np.float32)])
    bf = kernels.bf16_encode(bf_in)
    # rows for per-token quantisation edge cases
    rows = rng.standard_normal((12, 96)).astype(np.float32)
    rows[1] = 0.0
    rows[2, 5] = np.nan
    rows[3, 7] = np.inf
    rows[4, :] = np.nan
    rows[5] *= 1e-30
    rows[6] *= 1e30
    rows[7, 0] = -np.inf
    rows[8] = -0.0
    rows[9, 3] = 1e38
    rows[10] = np.float32(448.0)
    rows[11] = np.float32(-1e-40)
    spec = moe.RoutingSpec(ranks=1, experts=1, max_tokens=12, topk=1, hidden=96,
                           elem_size=1, scales=3)
    enc = moe.encode_tokens(spec, rows)
    dec = moe.decode_tokens(spec, enc)
    np.savez_compressed(HERE / "codecs.npz", fp8_in=x, fp8_out=fp8, bf16_in=bf_in,
                        bf16_out=bf, rows=rows, rows_enc=enc, rows_dec=dec,
                        fp8_table=kernels.FP8_DECODE)
    print("codecs.npz")


def make_weights(ref: Path) -> None:
    """weights.prepare outputs for the reference's small topology and a
    larger fp8 tensor (per-tensor quantisation incl. NaN/inf/zero words)."""
    _import_ref(ref)
    import struct
    from railtx import kernels
    from railtx.weights import build_schedule, fill_store, prepare
    import _invariants as inv
    train, infer = inv.small_topology()
    sched = build_schedule(train, infer)
    store = fill_store(train, 7)
    blob: dict[str, np.ndarray] = {}
    for k, t in enumerate(sched.tasks):
        full = np.concatenate([store.get(t.sources[0], i) for i in range(64)
                               if (t.sources[0], i) in store._data], axis=t.axis)
        width = t.full_shape[t.axis] // t.shard_count
        sl = [slice(None)] * len(t.full_shape)
        sl[t.axis] = slice(t.shard_index * width, (t.shard_index + 1) * width)
        words = np.ascontiguousarray(full[tuple(sl)]).reshape(-1)
        blob[f"t{k}_words"] = words
        blob[f"t{k}_dtype"] = np.array([0 if t.dtype == "bf16" else 1])
        blob[f"t{k}_prepared"] = np.frombuffer(prepare(t, store), np.uint8)
    rng = np.random.default_rng(77)
    x = (rng.standard_normal(1 << 16) * 3).astype(np.float32)
    x[5], x[6], x[7], x[8] = np.nan, np.inf, -np.inf, 0.0
    w = kernels.bf16_encode(x)
    q, scale = kernels.fp8_quantize(kernels.bf16_decode(w))
    blob["big_words"] = w
    blob["big_prepared"] = np.frombuffer(q.tobytes() + struct.pack("<f", scale), np.uint8)
    blob["ntasks"] = np.array([len(sched.tasks)])
    np.savez_compressed(HERE / "weights.npz", **blob)
    print("weights.npz", len(sched.tasks), "tasks")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference")
    a = ap.parse_args()
    ref = Path(a.ref)
    make_codecs(ref)
    make_weights(ref)
    make_moe(ref)


if __name__ == "__main__":
    main()
