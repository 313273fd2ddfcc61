"""Pin the CPU oracle against the reference's own outputs (golden vectors).

The fixtures come from running the reference railtx end to end
(tests/golden/make_golden.py).  Everything here is CPU-only.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

from golden_io import load_codecs, load_moe, moe_cases

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import moe_oracle as mo  # noqa: E402


def test_fp8_encode_matches_reference():
    c = load_codecs()
    got = mo.fp8_encode(c["fp8_in"].astype(np.float64))
    assert np.array_equal(got, c["fp8_out"])


def test_fp8_table_matches_reference():
    c = load_codecs()
    assert np.array_equal(mo.FP8_TABLE, c["fp8_table"], equal_nan=True)


def test_bf16_encode_matches_reference():
    c = load_codecs()
    assert np.array_equal(mo.bf16_encode(c["bf16_in"]), c["bf16_out"])


def test_encode_rows_edge_cases():
    c = load_codecs()
    spec = mo.Spec(1, 1, 12, 1, hidden=96, elem_size=1, scales=3)
    enc = mo.encode_tokens(spec, c["rows"])
    assert np.array_equal(enc, c["rows_enc"])
    dec = mo.decode_tokens(spec, enc)
    assert np.array_equal(dec, c["rows_dec"], equal_nan=True)


@pytest.mark.parametrize("name", moe_cases())
def test_moe_round_matches_reference(name):
    case = load_moe(name)
    spec = mo.Spec(**case.spec_args)
    for st in case.steps:
        payloads = [mo.encode_tokens(spec, v) for v in st.values]
        for q in range(spec.ranks):
            assert np.array_equal(payloads[q], st.payload[q])
        res = mo.dispatch(spec, st.routes, payloads)
        if st.counts is not None:
            assert np.array_equal(res.layout.counts, st.counts)
        for q in range(spec.ranks):
            rr = res.ranks[q]
            assert np.array_equal(rr.pos, st.pos[q])
            assert np.array_equal(rr.grouped.group_sizes, st.group_sizes[q])
            assert np.array_equal(rr.grouped.group_starts, st.group_starts[q])
            assert np.array_equal(rr.grouped.rows, st.rows[q])
            assert np.array_equal(rr.grouped.sources, st.sources[q])
            assert np.array_equal(rr.grouped.data, st.data[q])
        outs = mo.apply_experts(spec, res)
        for q in range(spec.ranks):
            assert np.array_equal(outs[q], st.outputs[q])
        comb = mo.combine(spec, res, outs, st.weights)
        for q in range(spec.ranks):
            assert comb[q].shape == st.combined[q].shape
            assert np.array_equal(comb[q], st.combined[q]), f"rank {q}"


def test_check_routes_errors():
    spec = mo.Spec(2, 4, 3, 2, hidden=8, elem_size=4, scales=0)
    with pytest.raises(mo.OracleProtocolError, match="duplicate"):
        mo.check_routes(spec, np.array([[0, 1], [2, 2]]))
    with pytest.raises(mo.OracleProtocolError, match="out of range"):
        mo.check_routes(spec, np.array([[0, 4]]))
    with pytest.raises(mo.OracleProtocolError, match="exceed"):
        mo.check_routes(spec, np.zeros((4, 2), np.int64))
    with pytest.raises(mo.OracleProtocolError, match="shape"):
        mo.check_routes(spec, np.zeros((2, 3), np.int64))


REF = Path(os.environ.get("RAILTX_REF", "/root/reference")) / "pkg" / "src"


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted (GPU box)")
def test_oracle_vs_live_reference_random_grid():
    """Beyond the fixtures: compare against the live reference on a small
    seeded grid of (N, E, T, R) (SPEC.md:553 acceptance grid, subsampled)."""
    sys.path.insert(0, str(REF))
    sys.path.insert(0, str(REF.parent / "tests"))
    from railtx import moe as rmoe
    import _fabric
    import _invariants as inv
    rng = np.random.default_rng(99)
    for (n, e, t, r) in [(2, 4, 3, 2), (4, 8, 6, 2), (2, 16, 5, 4), (8, 8, 2, 1)]:
        spec_r = rmoe.RoutingSpec(n, e, t, r, hidden=4, elem_size=4, scales=0)
        spec = mo.Spec(n, e, t, r, hidden=4, elem_size=4, scales=0)
        with _fabric.engines(_fabric.mode_config("reverse", 2), n) as es:
            mesh = rmoe.build_mesh(es, spec_r)
            try:
                routes, values, weights = inv.random_step(spec_r, rng)
                results = inv.run_moe_round(mesh, spec_r, routes, values, weights)
            finally:
                for m in mesh:
                    m.close()
        res = mo.dispatch(spec, routes, [mo.encode_tokens(spec, v) for v in values])
        outs = mo.apply_experts(spec, res)
        comb = mo.combine(spec, res, outs, weights)
        for q in range(n):
            g = results[q][0]
            assert np.array_equal(g.data, res.ranks[q].grouped.data)
            assert np.array_equal(g.rows, res.ranks[q].grouped.rows)
            assert np.array_equal(results[q][1], comb[q])


def test_weights_prepare_matches_reference():
    from oracle import transfer_oracle as to
    from golden_io import GOLDEN
    z = np.load(GOLDEN / "weights.npz")
    for k in range(int(z["ntasks"][0])):
        dt = "bf16" if int(z[f"t{k}_dtype"][0]) == 0 else "fp8"
        assert np.array_equal(to.prepare_words(z[f"t{k}_words"], dt), z[f"t{k}_prepared"]), k
    assert np.array_equal(to.prepare_words(z["big_words"], "fp8"), z["big_prepared"])
