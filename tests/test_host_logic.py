"""CPU tests of the host-side mirror of railtx.moe (no kernel launches)."""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import load_moe, moe_cases
from oracle import moe_oracle as mo
from paper_2510_27656_b200 import moe
from paper_2510_27656_b200.errors import ProtocolError, RailtxError


@pytest.mark.parametrize("kw,msg", [
    (dict(ranks=0, experts=4, max_tokens=1, topk=1), "rank count must be positive"),
    (dict(ranks=3, experts=4, max_tokens=1, topk=1), "expert count 4 is not a positive multiple of 3 ranks"),
    (dict(ranks=1, experts=4, max_tokens=1, topk=0), "topk 0 outside 1..4"),
    (dict(ranks=1, experts=4, max_tokens=0, topk=1), "max_tokens must be positive"),
    (dict(ranks=1, experts=4, max_tokens=1, topk=1, hidden=0), "hidden size must be positive"),
    (dict(ranks=1, experts=4, max_tokens=1, topk=1, scales=-1), "scale count must be non-negative"),
    (dict(ranks=1, experts=4, max_tokens=1, topk=1, scales=0), "at least one scale slot"),
])
def test_routing_spec_validation(kw, msg):
    with pytest.raises(ProtocolError, match=msg):
        moe.RoutingSpec(**kw)


def test_error_hierarchy():
    assert issubclass(ProtocolError, RailtxError)


def test_spec_properties():
    s = moe.RoutingSpec(8, 256, 128, 8, hidden=7168, elem_size=1, scales=56)
    assert (s.local_experts, s.payload_bytes, s.capacity) == (32, 7392, 32768)
    assert s.owner(33) == 1 and s.local_index(33) == 1
    s2 = moe.RoutingSpec(8, 256, 128, 8, hidden=7168, elem_size=1, scales=56, comb_elem_size=2)
    assert s2.comb_payload_bytes == 14336


def test_private_buffer_validation():
    s = moe.RoutingSpec(2, 4, 4, 2, hidden=8, elem_size=4, scales=0)
    moe.PrivateBufferConfig(4).validate(s)
    with pytest.raises(ProtocolError, match="private buffer"):
        moe.PrivateBufferConfig(5).validate(s)


def test_check_routes_messages_match_reference_order():
    s = moe.RoutingSpec(2, 4, 3, 2, hidden=8, elem_size=4, scales=0)
    with pytest.raises(ProtocolError, match=r"route array shape \(2, 3\) is not \(tokens, 2\)"):
        moe._check_routes(s, np.zeros((2, 3), np.int64))
    with pytest.raises(ProtocolError, match="4 tokens exceed the 3-token limit"):
        moe._check_routes(s, np.zeros((4, 2), np.int64))
    with pytest.raises(ProtocolError, match="expert index out of range"):
        moe._check_routes(s, np.array([[0, 4]]))
    with pytest.raises(ProtocolError, match="token 1 routes to a duplicate expert"):
        moe._check_routes(s, np.array([[0, 1], [3, 3]]))


@pytest.mark.parametrize("name", moe_cases())
def test_compute_layout_matches_golden(name):
    case = load_moe(name)
    spec = moe.RoutingSpec(**case.spec_args)
    for st in case.steps:
        counts = moe.RouteMatrix.from_routes(spec, st.routes).counts
        if st.counts is not None:
            assert np.array_equal(counts, st.counts)
        lay = moe.compute_layout(spec, counts)
        ol = mo.compute_layout(mo.Spec(**case.spec_args), counts)
        for k in ("assigned", "recv_start", "recv_total", "send_start"):
            assert np.array_equal(getattr(lay, k), getattr(ol, k)), k
        # range_of agrees with the golden grouped rows
        for d in range(spec.ranks):
            rows = []
            for (le, s), start, length in lay.ranges(d):
                rows.extend(range(start, start + length))
            got = st.rows[d][st.rows[d] >= 0]
            assert np.array_equal(np.array(rows, dtype=np.int64), got)


def test_capacity_error():
    s = moe.RoutingSpec(2, 4, 2, 2, hidden=8, elem_size=4, scales=0)
    with pytest.raises(ProtocolError, match="routes 5 copies, limit 4"):
        moe.RouteMatrix(s, np.array([[5, 0, 0, 0], [0, 0, 0, 0]]))


def test_trace_recorder_roundtrip(tmp_path):
    """TraceRecorder (railtx trace.py:33-99 semantics): total order, kind +
    field matching, transfer labels, JSON-lines dump/load; a disabled
    recorder keeps nothing."""
    from paper_2510_27656_b200.trace import TraceRecorder, load_path
    tr = TraceRecorder("e0")
    tr.label_transfer(7, "moe.comb")
    a = tr.record("wr_post", transfer=7, dst="r1")
    b = tr.record("moe_dispatch_done", step=1, used=3, capacity=8)
    tr.record("wr_post", transfer=8, dst="r2")
    assert a.seq < b.seq and len(tr) == 3
    assert [e.fields["dst"] for e in tr.events("wr_post")] == ["r1", "r2"]
    assert tr.events("wr_post", dst="r2")[0].fields["transfer"] == 8
    assert tr.labels() == {7: "moe.comb"} and tr.label_of(8) is None
    p = tmp_path / "t.jsonl"
    tr.dump_path(str(p))
    rows = load_path(str(p))
    assert [r["kind"] for r in rows] == ["wr_post", "moe_dispatch_done", "wr_post", "label"]
    assert rows[1]["used"] == 3 and rows[3]["label"] == "moe.comb" and rows[3]["transfer_id"] == 7
    off = TraceRecorder("e1", enabled=False)
    assert off.record("x") is None and len(off) == 0


@pytest.mark.parametrize("ranks", [1, 3])
def test_cpu_baseline_threaded_port_matches_oracle(ranks):
    """The reference arm's threaded oracle port (bench.cpu_baseline) checks
    itself against the serial oracle before timing; run it on a small shape,
    one rank and an EP=3 step (every rank on the host, as the reference's
    SimFabric runs it)."""
    import bench
    wl = dict(bench.WORKLOADS["decode"], tokens=16, experts=24, hidden=256, scales=4)
    r = bench.cpu_baseline(wl, 16, 0.05, ranks=ranks)
    assert r["kind"] == "port" and r["cores"] >= 1 and r["value"] > 0
    assert f"EP={ranks}" in r["sample"]
