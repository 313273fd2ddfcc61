"""GPU parity: the sm_100a dispatch/combine path vs the reference goldens
and the CPU oracle.  Bit-exact for payload bytes, indices, counts and the
fp32 combine; bf16 combine output within rtol 1e-2 / atol 1e-3
(BASELINE.json north_star)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from golden_io import load_moe, moe_cases
from oracle import moe_oracle as mo

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from moe_driver import check_device_round, close_mesh, device_round, make_mesh, ospec_of, run_moe_round
    from paper_2510_27656_b200 import moe
    from paper_2510_27656_b200.engine import local_engines
    from paper_2510_27656_b200.errors import ProtocolError


def _np(x):
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


@pytest.mark.parametrize("name", moe_cases())
def test_golden_round_bit_exact(name):
    """Whole reference rounds (goldens from railtx itself) through the
    device path, host-mode API, threaded driver like the reference's."""
    case = load_moe(name)
    spec = moe.RoutingSpec(**case.spec_args)
    mesh = make_mesh(spec)
    try:
        for st in case.steps:
            res = run_moe_round(mesh, spec, st.routes, st.values, st.weights)
            for q in range(spec.ranks):
                g, comb, pos = res[q]
                assert np.array_equal(pos, st.pos[q]), f"pos rank {q}"
                assert np.array_equal(_np(g.group_sizes), st.group_sizes[q])
                assert np.array_equal(_np(g.group_starts), st.group_starts[q])
                assert np.array_equal(_np(g.rows), st.rows[q]), f"rows rank {q}"
                assert np.array_equal(_np(g.sources), st.sources[q]), f"sources rank {q}"
                assert np.array_equal(_np(g.data), st.data[q]), f"data rank {q}"
                assert comb.shape == st.combined[q].shape
                assert np.array_equal(comb, st.combined[q]), f"combine rank {q}"
            if st.counts is not None:
                lay = mesh[0].last_layout
                assert np.array_equal(lay.counts, st.counts)
    finally:
        close_mesh(mesh)


def _oracle_round(ospec, routes, values_or_payloads, encoded=False):
    payloads = values_or_payloads if encoded else [mo.encode_tokens(ospec, v) for v in values_or_payloads]
    return mo.dispatch(ospec, routes, payloads), payloads


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("elem,src", [(1, torch.float32), (1, torch.bfloat16), (2, torch.float32),
                                      (2, torch.bfloat16), (4, torch.float32)])
def test_fused_encode_dispatch_matches_oracle(elem, src, fused):
    """Device mode: f32/bf16 values encoded inside the dispatch kernel
    (fp8 per-token scale / bf16 RNE / f32) == encode_tokens then dispatch."""
    N = 1
    spec = moe.RoutingSpec(ranks=N, experts=32, max_tokens=64, topk=4, hidden=512,
                           elem_size=elem, scales=8 if elem == 1 else 0)
    os_ = ospec_of(spec)
    rng = np.random.default_rng(5)
    routes, values, weights = mo.random_step(os_, rng, tokens=64)
    vals = [torch.from_numpy(v).to(src) for v in values]
    ref_vals = [v.float().numpy() for v in vals]      # bf16-rounded inputs for the oracle
    res, _ = _oracle_round(os_, routes, ref_vals)
    mesh = moe.build_mesh(local_engines([0]), spec)
    try:
        rk = mesh[0]
        rk.fused = fused
        rk.dispatch_send(vals[0].cuda(), torch.from_numpy(routes[0]).cuda())
        g = rk.dispatch_recv()
        want = res.ranks[0].grouped
        assert np.array_equal(_np(g.data), want.data)
        assert np.array_equal(_np(g.rows), want.rows)
        rk.combine_send(g.data)
        out = rk.combine_recv(torch.from_numpy(weights[0]).cuda())
        ref = mo.combine(os_, res, [want.data], weights)[0]
        assert np.array_equal(_np(out), ref)
    finally:
        close_mesh(mesh)


@pytest.mark.parametrize("topk,tokens,experts,elem,hidden", [
    (3, 37, 48, 1, 1024),     # R does not divide 32: loaded duplicate check, i % R ranks
    (12, 20, 64, 1, 512),     # R > 8: shuffle duplicate check past the unrolled part
    (8, 1, 256, 1, 7168),     # a single token
    (8, 148, 384, 1, 2048),   # as many tokens as SMs (last decode-shaped batch)
    (5, 64, 40, 2, 2048),     # bf16 rows that fit the token role (<= 2 chunks per thread)
    (2, 16, 8, 4, 256),       # f32 rows
])
def test_decode_roles_kernel_shapes(topk, tokens, experts, elem, hidden):
    """Odd decode shapes through the fused (warp-role) dispatch: payloads,
    rows, sources, pos and the combine bit-exact vs the oracle, two steps."""
    spec = moe.RoutingSpec(ranks=1, experts=experts, max_tokens=tokens, topk=topk, hidden=hidden,
                           elem_size=elem, scales=4 if elem == 1 else 0)
    os_ = ospec_of(spec)
    mesh = moe.build_mesh(local_engines([0]), spec)
    rk = mesh[0]
    try:
        for step in range(2):
            rng = np.random.default_rng(1000 * topk + tokens + step)
            routes, values, weights = mo.random_step(os_, rng, tokens=tokens)
            xb = torch.from_numpy(values[0]).to(torch.bfloat16)
            res, _ = _oracle_round(os_, routes, [xb.float().numpy()])
            rk.dispatch_send(xb.cuda(), torch.from_numpy(routes[0]).cuda())
            g = rk.dispatch_recv()
            want = res.ranks[0].grouped
            assert np.array_equal(_np(g.data), want.data)
            assert np.array_equal(_np(g.rows), want.rows)
            assert np.array_equal(_np(g.sources), want.sources)
            assert np.array_equal(rk.pos.cpu().numpy(), res.ranks[0].pos)
            rk.combine_send(g.data)
            out = rk.combine_recv(torch.from_numpy(weights[0]).cuda())
            assert np.array_equal(_np(out), mo.combine(os_, res, [want.data], weights)[0])
    finally:
        rk.close()


@pytest.mark.parametrize("bad", ["dup", "range"])
def test_device_route_errors_decode_path(bad):
    """Device-validated routes on the decode (warp-role) path: a duplicate
    or out-of-range expert is latched and raised at dispatch_recv."""
    spec = moe.RoutingSpec(ranks=1, experts=64, max_tokens=32, topk=8, hidden=1024, elem_size=1, scales=4)
    mesh = moe.build_mesh(local_engines([0]), spec)
    rk = mesh[0]
    try:
        routes = np.stack([np.random.default_rng(t).permutation(64)[:8] for t in range(32)]).astype(np.int64)
        if bad == "dup":
            routes[7, 5] = routes[7, 2]
        else:
            routes[30, 0] = 64
        x = torch.randn(32, 1024, device="cuda").to(torch.bfloat16)
        rk.dispatch_send(x, torch.from_numpy(routes).cuda())
        with pytest.raises(ProtocolError, match="duplicate" if bad == "dup" else "out of range"):
            rk.dispatch_recv()
    finally:
        rk.close()


@pytest.mark.parametrize("fused", [True, False])
def test_dsv3_decode_ep1_full_size(fused):
    """DeepSeek-V3 decode shape at EP=1 (128 tok, H=7168, E=256, top-8),
    fp8 dispatch from bf16 values, bf16 combine rows, bf16 out; several
    steps back to back on one mesh (counter epochs, buffer reuse)."""
    spec = moe.RoutingSpec(ranks=1, experts=256, max_tokens=128, topk=8, hidden=7168,
                           elem_size=1, scales=56, comb_elem_size=2, comb_scales=0)
    os_ = ospec_of(spec)
    cs = mo.Spec(1, 256, 128, 8, hidden=7168, elem_size=2, scales=0)
    mesh = moe.build_mesh(local_engines([0]), spec)
    rk = mesh[0]
    rk.fused = fused
    try:
        for step in range(3):
            rng = np.random.default_rng(100 + step)
            routes, values, weights = mo.random_step(os_, rng, tokens=128)
            xb = torch.from_numpy(values[0]).to(torch.bfloat16)
            res, _ = _oracle_round(os_, routes, [xb.float().numpy()])
            rk.dispatch_send(xb.cuda(), torch.from_numpy(routes[0]).cuda())
            g = rk.dispatch_recv()
            want = res.ranks[0].grouped
            assert np.array_equal(_np(g.data), want.data)
            assert np.array_equal(_np(g.sources), want.sources)
            # expert stand-in: decode the fp8 rows, scale by (1 + expert), bf16 rows back
            y = torch.zeros((g.data.shape[0], spec.hidden), dtype=torch.bfloat16, device="cuda")
            dec = moe.decode_tokens(spec, g.data)
            for le in range(spec.local_experts):
                s0, c = int(g.group_starts[le]), int(g.group_sizes[le])
                if c:
                    y[s0:s0 + c] = (dec[s0:s0 + c] * (1.0 + 0.01 * le)).to(torch.bfloat16)
            rk.combine_send(y)
            out = rk.combine_recv(torch.from_numpy(weights[0]).cuda(), out_dtype=torch.bfloat16)
            outs = [mo.bf16_encode(y.float().cpu().numpy()).view(np.uint8).reshape(y.shape[0], -1)]
            ref = mo.combine(os_, res, outs, weights, comb_spec=cs)[0]
            got = out.float().cpu().numpy()
            np.testing.assert_allclose(got, ref, rtol=1e-2, atol=1e-3)
            # the fp32 accumulation itself is exact: bf16(out) == bf16(ref)
            assert np.array_equal(mo.bf16_encode(ref), out.view(torch.int16).cpu().numpy().view(np.uint16))
    finally:
        rk.close()


@pytest.mark.parametrize("fused", [True, False])
def test_pinned_host_zero_copy_matches_device_mode(fused):
    """Page-locked host inputs (activations, routes, weights) and a pinned
    host `out`: the kernels read / write them in place over PCIe; the
    grouped payloads and the combined rows equal the device-mode step
    bit for bit, and the oracle's."""
    spec = moe.RoutingSpec(ranks=1, experts=256, max_tokens=128, topk=8, hidden=7168,
                           elem_size=1, scales=56, comb_elem_size=2, comb_scales=0)
    os_ = ospec_of(spec)
    cs = mo.Spec(1, 256, 128, 8, hidden=7168, elem_size=2, scales=0)
    mesh = moe.build_mesh(local_engines([0]), spec)
    rk = mesh[0]
    rk.fused = fused
    try:
        for step, T in enumerate([128, 77]):
            rng = np.random.default_rng(300 + step)
            routes, values, weights = mo.random_step(os_, rng, tokens=T)
            xb = torch.from_numpy(values[0]).to(torch.bfloat16)
            res, _ = _oracle_round(os_, routes, [xb.float().numpy()])
            rk.dispatch_send(xb.pin_memory(), torch.from_numpy(routes[0]).pin_memory())
            g = rk.dispatch_recv()
            assert np.array_equal(_np(g.data), res.ranks[0].grouped.data)
            y = (moe.decode_tokens(spec, g.data) * 0.75).to(torch.bfloat16)
            rk.combine_send(y)
            oh = torch.empty((T, spec.hidden), dtype=torch.bfloat16).pin_memory()
            out = rk.combine_recv(torch.from_numpy(weights[0]).pin_memory(), out_dtype=torch.bfloat16, out=oh)
            assert out is oh
            outs = [mo.bf16_encode(y.float().cpu().numpy()).view(np.uint8).reshape(y.shape[0], -1)]
            ref = mo.combine(os_, res, outs, weights, comb_spec=cs)[0]
            assert np.array_equal(mo.bf16_encode(ref), oh.view(torch.int16).numpy().view(np.uint16))
        with pytest.raises(ProtocolError, match="out must be"):
            rk.dispatch_send(xb.cuda(), torch.from_numpy(routes[0]).cuda())
            rk.dispatch_recv()
            rk.combine_send(y)
            rk.combine_recv(torch.from_numpy(weights[0]).cuda(), out=torch.empty(3, 3))
    finally:
        rk.close()


def test_check_moe_trace_audit():
    """check_moe (_invariants.py:334-364): results equal the oracle, the
    traced receive occupancy stays within capacity, and the per-peer write
    budget holds (<= 2 token writes, exactly 1 combine write per peer per
    step), audited from the engines' traces."""
    spec = moe.RoutingSpec(ranks=2, experts=4, max_tokens=4, topk=2, hidden=8, elem_size=4, scales=0)
    os_ = ospec_of(spec)
    mesh = make_mesh(spec, private=2, trace=True)
    try:
        rng = np.random.default_rng(104)
        steps = 3
        for _ in range(steps):
            routes, values, weights = mo.random_step(os_, rng)
            res = run_moe_round(mesh, spec, routes, values, weights)
            ref = mo.dispatch(os_, routes, [mo.encode_tokens(os_, v) for v in values])
            for q in range(spec.ranks):
                assert np.array_equal(_np(res[q][0].data), ref.ranks[q].grouped.data)
        for rk in mesh:
            tr = rk.engine.trace
            done = tr.events("moe_dispatch_done")
            assert len(done) == steps
            for ev in done:
                assert ev.fields["used"] <= ev.fields["capacity"]
            assert len(tr.events("moe_host_signal")) == steps
            assert len(tr.events("moe_combine_store")) == steps
            assert len(tr.events("moe_combine_done")) == steps
            labels = tr.labels()
            tok = comb = 0
            for ev in tr.events("wr_post"):
                lb = labels.get(ev.fields.get("transfer"), "")
                tok += lb.startswith("moe.tok.")
                comb += lb == "moe.comb"
            peers = spec.ranks - 1
            assert tok <= 2 * steps * peers
            assert comb == steps * peers
            # ordering: each step's host signal precedes its dispatch_done
            for a_, b_ in zip(tr.events("moe_host_signal"), done):
                assert a_.seq < b_.seq and a_.fields["step"] == b_.fields["step"]
    finally:
        close_mesh(mesh)


def test_multi_step_and_empty_steps():
    """Ragged token counts including empty steps, several steps in a row."""
    spec = moe.RoutingSpec(ranks=2, experts=8, max_tokens=12, topk=3, hidden=64, elem_size=4, scales=0)
    os_ = ospec_of(spec)
    mesh = make_mesh(spec)
    try:
        rng = np.random.default_rng(3)
        for step in range(6):
            tokens = 0 if step in (1, 4) else None
            routes, values, weights = mo.random_step(os_, rng, tokens)
            res = run_moe_round(mesh, spec, routes, values, weights)
            ref, pay = _oracle_round(os_, routes, values)
            outs = mo.apply_experts(os_, ref)
            comb = mo.combine(os_, ref, outs, weights)
            for q in range(spec.ranks):
                assert np.array_equal(_np(res[q][0].data), ref.ranks[q].grouped.data)
                assert np.array_equal(res[q][1], comb[q])
    finally:
        close_mesh(mesh)


def test_route_errors_host_and_device():
    spec = moe.RoutingSpec(ranks=1, experts=8, max_tokens=4, topk=2, hidden=16, elem_size=4, scales=0)
    mesh = moe.build_mesh(local_engines([0]), spec)
    rk = mesh[0]
    try:
        pay = np.zeros((2, spec.payload_bytes), np.uint8)
        with pytest.raises(ProtocolError, match="duplicate"):
            rk.dispatch_send(pay, np.array([[1, 1], [2, 3]]))
        with pytest.raises(ProtocolError, match="out of range"):
            rk.dispatch_send(pay, np.array([[1, 9], [2, 3]]))
        with pytest.raises(ProtocolError, match="token limit"):
            rk.dispatch_send(np.zeros((5, spec.payload_bytes), np.uint8), np.zeros((5, 2), np.int64))
        with pytest.raises(ProtocolError, match="payload shape"):
            rk.dispatch_send(np.zeros((2, 3), np.uint8), np.array([[1, 2], [2, 3]]))
        with pytest.raises(ProtocolError, match="combine before dispatch"):
            rk.combine_send(np.zeros((8, spec.payload_bytes), np.uint8))
        # device-validated routes: latched, raised at dispatch_recv
        rk.dispatch_send(torch.zeros((2, spec.payload_bytes), dtype=torch.uint8, device="cuda"),
                         torch.tensor([[1, 1], [2, 3]], device="cuda"))
        with pytest.raises(ProtocolError, match="duplicate"):
            rk.dispatch_recv()
    finally:
        rk.close()


def test_step_in_flight_error():
    spec = moe.RoutingSpec(ranks=1, experts=4, max_tokens=4, topk=1, hidden=16, elem_size=4, scales=0)
    mesh = moe.build_mesh(local_engines([0]), spec)
    rk = mesh[0]
    try:
        pay = np.zeros((1, spec.payload_bytes), np.uint8)
        rk.dispatch_send(pay, np.array([[0]]))
        with pytest.raises(ProtocolError, match="in flight"):
            rk.dispatch_send(pay, np.array([[0]]))
        g = rk.dispatch_recv()
        rk.combine_send(np.zeros_like(g.data))
        out = rk.combine_recv(np.ones((1, 1), np.float32))
        assert out.shape == (1, 16)
    finally:
        rk.close()


def test_no_sync_mode_matches_sync():
    """dispatch_recv(sync=False): max-shape views + device sizes; the whole
    step is launch-only (what the bench and CUDA graphs use)."""
    spec = moe.RoutingSpec(ranks=1, experts=64, max_tokens=32, topk=4, hidden=256,
                           elem_size=1, scales=4, comb_elem_size=2, comb_scales=0)
    os_ = ospec_of(spec)
    rng = np.random.default_rng(9)
    routes, values, weights = mo.random_step(os_, rng, tokens=32)
    mesh = moe.build_mesh(local_engines([0]), spec)
    rk = mesh[0]
    try:
        x = torch.from_numpy(values[0]).cuda()
        r = torch.from_numpy(routes[0]).cuda()
        w = torch.from_numpy(weights[0]).cuda()
        y = torch.randn(int(rk._shape.grouped_rows), spec.hidden, device="cuda").to(torch.bfloat16)
        rk.dispatch_send(x, r, sync=False)
        g = rk.dispatch_recv(sync=False)
        rk.combine_send(y)
        out1 = rk.combine_recv(w, sync=False)
        torch.cuda.synchronize()
        rk.dispatch_send(x, r)
        g2 = rk.dispatch_recv()
        total = g2.data.shape[0]
        assert int(g.padded_total) == total
        rk.combine_send(y[:total].contiguous())
        out2 = rk.combine_recv(w)
        assert torch.equal(out1, out2)
    finally:
        rk.close()


def test_codecs_match_reference_goldens():
    from golden_io import load_codecs
    from paper_2510_27656_b200 import kernels
    c = load_codecs()
    assert np.array_equal(kernels.fp8_encode(c["fp8_in"]), c["fp8_out"])
    assert np.array_equal(kernels.bf16_encode(c["bf16_in"]), c["bf16_out"])
    dec = kernels.fp8_decode(np.arange(256, dtype=np.uint8))
    assert np.array_equal(dec, c["fp8_table"], equal_nan=True)
    spec = moe.RoutingSpec(ranks=1, experts=1, max_tokens=12, topk=1, hidden=96, elem_size=1, scales=3)
    assert np.array_equal(moe.encode_tokens(spec, c["rows"]), c["rows_enc"])
    assert np.array_equal(moe.decode_tokens(spec, c["rows_enc"]), c["rows_dec"], equal_nan=True)


def test_kernel_registry_matches_oracle():
    from paper_2510_27656_b200 import kernels
    rng = np.random.default_rng(4)
    src = rng.integers(0, 256, (50, 37), dtype=np.uint8)
    rows = rng.integers(0, 50, 80)
    assert np.array_equal(kernels.pack_rows(src, rows), src[rows])
    y = rng.standard_normal((40, 24)).astype(np.float32)
    pos = rng.integers(0, 40, (10, 3))
    w = rng.random((10, 3)).astype(np.float32)
    assert np.array_equal(kernels.weighted_combine(y, pos, w), mo.weighted_combine(y, pos, w))


@pytest.mark.parametrize("src", ["values", "rows"])
@pytest.mark.parametrize("tokens,experts,elem", [(600, 256, 2), (300, 384, 1), (1024, 64, 4)])
def test_large_batch_generic_fused_path(tokens, experts, elem, src):
    """Batches larger than the SM count take the generic fused kernel:
    contiguous token ranges per CTA, segmented route counting with two grid
    barriers, the barrier-free token loop for rows without a per-token amax
    (f32/bf16 values, or pre-encoded payload rows of any element size).
    Bit-exact grouped data / metadata / combine vs the oracle."""
    spec = moe.RoutingSpec(ranks=1, experts=experts, max_tokens=tokens, topk=8, hidden=256,
                           elem_size=elem, scales=4 if elem == 1 else 0)
    os_ = ospec_of(spec)
    rng = np.random.default_rng(tokens)
    routes, values, weights = mo.random_step(os_, rng, tokens=tokens)
    res, _ = _oracle_round(os_, routes, values)
    mesh = moe.build_mesh(local_engines([0]), spec)
    rk = mesh[0]
    try:
        payload = (torch.from_numpy(values[0]).cuda() if src == "values"
                   else torch.from_numpy(mo.encode_tokens(os_, values[0])).cuda())
        for rep in range(2):
            rk.dispatch_send(payload, torch.from_numpy(routes[0]).cuda())
            g = rk.dispatch_recv()
            want = res.ranks[0].grouped
            assert np.array_equal(_np(g.data), want.data)
            assert np.array_equal(_np(g.rows), want.rows)
            assert np.array_equal(_np(g.sources), want.sources)
            assert np.array_equal(rk.pos.cpu().numpy(), res.ranks[0].pos)
            rk.combine_send(g.data)
            out = rk.combine_recv(torch.from_numpy(weights[0]).cuda())
            ref = mo.combine(os_, res, [want.data], weights)[0]
            assert np.array_equal(_np(out), ref)
    finally:
        rk.close()


@pytest.mark.parametrize("amax", [1.0, 3.14159265, 0.70710677, 1e-3, 12345.678, 65504.0, 2.0 ** -60,
                                  1.1, 1.9999999, 0.33333334, 7.77e-5, 2.5e10, 1.5, 5.0])
def test_fp8_encode_division_exhaustive(amax):
    """The fp8 encode divides by the per-token scale with a multiply and two
    FMAs (div_rn_by) instead of an IEEE division.  Every f32 value x with
    |x| <= amax (both signs; amax itself sits in each row so it sets the
    scale) must give the same e4m3 byte as RN(x / f32(amax/448)) through
    torch's e4m3fn cast, saturated (== the reference codec, SURVEY probe P3)."""
    H = 4096
    spec = moe.RoutingSpec(ranks=1, experts=8, max_tokens=1, topk=1, hidden=H, elem_size=1, scales=4)
    a32 = np.float32(amax)
    hi = int(a32.view(np.uint32))
    # IEEE f32 amax/448 (numpy; torch's tensor / python-scalar multiplies by
    # a rounded reciprocal instead) -- the scale the kernel computes
    s = torch.tensor(np.float32(a32) / np.float32(448.0), device="cuda")
    per = H - 1
    chunk_rows = 1 << 14
    step = chunk_rows * per
    bad = 0
    for sign in (0, 1 << 31):
        for lo in range(0, hi + 1, step):
            bits = torch.arange(lo, min(hi + 1, lo + step), dtype=torch.int64, device="cuda")
            n = bits.numel()
            rows = (n + per - 1) // per
            pad = rows * per - n
            bits = torch.cat([bits, torch.zeros(pad, dtype=torch.int64, device="cuda")]) | sign
            vals = (bits.to(torch.int32)).view(torch.float32).view(rows, per)
            x = torch.cat([torch.full((rows, 1), float(a32), device="cuda"), vals], dim=1)
            enc = moe.encode_tokens(spec, x)
            got = enc[:, :H]
            assert torch.equal(enc[:, H:H + 4].contiguous().view(torch.float32).flatten(), s.expand(rows))
            # satfinite like the reference codec: torch's e4m3fn cast does not
            # saturate, so clamp first (RNE maps (448, 464) to 448 anyway)
            want = (x / s).clamp(-448.0, 448.0).to(torch.float8_e4m3fn).view(torch.uint8)
            bad += int((got != want).sum())
    assert bad == 0, f"{bad} e4m3 bytes differ for amax={amax}"


PRIV_CASES = ["cfg1_full", "n3_e12_t11_r4", "n4_e16_t9_r4", "n8_e16_t7_r3", "fp8_dsv3ish", "fp8_n2_h33_odd"]


@pytest.mark.parametrize("name", PRIV_CASES)
@pytest.mark.parametrize("ptok", [0, 4, 32, "T"])
def test_private_rounds_match_goldens(name, ptok):
    """Speculative private-buffer round (moe.py:556-582, 693-698) at
    PrivateBufferConfig.tokens in {0, 4, 32, T}: the first min(P, assigned)
    rows of every (source, destination) slab travel through the receiver's
    private slab and are moved to their grouped rows there.  Outputs must
    not depend on P (the reference's own property, SURVEY.md probe P5):
    every step bit-exact against the railtx goldens.  Several ranks share
    this GPU (host-gated split kernels, which place the same rows)."""
    case = load_moe(name)
    spec = moe.RoutingSpec(**case.spec_args)
    p = spec.max_tokens if ptok == "T" else min(int(ptok), spec.max_tokens)
    mesh = make_mesh(spec, private=p)
    try:
        for st in case.steps:
            res = run_moe_round(mesh, spec, st.routes, st.values, st.weights)
            for q in range(spec.ranks):
                g, comb, pos = res[q]
                assert np.array_equal(pos, st.pos[q]), f"pos rank {q}"
                assert np.array_equal(_np(g.rows), st.rows[q]), f"rows rank {q}"
                assert np.array_equal(_np(g.data), st.data[q]), f"data rank {q} (P={p})"
                assert np.array_equal(comb, st.combined[q]), f"combine rank {q}"
    finally:
        close_mesh(mesh)


def test_route_timeout_names_the_silent_rank():
    """A rank that never sends: the waiting rank raises ProtocolError with
    the reference's message shape and the silent source in its diagnostics
    (moe.py:869-899: 'rank r step s timed out waiting for route counts;
    missing: {...}')."""
    spec = moe.RoutingSpec(ranks=2, experts=8, max_tokens=16, topk=2, hidden=256, elem_size=4, scales=0)
    mesh = moe.build_mesh(local_engines([0, 0]), spec, timeout=1.0)
    try:
        os_ = ospec_of(spec)
        routes, values, _ = mo.random_step(os_, np.random.default_rng(3), tokens=16)
        with pytest.raises(ProtocolError,
                           match=r"rank 0 step 0 timed out waiting for route counts; missing: \{'route': \[1\]\}"):
            mesh[0].dispatch_send(mo.encode_tokens(os_, values[0]), routes[0])
    finally:
        close_mesh(mesh)


def test_token_timeout_names_the_silent_rank():
    """Routes arrive but one rank's token rows never do: the receiver's
    token lane names that source (per-source counters vs the per-source
    expectations booked from the route matrix)."""
    spec = moe.RoutingSpec(ranks=2, experts=8, max_tokens=16, topk=2, hidden=256, elem_size=4, scales=0)
    mesh = moe.build_mesh(local_engines([0, 0]), spec, private=moe.PrivateBufferConfig(0), timeout=1.0)
    try:
        os_ = ospec_of(spec)
        # every token of rank 1 routes to rank 0's experts, so rank 0 waits on rank 1
        routes = [np.tile(np.array([[0, 1]], np.int64), (16, 1)), np.tile(np.array([[2, 3]], np.int64), (16, 1))]
        values = [np.ones((16, 256), np.float32), np.ones((16, 256), np.float32)]
        # rank 1 publishes its count row (route phase only) and stops there
        import ctypes as C
        from paper_2510_27656_b200 import _lib
        r1 = mesh[1]
        with r1._lock:
            r1._step_no += 1
        r_dev = torch.from_numpy(routes[1]).cuda()
        _lib.call("txb_moe_route", r1._shape_p, r1._bufs_p, C.c_void_p(r_dev.data_ptr()), 16, r1._sid())
        torch.cuda.synchronize()
        mesh[0].dispatch_send(mo.encode_tokens(os_, values[0]), routes[0])
        with pytest.raises(ProtocolError, match=r"rank 0 step 0 timed out waiting for token writes; "
                                                r"missing: \{'token': \[1\]\}"):
            mesh[0].dispatch_recv(1.0)
    finally:
        close_mesh(mesh)


def test_per_token_mode_odd_rows_host_gated():
    """max_tokens above the per-token threshold with combine rows that are
    not 16-byte vectorisable (fp8, hidden 100: 132-byte rows, the ADVICE
    case): every returned row also books its origin token's counter, and the
    payloads and combine stay bit-exact."""
    spec = moe.RoutingSpec(ranks=2, experts=8, max_tokens=300, topk=2, hidden=100, elem_size=1, scales=8)
    mesh = make_mesh(spec, private=32)
    try:
        for step, n in enumerate([300, 41, 300]):
            rng = np.random.default_rng(70 + step)
            routes, values, weights = mo.random_step(ospec_of(spec), rng, tokens=n)
            xb, got = device_round(mesh, spec, routes, values, weights, out_dtype=torch.float32)
            check_device_round(spec, routes, xb, weights, got, f"step {step}")
            for q in range(2):
                _, c = mesh[q].status()
                assert c["tok_ctr"] == c["tok_target"] and c["comb_ctr"] == c["comb_target"]
    finally:
        close_mesh(mesh)


def _grid_cases(count: int, seed: int):
    """A seeded subsample of the SPEC.md acceptance grid (criterion 6):
    (N, E, T, R) in {2,4,8} x {4,8,16} x {1..16} x {1,2,4}, E a multiple of
    N and R <= E (the reference RoutingSpec rejects the rest)."""
    combos = [(n, e, t, r) for n in (2, 4, 8) for e in (4, 8, 16) for t in range(1, 17) for r in (1, 2, 4)
              if e % n == 0 and r <= e]
    rng = np.random.default_rng(seed)
    return [combos[i] for i in rng.choice(len(combos), size=count, replace=False)]


@pytest.mark.parametrize("n,e,t,r", _grid_cases(24, 553))
def test_acceptance_grid_subsample(n, e, t, r):
    """SPEC.md criterion 6 through the device path: two seeded random steps
    (random token counts <= T, reference random_step) per grid point;
    grouped payloads, rows, sources, pos and the fp32 combine bit-exact vs
    the oracle (the criterion asks 1e-6; this is exact), the capacity bound
    N*T*max(R, E/N) respected (instrumented from the device layout).  The
    reference's own payload format (fp8, 8 scale slots, hidden 64)."""
    spec = moe.RoutingSpec(ranks=n, experts=e, max_tokens=t, topk=r, hidden=64, elem_size=1, scales=8)
    os_ = ospec_of(spec)
    mesh = make_mesh(spec, private=min(4, t))
    try:
        for seed in range(2):
            rng = np.random.default_rng(1000 * seed + 7 * n + 13 * e + 17 * t + r)
            routes, values, weights = mo.random_step(os_, rng)
            res = run_moe_round(mesh, spec, routes, values, weights)
            ref = mo.dispatch(os_, routes, [mo.encode_tokens(os_, v) for v in values])
            outs = mo.apply_experts(os_, ref)
            comb = mo.combine(os_, ref, outs, weights)
            for q in range(n):
                g, c, pos = res[q]
                want = ref.ranks[q].grouped
                assert np.array_equal(_np(g.data), want.data), (seed, q)
                assert np.array_equal(_np(g.rows), want.rows), (seed, q)
                assert np.array_equal(_np(g.sources), want.sources), (seed, q)
                assert np.array_equal(pos, ref.ranks[q].pos), (seed, q)
                assert np.array_equal(c, comb[q]), (seed, q)
            lay = mesh[0].last_layout
            assert int(lay.recv_total.max()) <= spec.capacity
    finally:
        close_mesh(mesh)


def test_dsv3_prefill_full_size_ep1():
    """DeepSeek-V3 prefill at full size (BASELINE configs[2]: 4096 tokens,
    hidden 7168, 256 experts, top-8, bf16 rows both ways) through the
    large-batch fused path at EP=1: 32768 grouped rows of 14 KiB bit-exact,
    bf16 combine bits exact, two steps."""
    spec = moe.RoutingSpec(ranks=1, experts=256, max_tokens=4096, topk=8, hidden=7168, elem_size=2, scales=0,
                           comb_elem_size=2, comb_scales=0)
    mesh = moe.build_mesh(local_engines([0]), spec)
    try:
        for step in range(2):
            rng = np.random.default_rng(4096 + step)
            routes, values, weights = mo.random_step(ospec_of(spec), rng, tokens=4096 - 1000 * step)
            xb, got = device_round(mesh, spec, routes, values, weights)
            check_device_round(spec, routes, xb, weights, got, f"step {step}")
    finally:
        close_mesh(mesh)


def test_kimi_k2_decode_ep1_full_size():
    """Kimi-K2 shape (BASELINE configs[3]: 384 experts, top-8, hidden 7168,
    128 tokens, bench.py's skewed routing) at EP=1 on the decode kernel,
    fp8 dispatch encoded in-kernel, bf16 combine: bit-exact, three steps."""
    import bench
    spec = moe.RoutingSpec(ranks=1, experts=384, max_tokens=128, topk=8, hidden=7168, elem_size=1, scales=56,
                           comb_elem_size=2, comb_scales=0)
    mesh = moe.build_mesh(local_engines([0]), spec)
    try:
        for step in range(3):
            rng = np.random.default_rng(3840 + step)
            _, values, weights = mo.random_step(ospec_of(spec), rng, tokens=128)
            routes = [bench.routes_for(bench.WORKLOADS["kimi"], rng, 128)]
            xb, got = device_round(mesh, spec, routes, values, weights)
            check_device_round(spec, routes, xb, weights, got, f"step {step}")
    finally:
        close_mesh(mesh)
