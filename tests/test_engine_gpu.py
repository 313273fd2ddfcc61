"""GPU tests of the WriteImm + ImmCounter engine primitives and the phase-2
data paths (paged KV-cache transfer, weight publication), modelled on the
reference invariant battery (tests/_invariants.py: check_engine_writes
42-70, check_imm_threshold 73-109, check_scatter_barrier 112-133,
check_kvcache 139-184, check_weights 215-244)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from golden_io import GOLDEN
from oracle import transfer_oracle as to

pytestmark = pytest.mark.gpu
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0

if NGPU:
    from paper_2510_27656_b200.engine import NvlinkFabric, Pages, ScatterDst, TransferEngine
    from paper_2510_27656_b200.errors import ProtocolError, TransferError
    from paper_2510_27656_b200 import kvcache, weights


def _pair():
    fab = NvlinkFabric()
    d1 = 1 if NGPU > 1 else 0
    if d1:
        from paper_2510_27656_b200.memory import enable_peer_access
        enable_peer_access([0, 1])
    return TransferEngine(fab, device=0, name="a"), TransferEngine(fab, device=d1, name="b")


def _u8(e, n, fill=None, seed=0):
    t = e.alloc_buffer(n)
    if fill == "rand":
        g = torch.Generator(device="cpu").manual_seed(seed)
        t.copy_(torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g).to(t.device))
    return t


@pytest.mark.parametrize("page_len,npages", [(4096, 64), (8192, 16), (100, 7), (40000, 3)])
def test_engine_writes_payload_complete_at_fire(page_len, npages):
    a, b = _pair()
    try:
        n = page_len * npages
        src = _u8(a, n, "rand", 101)
        dst1, dst2 = _u8(b, n), _u8(b, n)
        h, _ = a.reg_mr(src)
        _, d1 = b.reg_mr(dst1)
        _, d2 = b.reg_mr(dst2)
        f1 = b.expect_imm_count(11, 1)
        f2 = b.expect_imm_count(12, 1)
        order = tuple(np.random.default_rng(3).permutation(npages).tolist())
        pages = Pages(order, page_len)
        a.submit_paged_writes(page_len, (h, pages), (d1, pages), imm=11).result(30.0)
        a.submit_single_write(n, (h, 0), (d2, 0), imm=12).result(30.0)
        assert f1.wait(10.0) and f2.wait(10.0)
        want = src.cpu().numpy()
        assert np.array_equal(dst1.cpu().numpy(), want)
        assert np.array_equal(dst2.cpu().numpy(), want)
    finally:
        a.close()
        b.close()


def test_paged_write_scatter_matches_oracle():
    a, b = _pair()
    try:
        P = 2048
        src = _u8(a, P * 40, "rand", 5)
        dst = _u8(b, P * 80)
        h, _ = a.reg_mr(src)
        _, d = b.reg_mr(dst)
        si = tuple(np.random.default_rng(1).permutation(40)[:25].tolist())
        di = tuple(np.random.default_rng(2).permutation(80)[:25].tolist())
        a.submit_paged_writes(P, (h, Pages(si, P)), (d, Pages(di, P)), imm=9).result(30.0)
        want = np.zeros(P * 80, np.uint8)
        to.paged_copy(src.cpu().numpy(), want, P, (si, P, 0), (di, P, 0))
        assert np.array_equal(dst.cpu().numpy(), want)
    finally:
        a.close()
        b.close()


def test_imm_threshold_arm_before_and_after_arrival():
    a, b = _pair()
    try:
        src, dst = _u8(a, 16), _u8(b, 16)
        h, _ = a.reg_mr(src)
        _, desc = b.reg_mr(dst)
        counts = {imm: 2 + imm % 5 for imm in range(20, 28)}
        early = {imm: b.expect_imm_count(imm, counts[imm]) for imm in list(counts)[:4]}
        flags = []
        for imm, c in counts.items():
            for _ in range(c):
                flags.append(a.submit_single_write(1, (h, 0), (desc, 0), imm=imm))
        for f in flags:
            f.result(30.0)
        for imm, f in early.items():
            assert f.wait(10.0), f"imm {imm} never fired"
        for imm in list(counts)[4:]:
            assert b.imm_received_total(imm) == counts[imm]
            f = b.expect_imm_count(imm, counts[imm])
            assert f.wait(2.0), f"imm {imm} did not fire from residue"
        # re-arm consumes: one more expectation needs new receipts
        f = b.expect_imm_count(20, 1)
        assert not f.done()
        a.submit_single_write(0, (h, 0), (desc, 0), imm=20).result(10.0)
        assert f.wait(5.0)
        with pytest.raises(ProtocolError, match="already armed"):
            b.expect_imm_count(99, 1)
            b.expect_imm_count(99, 1)
        with pytest.raises(TransferError, match="zero-length write requires an immediate"):
            a.submit_single_write(0, (h, 0), (desc, 0))
        with pytest.raises(TransferError, match="outside region"):
            a.submit_single_write(17, (h, 0), (desc, 0), imm=1)
    finally:
        a.close()
        b.close()


def test_scatter_and_barrier():
    fab = NvlinkFabric()
    devs = [i % NGPU for i in range(4)]
    if NGPU > 1:
        from paper_2510_27656_b200.memory import enable_peer_access
        enable_peer_access(sorted(set(devs)))
    es = [TransferEngine(fab, device=d, name=f"e{i}") for i, d in enumerate(devs)]
    try:
        src = _u8(es[0], 3 * 8192, "rand", 103)
        h, _ = es[0].reg_mr(src)
        bufs, descs, flags = [], [], []
        for e in es[1:]:
            buf = _u8(e, 8192)
            _, d = e.reg_mr(buf)
            bufs.append(buf)
            descs.append(d)
            flags.append((e.expect_imm_count(31, 1), e.expect_imm_count(32, 1)))
        group = es[0].add_peer_group([d.owner for d in descs])
        dsts = [ScatterDst(8192, i * 8192, d, 0) for i, d in enumerate(descs)]
        es[0].submit_scatter(group, h, dsts, imm=31).result(30.0)
        es[0].submit_barrier(group, 32, [(d, 0) for d in descs]).result(30.0)
        want = src.cpu().numpy()
        for i, (ftok, fbar) in enumerate(flags):
            assert ftok.wait(10.0) and fbar.wait(10.0)
            assert np.array_equal(bufs[i].cpu().numpy(), want[i * 8192:(i + 1) * 8192])
    finally:
        for e in es:
            e.close()


@pytest.mark.parametrize("layers,chunks,ppc,page_len,heads", [(4, 2, 1, 8192, 1), (3, 2, 4, 4096, 2)])
def test_kvcache_pages_and_context_byte_identical(layers, chunks, ppc, page_len, heads):
    """check_kvcache fidelity: every decoder page equals page_bytes, the
    context equals context_bytes, and the completion fires only after all
    steps + the context write."""
    a, b = _pair()
    try:
        layout = kvcache.KvLayout(layers, chunks, ppc, page_len)
        dec = kvcache.KvReceiver(b, layout, pool_slots=layout.slots + 3, local_heads=heads,
                                 ctx_bytes=4096)
        t = dec.open_request(ctx_len=1024)
        req = t.request
        rid = req.request_id
        # prefiller fills its pages exactly as PrefillerNode._compute does
        kvb = np.zeros(layout.region_bytes(heads, layout.slots), np.uint8)
        for layer in range(layers):
            for j in range(heads):
                for slot in range(layout.slots):
                    idx = layout.page_index(heads, layout.slots, layer, j, slot)
                    kvb[idx * page_len:(idx + 1) * page_len] = np.frombuffer(
                        to.page_bytes(rid, layer, j, slot, page_len), np.uint8)
        kv = a.alloc_buffer(kvb.size)
        kv.copy_(torch.from_numpy(kvb).to(kv.device))
        ctx = a.alloc_buffer(1024)
        ctx.copy_(torch.from_numpy(np.frombuffer(to.context_bytes(rid, 1024), np.uint8).copy()).to(ctx.device))
        send = kvcache.KvSender(a, kv, ctx)
        flags = [send.send_step(req, k) for k in range(1, layout.steps + 1)]
        for f in flags:
            f.result(30.0)
        assert not t.flag.done(), "completion fired before the context write"
        send.send_context(req).result(30.0)
        assert t.wait(10.0)
        for layer in range(layers):
            for j in range(heads):
                for i in range(layout.slots):
                    got = dec.page_view(t, layer, j, i).cpu().numpy().tobytes()
                    assert got == to.page_bytes(rid, layer, j, i, page_len)
        assert dec.ctx[:1024].cpu().numpy().tobytes() == to.context_bytes(rid, 1024)
        dec.release(t)
    finally:
        a.close()
        b.close()


def test_weights_prepare_matches_reference_goldens():
    z = np.load(GOLDEN / "weights.npz")
    for k in range(int(z["ntasks"][0])):
        dt = "bf16" if int(z[f"t{k}_dtype"][0]) == 0 else "fp8"
        words = torch.from_numpy(z[f"t{k}_words"].view(np.int16)).cuda()
        got = weights.prepare_device(words, dt).cpu().numpy()
        assert np.array_equal(got, z[f"t{k}_prepared"]), k
    words = torch.from_numpy(z["big_words"].view(np.int16)).cuda()
    assert np.array_equal(weights.prepare_device(words, "fp8").cpu().numpy(), z["big_prepared"])


def test_weights_publish_to_two_destinations():
    a, b = _pair()
    try:
        z = np.load(GOLDEN / "weights.npz")
        words = torch.from_numpy(z["big_words"].view(np.int16)).cuda(a.device)
        prepared = weights.prepare_device(words, "fp8")
        n = prepared.numel()
        dst = _u8(b, 2 * n + 64)
        _, d = b.reg_mr(dst)
        f = b.expect_imm_count(77, 2)
        weights.publish(a, prepared, [(d, 0), (d, n + 64)], imm=77)
        assert f.wait(10.0)
        got = dst.cpu().numpy()
        assert np.array_equal(got[:n], z["big_prepared"])
        assert np.array_equal(got[n + 64:2 * n + 64], z["big_prepared"])
    finally:
        a.close()
        b.close()
