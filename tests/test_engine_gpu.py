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


def test_imm_counter_randomized_10k_writes_256_imms():
    """SPEC.md acceptance criterion 2 (ImmCounter semantics): 10,000 writes
    carrying 256 distinct imm values, submitted from 4 sender engines
    ("rails": 4 independent streams into one receiver).  Half the imms are
    armed before any write, half after every write has landed.  Every armed
    expectation fires exactly once at its threshold (its callback runs once,
    on the engine's callback thread), arming after arrival fires at once,
    and at fire time every payload of that imm is already complete (the
    atomicity probe).  Imm values are spread over the whole u32 range and
    include pairs congruent modulo the table size, which must not alias."""
    import threading
    rng = np.random.default_rng(549)
    nimm = 256
    base = rng.choice(1 << 31, size=nimm // 2, replace=False).astype(np.int64)
    imms = np.concatenate([base, base + 131072 * 3]).tolist()       # congruent pairs
    counts = rng.multinomial(10_000 - nimm, np.ones(nimm) / nimm) + 1  # >= 1 write each, 10k total
    assert counts.sum() == 10_000
    fab = NvlinkFabric()
    d1 = 1 if NGPU > 1 else 0
    if d1:
        from paper_2510_27656_b200.memory import enable_peer_access
        enable_peer_access([0, 1])
    recv = TransferEngine(fab, device=d1, name="recv")
    senders = [TransferEngine(fab, device=0, name=f"rail{i}") for i in range(4)]
    W = 16                                   # bytes per payload
    try:
        slot_of = np.concatenate([[0], np.cumsum(counts)[:-1]])
        dst = _u8(recv, 10_000 * W)
        _, desc = recv.reg_mr(dst)
        srcs = []
        for i, e in enumerate(senders):
            s = _u8(e, 10_000 * W)
            # payload of write k of imm i: bytes derived from (i, k), never zero
            pay = np.zeros((10_000, W), np.uint8)
            for ii in range(nimm):
                for k in range(counts[ii]):
                    pay[slot_of[ii] + k] = (np.arange(W) * 7 + ii * 13 + k + 1) % 255 + 1
            s.copy_(torch.from_numpy(pay.reshape(-1)).to(s.device))
            srcs.append((s, e.reg_mr(s)[0], pay))
        fired: dict = {}
        probe_bad: list = []
        lock = threading.Lock()

        def cb_for(ii):
            def cb(flag):
                got = dst[slot_of[ii] * W:(slot_of[ii] + counts[ii]) * W].cpu().numpy().reshape(-1, W)
                with lock:
                    fired[ii] = fired.get(ii, 0) + 1
                    if not np.array_equal(got, srcs[0][2][slot_of[ii]:slot_of[ii] + counts[ii]]):
                        probe_bad.append(ii)
            return cb

        early = {ii: recv.expect_imm_count(imms[ii], int(counts[ii]), cb=cb_for(ii)) for ii in range(0, nimm, 2)}
        # every write of every imm, interleaved over the 4 rails in a random order
        order = [(ii, k) for ii in range(nimm) for k in range(counts[ii])]
        perm = rng.permutation(len(order))
        last = [None] * 4
        for n, p in enumerate(perm):
            ii, k = order[p]
            r = n % 4
            s, h, _ = srcs[r]
            off = (slot_of[ii] + k) * W
            last[r] = senders[r].submit_single_write(W, (h, off), (desc, off), imm=imms[ii])
        for f in last:
            f.result(60.0)
        for e in senders:
            e._stream.synchronize()
        for ii, f in early.items():
            assert f.wait(20.0), f"imm {imms[ii]} never fired"
        late = {}
        for ii in range(1, nimm, 2):
            assert recv.imm_received_total(imms[ii]) == counts[ii]
            f = recv.expect_imm_count(imms[ii], int(counts[ii]), cb=cb_for(ii))
            assert f.done(), "arming after arrival must fire immediately"
            late[ii] = f
        t_end = __import__("time").monotonic() + 20.0
        while len(fired) < nimm and __import__("time").monotonic() < t_end:
            __import__("time").sleep(0.01)
        assert sorted(fired) == list(range(nimm)), "some callbacks never ran"
        assert all(v == 1 for v in fired.values()), "a callback ran more than once"
        assert not probe_bad, f"incomplete payloads at fire time for imms {probe_bad[:5]}"
        assert not recv._cbt.errors
        # exactly-once: re-arming needs new receipts
        again = recv.expect_imm_count(imms[0], 1)
        assert not again.done()
    finally:
        for e in senders + [recv]:
            e.close()


def test_callbacks_do_not_block_the_submitter():
    """on_done and ImmFlag callbacks run on the engine's callback thread;
    the submitting call returns before the transfer has completed."""
    import threading
    import time
    a, b = _pair()
    try:
        n = 256 << 20
        src, dst = _u8(a, n), _u8(b, n)
        h, _ = a.reg_mr(src)
        _, d = b.reg_mr(dst)
        seen = {}
        ev = threading.Event()
        f_imm = b.expect_imm_count(4242, 1, cb=lambda fl: seen.setdefault("imm", threading.current_thread().name))
        torch.cuda._sleep(50_000_000)                 # keep the GPU busy: the write cannot finish yet
        t0 = time.perf_counter()
        a.submit_single_write(n, (h, 0), (d, 0), imm=4242,
                              on_done=lambda cf: (seen.setdefault("done", threading.current_thread().name),
                                                  ev.set()))
        assert time.perf_counter() - t0 < 0.5, "submit_single_write blocked on completion"
        assert ev.wait(30.0) and f_imm.wait(30.0)
        t_end = time.monotonic() + 5.0
        while "imm" not in seen and time.monotonic() < t_end:
            time.sleep(0.01)
        assert seen["done"].endswith("-callbacks") and seen["imm"].endswith("-callbacks")
    finally:
        a.close()
        b.close()


def test_watcher_host_and_device_stores():
    """alloc_watcher (engine.py:621-638): the callback thread reports a
    strictly increasing subsequence of the stored values ending at the
    latest, for host stores and for device stores through device_ptr."""
    import time
    from paper_2510_27656_b200 import _lib
    import ctypes as C
    a = TransferEngine(NvlinkFabric(), device=0, name="w")
    try:
        seen = []
        w = a.alloc_watcher(lambda old, new: seen.append((old, new)), initial=0)
        for v in (1, 2, 5):
            w.store(v)
            time.sleep(0.02)
        st = torch.cuda.current_stream(0)
        _lib.call("txb_stream_write_value64", C.c_void_p(w.device_ptr), 9, C.c_void_p(st.cuda_stream))
        torch.cuda.synchronize()
        t_end = time.monotonic() + 5.0
        while (not seen or seen[-1][1] != 9) and time.monotonic() < t_end:
            time.sleep(0.01)
        news = [n for _, n in seen]
        assert news[-1] == 9 and news == sorted(set(news))
        assert all(o < n for o, n in seen)
        a.free_watcher(w)
    finally:
        a.close()


def test_kv_stream_device_clock_steps_and_bytes():
    """The persistent KV stream (kvcache LayerClock on the device): nothing
    moves before the clock, step k's receipt is released once the compute
    stream advanced the clock to k, and the whole request lands byte for
    byte (check_kvcache, _invariants.py:139-184)."""
    import time
    a, b = _pair()
    try:
        layers, chunks, ppc, page_len, heads = 6, 3, 4, 8192, 2
        layout = kvcache.KvLayout(layers, chunks, ppc, page_len)
        dec = kvcache.KvReceiver(b, layout, pool_slots=layout.slots + 5, local_heads=heads, ctx_bytes=4096)
        t = dec.open_request(ctx_len=512)
        req = t.request
        rid = req.request_id
        kvb = np.zeros(layout.region_bytes(heads, layout.slots), np.uint8)
        for layer in range(layers):
            for j in range(heads):
                for slot in range(layout.slots):
                    idx = layout.page_index(heads, layout.slots, layer, j, slot)
                    kvb[idx * page_len:(idx + 1) * page_len] = np.frombuffer(
                        to.page_bytes(rid, layer, j, slot, page_len), np.uint8)
        kv = a.alloc_buffer(kvb.size)
        kv.copy_(torch.from_numpy(kvb).to(kv.device))
        ctx = a.alloc_buffer(512)
        ctx.copy_(torch.from_numpy(np.frombuffer(to.context_bytes(rid, 512), np.uint8).copy()).to(ctx.device))
        send = kvcache.KvSender(a, kv, ctx)
        # the step lists equal the per-step Pages of step_pages
        si, di = send.step_indices(req)
        pps = heads * ppc
        for k in (1, 7, layout.steps):
            sp, dp = send.step_pages(req, k)
            assert list(si[(k - 1) * pps:k * pps]) == list(sp.indices)
            assert list(di[(k - 1) * pps:k * pps]) == list(dp.indices)
        clock = a.device_clock(layout.steps)
        comp = torch.cuda.Stream(a.device)
        flag = send.stream_all(req, clock, grid=16)
        time.sleep(0.05)
        assert b.imm_received_total(req.imm) == 0, "pages moved before the clock"
        for k in range(1, layout.steps + 1):
            clock.advance(comp)
            comp.synchronize()
            t_end = time.monotonic() + 10.0
            while b.imm_received_total(req.imm) < k and time.monotonic() < t_end:
                time.sleep(0.001)
            assert b.imm_received_total(req.imm) == k, f"step {k} receipt"
        flag.result(30.0)
        assert not t.flag.done()
        send.send_context(req).result(30.0)
        assert t.wait(10.0)
        for layer in range(layers):
            for j in range(heads):
                for i in range(layout.slots):
                    assert dec.page_view(t, layer, j, i).cpu().numpy().tobytes() == \
                        to.page_bytes(rid, layer, j, i, page_len)
        dec.release(t)
        # the retired imm can serve the next request
        t2 = dec.open_request(ctx_len=512)
        assert t2.request.imm != req.imm or not t2.flag.done()
    finally:
        a.close()
        b.close()


def test_kv_stream_cfg5_whole_request_byte_identical():
    """BASELINE configs[4] at full size: Llama-3-70B, 80 layers x 8 KV heads
    x 2048 slots of 8-KiB pages (16-token pages, 32k context) = 10 GiB in
    1280 (chunk, layer) steps, streamed by one persistent kernel into a
    scattered decoder slot list (prefill cuda:0 -> decode cuda:1 when there
    are two GPUs, else HBM loopback).  Every destination page must equal its
    source page (device-side comparison), and the request's receipt count
    must be steps + 1 (context write) exactly."""
    a, b = _pair()
    try:
        layers, chunks, heads, slots, page = 80, 16, 8, 2048, 8192
        layout = kvcache.KvLayout(layers, chunks, slots // chunks, page)
        dec = kvcache.KvReceiver(b, layout, pool_slots=slots, local_heads=heads, ctx_bytes=1 << 16)
        dec._free = list(np.random.default_rng(5).permutation(slots))
        t = dec.open_request(ctx_len=4096)
        total = layout.region_bytes(heads, slots)
        W = page // 8
        kv = a.alloc_buffer(total)
        kv.view(torch.int64).view(-1, W).copy_(
            torch.arange(total // 8, dtype=torch.int64, device=kv.device).view(-1, W))
        send = kvcache.KvSender(a, kv, a.alloc_buffer(4096))
        clock = a.device_clock(layout.steps)
        clock.advance(by=layout.steps)
        send.stream_all(t.request, clock).result(60.0)
        send.send_context(t.request).result(30.0)
        assert t.wait(30.0)
        assert b.imm_received_total(t.request.imm) == layout.steps + 1
        si, di = send.step_indices(t.request)
        dstw = dec.kv.view(torch.int64).view(-1, W)
        col = torch.arange(W, dtype=torch.int64, device=dstw.device)
        for c0 in range(0, si.size, 65536):
            s = torch.from_numpy(si[c0:c0 + 65536]).to(dstw.device)
            d = torch.from_numpy(di[c0:c0 + 65536]).to(dstw.device)
            assert torch.equal(dstw.index_select(0, d), s[:, None] * W + col[None, :]), c0
        dec.release(t)
    finally:
        a.close()
        b.close()
