"""CPU-side checks of the C ABI: the library loads, exports every symbol
declared in include/txb200.h, and the host-only planning call matches the
reference's RoutingSpec validation and capacity arithmetic."""

from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "txb200.h"
LIB = ROOT / "paper_2510_27656_b200" / "libtxb200.so"


def _declared() -> set[str]:
    txt = HEADER.read_text()
    return set(re.findall(r"^\s*(?:const char\*|int)\s+(txb_\w+)\s*\(", txt, re.M))


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists():
        subprocess.run(["make", "-C", str(ROOT)], check=True)
    from paper_2510_27656_b200 import _lib
    return _lib.load()


def test_header_declares_abi():
    names = _declared()
    assert {"txb_moe_route", "txb_moe_dispatch", "txb_moe_dispatch_recv", "txb_moe_combine_send",
            "txb_moe_combine_recv", "txb_last_error"} <= names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (txb_\w+)", out))
    missing = _declared() - exported
    assert not missing, f"declared but not exported: {sorted(missing)}"


def test_binding_covers_header(lib):
    from paper_2510_27656_b200 import _lib
    assert _declared() == set(_lib.SIGNATURES), "ctypes signature table out of sync with txb200.h"
    for name in _declared():
        assert hasattr(lib, name)


def test_sm100a_code_present():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _plan(**kw):
    from paper_2510_27656_b200 import _lib
    sh = _lib.Shape(**kw)
    rc = _lib.load().txb_moe_plan(C.byref(sh))
    return rc, sh


def test_plan_matches_reference_spec_arithmetic(lib):
    rc, sh = _plan(ranks=8, experts=256, max_tokens=128, topk=8, hidden=7168, elem_size=1,
                   scales=56, me=3)
    assert rc == 0
    assert sh.local_experts == 32
    assert sh.payload_bytes == 7168 + 4 * 56 == 7392
    assert sh.capacity == 8 * 128 * 32          # moe.py:80-83
    assert sh.comb_bytes == sh.payload_bytes   # default combine format = dispatch format
    assert sh.grouped_rows == 8 * 128 * 8 + 32 * 7
    assert sh.off_grouped % 4096 == 0 and sh.off_comb % 4096 == 0
    assert sh.region_bytes >= sh.off_comb + sh.comb_rows * sh.comb_bytes


@pytest.mark.parametrize("kw,msg", [
    (dict(ranks=0, experts=4, max_tokens=1, topk=1, hidden=1, elem_size=4), "rank count must be positive"),
    (dict(ranks=3, experts=4, max_tokens=1, topk=1, hidden=1, elem_size=4), "not a positive multiple"),
    (dict(ranks=1, experts=4, max_tokens=1, topk=5, hidden=1, elem_size=4), "topk 5 outside 1..4"),
    (dict(ranks=1, experts=4, max_tokens=0, topk=1, hidden=1, elem_size=4), "max_tokens must be positive"),
    (dict(ranks=1, experts=4, max_tokens=1, topk=1, hidden=1, elem_size=3), "element size 3"),
    (dict(ranks=1, experts=4, max_tokens=1, topk=1, hidden=1, elem_size=1, scales=0), "at least one scale"),
])
def test_plan_validation_messages(lib, kw, msg):
    from paper_2510_27656_b200 import _lib
    rc, _ = _plan(**kw)
    assert rc == _lib.TXB_ERR_PROTOCOL
    assert msg in _lib.last_error()
