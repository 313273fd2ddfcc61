"""INTEGRATION.md's stand-alone ctypes stub must lay out txb_moe_shape and
txb_moe_bufs exactly as the library binding (_lib.py) does, field for field
and byte for byte; a stub that drifts from the ABI would pass mis-laid
structs to txb_moe_dispatch_fused."""

from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

from paper_2510_27656_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def _stub_classes() -> dict:
    text = (ROOT / "INTEGRATION.md").read_text()
    code = "\n".join(re.findall(r"```python\n(.*?)```", text, re.S))
    src = []
    for name in ("Shape", "Bufs"):
        m = re.search(rf"^class {name}\(C\.Structure\):.*?(?=^\S)", code + "\nEND\n", re.S | re.M)
        assert m, f"class {name} missing from INTEGRATION.md"
        src.append(m.group(0))
    ns: dict = {"C": C}
    exec("\n".join(src), ns)  # noqa: S102  (our own documentation)
    return ns


def _layout(cls) -> list:
    return [(f[0], f[1], getattr(cls, f[0]).offset) for f in cls._fields_]


def test_integration_stub_matches_abi():
    ns = _stub_classes()
    for name, ref in (("Shape", _lib.Shape), ("Bufs", _lib.Bufs)):
        stub = ns[name]
        assert C.sizeof(stub) == C.sizeof(ref), name
        assert _layout(stub) == _layout(ref), name


def test_header_declares_the_same_fields():
    """include/txb200.h declares the struct fields in the binding's order."""
    h = (ROOT / "include" / "txb200.h").read_text()
    for cname, ref in (("txb_moe_shape", _lib.Shape), ("txb_moe_bufs", _lib.Bufs)):
        body = re.search(rf"typedef struct {cname} \{{(.*?)\}} {cname};", h, re.S).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        names = re.findall(r"\b([a-z_][a-z0-9_]*)\s*(?=[,;])", body)
        assert names == [f[0] for f in ref._fields_], cname
