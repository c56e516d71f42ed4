"""The C ABI (include/accelgen_b200.h) is what the built library exports and what the ctypes layer binds:
every AG_API declaration is exported by libaccelgen_b200.so (no GPU needed to dlopen it)."""
import ctypes
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _declared() -> set[str]:
    src = (ROOT / "include" / "accelgen_b200.h").read_text()
    return set(re.findall(r"AG_API\s+[\w\s\*]+?\b(ag_\w+)\s*\(", src))


def test_header_matches_binding_table():
    from paper_2503_13737_b200 import _lib
    assert _declared() == set(_lib.exported_symbols())


def test_library_exports_every_declared_symbol():
    from paper_2503_13737_b200.build import build
    lib = ctypes.CDLL(str(build()))  # in-tree nvcc build (no-op when up to date)
    missing = [n for n in sorted(_declared()) if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.ag_version() >= 1
