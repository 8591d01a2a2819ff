"""CPU-side checks of the C ABI: the library builds for sm_100a and exports every declared symbol."""

import re
import subprocess
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent


def _declared():
    text = (REPO / "include" / "hapigpu.h").read_text()
    return sorted(set(re.findall(r"\b(hg_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2504_03683_b200 import native

    lib = native.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", str(lib)], text=True)
    exported = set(re.findall(r" T (hg_[a-z_0-9]+)", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    assert set(native.EXPORTED) == set(_declared())


def test_library_loads_and_reports_abi_version():
    from paper_2504_03683_b200 import native

    native.build()
    L = native.lib()
    assert L.hg_abi_version() == 1


def test_cubin_is_sm100a():
    from paper_2504_03683_b200 import native

    lib = native.build()
    out = subprocess.check_output(["cuobjdump", "--list-elf", str(lib)], text=True)
    assert "sm_100a" in out
