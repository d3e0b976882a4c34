"""CPU-side checks of the drop-in boundary: the C-ABI library loads without a GPU and exports
every entry point include/lfdg.h declares; the Python mirror binds all of them."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "lfdg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lfdg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1812_06856_b200 import _native

    lib = os.path.join(ROOT, "paper_1812_06856_b200", "liblfdg.so")
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (lfdg_[a-z0-9_]+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, f"declared but not exported: {missing}"
    L = ctypes.CDLL(lib)  # loads without a GPU
    for s in declared_symbols():
        assert hasattr(L, s)
    assert set(declared_symbols()) == set(_native.EXPORTED)


def test_python_binding_covers_abi():
    from paper_1812_06856_b200 import _native

    L = _native.lib()
    for s in declared_symbols():
        assert getattr(L, s).argtypes is not None or s in ("lfdg_last_error",), s


def test_no_gpu_raises_cleanly():
    """Without a device the context constructor fails loudly (no CPU fallback)."""
    import pytest

    from conftest import has_gpu
    from paper_1812_06856_b200 import api

    if has_gpu():
        pytest.skip("GPU present")
    with pytest.raises(api.LfdgError):
        api.DeviceContext(0)


def test_sm100a_code_in_library():
    lib = os.path.join(ROOT, "paper_1812_06856_b200", "liblfdg.so")
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
