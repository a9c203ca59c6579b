"""CPU tests of the C-ABI boundary: the library loads without a GPU, exports every
symbol include/spava_b200.h declares, and fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

from paper_2601_21444_b200 import spava

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "spava_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spava_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_python_symbol_list():
    assert declared_symbols() == sorted(spava.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(spava.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert spava.lib().spava_version().decode().startswith("spava-b200")


def test_built_for_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {spava.LIB_PATH} 2>&1").read()
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, out


def test_compute_fails_loudly_without_device():
    """On this CPU container every compute entry point must return SPAVA_ECUDA."""
    if spava.device_ok():
        pytest.skip("a GPU is visible")
    L = spava.lib()
    rc = L.spava_score_block(None, 128, 1, None, 128, 1, None, 1, 1, 1, 128, 1, None, None,
                             1 << 30, None)
    assert rc == spava.ECUDA
    assert "no CPU fallback" in L.spava_last_error().decode()
    cfg = spava.LayerConfig.make(1000, 8, 2, 8, 16, 2, 2)
    with pytest.raises(spava.SpavaError) as e:
        spava.Fabric(cfg, 0)
    assert e.value.code == spava.ECUDA


def test_missing_library_raises(monkeypatch):
    monkeypatch.setattr(spava, "LIB_PATH", "/nonexistent/libspava_b200.so")
    monkeypatch.setattr(spava, "_lib", None)
    with pytest.raises(spava.SpavaError):
        spava.lib()


def test_error_mapping():
    """std::invalid_argument -> EINVAL, std::out_of_range -> ERANGE."""
    with pytest.raises(spava.SpavaError) as e:
        spava.make_plan(10, 1, 2, 10, 0)
    assert e.value.code == spava.EINVAL
    p = spava.make_plan(100, 1, 2, 4, 0)
    with pytest.raises(spava.SpavaError) as e:
        spava.physical_of(p, 4)
    assert e.value.code == spava.ERANGE
