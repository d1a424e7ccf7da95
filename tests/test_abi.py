"""CPU suite: the C-ABI library loads and exports every declared entry point."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "shardplan_gpu.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*|uint64_t)\s+(rs_\w+)\s*\(", src, re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("rs_profile_run", "rs_build_remap", "rs_simulate", "rs_emb_forward",
                 "rs_emb_backward", "rs_hash_value", "rs_build_icdf", "rs_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2201_10095_b200 import _lib

    L = _lib.lib()
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, missing
    assert set(declared_functions()) <= set(_lib.EXPORTS)
    assert L.rs_abi_version() == 1


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2201_10095_b200", "libshardplan_gpu.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_host_only_entry_points_without_gpu():
    """hash_value and hash_utilization need no device."""
    from paper_2201_10095_b200 import _lib

    L = _lib.lib()
    out = ctypes.c_uint32()
    assert L.rs_hash_value(42, 1 << 32, ctypes.byref(out)) == 0 and out.value == 3564271138
    assert L.rs_hash_value(7, 1000, ctypes.byref(out)) == 0 and out.value == 604
    assert L.rs_hash_value(1, 0, ctypes.byref(out)) == _lib.RS_ERR_INVALID_ARGUMENT
    assert b"hash_size" in L.rs_last_error()
    s, c = ctypes.c_double(), ctypes.c_double()
    assert L.rs_hash_utilization(1, 1, 2, ctypes.byref(s), ctypes.byref(c)) == 0
    assert s.value == 0.0 and c.value == 1.0  # tests/test_profiler.cpp:202-209


def test_python_api_mirrors_reference_names():
    import paper_2201_10095_b200 as p

    for n in ("profile", "build_icdf", "hash_utilization", "hash_value", "build_remap",
              "translate", "simulate", "TieredEmbeddingBag"):
        assert hasattr(p, n)
    assert p.hash_value(42, 1 << 32) == 3564271138
    with pytest.raises(p.InvalidArgument):
        p.hash_value(1, 0)
