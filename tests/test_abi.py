"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, exports every symbol
include/dawn.h declares, and its host-only logic (validation, shard rule) behaves."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2208_04514_b200 as dawn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dawn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dawn_[a-z_0-9]+)\s*\(", src)))


def test_builds_and_exports_every_declared_symbol():
    dawn.build()
    L = ctypes.CDLL(dawn._LIB)
    names = _declared()
    assert len(names) >= 10
    for n in names:
        assert hasattr(L, n), n
    assert dawn.version().endswith("sm_100a")
    hdr = open(os.path.join(ROOT, "include", "dawn.h")).read()
    assert f"#define DAWN_MS_BATCH {dawn.MS_BATCH}" in hdr


def test_sass_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", dawn._LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_workspace_bytes_limits():
    L = dawn.lib()
    assert L.dawn_workspace_bytes(1000, 8000, 0) > 0
    assert L.dawn_workspace_bytes(0, 0, 0) == 0
    assert L.dawn_workspace_bytes(10, 1 << 32, 1) == 0
    assert L.dawn_workspace_bytes(1 << 31, 10, 1) == 0
    assert L.dawn_workspace_bytes(1000, 8000, 1) <= L.dawn_workspace_bytes(1000, 8000, 0)


def test_host_validation_errors_before_device_work():
    L = dawn.lib()
    h = ctypes.c_void_p()
    assert L.dawn_graph_load_csr(0, 0, None, None, None, None, 0, None, 0, None,
                                 ctypes.byref(h)) == 1
    assert L.dawn_graph_load_csr(10, 5, None, None, None, None, 0, None, 0, None,
                                 ctypes.byref(h)) == 1
    assert L.dawn_graph_load_csr(10, 1 << 32, 1, 1, None, None, 0, 256, 1 << 40, None,
                                 ctypes.byref(h)) == 4
    assert L.dawn_graph_load_csr(10, 5, 256, 256, None, None, 0x100, 256, 1 << 40, None,
                                 ctypes.byref(h)) == 1
    assert L.dawn_graph_load_csr(10, 5, 256, 256, None, None, 0, 256, 10, None,
                                 ctypes.byref(h)) == 5
    assert b"workspace" in L.dawn_last_error()
    assert L.dawn_sssp(None, 0, 0, None, None, None) == 1
    assert L.dawn_sssp_batch(None, None, 4, 0, None, None, None) == 1
    assert L.dawn_sssp_batch(None, None, -1, 0, None, None, None) == 1
    assert L.dawn_graph_destroy(None) == 0
    assert L.dawn_graph_check(None, None) == 1
    assert L.dawn_largest_wcc(None, None, None, None, None) == 1
    assert L.dawn_msssp(None, None, 1, None, None, None) == 1


def test_lean_workspace_is_smaller():
    # DAWN_GRAPH_LEAN (PAPER L312-323 memory frugality): C4-sized graph
    L = dawn.lib()
    n, m = 1 << 24, 520_745_006
    full, lean = L.dawn_workspace_bytes(n, m, 1), L.dawn_workspace_bytes(n, m, 1 | 8)
    assert lean < full / 3, (full, lean)
    assert lean < 1.3e9, lean


@pytest.mark.parametrize("k,world", [(0, 1), (1, 1), (64, 2), (130, 2), (173778, 8), (200, 3)])
def test_apsp_shard_rule_partitions(k, world):
    parts = [dawn.apsp_shard(k, r, world) for r in range(world)]
    allidx = np.sort(np.concatenate(parts)) if k else np.zeros(0)
    assert np.array_equal(allidx, np.arange(k))
    for r, p in enumerate(parts):
        assert np.all(np.diff(p) > 0)
        assert np.all((p // dawn.MS_BATCH) % world == r)
    sizes = [len(p) for p in parts]
    assert sizes[0] == max(sizes)
    assert max(sizes) - min(sizes) <= dawn.MS_BATCH
    with pytest.raises(dawn.DawnError):
        dawn.apsp_shard(k, world, world)


def test_persistent_kernels_have_no_stack_frame():
    # A cooperative kernel with a stack frame (register spills) running next to other
    # cooperative launches (dawn_sssp_batch lanes) faulted or hung intermittently on B200 while
    # the spill-free build never did: every kernel must stay at STACK:0 / LOCAL:0.
    import subprocess
    dawn.build()
    out = subprocess.run(["cuobjdump", "-res-usage", dawn._LIB], capture_output=True,
                         text=True).stdout
    funcs = re.findall(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:\d+ LOCAL:(\d+)", out)
    assert len(funcs) >= 10
    bad = [(f, st, lo) for f, _, st, lo in funcs if st != "0" or lo != "0"]
    assert not bad, bad
    names = " ".join(f for f, *_ in funcs)
    for k in ("k_sssp", "k_ms64", "k_narrow", "k_wsssp", "k_part_level", "k_small"):
        assert k in names, k
