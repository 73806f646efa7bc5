"""The C-ABI library loads and exports every symbol include/vdmc.h declares; host-side
argument checking and the host planner work without a GPU (-m "not gpu")."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def vd():
    from paper_2201_11655_b200 import build as b
    b.build()
    from paper_2201_11655_b200 import vdmc
    return vdmc


def header_symbols():
    src = open(os.path.join(ROOT, "include", "vdmc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vdmc_[a-z_0-9]+)\s*\(", src)))


def test_exports_match_header(vd):
    syms = header_symbols()
    assert sorted(vd.EXPORTS) == syms
    out = subprocess.run(["nm", "-D", "--defined-only", vd.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (vdmc_\w+)", out))
    for s in syms:
        assert s in exported, s
    for s in syms:
        assert hasattr(vd.lib(), s)


def test_library_is_sm100a(vd):
    out = subprocess.run(["cuobjdump", "--list-elf", vd.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_class_ids_match_oracle(vd, oracle_mod):
    for k in (3, 4):
        assert vd.num_classes(k) == len(oracle_mod.class_table(k)["class_ids"])
        assert np.array_equal(vd.class_ids(k).astype(np.int64), oracle_mod.class_table(k)["class_ids"])
    assert vd.num_classes(6) == -1 and vd.num_classes(2) == -1
    with pytest.raises(vd.VdmcError, match="VDMC_EK"):
        vd.class_ids(6)


def test_class_ids_k5_match_oracle(vd, oracle_mod):
    """k = 5 (NEXT-3): the library's 16-bit table (host-built, 2^20 masks) lists the same 9364
    directed classes as the oracle; 21 undirected (OEIS A001349) = the oracle's all-mutual classes."""
    assert vd.num_classes(5) == 9364 and vd.num_classes(5, "undirected") == 21
    assert np.array_equal(vd.class_ids(5).astype(np.int64), oracle_mod.class_table(5)["class_ids"])
    assert np.array_equal(vd.class_ids(5, "undirected").astype(np.int64), oracle_mod.undirected_class_ids(5))


def test_options_validated_without_gpu(vd):
    """vdmc_count_ex checks k and every option before touching the graph or a device."""
    lib = vd.lib()
    for bad in ({"star_block": 5000}, {"cross_block": 7}, {"heavy_global": 3}, {"force_big": -1},
                {"ca_capacity": -5}, {"layered": 2}):
        o, _ = vd._options("directed", bad, None)
        assert vd.STATUS[lib.vdmc_count_ex(None, 4, None, None, vd.ctypes.byref(o), None)] == "VDMC_EINVAL", bad
    o, _ = vd._options("directed", {}, None)
    assert vd.STATUS[lib.vdmc_count_ex(None, 6, None, None, vd.ctypes.byref(o), None)] == "VDMC_EK"
    assert vd.STATUS[lib.vdmc_count_ex(None, 4, None, None, vd.ctypes.byref(o), None)] == "VDMC_EINVAL"   # NULL graph
    assert vd.STATUS[lib.vdmc_count_edges(None, 5, None, None, vd.ctypes.byref(o), None)] == "VDMC_EK"


def _build(vd, n, s, d, rank=None):
    h = ctypes.c_void_p()
    s = np.ascontiguousarray(s, np.int32)
    d = np.ascontiguousarray(d, np.int32)
    rk = None if rank is None else np.ascontiguousarray(rank, np.int32)
    st = vd.lib().vdmc_build_graph_edges(n, s.size, s.ctypes.data if s.size else None,
                                         d.ctypes.data if d.size else None, 0,
                                         rk.ctypes.data if rk is not None else None, 0, None, ctypes.byref(h))
    return st, vd.lib().vdmc_last_error().decode()


def test_host_validation_errors(vd):
    st, msg = _build(vd, 3, [0, 1], [1, 1])
    assert vd.STATUS[st] == "VDMC_ESELFLOOP" and "vertex 1" in msg
    st, msg = _build(vd, 3, [0], [7])
    assert vd.STATUS[st] == "VDMC_ERANGE" and "7" in msg
    st, _ = _build(vd, 1 << 30, [], [])
    assert vd.STATUS[st] == "VDMC_EINVAL"
    st, _ = _build(vd, 3, [0], [1], rank=[0, 0, 1])
    assert vd.STATUS[st] == "VDMC_EORDER"


def test_sym_csr_validation(vd):
    lib = vd.lib()
    h = ctypes.c_void_p()
    # 0 -> 1 recorded on 0's side only: no mirror
    ip = np.array([0, 1, 1], np.int64)
    nb = np.array([1], np.int32)
    dc = np.array([1], np.uint8)
    st = lib.vdmc_build_graph(2, ip.ctypes.data, nb.ctypes.data, dc.ctypes.data, None, 0, ctypes.byref(h))
    assert vd.STATUS[st] == "VDMC_EASYM"
    # mirror present but code not swapped
    ip = np.array([0, 1, 2], np.int64)
    nb = np.array([1, 0], np.int32)
    dc = np.array([1, 1], np.uint8)
    st = lib.vdmc_build_graph(2, ip.ctypes.data, nb.ctypes.data, dc.ctypes.data, None, 0, ctypes.byref(h))
    assert vd.STATUS[st] == "VDMC_EASYM"
    dc = np.array([1, 0], np.uint8)
    st = lib.vdmc_build_graph(2, ip.ctypes.data, nb.ctypes.data, dc.ctypes.data, None, 0, ctypes.byref(h))
    assert vd.STATUS[st] == "VDMC_EINVAL"
    ip = np.array([0, 1, 0], np.int64)
    st = lib.vdmc_build_graph(2, ip.ctypes.data, nb.ctypes.data, dc.ctypes.data, None, 0, ctypes.byref(h))
    assert vd.STATUS[st] == "VDMC_EINVAL"


def test_count_rejects_bad_k_and_null(vd):
    lib = vd.lib()
    assert vd.STATUS[lib.vdmc_count(None, 6, None, None, None)] == "VDMC_EK"
    assert vd.STATUS[lib.vdmc_count(None, 4, None, None, None)] == "VDMC_EINVAL"
    assert vd.STATUS[lib.vdmc_count(None, 5, None, None, None)] == "VDMC_EINVAL"   # k = 5 accepted (NEXT-3)


def test_no_device_fails_loudly(vd):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    st, msg = _build(vd, 3, [0, 1], [1, 2])
    assert vd.STATUS[st] == "VDMC_ENODEV", msg


@pytest.mark.parametrize("nparts", [1, 2, 3, 8])
def test_split_costs_partition(vd, nparts):
    rng = np.random.default_rng(nparts)
    cost = rng.integers(1, 1000, size=997)
    cost[:5] = 10 ** 6                        # heavy hub tasks first, like degree order
    prefix = np.cumsum(cost)
    parts = vd.split_costs(prefix, nparts)
    assert parts[0][0] == 0 and parts[-1][1] == cost.size
    for (a, b), (c, d) in zip(parts, parts[1:]):
        assert b == c and a <= b
    total = prefix[-1]
    for (a, b) in parts:
        share = (prefix[b - 1] if b else 0) - (prefix[a - 1] if a else 0)
        assert share <= total / nparts + cost.max()
    assert vd.split_costs(np.zeros(0, np.int64), nparts) == [(0, 0)] * nparts
