"""The C-ABI library loads and exports every symbol include/qmb200.h declares (no GPU needed)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2011_11762_b200 import _ffi, _build
from paper_2011_11762_b200.layout import MatrixParams

HEADER = Path(__file__).resolve().parent.parent / "include" / "qmb200.h"


def header_symbols():
    return sorted(set(re.findall(r"QM_API\s+[\w\s\*]+?\b(qm_\w+)\s*\(", HEADER.read_text())))


def test_library_is_built_in_tree():
    assert _build.LIB.exists(), "run __graft_entry__.build() first"
    assert _build.LIB.parent.name == "paper_2011_11762_b200"


def test_exports_every_header_symbol():
    lib = _ffi.load()
    names = header_symbols()
    assert len(names) >= 15
    assert sorted(_ffi.EXPORTS) == names
    for name in names:
        assert hasattr(lib, name), name


def test_abi_version_and_host_queries():
    lib = _ffi.load()
    assert lib.qm_abi_version() == _ffi.ABI_VERSION == 2
    lay = _ffi.make_layout(MatrixParams.create(4096, 64), 64)
    assert lib.qm_spgemm_workspace_bytes(ctypes.byref(lay), 556, 556) > 0
    assert lib.qm_compact_workspace_bytes(1016) > 0
    assert [lib.qm_numeric_path(b) for b in (16, 32, 64, 128, 8, 12)] == [2, 2, 2, 2, 0, 0]


def test_invalid_layout_is_reported_not_crashed():
    lib = _ffi.load()
    bad = _ffi.QmLayout(100, 12, 3, 5, 0)  # 5 does not divide 12
    rc = lib.qm_encode_keys(ctypes.byref(bad), None, None, 10, None, None)
    assert rc == _ffi.QM_ERR_INVALID
    assert b"divide" in lib.qm_last_error()
    with pytest.raises(Exception):
        _ffi.check(rc, "qm_encode_keys")


def test_workspace_and_argument_errors_before_any_device_work():
    """Status codes of the C ABI for caller mistakes (no GPU needed: they return before launching)."""
    lib = _ffi.load()
    lay = _ffi.make_layout(MatrixParams.create(4096, 64), 64)
    nc, nt = ctypes.c_int64(-1), ctypes.c_int64(-1)
    rc = lib.qm_spgemm_count(ctypes.byref(lay), None, 10, None, 10, None, 0, ctypes.byref(nc),
                             ctypes.byref(nt), None)
    assert rc == _ffi.QM_ERR_WORKSPACE and b"workspace" in lib.qm_last_error()
    rc = lib.qm_spgemm_count(ctypes.byref(lay), None, -1, None, 10, None, 0, ctypes.byref(nc),
                             ctypes.byref(nt), None)
    assert rc == _ffi.QM_ERR_INVALID
    assert lib.qm_numeric(ctypes.byref(lay), None, None, 0, None, 0, None, None, None, 0, 0, None, None, None,
                          None, None, 0, None) == _ffi.QM_OK  # nC == 0 is a no-op
    assert lib.qm_compact(64, -1, None, None, None, None, None, None, None, None, 0, None) == _ffi.QM_ERR_INVALID
    assert lib.qm_transpose_blocks(64, None, 4, None, None) == _ffi.QM_ERR_INVALID  # in place
    too_deep = _ffi.QmLayout(1 << 40, 1, 40, 1, 0)
    assert lib.qm_spgemm_workspace_bytes(ctypes.byref(too_deep), 1, 1) == 0
    assert lib.qm_encode_keys(ctypes.byref(too_deep), None, None, 1, None, None) == _ffi.QM_ERR_UNSUPPORTED


def test_multi_gpu_and_row_index_entry_points_reject_bad_arguments():
    """Caller mistakes on the staged multi-GPU and row-index entry points return status codes
    before any device work (no GPU needed)."""
    lib = _ffi.load()
    lay = _ffi.make_layout(MatrixParams.create(4096, 64), 64)
    counts = (ctypes.c_int64 * 3)()
    # ownership range outside the operand
    rc = lib.qm_stage_plan(None, 0, None, 0, 5, 3, 10, 0, 0, 10, 0, None, 0, None, None, None, None, counts, None)
    assert rc == _ffi.QM_ERR_INVALID and b"qm_stage_plan" in lib.qm_last_error()
    # b_is_a with different operand sizes
    rc = lib.qm_stage_plan(None, 0, None, 0, 0, 1, 10, 0, 1, 11, 1, None, 0, None, None, None, None, counts, None)
    assert rc == _ffi.QM_ERR_INVALID
    assert lib.qm_stage_plan_workspace_bytes(100, 100, 10, 0) > lib.qm_stage_plan_workspace_bytes(100, 100, 10, 1)
    # one operand's masks without the other's
    ia = _ffi.QmRowIndex(0, 0, 0, 0, 8)
    ib = _ffi.QmRowIndex(0, 0, 0, 0, 0)
    nc, nt = ctypes.c_int64(-1), ctypes.c_int64(-1)
    rc = lib.qm_spgemm_count_ix(ctypes.byref(lay), ctypes.byref(ia), 1, ctypes.byref(ib), 1, 0, 0, 0, None, 0,
                                ctypes.byref(nc), ctypes.byref(nt), None, None, None)
    assert rc == _ffi.QM_ERR_INVALID and b"masks" in lib.qm_last_error()
    # a halo with more ranks than the ABI carries
    h = _ffi.QmHalo()
    h.world = 9
    h.count[0] = 1
    one = (ctypes.c_void_p * 1)(8)
    n1 = (ctypes.c_int64 * 1)(1)
    rc = lib.qm_numeric_pools_ex(ctypes.byref(lay), one, n1, 1, one, n1, 1, None, None, None, None, None, None, None,
                                 ctypes.byref(h), 0, None, 1, 1, None, None, None, None, None, None, 0, None)
    assert rc == _ffi.QM_ERR_INVALID and b"halo" in lib.qm_last_error()
    assert lib.qm_row_index_workspace_bytes(ctypes.byref(lay), 1000) > 0


def test_numeric_kernel_selection(monkeypatch):
    """qm_numeric_kernel names the kernel qm_numeric launches: grouped C blocks (bs 16 groups, bs 32
    quads) only for products with long enough k lists, per-block kernels otherwise (host query)."""
    for v in ("QM_QUAD32", "QM_G16_GROUPS", "QM_NUMERIC"):
        monkeypatch.delenv(v, raising=False)
    lib = _ffi.load()

    def kernel(n, leaf, bs, n_c, n_t, masked=0, flags=0):
        lay = _ffi.make_layout(MatrixParams.create(n, leaf), bs)
        return lib.qm_numeric_kernel(ctypes.byref(lay), n_c, n_t, masked, flags).decode()

    assert kernel(1 << 20, 64, 64, 1063904, 17827216) == "k_numeric_tma"        # C5-64
    assert kernel(1 << 20, 32, 32, 4227008, 138330400) == "k_numeric_quad32"    # C5-32: 33 triples per block
    assert kernel(65536, 32, 32, 63720, 65536) == "k_numeric_tma"               # random: ~1 triple per block
    assert kernel(1 << 20, 32, 32, 4227008, 138330400, masked=1) == "k_numeric_tma"
    assert kernel(1 << 20, 32, 32, 4227008, 138330400, flags=1) == "k_numeric_tma"  # transposed references
    assert kernel(65536, 128, 32, 1000, 100000) == "k_numeric_tma"              # 4x4 blocks per leaf: no quads
    assert kernel(32768, 128, 16, 132064, 2215312) == "k_numeric_group16"       # banded, leaf 128
    assert kernel(32768, 128, 16, 128694, 130472) == "k_numeric_dmma"           # random
    assert kernel(32768, 16, 16, 132064, 2215312) == "k_numeric_dmma"           # one block per leaf
    assert kernel(4800, 48, 12, 100, 1000) == "k_numeric_generic"
    monkeypatch.setenv("QM_QUAD32", "0")
    assert kernel(1 << 20, 32, 32, 4227008, 138330400) == "k_numeric_tma"
    monkeypatch.setenv("QM_G16_GROUPS", "1")
    assert kernel(32768, 128, 16, 128694, 130472) == "k_numeric_group16"
