"""The C ABI: the library loads without a GPU and exports exactly the
functions include/tricount_b200.h declares (no compute calls here)."""
from __future__ import annotations

import ctypes
import subprocess

import pytest

from paper_2403_02997_b200 import _lib


def test_header_declares_entry_points():
    syms = _lib.header_symbols()
    for s in ("tcb_csr_build", "tcb_bfs_levels", "tcb_cover_select", "tcb_cetc_count",
              "tcb_cetc", "tcb_cetc_host", "tcb_rmat_generate", "tcb_context_create"):
        assert s in syms


def test_library_loads_and_exports_header_symbols():
    if not _lib.LIB_PATH.exists():
        pytest.fail("libtricount_b200.so missing: run __graft_entry__.build()")
    L = _lib.load_library()
    for s in _lib.header_symbols():
        assert hasattr(L, s), s
    assert L.tcb_version() == 6
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert exported == set(_lib.header_symbols())


def test_library_targets_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_null_context_is_rejected():
    L = _lib.load_library()
    assert L.tcb_context_set_stream(None, None) == _lib.TCB_ERR_INVALID
    assert L.tcb_launch_count(None) == -1
    assert L.tcb_last_error(None) == b"null context"


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import numpy as np
    import paper_2403_02997_b200 as tb
    with pytest.raises(RuntimeError, match="CUDA"):
        tb.normalize(tb.EdgeList(n=3, edges=np.array([[0, 1], [1, 2], [0, 2]])))


@pytest.mark.gpu
def test_size_ceiling_is_rejected():
    """n >= 2^31 or 2m >= 2^31 fails with TCB_ERR_INVALID before any launch
    (common.cuh require_sizes), instead of overflowing the 32-bit layout."""
    from paper_2403_02997_b200 import _lib
    ctx = _lib.context(0)
    lib = ctx.lib
    assert lib.tcb_bfs_levels(ctx.h, None, None, None, 1 << 31, 0, None, None, None) == 1
    assert lib.tcb_bfs_levels(ctx.h, None, None, None, 16, 1 << 30, None, None, None) == 1
    assert lib.tcb_cover_select(ctx.h, None, None, None, 1 << 30, None, None, None) == 1
    assert b"2^31" in lib.tcb_last_error(ctx.h)
    # the host-buffer entries check m from the row offsets too
    import ctypes
    import numpy as np
    row = np.array([0, 1 << 31], dtype=np.int64)
    r = _lib.TcbResult()
    assert lib.tcb_cetc_host(ctx.h, row.ctypes.data_as(ctypes.c_void_p), None, 1, None,
                             ctypes.byref(r)) == 1
    assert lib.tcb_cetc_host_shard(ctx.h, row.ctypes.data_as(ctypes.c_void_p), None, 1, 0, 1,
                                   ctypes.byref(r)) == 1
    bad = np.array([0, -2], dtype=np.int64)
    assert lib.tcb_cetc_host(ctx.h, bad.ctypes.data_as(ctypes.c_void_p), None, 1, None,
                             ctypes.byref(r)) == 1
    two = np.array([0, 2], dtype=np.int64)
    assert lib.tcb_cetc_host(ctx.h, two.ctypes.data_as(ctypes.c_void_p), None, 1, None,
                             ctypes.byref(r)) == 1  # null neighbours
