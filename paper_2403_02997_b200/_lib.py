"""ctypes binding of libtricount_b200.so (the C ABI in include/tricount_b200.h).

This is the only route to compute in the package: there is no CPU fallback.
If the library or a CUDA device is missing, every compute call raises.
PyTorch supplies device memory and streams; arguments crossing the ABI are
plain pointers and sizes.
"""
from __future__ import annotations

import ctypes
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libtricount_b200.so"
HEADER_PATH = Path(__file__).resolve().parents[1] / "include" / "tricount_b200.h"

TCB_OK = 0
TCB_ERR_INVALID = 1
TCB_ERR_CUDA = 2
TCB_ERR_NOMEM = 3
TCB_ERR_ASSERT = 4
TCB_ERR_INTERNAL = 5

STAGES = ("components", "bfs", "select", "intersect", "h2d", "d2h", "isect_cta", "isect_hub")


class TcbResult(ctypes.Structure):
    _fields_ = [
        ("triangles", ctypes.c_int64),
        ("c1", ctypes.c_int64),
        ("c2", ctypes.c_int64),
        ("ncover", ctypes.c_int64),
        ("components", ctypes.c_int64),
        ("max_level", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


_lib = None
_lib_lock = threading.Lock()


def load_library(path: Path | None = None):
    """Load the shared library and declare every exported signature."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        import os
        p = Path(path or os.environ.get("TCB_LIBRARY") or LIB_PATH)
        if not p.exists():
            raise RuntimeError(
                f"libtricount_b200.so not found at {p}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(str(p))
        vp = ctypes.c_void_p
        i64 = ctypes.c_int64
        u64 = ctypes.c_uint64
        i32 = ctypes.c_int
        pi64 = ctypes.POINTER(ctypes.c_int64)
        sigs = {
            "tcb_version": ([], i32),
            "tcb_context_create": ([i32, vp, ctypes.POINTER(vp)], i32),
            "tcb_context_destroy": ([vp], i32),
            "tcb_context_set_stream": ([vp, vp], i32),
            "tcb_last_error": ([vp], ctypes.c_char_p),
            "tcb_launch_count": ([vp], i64),
            "tcb_set_timing": ([vp, i32], i32),
            "tcb_set_tuning": ([vp, i32, i32], i32),
            "tcb_set_test_flags": ([vp, i32], i32),
            "tcb_stage_times": ([vp, ctypes.POINTER(ctypes.c_float), i32], i32),
            "tcb_level_records": ([vp, pi64, i32], i32),
            "tcb_rmat_generate": ([vp, i32, i64, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_double, u64, u64, u64, u64, vp, vp], i32),
            "tcb_er_generate": ([vp, i64, ctypes.c_double, u64, u64, u64, u64, vp, pi64], i32),
            "tcb_lattice_generate": ([vp, i64, vp], i32),
            "tcb_csr_build": ([vp, vp, i64, i64, vp, vp, vp, vp, vp, pi64], i32),
            "tcb_csr_rows": ([vp, vp, i64, vp], i32),
            "tcb_copy_to_device": ([vp, vp, vp, i64], i32),
            "tcb_split_by_level": ([vp, vp, vp, vp, i64, i64, vp, vp, vp, vp,
                                    ctypes.POINTER(ctypes.c_int64)], i32),
            "tcb_split_cross_count": ([vp, vp, vp, vp, i64, i64, vp,
                                       ctypes.POINTER(ctypes.c_int64)], i32),
            "tcb_csr_edges": ([vp, vp, vp, i64, i64, vp, vp], i32),
            "tcb_bfs_levels": ([vp, vp, vp, vp, i64, i64, vp, pi64, pi64], i32),
            "tcb_bfs_parent": ([vp, vp, vp, i64, vp, i64, vp], i32),
            "tcb_edge_classes": ([vp, vp, vp, vp, i64, i64, vp, vp, vp], i32),
            "tcb_cover_select": ([vp, vp, vp, vp, i64, vp, vp, pi64], i32),
            "tcb_cetc_count": ([vp, vp, vp, vp, i64, vp, vp, i64, i64, pi64], i32),
            "tcb_cetc_count_restricted": ([vp, vp, vp, vp, i64, vp, vp, i64, i64, i64, pi64],
                                          i32),
            "tcb_cetc": ([vp, vp, vp, vp, i64, i64, vp, vp, vp,
                          ctypes.POINTER(TcbResult)], i32),
            "tcb_cetc_shard": ([vp, vp, vp, vp, i64, i64, i32, i32,
                                ctypes.POINTER(TcbResult)], i32),
            "tcb_forward_count": ([vp, vp, vp, vp, i64, i64, pi64], i32),
            "tcb_cetc_fe": ([vp, vp, vp, vp, i64, i64, ctypes.c_double,
                             ctypes.POINTER(TcbResult), ctypes.POINTER(ctypes.c_int32)], i32),
            "tcb_degree_order": ([vp, vp, vp, vp, i64, i64, vp, vp, vp], i32),
            "tcb_cetc_host": ([vp, vp, vp, i64, vp, ctypes.POINTER(TcbResult)], i32),
            "tcb_cetc_host_shard": ([vp, vp, vp, i64, i32, i32, ctypes.POINTER(TcbResult)], i32),
        }
        for name, (args, res) in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


def header_symbols() -> list[str]:
    """Function names declared TCB_API in include/tricount_b200.h."""
    import re
    text = HEADER_PATH.read_text()
    return re.findall(r"TCB_API\s+[\w\s\*]+?\b(tcb_\w+)\s*\(", text)


class TcbError(RuntimeError):
    pass


def _raise(code: int, msg: str):
    if code == TCB_ERR_INVALID:
        raise ValueError(msg)
    if code == TCB_ERR_ASSERT:
        raise AssertionError(msg)
    if code == TCB_ERR_NOMEM:
        raise MemoryError(msg)
    raise TcbError(f"tcb error {code}: {msg}")


class Context:
    """One libtricount_b200 context (workspace + stream) per device per thread."""

    def __init__(self, device: int):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2403_02997_b200 needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.device = device
        h = ctypes.c_void_p()
        with torch.cuda.device(device):
            stream = torch.cuda.current_stream(device).cuda_stream
            rc = self.lib.tcb_context_create(device, ctypes.c_void_p(stream), ctypes.byref(h))
        if rc != TCB_OK:
            _raise(rc, "tcb_context_create failed")
        self.h = h

    def sync_stream(self):
        import torch
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self.check(self.lib.tcb_context_set_stream(self.h, ctypes.c_void_p(stream)))

    def check(self, rc: int):
        if rc != TCB_OK:
            msg = self.lib.tcb_last_error(self.h)
            _raise(rc, msg.decode() if msg else "")

    def launches(self) -> int:
        return int(self.lib.tcb_launch_count(self.h))

    def set_timing(self, on: bool):
        self.check(self.lib.tcb_set_timing(self.h, int(bool(on))))

    def set_test_flags(self, flags: int = 0):
        """Test hook: force rarely taken device paths (tcb_set_test_flags)."""
        self.check(self.lib.tcb_set_test_flags(self.h, int(flags)))

    def set_tuning(self, warp_tier_max_degree: int = 0, cta_stage_max: int = 0):
        """Intersection work-split knobs (0 = defaults); results are unchanged."""
        self.check(self.lib.tcb_set_tuning(self.h, int(warp_tier_max_degree),
                                           int(cta_stage_max)))

    def stage_times(self) -> dict:
        arr = (ctypes.c_float * len(STAGES))()
        self.check(self.lib.tcb_stage_times(self.h, arr, len(STAGES)))
        return {k: float(arr[i]) for i, k in enumerate(STAGES)}

    def level_records(self) -> list[tuple[str, float, int]]:
        """Per-level BFS records of the last call (diagnostics):
        (mode "TD"/"BU", step end in us from the BFS start, next frontier)."""
        cap = 64
        arr = (ctypes.c_int64 * (3 * cap))()
        k = int(self.lib.tcb_level_records(self.h, arr, cap))
        if k < 0:
            self.check(-k)
        return [("BU" if arr[3 * i] else "TD", arr[3 * i + 1] / 1e3, int(arr[3 * i + 2]))
                for i in range(k)]

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.tcb_context_destroy(self.h)
        except Exception:
            pass


_tls = threading.local()


def context(device: int | None = None) -> Context:
    """The calling thread's context for `device` (default: current CUDA device),
    bound to torch's current stream."""
    import torch
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2403_02997_b200 needs a CUDA device (no CPU fallback)")
        device = torch.cuda.current_device()
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    ctx = ctxs.get(device)
    if ctx is None:
        ctx = ctxs[device] = Context(device)
    ctx.sync_stream()
    return ctx


def ptr(t) -> ctypes.c_void_p:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(t.data_ptr())
