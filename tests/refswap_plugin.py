"""pytest plugin: the reference's own test suite with its cover-edge path
swapped for the GPU one (registry swap).

Loaded with ``-p refswap_plugin`` by tests/test_reference_harness.py when an
installed copy of the reference (``baseline/_ref``: ``pip install --target``,
plus its tests and data, git-ignored) is present.  At import — before any
reference test module does ``import tricount`` / ``from tricount.x import y``
— every cover-edge entry point of the installed ``tricount`` is replaced by
the B200 one, the way the reference's own tests swap registry entries
(pkg/tests/test_bench_cli.py:117-121 monkeypatches SEQUENTIAL_IDS):

* ``SEQUENTIAL_IDS["CETC*"]`` and ``PARALLEL_IDS["CETC-SM"]`` (so
  ``count_sequential``, ``tc_par`` and ``bench._runner`` dispatch to the GPU),
* ``tc_cetc``, ``tc_cetc_degree``, ``tc_cetc_fe``, ``tc_cetc_split*``,
  ``tc_cetc_sm`` and ``parallel._cetc_sm_counts``,
* ``bfs_label`` / ``cover_edges`` in ``tricount``, ``tricount.bfs`` and
  ``tricount.cli`` (``--dump-cover``, cli.py:61-69).

The GPU functions receive the reference's own ``Graph`` objects.  Every
swapped call is counted; the count is written to $REFSWAP_REPORT at exit so
the caller can assert the GPU path actually ran.
"""
from __future__ import annotations

import atexit
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = Path(os.environ.get("REFSWAP_REF", ROOT / "baseline" / "_ref"))
for p in (str(REF), str(ROOT)):
    if p not in sys.path:
        sys.path.insert(0, p)

import tricount  # noqa: E402  (the installed reference)
import tricount.bfs  # noqa: E402
import tricount.cli  # noqa: E402
import tricount.parallel  # noqa: E402
import tricount.sequential  # noqa: E402

import paper_2403_02997_b200 as tb  # noqa: E402

CALLS = {"n": 0}


def _counted(fn):
    def wrapper(*a, **k):
        CALLS["n"] += 1
        return fn(*a, **k)
    wrapper.__name__ = getattr(fn, "__name__", "gpu_fn")
    wrapper.__doc__ = fn.__doc__
    return wrapper


def _swap_entry_points():
    gpu = {
        "tc_cetc": tb.tc_cetc,
        "tc_cetc_degree": tb.tc_cetc_degree,
        "tc_cetc_fe": tb.tc_cetc_fe,
        "tc_cetc_split": tb.tc_cetc_split,
        "tc_cetc_split_degree": tb.tc_cetc_split_degree,
        "tc_cetc_split_recursive": tb.tc_cetc_split_recursive,
        "tc_cetc_sm": tb.tc_cetc_sm,
        "bfs_label": tb.bfs_label,
        "cover_edges": tb.cover_edges,
    }
    wrapped = {k: _counted(v) for k, v in gpu.items()}
    mods = (tricount, tricount.sequential, tricount.parallel, tricount.bfs, tricount.cli)
    for mod in mods:
        for name, fn in wrapped.items():
            if hasattr(mod, name):
                setattr(mod, name, fn)
    tricount.parallel._cetc_sm_counts = _counted(tb.parallel._cetc_sm_counts)
    seq_gpu = {k: _counted(v) for k, v in tb.SEQUENTIAL_IDS.items()}
    swapped = []
    for reg in {id(tricount.SEQUENTIAL_IDS): tricount.SEQUENTIAL_IDS,
                id(tricount.sequential.SEQUENTIAL_IDS): tricount.sequential.SEQUENTIAL_IDS}.values():
        for alg in list(reg):
            if alg.startswith("CETC"):
                reg[alg] = seq_gpu[alg]
                swapped.append(alg)
    for reg in {id(tricount.PARALLEL_IDS): tricount.PARALLEL_IDS,
                id(tricount.parallel.PARALLEL_IDS): tricount.parallel.PARALLEL_IDS}.values():
        reg["CETC-SM"] = _counted(tb.PARALLEL_IDS["CETC-SM"])
        swapped.append("CETC-SM")
    return sorted(set(swapped))


SWAPPED = _swap_entry_points()


def _report():
    out = os.environ.get("REFSWAP_REPORT")
    if out:
        Path(out).write_text(f"{CALLS['n']} {' '.join(SWAPPED)}\n")


atexit.register(_report)


def pytest_report_header(config):
    return f"refswap: GPU cover-edge path swapped into the reference ({', '.join(SWAPPED)})"
