"""The reference's OWN hot-path tests and harness, driven through the GPU path.

SURVEY.md §8(c) (2): swap the reference's CETC registry entries and entry
points for the GPU functions (the pattern of ref pkg/tests/test_bench_cli.py
:117-121) and re-run its ``test_sequential.py -k CETC``, ``test_parallel.py``
and ``test_bench_cli.py`` — the last includes ``--dump-cover`` on karate
("28 cover edges", cli.py:61-69) and ``bench._runner`` (bench.py:122-129)
dispatching the ``cetc-family`` ids.  The swap lives in
tests/refswap_plugin.py.

Needs the installed reference in ``baseline/_ref`` (tools/install_reference.sh:
``pip install --target`` of /root/reference plus its tests and data; the
directory is git-ignored and travels to the GPU box with the snapshot) and
numba (the reference's kernels run the non-swapped parts of its suite).
Skipped when either is missing.  Nothing here reads /root/reference.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


def _available() -> str | None:
    if not (REF / "tricount" / "__init__.py").exists() or not (REF / "tests").is_dir():
        return "baseline/_ref (tools/install_reference.sh) not present"
    try:
        import numba  # noqa: F401
    except Exception:
        return "numba missing"
    return None


def _run(tmp_path, args):
    report = tmp_path / "refswap.txt"
    env = dict(os.environ,
               PYTHONPATH=os.pathsep.join([str(ROOT / "tests"), str(REF), str(ROOT)]),
               TRICOUNT_DATA=str(REF / "data"),
               NUMBA_CACHE_DIR=str(tmp_path / "numba"),
               PYTHONDONTWRITEBYTECODE="1",
               REFSWAP_REPORT=str(report))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "refswap_plugin", "-p",
           "no:cacheprovider", "--rootdir", str(REF / "tests"), *args]
    out = subprocess.run(cmd, cwd=str(REF / "tests"), env=env, capture_output=True,
                         text=True, timeout=1500)
    calls, *swapped = report.read_text().split() if report.exists() else ("0",)
    return out, int(calls), swapped


@pytest.mark.parametrize("suite", [
    ["test_sequential.py", "-k", "CETC or CoverEdge or Split or dispatch"],
    ["test_parallel.py"],
    ["test_bench_cli.py"],
], ids=["sequential-CETC", "parallel", "bench_cli"])
def test_reference_suite_with_gpu_cover_edge_path(tmp_path, suite):
    why = _available()
    if why:
        pytest.skip(why)
    out, calls, swapped = _run(tmp_path, suite)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "passed" in out.stdout
    # the swap really happened and the GPU path really ran
    assert {"CETC-Seq", "CETC-SM", "CETC-Seq-FE"} <= set(swapped), swapped
    assert calls > 0, "no GPU cover-edge call was made"
