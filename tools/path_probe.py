"""Time the general path against the low-degree merge path on synthetic
low-degree graphs (ER with mean degree k, n vertices), toggling
TCB_NO_LOWDEG per call.  Run on the GPU box:
    python tools/path_probe.py
"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2403_02997_b200 as tb  # noqa: E402
from paper_2403_02997_b200 import configs as C  # noqa: E402
from paper_2403_02997_b200.graph import normalize_device  # noqa: E402


def timed(dg, reps=5):
    tb.cetc(dg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = tb.cetc(dg)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, r


for n, k in ((1 << 18, 8), (1 << 20, 8), (1 << 20, 16), (1 << 22, 12), (1 << 20, 24)):
    pairs = C.er_pairs_device(n, k / (n - 1), 7) if n <= 4096 else None
    # sparse ER by uniform random pairs (the fixture recipe is O(n^2))
    g = torch.Generator(device="cuda").manual_seed(n + k)
    pr = torch.randint(0, n, (n * k // 2, 2), device="cuda", generator=g)
    dg = normalize_device(n, pr)
    deg = (dg.row_offsets[1:] - dg.row_offsets[:-1])
    os.environ.pop("TCB_NO_LOWDEG", None)
    t_low, r1 = timed(dg)
    os.environ["TCB_NO_LOWDEG"] = "1"
    t_gen, r2 = timed(dg)
    os.environ.pop("TCB_NO_LOWDEG", None)
    assert (r1.triangles, r1.c1, r1.c2) == (r2.triangles, r2.c1, r2.c2)
    print(f"n={n} k={k} m={dg.m} dmax={int(deg.max())} T={r1.triangles}: "
          f"dispatch {t_low:.3f} ms, general {t_gen:.3f} ms", flush=True)
