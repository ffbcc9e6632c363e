"""Capacity probe: build an RMAT config in HBM, time the fused step
(CUDA events, 2 warm-up + 3 timed), cross-check T against the GPU forward
count and report peak HBM.  python tools/scale_probe.py rmat25 rmat26
"""
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
import paper_2403_02997_b200 as tb  # noqa: E402
from paper_2403_02997_b200 import configs as C  # noqa: E402

for name in sys.argv[1:] or ["rmat25"]:
    torch.cuda.reset_peak_memory_stats()
    t0 = time.time()
    dg = C.build_device_graph(name)
    torch.cuda.synchronize()
    tb_s = time.time() - t0
    deg = dg.row_offsets[1:] - dg.row_offsets[:-1]
    for _ in range(2):
        r = tb.cetc(dg)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(3):
        r = tb.cetc(dg)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 3
    free, total = torch.cuda.mem_get_info()
    f = tb.ops.forward_count(dg)
    print(f"{name}: n {dg.n} m {dg.m} 2m {2 * dg.m} max_deg {int(deg.max())} build {tb_s:.1f}s "
          f"step {ms:.1f} ms ({dg.m / ms / 1e6:.3f} G edges/s) T {r.triangles} c1 {r.c1} c2 {r.c2} "
          f"levels {r.max_level} cover {r.ncover} forward {f} match {f == r.triangles} "
          f"torch peak {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB, "
          f"device in use {(total - free) / 2**30:.1f} GiB", flush=True)
    del dg, deg, r
    torch.cuda.empty_cache()
