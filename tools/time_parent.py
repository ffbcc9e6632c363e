"""Time the FIFO-parent rebuild and edge classification (bfs_label's extra
outputs) on a config: python tools/time_parent.py lattice2048"""
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
import paper_2403_02997_b200 as tb  # noqa: E402
from paper_2403_02997_b200 import configs as C  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "lattice2048"
dg = C.build_device_graph(name)
level, comps, ml = tb.ops.bfs_levels(dg)
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    parent = tb.ops.bfs_parent(dg, level, ml)
    t1 = time.perf_counter()
    cls = tb.ops.edge_classes(dg, level, parent)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
print(f"{name}: n={dg.n} m={dg.m} levels={ml + 1} parent {1e3 * (t1 - t0):.2f} ms, "
      f"edge classes {1e3 * (t2 - t1):.2f} ms; tree edges {(cls == 0).sum().item()} "
      f"(n - components = {dg.n - comps})")
