"""Per-level BFS records of the fused step (tcb_level_records) for a config.

    python tools/bfs_levels_probe.py rmat24 [steps]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2403_02997_b200 as tb  # noqa: E402
from paper_2403_02997_b200 import configs as C  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dg = C.build_device_graph(name)
ctx = tb._lib.context()
ctx.set_timing(True)
for i in range(steps):
    r = tb.cetc(dg)
    st = ctx.stage_times()
    recs = ctx.level_records()
    print(f"step {i}: T={r.triangles} comps={r.components} max_level={r.max_level} "
          + " ".join(f"{k}={v:.3f}" for k, v in st.items() if v), flush=True)
    prev = 0.0
    for L, (mode, t_us, nf) in enumerate(recs[:12]):
        print(f"   L{L} {mode} {t_us - prev:8.1f} us  next={nf}")
        prev = t_us
    if len(recs) > 12:
        print(f"   ... {len(recs)} records, last at {recs[-1][1]:.1f} us")
