"""Run the fused CETC step on one config a few times (for ncu / nsight captures).

    python tools/profile_step.py rmat22 [steps]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2403_02997_b200 as tb  # noqa: E402
from paper_2403_02997_b200 import configs as C  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rmat22"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dg = C.build_device_graph(name)
ctx = tb._lib.context()
ctx.set_timing(True)
for i in range(steps):
    t0 = time.time()
    r = tb.cetc(dg)
    st = ctx.stage_times()
    print(f"step {i}: T={r.triangles} c1={r.c1} c2={r.c2} |S|={r.ncover} "
          f"wall={1e3*(time.time()-t0):.1f}ms stages=" +
          " ".join(f"{k}={v:.2f}" for k, v in st.items() if v), flush=True)
