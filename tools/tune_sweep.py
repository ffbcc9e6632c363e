"""Sweep the runtime tier knobs (tcb_set_tuning: warp-tier max owner degree,
ids staged per CTA pass) on one config; prints stage times per setting.
    python tools/tune_sweep.py rmat24 "512,0 256,0 128,0"
"""
import sys

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
import paper_2403_02997_b200 as tb  # noqa: E402
from paper_2403_02997_b200 import configs as C  # noqa: E402

name = sys.argv[1]
settings = [tuple(int(v) for v in s.split(",")) for s in sys.argv[2].split()]
dg = C.build_device_graph(name)
ctx = tb._lib.context()
ctx.set_timing(True)
for wt, hc in settings:
    ctx.set_tuning(wt, hc)
    for _ in range(2):
        r = tb.cetc(dg)
    st = ctx.stage_times()
    tot = sum(v for k, v in st.items() if k in ("components", "bfs", "select", "intersect"))
    print(f"wt={wt:4d} hc={hc:5d}: T={r.triangles} total={tot:.2f} ms " +
          " ".join(f"{k}={v:.2f}" for k, v in st.items() if v), flush=True)
ctx.set_tuning(0, 0)
