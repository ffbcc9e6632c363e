"""Run one config under several intersection tunings, one process each
(a fault poisons the CUDA context).  python tools/debug_tiers.py rmat16 wt hc"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2403_02997_b200 as tb  # noqa: E402
from paper_2403_02997_b200 import configs as C  # noqa: E402

name, wt, hc = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
dg = C.build_device_graph(name)
ctx = tb._lib.context()
ctx.set_tuning(wt, hc)
r = tb.cetc(dg)
print(name, wt, hc, "T", r.triangles, "c1", r.c1, "c2", r.c2, flush=True)
