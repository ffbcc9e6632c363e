"""Time the CETC variants on a config: python tools/time_variants.py rmat22
(forward count, CETC-Seq-FE fused, degree_order relabel, CETC on the
relabelled graph).  Wall time around synchronous calls, after one warm-up."""
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
import paper_2403_02997_b200 as tb  # noqa: E402
from paper_2403_02997_b200 import configs as C  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rmat22"
dg = C.build_device_graph(name)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, 1e3 * (time.perf_counter() - t0)


cetc, t_cetc = timed(lambda: tb.cetc(dg))
fwd, t_fwd = timed(lambda: tb.ops.forward_count(dg))
(fe, used), t_fe = timed(lambda: tb.ops.cetc_fe(dg))
dd, t_dd = timed(lambda: tb.degree_order_device(dg))
cd, t_cd = timed(lambda: tb.cetc(dd))
print(f"{name}: T={cetc.triangles} ratio={cetc.ncover / max(dg.m, 1):.3f} | cetc {t_cetc:.2f} ms | "
      f"forward {t_fwd:.2f} ms (T={fwd}) | FE {t_fe:.2f} ms ({'forward' if used else 'cetc'}, "
      f"T={fe.triangles}) | degree_order {t_dd:.2f} ms | cetc on relabelled {t_cd:.2f} ms "
      f"(T={cd.triangles}, ratio {cd.ncover / max(dg.m, 1):.3f})")
