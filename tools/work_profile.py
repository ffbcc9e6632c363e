"""Where the CTA-tier probe work sits: sum over cover edges of min(d(u), d(v))
bucketed by owner degree, plus partner-degree buckets and partner reuse
(how often each partner list is streamed).  Run on the GPU box:
    python tools/work_profile.py rmat24
"""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
import paper_2403_02997_b200 as tb  # noqa: E402
from paper_2403_02997_b200 import configs as C  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rmat22"
dg = C.build_device_graph(name)
r = tb.cetc(dg, keep_level=True, keep_cover=True)
deg = dg.row_offsets[1:] - dg.row_offsets[:-1]
u, v = r.cover_u.long(), r.cover_v.long()
du, dv = deg[u], deg[v]
own_u = (du > dv) | ((du == dv) & (u < v))
d_own = torch.where(own_u, du, dv)
d_par = torch.where(own_u, dv, du)
par = torch.where(own_u, v, u)
wmin = torch.minimum(du, dv)
tot = wmin.sum().item()
print(f"{name}: |S|={len(u)} W_min={tot:.4g}")
edges = [0, 16, 512, 2048, 4096, 16384, 65536, 1 << 40]
for lo, hi in zip(edges[:-1], edges[1:]):
    m = (d_own > lo) & (d_own <= hi)
    print(f"  owner d in ({lo},{hi}]: owners={torch.unique(torch.where(own_u, u, v)[m]).numel():>9} "
          f"edges={int(m.sum()):>11} W={wmin[m].sum().item() / tot * 100:6.2f}%")
cta = d_own > 512
for lo, hi in zip(edges[:-1], edges[1:]):
    m = cta & (d_par > lo) & (d_par <= hi)
    print(f"  CTA tier, partner d in ({lo},{hi}]: edges={int(m.sum()):>11} "
          f"W={wmin[m].sum().item() / tot * 100:6.2f}%")
cnt = torch.bincount(par[cta], minlength=dg.n)
streamed = (cnt * deg).sum().item()
uniq = deg[cnt > 0].sum().item()
print(f"  CTA tier: streamed ids {streamed:.4g}, distinct partner ids {uniq:.4g}, "
      f"reuse {streamed / max(uniq, 1):.1f}x, partners {(cnt > 0).sum().item()}")
