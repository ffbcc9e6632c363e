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

# multi-GPU balance: probe work per shard under owner sharding (x % N)
# and under (owner, id-range group, 1024-partner block) item sharding
ow = torch.where(own_u, u, v)
for N in (2, 4, 8):
    per_owner = torch.zeros(dg.n, dtype=torch.float64, device=ow.device)
    per_owner.index_add_(0, ow, wmin.double())
    owners = torch.arange(dg.n, device=ow.device)
    shard_w = torch.zeros(N, dtype=torch.float64, device=ow.device)
    shard_w.index_add_(0, owners % N, per_owner)
    print(f"  N={N}: owner sharding  max/mean shard work = "
          f"{(shard_w.max() / shard_w.mean()).item():.3f}")
    # finer: each cover edge's block index within its owner (rank of the edge
    # among the owner's partners // 1024) and range group g in [0, 32)
    order = torch.argsort(ow, stable=True)
    ow_s = ow[order]
    first = torch.searchsorted(ow_s, ow_s, right=False)
    blk = (torch.arange(len(ow_s), device=ow.device) - first) // 1024
    wm_s = wmin[order].double()
    key = (ow_s * 7 + blk) % N
    sw2 = torch.zeros(N, dtype=torch.float64, device=ow.device)
    sw2.index_add_(0, key, wm_s)
    print(f"  N={N}: (owner, block) sharding max/mean = {(sw2.max() / sw2.mean()).item():.3f}")
