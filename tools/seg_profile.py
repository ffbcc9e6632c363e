"""Stream-segment length distribution of the CTA tier (owners with d > 512):
an edge (owner x, partner p) streams OFF(p) and SUP(p) above x, each cut
into G(x) id-range slices when x's staged lists exceed HC.  Prints the share
of streamed ids by slice length.  Run on the GPU box:
    python tools/seg_profile.py rmat24
"""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
import paper_2403_02997_b200 as tb  # noqa: E402
from paper_2403_02997_b200 import configs as C  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rmat22"
HC = 4096
dg = C.build_device_graph(name)
r = tb.cetc(dg, keep_level=True, keep_cover=True)
n = dg.n
deg = dg.row_offsets[1:] - dg.row_offsets[:-1]
u, v = r.cover_u.long(), r.cover_v.long()
du, dv = deg[u], deg[v]
own_u = (du > dv) | ((du == dv) & (u < v))
x = torch.where(own_u, u, v)
p = torch.where(own_u, v, u)
dx = deg[x]
cta = dx > 512
x, p = x[cta], p[cta]
lev = r.level
srcl, nbl = dg.src.long(), dg.neighbors.long()
same = lev[srcl] == lev[nbl]
n_off = torch.bincount(srcl[~same], minlength=n)
sup = same & (nbl > srcl)
n_sup = torch.bincount(srcl[sup], minlength=n)
keys = srcl[sup] * (n + 1) + nbl[sup]
above = torch.cumsum(n_sup, 0)[p] - torch.searchsorted(keys, p * (n + 1) + x, right=True)
st = (n_off + n_sup)[x]
G = torch.ones_like(st)
while True:
    big = (st + G - 1) // G > HC
    if not big.any() or int(G.max()) >= 32:
        break
    G = torch.where(big, G * 2, G)
print(f"{name}: CTA edges {len(x)}, owners split (G>1): {int((G > 1).sum())} edges, "
      f"{int(torch.unique(x[G > 1]).numel())} owners")
so = n_off[p].float() / G
ss = above.float() / G
tot = float(n_off[p].sum() + above.sum())
bins = [0, 8, 32, 128, 512, 2048, 1e12]
for name_, L, cnt in (("OFF", so, n_off[p] * 1.0), ("SUP", ss, above * 1.0)):
    for lo, hi in zip(bins[:-1], bins[1:]):
        m = (L >= lo) & (L < hi)
        print(f"  {name_} slice len [{lo},{hi}): ids {float(cnt[m].sum()) / tot * 100:6.2f}%  "
              f"slices {int(m.sum() * 1)}")
for g in (1, 2, 4, 8, 16, 32):
    m = G == g
    print(f"  G={g:2d}: edges {int(m.sum()):>10}  ids {float((n_off[p] + above)[m].sum()) / tot * 100:6.2f}%")
# CTA items: ceil(partners / 1024) per owner and group, and stream ids per item
own_ids, per_owner = torch.unique(x, return_counts=True)
first = torch.searchsorted(x.sort().values, own_ids)
Gx = G[x.argsort()][first]
items = ((per_owner + 1023) // 1024) * Gx
tot_items = int(items.sum())
print(f"  CTA items {tot_items}, owners {len(own_ids)}, stream ids/item {tot / max(tot_items, 1):.0f}")
ids_per_owner = torch.zeros(n, dtype=torch.float64, device=x.device)
ids_per_owner.index_add_(0, x, (n_off[p] + above).double())
ipi = ids_per_owner[own_ids] / items.double()
for lo, hi in [(0, 1024), (1024, 4096), (4096, 16384), (16384, 65536), (65536, 1e12)]:
    m = (ipi >= lo) & (ipi < hi)
    print(f"   items with [{lo},{hi}) ids: {int(items[m].sum()):>9} items, "
          f"{float(ids_per_owner[own_ids][m].sum()) / tot * 100:6.2f}% of ids")
