"""Same-level stream volume under two dedup orientations (measurement only):
id rule (stream SUP(p) above x: same-level w > max(x, p)) vs degree-rank rule
(stream same-level w of p ranked above the owner x).  Run on the GPU box:
    python tools/rank_profile.py rmat24
"""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
import paper_2403_02997_b200 as tb  # noqa: E402
from paper_2403_02997_b200 import configs as C  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rmat22"
dg = C.build_device_graph(name)
r = tb.cetc(dg, keep_level=True, keep_cover=True)
n = dg.n
deg = dg.row_offsets[1:] - dg.row_offsets[:-1]
u, v = r.cover_u.long(), r.cover_v.long()
du, dv = deg[u], deg[v]
own_u = (du > dv) | ((du == dv) & (u < v))
x = torch.where(own_u, u, v)
p = torch.where(own_u, v, u)
del du, dv, own_u, u, v
lev = r.level
srcl, nbl = dg.src.long(), dg.neighbors.long()
same = lev[srcl] == lev[nbl]
n_off = torch.bincount(srcl[~same], minlength=n)
# rank: degree desc, id asc -> rank value (higher = higher rank)
order = torch.argsort(deg * (n + 1) + (n - torch.arange(n, device=deg.device)), descending=False)
rank = torch.empty(n, dtype=torch.long, device=deg.device)
rank[order] = torch.arange(n, device=deg.device)
s_src, s_nb = srcl[same], nbl[same]
del srcl, nbl, same
n_same = torch.bincount(s_src, minlength=n)
end = torch.cumsum(n_same, 0)
keys = s_src * n + rank[s_nb]
keys, _ = torch.sort(keys)
above_rank = end[p] - torch.searchsorted(keys, p * n + rank[x], right=True)
keys = s_src * (n + 1) + s_nb  # CSR order is already sorted
above_id = end[p] - torch.searchsorted(keys, p * (n + 1) + x, right=True)
off = int(n_off[p].sum())
a, b = int(above_id.sum()), int(above_rank.sum())
print(f"{name}: OFF stream {off:.4e}  same-level: id rule {a:.4e}  rank rule {b:.4e}  "
      f"total id {off + a:.4e}  total rank {off + b:.4e} ({(off + b) / (off + a):.3f})")
# owner tables: id rule SUP(x) (same-level > x) vs rank rule (same-level ranked above x)
# degree-bucket prefixes (what the kernels stream): w in UP(p) with
# bucket(d(w)) >= bucket(d(x)), at 1 and 2 buckets per octave, per tier
dx = deg[x]
for per_oct in (1, 2, 4):
    def bk(d):
        lg = torch.floor(torch.log2(d.clamp(min=1).double())).long()
        frac = d.double() / torch.pow(2.0, lg.double())
        return lg * per_oct + torch.floor((frac - 1.0) * per_oct).long()
    rk_src = rank[s_src] if False else None
    up = rank[s_nb] > rank[s_src]
    b_nb = bk(deg[s_nb])
    keys2, _ = torch.sort(s_src[up] * 256 + (255 - b_nb[up]))
    kx = bk(dx)
    pref = torch.searchsorted(keys2, p * 256 + (255 - kx), right=True) - \
        torch.searchsorted(keys2, p * 256, right=False)
    for tier, m in (("warp", (dx > 16) & (dx <= 512)), ("cta", dx > 512), ("all", dx > 0)):
        print(f"  {per_oct}/octave {tier}: bucket prefix {int(pref[m].sum()):.4e}  exact {int(above_rank[m].sum()):.4e}  "
              f"OFF {int(n_off[p][m].sum()):.4e}")
