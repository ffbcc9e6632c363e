"""Same-level work under the two stream directions (measurement only).
For every cover edge (owner x ranked above partner p) the same-level apexes
are UP(x) ∩ UP(p) with every w ranked above x.  Current kernels stream
A_e = |{w in UP(p): w above x}| past a hash of the owner's lists; the other
direction streams B_e = |UP(x)| past a structure over p.  Prints sums of A,
B and min(A, B), split by owner tier (thread/warp/cta by owner degree).
    python tools/orient_profile.py rmat24
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
order = torch.argsort(deg * (n + 1) + (n - torch.arange(n, device=deg.device)))
rank = torch.empty(n, dtype=torch.long, device=deg.device)
rank[order] = torch.arange(n, device=deg.device)
s_src, s_nb = srcl[same], nbl[same]
del srcl, nbl, same
up = rank[s_nb] > rank[s_src]
n_up = torch.bincount(s_src[up], minlength=n)
n_same = torch.bincount(s_src, minlength=n)
end = torch.cumsum(n_same, 0)
keys, _ = torch.sort(s_src * n + rank[s_nb])
A = end[p] - torch.searchsorted(keys, p * n + rank[x], right=True)
B = n_up[x]
M = torch.minimum(A, B)
dx = deg[x]
for tier, sel in (("thread", dx <= 16), ("warp", (dx > 16) & (dx <= 256)), ("cta", dx > 256),
                  ("all", torch.ones_like(dx, dtype=torch.bool))):
    oa, ob = n_off[p][sel].sum().item(), n_off[x][sel].sum().item()
    print(f"{name} {tier:6s} edges {int(sel.sum()):.3e}  same: A {A[sel].sum().item():.3e} "
          f"B {B[sel].sum().item():.3e} min {M[sel].sum().item():.3e}   "
          f"off: |OFF(p)| {oa:.3e} |OFF(x)| {ob:.3e} "
          f"min {torch.minimum(n_off[p], n_off[x])[sel].sum().item():.3e}")
