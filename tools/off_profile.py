import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2403_02997_b200 as tb
from paper_2403_02997_b200 import configs as C
name = sys.argv[1]
dg = C.build_device_graph(name)
r = tb.cetc(dg, keep_level=True, keep_cover=True)
n = dg.n
deg = dg.row_offsets[1:] - dg.row_offsets[:-1]
u, v = r.cover_u.long(), r.cover_v.long()
own_u = (deg[u] > deg[v]) | ((deg[u] == deg[v]) & (u < v))
x = torch.where(own_u, u, v); p = torch.where(own_u, v, u)
cta = deg[x] > 256
x, p = x[cta], p[cta]
lev = r.level.long()
srcl, nbl = dg.src.long(), dg.neighbors.long()
ls, ln = lev[srcl], lev[nbl]
dn = torch.bincount(srcl[ln < ls], minlength=n)
upl = torch.bincount(srcl[ln > ls], minlength=n)
tot = int((dn[p] + upl[p]).sum())
skip = int((dn[p] * (dn[x] == 0)).sum() + (upl[p] * (upl[x] == 0)).sum())
print(f"{name}: OFF stream {tot:.4e}  skippable (owner side empty) {skip:.4e} ({skip/tot:.3f})")
# min-side choice if each part could be oriented independently
alt = int((torch.minimum(dn[p], dn[x]) + torch.minimum(upl[p], upl[x])).sum())
print(f"  per-part min-side stream {alt:.4e} ({alt/tot:.3f})")
