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
lev = r.level
srcl, nbl = dg.src.long(), dg.neighbors.long()
same = lev[srcl] == lev[nbl]
ds, dn = deg[srcl], deg[nbl]
up = same & ((dn > ds) | ((dn == ds) & (nbl < srcl)))
us, un = srcl[up], nbl[up]
del srcl, nbl, same, ds, dn
bk = lambda d: torch.floor(torch.log2(d.clamp(min=1).double())).long()
# per UP entry key sorted by (src, degree) to count by degree thresholds
du = deg[un]
keys, idx = torch.sort(us * (1 << 22) + du)
un_sorted = un[idx]
dx = deg[x]; kx = bk(dx)
lo_b = p * (1 << 22) + (1 << kx)          # d >= 2^kx
lo_eq = p * (1 << 22) + dx                # d >= d(x)
lo_gt = p * (1 << 22) + dx + 1            # d > d(x)
end = p * (1 << 22) + (1 << 22)
c_b = torch.searchsorted(keys, end) - torch.searchsorted(keys, lo_b)
c_eq = torch.searchsorted(keys, end) - torch.searchsorted(keys, lo_eq)
c_gt = torch.searchsorted(keys, end) - torch.searchsorted(keys, lo_gt)
print(f"{name}: bucket prefix {int(c_b.sum()):.4e}  d>=d(x) {int(c_eq.sum()):.4e}  d>d(x) {int(c_gt.sum()):.4e}")
def fb(d):
    d = d.clamp(min=1)
    lg = torch.floor(torch.log2(d.double())).long()
    sub = torch.where(d >= 8, (d >> (lg - 3).clamp(min=0)) & 7, torch.zeros_like(d))
    return torch.where(d < 8, d, 8 * lg + sub)
fk, _ = torch.sort(us * 256 + fb(du))
fx = fb(dx)
c_f = torch.searchsorted(fk, p * 256 + 256) - torch.searchsorted(fk, p * 256 + fx)
print(f"{name}: fine-bucket prefix {int(c_f.sum()):.4e}")
