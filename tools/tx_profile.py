import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2403_02997_b200 as tb
from paper_2403_02997_b200 import configs as C
for name in sys.argv[1:]:
    dg = C.build_device_graph(name)
    r = tb.cetc(dg, keep_level=True, keep_cover=True)
    n = dg.n
    deg = dg.row_offsets[1:] - dg.row_offsets[:-1]
    order = torch.argsort(-deg * (n + 1) + torch.arange(n, device=deg.device))  # deg desc, id asc
    t = torch.empty(n, dtype=torch.long, device=deg.device); t[order] = torch.arange(n, device=deg.device)
    u, v = r.cover_u.long(), r.cover_v.long()
    x = torch.where(t[u] < t[v], u, v); p = torch.where(t[u] < t[v], v, u)
    dx = deg[x]
    cta = dx > 256
    lev = r.level
    srcl, nbl = dg.src.long(), dg.neighbors.long()
    same = lev[srcl] == lev[nbl]
    up = same & (t[nbl] < t[srcl])
    keys, _ = torch.sort(srcl[up] * n + t[nbl[up]])
    start = torch.searchsorted(keys, p * n)
    above = torch.searchsorted(keys, p * n + t[x]) - start
    for B in (65536, 131072, 262144):
        m = cta & (t[x] < B)
        print(f"{name} B={B}: CTA edges with t(x)<B {int(m.sum())}/{int(cta.sum())}  UP-above share {float(above[m].sum())/float(above[cta].sum()):.3f}")
    print(name, "vertices deg>256:", int((deg > 256).sum()), "deg>1024:", int((deg > 1024).sum()))
