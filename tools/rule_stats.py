"""CPU-side what-if statistics for the intersection's stream rules (no GPU).

For a config's CSR and BFS levels (built with the oracle), count the ids
the CTA/warp tiers would stream per cover edge under alternative rules:

  OFF part (c1):  sum_S |OFF(p)|  (p = lower-ranked endpoint, today)
                  sum_S min(|OFF(x)|, |OFF(p)|)
  UP part (same-level): with UP(v) = same-level neighbours ranked above v,
                  bucket prefix  : |{w in UP(p): bucket(d(w)) >= bucket(d(x))}|
                  exact cut      : |{w in UP(p): rank(w) > rank(x)}|
  for rank = (degree desc, id asc) and rank = (same-level degree desc, id asc).

    python tools/rule_stats.py rmat22
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
import oracle  # noqa: E402
from paper_2403_02997_b200 import configs as C  # noqa: E402

torch.set_num_threads(8)
name = sys.argv[1] if len(sys.argv) > 1 else "rmat22"
cfg = C.CONFIGS[name]
t0 = time.time()
if cfg.kind == "rmat":
    pairs = oracle.rmat_pairs(cfg.scale, cfg.edge_factor, seed=cfg.seed,
                              perm=C.id_permutation(cfg.n, cfg.perm_seed))
elif cfg.kind == "er":
    pairs = C.er_pairs(cfg.n, cfg.p, cfg.seed)
else:
    pairs = C.lattice_pairs(cfg.side)
row, nb, eu, ev = oracle.normalize(cfg.n, pairs)
del pairs, eu, ev
level, _, _, _ = oracle.bfs_levels(row, nb, cfg.n)
print(f"{name}: built in {time.time() - t0:.1f} s")
n = cfg.n
row_t = torch.from_numpy(row)
deg = row_t[1:] - row_t[:-1]
src = torch.repeat_interleave(torch.arange(n), deg)
dst = torch.from_numpy(nb).long()
lev = torch.from_numpy(level)
same = lev[src] == lev[dst]
n_off = torch.bincount(src[~same], minlength=n)
hdeg = torch.bincount(src[same], minlength=n)
ss, sd = src[same], dst[same]
del src, dst, same


def rank_of(key):
    """rank: higher = ranked higher; key desc, id asc."""
    order = torch.argsort(key * (n + 1) + (n - torch.arange(n)))
    rk = torch.empty(n, dtype=torch.long)
    rk[order] = torch.arange(n)
    return rk


def bucket(d):
    return torch.floor(torch.log2(d.clamp(min=1).double())).long()


for rname, key in (("degree", deg), ("same-level degree", hdeg),
                   ("same-level deg, OFF by degree", None)):
    rk = rank_of(key if key is not None else hdeg)
    rk_off = rank_of(deg) if key is None else rk
    # cover edges, owner = higher rank
    fwd = ss < sd
    cu, cv = ss[fwd], sd[fwd]
    xo = torch.where(rk_off[cu] > rk_off[cv], cu, cv)
    po = torch.where(rk_off[cu] > rk_off[cv], cv, cu)
    off_now = n_off[po].sum().item()
    off_min = torch.minimum(n_off[xo], n_off[po]).sum().item()
    x = torch.where(rk[cu] > rk[cv], cu, cv)
    p = torch.where(rk[cu] > rk[cv], cv, cu)
    # UP(v) entries: (v, w) same level, rank(w) > rank(v)
    upm = rk[sd] > rk[ss]
    us, uw = ss[upm], sd[upm]
    # exact: count entries of UP(p) with rank > rank(x): sort keys p*n + rank(w)
    keys, _ = torch.sort(us * n + rk[uw])
    ends = torch.searchsorted(keys, p * n + n)
    exact = (ends - torch.searchsorted(keys, p * n + rk[x], right=True)).sum().item()
    # bucket prefix by the rank key's bucket
    kk = key if key is not None else hdeg
    bkeys, _ = torch.sort(us * 64 + bucket(kk[uw]))
    bend = torch.searchsorted(bkeys, p * 64 + 64)
    bpre = (bend - torch.searchsorted(bkeys, p * 64 + bucket(kk[x]))).sum().item()
    up_total = len(us)
    print(f"rank by {rname}: |S|={len(cu)} OFF stream {off_now:.4e} (min rule {off_min:.4e}); "
          f"UP entries {up_total:.4e}; UP stream bucket-prefix {bpre:.4e}, exact {exact:.4e}; "
          f"total now-style {off_now + bpre:.4e}, best {off_min + exact:.4e}")
    del keys, bkeys, ends, bend

# galloping what-if on the degree rank: per edge min(cut, |UP(x)| * ceil(log2(cut + 1)))
rk = rank_of(deg)
fwd = ss < sd
cu, cv = ss[fwd], sd[fwd]
x = torch.where(rk[cu] > rk[cv], cu, cv)
p = torch.where(rk[cu] > rk[cv], cv, cu)
upm = rk[sd] > rk[ss]
us, uw = ss[upm], sd[upm]
n_up = torch.bincount(us, minlength=n)
keys, _ = torch.sort(us * n + rk[uw])
cut = torch.searchsorted(keys, p * n + n) - torch.searchsorted(keys, p * n + rk[x], right=True)
ux = n_up[x]
gal = ux * torch.ceil(torch.log2(cut.double() + 1)).long()
best = torch.minimum(cut, gal)
print(f"UP exact {cut.sum().item():.4e}; galloping-or-stream {best.sum().item():.4e}; "
      f"edges where galloping wins {(gal < cut).sum().item()} of {len(cut)}; "
      f"sum |UP(x)| over edges {ux.sum().item():.4e}")
for lo, hi in ((0, 256), (256, 4096), (4096, 1 << 40)):
    msk = (deg[x] > lo) & (deg[x] <= hi)
    print(f"  owner d in ({lo},{hi}]: edges {msk.sum().item()}, UP exact {cut[msk].sum().item():.4e}, "
          f"best {best[msk].sum().item():.4e}, OFF(p) {n_off[p[msk]].sum().item():.4e}")
