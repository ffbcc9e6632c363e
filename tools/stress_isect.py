"""One-off randomized stress of the intersection tiers against the oracle
(bigger graphs than tests/test_gpu_sweep.py, default thresholds and a few
shrunk ones).  Run on a GPU box:  python tools/stress_isect.py [SEEDS]
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle  # noqa: E402
import paper_2403_02997_b200 as tb  # noqa: E402
import test_gpu_sweep as sw  # noqa: E402


def g_union(rng):
    """A wide dense layer, an RMAT graph and a sparse ER graph, ids shuffled."""
    parts, base = [], 0
    for gen in (sw.g_wide_layer, sw.g_large, sw.g_rooted_dense):
        n_i, p_i = gen(rng)
        parts.append(np.asarray(p_i, dtype=np.int64).reshape(-1, 2) + base)
        base += n_i
    pairs = np.concatenate(parts)
    return base, rng.permutation(base)[pairs]


def main():
    seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    ctx = tb._lib.context()
    bad = 0
    for gen in (sw.g_wide_layer, sw.g_large, g_union):
        for s in range(seeds):
            t0 = time.time()
            n, pairs, row, nb, ref = sw._case(gen, 777_000 + 1000 * hash(gen.__name__) % 997 + s)
            dg = tb.device_graph(tb.normalize(tb.EdgeList(n=n, edges=pairs)))
            for flags in (8, 8 | 4):
                for t in ((0, 0), (256, 64), (32, 1024), (8, 16)):
                    ctx.set_test_flags(flags)
                    ctx.set_tuning(*t)
                    r = tb.cetc(dg)
                    ok = (r.triangles, r.c1, r.c2) == (ref["T"], ref["c1"], ref["c2"])
                    bad += not ok
                    if not ok:
                        print("MISMATCH", gen.__name__, s, flags, t, (r.triangles, r.c1, r.c2),
                              (ref["T"], ref["c1"], ref["c2"]), flush=True)
            ctx.set_tuning(0, 0)
            ctx.set_test_flags(0)
            print(f"{gen.__name__} seed {s}: n={n} m={len(row) and int(row[-1]) // 2} "
                  f"dmax={int(np.diff(row).max())} T={ref['T']} ok ({time.time() - t0:.1f}s)", flush=True)
    print("mismatches:", bad)
    return 1 if bad else 0


if __name__ == "__main__":
    raise SystemExit(main())
