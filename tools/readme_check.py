import sys; sys.path.insert(0, ".")
import paper_2403_02997_b200 as tb
g = tb.normalize(tb.generate_rmat(tb.RmatParams(scale=16, edge_factor=16, seed=1)))
lab = tb.bfs_label(g)
cov = tb.cover_edges(lab, g)
T1 = tb.tc_cetc(g)
T2 = tb.tc_cetc_sm(g, tb.ParallelConfig(workers=8))
T3 = tb.count_sequential("CETC-Seq-SR", g)
from paper_2403_02997_b200 import configs
dg = configs.build_device_graph("rmat16")
r = tb.cetc(dg, keep_level=True)
print("readme ok", T1, T2, T3, len(cov), lab.components, r.triangles, r.c1, r.c2, r.ncover)
