import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["HF_WIDE"] = "1"
import hfgen, oracle
from paper_2203_08395_b200 import hf
g = hfgen.config(sys.argv[1], float(sys.argv[2]))
G = hf.hf_graph_create(g.n, g.m, g.in_ptr, g.in_src, delay=g.delay)
L, level, lptr, order = hf.levelize_np(G)
lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
at_o = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.at_src, lv)
rat_o, slack_o, wns_o = oracle.backward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.t_req, at_o, lv)
at = np.zeros(g.n, np.float32); hf.hf_propagate_forward(G, g.at_src, at)
rat = np.zeros(g.n, np.float32); hf.hf_propagate_backward(G, g.t_req, at_o, rat)
op, od, oe = oracle.fanout(g.n, g.m, g.in_ptr, g.in_src)
outdeg = np.diff(op); indeg = np.diff(g.in_ptr)
print("L", L, "level sizes max", np.bincount(level).max())
for name, x, y, deg in (("at", at, at_o, indeg), ("rat", rat, rat_o, outdeg)):
    bad = np.nonzero(x.view(np.uint32) != y.view(np.uint32))[0]
    print(name, "mismatches", len(bad))
    for v in bad[:10]:
        print("  node", v, "level", level[v], "deg", deg[v], "gpu", x[v], "oracle", y[v])
    if len(bad):
        print("  deg hist of bad:", np.bincount(deg[bad])[:30], "levels:", np.bincount(level[bad]))
