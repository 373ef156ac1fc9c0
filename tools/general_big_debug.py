import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2411_13507_b200 import _native as nat, graph as G
from tests.conftest import load_golden
from tests.helpers import inputs_from_golden
g = load_golden("general_big60")
N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(g)
ctx = nat.Context(0)
gr = G.build_graph(N, spec, orc, bounds, seed, include, ctx=ctx)
m = G.cut_graph(gr, obstacles)
r = m.qp_records()
kd = r["edge"]*64 + r["obstacle"]; kr = g["qp_edge"]*64 + g["qp_obstacle"]
od, orr = np.argsort(kd), np.argsort(kr)
rows = [o.A.shape[0] for o in obstacles]
for i in range(kd.size):
    a, b = od[i], orr[i]
    print(int(r["obstacle"][a]), rows[int(r["obstacle"][a])], int(r["status"][a]), int(g["qp_status"][b]), int(r["iterations"][a]), int(g["qp_iters"][b]), float(r["delta"][a]), float(g["qp_delta"][b]))
