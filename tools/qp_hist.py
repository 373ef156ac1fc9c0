import sys, numpy as np
sys.path.insert(0, '.')
from paper_2411_13507_b200 import _native as nat, configs, graph as G
ctx = nat.Context(0)
w = configs.BUILDERS['cfg3']()
g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
m = G.cut_graph(g, w.obstacles)
r = m.qp_records()
it = r['iterations'].astype(np.int64); st = r['status']
print('n', it.size, 'sum', it.sum(), 'mean', it.mean())
for s in range(4): print('status', s, (st == s).sum(), 'iters', it[st == s].sum())
print('pct', np.percentile(it, [10, 25, 50, 75, 90, 95, 99]))
print('hist', np.histogram(it, bins=[0, 25, 50, 75, 100, 150, 200, 300, 400, 499, 501])[0])
