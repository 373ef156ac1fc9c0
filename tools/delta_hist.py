import sys, numpy as np
sys.path.insert(0, '.')
from paper_2411_13507_b200 import _native as nat, configs, graph as G
ctx = nat.Context(0)
w = configs.BUILDERS['cfg3']()
g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
m = G.cut_graph(g, w.obstacles)
r = m.qp_records()
st = r['status']; d = r['delta']
s = st == 0
print('solved', s.sum(), 'polished<1e-2', (s & (d < 1e-2)).sum())
edges = [0, 1e-12, 1e-9, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2]
print(np.histogram(d[s], bins=edges)[0])
