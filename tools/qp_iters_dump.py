"""Dump the cfg3 Cut-QP per-instance iteration counts (instance = fetch order of k_qp_admm)
to gpurun_out/qp_iters_cfg3.npy, for offline tail/scheduling estimates."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2411_13507_b200 import _native as nat, configs, graph as G
ctx = nat.Context(0)
w = configs.BUILDERS['cfg3']()
g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
m = G.cut_graph(g, w.obstacles)
r = m.qp_records()
np.save('gpurun_out/qp_iters_cfg3.npy', r['iterations'].astype(np.int32))
np.save('gpurun_out/qp_status_cfg3.npy', np.asarray(r['status']).astype(np.int8))
print('n', r['iterations'].size)
