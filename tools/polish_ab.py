"""Dump the Cut-QP records of one cut (for comparing polish implementations across processes).

    BZG_POLISH_IMPL=lu python tools/polish_ab.py cfg3 out_lu.npz ; python tools/polish_ab.py cfg3 out_reg.npz
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from paper_2411_13507_b200 import _native as nat, configs, graph as G  # noqa: E402


def main(name, out):
    ctx = nat.Context(0)
    w = configs.BUILDERS[name]()
    g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
    m = G.cut_graph(g, w.obstacles)
    r = m.qp_records()
    np.savez(out, edge=r["edge"], obstacle=r["obstacle"], status=r["status"], delta=r["delta"], alive=m.alive)


if __name__ == "__main__":
    main(*sys.argv[1:])
