"""A few captured replanning cycles (Replanner, obstacle 0 dynamic) on one config -- the command
to put under ncu for the per-kernel split of a cycle.

    python tools/replan_cycle.py cfg1-demo 5
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from paper_2411_13507_b200 import _native as nat, configs, graph as G  # noqa: E402
from paper_2411_13507_b200.geometry import Polytope  # noqa: E402
from paper_2411_13507_b200.replan import Replanner  # noqa: E402


def main(cfg="cfg1-demo", cycles="5"):
    ctx = nat.Context(0)
    nat.set_default_context(ctx)
    w = configs.BUILDERS[cfg]()
    g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
    obs = list(w.obstacles)
    rp = Replanner(g, obs, position_only_snap=True, require_tube_snap=False,
                   dynamic=[True] + [False] * (len(obs) - 1))
    for k in range(int(cycles)):
        A = np.asarray(obs[0].A, float)
        obs[0] = Polytope(A, np.asarray(obs[0].b, float) + A @ np.full(w.spec.m, 0.01))
        p = rp(obs, w.start, w.goal)
    print(cfg, rp.info(), "hops", len(p or []))


if __name__ == "__main__":
    main(*sys.argv[1:])
