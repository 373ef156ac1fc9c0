"""Kernel time vs device wall time of one cached re-cut + relaxed search cycle (cfg2, one moved
obstacle): how much of a replanning cycle is launch/host overhead."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_13507_b200 import _native as nat, configs, graph as G  # noqa: E402
from paper_2411_13507_b200.geometry import Polytope  # noqa: E402


def main(cfg="cfg2"):
    stream = torch.cuda.Stream()
    ctx = nat.Context(0, stream=stream.cuda_stream)
    w = configs.BUILDERS[cfg]()
    g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
    g.set_cut_cache(64)
    obs = list(w.obstacles)
    G.cut_graph(g, obs)
    walls, kern = [], []
    for k in range(12):
        A = np.asarray(obs[k % len(obs)].A)
        obs[k % len(obs)] = Polytope(A, np.asarray(obs[k % len(obs)].b) + A @ np.full(2, 0.01))
        ctx.reset_stats()
        ctx.set_profiling(k >= 6)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        m = G.cut_graph(g, obs)
        G.find_path(g, m, w.start, w.goal, position_only_snap=True, require_tube_snap=False)
        b.record(stream)
        b.synchronize()
        if k >= 6:
            n, st = ctx.stats()
            kern.append(sum(v[0] for v in st.values()))
            walls.append(a.elapsed_time(b))
            top = sorted(st.items(), key=lambda kv: -kv[1][0])[:6]
    ctx.set_profiling(False)
    print(cfg, "cycle device ms", round(float(np.median(walls)), 3), "kernel sum", round(float(np.median(kern)), 3),
          "launches", n, [(k, round(v[0], 3)) for k, v in top])


if __name__ == "__main__":
    main(*sys.argv[1:])
