"""Run one build -> cut -> find_path step of a workload (profiling driver for ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2411_13507_b200 import _native as nat, configs, graph as G  # noqa: E402


def main(name="cfg3", reps=1):
    ctx = nat.Context(0)
    w = configs.BUILDERS[name]()
    for _ in range(int(reps)):
        g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
        mask = G.cut_graph(g, w.obstacles)
        path = G.find_path(g, mask, w.start, w.goal)
    print(w.name, "V", g.num_vertices, "E", g.num_edges, "qp", mask.pairs_qp, "path", path)


if __name__ == "__main__":
    main(*sys.argv[1:])
