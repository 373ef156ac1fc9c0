"""The replanning-cycle benchmark (bench.recut_bench: one moving obstacle, re-cut + relaxed-snap
search per cycle; eager full cut, eager re-cut cache, captured Replanner with and without the
static / dynamic split) on the graph of any config.

    python tools/replan_probe.py cfg1-demo cfg2 cfg3
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_13507_b200 import _native as nat, configs, graph as G  # noqa: E402


def main(*cfgs):
    stream = torch.cuda.Stream()
    ctx = nat.Context(0, stream=stream.cuda_stream)
    nat.set_default_context(ctx)
    for cfg in cfgs or ("cfg1-demo", "cfg2"):
        w = configs.BUILDERS[cfg]()
        g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
        with torch.cuda.stream(stream):
            res = bench.recut_bench(ctx, stream, w, g, steps=20)
        print(json.dumps({"config": cfg, "V": g.num_vertices, "E": g.num_edges, **res}), flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
