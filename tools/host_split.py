"""Host time of each public call of one step (wall, synchronised) split into its Python
preparation and its C call, for small scenes where the host bounds the step.

    python tools/host_split.py cfg1-demo cfg1
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2411_13507_b200 import _native as nat, graph as G  # noqa: E402


def main(*cfgs):
    ctx = nat.Context(0)
    nat.set_default_context(ctx)
    for cfg in cfgs or ("cfg1-demo",):
        w = bench.workload(cfg)
        lib = ctx.lib
        calls = {}
        orig = {}
        for name in ("bzg_build_graph", "bzg_cut_graph", "bzg_find_path", "bzg_sample_region_states",
                     "bzg_mask_copy"):
            f = getattr(lib, name)
            orig[name] = f

            def wrap(*a, _f=f, _n=name):
                t = time.perf_counter()
                r = _f(*a)
                calls.setdefault(_n, []).append(1e3 * (time.perf_counter() - t))
                return r
            setattr(lib, name, wrap)
        tot = []
        for k in range(25):
            if k == 5:
                calls.clear()
                tot.clear()
            ctx.synchronize()
            t = time.perf_counter()
            bench.public_api_step(w, ctx, 0, 1)
            ctx.synchronize()
            tot.append(1e3 * (time.perf_counter() - t))
        for name, f in orig.items():
            setattr(lib, name, f)
        med = {k: round(float(np.median(v)), 3) for k, v in calls.items()}
        print(cfg, "step wall p50", round(float(np.median(tot)), 3), "C calls p50", med,
              "python+other", round(float(np.median(tot)) - sum(med.values()), 3), flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
