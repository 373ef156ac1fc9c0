"""One graph-stage step (build -> cut -> find_path) through the captured Planner vs the eager
public API, per config: device ms (events around the call, L2 flushed) and wall ms.

    python tools/planner_probe.py cfg1-demo cfg2 cfg3
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_13507_b200 import _native as nat  # noqa: E402
from paper_2411_13507_b200.plan import Planner  # noqa: E402


def main(*cfgs):
    stream = torch.cuda.Stream()
    ctx = nat.Context(0, stream=stream.cuda_stream)
    nat.set_default_context(ctx)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for cfg in cfgs or ("cfg1-demo", "cfg2"):
        w = bench.workload(cfg)
        pl = Planner(w.N, w.spec, w.oracle, w.sample_bounds, w.obstacles, seed=w.seed, include=w.include)

        def planner_step():
            return pl(w.seed, w.obstacles, w.start, w.goal, include=w.include)

        def eager_step():
            return bench.public_api_step(w, ctx, 0, 1)

        out = {}
        for name, fn in (("eager", eager_step), ("planner", planner_step)):
            for _ in range(3):
                p = fn()
            dev, wall = [], []
            for _ in range(15):
                with torch.cuda.stream(stream):
                    flush.zero_()
                torch.cuda.synchronize()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                t0 = time.perf_counter()
                a.record(stream)
                p = fn()
                b.record(stream)
                b.synchronize()
                wall.append(1e3 * (time.perf_counter() - t0))
                dev.append(a.elapsed_time(b))
            out[name] = (round(float(np.median(dev)), 3), round(float(np.median(wall)), 3), len(p or []))
        print(cfg, "device/wall ms p50, hops:", out, pl.info(), flush=True)
        pl.close()


if __name__ == "__main__":
    main(*sys.argv[1:])
