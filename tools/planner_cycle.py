"""A few Planner calls on one config -- the command to put under ncu for the per-kernel split
of a captured step.      python tools/planner_cycle.py cfg1-demo 3
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_2411_13507_b200 import _native as nat  # noqa: E402
from paper_2411_13507_b200.plan import Planner  # noqa: E402


def main(cfg="cfg1-demo", calls="3"):
    ctx = nat.Context(0)
    nat.set_default_context(ctx)
    w = bench.workload(cfg)
    kw = {}
    if w.extra.get("regions"):
        rr, smp = bench.region_constants(w)
        kw = dict(regions=w.extra["regions"], per_region=w.extra["per_region"], rows_added=rr, sampling=smp)
    pl = Planner(w.N, w.spec, w.oracle, w.sample_bounds, w.obstacles, seed=w.seed, include=w.include, **kw)
    for _ in range(int(calls)):
        p = pl(w.seed, w.obstacles, w.start, w.goal, include=w.include)
    print(cfg, pl.info(), "hops", len(p or []))


if __name__ == "__main__":
    main(*sys.argv[1:])
