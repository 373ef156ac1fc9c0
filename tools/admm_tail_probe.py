"""Per-pass ADMM timing under different schedules (BZG_ADMM_* env), one workload.

    python tools/admm_tail_probe.py cfg2 "BZG_ADMM_PASSES=1" "BZG_ADMM_PASSES=3 BZG_ADMM_DUMP=12" ...
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2411_13507_b200 import _native as nat, configs, graph as G  # noqa: E402


def main(cfg, *specs):
    ctx = nat.Context(0)
    w = configs.BUILDERS[cfg]() if cfg != "cfg5" else configs.scaling_sweep(20000)
    if w.extra.get("regions"):
        from paper_2411_13507_b200 import regions as R
        g = R.build_region_graph(w.extra["per_region"], w.spec, w.oracle, w.extra["regions"], w.sample_bounds,
                                 w.seed, include=w.include, ctx=ctx)
    else:
        g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
    for spec in specs:
        for k in ("BZG_ADMM_LANES", "BZG_ADMM_PASSES", "BZG_ADMM_DUMP"):
            os.environ.pop(k, None)
        for kv in spec.split():
            k, v = kv.split("=")
            os.environ[k] = v
        G.cut_graph(g, w.obstacles)  # warm
        ctx.reset_stats()
        ctx.set_profiling(True)
        reps = 5
        for _ in range(reps):
            m = G.cut_graph(g, w.obstacles)
        ctx.synchronize()
        _, st = ctx.stats()
        ctx.set_profiling(False)
        ad = {k: round(v[0] / reps, 4) for k, v in st.items() if k.startswith("k_qp_admm")}
        print(f"{cfg} {spec:45s} qp={m.pairs_qp} admm={ad} total={round(sum(ad.values()), 4)}", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
