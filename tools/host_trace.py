"""Host wall time per public call of one step (build / cut / find_path) after warm-up, and the
kernel time inside each (profiling on): where a small scene's step time goes."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2411_13507_b200 import _native as nat  # noqa: E402


def main(cfg="cfg1", reps="20"):
    ctx = nat.Context(0)
    nat.set_default_context(ctx)
    w = bench.workload(cfg)
    for _ in range(3):
        bench.public_api_step(w, ctx, 0, 1)
    ts = []
    for _ in range(int(reps)):
        t0 = time.perf_counter()
        bench.public_api_step(w, ctx, 0, 1)
        ts.append((time.perf_counter() - t0) * 1e3)
    print(cfg, "public-API step wall ms p50", round(float(np.median(ts)), 3))
    step = bench.DeviceStep(ctx, w)
    for _ in range(3):
        step.run()
    ph = []
    for _ in range(int(reps)):
        step.run()
        ph.append(step.last["host_phase_ms"])
    print("device-step host phases p50:", {k: round(float(np.median([p[k] for p in ph])), 3) for k in ph[0]})
    ctx.set_profiling(True)
    ctx.reset_stats()
    step.run()
    ctx.synchronize()
    n, st = ctx.stats()
    ctx.set_profiling(False)
    print("launches", n, "kernel ms", round(sum(v[0] for v in st.values()), 3))


if __name__ == "__main__":
    main(*sys.argv[1:])
