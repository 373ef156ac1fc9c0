"""Per-step wall time of bench.DeviceStep (host phases), with and without kernel profiling.

    python tools/step_timing.py cfg5 50000
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_2411_13507_b200 import _native as nat  # noqa: E402


def main(config="cfg5", nodes="50000", reps=6):
    import torch

    ctx = nat.Context(0)
    nat.set_default_context(ctx)
    w = bench.workload(config, int(nodes))
    step = bench.DeviceStep(ctx, w)
    for mode in ("plain", "profile_only", "profile_all"):
        ctx.reset_stats()
        if mode == "profile_only":
            ctx.set_profiling(True)
            ctx.profile_only("k_pair_tiles")
        elif mode == "profile_all":
            ctx.set_profiling(True)
            ctx.profile_only(None)
        for r in range(int(reps)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            step.run()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            print(f"{mode:13s} rep {r}: {1e3 * (t1 - t0):8.2f} ms  phases {step.last['host_phase_ms']}", flush=True)
        ctx.set_profiling(False)
        ctx.profile_only(None)


if __name__ == "__main__":
    main(*sys.argv[1:])
