"""One bench step of cfg5 at N nodes (profiling driver for ncu):  python tools/run_cfg5_once.py 100000"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_2411_13507_b200 import _native as nat  # noqa: E402

if __name__ == "__main__":
    ctx = nat.Context(0)
    nat.set_default_context(ctx)
    step = bench.DeviceStep(ctx, bench.workload("cfg5", int(sys.argv[1]) if len(sys.argv) > 1 else 100000))
    for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
        step.run()
    print("ok")
