"""Bellman-Ford statistics of one bench step (sweeps, frontier expansions, V, E_alive).

    BZG_TRACE=1 python tools/bf_probe.py cfg5 100000
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_2411_13507_b200 import _native as nat  # noqa: E402


def main(config="cfg5", nodes="100000"):
    ctx = nat.Context(0)
    nat.set_default_context(ctx)
    w = bench.workload(config, int(nodes))
    step = bench.DeviceStep(ctx, w)
    for _ in range(2):
        step.run()
    m = step.local_mask
    print(config, nodes, "E", m.alive.size, "E_alive", int(m.alive.sum()), "path_hops", len(step.last.get("path") or []),
          flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
