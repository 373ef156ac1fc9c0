"""Per-rank local step of a G-way row-block split, timed on one GPU (DESIGN.md §5 evidence).

For G in (1, 2, 4, 8) and the first / last rank: build (rows of the block) -> cut (its edges,
its QPs) -> find_path on the local graph (a stand-in for rank 0's search over the gathered
alive edges).  Prints device ms per step (CUDA events, L2 flushed), the per-kernel split and
the bytes rank g sends in the alive-edge gather (16 B per alive edge + 1 B provenance).

    python tools/row_block_probe.py [cfg3] [steps]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import json  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_13507_b200 import _native as nat  # noqa: E402


def main(cfg="cfg3", steps="5", nodes="0"):
    steps = int(steps)
    stream = torch.cuda.Stream()
    ctx = nat.Context(0, stream=stream.cuda_stream)
    nat.set_default_context(ctx)
    w = bench.workload(cfg, int(nodes))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    out = []
    for G in (1, 2, 4, 8):
        for g in sorted({0, G - 1}):
            step = bench.DeviceStep(ctx, w, rank=g, world=G)
            step.world, step.rank = 1, 0  # local work only: no gather, search the local graph
            for _ in range(2):
                step.run()
            ctx.reset_stats()
            ctx.set_profiling(True)
            ms = []
            for _ in range(steps):
                with torch.cuda.stream(stream):
                    flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                step.run()
                b.record(stream)
                b.synchronize()
                ms.append(a.elapsed_time(b))
            _, st = ctx.stats()
            ctx.set_profiling(False)
            alive = int(step.last_mask.alive.sum())
            top = sorted(((k, v[0] / steps) for k, v in st.items()), key=lambda kv: -kv[1])[:6]
            rec = {"G": G, "rank": g, "rows": list(step.rows or (0, w.num_vertices)), "ms": round(float(np.median(ms)), 4),
                   "edges": step.last["E"], "qp": int(step.last["qp"]), "alive": alive,
                   "gather_bytes": alive * 18, "top": [(k, round(v, 4)) for k, v in top]}
            out.append(rec)
            print(json.dumps(rec), flush=True)
    return out


if __name__ == "__main__":
    main(*sys.argv[1:])
