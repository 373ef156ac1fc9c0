"""Per-QP iteration counts and cheap geometric features of a workload's cut (ADMM ordering study).
Writes gpurun_out/qp_features_<cfg>.npz: iterations, status, work-list order, and per instance
dmin (smallest control-point distance to the box), ovmin (smallest bbox overlap)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2411_13507_b200 import _native as nat, configs, graph as G  # noqa: E402


def main(cfg="cfg3"):
    ctx = nat.Context(0)
    w = configs.BUILDERS[cfg]()
    g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
    m = G.cut_graph(g, w.obstacles)
    r = m.qp_records()
    P = g.edge_points
    lo = np.stack([-np.asarray(o.b)[2:4] for o in w.obstacles])
    hi = np.stack([np.asarray(o.b)[:2] for o in w.obstacles])
    pts = P[r["edge"]]  # (n, 2, J)
    l = lo[r["obstacle"]][:, :, None]
    h = hi[r["obstacle"]][:, :, None]
    dx = np.maximum(l - pts, 0) + np.maximum(pts - h, 0)
    dist = np.sqrt((dx ** 2).sum(1))
    mn, mx = pts.min(2), pts.max(2)
    ov = np.minimum(mx, h[:, :, 0]) - np.maximum(mn, l[:, :, 0])
    Path("gpurun_out").mkdir(exist_ok=True)
    np.savez_compressed(f"gpurun_out/qp_features_{cfg}.npz", iters=r["iterations"], status=r["status"],
                        edge=r["edge"], obstacle=r["obstacle"], dmin=dist.min(1), ovmin=ov.min(1))
    print(cfg, r["iterations"].size)


if __name__ == "__main__":
    main(*sys.argv[1:])
