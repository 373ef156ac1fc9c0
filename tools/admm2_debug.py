"""Compare k_qp_admm (BZG_ADMM_LANES=1) with k_qp_admm2 (=2) instance by instance on a golden scene."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2411_13507_b200 import _native as nat  # noqa: E402
from paper_2411_13507_b200 import graph as G  # noqa: E402
from tests.conftest import load_golden  # noqa: E402
from tests.helpers import inputs_from_golden  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rf300_s5"
g = load_golden(name)
ctx = nat.Context(0)
N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(g)
gr = G.build_graph(N, spec, orc, bounds, seed, include, ctx=ctx)
rec = {}
for lanes in ("1", "2"):
    os.environ["BZG_ADMM_LANES"] = lanes
    rec[lanes] = G.cut_graph(gr, obstacles).qp_records()
a, b = rec["1"], rec["2"]
for r in (a, b):
    o = np.argsort(r["edge"] * 1_000_003 + r["obstacle"], kind="stable")
    for k in list(r):
        r[k] = r[k][o]
print("n", a["status"].size, "status eq", (a["status"] == b["status"]).mean(), "iters eq",
      (a["iterations"] == b["iterations"]).mean(), "delta eq", (a["delta"] == b["delta"]).mean())
print("status hist 1", np.bincount(a["status"], minlength=4), "2", np.bincount(b["status"], minlength=4))
print("iters mean", a["iterations"].mean(), b["iterations"].mean())
d = np.nonzero(a["iterations"] != b["iterations"])[0][:10]
for i in d:
    print(i, a["status"][i], b["status"][i], a["iterations"][i], b["iterations"][i], a["delta"][i], b["delta"][i])
