"""The N > 1 row-block path on a real device: every rank on cuda:0, host-side (gloo)
collectives, result checked against one process by tools/dist_check.py (rank 0).

The one-GPU box cannot run NCCL ranks on separate devices; this covers the sharded build,
local cut, gather and adoption of the union through libbzg on the device, and the
gloo tests in test_shard_gloo.py cover the same exchange logic on CPU."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("world", [2, 3])
def test_row_block_gather_matches_single_process(world):
    env = dict(os.environ, BZG_DIST_BACKEND="gloo", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world), str(ROOT / "tools" / "dist_check.py"),
           "cfg2"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    print(res.stdout[-2000:])
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "checks=" in res.stdout
