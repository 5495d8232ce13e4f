"""Multi-GPU parity (tests/mgpu_check.py) under pytest: one process per GPU via
torchrun over every visible GPU (2, 4 or 8).  Skipped on boxes with fewer
than two GPUs; the development runner's 2- and 4-GPU results are under
profiles/ (mgpu_check_*)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs at least 2 GPUs")
@pytest.mark.timeout(900)
def test_multi_gpu_parity_all_algorithms():
    n = torch.cuda.device_count()
    n = 8 if n >= 8 else (4 if n >= 4 else 2)
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29977",
           str(ROOT / "tests" / "mgpu_check.py")]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=850)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    res = json.loads(line)["results"]
    bad = {k: v for k, v in res.items() if not v["ok"]}
    assert not bad, bad
    assert {"zero", "ordered", "ring", "zero_inc"} <= set(res)
