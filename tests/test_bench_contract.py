"""bench.py's reference arm runs on the host and prints the contract's JSON
line (CPU test: the reference arm needs no GPU)."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--model", "shufflenet_v2_x0_5", "--theta", str(256 << 10),
                          "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "ms" and d["higher_is_better"] is False
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 1
    cfg = d["config"]
    assert cfg["model"] == "shufflenet_v2_x0_5" and cfg["params"] == 1366792
    assert cfg["tensors"] == 170 and cfg["theta"] == 256 << 10 and cfg["buckets"] == 4
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["value"] == d["value"] and cb["cores"] >= 1
    assert set(cb["stages_ms"]) == {"pack", "fold", "unscale", "lars"}
    assert d["e2e"] == {"value": d["value"], "unit": "ms", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_both_arms_print_the_same_config_keys():
    """run_ours and run_reference both print workload_config(args, world)."""
    sys.path.insert(0, str(ROOT))
    import bench

    args = bench.parse(["--gpus", "2", "--algorithm", "zero"])
    a = bench.workload_config(args, 2)
    assert a["parallelism"] == "dp2" and a["topology"] == "Topology(2,1)"
    assert a["algorithm"] == "zero" and a["buckets"] == 3 and "loss_scale" not in a
    src = (ROOT / "bench.py").read_text()
    assert src.count('"config": workload_config(args, world)') == 2
    b = bench.workload_config(bench.parse(["--loss-scale", "1000"]), 1)
    assert b["loss_scale"] == 1000.0 and b["algorithm"] == "none"
