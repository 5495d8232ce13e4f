"""Calibrate the α-β model on the measured all-reduce sweeps and seed η.

    python tools/calibrate_netsim.py > profiles/netsim_calibration.json
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1807_11205_b200.collectives import Topology, hierarchical_schedule, ring_schedule  # noqa: E402
from paper_1807_11205_b200.netsim import calibrate_from_sweep, calibrated_eta, load_sweep, simulate  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
out = []
for path, p, k in [("profiles/final_n4/sweep_fin_n4.jsonl", 4, 2),
                   ("profiles/final_n2/sweep_fin_n2.jsonl", 2, 1)]:
    rows = load_sweep(ROOT / path)
    link = calibrate_from_sweep(rows, p, k)
    eta, _ = calibrated_eta(p, k, link)
    fit = []
    for r in rows:
        if r["variant"] == "ring" or r["variant"] == f"hierarchical_{k}x{p // k}":
            n = r["bytes"] // 2
            s = (ring_schedule(p, n, 2, k=k) if r["variant"] == "ring"
                 else hierarchical_schedule(Topology(p, k), n, 2))
            fit.append({"variant": r["variant"], "bytes": r["bytes"], "measured_us": r["us"],
                        "model_us": round(simulate(s, link).total_time * 1e6, 2)})
    out.append({"sweep": path, "p": p, "k": k, "link": link.to_dict(),
                "eta_bytes": eta, "fit": fit})
print(json.dumps(out, indent=1))
