#!/usr/bin/env python
"""Summarise a multi-GPU session (tools/mgpu_quick.sh / mgpu_full.sh output)
into markdown: step time per algorithm with its phase split, the sharded
kernels' NVLink rates, whole-gradient busBW, parity verdicts, and the
message-size sweep.

usage: python tools/mgpu_summary.py gpurun_out TAG N > profiles/<name>.md
"""

import glob
import json
import os
import re
import sys


def last_json(path):
    line = None
    with open(path) as f:
        for ln in f:
            if ln.startswith("{"):
                line = ln
    return json.loads(line) if line else None


def main():
    d, tag, n = sys.argv[1], sys.argv[2], sys.argv[3]
    print(f"# multi-GPU session `{tag}`, N = {n} B200\n")
    print("Step = one fused MP-LARS step on ResNet-50 gradients (25.6 M params) unless "
          "the name says otherwise; ms per step, max over ranks, CUDA events, L2 flushed "
          "(write + read) and ranks lined up by a 4-byte all-reduce before every step.\n")
    print("| run | step ms | e2e ms | buckets | phases (µs) | NVLink GB/s (rs_pass1 in / pass2_push out) |")
    print("|---|---|---|---|---|---|")
    ar = None
    for f in sorted(glob.glob(os.path.join(d, f"bench_{tag}_n{n}_*.log"))):
        j = last_json(f)
        name = re.sub(rf"^bench_{tag}_n{n}_", "", os.path.basename(f))[:-4]
        if j is None:
            print(f"| {name} | failed | | | | |")
            continue
        ph = ", ".join(f"{k} {v * 1e3:.0f}" for k, v in (j.get("phases_ms") or {}).items())
        nv = (j.get("roofline") or {}).get("nvlink") or {}
        nvs = f"{nv.get('rs_pass1_in_gbs', '')} / {nv.get('pass2_push_out_gbs', '')}" if nv else ""
        e2e = (j.get("e2e") or {}).get("value", "")
        print(f"| {name} | {j['value']} | {e2e} | {j['config'].get('buckets')} | {ph} | {nvs} |")
        if j.get("allreduce"):
            ar = j["allreduce"]
    if ar:
        print(f"\n## whole-gradient all-reduce ({ar['bytes']} B fp16)\n")
        print("| variant | µs | busBW GB/s | algBW GB/s |")
        print("|---|---|---|---|")
        for k, v in ar.items():
            if isinstance(v, dict):
                print(f"| {k} | {v['us']} | {v['busbw_gbs']} | {v['algbw_gbs']} |")
    print("\n## parity (tests/mgpu_check.py)\n")
    for f in sorted(glob.glob(os.path.join(d, f"mgpu_check_{tag}_n{n}*.log"))):
        j = last_json(f)
        if j is None:
            print(f"* {os.path.basename(f)}: no result")
            continue
        res = ", ".join(f"{k} {'ok' if v['ok'] else 'FAIL'}" for k, v in j["results"].items())
        print(f"* {os.path.basename(f)} ({j['model']}, theta {j['theta']}): {res}")
    for f in sorted(glob.glob(os.path.join(d, f"sweep_{tag}_n{n}*.jsonl"))):
        rows = {}
        summ = None
        for ln in open(f):
            x = json.loads(ln)
            if "bytes" in x:
                rows.setdefault(x["bytes"], {})[x["variant"]] = x
            else:
                summ = x
        vs = sorted({v for r in rows.values() for v in r})
        print(f"\n## message-size sweep {os.path.basename(f)} (+Inf forced on rank 0)\n")
        print("| bytes | " + " | ".join(f"{v} µs / busBW" for v in vs) + " |")
        print("|---|" + "---|" * len(vs))
        for b in sorted(rows):
            cells = []
            for v in vs:
                x = rows[b].get(v)
                cells.append(f"{x['us']} / {x['busbw_gbs']}{'' if x['overflow_propagated'] else ' (!)'}"
                             if x else "")
            print(f"| {b} | " + " | ".join(cells) + " |")
        if summ:
            print(f"\nall overflow propagated: {summ.get('all_overflow_propagated')}; "
                  f"peak busBW: {summ.get('peak_busbw_gbs')}")


if __name__ == "__main__":
    main()
