"""NVLink peer-access probe (tools only): pull / push of a rank's 1/p slice
from / into every peer of a symmetric-memory buffer, timed with CUDA events,
max over ranks.  Run under torchrun, e.g.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        tools/nvlink_probe.py --mbytes 51
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent
LIB = ROOT / "_probe" / "libnvprobe.so"


def build():
    LIB.parent.mkdir(exist_ok=True)
    if not LIB.exists() or LIB.stat().st_mtime < (ROOT / "nvlink_probe.cu").stat().st_mtime:
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                        "-Xcompiler", "-fPIC", str(ROOT / "nvlink_probe.cu"), "-o", str(LIB)],
                       check=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mbytes", type=float, default=51.1)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        build()
    dist.barrier()
    lib = ctypes.CDLL(str(LIB))
    lib.probe_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                              ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                              ctypes.c_int, ctypes.c_void_p]
    import torch.distributed._symmetric_memory as symm
    p = world
    total = int(args.mbytes * 1e6) // (p * 65536) * p * 65536
    slice_bytes = total // p
    buf = symm.empty(total, dtype=torch.uint8, device=dev)
    buf.fill_(rank + 1)
    hdl = symm.rendezvous(buf, dist.group.WORLD.group_name)
    peers = torch.tensor([int(x) for x in hdl.buffer_ptrs], dtype=torch.int64, device=dev)
    scratch = torch.zeros(1 << 20, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream()
    sh = int(s.cuda_stream)
    tok = torch.zeros(1, device=dev)
    configs = []
    for U in (1, 2, 4):
        for g in (148 * 2, 148 * 4, 148 * 8):
            configs.append(("pull_ldg", 0, U, g, 0))
    for S in (2, 4, 8):
        for blk in (8192, 16384, 32768):
            if S * blk > 200 * 1024:
                continue
            for g in (148, 148 * 2):
                if g == 296 and S * blk > 100 * 1024:
                    continue
                configs.append(("pull_tma", 2, S, g, blk))
    for U in (1, 2, 4):
        for g in (148 * 2, 148 * 4, 148 * 8):
            configs.append(("push_st", 1, U, g, 0))
    results = []
    for name, mode, U, g, blk in configs:
        ts = []
        for r in range(args.reps + 2):
            dist.barrier()
            torch.cuda._sleep(500_000)
            dist.all_reduce(tok)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            rc = lib.probe_run(mode, U, peers.data_ptr(), p, rank, slice_bytes, scratch.data_ptr(),
                               g, blk, sh)
            b.record(s)
            b.synchronize()
            if rc != 0:
                raise RuntimeError(f"{name} rc={rc}")
            if r >= 2:
                ts.append(a.elapsed_time(b))
        t = torch.tensor([sorted(ts)[len(ts) // 2]], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        us = float(t[0]) * 1e3
        nv = (p - 1) * slice_bytes
        results.append({"kernel": name, "U_or_stages": U, "grid": g, "blk": blk, "us": round(us, 2),
                        "nvlink_gbs": round(nv / us / 1e3, 1),
                        "all_bytes_gbs": round(p * slice_bytes / us / 1e3, 1)})
        if rank == 0:
            print(json.dumps(results[-1]), flush=True)
    if rank == 0:
        best = {}
        for r in results:
            if r["nvlink_gbs"] > best.get(r["kernel"], {}).get("nvlink_gbs", 0):
                best[r["kernel"]] = r
        print(json.dumps({"summary": "nvlink_probe", "p": p, "slice_bytes": slice_bytes,
                          "best": best}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
