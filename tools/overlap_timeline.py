#!/usr/bin/env python
"""Timeline evidence for the backward-overlap driver.

nsys is not in this image; torch.profiler (Kineto over CUPTI) records the
same device timeline.  A conv net runs fp16 forward/backward with
BackwardOverlap hooking its parameters into a GradientPipeline; with NVTX
phase ranges on (GS_NVTX=1) three steps are profiled and the chrome trace is
analysed:

  * every kernel of ours (pack / pass 1 on the side stream, trust / pass 2
    on the compute stream) and every backward kernel, by stream;
  * for the side-stream bucket kernels, the fraction of their time that
    overlaps a backward kernel on the compute stream (> 0: the bucket work
    runs UNDER backward, as PAPER.md:177 describes);
  * the exposed tail: from the last backward kernel to the end of pass 2.

  python tools/overlap_timeline.py [--out gpurun_out/overlap] > summary.json
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ["GS_NVTX"] = "1"

import torch  # noqa: E402

import paper_1807_11205_b200 as gs  # noqa: E402

OURS = ("lars_pass1", "lars_trust", "lars_pass2", "batched_copy", "ordered_allreduce",
        "oneshot_allreduce", "rs_pass1", "pass2_push", "peer_fence", "fold_")


class Net(torch.nn.Module):
    def __init__(self, width=128, depth=10):
        super().__init__()
        layers, c = [], 3
        for i in range(depth):
            layers += [torch.nn.Conv2d(c, width, 3, padding=1, bias=False),
                       torch.nn.BatchNorm2d(width), torch.nn.ReLU()]
            c = width
        self.body = torch.nn.Sequential(*layers)
        self.fc = torch.nn.Linear(width, 100)

    def forward(self, x):
        return self.fc(self.body(x).mean(dim=(2, 3)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/overlap")
    ap.add_argument("--theta", type=int, default=1 << 20)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--res", type=int, default=64)
    ap.add_argument("--width", type=int, default=256)
    ap.add_argument("--algorithm", default="zero", choices=["zero", "ordered"],
                    help="multi-GPU (torchrun): the sharded fused step or the ordered all-reduce")
    args = ap.parse_args()
    torch.manual_seed(0)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = 0
    kw = {}
    if world > 1:
        from paper_1807_11205_b200.dist import Communicator, init_from_env
        rank, world, local = init_from_env("nccl")
        torch.cuda.set_device(local)
        comm = Communicator(gs.Topology(world, 1))
        kw = dict(comm=comm, sharded_update=args.algorithm == "zero",
                  flat_variant="ordered", eta_bytes=0)
        args.out = f"{args.out}_rank{rank}"
    # GPU-bound backward (each conv's backward takes longer than the host
    # needs to launch it), so a side-stream kernel CAN run beside it
    net = Net(width=args.width).cuda()
    cfg = gs.LarsConfig(gs.Schedule(0.1), eta=0.001, weight_decay=5e-4, momentum=0.9)
    drv = gs.BackwardOverlap.for_module(net, cfg, threshold_bytes=args.theta,
                                        loss_scale=gs.LossScale(1024.0), **kw)
    x = torch.randn(args.batch, 3, args.res, args.res, device="cuda").half()
    y = torch.randint(0, 100, (args.batch,), device="cuda")

    def one(step):
        drv.begin(step)
        loss = torch.nn.functional.cross_entropy(net(x).float(), y)
        (loss * drv.loss_scale).backward()
        return drv.finish()

    for s in range(3):
        one(s)
    torch.cuda.synchronize()
    acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
    with torch.profiler.profile(activities=acts) as prof:
        for s in range(3, 6):
            one(s)
        torch.cuda.synchronize()
    out = Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    trace = str(out) + "_trace.json"
    prof.export_chrome_trace(trace)
    ev = json.load(open(trace))["traceEvents"]
    kern = [e for e in ev if e.get("cat") == "kernel"]
    ours = [e for e in kern if any(k in e["name"] for k in OURS)]
    other = [e for e in kern if e not in ours]
    by_stream: dict = {}
    for e in ours:
        by_stream.setdefault(e["args"].get("stream"), []).append(e)
    comp_stream = max({e["args"].get("stream") for e in other},
                      key=lambda s: sum(e["dur"] for e in other if e["args"].get("stream") == s))
    side = [e for e in ours if e["args"].get("stream") != comp_stream]
    comp = sorted((e["ts"], e["ts"] + e["dur"]) for e in other
                  if e["args"].get("stream") == comp_stream)

    def overlap(a, b):
        tot = 0.0
        for s, t in comp:
            lo, hi = max(a, s), min(b, t)
            if hi > lo:
                tot += hi - lo
        return tot

    side_time = sum(e["dur"] for e in side)
    side_under = sum(overlap(e["ts"], e["ts"] + e["dur"]) for e in side)
    # per step: the compute stream's last non-optimizer kernel (end of
    # backward) to the end of pass 2 = what the optimizer step adds
    p2 = sorted(e["ts"] + e["dur"] for e in ours
                if "lars_pass2" in e["name"] or "pass2_push" in e["name"])
    tails = []
    for end in p2:
        before = [t for s_, t in comp if t <= end]
        if before:
            tails.append(end - max(before))
    ranges = [e for e in ev if e.get("cat") == "user_annotation" and e["name"].startswith("gs.")]
    summary = {
        "trace": trace, "theta": args.theta, "buckets": len(drv.pipe.buckets),
        "params": sum(drv.pipe.sizes), "compute_stream": comp_stream,
        "our_kernels_by_stream": {str(k): sorted({next(o for o in OURS if o in e["name"])
                                                  for e in v}) for k, v in by_stream.items()},
        "side_stream_kernel_us": round(side_time, 1),
        "side_stream_us_under_backward": round(side_under, 1),
        "side_overlap_fraction": round(side_under / side_time, 3) if side_time else None,
        "exposed_tail_us_per_step": [round(t, 1) for t in tails],
        "config": {"batch": args.batch, "res": args.res, "width": args.width, "depth": 10,
                   "world": world, "rank": rank,
                   "algorithm": args.algorithm if world > 1 else "none"},
        "nvtx_ranges": sorted({e["name"] for e in ranges}),
        "steps_profiled": 3,
    }
    print(json.dumps(summary, indent=1))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
