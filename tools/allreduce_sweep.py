#!/usr/bin/env python
"""All-reduce message-size sweep (BASELINE.json config 5).

fp16 sum all-reduce of 2^10 ... 2^30 bytes at p = WORLD_SIZE GPUs, for every
variant the pipeline can pick per bucket (collectives.py:238-340):

  ring                 flat 1xp ncclAllReduce (fp16 wire)
  hierarchical_GxK     the paper's literal reduce -> masters all-reduce ->
                       broadcast on Topology(p, K) sub-communicators
  sharded_GxK          intra-group reduce-scatter -> same-offset all-reduce ->
                       intra-group all-gather
  ordered              our symmetric-memory NVLink kernel, reference fold order

with FORCED OVERFLOW: rank 0's buffer carries 0x7C00 (+Inf) at element 0 and
every other element is a finite binary16, so every result must carry Inf
there — the overflow flag the loss scale's skip decision reads
(halfprec.py:209-216).  The ordered kernel reports it through its own
non-finite flag; NCCL results are checked directly.  busBW = S/t * 2(p-1)/p
(nccl-tests convention) for every variant; max over ranks of the per-rank
CUDA-event time on the launching stream, with the calls queued behind a
device sleep so the events time the GPU, not the host launch rate.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
      --master-addr 127.0.0.1 --master-port P tools/allreduce_sweep.py [--max-log2 30]

Rank 0 prints one JSON line per (size, variant) and a final summary line.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log2", type=int, default=10)
    ap.add_argument("--max-log2", type=int, default=30)
    ap.add_argument("--variants",
                    default="ring,hierarchical,sharded,ordered,ordered_push,ordered_oneshot,ordered_ll,"
                            "ordered_hier,ordered_hier_push")
    ap.add_argument("--out", default=None, help="also write the lines to this file (rank 0)")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    import paper_1807_11205_b200 as gs
    from paper_1807_11205_b200 import _device as dv
    from paper_1807_11205_b200._peer import launch
    from paper_1807_11205_b200.dist import Communicator, OrderedWire, init_from_env

    rank, world, local = init_from_env("nccl")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    s0 = torch.cuda.current_stream(dev)
    want = set(args.variants.split(","))
    max_elems = (1 << args.max_log2) // 2

    variants = []
    if "ring" in want:
        variants.append(("ring", 1))
    for k in (4, 2):
        if 1 < k < world and world % k == 0:
            if "hierarchical" in want:
                variants.append((f"hierarchical_{world // k}x{k}", k))
            if "sharded" in want:
                variants.append((f"sharded_{world // k}x{k}", k))
    if "ordered" in want:
        variants.append(("ordered", 1))
    if "ordered_push" in want:
        variants.append(("ordered_push", 1))
    if "ordered_oneshot" in want:
        variants.append(("ordered_oneshot", 1))
    if "ordered_ll" in want:
        variants.append(("ordered_ll", 1))
    for form in ("ordered_hier", "ordered_hier_push"):
        if form in want:
            for k in (4, 2):
                if 1 < k < world and world % k == 0:
                    variants.append((f"{form}_{world // k}x{k}", k))
    comms = {k: Communicator(gs.Topology(world, k)) for k in sorted({k for _, k in variants})}
    # bookkeeping reductions on CPU (gloo): NCCL_ALGO=NVLS runs have no fp64/int path
    host = dist.new_group(backend="gloo")

    # finite binary16 payload (small values: no finite sum overflows), Inf at 0 on rank 0
    g = torch.Generator(device="cpu").manual_seed(1234 + rank)
    base = (torch.rand(max_elems, generator=g) * 2e-3 - 1e-3).to(torch.float16).to(dev)
    buf = torch.empty_like(base)
    # small-bucket inboxes up to 2 MB buckets, so the sweep shows the crossover
    OrderedWire.SMALL_CAP_ELEMS = 1 << 20
    OrderedWire.PUSH_MAX_BYTES = 0  # "ordered" is the pure pull form here
    ow = OrderedWire(comms[1], max_elems, dev) if any(v[0].startswith("ordered") for v in variants) \
        else None
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    if ow is not None:
        ow.ctx["nonfinite"] = dv.ptr(flag)  # the kernels OR 1 here on a non-finite sum
    tok = torch.zeros(1, dtype=torch.float32, device=dev)
    sleep_cycles = 1.0e7  # ~5 ms at 2 GHz, longer than queueing 50 eager calls
    half = [0]
    lines = []
    for lg in range(args.min_log2, args.max_log2 + 1):
        S = 1 << lg
        n = S // 2
        for name, k in variants:
            comm = comms[k]
            algo = "ordered" if name.startswith("ordered") else name.split("_")[0]
            nn = n - n % k if algo == "sharded" else n
            if nn == 0 or (name in ("ordered_oneshot", "ordered_ll") and nn > ow.cap):
                continue
            if algo == "ordered":
                def refill():
                    h = ow.halves[half[0]]
                    h[:nn].view(torch.float16).copy_(base[:nn])
                    if rank == 0:
                        h[:1].view(torch.int16).fill_(0x7C00)

                def run(_push="push" in name,
                        _k=k if name.startswith("ordered_hier") else 0):
                    ow.push = _push
                    sh = int(s0.cuda_stream)
                    op = ow.hier_op(half[0], 0, nn, _k, sh) if _k else \
                        ow.allreduce_op(half[0], 0, nn, sh, small={"ordered_oneshot": "oneshot",
                                                                   "ordered_ll": "ll"}.get(name, "none"))
                    launch([op])
                    ow.advance(1, sh)
                    half[0] ^= 1

                def result():
                    return ow.halves[half[0] ^ 1][:nn].view(torch.float16)
            else:
                t = buf[:nn]

                def refill(_t=t):
                    _t.copy_(base[:nn])
                    if rank == 0:
                        _t[:1].view(torch.int16).fill_(0x7C00)

                def run(_t=t, _c=comm, _a=algo):
                    _c.allreduce(_t, _a)

                def result(_t=t):
                    return _t
            # correctness of the forced-overflow path (one untimed call)
            flag.zero_()
            refill()
            if algo == "ordered":
                refill()  # both halves hold the payload
                half[0] ^= 1
                refill()
                half[0] ^= 1
            torch.cuda.synchronize(dev)
            dist.barrier(group=host)
            run()
            torch.cuda.synchronize(dev)
            r = result()
            inf_ok = bool(torch.isinf(r[0]).item())
            finite_rest = bool(torch.isfinite(r[1:]).all().item()) if nn > 1 else True
            # the ordered kernel flags the slice its rank folded: OR over ranks
            flag_any = torch.tensor([int(flag.item())], dtype=torch.int64)
            dist.all_reduce(flag_any, op=dist.ReduceOp.MAX, group=host)
            flag_ok = bool(flag_any.item() != 0) if algo == "ordered" else None
            # timing: in-place repeats grow the values by ~p per call until they
            # saturate to Inf; binary16 adds cost the same on any value
            iters = 50 if S <= (1 << 20) else (20 if S <= (1 << 26) else 5)
            for _ in range(3):
                run()
            torch.cuda.synchronize(dev)
            dist.barrier(group=host)
            # line the ranks' streams up, then let the host queue every call
            # while the GPU sleeps, so the events time device work and not the
            # host's launch rate (which bounds eager small-message calls)
            comms[1].allreduce_ring(tok)
            torch.cuda._sleep(int(sleep_cycles))
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s0)
            for _ in range(iters):
                run()
            b.record(s0)
            b.synchronize()
            ms = torch.tensor([a.elapsed_time(b) / iters], dtype=torch.float64)
            dist.all_reduce(ms, op=dist.ReduceOp.MAX, group=host)
            ok = torch.tensor([int(inf_ok and finite_rest and flag_ok is not False)],
                              dtype=torch.int64)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=host)
            sec = float(ms) * 1e-3
            Sb = 2 * nn
            line = {"bytes": Sb, "variant": name, "p": world, "us": round(sec * 1e6, 2),
                    "algbw_gbs": round(Sb / sec / 1e9, 2),
                    "busbw_gbs": round(Sb / sec * 2 * (world - 1) / world / 1e9, 2),
                    "overflow_propagated": bool(ok.item()), "iters": iters}
            if rank == 0:
                print(json.dumps(line), flush=True)
            lines.append(line)
    if rank == 0:
        best = {}
        for ln in lines:
            v = ln["variant"]
            best[v] = max(best.get(v, 0.0), ln["busbw_gbs"])
        summary = {"summary": "allreduce_sweep", "p": world,
                   "nccl_algo_env": os.environ.get("NCCL_ALGO"),
                   "peak_busbw_gbs": best,
                   "all_overflow_propagated": all(ln["overflow_propagated"] for ln in lines)}
        print(json.dumps(summary), flush=True)
        if args.out:
            Path(args.out).write_text("\n".join(json.dumps(x) for x in lines + [summary]) + "\n")
    dist.barrier(group=host)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
