#!/usr/bin/env python
"""Isolate the costs inside the sharded step's reduce-scatter + pass 1.

torchrun --nproc-per-node N tools/rs_probe.py   (N = 2, 4 or 8)

For bucket 0 of the ResNet-50 wire (theta = 16 MiB) times, per call, max
over ranks, back-to-back calls after a device barrier:
  rs_pass1_staged   gs_rs_pass1, cp.async-staged chunk
  rs_pass1_direct   gs_rs_pass1, register loads
  rs_fold           gs_ordered_reduce_scatter_f16 over the same slices
  pass1_local       gs_lars_pass1 over the rank's owned chunks (no NVLink)
  copy_local        gs_fill_zero of the rank's slice bytes (HBM write only)
"""

import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    import torch.distributed as dist

    import paper_1807_11205_b200 as gs
    from paper_1807_11205_b200 import _device as dv, _native, shapes as sh
    from paper_1807_11205_b200.dist import Communicator, init_from_env

    rank, world, local = init_from_env("nccl")
    dev = torch.device("cuda", local)
    specs = sh.load_shapes("resnet50")
    comm = Communicator(gs.Topology(world, 1))
    cfg = gs.LarsConfig(gs.Schedule(0.1), eta=0.001, weight_decay=5e-4, momentum=0.9)
    pipe = gs.GradientPipeline(specs, cfg, threshold_bytes=16 << 20, comm=comm,
                               sharded_update=True, init_master=sh.synth_master(specs),
                               loss_scale=gs.LossScale(1024.0), device=dev)
    grads = torch.from_numpy(sh.synth_wire_grads(specs, rank=rank, seed=0)).to(dev)
    for i in range(3):
        pipe.step(grads, i)
    torch.cuda.synchronize(dev)
    s0 = torch.cuda.current_stream(dev)
    sh_ = int(s0.cuda_stream)
    plan, a = pipe.plan, pipe.arena
    wire = pipe._halves[0]
    plan.use_segments(plan.alt_segments([wire.data_ptr() + 2 * o for o in pipe.wire_off]))
    plan.upload_params(s0)
    wires = a.peers("wireA")
    sig, ebase = dv.ptr(a.peers("sig")), dv.ptr(pipe.epoch_base)
    tok = torch.zeros(1, device=dev)
    out = {}
    for b in range(len(pipe.buckets)):
        c0, c1 = pipe._own_bucket[b]
        E = pipe._bucket_E[b]
        elems = E[rank + 1] - E[rank]
        scratch = torch.empty(2 * elems, dtype=torch.uint8, device=dev)

        def rs(direct):
            hint = plan.hint | (0 if direct else _native.HINT_RS_STAGE)
            _native.call("gs_rs_pass1", dv.ptr(wires), None, sig, rank, world, dv.ptr(plan.d_segs),
                         dv.ptr(plan.d_chunks), c0, c1, None, dv.ptr(plan.params), hint,
                         dv.ptr(a.peers("partials")), dv.ptr(a.peers("flags")), 1, ebase,
                         pipe._nblocks, sh_)
            _native.call("gs_counter_add", ebase, 1, sh_)

        def fold():
            _native.call("gs_ordered_reduce_scatter_f16", dv.ptr(wires), sig, rank, world,
                         dv.ptr(pipe._rs_bounds[b]), 1, ebase, pipe._nblocks, None, sh_)
            _native.call("gs_counter_add", ebase, 1, sh_)

        def p1():
            plan.pass1(sh_, g_is_f16=True, chunk0=c0, nchunk=c1 - c0)

        def wr():
            _native.call("gs_fill_zero", scratch.data_ptr(), scratch.numel(), sh_)

        res = {}
        for name, fn in (("rs_pass1_staged", lambda: rs(False)), ("rs_pass1_direct", lambda: rs(True)),
                         ("rs_fold", fold), ("pass1_local", p1), ("copy_local", wr)):
            times = []
            for rep in range(5):
                dist.all_reduce(tok)
                # the host queues every call while the GPU sleeps: the events
                # then time device work, not the host's launch rate
                torch.cuda._sleep(8_000_000)
                ev0 = torch.cuda.Event(enable_timing=True)
                ev1 = torch.cuda.Event(enable_timing=True)
                ev0.record(s0)
                for _ in range(10):
                    fn()
                ev1.record(s0)
                ev1.synchronize()
                times.append(ev0.elapsed_time(ev1) / 10 * 1e3)
            t = torch.tensor([statistics.median(times)], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            res[name] = round(float(t), 2)
        res["elems_per_rank"] = elems
        res["chunks_per_rank"] = c1 - c0
        res["nvlink_in_gbs_rs_pass1"] = round((world - 1) * 2 * elems / (res["rs_pass1_direct"] * 1e-6) / 1e9, 1)
        res["nvlink_in_gbs_fold"] = round((world - 1) * 2 * elems / (res["rs_fold"] * 1e-6) / 1e9, 1)
        out[f"bucket{b}"] = res
    plan.use_segments(None)
    if rank == 0:
        print(json.dumps({"probe": "rs", "p": world, "nblocks": pipe._nblocks, **out}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
