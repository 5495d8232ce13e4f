"""Multi-GPU parity check of the pipeline (run on a GPU box, not by pytest):

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mgpu_check.py

"ordered" (symmetric-memory peer fold) must be bit-exact at every N.
Every rank steps GradientPipeline(comm=Communicator(Topology(N, k))) on its own
synthetic fp16 gradients; rank 0 recomputes the reference composition with the
CPU oracle.  Checks per algorithm (ring / hierarchical / sharded):
  * N = 2: NCCL's fp16 sum of two operands is one correctly rounded add, the
    same as the reference's pairwise tree -> master/velocity/working and the
    trust scales must be BIT-EXACT;
  * N > 2: NCCL's order differs from the tree -> the reduced buckets must be
    within 2^-9 * sum|x| (test_collectives.py:237-250 bound) and the update,
    recomputed by the oracle from the GPU's own reduced buckets, bit-exact.
Also an injected Inf on one rank must skip the step on every rank.
"""

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1807_11205_b200 as gs  # noqa: E402
from oracle import reference_port as rp  # noqa: E402
from paper_1807_11205_b200 import shapes as sh  # noqa: E402
from paper_1807_11205_b200.dist import Communicator, init_from_env  # noqa: E402


def split(flat, specs):
    out, o = [], 0
    for s in specs:
        out.append(flat[o:o + s.numel])
        o += s.numel
    return out


def main():
    rank, world, local = init_from_env("nccl")
    dev = torch.device("cuda", local)
    model = os.environ.get("MGPU_MODEL", "shufflenet_v2_x0_5")
    theta = int(os.environ.get("MGPU_THETA", str(256 << 10)))
    specs = sh.load_shapes(model)
    master = sh.synth_master(specs)
    order = list(reversed(range(len(specs))))
    results = {}
    algos = os.environ.get("MGPU_ALGOS", "zero,zero_unfused,ordered,ordered_push,ordered_hier,ring,"
                           "hierarchical,sharded,zero_inc,ordered_inc,ring_inc,zero_host,"
                           "ordered_host,zero_busy,ordered_busy,ordered_hier_push").split(",")
    for algo_name, k in (("zero", 1), ("zero_unfused", 1), ("ordered", 1), ("ordered_push", 1),
                         ("ordered_hier", 2), ("ring", 1),
                         ("hierarchical", 2), ("sharded", 2), ("zero_inc", 1), ("ordered_inc", 1),
                         ("ring_inc", 1), ("zero_host", 1), ("ordered_host", 1),
                         ("zero_busy", 1), ("ordered_busy", 1), ("ordered_hier_push", 2)):
        if algo_name not in algos:
            continue
        # *_inc: the same step driven through the incremental API the
        # backward-overlap driver uses (begin / submit per bucket / end),
        # buckets submitted in REVERSE order to exercise the in-order gating
        # *_busy: the incremental path while another stream keeps every SM
        # busy with GEMMs of a rank-dependent length (the backward pass the
        # overlap driver runs against): the spin-waiting peer kernels must
        # still make progress and give the same bits
        busy = algo_name.endswith("_busy")
        inc = algo_name.endswith("_inc") or busy
        # *_host: the same step from a pinned HOST gradient (enqueue_host:
        # per-bucket H2D overlapped with the incremental submission)
        host = algo_name.endswith("_host")
        algo = algo_name[:-5] if busy else algo_name[:-4] if inc else \
            algo_name[:-5] if host else algo_name
        push = algo in ("ordered_push", "ordered_hier_push")
        if push:
            algo = "ordered" if algo == "ordered_push" else "ordered_hier"
        if world % k or (algo != "ring" and world == 1):
            continue
        comm = Communicator(gs.Topology(world, k))
        cfg = gs.LarsConfig(gs.Schedule(0.1), eta=0.001, weight_decay=5e-4, momentum=0.9)
        pipe = gs.GradientPipeline(specs, cfg, threshold_bytes=theta, comm=comm,
                                   eta_bytes=0 if algo in ("ring", "ordered") else 1 << 62,
                                   hier_variant=algo if algo not in ("ring", "ordered") else "hierarchical",
                                   flat_variant="ordered" if algo == "ordered" else "ring",
                                   ordered_push=push,
                                   sharded_update=algo.startswith("zero"),
                                   fused_collective=algo == "zero",
                                   init_master=master, loss_scale=gs.LossScale(1024.0), device=dev)
        groups = [rp.Group(s.name, s.kind, w.copy(), np.zeros(s.numel, np.float32),
                           np.zeros(s.numel, np.float32), rp.narrow(w))
                  for s, w in zip(specs, split(master, specs))]
        oloss = rp.LossScaleState(1024.0)
        ok = True
        notes = []
        for step in range(3):
            wires = [sh.synth_wire_grads(specs, rank=r, seed=step, loss_scale=oloss.scale)
                     for r in range(world)]
            if step == 2:
                wires[world - 1][4321] = 0x7C00
            flat = torch.from_numpy(wires[rank]).to(dev)
            if host:
                pipe.enqueue_host(torch.from_numpy(wires[rank]).pin_memory(), step)
                res = pipe.finish()
            elif inc:
                views = split(flat, specs)
                if busy:
                    hog = torch.cuda.Stream(dev)
                    hog.wait_stream(torch.cuda.current_stream(dev))
                    a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
                    with torch.cuda.stream(hog):
                        for _ in range(8 + 8 * rank):
                            a = (a @ a).clamp_(-1, 1)
                pipe.begin(step)
                for b in reversed(range(len(pipe.buckets))):
                    pipe.submit(b, [views[i] for i in pipe.buckets[b].params])
                pipe.end()
                res = pipe.finish()
                if busy:
                    torch.cuda.current_stream(dev).wait_stream(hog)
            else:
                res = pipe.step(flat, step)
            reduced = [pipe.bucket_payload(b).cpu().numpy() for b in range(len(pipe.buckets))]
            if algo.startswith("zero"):
                pipe.gather_state()  # masters/velocities are sharded (ZeRO-1)
                torch.cuda.synchronize(dev)
            if rank == 0:
                parts = [split(w, specs) for w in wires]
                exact = world == 2 or algo in ("ordered", "ordered_hier", "zero", "zero_unfused")
                out = rp.compose_step_fp16(parts, [s.name for s in specs], [s.numel for s in specs],
                                           order, groups, rp.LarsHyper(0.001, 0.0, 5e-4, 0.9), 0.1,
                                           oloss, theta, 0,
                                           reduced_override=None if exact else reduced)
                if not exact and not algo.startswith("zero"):
                    # reduced buckets within the reference's fp16 bound
                    tree = rp.compose_step_fp16  # noqa: F841 (documentation)
                    for b, bk in enumerate(pipe.buckets):
                        xs = np.stack([np.concatenate([parts[r][i] for i in bk.params])
                                       for r in range(world)])
                        bound = 2.0 ** -9 * np.abs(rp.widen(xs)).sum(0)
                        fin = np.isfinite(bound)
                        err = np.abs(rp.widen(reduced[b]) - rp.fold_ascending(list(rp.widen(xs))))
                        if not np.all(err[fin] <= bound[fin] + 2.0 ** -24):
                            ok = False
                            notes.append(f"step {step} bucket {b}: fp16 sum outside 2^-9 bound")
                if res.applied != out.applied:
                    ok = False
                    notes.append(f"step {step}: applied {res.applied} vs {out.applied}")
                got = pipe.registration_view(pipe.master).cpu().numpy()
                want = np.concatenate([g.master for g in groups])
                if not np.array_equal(got.view(np.uint32), want.view(np.uint32)):
                    ok = False
                    notes.append(f"step {step}: master differs in "
                                 f"{int((got.view(np.uint32) != want.view(np.uint32)).sum())} elems")
                gotv = pipe.registration_view(pipe.velocity).cpu().numpy()
                wantv = np.concatenate([g.velocity for g in groups])
                if not np.array_equal(gotv.view(np.uint32), wantv.view(np.uint32)):
                    ok = False
                    notes.append(f"step {step}: velocity differs")
                goth = pipe.registration_view(pipe.working).cpu().numpy()
                wanth = np.concatenate([g.working for g in groups])
                if not np.array_equal(goth, wanth):
                    ok = False
                    notes.append(f"step {step}: working copy differs")
                if out.applied and not np.array_equal(pipe.seg_scales(), out.scales):
                    ok = False
                    notes.append(f"step {step}: trust scales differ")
            flag = torch.tensor([0 if res.applied else 1], device=dev)
            dist.all_reduce(flag)
            if step == 2 and int(flag) != world:
                ok = False
                notes.append("injected Inf did not skip on every rank")
        results[algo_name] = {"ok": ok, "notes": notes[:5], "k": k}
    if rank == 0:
        print(json.dumps({"world": world, "model": model, "theta": theta, "results": results}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
