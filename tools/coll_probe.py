"""Time the symmetric-memory collectives in isolation (torchrun, N GPUs).

ordered all-reduce of S bytes, reduce-scatter with equal slices, all-gather of
the slices — each 10x back to back after a barrier, device time by events,
max over ranks.
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1807_11205_b200 as gs  # noqa: E402
from paper_1807_11205_b200 import _device as dev, _native  # noqa: E402
from paper_1807_11205_b200.dist import Communicator, SymmetricArena, init_from_env  # noqa: E402


def main():
    rank, world, local = init_from_env("nccl")
    d = torch.device("cuda", local)
    comm = Communicator(gs.Topology(world, 1))
    n = 1 << 27  # capacity (elements)
    sms = torch.cuda.get_device_properties(d).multi_processor_count
    nb = int(os.environ.get("NB", str(2 * sms)))
    a = SymmetricArena(comm, {"w": 2 * n, "x": 2 * n}, d, sig_words=2 * nb * world)
    ebase = torch.zeros(1, dtype=torch.int32, device=d)
    s0 = torch.cuda.current_stream(d)
    sh = int(s0.cuda_stream)
    sig = dev.ptr(a.peers("sig"))
    slot = [0]

    def rs():
        slot[0] += 1
        _native.call("gs_ordered_reduce_scatter_f16", dev.ptr(a.peers("w")), sig, rank, world,
                     dev.ptr(bounds_e), slot[0], dev.ptr(ebase), nb, None, sh)

    def ag():
        slot[0] += 1
        _native.call("gs_ordered_allgather", dev.ptr(a.peers("x")), sig, rank, world,
                     dev.ptr(bounds_b), slot[0], dev.ptr(ebase), nb, sh)

    def ar():
        slot[0] += 1
        _native.call("gs_ordered_allreduce_f16", dev.ptr(a.peers("w")), sig, rank, world, 0, n,
                     slot[0], dev.ptr(ebase), nb, None, sh)

    sizes = [int(x) for x in os.environ.get("SIZES", "512,65536,1048576,8388608,25557248,67108864").split(",")]
    for m in sizes:
      E = [r * m // world // 8 * 8 for r in range(world)] + [m]
      bounds_e = dev.upload(np.array(E, dtype=np.int64), d)
      bounds_b = dev.upload(np.array([2 * e for e in E], dtype=np.int64), d)
      n = m
      out = {}
      for name, fn in (("allreduce", ar), ("reduce_scatter", rs), ("allgather", ag),
                       ("nccl_allreduce", lambda: dist.all_reduce(a.view("x", torch.float16)[:m]))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(d)
        dist.barrier()
        torch.cuda.synchronize(d)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s0)
        for _ in range(10):
            fn()
        e1.record(s0)
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 10 * 1e3], dtype=torch.float64, device=d)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[name] = round(float(t), 1)
      if rank == 0:
        print({"world": world, "bytes": 2 * m, "nblocks": nb, "us": out,
               "busbw_gbs": {k: round(2 * m / (v * 1e-6) * 2 * (world - 1) / world / 1e9, 1)
                             for k, v in out.items() if k in ("allreduce", "nccl_allreduce")}},
              flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
