"""p data-parallel ranks emulated on ONE device, running the real peer kernels.

The reference executes its p workers inside one process (the in-memory
executor, collectives.py:286-340).  This module does the same for the
B200 pipeline, but through the very kernels a multi-GPU job runs:
each emulated rank owns a full arena (wire halves, masters, velocities,
partials, control block, signal area) in this device's memory, every rank's
peer tables point at the other ranks' arenas, and each peer-synchronised
launch (the ordered all-reduce, reduce-scatter / all-gather, gs_rs_pass1,
gs_zero_update, gs_peer_fence) is issued ONCE for all p ranks over a
gs_rank_ctx table (CTA b serves rank b / nb), so every rank's CTAs are
co-resident and the cross-rank waits resolve inside one kernel — on one
stream, deterministically, and under ncu's kernel serialisation too.

The ranks' step programs are Python generators (GradientPipeline._*_gen):
everything between two peer launches is launched per rank, and the peer
launch of all ranks is batched, in lockstep.  Nothing here is a CPU model:
the arithmetic and the exchange are the product kernels, only the NVLink
transport is replaced by local memory.  NCCL algorithms (ring /
hierarchical / sharded via torch.distributed) cannot be emulated.

Use::

    world = LocalWorld(Topology(8, 1), device)
    pipes = [GradientPipeline(specs, cfg, comm=c, sharded_update=True, ...)
             for c in world.comms]
    results = world.step(pipes, [grads_of_rank(r) for r in range(8)], step)
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as dev
from ._peer import launch
from .collectives import Topology, choose_algorithm

__all__ = ["LocalWorld", "LocalComm"]


class LocalComm:
    """The Communicator of emulated rank `rank` (same attributes the pipeline
    reads from dist.Communicator)."""

    emulated = True

    def __init__(self, world: "LocalWorld", rank: int):
        self.world = world
        self.topo = world.topo
        self.rank = rank
        self.world_size = world.topo.p
        self.peer_ctas = world.peer_ctas
        self.timeout_s = world.timeout_s
        k = world.topo.k
        self.group = world.topo.group_of(rank)
        self.offset = rank - self.group * k
        self.master = self.group * k

    def pick(self, nbytes: int, eta_bytes: int, hier_variant: str = "hierarchical",
             flat_variant: str = "ring") -> str:
        return hier_variant if choose_algorithm(nbytes, eta_bytes) == "hierarchical" \
            else flat_variant

    def make_arena(self, regions: dict, device, sig_words: int) -> "LocalArena":
        return self.world._arena(self.rank, regions, device, sig_words)

    def make_ordered_wire(self, total: int, device, push: bool = False,
                          itemsize: int = 2) -> "LocalOrderedWire":
        return self.world._ordered_wire(self.rank, total, device, push, itemsize)

    def _no_nccl(self, *a, **k):
        raise NotImplementedError("NCCL collectives cannot be emulated on one device; use the "
                                  "own-kernel paths (sharded_update, flat_variant='ordered', "
                                  "hier_variant='ordered_hier')")

    allreduce = allreduce_ring = allreduce_hierarchical = allreduce_sharded = _no_nccl


class LocalArena:
    """SymmetricArena of one emulated rank: its own allocation, and peer
    tables (shared by all ranks, so a batched launch passes one table)."""

    from .dist import SymmetricArena as _SA
    ALIGN = _SA.ALIGN
    layout = _SA.layout
    view = _SA.view
    peers = _SA.peers

    def __init__(self, p, rank, buf, offsets, sizes, bases, tabs):
        self.p, self.rank, self.buf = p, rank, buf
        self.offsets, self.sizes, self.bases, self._tabs = offsets, sizes, bases, tabs


class LocalOrderedWire:
    """OrderedWire of one emulated rank (see dist.OrderedWire)."""

    from .dist import OrderedWire as _OW
    MIN_ELEMS_PER_CTA = _OW.MIN_ELEMS_PER_CTA
    small_form = _OW.small_form
    nbytes_for = _OW.nbytes_for
    oneshot_cap = staticmethod(_OW.oneshot_cap)
    sig_bytes = staticmethod(_OW.sig_bytes)
    _setup = _OW._setup
    grid_for = _OW.grid_for
    push_for = _OW.push_for
    allreduce_op = _OW.allreduce_op
    hier_op = _OW.hier_op
    allreduce = _OW.allreduce
    advance = _OW.advance
    status_word = _OW.status_word

    def __init__(self, p, rank, total, itemsize, buf, bases, nblocks, device, push, timeout_s):
        self.p, self.rank, self.total, self.buf, self.nblocks = p, rank, total, buf, nblocks
        self.itemsize = itemsize
        self._setup(bases, device, push, timeout_s)


class LocalWorld:
    """p ranks of one job on one device (see the module docstring).

    peer_ctas: CTAs per rank of every peer kernel (the whole launch, p x
    peer_ctas CTAs, must be co-resident; the kernels clamp it further).
    timeout_s: bound of every device-side peer wait; a timeout is reported by
    GradientPipeline.finish (PeerTimeoutError), the GPU never hangs."""

    def __init__(self, topo: Topology, device=None, peer_ctas: int = 16, timeout_s: float = 30.0):
        self.topo = topo
        self.device = device or dev.require_cuda()
        self.peer_ctas = int(peer_ctas)
        self.timeout_s = float(timeout_s)
        self.comms = [LocalComm(self, r) for r in range(topo.p)]
        self._arenas = None
        self._wires = None

    # -- allocation: the first rank to ask allocates every rank's copy ------
    def _arena(self, rank, regions, device, sig_words) -> LocalArena:
        p = self.topo.p
        if self._arenas is None or self._arenas[0] != (tuple(regions.items()), sig_words) \
                or self._arenas[1][rank] is None:
            proto = LocalArena(p, 0, None, None, None, None, None)
            proto.layout(regions, sig_words)
            bufs = [torch.zeros(proto.nbytes, dtype=torch.uint8, device=device) for _ in range(p)]
            bases = [b.data_ptr() for b in bufs]
            tabs = {name: dev.upload(np.array([b + off for b in bases], dtype=np.uint64), device)
                    for name, off in proto.offsets.items()}
            self._arenas = ((tuple(regions.items()), sig_words),
                            [LocalArena(p, r, bufs[r], proto.offsets, proto.sizes, bases, tabs)
                             for r in range(p)])
        arena = self._arenas[1][rank]
        self._arenas[1][rank] = None  # each rank takes its arena once
        return arena

    def _ordered_wire(self, rank, total, device, push, itemsize=2) -> LocalOrderedWire:
        p = self.topo.p
        total = (total + 255) // 256 * 256
        key = (total, itemsize)
        if self._wires is None or self._wires[0] != key or self._wires[1][rank] is None:
            nb = self.peer_ctas
            nbytes = LocalOrderedWire.nbytes_for(total, itemsize, nb, p)
            bufs = [torch.zeros(nbytes, dtype=torch.uint8, device=device) for _ in range(p)]
            bases = [b.data_ptr() for b in bufs]
            wires = [LocalOrderedWire(p, r, total, itemsize, bufs[r], bases, nb, device, push,
                                      self.timeout_s) for r in range(p)]
            # one bufs/sig table for every rank: the batched launch passes
            # rank 0's, so all must be the same tensors
            for w in wires[1:]:
                w.bufs_dev, w.sig_dev = wires[0].bufs_dev, wires[0].sig_dev
                w.inbox_dev = wires[0].inbox_dev
            self._wires = (key, wires)
        w = self._wires[1][rank]
        self._wires[1][rank] = None
        return w

    # -- lockstep driver ----------------------------------------------------
    @staticmethod
    def drive(gens) -> int:
        """Run one generator per rank in lockstep: each rank's local launches
        up to its next peer op, then the ops of all ranks as one launch.
        Returns the number of batched peer launches."""
        n = 0
        gens = list(gens)
        while True:
            ops = [next(g, None) for g in gens]
            if all(op is None for op in ops):
                return n
            if any(op is None for op in ops):
                raise RuntimeError("emulated ranks diverged: one finished its step while "
                                   "another still has peer launches")
            launch(ops)
            n += 1

    def enqueue(self, pipes, grads, step: int, executor: bool = True) -> None:
        """One step of every rank (grads[r] = rank r's gradients), launched on
        the current stream; finish() each pipe afterwards.  The fused sharded
        step goes through the native executor (gs_step_zero over all p ranks
        in one call) unless executor=False, which drives the per-kernel
        generators in lockstep instead (same kernels, same order)."""
        if executor and all(pp.sharded and pp.fused_collective for pp in pipes):
            import numpy as np_
            from . import _native
            from ._peer import batched_table
            tabs = [pp._open_step(g, step) for pp, g in zip(pipes, grads)]
            recs = np_.concatenate([pp._zero_record(t) for pp, t in zip(pipes, tabs)])
            ctx = batched_table([pp._ctx for pp in pipes], self.device)
            sh = int(torch.cuda.current_stream(self.device).cuda_stream)
            max_own = max(pp._n_own for pp in pipes)
            _native.call("gs_step_zero", recs.ctypes.data, len(pipes), dev.ptr(ctx),
                         *pipes[0]._zero_args(max_own, sh))
            for pp in pipes:
                pp._last_wire = pp.red
                pp.plan.end_step()
            return
        self.drive(pipe._enqueue_gen(g, step) for pipe, g in zip(pipes, grads))

    def step(self, pipes, grads, step: int, executor: bool = True):
        self.enqueue(pipes, grads, step, executor)
        return [pipe.finish() for pipe in pipes]

    def gather_state(self, pipes) -> None:
        """Sharded masters / velocities made whole on every rank."""
        self.drive(pipe._gather_gen() for pipe in pipes)
        for pipe in pipes:
            pipe._gathered = True

    # the incremental API, lockstep over ranks
    def begin(self, pipes, step: int) -> None:
        self.drive(pipe._begin_gen(step) for pipe in pipes)

    def submit(self, pipes, b: int, grads) -> None:
        self.drive(pipe._submit_gen(b, g) for pipe, g in zip(pipes, grads))

    def end(self, pipes) -> None:
        self.drive(pipe._end_gen() for pipe in pipes)
