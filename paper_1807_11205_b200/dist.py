"""Multi-GPU gradient all-reduce over NCCL / NVLink, one process per GPU.

The reference executes p workers in one process (collectives.py:286-340) or
over loopback TCP (tcp.py); on a B200 box each worker is a process that owns
one GPU and the bucket all-reduce runs over NVLink 5 / NVSwitch:

  "ring"          flat 1xp: ncclAllReduce(sum) on the world communicator
                  (ring_allreduce / allreduce_f16 "ring", collectives.py:291-302,
                  322-340; NCCL picks ring or NVLS itself);
  "hierarchical"  the paper's three phases (hierarchical_schedule,
                  collectives.py:183-235) on sub-communicators of
                  Topology(p, k): ncclReduce to the group master (lowest rank,
                  collectives.py:76-77) -> ncclAllReduce among the masters ->
                  ncclBroadcast inside the group;
  "ordered"       the reference's own summation order, bit-exact: a single
                  kernel per rank folds its slice out of every peer's
                  symmetric-memory buffer over NVLink in pairwise-tree order
                  and gathers the other slices back (OrderedWire);
  "sharded"       bandwidth-optimal hierarchy for NVSwitch: intra-group
                  reduce-scatter -> all-reduce among same-offset ranks of all
                  groups -> intra-group all-gather (moves 2(p-1)/p S per GPU,
                  the flat ring's volume, instead of the master's 3S);
  "ordered_hier"  the same two-level structure in ONE own kernel
                  (gs_hier_allreduce_f16), bit-exact: the reference's rank
                  tree factors over power-of-two groups.

Sums never use ncclAvg: the reference sums and then divides by float32(p)
(collectives.py:268-269), which the LARS pass-1 kernel does on the fly.
NCCL's summation order differs from the reference's pairwise tree, so these
paths match the oracle within the reference's own fp16 tolerance (2^-9
relative, test_collectives.py:237-250); the skip decision is order-free for
Inf/NaN inputs.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist

from .collectives import Topology, choose_algorithm

__all__ = ["Communicator", "init_from_env", "ALGORITHMS"]

ALGORITHMS = ("ring", "hierarchical", "sharded", "ordered", "ordered_hier")


def init_from_env(backend: str | None = None) -> tuple[int, int, int]:
    """Initialise torch.distributed from torchrun's env (127.0.0.1 rendezvous).
    Returns (rank, world_size, local_rank)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29512")
        be = backend or ("nccl" if torch.cuda.is_available() else "gloo")
        if be == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(be, rank=rank, world_size=world,
                                    device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(be, rank=rank, world_size=world)
    return rank, world, local


class Communicator:
    """World + Topology(p, k) sub-groups for one rank.

    Every rank must construct it (group creation is collective).  Groups:
      intra[g]  = ranks of group g            (contiguous, collectives.py:70-74)
      masters   = lowest rank of every group  (collectives.py:76-77)
      cross[j]  = member j of every group     (the sharded middle phase)
    """

    def __init__(self, topo: Topology, rank: int | None = None):
        self.topo = topo
        self.rank = dist.get_rank() if rank is None else rank
        self.world_size = topo.p
        if dist.is_initialized() and dist.get_world_size() != topo.p:
            raise ValueError(f"topology is for p={topo.p}, world size is {dist.get_world_size()}")
        self.world = dist.group.WORLD
        p, k, G = topo.p, topo.k, topo.group_count
        self.group = topo.group_of(self.rank)
        self.offset = self.rank - self.group * k
        self.master = self.group * k
        self.intra = None
        self.masters = None
        self.cross = None
        if p > 1 and k > 1:
            for g in range(G):
                pg = dist.new_group(list(topo.members(g)))
                if g == self.group:
                    self.intra = pg
        if p > 1 and G > 1:
            pg = dist.new_group(topo.masters())
            if self.rank == self.master:
                self.masters = pg
            for j in range(k):
                pg = dist.new_group([g * k + j for g in range(G)])
                if j == self.offset:
                    self.cross = pg

    # -- the three algorithms; all in place, sum, on the caller's current stream
    # (binary16 bit patterns travel as float16: NCCL has no uint16 type)
    @staticmethod
    def _wire(t: torch.Tensor) -> torch.Tensor:
        return t.view(torch.float16) if t.dtype == torch.uint16 else t

    def allreduce_ring(self, t: torch.Tensor, async_op: bool = False):
        return dist.all_reduce(self._wire(t), op=dist.ReduceOp.SUM, group=self.world,
                               async_op=async_op)

    def allreduce_hierarchical(self, t: torch.Tensor):
        """Literal three-phase: reduce to master, masters all-reduce, broadcast."""
        t = self._wire(t)
        topo = self.topo
        if topo.k > 1:
            dist.reduce(t, dst=self.master, op=dist.ReduceOp.SUM, group=self.intra)
        if topo.group_count > 1 and self.rank == self.master:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.masters)
        if topo.k > 1:
            dist.broadcast(t, src=self.master, group=self.intra)

    def allreduce_sharded(self, t: torch.Tensor):
        """Reduce-scatter inside the group, all-reduce the shard across groups,
        all-gather inside the group.  t.numel() must be a multiple of k."""
        t = self._wire(t)
        topo = self.topo
        k = topo.k
        if k == 1:
            if topo.group_count > 1:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.cross)
            return
        n = t.numel()
        if n % k:
            raise ValueError(f"sharded all-reduce needs a multiple of k={k} elements, got {n}")
        shard = t.view(k, n // k)[self.offset]
        dist.reduce_scatter_tensor(shard, t, op=dist.ReduceOp.SUM, group=self.intra)
        if topo.group_count > 1:
            dist.all_reduce(shard, op=dist.ReduceOp.SUM, group=self.cross)
        dist.all_gather_into_tensor(t, shard, group=self.intra)

    def allreduce(self, t: torch.Tensor, algorithm: str) -> None:
        if self.topo.p == 1:
            return
        if algorithm == "ring":
            self.allreduce_ring(t)
        elif algorithm == "hierarchical":
            self.allreduce_hierarchical(t)
        elif algorithm == "sharded":
            self.allreduce_sharded(t)
        else:
            raise ValueError(f"unknown algorithm {algorithm!r}")

    def pick(self, nbytes: int, eta_bytes: int, hier_variant: str = "hierarchical",
             flat_variant: str = "ring") -> str:
        """Hybrid rule (collectives.py:238-244) mapped onto the variants."""
        return hier_variant if choose_algorithm(nbytes, eta_bytes) == "hierarchical" else flat_variant

    # -- peer-memory plumbing of the own-kernel paths (emulation.LocalComm
    # provides the same three on one device)
    emulated = False
    #: CTAs per rank of the peer kernels (None: the pipeline's default)
    peer_ctas = None
    #: bound of every device-side peer wait (gs_rank_ctx.timeout_ns)
    timeout_s = 120.0

    def make_arena(self, regions: dict, device, sig_words: int) -> "SymmetricArena":
        return SymmetricArena(self, regions, device, sig_words)

    def make_ordered_wire(self, total: int, device, push: bool = False,
                          itemsize: int = 2) -> "OrderedWire":
        return OrderedWire(self, total, device, push=push, itemsize=itemsize)


class OrderedWire:
    """Double-buffered symmetric-memory wire for the bit-exact ordered
    all-reduce (gs_ordered_allreduce_f16): one allocation per rank,
    [wire A | wire B | signal area | control], exchanged once through torch's
    symmetric-memory rendezvous so every rank holds every peer's NVLink-mapped
    base address.  Both halves have the pipeline's wire layout, so a bucket is
    the same element range in every rank's buffer.  `push` selects the push
    form of the kernel (fold + remote stores, one exit barrier) over the pull
    form (fold, barrier, gather by remote loads); same result bit for bit."""

    def __init__(self, comm: "Communicator", total: int, device, nblocks: int | None = None,
                 push: bool = False, itemsize: int = 2):
        import torch.distributed._symmetric_memory as symm

        self.p = comm.topo.p
        self.rank = comm.rank
        sms = torch.cuda.get_device_properties(device).multi_processor_count
        # all CTAs must be co-resident (they wait on their peers' CTAs): two
        # 512-thread CTAs per SM fit next to anything else that is running
        self.nblocks = nblocks or comm.peer_ctas or 2 * sms
        self.total = (total + 255) // 256 * 256
        self.itemsize = itemsize
        self.buf = symm.empty(self.nbytes_for(self.total, itemsize, self.nblocks, self.p),
                              dtype=torch.uint8, device=device)
        self.buf.zero_()
        torch.cuda.synchronize(device)
        self.hdl = symm.rendezvous(self.buf, dist.group.WORLD.group_name)
        bases = [int(x) for x in self.hdl.buffer_ptrs]
        self._setup(bases, device, push, comm.timeout_s)
        dist.barrier()

    #: inbox slot capacity (binary16 elements) for the small-bucket kernels
    SMALL_CAP_ELEMS = 1 << 18
    #: buckets up to this many elements take the one-shot kernel
    #: (gs_oneshot_allreduce_f16: one barrier, (p-1) x S bytes out).
    #: Measured at p = 4 (profiles/r02/y_n4, aa_n4): 13.1-14.3 µs up to 8 KB
    #: vs 19-20 (pull) / 15.3-16.1 (push) and NCCL's 14.6-15.0; from 16 KB
    #: on the (p-1) x S bytes make it tie or lose to the push form.
    ONESHOT_MAX_ELEMS = 4096
    #: buckets up to this many elements take the LL kernel when whole
    #: 8-element vectors (gs_ll_allreduce_f16: no fence, no barrier).
    #: Measured at p = 4 (profiles/r02/ii_n4, fp16 bytes): 9.0-12.7 µs up to
    #: 128 KB, 15.5 µs at 256 KB and 20.9 µs at 512 KB vs NCCL ring 15.2-17.4
    #: and the push form 16.4-25.2; at 1 MB its doubled bytes lose (32.5 vs
    #: 24.7 push).  512 KB rather than 256 KB: a θ = 256 KiB bucket closes just
    #: above θ and would otherwise miss the LL form
    LL_MAX_ELEMS = 1 << 18

    @staticmethod
    def oneshot_cap(total: int, itemsize: int) -> int:
        """Elements per inbox slot (0: no small-bucket forms, e.g. the fp32
        wire or SMALL_CAP_ELEMS = 0)."""
        if itemsize != 2:
            return 0
        return (min(total, OrderedWire.SMALL_CAP_ELEMS) + 255) // 256 * 256

    @staticmethod
    def sig_bytes(nblocks: int, p: int) -> int:
        return (4 * 3 * nblocks * p + 512 + 255) // 256 * 256

    @staticmethod
    def nbytes_for(total: int, itemsize: int, nblocks: int, p: int) -> int:
        """[wire A | wire B | signal area (3 barrier phases) | inbox (2 parities
        x p slots of oneshot_cap elements) | status]"""
        cap = OrderedWire.oneshot_cap(total, itemsize)
        # 4 bytes per element and slot: the LL form's {payload, epoch} words
        return 2 * total * itemsize + OrderedWire.sig_bytes(nblocks, p) + 2 * p * cap * 4 + 128

    def _setup(self, bases, device, push: bool, timeout_s: float) -> None:
        """Tables and this rank's context from every rank's base address
        (shared with emulation.LocalOrderedWire)."""
        import numpy as np

        from . import _device as dev
        from ._peer import rank_ctx

        z, t = self.itemsize, self.total
        dt = torch.uint16 if z == 2 else torch.float32
        self.halves = (self.buf[: z * t].view(dt), self.buf[z * t: 2 * z * t].view(dt))
        self.bufs_dev = [dev.upload(np.array([b + h * z * t for b in bases], dtype=np.uint64),
                                    device) for h in range(2)]
        self.sig_dev = dev.upload(np.array([b + 2 * z * t for b in bases], dtype=np.uint64),
                                  device)
        # one-shot inboxes (small buckets): after the signal area
        self.cap = self.oneshot_cap(t, z)
        ib = 2 * z * t + self.sig_bytes(self.nblocks, self.p)
        self.inbox_dev = dev.upload(np.array([b + ib for b in bases], dtype=np.uint64), device) \
            if self.cap else None
        self._oneshot_calls = 0
        # device-resident epoch base: every call of a step uses base + slot,
        # and advance() bumps the base once per step on the stream
        self.epoch_base = torch.zeros(1, dtype=torch.int32, device=device)
        # status word (a timed-out peer wait is reported here) at the tail
        self.status = self.buf[-128:].view(torch.int32)
        self.ctx = rank_ctx(self.rank, timeout_s=timeout_s, status=dev.ptr(self.status),
                            epoch_base=dev.ptr(self.epoch_base))
        self.push = bool(push)
        self.device = device

    #: elements per CTA below which a call uses fewer CTAs: a small bucket
    #: then pays the barriers of a few CTAs instead of the whole co-resident
    #: grid (every rank derives the same grid from n, so the per-CTA signal
    #: slots still pair up)
    MIN_ELEMS_PER_CTA = 16384

    #: buckets up to this many bytes take the push form at p >= 4 even on a
    #: pull wire: p = 4 sweeps (r2ii, r2tt, r2ac) put it 2-4 µs ahead from
    #: 128 KB to 2 MB, even from 4 MB on; at p = 2 neither form leads there
    #: (r2t).  fp16 wire only (measured there).  Same fold order,
    #: bit-identical; 0 disables
    PUSH_MAX_BYTES = 2 << 20

    def push_for(self, n: int) -> bool:
        return self.push or (self.p >= 4 and self.itemsize == 2
                             and n * 2 <= OrderedWire.PUSH_MAX_BYTES)

    def grid_for(self, n: int) -> int:
        return max(1, min(self.nblocks, -(-int(n) // self.MIN_ELEMS_PER_CTA)))

    def small_form(self, offset: int, n: int) -> str:
        """The size rule: "ll", "oneshot" or "none" (the pull / push kernel)."""
        if not self.cap or not 0 < n <= self.cap:
            return "none"
        if n <= OrderedWire.LL_MAX_ELEMS and n % 8 == 0 and offset % 8 == 0:
            return "ll"
        return "oneshot" if n <= OrderedWire.ONESHOT_MAX_ELEMS else "none"

    def allreduce_op(self, half: int, offset: int, n: int, stream_h: int, slot: int = 0,
                     small: str | None = None):
        """The bucket all-reduce as a peer op; `slot` (0-based within the
        step, < per_step) makes the epoch unique among the step's calls.
        small: "oneshot" (one barrier), "ll" (no barrier; whole 8-element
        vectors) or "none" (pull / push kernel); None = small_form's size
        rule.  Bit-identical either way."""
        from . import _device as dev
        from ._peer import PeerOp

        if small is None:
            small = self.small_form(offset, n)
        if small == "ll" and not (n % 8 == 0 and offset % 8 == 0):
            small = "oneshot"
        if small != "none" and self.cap and 0 < n <= self.cap:
            parity = self._oneshot_calls & 1
            self._oneshot_calls += 1
            if small == "ll":
                grid = max(1, min(self.nblocks, -(-n // (8 * 256))))
                return PeerOp("gs_ll_allreduce_f16", self.ctx,
                              (self.p, dev.ptr(self.bufs_dev[half]), dev.ptr(self.inbox_dev),
                               offset, n, self.cap, slot + 1, grid, parity, stream_h),
                              device=self.device)
            return PeerOp("gs_oneshot_allreduce_f16", self.ctx,
                          (self.p, dev.ptr(self.bufs_dev[half]), dev.ptr(self.inbox_dev),
                           dev.ptr(self.sig_dev), offset, n, self.cap, slot + 1, self.grid_for(n),
                           parity, stream_h), device=self.device)
        return PeerOp("gs_ordered_allreduce_f16" if self.itemsize == 2 else
                      "gs_ordered_allreduce_f32", self.ctx,
                      (self.p, dev.ptr(self.bufs_dev[half]), dev.ptr(self.sig_dev), offset, n,
                       slot + 1, self.grid_for(n), 1 if self.push_for(n) else 0, stream_h),
                      device=self.device)

    def hier_op(self, half: int, offset: int, n: int, k: int, stream_h: int, slot: int = 0):
        """The bucket all-reduce over Topology(p, k)'s two levels
        (gs_hier_allreduce_f16; bit-identical to allreduce_op).  Buckets the
        one-shot kernel takes (n <= ONESHOT_MAX_ELEMS) use it here too: the
        reference's rank tree factors over the groups, so the flat one-shot
        fold gives the hierarchy's bits with one barrier instead of three."""
        from . import _device as dev
        from ._peer import PeerOp

        if self.small_form(offset, n) != "none":
            return self.allreduce_op(half, offset, n, stream_h, slot)

        return PeerOp("gs_hier_allreduce_f16", self.ctx,
                      (self.p, k, dev.ptr(self.bufs_dev[half]), dev.ptr(self.sig_dev), offset, n,
                       slot + 1, self.grid_for(n), 1 if self.push else 0, stream_h),
                      device=self.device)

    def allreduce(self, half: int, offset: int, n: int, stream_h: int, slot: int = 0,
                  small: str | None = None) -> None:
        from ._peer import launch
        launch([self.allreduce_op(half, offset, n, stream_h, slot, small)])

    def advance(self, per_step: int, stream_h: int) -> None:
        from . import _device as dev
        from . import _native

        _native.call("gs_counter_add", dev.ptr(self.epoch_base), per_step, stream_h)

    def status_word(self) -> int:
        return int(self.status[0].item())


class SymmetricArena:
    """One symmetric-memory allocation per rank carved into named regions
    (byte sizes given up front), plus device tables of every peer's address
    of each region — the building block of the sharded (ZeRO-1) update, in
    which the wire, the binary16 working weights, the masters, the
    velocities, the LARS chunk partials and the control block (step flags)
    are all reachable by every peer over NVLink."""

    ALIGN = 512

    def __init__(self, comm: "Communicator", regions: dict, device, sig_words: int):
        import torch.distributed._symmetric_memory as symm

        self.p, self.rank = comm.topo.p, comm.rank
        self.layout(regions, sig_words)
        self.buf = symm.empty(self.nbytes, dtype=torch.uint8, device=device)
        self.buf.zero_()
        torch.cuda.synchronize(device)
        self.hdl = symm.rendezvous(self.buf, dist.group.WORLD.group_name)
        self.bases = [int(x) for x in self.hdl.buffer_ptrs]
        self.tables(device)
        dist.barrier()

    def layout(self, regions: dict, sig_words: int) -> None:
        self.offsets, off = {}, 0
        for name, nbytes in list(regions.items()) + [("sig", 4 * sig_words)]:
            self.offsets[name] = off
            off += (int(nbytes) + self.ALIGN - 1) // self.ALIGN * self.ALIGN
        self.sizes = dict(regions, sig=4 * sig_words)
        self.nbytes = off

    def tables(self, device) -> None:
        import numpy as np

        from . import _device as dev

        self._tabs = {}
        for name in self.offsets:
            self._tabs[name] = dev.upload(
                np.array([b + self.offsets[name] for b in self.bases], dtype=np.uint64), device)

    def view(self, name: str, dtype: torch.dtype) -> torch.Tensor:
        o, n = self.offsets[name], self.sizes[name]
        return self.buf[o:o + n].view(dtype)

    def peers(self, name: str) -> torch.Tensor:
        """Device uint64[p]: every rank's address of region `name`."""
        return self._tabs[name]
