"""The fused per-step gradient pipeline of one data-parallel rank.

This composes the reference's step body (experiment.py:368-413) on the fp16
wire that the north star asks for, device-resident:

  1. pack       per-parameter fp16 gradients -> theta-buckets of the wire
                buffer, in enqueue (backward) order; bucket boundaries are
                exactly FusionBuffer's (fusion.py:58-94)       gs_batched_copy
  2. all-reduce every bucket, sum: own bit-exact NVLink kernels (ordered /
                sharded) or NCCL (flat ring / hierarchical / sharded), bucket
                i in flight while bucket i+1 is packed and bucket i-1 runs
                pass 1
  3. pass 1     widen, /float32(p) (mean, collectives.py:268-269), finite test
                on the scaled mean (LossScale.update, experiment.py:403),
                /float32(step_scale) (unscale, experiment.py:407), finite
                gate (lars.py:161-163), fp64 partial norms      gs_lars_pass1
  4. trust      per-group trust ratio and fp32 scale            gs_lars_trust
  5. pass 2     momentum / master / working-copy update, skipped on the
                device when either flag is set                  gs_lars_pass2

Memory layout (HBM): one uint16 wire buffer holding every bucket back to
back (each bucket starts on a 512-byte boundary; the zero slack after a
bucket's payload is never part of any tensor, so the per-bucket unpack_map is
the reference's), and fp32 master / fp32 velocity / uint16 working arenas
laid out at the SAME element offsets as the wire, so pass 1/2 stream four
arrays with one index.  ParamGroup objects are views into the arenas.

Every step is a Python generator (``_enqueue_gen`` and friends) that launches
the rank-local kernels itself and YIELDS each peer-synchronised launch as a
``_peer.PeerOp``: on a multi-GPU box ``enqueue`` launches each op for this
rank alone; ``emulation.LocalWorld`` runs the p ranks' generators in
lockstep on one device and launches each op once for all of them.
"""

from __future__ import annotations

import os

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dev
from . import _native
from . import _trace
from ._peer import PeerOp, PeerTimeoutError, decode_status, launch, rank_ctx
from ._plan import LarsPlan, SegmentSpec, build_chunks, step_params
from .fusion import copy_table, plan_buckets
from .halfprec import LossScale
from .lars import LarsConfig, ParamGroup, segment_flags

__all__ = ["ParamSpec", "Bucket", "GradientPipeline", "StepResult", "BUCKET_ALIGN",
           "plan_layout", "shard_buckets"]

#: wire-buffer granularity (elements): bucket starts are 512-byte aligned and
#: padded lengths are multiples of 256 so any k <= 8 shards 16-byte aligned
BUCKET_ALIGN = 256

_MASK = _native.FLAG_SCALED_NONFINITE | _native.FLAG_GRAD_NONFINITE


@dataclass(frozen=True)
class ParamSpec:
    name: str
    shape: tuple
    kind: str

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape, dtype=np.int64)) if len(self.shape) else 1


@dataclass
class Bucket:
    start: int                 # wire offset (elements)
    length: int                # payload elements (the reference batch size)
    padded: int                # allocated elements (multiple of BUCKET_ALIGN)
    params: list               # registration indices, wire order
    unpack_map: tuple          # ((name, offset, length), ...) as fusion.py:84-88
    chunk0: int = 0
    nchunk: int = 0
    algorithm: str = "ring"
    itemsize: int = 2          # wire element: binary16 (2) or fp32 (4)

    @property
    def nbytes(self) -> int:
        return self.itemsize * self.length


@dataclass
class StepResult:
    applied: bool
    scale: float               # the loss scale the step was unscaled with
    grad_norm: float           # experiment.py:408-411 (0.0 when not applied)
    flags: int
    algorithms: list = field(default_factory=list)


def resolve_eta(eta_bytes, topo=None, itemsize: int = 2):
    """The pipeline's hybrid threshold: an int (bytes), float("inf") (every
    bucket hierarchical, the reference's config 1) or the path of a measured
    sweep file (`tools/allreduce_sweep.py` JSONL), from which netsim seeds η
    for `topo` (netsim.eta_from_sweep)."""
    if isinstance(eta_bytes, (str, os.PathLike)):
        if topo is None:
            raise ValueError("eta_bytes from a sweep file needs a Communicator (p > 1)")
        from .netsim import eta_from_sweep
        eta_bytes = eta_from_sweep(eta_bytes, topo.p, topo.k, itemsize)
    return eta_bytes if eta_bytes == float("inf") else int(eta_bytes)


def _roundup(n: int, a: int) -> int:
    return (n + a - 1) // a * a


def plan_layout(specs, order, threshold_bytes: int, itemsize: int = 2):
    """Host-only wire layout: (wire offset per parameter, buckets, total).

    Bucket membership and per-bucket unpack maps are exactly what
    FusionBuffer(threshold) emits for tensors of `itemsize` bytes (uint16
    binary16 or float32) enqueued in `order` (fusion.py:58-94); bucket b
    starts at a BUCKET_ALIGN-aligned wire offset.
    """
    sizes = [s.numel for s in specs]
    groups_pos = plan_buckets([sizes[i] for i in order], itemsize, threshold_bytes)
    wire_off = [0] * len(specs)
    buckets, off = [], 0
    for pos_list in groups_pos:
        start, umap = off, []
        idxs = [order[q] for q in pos_list]
        for i in idxs:
            wire_off[i] = off
            umap.append((specs[i].name, off - start, sizes[i]))
            off += sizes[i]
        length = off - start
        off = start + max(BUCKET_ALIGN, _roundup(length, BUCKET_ALIGN))
        buckets.append(Bucket(start, length, off - start, idxs, tuple(umap), itemsize=itemsize))
    return wire_off, buckets, max(off, BUCKET_ALIGN)


def shard_buckets(buckets, chunk_abs_start, p: int):
    """Per-bucket ownership of the sharded update: for bucket b, rank r owns
    chunks [C_b[r], C_b[r+1]) = wire elements [E_b[r], E_b[r+1]), split at
    chunk starts so each rank gets ~length/p elements; E_b spans the padded
    bucket (the zero slack goes to the last owner).  Returns (C, E) lists."""
    Cs, Es = [], []
    for bk in buckets:
        cb0, cb1 = bk.chunk0, bk.chunk0 + bk.nchunk
        C = [cb0]
        for q in range(1, p):
            target = bk.start + q * bk.length // p
            C.append(cb0 + int(np.searchsorted(chunk_abs_start[cb0:cb1], target)))
        C.append(cb1)
        E = [bk.start] + [int(chunk_abs_start[c]) if c < cb1 else bk.start + bk.padded
                          for c in C[1:p]] + [bk.start + bk.padded]
        Cs.append(C)
        Es.append(E)
    return Cs, Es


class GradientPipeline:
    """Device-resident fp16-wire MP-LARS step for one rank.

    Args:
      specs: parameters in registration order (ParamSpec or (name, shape, kind)).
      cfg: LarsConfig.
      threshold_bytes: fusion threshold theta (fusion.py:42-44).
      loss_scale: LossScale (host state, updated from the device flag).
      order: enqueue order as registration indices (default: backward order,
        i.e. reversed registration).
      comm: dist.Communicator (or emulation.LocalComm) for p > 1; None = a
        single worker, no collective.
      eta_bytes: hybrid threshold (collectives.py:238-244) on fp16 bucket bytes;
        float("inf") = every bucket hierarchical; a path = seed it from a
        measured sweep file through the netsim model (resolve_eta).
      hier_variant: variant for hierarchical buckets: "hierarchical" = the
        literal master path over NCCL, "sharded" = RS/AR/AG over NCCL,
        "ordered_hier" = own bit-exact two-level kernel (power-of-two k).
      flat_variant: flat buckets: "ring" (NCCL) or "ordered" (own bit-exact
        NVLink all-reduce, gs_ordered_allreduce_f16).
      ordered_push: the ordered all-reduce's push form (same bits).
      sharded_update: ZeRO-1 step: each rank folds and updates only its
        chunks of every bucket (masters / velocities sharded, working copy
        replicated); fused_collective selects the fused kernels
        (gs_rs_pass1 / gs_zero_update) over separate collectives.
      init_master: flat fp32 initial weights in registration order.
      grad_norm: compute the experiment's grad-norm metric.
      local_workers: with comm=None, simulate p workers on this GPU the way
        the reference's in-memory executor does (collectives.py:286-340):
        each worker's gradients are packed into its own wire buffer and every
        bucket is reduced by the ordered pairwise-tree fold kernel
        (gs_fold_f16_tree), bit-identical to allreduce_f16.  enqueue() then
        takes one gradient set per worker.
      snapshot_wire: p = 1 only.  No collective consumes the fused batches, so
        by default the wire is LAZY: the kernels read the gradients where they
        lie and bucket_payload() packs the reference's FusedBatch payloads
        from them on request (the gradients must then be unchanged since the
        step).  snapshot_wire=True packs the wire inside every step instead
        (2 B/element more HBM traffic).
      wire_dtype: "f16" (the north star's binary16 wire) or "f32" — the
        reference's own run_experiment path: fp32 gradients fused at 4 bytes
        per element and all-reduced as the ascending fp32 left fold, mean
        applied by pass 1 (experiment.py:282-301, 368-413).  Replicated
        update only (no sharded_update).
    """

    def __init__(self, specs, cfg: LarsConfig, *, threshold_bytes: int = 4 << 20,
                 loss_scale: LossScale | None = None, order=None, comm=None,
                 eta_bytes: int = 0, hier_variant: str = "hierarchical",
                 init_master=None, grad_norm: bool = True, device=None,
                 local_workers: int = 1, flat_variant: str = "ring", ordered_push: bool = False,
                 sharded_update: bool = False, fused_collective: bool = True,
                 snapshot_wire: bool = False, wire_dtype: str = "f16"):
        self.specs = [s if isinstance(s, ParamSpec) else ParamSpec(s[0], tuple(s[1]), s[2])
                      for s in specs]
        self.cfg = cfg
        self.loss_scale = loss_scale if loss_scale is not None else LossScale()
        self.comm = comm
        if comm is not None and local_workers != 1:
            raise ValueError("local_workers is only for the single-process (comm=None) mode")
        self.p = comm.topo.p if comm is not None else int(local_workers)
        self.local = comm is None and self.p > 1
        self.emulated = bool(getattr(comm, "emulated", False))
        self.eta_bytes = resolve_eta(eta_bytes, comm.topo if comm is not None else None,
                                     2 if wire_dtype == "f16" else 4)
        self.hier_variant = hier_variant
        self.grad_norm_enabled = grad_norm
        self.device = device or dev.require_cuda()
        n = len(self.specs)
        self.order = list(reversed(range(n))) if order is None else list(order)
        if sorted(self.order) != list(range(n)):
            raise ValueError("order must be a permutation of the parameter indices")
        sizes = [s.numel for s in self.specs]
        self.sizes = sizes
        if wire_dtype not in ("f16", "f32"):
            raise ValueError(f"wire_dtype must be 'f16' or 'f32', got {wire_dtype!r}")
        self.wire_dtype = wire_dtype
        self.f16 = wire_dtype == "f16"
        #: bytes per wire element and the wire's torch dtype
        self.isz = 2 if self.f16 else 4
        self.wdt = torch.uint16 if self.f16 else torch.float32

        # ---- wire layout: FusionBuffer boundaries over the enqueue order
        self.wire_off, self.buckets, self.total = plan_layout(self.specs, self.order,
                                                              threshold_bytes, self.isz)

        d = self.device
        self.sharded = bool(sharded_update)
        if self.sharded and (comm is None or comm.topo.p < 2):
            raise ValueError("sharded_update needs a Communicator with p >= 2")
        if self.sharded and not self.f16:
            raise ValueError("the sharded update runs on the binary16 wire (wire_dtype='f16')")
        self.fused_collective = bool(fused_collective) and self.sharded and \
            comm.topo.p in (2, 4, 8)
        for b in self.buckets:
            if self.sharded:
                b.algorithm = "sharded-update"
            elif comm is not None:
                b.algorithm = comm.pick(b.nbytes, self.eta_bytes, hier_variant, flat_variant)
            else:
                b.algorithm = "ordered" if self.local else "none"
        if self.emulated and any(b.algorithm not in ("ordered", "ordered_hier", "sharded-update")
                                 for b in self.buckets):
            raise ValueError("emulated ranks run the own-kernel paths only: sharded_update=True "
                             "or flat_variant='ordered' with eta_bytes=0")
        self.snapshot_wire = bool(snapshot_wire) and comm is None and not self.local
        self.ordered = None
        self.arena = None
        self._half = 0
        if self.sharded:
            self._init_sharded_arena(comm, d)
        elif comm is not None and any(b.algorithm in ("ordered", "ordered_hier")
                                      for b in self.buckets):
            # the ordered (bit-exact) collective reads peers' wires over
            # NVLink: the wire lives in a double-buffered symmetric window
            self.ordered = comm.make_ordered_wire(self.total, d, push=ordered_push,
                                                  itemsize=self.isz)
            self.wire = self.ordered.halves[0]
        else:
            self.wire = torch.zeros(self.total, dtype=self.wdt, device=d)
        self._last_wire = self.wire
        if not self.sharded:
            self.master = torch.zeros(self.total, dtype=torch.float32, device=d)
            self.velocity = torch.zeros(self.total, dtype=torch.float32, device=d)
            self.working = torch.zeros(self.total, dtype=torch.uint16, device=d)
        self.grad32 = torch.zeros(self.total, dtype=torch.float32, device=d)
        if init_master is not None:
            self.load_master(init_master)

        self.groups = [self._group_view(i) for i in range(n)]

        # ---- segment table (registration order = group order, so the
        # grad-norm sum runs in the reference's group order) and chunk table
        # in wire order, so every bucket owns a contiguous chunk range
        gsrc = self.red if self.sharded else self.wire
        gb, mb, vb, hb = (t.data_ptr() for t in (gsrc, self.master, self.velocity, self.working))
        segs = [SegmentSpec(gb + self.isz * self.wire_off[i], mb + 4 * self.wire_off[i],
                            vb + 4 * self.wire_off[i], hb + 2 * self.wire_off[i], sizes[i],
                            segment_flags(self.groups[i])) for i in range(n)]
        if self.sharded:
            self.plan = LarsPlan(segs, d, order=self.order,
                                 partials=self.arena.view("partials", torch.float64),
                                 ctl=self.arena.view("ctl", torch.uint8))
        else:
            self.plan = LarsPlan(segs, d, order=self.order)
        if not self.fused_collective:
            # the pipeline owns the master arena: pass 2 hands the updated
            # masters' sum w^2 to the next step's pass 1
            self.plan.enable_w2_cache()
        begin, count = self.plan.host_segs["chunk_begin"], self.plan.host_segs["chunk_count"]
        c = 0
        for b in self.buckets:
            b.chunk0 = c
            b.nchunk = int(sum(int(count[i]) for i in b.params))
            if b.nchunk:
                assert int(begin[b.params[0]]) == c or sizes[b.params[0]] == 0
            c += b.nchunk
        assert c == self.plan.nchunk
        if self.ordered is not None:
            self._half_segs = [self.plan.alt_segments(
                [h.data_ptr() + self.isz * o for o in self.wire_off]) for h in self.ordered.halves]
        if self.sharded:
            self._init_ownership(d)

        self._pack_cache: dict = {}
        self._src_cache: dict = {}
        self._grad_arena = None
        self._wire_src = None
        self._prepared = None
        self._pending = False
        self._inc = None
        real_comm = comm is not None and not self.emulated
        self._pack_stream = torch.cuda.Stream(device=d) if real_comm else None
        # replicated update at p > 1: pass 1 of bucket b runs on its own
        # stream so it overlaps the all-reduce of bucket b + 1
        self._p1_stream = torch.cuda.Stream(device=d) if real_comm else None
        # the incremental API's side stream (bucket work under backward);
        # emulated ranks keep one stream so their peer launches batch
        self._side_stream = torch.cuda.Stream(device=d) if not self.emulated else None
        if self.local:
            self.rank_wire = [torch.zeros(self.total, dtype=self.wdt, device=d)
                              for _ in range(self.p)]
            self._slots = dev.upload(np.array([t.data_ptr() for t in self.rank_wire],
                                              dtype=np.uint64), d)

    # ------------------------------------------------------------ sharded
    def _init_sharded_arena(self, comm, d) -> None:
        """ZeRO-1 layout: one symmetric window holding the raw wire (the
        gradients as packed, or written in place through grad_views()), the
        reduced wire (this rank's folded slices), the binary16 working
        weights, the masters, the velocities, the chunk partials and the
        control block, so every peer can reach them."""
        p = comm.topo.p
        chunks, _, _ = build_chunks(self.sizes, self.order)
        self._host_chunks = chunks
        nchunk = len(chunks)
        sms = torch.cuda.get_device_properties(d).multi_processor_count
        # CTAs per rank of the peer-synchronised kernels (each clamps to what
        # is co-resident: 4 CTAs per SM for gs_rs_pass1 at p = 2 / 4)
        self._nblocks = comm.peer_ctas or 4 * sms
        regions = {
            "wire": 2 * self.total, "red": 2 * self.total, "working": 2 * self.total,
            "master": 4 * self.total, "velocity": 4 * self.total,
            "partials": 8 * max(1, 3 * nchunk), "ctl": _native.CTL_DTYPE.itemsize,
        }
        self.arena = comm.make_arena(regions, d, 2 * self._nblocks * p)
        a = self.arena
        self.wire = a.view("wire", torch.uint16)
        self.red = a.view("red", torch.uint16)
        self.master = a.view("master", torch.float32)
        self.velocity = a.view("velocity", torch.float32)
        self.working = a.view("working", torch.uint16)
        self.epoch_base = torch.zeros(1, dtype=torch.int32, device=d)

    def _shared_upload(self, arr: np.ndarray) -> torch.Tensor:
        """A device table every rank passes to a peer launch: identical
        content on every rank; emulated ranks share one tensor so the batched
        launch's arguments agree."""
        if not self.emulated:
            return dev.upload(arr, self.device)
        cache = self.comm.world.__dict__.setdefault("_tables", {})
        key = (arr.dtype.str, arr.tobytes())
        t = cache.get(key)
        if t is None:
            t = cache[key] = dev.upload(arr, self.device)
        return t

    def _init_ownership(self, d) -> None:
        """Sharded update: which chunks this rank folds and updates (needs
        the buckets' chunk ranges, i.e. runs after the LARS plan is built)."""
        p, r = self.comm.topo.p, self.comm.rank
        chunks = self._host_chunks
        # ownership, PER BUCKET: rank r owns chunks [C_b[r], C_b[r+1]) of bucket
        # b (balanced by elements, in wire order) = wire elements [E_b[r],
        # E_b[r+1]); every bucket's fold is spread over all ranks
        abs_start = np.array([self.wire_off[int(c["seg"])] + int(c["start"]) for c in chunks],
                             dtype=np.int64)
        clen = np.array([int(c["len"]) for c in chunks], dtype=np.int64)
        self._bucket_C, self._bucket_E = shard_buckets(self.buckets, abs_start, p)
        self._own_bucket = [(C[r], C[r + 1]) for C in self._bucket_C]
        self._rs_bounds, self._part_bounds, self._w16_bounds, self._m_bounds = [], [], [], []
        own_list, own_off = [], [0]
        for C, E in zip(self._bucket_C, self._bucket_E):
            own_list.extend(range(C[r], C[r + 1]))
            own_off.append(len(own_list))
            self._rs_bounds.append(self._shared_upload(np.array(E, dtype=np.int64)))
            self._part_bounds.append(self._shared_upload(np.array([24 * c for c in C],
                                                                  dtype=np.int64)))
            self._w16_bounds.append(self._shared_upload(np.array([2 * e for e in E],
                                                                 dtype=np.int64)))
            self._m_bounds.append(self._shared_upload(np.array([4 * e for e in E],
                                                               dtype=np.int64)))
        self._own_list = dev.upload(np.array(own_list or [0], dtype=np.int32), d)
        self._own_off = dev.upload(np.array(own_off, dtype=np.int32), d)
        self._own_count = [own_off[b + 1] - own_off[b] for b in range(len(self.buckets))]
        self._n_own = len(own_list)
        #: elements this rank updates (pass 2) per step
        self.owned_elems = int(clen[own_list].sum()) if own_list else 0
        plan, a = self.plan, self.arena
        # per-segment "scale published" epochs of gs_zero_update
        self._seg_ready = torch.zeros(max(1, plan.nseg), dtype=torch.int32, device=d)
        self._ctx = rank_ctx(r, timeout_s=self.comm.timeout_s, status=dev.ptr(plan.ctl) + 16,
                             epoch_base=dev.ptr(self.epoch_base), segs=dev.ptr(plan.base_segs),
                             chunks=dev.ptr(plan.d_chunks), own_list=dev.ptr(self._own_list),
                             own_off=dev.ptr(self._own_off), ctl=dev.ptr(plan.ctl),
                             seg_scale=dev.ptr(plan.seg_scale), red=dev.ptr(self.red),
                             partials=dev.ptr(plan.partials), seg_out=dev.ptr(plan.seg_out),
                             seg_ready=dev.ptr(self._seg_ready))
        # this rank's one-entry context table for the native executor
        self._ctx_dev = dev.upload(self._ctx, d)

    def _op(self, fn: str, *args, count: int | None = None) -> PeerOp:
        return PeerOp(fn, self._ctx, args, count=count, device=self.device)

    def _gather_gen(self):
        """Masters and velocities made whole on every rank (inspection,
        checkpoints; the step only keeps the working copy replicated)."""
        if not self.sharded:
            return
        sh = int(torch.cuda.current_stream(self.device).cuda_stream)
        p, a, nb = self.comm.topo.p, self.arena, len(self.buckets)
        for j, name in enumerate(("master", "velocity")):
            for b in range(nb):
                yield self._op("gs_ordered_allgather", p, dev.ptr(a.peers(name)),
                               dev.ptr(a.peers("sig")), dev.ptr(self._m_bounds[b]),
                               j * nb + b + 1, self._nblocks, sh)
        _native.call("gs_counter_add", dev.ptr(self.epoch_base), 2 * nb, sh)

    def gather_state(self) -> None:
        """Make the sharded masters and velocities whole on every rank."""
        self._drive(self._gather_gen())
        self._gathered = True

    def state_groups(self) -> list:
        """The ParamGroups with current masters / velocities on this rank: a
        sharded pipeline keeps only its own chunks of them current between
        steps, so this gathers first when a step ran since the last gather
        (collective: every rank calls it).  Replicated pipelines: `groups`."""
        if self.sharded and not getattr(self, "_gathered", True):
            self.gather_state()
        return self.groups

    def _drive(self, gen) -> None:
        """Launch this rank's peer ops as they come (one rank per launch)."""
        if self.emulated:
            raise RuntimeError("an emulated rank is driven by its LocalWorld (world.step / "
                               "world.gather_state / world.begin ...), with its peers in lockstep")
        for op in gen:
            launch([op])

    def _gen_sharded(self, tabs, s0, timer):
        """The ZeRO-1 step.  Fused: [pack] -> gs_rs_pass1 over the rank's
        owned chunks of every bucket (fold from the peers' raw wires into the
        reduced wire + pass 1, partials and flags pushed to every peer) ->
        gs_zero_update (fence, trust, pass 2 + working-weight push) ->
        fence.  Separate collectives: pack -> per bucket reduce-scatter +
        pass 1 -> all-gather of the partials -> trust -> pass 2 -> all-gather
        of the working weights."""
        plan, a = self.plan, self.arena
        sh = int(s0.cuda_stream)
        p = self.comm.topo.p
        nb = len(self.buckets)
        sig, ebase = dev.ptr(a.peers("sig")), dev.ptr(self.epoch_base)
        plan.use_segments(None)
        if self.fused_collective:
            if tabs is not None:
                if timer:
                    timer("pack")
                self._pack(tabs, nb, sh)
            if timer:
                timer("rs_pass1")
            yield self._op("gs_rs_pass1", p, dev.ptr(a.peers("wire")), sig,
                           dev.ptr(a.peers("partials")), dev.ptr(a.peers("ctl")), 0, nb,
                           plan.sp, plan.hint, plan.parity, 1, self._nblocks, sh)
            if timer:
                timer("update")
            # the peer fence, the trust kernel and pass 2 with the working-
            # weight push in one launch
            yield self._op("gs_zero_update", p, sig, dev.ptr(a.peers("working")), 2, plan.nseg,
                           plan.nchunk, 0, nb, None, plan.sp, plan.hint, plan.parity, _MASK, sh,
                           count=self._n_own)
            if timer:
                timer("fence_end")
            # the closing fence also advances the epoch base for the next step
            yield self._op("gs_peer_fence", p, sig, 3, 4, sh)
        else:
            # the reduce-scatter folds in place in the reduced wire
            if timer:
                timer("pack")
            self._pack(tabs, nb, sh)
            for b in range(nb):
                if timer:
                    timer(f"rs{b}")
                yield self._op("gs_ordered_reduce_scatter_f16", p, dev.ptr(a.peers("red")), sig,
                               dev.ptr(self._rs_bounds[b]), b + 1, self._nblocks, sh)
                c0, c1 = self._own_bucket[b]
                if timer:
                    timer(f"pass1_{b}")
                if c1 > c0:
                    plan.pass1(sh, g_is_f16=self.f16, chunk0=c0, nchunk=c1 - c0)
            if timer:
                timer("gather_partials")
            for b in range(nb):
                yield self._op("gs_ordered_allgather", p, dev.ptr(a.peers("partials")), sig,
                               dev.ptr(self._part_bounds[b]), nb + 1 + b, self._nblocks, sh)
            if timer:
                timer("trust")
            plan.trust(sh, peer_ctl=a.peers("ctl"), npeers=p)
            if timer:
                timer("pass2")
            for b in range(nb):
                c0, c1 = self._own_bucket[b]
                if c1 > c0:
                    plan.pass2(sh, g_is_f16=self.f16, flag_mask=_MASK, chunk0=c0, nchunk=c1 - c0)
            if timer:
                timer("gather_w16")
            for b in range(nb):
                yield self._op("gs_ordered_allgather", p, dev.ptr(a.peers("working")), sig,
                               dev.ptr(self._w16_bounds[b]), 2 * nb + 1 + b, self._nblocks, sh)
            _native.call("gs_counter_add", ebase, 3 * nb + 1, sh)
        self._last_wire = self.red
        if timer:
            timer("end")

    # ------------------------------------------------------------ layout
    def _group_view(self, i: int) -> ParamGroup:
        s, o, n = self.specs[i], self.wire_off[i], self.sizes[i]
        return ParamGroup(name=s.name, kind=s.kind, master_w=self.master[o:o + n],
                          grad=self.grad32[o:o + n], velocity=self.velocity[o:o + n],
                          working_w16=self.working[o:o + n])

    def load_master(self, flat) -> None:
        """Set master weights from a flat fp32 vector in registration order and
        refresh the working copy (make_param_group, lars.py:128-139)."""
        src = dev.to_cuda(np.asarray(flat, dtype=np.float32) if not dev.is_tensor(flat)
                          else flat.to(torch.float32), self.device).reshape(-1)
        if src.numel() != sum(self.sizes):
            raise ValueError(f"expected {sum(self.sizes)} master values, got {src.numel()}")
        ro = 0
        for i, n in enumerate(self.sizes):
            o = self.wire_off[i]
            self.master[o:o + n].copy_(src[ro:ro + n])
            ro += n
        from .halfprec import f32_to_f16
        self.working.copy_(f32_to_f16(self.master))
        self.invalidate_master_cache()

    def invalidate_master_cache(self) -> None:
        """Call after writing the master arena other than through step()
        (e.g. through ``groups[i].master_w``): pass 1 then re-derives the
        per-chunk sum w^2 that pass 2 otherwise carries over."""
        if hasattr(self, "plan"):
            self.plan.invalidate_w2_cache()

    def registration_view(self, arena: torch.Tensor) -> torch.Tensor:
        """Gather an arena (wire layout) into registration order (host checks)."""
        return torch.cat([arena[self.wire_off[i]:self.wire_off[i] + n]
                          for i, n in enumerate(self.sizes)])

    def bucket_payload(self, b: int) -> torch.Tensor:
        """Bucket b of the last step's wire (the reference's FusedBatch
        payload, fusion.py:84-90; after a collective, the reduced bucket —
        with the sharded update only this rank's slices are reduced).  At
        p = 1 with the lazy wire it is packed from the last step's gradients
        on first request, so those must be unchanged since the step."""
        src = self._wire_src
        if src is not None:
            tabs = self._tables_for(src, self.wire)
            self._pack(tabs, len(self.buckets),
                       int(torch.cuda.current_stream(self.device).cuda_stream))
            self._wire_src = None
        bk = self.buckets[b]
        return self._last_wire[bk.start:bk.start + bk.length]

    # ------------------------------------------------------------ packing
    def grad_arena(self) -> torch.Tensor:
        """A device gradient arena (binary16 as uint16, or fp32) in
        registration order that a backward pass (or a host copy) can write
        into; step() accepts it."""
        if self._grad_arena is None:
            self._grad_arena = torch.zeros(sum(self.sizes), dtype=self.wdt, device=self.device)
        return self._grad_arena

    def grad_views(self) -> list:
        """Sharded update: per-parameter views of this rank's raw wire (the
        gradients' bucket slots, DDP's gradient-as-bucket-view).  Gradients
        written there need no pack: step(pipe.grad_views(), k) reads them in
        place, and the fused step never modifies them."""
        if not self.sharded:
            raise ValueError("grad_views() is for the sharded update; at p = 1 the kernels "
                             "read any gradient buffer in place")
        return [self.wire[o:o + n] for o, n in zip(self.wire_off, self.sizes)]

    def _grad_list(self, grads):
        if dev.is_tensor(grads):
            flat = grads.reshape(-1)
            if flat.numel() != sum(self.sizes):
                raise ValueError("flat gradient length does not match the parameters")
            views, ro = [], 0
            for n in self.sizes:
                views.append(flat[ro:ro + n])
                ro += n
            return views
        views = list(grads)
        if len(views) != len(self.sizes):
            raise ValueError(f"expected {len(self.sizes)} gradients, got {len(views)}")
        return views

    def _dtype_ok(self, t) -> bool:
        return t.dtype in ((torch.uint16, torch.float16) if self.f16 else (torch.float32,))

    def _check_grads(self, views) -> None:
        for t, n in zip(views, self.sizes):
            if t.numel() != n or not self._dtype_ok(t) or not t.is_cuda:
                raise ValueError("gradients must be CUDA " + ("fp16/uint16" if self.f16 else "fp32")
                                 + " tensors of the parameter sizes")

    def _tables_for(self, views, dst: torch.Tensor):
        """Per-bucket gs_copy tables packing `views` into `dst`, plus entry
        len(buckets) = every bucket in one table (cached, bounded)."""
        key = (dst.data_ptr(),) + tuple((t.data_ptr(), t.numel()) for t in views)
        tabs = self._pack_cache.get(key)
        if tabs is None:
            self._check_grads(views)
            wb = dst.data_ptr()
            tabs, host = [], []
            for b in self.buckets:
                z = self.isz
                t = copy_table((views[i].data_ptr(), wb + z * self.wire_off[i], z * self.sizes[i])
                               for i in b.params if self.sizes[i])
                tabs.append((dev.upload(t, self.device), len(t)))
                host.append(t)
            allt = np.concatenate(host) if host else copy_table([])
            tabs.append((dev.upload(allt, self.device), len(allt)))
            if len(self._pack_cache) >= 16:
                self._pack_cache.pop(next(iter(self._pack_cache)))
            self._pack_cache[key] = tabs
        return tabs

    @staticmethod
    def _pack(tabs, b: int, stream_h: int) -> None:
        tab, n = tabs[b]
        if n:
            _native.call("gs_batched_copy", dev.ptr(tab), n, stream_h)

    # ------------------------------------------------------------ the step
    def params_for(self, step: int) -> np.ndarray:
        cfg = self.cfg
        return step_params(eta=cfg.eta, epsilon=cfg.epsilon, gamma=cfg.schedule.lr(step),
                           weight_decay=cfg.weight_decay, momentum=cfg.momentum,
                           mean_divisor=self.p if self.p > 1 else None,
                           unscale_divisor=self.loss_scale.scale,
                           grad_norm=self.grad_norm_enabled)

    def prepare(self, step: int) -> None:
        """Host-only part of a step (schedule, loss scale, launch hint)."""
        self.plan.set_params(self.params_for(step), g_is_f16=self.f16)
        self._prepared = step

    def _sources(self, grads):
        """Launch tables for this gradient set, cached on the buffer
        addresses so a steady-state step does no per-tensor host work."""
        if dev.is_tensor(grads):
            ck = (grads.data_ptr(), grads.numel(), grads.dtype)
        else:
            ck = tuple((g.data_ptr(), g.numel()) if dev.is_tensor(g) else id(g) for g in grads)
        hit = self._src_cache.get(ck)
        if hit is not None:
            return hit
        res = self._sources_uncached(grads)
        if len(self._src_cache) >= 16:
            self._src_cache.pop(next(iter(self._src_cache)))
        self._src_cache[ck] = res
        return res

    def _sources_uncached(self, grads):
        if self.local:
            if len(grads) != self.p:
                raise ValueError(f"expected gradients of {self.p} workers, got {len(grads)}")
            return [self._tables_for(self._grad_list(g), w) for g, w in zip(grads, self.rank_wire)]
        views = self._grad_list(grads)
        self._check_grads(views)
        if self.comm is None:
            # the kernels read the gradients where they lie (lazy wire)
            tab = self.plan.alt_segments([t.data_ptr() for t in views])
            return ("direct", tab, views,
                    self._tables_for(views, self.wire) if self.snapshot_wire else None)
        if self.ordered is not None:
            return tuple(self._tables_for(views, h) for h in self.ordered.halves)
        if self.sharded:
            if not self.fused_collective:
                # the separate reduce-scatter folds in place: pack into the
                # reduced wire (also from grad_views(), a wire -> red copy)
                return self._tables_for(views, self.red)
            if all(t.data_ptr() == self.wire.data_ptr() + 2 * o
                   for t, o, n in zip(views, self.wire_off, self.sizes) if n):
                return None  # gradients already in the raw wire: no pack
        return self._tables_for(views, self.wire)

    def enqueue(self, grads, step: int, timer=None) -> None:
        """Launch one step on the current stream (no host sync).

        `timer`, if given, is called with a phase name before each phase
        (the bench records CUDA events there).  finish() must be called
        before the next step is enqueued: the LossScale update needs this
        step's flags (experiment.py:403-413).

        The two hot steps (p = 1 and the fused sharded step) go through the
        native executor (one C call, gs_step_replicated / gs_step_zero) unless
        a timer or NVTX ranges ask for the per-kernel path; both launch the
        same kernels in the same order."""
        if timer is None and not _trace.enabled() and self._fast_ok():
            tabs = self._open_step(grads, step)
            sh = int(torch.cuda.current_stream(self.device).cuda_stream)
            if self.sharded:
                rec = self._zero_record(tabs)
                _native.call("gs_step_zero", rec.ctypes.data, 1, dev.ptr(self._ctx_dev),
                             *self._zero_args(self._n_own, sh))
                self._last_wire = self.red
            else:
                _, seg_tab, views, snap = tabs
                rec = self._replicated_record(seg_tab, snap)
                plan = self.plan
                _native.call("gs_step_replicated", rec.ctypes.data, 1 if self.f16 else 0,
                             plan.sp, plan.hint, plan.parity, _MASK, sh)
                self._wire_src = views if snap is None else None
                self._last_wire = self.wire
            self.plan.end_step()
            return
        self._drive(self._enqueue_gen(grads, step, timer))

    # ---- the native executor's records (host structs, rebuilt only when a
    # pointer changes)
    def _fast_ok(self) -> bool:
        if self.emulated:
            return False
        if self.sharded:
            return self.fused_collective
        return self.comm is None and not self.local

    def _replicated_record(self, seg_tab, snap) -> np.ndarray:
        plan = self.plan
        key = (dev.ptr(seg_tab), id(snap))
        rec = getattr(self, "_rep_rec", None)
        if rec is None or self._rep_key != key:
            rec = np.zeros(1, dtype=_native.STEP_RANK_DTYPE)
            nb = len(self.buckets)
            if snap is not None and snap[nb][1]:
                rec["pack"], rec["npack"] = dev.ptr(snap[nb][0]), snap[nb][1]
            rec["segs"], rec["chunks"] = dev.ptr(seg_tab), dev.ptr(plan.d_chunks)
            rec["nseg"], rec["nchunk"] = plan.nseg, plan.nchunk
            rec["partials"], rec["seg_scale"] = dev.ptr(plan.partials), dev.ptr(plan.seg_scale)
            rec["seg_out"], rec["ctl"] = dev.ptr(plan.seg_out), dev.ptr(plan.ctl)
            self._rep_rec, self._rep_key = rec, key
            self._rep_refs = (seg_tab, snap)  # keep the tables alive with the record
        wsq = plan.wsq
        rec["wsq_out"] = dev.ptr(wsq) if wsq is not None else 0
        rec["wsq_in"] = dev.ptr(wsq) if wsq is not None and plan.wsq_valid else 0
        return rec

    def _zero_record(self, tabs) -> np.ndarray:
        """gs_step_zero's rank record (pack table = the all-bucket table, or
        none when the gradients already lie in the raw wire)."""
        key = id(tabs)
        rec = getattr(self, "_zero_rec", None)
        if rec is None or self._zero_key != key:
            plan, nb = self.plan, len(self.buckets)
            rec = np.zeros(1, dtype=_native.STEP_RANK_DTYPE)
            if tabs is not None and tabs[nb][1]:
                rec["pack"], rec["npack"] = dev.ptr(tabs[nb][0]), tabs[nb][1]
            rec["segs"], rec["chunks"] = dev.ptr(plan.base_segs), dev.ptr(plan.d_chunks)
            rec["nseg"], rec["nchunk"] = plan.nseg, plan.nchunk
            rec["partials"], rec["seg_scale"] = dev.ptr(plan.partials), dev.ptr(plan.seg_scale)
            rec["seg_out"], rec["ctl"] = dev.ptr(plan.seg_out), dev.ptr(plan.ctl)
            rec["epoch_base"] = dev.ptr(self.epoch_base)
            self._zero_rec, self._zero_key, self._zero_refs = rec, key, tabs
        return rec

    def _zero_args(self, max_own: int, sh: int) -> tuple:
        """The arguments of gs_step_zero after (ranks, nranks, ctx)."""
        a, plan = self.arena, self.plan
        return (self.comm.topo.p, dev.ptr(a.peers("wire")), dev.ptr(a.peers("sig")),
                dev.ptr(a.peers("partials")), dev.ptr(a.peers("ctl")),
                dev.ptr(a.peers("working")), len(self.buckets), max_own, plan.sp, plan.hint,
                plan.parity, _MASK, self._nblocks, sh)

    def _open_step(self, grads, step: int):
        """Host prologue of every step: the previous step finished, scalars
        staged, launch tables for these gradients."""
        if self._pending:
            raise RuntimeError("the previous step was not finished: call finish() before "
                               "enqueueing the next step (its flags drive the loss scale)")
        if self._prepared != step:
            self.prepare(step)
        self._prepared = None
        tabs = self._sources(grads)
        self._pending = True
        self._wire_src = None
        self._gathered = False
        return tabs

    def _enqueue_gen(self, grads, step: int, timer=None):
        tabs = self._open_step(grads, step)
        s0 = torch.cuda.current_stream(self.device)
        timer = _trace.hook(timer)
        if self.sharded:
            yield from self._gen_sharded(tabs, s0, timer)
        else:
            yield from self._gen_replicated(tabs, s0, timer)
        if isinstance(timer, _trace.PhaseRanges):
            timer.close()
        self.plan.end_step()

    def _gen_replicated(self, tabs, s0, timer):
        plan = self.plan
        sh = int(s0.cuda_stream)
        nb = len(self.buckets)
        if self.comm is None and not self.local:
            _, seg_tab, views, snap = tabs
            plan.use_segments(seg_tab)
            if snap is not None:
                if timer:
                    timer("pack")
                self._pack(snap, nb, sh)
                self._last_wire = self.wire
            else:
                self._wire_src = views  # bucket_payload() packs these on demand
                self._last_wire = self.wire
            if timer:
                timer("pass1")
            plan.pass1(sh, g_is_f16=self.f16)
        elif self.local:
            plan.use_segments(None)
            if timer:
                timer("pack")
            for b in range(nb):
                for t in tabs:
                    self._pack(t, b, sh)
            if timer:
                timer("fold")
            wb = self.wire.data_ptr()
            for bk in self.buckets:
                if not bk.length:
                    continue
                if self.f16:
                    _native.call("gs_fold_f16_tree", dev.ptr(self._slots), self.p, bk.start,
                                 wb + 2 * bk.start, bk.length, None, sh)
                else:  # ascending fp32 sum; pass 1 divides by float32(p)
                    _native.call("gs_fold_f32", dev.ptr(self._slots), self.p, bk.start,
                                 wb + 4 * bk.start, bk.length, 0, sh)
            self._last_wire = self.wire
            if timer:
                timer("pass1")
            plan.pass1(sh, g_is_f16=self.f16)
        else:
            # bucket b+1 is packed (pack stream) while bucket b's all-reduce is
            # in flight and bucket b-1 runs pass 1 (compute stream)
            ps = self._pack_stream if self._pack_stream is not None else s0
            if ps is not s0:
                ps.wait_stream(s0)
            half = self._half
            wire = self.ordered.halves[half] if self.ordered is not None else self.wire
            ptabs = tabs[half] if self.ordered is not None else tabs
            plan.use_segments(self._half_segs[half] if self.ordered is not None else None)
            works = []
            for b, bk in enumerate(self.buckets):
                with torch.cuda.stream(ps):
                    self._pack(ptabs, b, int(ps.cuda_stream))
                    payload = wire[bk.start:bk.start + bk.padded]
                    if bk.algorithm == "ring":
                        works.append(self.comm.allreduce_ring(payload, async_op=True))
                    else:
                        if bk.algorithm not in ("ordered", "ordered_hier"):
                            self.comm.allreduce(payload, bk.algorithm)
                        ev = torch.cuda.Event()
                        ev.record(ps)
                        works.append(ev)
            p1s = self._p1_stream if self._p1_stream is not None and not timer else s0
            if p1s is not s0:
                p1s.wait_stream(s0)
            sh1 = int(p1s.cuda_stream)
            for b, bk in enumerate(self.buckets):
                w = works[b]
                if isinstance(w, torch.cuda.Event):
                    s0.wait_event(w)
                else:
                    w.wait()
                if bk.algorithm in ("ordered", "ordered_hier"):
                    if timer:
                        timer(f"allreduce{b}")
                    yield self._ordered_op(half, bk, sh, b)
                if timer:
                    timer(f"pass1_{b}")
                if p1s is not s0:
                    p1s.wait_stream(s0)
                plan.pass1(sh1, g_is_f16=self.f16, chunk0=bk.chunk0, nchunk=bk.nchunk)
            if p1s is not s0:
                s0.wait_stream(p1s)
            if ps is not s0:
                s0.wait_stream(ps)
            if self.ordered is not None:
                self.ordered.advance(nb + 1, sh)
                self._half ^= 1
            self._last_wire = wire
        if timer:
            timer("trust")
        plan.trust(sh)
        if timer:
            timer("pass2")
        plan.pass2(sh, g_is_f16=self.f16, flag_mask=_MASK)
        plan.use_segments(None)
        if timer:
            timer("end")

    def _ordered_op(self, half: int, bk: Bucket, sh: int, slot: int) -> PeerOp:
        """Own bit-exact all-reduce of one bucket: flat, or over
        Topology(p, k)'s two levels (hierarchical buckets, hier_variant =
        'ordered_hier'); identical results."""
        # the padded range (its zero slack stays zero under the fold): whole
        # 8-element vectors, so small buckets qualify for the LL kernel
        if bk.algorithm == "ordered_hier" and self.f16:
            return self.ordered.hier_op(half, bk.start, bk.padded, self.comm.topo.k, sh, slot=slot)
        # fp32: the reference's left fold does not factor over groups, so the
        # hierarchical buckets take the flat kernel (the same fold)
        return self.ordered.allreduce_op(half, bk.start, bk.padded, sh, slot=slot)

    def _bucket_host_ranges(self):
        """Per bucket, the [lo, hi) element range of the registration-order
        flat gradient that holds exactly its tensors, or None when a bucket's
        tensors are not contiguous in registration order (custom orders)."""
        if getattr(self, "_host_ranges", "unset") != "unset":
            return self._host_ranges
        offs = np.concatenate([[0], np.cumsum(self.sizes)])
        ranges = []
        for bk in self.buckets:
            idx = sorted(bk.params)
            if idx != list(range(idx[0], idx[-1] + 1)):
                ranges = None
                break
            ranges.append((int(offs[idx[0]]), int(offs[idx[-1] + 1])))
        self._host_ranges = ranges
        return ranges

    def enqueue_host(self, host_flat: torch.Tensor, step: int) -> None:
        """One step from a pinned host fp16 gradient (registration order).
        p = 1: the host->device copy is split per bucket on a copy stream and
        pass 1 of bucket b starts as soon as bucket b has landed, so the PCIe
        transfer overlaps the update; p > 1: one copy, then the regular
        step."""
        arena = self.grad_arena()
        s0 = torch.cuda.current_stream(self.device)
        ranges = self._bucket_host_ranges() if self.comm is None and not self.local else None
        if ranges is None or self.snapshot_wire:
            arena.copy_(host_flat.reshape(-1), non_blocking=True)
            self.enqueue(arena, step)
            return
        if self._pending:
            raise RuntimeError("the previous step was not finished: call finish() first")
        if self._prepared != step:
            self.prepare(step)
        self._prepared = None
        _, seg_tab, views, _ = self._sources(arena)
        plan = self.plan
        sh = int(s0.cuda_stream)
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream(device=self.device)
        cs = self._copy_stream
        cs.wait_stream(s0)
        src = host_flat.reshape(-1)
        evs = []
        with torch.cuda.stream(cs):
            for lo, hi in ranges:
                arena[lo:hi].copy_(src[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
                evs.append(ev)
        self._pending = True
        plan.use_segments(seg_tab)
        self._wire_src = views
        for bk, ev in zip(self.buckets, evs):
            s0.wait_event(ev)
            plan.pass1(sh, g_is_f16=self.f16, chunk0=bk.chunk0, nchunk=bk.nchunk)
        plan.finish(sh, self.f16, _MASK)
        plan.use_segments(None)
        plan.end_step()
        self._last_wire = self.wire

    # ------------------------------------------------------------ incremental
    # The step split at bucket granularity, for a backward pass that hands
    # gradients over as they are produced (overlap.py): bucket b
    # is packed, reduced and run through pass 1 on a side stream as soon as
    # its last gradient exists, while the backward pass keeps computing.
    def begin(self, step: int) -> None:
        """Open a step: stage the scalars (current stream)."""
        self._drive(self._begin_gen(step))

    def _begin_gen(self, step: int):
        if self.local:
            raise ValueError("incremental steps need one gradient set per rank "
                             "(local_workers > 1 takes whole gradient sets)")
        if self.sharded and not self.fused_collective:
            raise ValueError("incremental sharded steps use the fused kernels (p in 2, 4, 8)")
        if self._pending:
            raise RuntimeError("the previous step was not finished: call finish() first")
        if self._prepared != step:
            self.prepare(step)
        self._prepared = None
        s0 = torch.cuda.current_stream(self.device)
        half = self._half
        if self.sharded:
            wire = self.wire
            self.plan.use_segments(None)
        elif self.ordered is not None:
            wire = self.ordered.halves[half]
            self.plan.use_segments(self._half_segs[half])
        else:
            wire = self.wire
            self.plan.use_segments(None)
        ss = self._side_stream if self._side_stream is not None else s0
        if ss is not s0:
            ss.wait_stream(s0)
        self._pending = True
        self._gathered = False
        self._inc = {"step": step, "half": half, "wire": wire, "next": 0, "stream": ss,
                     "ready": [None] * len(self.buckets)}
        return
        yield  # a generator with no peer launch

    def submit(self, b: int, grads) -> None:
        """Bucket b's gradients (tensors of its parameters, in `buckets[b].params`
        order, fp16/uint16, on this device) are complete on the current stream.
        Buckets launch strictly in bucket order (every rank issues the same
        collective sequence), each as soon as it and all earlier ones are in."""
        self._drive(self._submit_gen(b, grads))

    def _submit_gen(self, b: int, grads):
        inc = self._inc
        if inc is None:
            raise RuntimeError("submit() outside begin()/end()")
        if inc["ready"][b] is not None:
            raise ValueError(f"bucket {b} submitted twice in one step")
        bk = self.buckets[b]
        grads = list(grads)
        if len(grads) != len(bk.params):
            raise ValueError(f"bucket {b} holds {len(bk.params)} tensors, got {len(grads)}")
        wb = inc["wire"].data_ptr()
        pairs = []
        for i, t in zip(bk.params, grads):
            if t.numel() != self.sizes[i] or not self._dtype_ok(t) \
                    or not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"gradient of {self.specs[i].name!r} must be a contiguous CUDA "
                                 f"{self.wire_dtype} tensor of {self.sizes[i]} elements")
            z = self.isz
            if self.sizes[i] and t.data_ptr() != wb + z * self.wire_off[i]:
                pairs.append((t.data_ptr(), wb + z * self.wire_off[i], z * self.sizes[i]))
        key = ("inc", b, wb) + tuple(p[0] for p in pairs)
        tab = self._pack_cache.get(key)
        if tab is None:
            t = copy_table(pairs)
            if len(self._pack_cache) >= 64:
                self._pack_cache.pop(next(iter(self._pack_cache)))
            tab = self._pack_cache[key] = (dev.upload(t, self.device), len(t))
        ss = inc["stream"]
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        if ss is not torch.cuda.current_stream(self.device):
            for t in grads:
                t.record_stream(ss)  # read there; keep the allocator off it
        inc["ready"][b] = (tab, ev, grads)
        while inc["next"] < len(self.buckets) and inc["ready"][inc["next"]] is not None:
            yield from self._launch_bucket(inc["next"])
            inc["next"] += 1

    def _launch_bucket(self, b: int):
        inc = self._inc
        tab, ev, _ = inc["ready"][b]
        bk, plan, ss = self.buckets[b], self.plan, inc["stream"]
        ss.wait_event(ev)
        sh = int(ss.cuda_stream)
        rng = _trace.hook(None, f"gs.bucket{b}")
        with torch.cuda.stream(ss):
            yield from self._bucket_ops(b, tab, inc, bk, plan, sh)
        if isinstance(rng, _trace.PhaseRanges):
            rng.close()

    def _bucket_ops(self, b, tab, inc, bk, plan, sh):
        """Bucket b on the side stream: pack, reduce, pass 1."""
        if tab[1]:
            _native.call("gs_batched_copy", dev.ptr(tab[0]), tab[1], sh)
        if self.sharded:
            a, p = self.arena, self.comm.topo.p
            yield self._op("gs_rs_pass1", p, dev.ptr(a.peers("wire")), dev.ptr(a.peers("sig")),
                           dev.ptr(a.peers("partials")), dev.ptr(a.peers("ctl")), b, b + 1,
                           plan.sp, plan.hint, plan.parity, b + 1, self._nblocks, sh)
            return
        if bk.algorithm in ("ordered", "ordered_hier"):
            yield self._ordered_op(inc["half"], bk, sh, b)
        elif bk.algorithm != "none":
            self.comm.allreduce(inc["wire"][bk.start:bk.start + bk.padded], bk.algorithm)
        if bk.nchunk:
            plan.pass1(sh, g_is_f16=self.f16, chunk0=bk.chunk0, nchunk=bk.nchunk)

    def end(self) -> None:
        """Close the step: every bucket must have been submitted; trust and
        pass 2 run on the current stream after the side stream's work."""
        self._drive(self._end_gen())

    def _end_gen(self):
        inc = self._inc
        if inc is None:
            raise RuntimeError("end() without begin()")
        missing = [b for b, r in enumerate(inc["ready"]) if r is None]
        if missing:
            names = [self.specs[i].name for i in self.buckets[missing[0]].params]
            raise RuntimeError(f"step ended with {len(missing)} bucket(s) never submitted "
                               f"(first: bucket {missing[0]}, tensors {names[:4]}...)")
        s0 = torch.cuda.current_stream(self.device)
        if inc["stream"] is not s0:
            s0.wait_stream(inc["stream"])
        sh = int(s0.cuda_stream)
        plan = self.plan
        nb = len(self.buckets)
        if self.sharded:
            p, a = self.comm.topo.p, self.arena
            sig = dev.ptr(a.peers("sig"))
            # fence + trust + pass 2 with the working-weight push, one launch
            yield self._op("gs_zero_update", p, sig, dev.ptr(a.peers("working")), nb + 1,
                           plan.nseg, plan.nchunk, 0, nb, None, plan.sp, plan.hint, plan.parity,
                           _MASK, sh, count=self._n_own)
            yield self._op("gs_peer_fence", p, sig, nb + 2, nb + 3, sh)
            self._last_wire = self.red
        else:
            plan.finish(sh, self.f16, _MASK)
            if self.ordered is not None:
                self.ordered.advance(nb + 1, sh)
                self._half ^= 1
            self._last_wire = inc["wire"]
        plan.use_segments(None)
        plan.end_step()
        self._inc = None

    def finish(self) -> StepResult:
        """Read the step's control block (the one host sync) and advance
        LossScale exactly as experiment.py:403-413 does.  Raises
        PeerTimeoutError when a peer wait of the step timed out."""
        if not self._pending:
            raise RuntimeError("finish() without an enqueued step")
        rec = self.plan.read_ctl()
        self._pending = False
        status = int(rec["status"])
        if not status and self.ordered is not None:
            status = self.ordered.status_word()
        if status:
            raise PeerTimeoutError(decode_status(status & 0xFFFFFFFF))
        flags = self.plan.last_flags(rec)
        if not flags & _MASK:
            # pass 2 ran: its per-chunk sum w^2 of the new masters is current
            self.plan.wsq_valid = self.plan.wsq is not None
        step_scale = self.loss_scale.scale
        applied = self.loss_scale.update_from_flag(bool(flags & _native.FLAG_SCALED_NONFINITE))
        grad_norm = 0.0
        if applied:
            grad_norm = float(rec["grad_norm"]) if self.grad_norm_enabled else 0.0
            applied = not (flags & _native.FLAG_GRAD_NONFINITE)
        return StepResult(applied=applied, scale=step_scale, grad_norm=grad_norm, flags=flags,
                          algorithms=sorted({b.algorithm for b in self.buckets}))

    def step(self, grads, step: int) -> StepResult:
        self.enqueue(grads, step)
        return self.finish()

    # ------------------------------------------------------------ state
    def save_checkpoint(self, path, step: int = 0) -> None:
        """LARS v1 checkpoint (lars.py:184-237) straight from the arenas,
        byte-identical to the reference's save_checkpoint of the same groups.
        Sharded: gathers the masters / velocities first (collective: every
        rank calls it; each may write its own file)."""
        from .lars import save_checkpoint
        save_checkpoint(path, self.state_groups(), step)

    def load_checkpoint(self, path) -> int:
        """Restore masters, velocities and working copies from a LARS v1 file
        whose groups match this pipeline (names, kinds, sizes, flag bits);
        returns the checkpoint's step.  Every rank of a sharded pipeline
        loads the whole file."""
        from .lars import read_checkpoint_arrays
        step, groups = read_checkpoint_arrays(path)
        if len(groups) != len(self.specs):
            raise ValueError(f"checkpoint has {len(groups)} groups, pipeline {len(self.specs)}")
        for (name, kind, flags, m, v, w16), s, g in zip(groups, self.specs, self.groups):
            if name != s.name or kind != s.kind or m.size != s.numel:
                raise ValueError(f"checkpoint group {name!r} ({kind}, {m.size}) does not match "
                                 f"{s.name!r} ({s.kind}, {s.numel})")
            if flags != segment_flags(g):
                raise ValueError(f"checkpoint group {name!r}: flag bits {flags} differ from the "
                                 f"pipeline's {segment_flags(g)}")
        for (name, kind, flags, m, v, w16), g in zip(groups, self.groups):
            g.master_w.copy_(torch.from_numpy(m))
            g.velocity.copy_(torch.from_numpy(v))
            g.working_w16.copy_(torch.from_numpy(w16))
        torch.cuda.current_stream(self.device).synchronize()
        self.invalidate_master_cache()
        return step

    # ------------------------------------------------------------ inspection
    def seg_scales(self) -> np.ndarray:
        return dev.to_host(self.plan.seg_scale)[: len(self.specs)]

    def seg_stats(self) -> np.ndarray:
        """(nseg, 4): ||w||, ||eff||, local lr, sum g^2 of the last step."""
        return dev.to_host(self.plan.seg_out).reshape(-1, 4)[: len(self.specs)]
