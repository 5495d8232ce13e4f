"""The fused per-step gradient pipeline of one data-parallel rank.

This composes the reference's step body (experiment.py:368-413) on the fp16
wire that the north star asks for, device-resident:

  1. pack       per-parameter fp16 gradients -> theta-buckets of the wire
                buffer, in enqueue (backward) order; bucket boundaries are
                exactly FusionBuffer's (fusion.py:58-94)       gs_batched_copy
  2. all-reduce every bucket, sum, over NCCL (flat ring / hierarchical /
                sharded), bucket i in flight while bucket i+1 is packed and
                bucket i-1 runs pass 1                          dist.Communicator
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
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dev
from . import _native
from ._plan import LarsPlan, SegmentSpec, step_params
from .fusion import copy_table, plan_buckets
from .halfprec import LossScale
from .lars import LarsConfig, ParamGroup, segment_flags

__all__ = ["ParamSpec", "Bucket", "GradientPipeline", "StepResult", "BUCKET_ALIGN",
           "plan_layout", "shard_buckets"]

#: wire-buffer granularity (elements): bucket starts are 512-byte aligned and
#: padded lengths are multiples of 256 so any k <= 8 shards 16-byte aligned
BUCKET_ALIGN = 256


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

    @property
    def nbytes(self) -> int:
        return 2 * self.length


@dataclass
class StepResult:
    applied: bool
    scale: float               # the loss scale the step was unscaled with
    grad_norm: float           # experiment.py:408-411 (0.0 when not applied)
    flags: int
    algorithms: list = field(default_factory=list)


def _roundup(n: int, a: int) -> int:
    return (n + a - 1) // a * a


def plan_layout(specs, order, threshold_bytes: int):
    """Host-only wire layout: (wire offset per parameter, buckets, total).

    Bucket membership and per-bucket unpack maps are exactly what
    FusionBuffer(threshold) emits for uint16 tensors enqueued in `order`
    (fusion.py:58-94); bucket b starts at a BUCKET_ALIGN-aligned wire offset.
    """
    sizes = [s.numel for s in specs]
    groups_pos = plan_buckets([sizes[i] for i in order], 2, threshold_bytes)
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
        buckets.append(Bucket(start, length, off - start, idxs, tuple(umap)))
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
      comm: dist.Communicator for p > 1 (None = single worker, no collective).
      eta_bytes: hybrid threshold (collectives.py:238-244) on fp16 bucket bytes.
      hier_variant: NCCL variant for hierarchical buckets ("hierarchical" =
        literal master path, "sharded" = RS/AR/AG).
      init_master: flat fp32 initial weights in registration order.
      grad_norm: compute the experiment's grad-norm metric in pass 1.
      local_workers: with comm=None, simulate p workers on this GPU the way
        the reference's in-memory executor does (collectives.py:286-340):
        each worker's gradients are packed into its own wire buffer and every
        bucket is reduced by the ordered pairwise-tree fold kernel
        (gs_fold_f16_tree), bit-identical to allreduce_f16.  enqueue() then
        takes one gradient set per worker.
    """

    def __init__(self, specs, cfg: LarsConfig, *, threshold_bytes: int = 4 << 20,
                 loss_scale: LossScale | None = None, order=None, comm=None,
                 eta_bytes: int = 0, hier_variant: str = "hierarchical",
                 init_master=None, grad_norm: bool = True, device=None,
                 local_workers: int = 1, use_graph: bool = True, fused_pack: bool = True,
                 bulk: bool = False, fuse_trust: bool = False, trust_in_pass2: bool = False,
                 flat_variant: str = "ring", sharded_update: bool = False,
                 fused_collective: bool = True, lazy_wire: bool = True):
        self.specs = [s if isinstance(s, ParamSpec) else ParamSpec(s[0], tuple(s[1]), s[2])
                      for s in specs]
        self.cfg = cfg
        self.loss_scale = loss_scale if loss_scale is not None else LossScale()
        self.comm = comm
        if comm is not None and local_workers != 1:
            raise ValueError("local_workers is only for the single-process (comm=None) mode")
        self.p = comm.topo.p if comm is not None else int(local_workers)
        self.local = comm is None and self.p > 1
        # eta = inf (every bucket hierarchical, the reference's config 1 and
        # netsim.calibrated_eta when ring never wins) is kept as a float
        self.eta_bytes = eta_bytes if eta_bytes == float("inf") else int(eta_bytes)
        self.hier_variant = hier_variant
        self.grad_norm_enabled = grad_norm
        self.device = device or dev.require_cuda()
        n = len(self.specs)
        self.order = list(reversed(range(n))) if order is None else list(order)
        if sorted(self.order) != list(range(n)):
            raise ValueError("order must be a permutation of the parameter indices")
        sizes = [s.numel for s in self.specs]
        self.sizes = sizes

        # ---- wire layout: FusionBuffer boundaries over the enqueue order
        self.wire_off, self.buckets, self.total = plan_layout(self.specs, self.order,
                                                              threshold_bytes)

        d = self.device
        self.sharded = bool(sharded_update)
        # sharded update: reduce-scatter fused with pass 1 and pass 2 fused
        # with the working-weight push (gs_fused.cu) instead of separate
        # collective kernels
        self.fused_collective = bool(fused_collective) and self.sharded and \
            comm is not None and comm.topo.p in (2, 4, 8)
        if self.sharded and (comm is None or comm.topo.p < 2):
            raise ValueError("sharded_update needs a Communicator with p >= 2")
        for b in self.buckets:
            if self.sharded:
                b.algorithm = "sharded-update"
            elif comm is not None:
                b.algorithm = comm.pick(b.nbytes, self.eta_bytes, hier_variant, flat_variant)
            else:
                b.algorithm = "ordered" if self.local else "none"
        # the ordered (bit-exact) collective reads peers' wires over NVLink:
        # the wire then lives in a double-buffered symmetric-memory window
        self.ordered = None
        self.arena = None
        if self.sharded:
            self._init_sharded_arena(comm, d)
        elif comm is not None and any(b.algorithm == "ordered" for b in self.buckets):
            from .dist import OrderedWire
            self.ordered = OrderedWire(comm, self.total, d)
            self.wire = self.ordered.halves[0]
        else:
            self.wire = torch.zeros(self.total, dtype=torch.uint16, device=d)
        self._last_wire = self.wire
        self._half = 0
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
        wb, mb, vb, hb = (t.data_ptr() for t in (self.wire, self.master, self.velocity,
                                                   self.working))
        segs = [SegmentSpec(wb + 2 * self.wire_off[i], mb + 4 * self.wire_off[i],
                            vb + 4 * self.wire_off[i], hb + 2 * self.wire_off[i], sizes[i],
                            segment_flags(self.groups[i])) for i in range(n)]
        if self.sharded:
            self.plan = LarsPlan(segs, d, order=self.order,
                                 partials=self.arena.view("partials", torch.float64),
                                 flagbuf=self.arena.view("flags", torch.int32))
        else:
            self.plan = LarsPlan(segs, d, order=self.order)
        if bulk:
            self.plan.extra_hint &= ~_native.HINT_NO_BULK
        if self.sharded and os.environ.get("GS_RS_STAGE", "0") == "1":
            # A/B switch: gs_rs_pass1 staging each chunk through shared memory
            # with cp.async instead of register loads (same results; slower)
            self.plan.extra_hint |= _native.HINT_RS_STAGE
        self.plan.fuse_trust = fuse_trust
        self.plan.trust_in_pass2 = trust_in_pass2
        begin, count = self.plan.host_segs["chunk_begin"], self.plan.host_segs["chunk_count"]
        c = 0
        for b in self.buckets:
            b.chunk0 = c
            b.nchunk = int(sum(int(count[i]) for i in b.params))
            if b.nchunk:
                assert int(begin[b.params[0]]) == c or sizes[b.params[0]] == 0
            c += b.nchunk
        assert c == self.plan.nchunk
        if self.sharded:
            self._init_ownership(d)

        self._pack_cache: dict = {}
        self.use_graph = use_graph
        self._graphs: dict = {}
        # p = 1: pass 1 reads the gradients where they lie and writes the wire
        # copy itself (gs_segment.gcopy), so packing costs no extra launch and
        # no re-read of the wire
        self.fused_pack = fused_pack and comm is None and not self.local
        #: p = 1: no collective consumes the fused batches, so the wire copy is
        #: written only when bucket_payload() asks for it (saves 2 B/element
        #: of HBM writes per step); lazy_wire=False restores pass 1's copy
        self.lazy_wire = bool(lazy_wire) and self.fused_pack
        self._wire_src = None
        self._prepared = None
        self._src_cache: dict = {}
        self._grad_arena = None
        self._pack_stream = torch.cuda.Stream(device=d) if comm is not None else None
        if self.local:
            self.rank_wire = [torch.zeros(self.total, dtype=torch.uint16, device=d)
                              for _ in range(self.p)]
            self._slots = dev.upload(np.array([t.data_ptr() for t in self.rank_wire],
                                              dtype=np.uint64), d)
        self._result_host = torch.zeros(2, dtype=torch.float64).pin_memory()
        self._flags_host = torch.zeros(1, dtype=torch.int32).pin_memory()

    # ------------------------------------------------------------ sharded
    def _init_sharded_arena(self, comm, d) -> None:
        """ZeRO-1 layout: one symmetric window holding both wire halves, the
        binary16 working weights, the masters, the velocities, the chunk
        partials and the step flags, so every peer can reach them."""
        from ._plan import build_chunks
        from .dist import SymmetricArena

        p = comm.topo.p
        #: whole-step reduce-scatter form: "pull" (pack locally, the owner
        #: loads its peers' shares over NVLink) or "inbox" (the packer stores
        #: each owner's share straight into its inbox over NVLink, the fold
        #: reads local memory); measured equal within noise, pull is default
        self.rs_mode = os.environ.get("GS_RS_MODE", "pull")
        if self.rs_mode not in ("pull", "inbox"):
            raise ValueError(f"GS_RS_MODE must be 'pull' or 'inbox', got {self.rs_mode!r}")
        chunks, _, _ = build_chunks(self.sizes, self.order)
        self._host_chunks = chunks
        nchunk = len(chunks)
        sms = torch.cuda.get_device_properties(d).multi_processor_count
        # grid of the peer-synchronised kernels (each clamps to what is
        # co-resident: 4 CTAs per SM for gs_rs_pass1 at p = 2 / 4)
        self._nblocks = 4 * sms
        regions = {
            "wireA": 2 * self.total, "wireB": 2 * self.total, "working": 2 * self.total,
            "master": 4 * self.total, "velocity": 4 * self.total,
            "partials": 8 * max(1, 3 * nchunk), "flags": 4 * (4 + len(self.specs) + 1),
            # inbox form of the reduce-scatter: p wire-shaped slots, slot q
            # receives rank q's raw values of this rank's slices
            "inbox": 2 * self.total * p if self.rs_mode == "inbox" else 0,
        }
        self.arena = SymmetricArena(comm, regions, d, sig_words=2 * self._nblocks * p)
        a = self.arena
        self.wire = a.view("wireA", torch.uint16)
        self._halves = (a.view("wireA", torch.uint16), a.view("wireB", torch.uint16))
        self.master = a.view("master", torch.float32)
        self.velocity = a.view("velocity", torch.float32)
        self.working = a.view("working", torch.uint16)
        self.epoch_base = torch.zeros(1, dtype=torch.int32, device=d)
        self._ps_events = None

    def _init_ownership(self, d) -> None:
        """Sharded update: which chunks this rank folds and updates (needs
        the buckets' chunk ranges, i.e. runs after the LARS plan is built)."""
        p = self.comm.topo.p
        chunks = self._host_chunks
        # ownership, PER BUCKET: rank r owns chunks [C_b[r], C_b[r+1]) of bucket
        # b (balanced by elements, in wire order) = wire elements [E_b[r],
        # E_b[r+1]); every bucket's fold is spread over all ranks, so the
        # bucket pipeline never waits on one rank's share
        abs_start = np.array([self.wire_off[int(c["seg"])] + int(c["start"]) for c in chunks],
                             dtype=np.int64)
        clen = np.array([int(c["len"]) for c in chunks], dtype=np.int64)
        r = self.comm.rank
        self._bucket_C, self._bucket_E = shard_buckets(self.buckets, abs_start, p)
        self._own_bucket = [(C[r], C[r + 1]) for C in self._bucket_C]
        self._rs_bounds, self._part_bounds, self._w16_bounds, self._m_bounds = [], [], [], []
        own_list = []
        for C, E in zip(self._bucket_C, self._bucket_E):
            own_list.extend(range(C[r], C[r + 1]))
            self._rs_bounds.append(dev.upload(np.array(E, dtype=np.int64), d))
            self._part_bounds.append(dev.upload(np.array([24 * c for c in C], dtype=np.int64), d))
            self._w16_bounds.append(dev.upload(np.array([2 * e for e in E], dtype=np.int64), d))
            self._m_bounds.append(dev.upload(np.array([4 * e for e in E], dtype=np.int64), d))
        self._own_list = dev.upload(np.array(own_list or [0], dtype=np.int32), d)
        self._n_own = len(own_list)
        #: elements this rank updates (pass 2) per step
        self.owned_elems = int(clen[own_list].sum()) if own_list else 0
        ib = self.arena.bases[r] + self.arena.offsets["inbox"]
        self._inbox_src = dev.upload(np.array([ib + 2 * self.total * q for q in range(p)],
                                              dtype=np.uint64), d)
        #: NVLS multicast address of the working arena (GS_MULTICAST=1): pass 2
        #: then pushes each updated binary16 vector to every rank with ONE
        #: store.  Off by default: the all-gather is bound by each rank's
        #: INBOUND traffic, (p-1)/p of the arena either way, and the multicast
        #: stores measured slower (p=4: pass2_push 87 vs 73 us, r01p)
        self._mc_working = self.arena.multicast("working") \
            if os.environ.get("GS_MULTICAST", "0") == "1" else None

    def gather_state(self) -> None:
        """Make the sharded masters and velocities whole on every rank (for
        inspection / checkpoints; the step itself only keeps the working
        copy replicated, ZeRO-1)."""
        if not self.sharded:
            return
        sh = int(torch.cuda.current_stream(self.device).cuda_stream)
        p, r = self.comm.topo.p, self.comm.rank
        nb = len(self.buckets)
        for name in ("master", "velocity"):
            for b in range(nb):
                _native.call("gs_ordered_allgather", dev.ptr(self.arena.peers(name)),
                             dev.ptr(self.arena.peers("sig")), r, p, dev.ptr(self._m_bounds[b]),
                             b + 1, dev.ptr(self.epoch_base), self._nblocks, sh)
            _native.call("gs_counter_add", dev.ptr(self.epoch_base), nb, sh)

    def _launch_sharded(self, tabs, s0, timer) -> None:
        """reduce-scatter (own slice, reference tree order) -> pass 1 on own
        chunks -> all-gather of the chunk partials -> trust (flags OR-ed over
        ranks) -> pass 2 on own chunks -> all-gather of the working weights."""
        plan, a = self.plan, self.arena
        sh = int(s0.cuda_stream)
        p, r = self.comm.topo.p, self.comm.rank
        half = self._half
        wire = self._halves[half]
        ptabs = tabs[half]
        wb = wire.data_ptr()
        plan.use_segments(plan.alt_segments([wb + 2 * o for o in self.wire_off]))
        plan.reset_flags(sh)
        sig, ebase = dev.ptr(a.peers("sig")), dev.ptr(self.epoch_base)
        wires = a.peers("wireA" if half == 0 else "wireB")
        nb = len(self.buckets)
        if self.fused_collective:
            # one reduce-scatter launch follows all packs: pack every bucket
            # with one launch on the compute stream
            if timer:
                timer("pack")
            if self.rs_mode == "inbox":
                self._pack([tabs[2]], 0, sh)  # owners' shares straight into their inboxes
            else:
                self._pack(ptabs, nb, sh)
            self._launch_sharded_fused(s0, sh, sig, ebase, wires, timer, wire)
            self._last_wire = wire
            self._half ^= 1
            plan.use_segments(None)
            return
        ps = self._pack_stream
        ps.wait_stream(s0)
        evs = []
        for b in range(nb):
            with torch.cuda.stream(ps):
                self._pack(ptabs, b, int(ps.cuda_stream))
                ev = torch.cuda.Event()
                ev.record(ps)
                evs.append(ev)
        for b in range(nb):
            s0.wait_event(evs[b])
            if timer:
                timer(f"rs{b}")
            _native.call("gs_ordered_reduce_scatter_f16", dev.ptr(wires), sig, r, p,
                         dev.ptr(self._rs_bounds[b]), b + 1, ebase, self._nblocks, None, sh)
            c0, c1 = self._own_bucket[b]
            if timer:
                timer(f"pass1_{b}")
            if c1 > c0:
                plan.pass1(sh, g_is_f16=True, chunk0=c0, nchunk=c1 - c0)
        s0.wait_stream(ps)
        if timer:
            timer("gather_partials")
        for b in range(nb):
            _native.call("gs_ordered_allgather", dev.ptr(a.peers("partials")), sig, r, p,
                         dev.ptr(self._part_bounds[b]), nb + 1 + b, ebase, self._nblocks, sh)
        if timer:
            timer("trust")
        plan.trust(sh, peer_flags=a.peers("flags"), npeers=p)
        if timer:
            timer("pass2")
        mask = _native.FLAG_SCALED_NONFINITE | _native.FLAG_GRAD_NONFINITE
        for b in range(nb):
            c0, c1 = self._own_bucket[b]
            if c1 > c0:
                plan.pass2(sh, g_is_f16=True, flag_mask=mask, chunk0=c0, nchunk=c1 - c0)
        if timer:
            timer("gather_w16")
        for b in range(nb):
            _native.call("gs_ordered_allgather", dev.ptr(a.peers("working")), sig, r, p,
                         dev.ptr(self._w16_bounds[b]), 2 * nb + 1 + b, ebase, self._nblocks, sh)
        _native.call("gs_counter_add", ebase, 3 * nb + 1, sh)
        plan.use_segments(None)
        self._last_wire = wire
        self._half ^= 1
        if timer:
            timer("end")

    def _launch_sharded_fused(self, s0, sh, sig, ebase, wires, timer, wire) -> None:
        """The sharded step in fused kernels, after the pack: one gs_rs_pass1
        over the rank's owned chunks of every bucket (reduce-scatter + pass 1,
        partials and flags pushed to every peer), a one-CTA peer fence, trust,
        gs_pass2_push (pass 2 + working-weight push to every peer), and a
        closing fence."""
        plan, a = self.plan, self.arena
        p, r = self.comm.topo.p, self.comm.rank
        parts, flags = dev.ptr(a.peers("partials")), dev.ptr(a.peers("flags"))
        # every gradient is already resident: ONE reduce-scatter + pass 1 launch
        # over the rank's owned chunks of all buckets (one entry barrier, one
        # NVLink ramp-up) instead of one per bucket -- per-bucket launches each
        # paid ~20 us of barrier and ramp latency (tools/rs_probe.py); the
        # per-bucket form is the incremental API's (submit / overlap.py)
        if timer:
            timer("rs_pass1")
        inbox = self.rs_mode == "inbox"
        _native.call("gs_rs_pass1", dev.ptr(self._inbox_src if inbox else wires),
                     wire.data_ptr() if inbox else None, sig, r, p, dev.ptr(plan.d_segs),
                     dev.ptr(plan.d_chunks), 0, self._n_own, dev.ptr(self._own_list),
                     dev.ptr(plan.params), plan.hint, parts, flags, 1, ebase, self._nblocks, sh)
        if timer:
            timer("fence")
        _native.call("gs_peer_fence", sig, r, p, 2, ebase, sh)
        if timer:
            timer("trust")
        plan.trust(sh)
        if timer:
            timer("pass2_push")
        mask = _native.FLAG_SCALED_NONFINITE | _native.FLAG_GRAD_NONFINITE
        _native.call("gs_pass2_push", dev.ptr(plan.d_segs), dev.ptr(plan.d_chunks), 0,
                     self._n_own, dev.ptr(self._own_list), dev.ptr(plan.params), plan.hint,
                     dev.ptr(plan.seg_scale), dev.ptr(plan.flags), mask,
                     dev.ptr(a.peers("working")), p, r, self._mc_working, sh)
        if timer:
            timer("fence_end")
        _native.call("gs_peer_fence", sig, r, p, 3, ebase, sh)
        _native.call("gs_counter_add", ebase, 4, sh)
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

    def registration_view(self, arena: torch.Tensor) -> torch.Tensor:
        """Gather an arena (wire layout) into registration order (host checks)."""
        return torch.cat([arena[self.wire_off[i]:self.wire_off[i] + n]
                          for i, n in enumerate(self.sizes)])

    def bucket_payload(self, b: int) -> torch.Tensor:
        """Bucket b of the last step's wire (the reference's FusedBatch
        payload, fusion.py:84-90); at p = 1 with the lazy wire it is packed
        from the last step's gradients on first request."""
        src = getattr(self, "_wire_src", None)
        if src is not None:
            tabs = self._tables_for(src, self.wire)
            self._pack(tabs, len(self.buckets), int(torch.cuda.current_stream(self.device).cuda_stream))
            self._wire_src = None
        bk = self.buckets[b]
        return self._last_wire[bk.start:bk.start + bk.length]

    # ------------------------------------------------------------ packing
    def grad_arena(self) -> torch.Tensor:
        """A device fp16 (uint16) gradient arena in registration order that a
        backward pass (or a host copy) can write into; step() accepts it."""
        if self._grad_arena is None:
            self._grad_arena = torch.zeros(sum(self.sizes), dtype=torch.uint16, device=self.device)
        return self._grad_arena

    def _grad_views(self, grads):
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

    def _tables_for(self, views, dst: torch.Tensor):
        """Per-bucket gs_copy tables packing `views` into `dst` (cached)."""
        key = (dst.data_ptr(),) + tuple((t.data_ptr(), t.numel()) for t in views)
        tabs = self._pack_cache.get(key)
        if tabs is None:
            for t, n in zip(views, self.sizes):
                if t.numel() != n or t.dtype not in (torch.uint16, torch.float16) or not t.is_cuda:
                    raise ValueError("gradients must be CUDA fp16/uint16 tensors of the "
                                     "parameter sizes")
            wb = dst.data_ptr()
            tabs, host = [], []
            for b in self.buckets:
                t = copy_table((views[i].data_ptr(), wb + 2 * self.wire_off[i], 2 * self.sizes[i])
                               for i in b.params if self.sizes[i])
                tabs.append((dev.upload(t, self.device), len(t)))
                host.append(t)
            # entry len(buckets): every bucket in one table (one launch when all
            # gradients are packed before the first collective)
            allt = np.concatenate(host) if host else copy_table([])
            tabs.append((dev.upload(allt, self.device), len(allt)))
            if len(self._pack_cache) > 8:
                self._pack_cache.clear()
                self._graphs.clear()
            self._pack_cache[key] = tabs
        return tabs

    def _inbox_table(self, views):
        """One gs_copy table storing this rank's gradients straight into the
        owners' inboxes (slot = this rank), split at the per-bucket ownership
        bounds; cached on the gradient addresses."""
        key = ("inbox",) + tuple((t.data_ptr(), t.numel()) for t in views)
        tab = self._pack_cache.get(key)
        if tab is None:
            p, r = self.comm.topo.p, self.comm.rank
            off = self.arena.offsets["inbox"]
            slot = [self.arena.bases[q] + off + 2 * self.total * r for q in range(p)]
            bucket_of = {}
            for b, bk in enumerate(self.buckets):
                for i in bk.params:
                    bucket_of[i] = b
            pairs = []
            for i, t in enumerate(views):
                n = self.sizes[i]
                if not n:
                    continue
                wo = self.wire_off[i]
                E = self._bucket_E[bucket_of[i]]
                for q in range(p):
                    lo, hi = max(wo, E[q]), min(wo + n, E[q + 1])
                    if lo < hi:
                        pairs.append((t.data_ptr() + 2 * (lo - wo), slot[q] + 2 * lo, 2 * (hi - lo)))
            host = copy_table(pairs)
            tab = (dev.upload(host, self.device), len(host))
            if len(self._pack_cache) > 8:
                self._pack_cache.clear()
                self._graphs.clear()
            self._pack_cache[key] = tab
        return tab

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
        """Host-only part of a step (schedule, loss scale, launch hint) so the
        device part can be enqueued without host work in between."""
        self.plan.stage_params(self.params_for(step), g_is_f16=True)
        self._prepared = step

    def _sources(self, grads):
        """(launch tables, graph key) for this gradient set, cached on the
        buffer addresses so a steady-state step does no per-tensor host work."""
        if dev.is_tensor(grads):
            ck = (grads.data_ptr(), grads.numel(), grads.dtype)
        else:
            ck = tuple((g.data_ptr(), g.numel()) if dev.is_tensor(g) else id(g) for g in grads)
        hit = self._src_cache.get(ck)
        if hit is not None:
            return hit
        res = self._sources_uncached(grads)
        if len(self._src_cache) > 16:
            self._src_cache.clear()
        self._src_cache[ck] = res
        return res

    def _sources_uncached(self, grads):
        if self.local:
            if len(grads) != self.p:
                raise ValueError(f"expected gradients of {self.p} workers, got {len(grads)}")
            tabs = [self._tables_for(self._grad_views(g), w) for g, w in zip(grads, self.rank_wire)]
            return tabs, tuple(id(t) for t in tabs)
        views = self._grad_views(grads)
        if self.fused_pack:
            for t, n in zip(views, self.sizes):
                if t.numel() != n or t.dtype not in (torch.uint16, torch.float16) or not t.is_cuda:
                    raise ValueError("gradients must be CUDA fp16/uint16 tensors of the "
                                     "parameter sizes")
            wb = self.wire.data_ptr()
            # lazy wire (default): with no collective to feed, pass 1 and
            # pass 2 read the gradients where they lie and the fused batches
            # are only materialised when asked for (bucket_payload); eager:
            # pass 1 also writes the wire copy (gs_segment.gcopy)
            tab = self.plan.alt_segments([t.data_ptr() for t in views],
                                         None if self.lazy_wire else
                                         [wb + 2 * o for o in self.wire_off])
            return ("fused", tab, views), id(tab)
        if self.ordered is not None:
            tabs = tuple(self._tables_for(views, h) for h in self.ordered.halves)
            return tabs, tuple(id(t) for t in tabs)
        if self.sharded:
            tabs = tuple(self._tables_for(views, h) for h in self._halves)
            if self.fused_collective and self.rs_mode == "inbox":
                tabs = tabs + (self._inbox_table(views),)
            return tabs, tuple(id(t) for t in tabs)
        tabs = self._tables_for(views, self.wire)
        return tabs, id(tabs)

    def _half_segments(self, half: int):
        """Segment table whose gradient pointers address wire half `half`."""
        wb = self.ordered.halves[half].data_ptr()
        return self.plan.alt_segments([wb + 2 * o for o in self.wire_off])

    def enqueue(self, grads, step: int, timer=None) -> None:
        """Launch one step on the current stream (no host sync).

        `timer`, if given, is called with a phase name before each phase
        (the bench records CUDA events there); timed launches run eagerly.
        Otherwise, with comm=None and use_graph, the kernel sequence is
        captured once per (gradient-buffer set, launch hint) into a CUDA graph
        and replayed: the per-step scalars live in device memory
        (gs_step_params), so a replay picks up the new loss scale / rate.
        """
        s0 = torch.cuda.current_stream(self.device)
        if self._prepared != step:
            self.prepare(step)
        self._prepared = None
        tabs, key = self._sources(grads)
        if self.lazy_wire:
            self._wire_src = tabs[2]  # bucket_payload() packs these on demand
        key = (key, self.plan.hint, self._half)
        self.plan.upload_params(s0)
        # graph replay needs every kernel of the step to be ours: comm = None,
        # or only ordered (symmetric-memory) buckets, whose epochs live on
        # the device (NCCL buckets run eagerly)
        graphable = self.comm is None or self.sharded or \
            all(b.algorithm == "ordered" for b in self.buckets)
        if timer is not None or not self.use_graph or not graphable:
            self._launch(tabs, s0, timer)
            return
        entry = self._graphs.get(key)
        if entry is None:
            # first sight of these buffers: run eagerly (warms every kernel),
            # capture on the next call
            self._graphs[key] = "warm"
            self._launch(tabs, s0, None)
            return
        if entry == "warm":
            g = torch.cuda.CUDAGraph()
            n0 = _native.launch_count
            half = self._half
            with torch.cuda.graph(g):
                self._launch(tabs, torch.cuda.current_stream(self.device), None)
            self._half = half  # capture executes nothing: the replay below does
            entry = (g, _native.launch_count - n0)
            _native.launch_count = n0
            self._graphs[key] = entry
        g, nk = entry
        g.replay()
        _native.launch_count += nk
        if self.ordered is not None:
            self._last_wire = self.ordered.halves[self._half]
            self._half ^= 1
        elif self.sharded:
            self._last_wire = self._halves[self._half]
            self._half ^= 1

    def _launch(self, tabs, s0, timer) -> None:
        if self.sharded:
            self._launch_sharded(tabs, s0, timer)
            return
        plan = self.plan
        sh = int(s0.cuda_stream)
        fused = isinstance(tabs, tuple) and tabs[0] == "fused"
        plan.use_segments(tabs[1] if fused else None)
        plan.reset_flags(sh)
        if fused:
            if timer:
                timer("pass1")
            plan.pass1(sh, g_is_f16=True)
        elif self.comm is None:
            if timer:
                timer("pack")
            for b in range(len(self.buckets)):
                if self.local:
                    for t in tabs:
                        self._pack(t, b, sh)
                else:
                    self._pack(tabs, b, sh)
            if self.local:
                if timer:
                    timer("fold")
                wb = self.wire.data_ptr()
                for bk in self.buckets:
                    if bk.length:
                        _native.call("gs_fold_f16_tree", dev.ptr(self._slots), self.p, bk.start,
                                     wb + 2 * bk.start, bk.length, None, sh)
            if timer:
                timer("pass1")
            plan.pass1(sh, g_is_f16=True)
        else:
            # bucket b+1 is packed (pack stream) while bucket b's all-reduce is
            # in flight and bucket b-1 runs pass 1 (compute stream)
            ps = self._pack_stream
            ps.wait_stream(s0)
            half = self._half
            wire = self.ordered.halves[half] if self.ordered is not None else self.wire
            ptabs = tabs[half] if self.ordered is not None else tabs
            if self.ordered is not None:
                plan.use_segments(self._half_segments(half))
            works = []
            for b, bk in enumerate(self.buckets):
                with torch.cuda.stream(ps):
                    self._pack(ptabs, b, int(ps.cuda_stream))
                    payload = wire[bk.start:bk.start + bk.padded]
                    if bk.algorithm == "ring":
                        works.append(self.comm.allreduce_ring(payload, async_op=True))
                    else:
                        if bk.algorithm != "ordered":
                            self.comm.allreduce(payload, bk.algorithm)
                        ev = torch.cuda.Event()
                        ev.record(ps)
                        works.append(ev)
            for b, bk in enumerate(self.buckets):
                w = works[b]
                if isinstance(w, torch.cuda.Event):
                    s0.wait_event(w)
                else:
                    w.wait()
                if bk.algorithm == "ordered":
                    self.ordered.allreduce(half, bk.start, bk.length, sh, slot=b)
                plan.pass1(sh, g_is_f16=True, chunk0=bk.chunk0, nchunk=bk.nchunk)
            s0.wait_stream(ps)
            if self.ordered is not None:
                self.ordered.advance(len(self.buckets) + 1, sh)
            self._last_wire = wire
            if self.ordered is not None:
                self._half ^= 1
        mask = _native.FLAG_SCALED_NONFINITE | _native.FLAG_GRAD_NONFINITE
        if plan.trust_via_pass2:
            if timer:
                timer("pass2")
            plan.pass2(sh, g_is_f16=True, flag_mask=mask, trust=True)
        else:
            if timer:
                timer("trust")
            if not plan.fused:
                plan.trust(sh)
            if timer:
                timer("pass2")
            plan.pass2(sh, g_is_f16=True, flag_mask=mask)
        plan.use_segments(None)
        if timer:
            timer("end")

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
        """One step from a pinned host fp16 gradient (registration order): the
        host->device copy is split per bucket on a copy stream and pass 1 of
        bucket b starts as soon as bucket b has landed, so the PCIe transfer
        overlaps the update (p = 1, fused packer); otherwise one copy then
        the regular step."""
        arena = self.grad_arena()
        s0 = torch.cuda.current_stream(self.device)
        # p > 1: per-bucket H2D + incremental submission is available but
        # measured slower than one copy + the whole (graph-replayed) step
        # (p=2: 1.36 vs 1.21 ms, same box A/B, profiles/r01r_n2_host_ab.md)
        if self.comm is not None and (self.fused_collective or not self.sharded) and \
                os.environ.get("GS_HOST_INCREMENTAL", "0") == "1":
            ranges = self._bucket_host_ranges()
            if ranges is not None:
                self._enqueue_host_incremental(host_flat, arena, ranges, step)
                return
        ranges = self._bucket_host_ranges() if self.fused_pack else None
        if ranges is None:
            arena.copy_(host_flat.reshape(-1), non_blocking=True)
            self.enqueue(arena, step)
            return
        if self._prepared != step:
            self.prepare(step)
        self._prepared = None
        tabs, _ = self._sources(arena)
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
        plan.upload_params(s0)
        plan.use_segments(tabs[1])
        if self.lazy_wire:
            self._wire_src = tabs[2]
        plan.reset_flags(sh)
        for bk, ev in zip(self.buckets, evs):
            s0.wait_event(ev)
            plan.pass1(sh, g_is_f16=True, chunk0=bk.chunk0, nchunk=bk.nchunk)
        mask = _native.FLAG_SCALED_NONFINITE | _native.FLAG_GRAD_NONFINITE
        plan.finish(sh, True, mask)
        plan.use_segments(None)
        self._last_wire = self.wire

    # ------------------------------------------------------------ incremental
    # The step split at bucket granularity, for a backward pass that hands
    # gradients over as they are produced (overlap.py): bucket b
    # is packed, reduced and run through pass 1 on a side stream as soon as
    # its last gradient exists, while the backward pass keeps computing.
    def begin(self, step: int) -> None:
        """Open a step: stage the scalars, reset the flags (current stream)."""
        if self.local:
            raise ValueError("incremental steps need one gradient set per rank "
                             "(local_workers > 1 takes whole gradient sets)")
        if self.sharded and not self.fused_collective:
            raise ValueError("incremental sharded steps use the fused kernels (p in 2, 4, 8)")
        s0 = torch.cuda.current_stream(self.device)
        if self._prepared != step:
            self.prepare(step)
        self._prepared = None
        plan = self.plan
        plan.upload_params(s0)
        sh = int(s0.cuda_stream)
        half = self._half
        if self.sharded:
            wire = self._halves[half]
            plan.use_segments(plan.alt_segments([wire.data_ptr() + 2 * o for o in self.wire_off]))
        elif self.ordered is not None:
            wire = self.ordered.halves[half]
            plan.use_segments(self._half_segments(half))
        else:
            wire = self.wire
            plan.use_segments(None)
        plan.reset_flags(sh)
        if getattr(self, "_side_stream", None) is None:
            self._side_stream = torch.cuda.Stream(device=self.device)
        ss = self._side_stream
        ss.wait_stream(s0)
        self._inc = {"step": step, "half": half, "wire": wire, "next": 0,
                     "ready": [None] * len(self.buckets)}

    def submit(self, b: int, grads) -> None:
        """Bucket b's gradients (tensors of its parameters, in `buckets[b].params`
        order, fp16/uint16, on this device) are complete on the current stream.
        Buckets launch strictly in bucket order (every rank issues the same
        collective sequence), each as soon as it and all earlier ones are in."""
        inc = getattr(self, "_inc", None)
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
            if t.numel() != self.sizes[i] or t.dtype not in (torch.uint16, torch.float16) \
                    or not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"gradient of {self.specs[i].name!r} must be a contiguous CUDA "
                                 f"fp16 tensor of {self.sizes[i]} elements")
            if self.sizes[i]:
                pairs.append((t.data_ptr(), wb + 2 * self.wire_off[i], 2 * self.sizes[i]))
        key = ("inc", b, wb) + tuple(p[0] for p in pairs)
        tab = self._pack_cache.get(key)
        if tab is None:
            t = copy_table(pairs)
            if len(self._pack_cache) > 64:
                self._pack_cache.clear()
                self._graphs.clear()
            tab = self._pack_cache[key] = (dev.upload(t, self.device), len(t))
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        for t in grads:
            t.record_stream(self._side_stream)  # read there; keep the allocator off it
        inc["ready"][b] = (tab, ev, grads)
        while inc["next"] < len(self.buckets) and inc["ready"][inc["next"]] is not None:
            self._launch_bucket(inc["next"])
            inc["next"] += 1

    def _launch_bucket(self, b: int) -> None:
        inc = self._inc
        tab, ev, _ = inc["ready"][b]
        bk, plan, ss = self.buckets[b], self.plan, self._side_stream
        ss.wait_event(ev)
        sh = int(ss.cuda_stream)
        with torch.cuda.stream(ss):
            if tab[1]:
                _native.call("gs_batched_copy", dev.ptr(tab[0]), tab[1], sh)
            if self.sharded:
                p, r = self.comm.topo.p, self.comm.rank
                c0, c1 = self._own_bucket[b]
                wires = self.arena.peers("wireA" if inc["half"] == 0 else "wireB")
                _native.call("gs_rs_pass1", dev.ptr(wires), None, dev.ptr(self.arena.peers("sig")), r,
                             p, dev.ptr(plan.d_segs), dev.ptr(plan.d_chunks), c0, c1, None,
                             dev.ptr(plan.params), plan.hint, dev.ptr(self.arena.peers("partials")),
                             dev.ptr(self.arena.peers("flags")), b + 1, dev.ptr(self.epoch_base),
                             self._nblocks, sh)
                return
            if bk.algorithm == "ordered":
                self.ordered.allreduce(inc["half"], bk.start, bk.length, sh, slot=b)
            elif bk.algorithm != "none":
                self.comm.allreduce(inc["wire"][bk.start:bk.start + bk.padded], bk.algorithm)
            if bk.nchunk:
                plan.pass1(sh, g_is_f16=True, chunk0=bk.chunk0, nchunk=bk.nchunk)

    def end(self) -> None:
        """Close the step: every bucket must have been submitted; trust and
        pass 2 run on the current stream after the side stream's work."""
        inc = getattr(self, "_inc", None)
        if inc is None:
            raise RuntimeError("end() without begin()")
        missing = [b for b, r in enumerate(inc["ready"]) if r is None]
        if missing:
            names = [self.specs[i].name for i in self.buckets[missing[0]].params]
            raise RuntimeError(f"step ended with {len(missing)} bucket(s) never submitted "
                               f"(first: bucket {missing[0]}, tensors {names[:4]}...)")
        s0 = torch.cuda.current_stream(self.device)
        s0.wait_stream(self._side_stream)
        sh = int(s0.cuda_stream)
        plan = self.plan
        mask = _native.FLAG_SCALED_NONFINITE | _native.FLAG_GRAD_NONFINITE
        nb = len(self.buckets)
        if self.sharded:
            p, r = self.comm.topo.p, self.comm.rank
            sig, ebase = dev.ptr(self.arena.peers("sig")), dev.ptr(self.epoch_base)
            _native.call("gs_peer_fence", sig, r, p, nb + 1, ebase, sh)
            plan.trust(sh)
            _native.call("gs_pass2_push", dev.ptr(plan.d_segs), dev.ptr(plan.d_chunks), 0,
                         self._n_own, dev.ptr(self._own_list), dev.ptr(plan.params), plan.hint,
                         dev.ptr(plan.seg_scale), dev.ptr(plan.flags), mask,
                         dev.ptr(self.arena.peers("working")), p, r, self._mc_working, sh)
            _native.call("gs_peer_fence", sig, r, p, nb + 2, ebase, sh)
            _native.call("gs_counter_add", ebase, nb + 3, sh)
            self._half ^= 1
        else:
            plan.finish(sh, True, mask)
            if self.ordered is not None:
                self.ordered.advance(nb + 1, sh)
                self._half ^= 1
        plan.use_segments(None)
        self._last_wire = inc["wire"]
        self._inc = None

    def _enqueue_host_incremental(self, host_flat, arena, ranges, step: int) -> None:
        """p > 1 from host gradients: bucket b's host->device copy runs on a
        copy stream and the bucket is submitted (pack + collective + pass 1,
        the incremental API) as soon as it has landed, so the PCIe transfer
        of the later buckets hides the earlier buckets' reduction."""
        s0 = torch.cuda.current_stream(self.device)
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream(device=self.device)
        cs = self._copy_stream
        cs.wait_stream(s0)
        src = host_flat.reshape(-1)
        views = self._grad_views(arena)
        evs = []
        with torch.cuda.stream(cs):
            for lo, hi in ranges:
                arena[lo:hi].copy_(src[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
                evs.append(ev)
        self.begin(step)
        for b, ev in enumerate(evs):
            s0.wait_event(ev)
            self.submit(b, [views[i] for i in self.buckets[b].params])
        self.end()

    def finish(self) -> StepResult:
        """Read the step's flags (the one host sync) and advance LossScale
        exactly as experiment.py:403-413 does."""
        self._flags_host.copy_(self.plan.flags, non_blocking=True)
        self._result_host[0:1].copy_(self.plan.grad_norm, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        flags = int(self._flags_host.item())
        step_scale = self.loss_scale.scale
        applied = self.loss_scale.update_from_flag(bool(flags & _native.FLAG_SCALED_NONFINITE))
        grad_norm = 0.0
        if applied:
            grad_norm = float(self._result_host[0].item()) if self.grad_norm_enabled else 0.0
            applied = not (flags & _native.FLAG_GRAD_NONFINITE)
        return StepResult(applied=applied, scale=step_scale, grad_norm=grad_norm, flags=flags,
                          algorithms=sorted({b.algorithm for b in self.buckets}))

    def step(self, grads, step: int) -> StepResult:
        self.enqueue(grads, step)
        return self.finish()

    # ------------------------------------------------------------ inspection
    def seg_scales(self) -> np.ndarray:
        return dev.to_host(self.plan.seg_scale)[: len(self.specs)]

    def seg_stats(self) -> np.ndarray:
        """(nseg, 4): ||w||, ||eff||, local lr, sum g^2 of the last step."""
        return dev.to_host(self.plan.seg_out).reshape(-1, 4)[: len(self.specs)]
