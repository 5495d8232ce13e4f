"""The multi-rank (NVLink) kernels at p = 2 / 4 / 8 on ONE GPU, bit-exact
against the oracle.

emulation.LocalWorld gives every rank its own arena in this device's memory
and launches each peer-synchronised kernel once for all ranks (CTA b serves
rank b / nb), so the cross-rank barriers, the peer loads / remote stores and
the fused reduce-scatter + LARS kernels run exactly as on an 8-GPU box — only
the transport is local memory.  Reference semantics: fold_f16_tree
(collectives.py:273-283), allreduce_f16 (collectives.py:322-340), the step
composition of SURVEY.md §8a-14 (experiment.py:368-413 on the fp16 wire).
"""

import numpy as np
import pytest
import torch

from oracle import reference_port as rp
import paper_1807_11205_b200 as gs
from paper_1807_11205_b200 import _device as dev
from paper_1807_11205_b200 import _native, shapes as sh
from paper_1807_11205_b200._peer import PeerOp, PeerTimeoutError, launch, rank_ctx
from paper_1807_11205_b200.dist import OrderedWire
from paper_1807_11205_b200.emulation import LocalWorld

pytestmark = pytest.mark.gpu


def split(flat, specs):
    out, o = [], 0
    for s in specs:
        out.append(flat[o:o + s.numel])
        o += s.numel
    return out


def random_f16(rng, n, special=True):
    """binary16 patterns: mostly finite values of mixed magnitude, plus
    subnormals, near-overflow values and (optionally) Inf / NaN."""
    if n == 0:
        return np.zeros(0, np.uint16)
    x = (rng.standard_normal(n) * np.exp2(rng.integers(-20, 12, n))).astype(np.float16)
    h = x.view(np.uint16).copy()
    h[rng.integers(0, n, max(1, n // 97))] = rng.integers(1, 0x400, max(1, n // 97))  # subnormal
    h[rng.integers(0, n, max(1, n // 131))] = 0x7BFF  # 65504: sums overflow
    if special:
        h[rng.integers(0, n, 2)] = 0x7C00
        h[rng.integers(0, n, 1)] = 0xFE01  # a NaN with payload
    return h


# ---------------------------------------------------------------- collectives
@pytest.mark.parametrize("p", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("form", ["pull", "push", "oneshot", "ll"])
def test_ordered_allreduce_bit_exact(p, form, monkeypatch):
    """gs_ordered_allreduce_f16 (pull and push forms) and
    the small-bucket gs_oneshot_allreduce_f16 == fold_f16_tree on every
    rank, incl. ragged lengths, an unaligned bucket offset, Inf/NaN and
    pairwise overflow; the one-shot calls alternate their inbox parity."""
    d = dev.require_cuda()
    world = LocalWorld(gs.Topology(p, 1), d, peer_ctas=8, timeout_s=20.0)
    total = 1 << 16
    push = form == "push"
    if form == "pull":
        # keep the pull kernel on every bucket (no size rule)
        monkeypatch.setattr(OrderedWire, "PUSH_MAX_BYTES", 0)
    wires = [c.make_ordered_wire(total, d, push=push) for c in world.comms]
    rng = np.random.default_rng(100 + p)
    sh_ = torch.cuda.current_stream().cuda_stream
    for slot, (off, n) in enumerate([(0, 40000), (8, 1), (1003, 12345), (4096, 0),
                                     (2048, 8 * 1001)]):
        data = [random_f16(rng, n) for _ in range(p)]
        for w, x in zip(wires, data):
            w.halves[0][off:off + n].copy_(torch.from_numpy(x))
        small = form if form in ("oneshot", "ll") else "none"
        launch([w.allreduce_op(0, off, n, sh_, slot=slot, small=small) for w in wires])
        torch.cuda.synchronize()
        want = rp.fold_f16_tree([x for x in data]) if n else np.zeros(0, np.uint16)
        for r, w in enumerate(wires):
            got = w.halves[0][off:off + n].cpu().numpy()
            assert np.array_equal(got, want), f"p={p} push={push} rank {r} bucket {slot}"
            assert w.status_word() == 0


@pytest.mark.parametrize("push", [False, True])
@pytest.mark.parametrize("p,k", [(2, 2), (4, 2), (4, 4), (6, 2), (8, 2), (8, 4), (8, 8)])
def test_hierarchical_allreduce_bit_exact(p, k, push, monkeypatch):
    """gs_hier_allreduce_f16 over Topology(p, k): intra-group reduce-scatter,
    inter-group fold of the group partials, all-gather (or, push form, the
    final sub-slices stored into every rank) — the reference's rank tree
    (fold_f16_tree) bit for bit."""
    from paper_1807_11205_b200.dist import OrderedWire
    # no one-shot inbox: every bucket below runs the two-level kernel (small
    # buckets take the one-shot kernel by default: test_hier_op_small_buckets)
    monkeypatch.setattr(OrderedWire, "SMALL_CAP_ELEMS", 0)
    d = dev.require_cuda()
    world = LocalWorld(gs.Topology(p, k), d, peer_ctas=8, timeout_s=20.0)
    wires = [c.make_ordered_wire(1 << 16, d, push=push) for c in world.comms]
    rng = np.random.default_rng(300 + 10 * p + k)
    sh_ = torch.cuda.current_stream().cuda_stream
    for slot, (off, n) in enumerate([(0, 50001), (24, 7), (1000, 8 * p * 16 + 3)]):
        data = [random_f16(rng, n) for _ in range(p)]
        for w, x in zip(wires, data):
            w.halves[0][off:off + n].copy_(torch.from_numpy(x))
        launch([w.hier_op(0, off, n, k, sh_, slot=slot) for w in wires])
        torch.cuda.synchronize()
        want = rp.fold_f16_tree(data)
        for r, w in enumerate(wires):
            assert np.array_equal(w.halves[0][off:off + n].cpu().numpy(), want), \
                f"Topology({p},{k}) rank {r} bucket {slot}"
            assert w.status_word() == 0


@pytest.mark.parametrize("p,k", [(4, 2), (8, 4)])
def test_hier_op_small_buckets(p, k):
    """hier_op sends small buckets to the LL (whole vectors) or one-shot
    kernel (the reference's tree factors over the groups, so the bits are the
    hierarchy's); alternating parities over consecutive calls."""
    d = dev.require_cuda()
    world = LocalWorld(gs.Topology(p, k), d, peer_ctas=8, timeout_s=20.0)
    wires = [c.make_ordered_wire(1 << 16, d) for c in world.comms]
    rng = np.random.default_rng(900 + p)
    sh_ = torch.cuda.current_stream().cuda_stream
    for slot, (off, n) in enumerate([(0, 4096), (24, 7), (512, 3001), (8, 1)]):
        data = [random_f16(rng, n) for _ in range(p)]
        for w, x in zip(wires, data):
            w.halves[0][off:off + n].copy_(torch.from_numpy(x))
        ops = [w.hier_op(0, off, n, k, sh_, slot=slot) for w in wires]
        want_fn = "gs_ll_allreduce_f16" if n % 8 == 0 and off % 8 == 0 else \
            "gs_oneshot_allreduce_f16"
        assert ops[0].fn == want_fn
        launch(ops)
        torch.cuda.synchronize()
        want = rp.fold_f16_tree(data)
        for r, w in enumerate(wires):
            assert np.array_equal(w.halves[0][off:off + n].cpu().numpy(), want), (p, k, r, slot)
            assert w.status_word() == 0


@pytest.mark.parametrize("p", [2, 4, 8])
def test_reduce_scatter_and_allgather_bit_exact(p):
    """gs_ordered_reduce_scatter_f16 folds rank r's slice in tree order;
    gs_ordered_allgather then makes every slice whole everywhere."""
    d = dev.require_cuda()
    world = LocalWorld(gs.Topology(p, 1), d, peer_ctas=8)
    n = 50000 + 3 * p
    arenas = [c.make_arena({"buf": 2 * n}, d, 2 * 8 * p) for c in world.comms]
    status = torch.zeros(p * 16, dtype=torch.int32, device=d)
    ctx = [rank_ctx(r, timeout_s=20.0, status=dev.ptr(status) + 64 * r) for r in range(p)]
    bounds_e = np.linspace(0, n, p + 1).astype(np.int64) // 8 * 8
    bounds_e[-1] = n
    bounds = dev.upload(bounds_e, d)
    bytes_b = dev.upload(2 * bounds_e, d)
    rng = np.random.default_rng(7)
    data = [random_f16(rng, n) for _ in range(p)]
    for a, x in zip(arenas, data):
        a.view("buf", torch.uint16)[:n].copy_(torch.from_numpy(x))
    sh_ = torch.cuda.current_stream().cuda_stream
    tab, sig = dev.ptr(arenas[0].peers("buf")), dev.ptr(arenas[0].peers("sig"))
    launch([PeerOp("gs_ordered_reduce_scatter_f16", ctx[r], (p, tab, sig, dev.ptr(bounds), 1, 8, sh_))
            for r in range(p)])
    torch.cuda.synchronize()
    want = rp.fold_f16_tree(data)
    for r, a in enumerate(arenas):
        lo, hi = bounds_e[r], bounds_e[r + 1]
        assert np.array_equal(a.view("buf", torch.uint16)[lo:hi].cpu().numpy(), want[lo:hi])
    launch([PeerOp("gs_ordered_allgather", ctx[r], (p, tab, sig, dev.ptr(bytes_b), 2, 8, sh_))
            for r in range(p)])
    torch.cuda.synchronize()
    for a in arenas:
        assert np.array_equal(a.view("buf", torch.uint16)[:n].cpu().numpy(), want)
    assert int(status.abs().sum()) == 0


def test_missing_peer_times_out_without_hanging():
    """A rank that never arrives: the waits give up after the bound, record
    the site / phase / peer in the status word and the kernel completes (no
    trap, the context stays usable); the pipeline raises PeerTimeoutError."""
    d = dev.require_cuda()
    world = LocalWorld(gs.Topology(2, 1), d, peer_ctas=4, timeout_s=0.5)
    wires = [c.make_ordered_wire(4096, d) for c in world.comms]
    sh_ = torch.cuda.current_stream().cuda_stream
    launch([wires[0].allreduce_op(0, 0, 4096, sh_)])  # rank 1 never launches
    torch.cuda.synchronize()
    st = wires[0].status_word() & 0xFFFFFFFF
    assert st >> 31 == 1 and (st >> 20) & 0xFF == 1 and (st >> 8) & 0xFF == 1 and st & 0xFF == 0
    # the device is still healthy
    assert float(torch.ones(4, device=d).sum()) == 4.0


# ---------------------------------------------------------------- pipelines
def run_emulated(p, model="shufflenet_v2_x0_5", theta=256 << 10, steps=3, inject_step=2,
                 incremental=False, in_place=False, specs=None, k=1, executor=True, **kw):
    d = dev.require_cuda()
    specs = specs or sh.load_shapes(model)
    master = sh.synth_master(specs, seed=0)
    world = LocalWorld(gs.Topology(p, k), d, peer_ctas=16)
    cfg = gs.LarsConfig(gs.Schedule(0.1), eta=0.001, weight_decay=5e-4, momentum=0.9)
    pipes = [gs.GradientPipeline(specs, cfg, threshold_bytes=theta, comm=c, init_master=master,
                                 loss_scale=gs.LossScale(1024.0), device=d, **kw)
             for c in world.comms]
    groups = [rp.Group(s.name, s.kind, w.copy(), np.zeros(s.numel, np.float32),
                       np.zeros(s.numel, np.float32), rp.narrow(w))
              for s, w in zip(specs, split(master, specs))]
    oloss = rp.LossScaleState(1024.0)
    order = list(reversed(range(len(specs))))
    for step in range(steps):
        wires = [sh.synth_wire_grads(specs, rank=r, seed=step, loss_scale=oloss.scale)
                 for r in range(p)]
        if step == inject_step:
            wires[p - 1][4321] = 0x7C00
        flats = [torch.from_numpy(w).to(d) for w in wires]
        if in_place:
            for pipe, f in zip(pipes, flats):
                for v, t in zip(pipe.grad_views(), split(f, specs)):
                    v.copy_(t)
            grads = [pipe.grad_views() for pipe in pipes]
        else:
            grads = flats
        if incremental:
            world.begin(pipes, step)
            views = [split(f, specs) for f in flats]
            for b in reversed(range(len(pipes[0].buckets))):
                world.submit(pipes, b, [[v[i] for i in pipes[0].buckets[b].params]
                                        for v in views])
            world.end(pipes)
            res = [pipe.finish() for pipe in pipes]
        else:
            res = world.step(pipes, grads, step, executor=executor)
        out = rp.compose_step_fp16([split(w, specs) for w in wires], [s.name for s in specs],
                                   [s.numel for s in specs], order, groups,
                                   rp.LarsHyper(0.001, 0.0, 5e-4, 0.9), 0.1, oloss, theta,
                                   kw.get("eta_bytes", 0), threads=rp.default_threads())
        if pipes[0].sharded:
            world.gather_state(pipes)
        for r, (pipe, rr) in enumerate(zip(pipes, res)):
            what = f"p={p} step={step} rank={r}"
            assert rr.applied == out.applied, what
            assert rr.scale == out.scale_used and pipe.loss_scale.scale == oloss.scale, what
            if out.applied:
                assert rr.grad_norm == pytest.approx(out.grad_norm, rel=1e-12), what
                assert np.array_equal(pipe.seg_scales(), out.scales), what
            for name, want in (("master", np.concatenate([g.master for g in groups])),
                               ("velocity", np.concatenate([g.velocity for g in groups]))):
                got = pipe.registration_view(getattr(pipe, name)).cpu().numpy()
                bad = np.flatnonzero(got.view(np.uint32) != want.view(np.uint32))
                assert bad.size == 0, f"{what}: {name} differs in {bad.size} elements"
            got = pipe.registration_view(pipe.working).cpu().numpy()
            assert np.array_equal(got, np.concatenate([g.working for g in groups])), what
    return pipes


@pytest.mark.parametrize("p,executor", [(2, True), (4, True), (8, True), (2, False), (8, False)])
def test_sharded_fused_step_bit_exact(p, executor):
    """gs_rs_pass1 + gs_zero_update + gs_peer_fence (ZeRO-1 step),
    shufflenet shapes, theta = 256 KiB, 3 steps, +Inf on the last rank at
    step 2 (skipped everywhere, loss scale halved) — through the native
    executor (gs_step_zero, all ranks in one call) and through the
    per-kernel generators in lockstep."""
    pipes = run_emulated(p, sharded_update=True, executor=executor)
    assert pipes[0].fused_collective
    assert pipes[0].loss_scale.scale == 512.0


@pytest.mark.parametrize("p", [2, 8])
def test_sharded_fused_step_gradients_in_place(p):
    """Gradients written straight into the raw wire (grad_views): no pack,
    and the step leaves them untouched."""
    run_emulated(p, sharded_update=True, in_place=True, steps=2, inject_step=-1)


@pytest.mark.parametrize("p", [2, 4, 8])
def test_sharded_separate_collectives_bit_exact(p):
    """Reduce-scatter + pass 1 + all-gather of the partials + trust + pass 2 +
    all-gather of the working weights (the unfused ZeRO-1 form)."""
    run_emulated(p, sharded_update=True, fused_collective=False)


@pytest.mark.parametrize("p,push", [(2, False), (4, True), (8, False), (8, True)])
def test_ordered_allreduce_step_bit_exact(p, push):
    """Replicated update after the own ordered all-reduce of every bucket."""
    run_emulated(p, flat_variant="ordered", eta_bytes=0, ordered_push=push)


@pytest.mark.parametrize("p,k", [(4, 2), (8, 4), (8, 2)])
def test_hierarchical_step_bit_exact(p, k):
    """Every bucket hierarchical (eta = inf, the reference's config 1 rule)
    through the own two-level kernel, replicated update."""
    pipes = run_emulated(p, k=k, eta_bytes=float("inf"), hier_variant="ordered_hier")
    assert {b.algorithm for b in pipes[0].buckets} == {"ordered_hier"}


def test_config1_emulated_hierarchy_matches_reference_hashes(golden):
    """Config 1 (shufflenet shapes, p = 4 as Topology(4, 2),
    theta = 256 KiB, eta = inf, an injected +Inf at step 2) with the four
    ranks emulated on the device and the two-level own kernel: master,
    velocity and working copy equal the SHA-256 the reference produced."""
    import hashlib
    doc = golden.json("step_golden.json")
    d = dev.require_cuda()
    specs = sh.load_shapes(doc["model"])
    world = LocalWorld(gs.Topology(doc["p"], doc["k"]), d, peer_ctas=16)
    cfg = gs.LarsConfig(gs.Schedule(base_lr=doc["lr"]), eta=doc["eta"], epsilon=doc["epsilon"],
                        weight_decay=doc["weight_decay"], momentum=doc["momentum"])
    pipes = [gs.GradientPipeline(specs, cfg, threshold_bytes=doc["theta"], comm=c,
                                 eta_bytes=float("inf"), hier_variant="ordered_hier",
                                 init_master=sh.synth_master(specs, seed=0),
                                 loss_scale=gs.LossScale(doc["loss_scale"]), device=d)
             for c in world.comms]
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    for step, want in enumerate(doc["steps"]):
        grads = []
        for r in range(doc["p"]):
            flat = sh.synth_wire_grads(specs, rank=r, seed=step,
                                       loss_scale=pipes[0].loss_scale.scale)
            inj = doc["inject"]
            if step == inj["step"] and r == inj["rank"]:
                flat[inj["index"]] = 0x7C00
            grads.append(torch.from_numpy(flat).to(d))
        res = world.step(pipes, grads, step)
        for pipe, rr in zip(pipes, res):
            assert rr.applied == want["applied"] and rr.scale == want["scale_used"]
            assert pipe.loss_scale.scale == want["scale_after"]
            assert sha(pipe.registration_view(pipe.master).cpu().numpy()) == want["master_sha"]
            assert sha(pipe.registration_view(pipe.velocity).cpu().numpy()) == want["velocity_sha"]
            assert sha(pipe.registration_view(pipe.working).cpu().numpy()) == want["working_sha"]


@pytest.mark.parametrize("p", [4, 8])
def test_incremental_sharded_step_bit_exact(p):
    """begin / submit (buckets in reverse) / end: per-bucket gs_rs_pass1 as
    the backward-overlap driver issues it."""
    run_emulated(p, sharded_update=True, incremental=True)


@pytest.mark.timeout(900)
def test_resnet50_p8_sharded_fused_bit_exact():
    """ResNet-50 (25.6 M params, 161 tensors), theta = 16 MiB, p = 8."""
    run_emulated(8, model="resnet50", theta=16 << 20, steps=1, inject_step=-1,
                 sharded_update=True)


@pytest.mark.timeout(900)
def test_resnet50_p8_ordered_bit_exact():
    run_emulated(8, model="resnet50", theta=16 << 20, steps=1, inject_step=-1,
                 flat_variant="ordered", eta_bytes=0)


def test_pipeline_reports_peer_timeout():
    """finish() raises PeerTimeoutError when a peer wait timed out."""
    d = dev.require_cuda()
    specs = sh.load_shapes("shufflenet_v2_x0_5")
    world = LocalWorld(gs.Topology(2, 1), d, peer_ctas=4, timeout_s=0.5)
    cfg = gs.LarsConfig(gs.Schedule(0.1))
    pipes = [gs.GradientPipeline(specs, cfg, threshold_bytes=1 << 20, comm=c,
                                 sharded_update=True, device=d) for c in world.comms]
    g = torch.from_numpy(sh.synth_wire_grads(specs, rank=0)).to(d)
    # drive rank 0 alone: its peer waits can never be satisfied
    for op in pipes[0]._enqueue_gen(g, 0):
        launch([op])
    with pytest.raises(RuntimeError, match="driven by its LocalWorld"):
        pipes[1].enqueue(g, 0)
    with pytest.raises(PeerTimeoutError, match="peer 1"):
        pipes[0].finish()
