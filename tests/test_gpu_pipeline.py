"""Parity of the fused pipeline (GradientPipeline) against the oracle / golden.

Bit-exact expectations: bucket layout, overflow flags, skip
decision, loss scale; with the ordered fold (local workers) and at p=1 also
master, velocity, working copy and the per-group fp32 trust scale.  The fp64
norms are summed in a different order than OpenBLAS' ddot, so the fp64 local
rate is checked at rel 1e-12 and the grad-norm metric at rel 1e-12.
"""

import hashlib

import numpy as np
import pytest
import torch

from oracle import reference_port as rp
import paper_1807_11205_b200 as gs
from paper_1807_11205_b200 import shapes as sh

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def split(flat, specs):
    out, o = [], 0
    for s in specs:
        out.append(flat[o:o + s.numel])
        o += s.numel
    return out


def oracle_groups(specs, master):
    groups = []
    for s, w in zip(specs, split(master, specs)):
        w = w.copy()
        groups.append(rp.Group(s.name, s.kind, w, np.zeros(s.numel, np.float32),
                               np.zeros(s.numel, np.float32), rp.narrow(w)))
    return groups


def check_state(pipe, groups, what=""):
    got_w = pipe.registration_view(pipe.master).cpu().numpy()
    got_v = pipe.registration_view(pipe.velocity).cpu().numpy()
    got_h = pipe.registration_view(pipe.working).cpu().numpy()
    want_w = np.concatenate([g.master for g in groups])
    want_v = np.concatenate([g.velocity for g in groups])
    want_h = np.concatenate([g.working for g in groups])
    bad = np.flatnonzero(got_w.view(np.uint32) != want_w.view(np.uint32))
    assert bad.size == 0, f"{what}: master differs at {bad[:8]} ({bad.size} elems)"
    assert np.array_equal(got_v.view(np.uint32), want_v.view(np.uint32)), f"{what}: velocity"
    assert np.array_equal(got_h, want_h), f"{what}: working copy"


def test_config1_ordered_matches_reference_golden(golden):
    """Config 1 (shufflenet shapes, 4 workers, Topology(4,2), theta=256 KiB,
    eta=inf): 3 steps incl. an injected overflow, against the hashes the
    reference itself produced."""
    doc = golden.json("step_golden.json")
    specs = sh.load_shapes(doc["model"])
    cfg = gs.LarsConfig(gs.Schedule(base_lr=doc["lr"]), eta=doc["eta"], epsilon=doc["epsilon"],
                        weight_decay=doc["weight_decay"], momentum=doc["momentum"])
    loss = gs.LossScale(doc["loss_scale"])
    pipe = gs.GradientPipeline(specs, cfg, threshold_bytes=doc["theta"], local_workers=doc["p"],
                               init_master=sh.synth_master(specs, seed=0), loss_scale=loss)
    assert [[list(m) for m in b.unpack_map] for b in pipe.buckets] == doc["steps"][0]["maps"]
    for step, want in enumerate(doc["steps"]):
        grads = []
        for r in range(doc["p"]):
            flat = sh.synth_wire_grads(specs, rank=r, seed=step, loss_scale=loss.scale)
            inj = doc["inject"]
            if step == inj["step"] and r == inj["rank"]:
                flat[inj["index"]] = 0x7C00
            grads.append(torch.from_numpy(flat).cuda())
        res = pipe.step(grads, step)
        assert res.applied == want["applied"]
        assert res.scale == want["scale_used"] and loss.scale == want["scale_after"]
        assert res.grad_norm == pytest.approx(want["grad_norm"], rel=1e-12)
        assert sha(pipe.registration_view(pipe.master).cpu().numpy()) == want["master_sha"]
        assert sha(pipe.registration_view(pipe.velocity).cpu().numpy()) == want["velocity_sha"]
        assert sha(pipe.registration_view(pipe.working).cpu().numpy()) == want["working_sha"]


def run_vs_oracle(model, p, theta, steps=2, loss_scale=1024.0, wd=5e-4, eta_bytes=0,
                  inject=None, order=None, specs=None, **kw):
    specs = specs or sh.load_shapes(model)
    master = sh.synth_master(specs, seed=0)
    cfg = gs.LarsConfig(gs.Schedule(base_lr=0.1), eta=0.001, epsilon=0.0, weight_decay=wd,
                        momentum=0.9)
    pipe = gs.GradientPipeline(specs, cfg, threshold_bytes=theta, local_workers=p,
                               init_master=master, loss_scale=gs.LossScale(loss_scale),
                               order=order, **kw)
    groups = oracle_groups(specs, master)
    oloss = rp.LossScaleState(loss_scale)
    order = order or list(reversed(range(len(specs))))
    for step in range(steps):
        wires = [sh.synth_wire_grads(specs, rank=r, seed=step, loss_scale=oloss.scale)
                 for r in range(p)]
        if inject is not None and inject[0] == step:
            wires[inject[1]][inject[2]] = inject[3]
        dev_grads = [torch.from_numpy(w).cuda() for w in wires]
        res = pipe.step(dev_grads if p > 1 else dev_grads[0], step)
        out = rp.compose_step_fp16([split(w, specs) for w in wires], [s.name for s in specs],
                                   [s.numel for s in specs], order, groups,
                                   rp.LarsHyper(0.001, 0.0, wd, 0.9), 0.1, oloss, theta,
                                   eta_bytes)
        assert res.applied == out.applied, step
        assert res.scale == out.scale_used and pipe.loss_scale.scale == oloss.scale
        assert res.grad_norm == pytest.approx(out.grad_norm, rel=1e-12, abs=0)
        if out.applied:
            assert np.array_equal(pipe.seg_scales(), out.scales)
            local = pipe.seg_stats()[:, 2]
            np.testing.assert_allclose(local, out.locals, rtol=1e-12, atol=0)
        check_state(pipe, groups, f"{model} p={p} step={step}")
        for b, m in zip(pipe.buckets, out.maps):
            assert b.unpack_map == m
    return pipe


@pytest.mark.parametrize("theta", [4 << 20, 16 << 20])
@pytest.mark.parametrize("kw", [{}, {"snapshot_wire": True}])
def test_resnet50_single_gpu_matches_oracle(kw, theta):
    """The bench configuration (theta = 16 MiB) and theta = 4 MiB; lazy wire
    (payloads packed on request) and the in-step snapshot."""
    pipe = run_vs_oracle("resnet50", 1, theta, steps=3, **kw)
    # the wire holds the reference's bucket payloads of the last step
    specs = sh.load_shapes("resnet50")
    flat = sh.synth_wire_grads(specs, rank=0, seed=2)
    parts = split(flat, specs)
    for b in range(len(pipe.buckets)):
        want = np.concatenate([parts[i] for i in pipe.buckets[b].params])
        assert np.array_equal(pipe.bucket_payload(b).cpu().numpy(), want)


def test_resnet50_p8_ordered_matches_oracle():
    run_vs_oracle("resnet50", 8, 16 << 20, steps=1)


def test_alexnet_single_gpu_matches_oracle():
    run_vs_oracle("alexnet", 1, 4 << 20, steps=1)


def test_non_power_of_two_workers_and_scale():
    # p = 3 and loss scale 1000 take the IEEE-division path of the kernels
    run_vs_oracle("shufflenet_v2_x0_5", 3, 256 << 10, steps=2, loss_scale=1000.0)


def test_overflow_skip_mutates_nothing():
    pipe = run_vs_oracle("shufflenet_v2_x0_5", 2, 256 << 10, steps=2,
                         inject=(1, 0, 777, 0x7C00))
    assert pipe.loss_scale.scale == 512.0


def test_near_overflow_sum_sets_flag():
    # every worker holds 65504 at one element: the pairwise sum overflows
    specs = sh.load_shapes("shufflenet_v2_x0_5")
    p = 4
    pipe = gs.GradientPipeline(specs, gs.LarsConfig(gs.Schedule(0.1)), threshold_bytes=1 << 20,
                               local_workers=p, init_master=sh.synth_master(specs))
    before = pipe.master.clone()
    grads = []
    for r in range(p):
        w = sh.synth_wire_grads(specs, rank=r)
        w[5000] = 0x7BFF
        grads.append(torch.from_numpy(w).cuda())
    res = pipe.step(grads, 0)
    assert not res.applied and res.flags & 1
    assert torch.equal(before, pipe.master)


def test_odd_sizes_and_unaligned_segments():
    rng = np.random.default_rng(3)
    specs = []
    for i in range(40):
        kind = ["weight", "bias", "bn_gamma", "bn_beta"][i % 4]
        shape = (int(rng.integers(1, 40)), int(rng.integers(1, 300))) if kind == "weight" \
            else (int(rng.integers(1, 700)),)
        specs.append(gs.ParamSpec(f"p{i}", shape, kind))
    specs.append(gs.ParamSpec("big", (3, 40001), "weight"))
    specs.append(gs.ParamSpec("empty", (0,), "bias"))
    order = list(rng.permutation(len(specs)))
    run_vs_oracle(None, 3, 3000, steps=2, specs=specs, order=[int(i) for i in order])


def test_fp32_lars_step_api_matches_oracle(golden):
    """lars_step drop-in (fp32 grads) on the golden trajectories."""
    g = golden.npz("lars_golden.npz")
    meta = golden.json("lars_golden_meta.json")
    kinds = ["weight", "bias", "bn_gamma", "bn_beta", "weight", "weight", "bias"]
    sizes = list(g["sizes"])
    for ci, c in enumerate(meta):
        sched = gs.Schedule(base_lr=c["base_lr"], kind=c.get("kind", "constant"),
                            warmup_steps=c.get("warmup_steps", 0),
                            total_steps=c.get("total_steps", 1), end_lr=c.get("end_lr", 0.0))
        cfg = gs.LarsConfig(sched, eta=c["eta"], epsilon=c["epsilon"],
                            weight_decay=c["weight_decay"], momentum=c["momentum"])
        groups = [gs.make_param_group(f"g{gi}", k, g[f"c{ci}_w0_{gi}"])
                  for gi, (k, n) in enumerate(zip(kinds, sizes))]
        for step in range(4):
            for gi, grp in enumerate(groups):
                grp.grad.copy_(torch.from_numpy(g[f"c{ci}_s{step}_g_{gi}"]))
            assert gs.lars_step(groups, cfg, step) == bool(g[f"c{ci}_s{step}_ok"])
            for gi, grp in enumerate(groups):
                assert np.array_equal(grp.master_w.cpu().numpy().view(np.uint32),
                                      g[f"c{ci}_s{step}_w_{gi}"].view(np.uint32)), (ci, step, gi)
                assert np.array_equal(grp.velocity.cpu().numpy().view(np.uint32),
                                      g[f"c{ci}_s{step}_v_{gi}"].view(np.uint32))
                assert np.array_equal(grp.working_w16.cpu().numpy(), g[f"c{ci}_s{step}_h_{gi}"])


def test_host_gradient_path_matches_device_path():
    """enqueue_host (per-bucket H2D overlapped with pass 1) == device path."""
    specs = sh.load_shapes("resnet50")
    master = sh.synth_master(specs, seed=0)
    cfg = gs.LarsConfig(gs.Schedule(base_lr=0.1), eta=0.001, weight_decay=5e-4, momentum=0.9)
    a = gs.GradientPipeline(specs, cfg, threshold_bytes=4 << 20, init_master=master)
    b = gs.GradientPipeline(specs, cfg, threshold_bytes=4 << 20, init_master=master)
    for step in range(2):
        host = torch.from_numpy(sh.synth_wire_grads(specs, rank=0, seed=step)).pin_memory()
        ra = a.step(host.cuda(), step)
        b.enqueue_host(host, step)
        rb = b.finish()
        assert ra.applied == rb.applied and ra.grad_norm == rb.grad_norm
        assert torch.equal(a.master, b.master) and torch.equal(a.working, b.working)
        assert torch.equal(a.velocity, b.velocity)


def test_per_kernel_path_equals_executor():
    """The per-kernel launch path (taken when a timer or NVTX asks for
    phases) and the native executor (gs_step_replicated) give the same
    state bit for bit, step after step."""
    specs = sh.load_shapes("shufflenet_v2_x0_5")
    master = sh.synth_master(specs, seed=0)
    cfg = gs.LarsConfig(gs.Schedule(0.1), eta=0.001, weight_decay=5e-4, momentum=0.9)
    a = gs.GradientPipeline(specs, cfg, threshold_bytes=256 << 10, init_master=master)
    b = gs.GradientPipeline(specs, cfg, threshold_bytes=256 << 10, init_master=master)
    phases = []
    for step in range(3):
        g = torch.from_numpy(sh.synth_wire_grads(specs, rank=0, seed=step)).cuda()
        ra = a.step(g, step)
        b.enqueue(g, step, timer=phases.append)
        rb = b.finish()
        assert (ra.applied, ra.grad_norm, ra.flags) == (rb.applied, rb.grad_norm, rb.flags)
        for name in ("master", "velocity", "working"):
            assert torch.equal(getattr(a, name), getattr(b, name)), (step, name)
    assert phases[:4] == ["pass1", "trust", "pass2", "end"]
