"""The reference's own fp32-wire step (run_experiment, experiment.py:368-413:
fp32 gradients fused by FusionBuffer at 4 bytes per element, all-reduced with
op="mean" as the ascending fp32 left fold, then LossScale / unscale / LARS)
through GradientPipeline(wire_dtype="f32").

Pinned by tests/golden/step32_golden.json, written by running the
reference's experiment._fused_allreduce and lars_step (make_golden.py
make_step32): config-1 shapes, p = 4 as Topology(4, 2), theta = 256 KiB,
eta = inf, registration order (experiment.py:371), an injected +Inf at
step 2 (skip, loss scale halved)."""

import hashlib

import numpy as np
import pytest
import torch

from oracle import reference_port as rp
import paper_1807_11205_b200 as gs
from paper_1807_11205_b200 import _device as dev
from paper_1807_11205_b200 import shapes as sh
from paper_1807_11205_b200.emulation import LocalWorld

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def grads_of(doc, specs, step, scale):
    out = []
    for r in range(doc["p"]):
        flat = sh.synth_grads_f32(specs, rank=r, seed=step) * np.float32(scale)
        if step == doc["inject"]["step"] and r == doc["inject"]["rank"]:
            flat[doc["inject"]["index"]] = np.inf
        out.append(torch.from_numpy(flat).cuda())
    return out


def check(doc, pipes, run):
    specs = pipes[0].specs
    for step, want in enumerate(doc["steps"]):
        res = run(grads_of(doc, specs, step, pipes[0].loss_scale.scale), step)
        for pipe, r in zip(pipes, res):
            assert r.applied == want["applied"] and r.scale == want["scale_used"]
            assert pipe.loss_scale.scale == want["scale_after"]
            if want["applied"]:
                assert r.grad_norm == pytest.approx(want["grad_norm"], rel=1e-12)
            assert [[list(m) for m in b.unpack_map] for b in pipe.buckets] == want["maps"]
            assert sha(pipe.registration_view(pipe.master).cpu().numpy()) == want["master_sha"]
            assert sha(pipe.registration_view(pipe.velocity).cpu().numpy()) == want["velocity_sha"]
            assert sha(pipe.registration_view(pipe.working).cpu().numpy()) == want["working_sha"]


def _cfg(doc):
    return gs.LarsConfig(gs.Schedule(base_lr=doc["lr"]), eta=doc["eta"], epsilon=doc["epsilon"],
                         weight_decay=doc["weight_decay"], momentum=doc["momentum"])


def test_fp32_wire_local_workers_match_reference_hashes(golden):
    doc = golden.json("step32_golden.json")
    specs = sh.load_shapes(doc["model"])
    pipe = gs.GradientPipeline(specs, _cfg(doc), threshold_bytes=doc["theta"],
                               local_workers=doc["p"], order=list(range(len(specs))),
                               wire_dtype="f32", init_master=sh.synth_master(specs, seed=0),
                               loss_scale=gs.LossScale(doc["loss_scale"]))
    check(doc, [pipe], lambda g, step: [pipe.step(g, step)])


@pytest.mark.parametrize("variant", ["ordered", "ordered_hier"])
def test_fp32_wire_emulated_ranks_match_reference_hashes(golden, variant):
    """The four ranks emulated on the device, every bucket through the own
    fp32 all-reduce kernel (gs_ordered_allreduce_f32) — flat, or requested as
    hierarchical (the fp32 left fold does not factor over groups: the flat
    kernel serves both, as the reference's algorithms agree bitwise)."""
    doc = golden.json("step32_golden.json")
    d = dev.require_cuda()
    specs = sh.load_shapes(doc["model"])
    world = LocalWorld(gs.Topology(doc["p"], doc["k"]), d, peer_ctas=16)
    kw = dict(flat_variant="ordered", eta_bytes=0) if variant == "ordered" else \
        dict(hier_variant="ordered_hier", eta_bytes=float("inf"))
    pipes = [gs.GradientPipeline(specs, _cfg(doc), threshold_bytes=doc["theta"], comm=c,
                                 order=list(range(len(specs))), wire_dtype="f32",
                                 init_master=sh.synth_master(specs, seed=0),
                                 loss_scale=gs.LossScale(doc["loss_scale"]), device=d, **kw)
             for c in world.comms]
    check(doc, pipes, lambda g, step: world.step(pipes, g, step))


@pytest.mark.parametrize("p,scale", [(1, 1024.0), (3, 1000.0)])
def test_fp32_wire_matches_oracle(p, scale):
    """p = 1 (no collective) and p = 3 with a non-power-of-two loss scale
    (the IEEE-division kernels) against the oracle's fp32 composition."""
    specs = sh.load_shapes("shufflenet_v2_x0_5")
    master = sh.synth_master(specs, seed=0)
    cfg = gs.LarsConfig(gs.Schedule(0.1), eta=0.001, weight_decay=5e-4, momentum=0.9)
    order = list(reversed(range(len(specs))))
    pipe = gs.GradientPipeline(specs, cfg, threshold_bytes=1 << 20, local_workers=p,
                               wire_dtype="f32", init_master=master,
                               loss_scale=gs.LossScale(scale))
    groups, o = [], 0
    for s in specs:
        w = master[o:o + s.numel].copy()
        groups.append(rp.Group(s.name, s.kind, w, np.zeros(s.numel, np.float32),
                               np.zeros(s.numel, np.float32), rp.narrow(w)))
        o += s.numel
    oloss = rp.LossScaleState(scale)
    for step in range(2):
        flats = [sh.synth_grads_f32(specs, rank=r, seed=step) * np.float32(oloss.scale)
                 for r in range(p)]
        dev_g = [torch.from_numpy(f).cuda() for f in flats]
        res = pipe.step(dev_g if p > 1 else dev_g[0], step)
        parts = []
        for f in flats:
            q, o = [], 0
            for s in specs:
                q.append(f[o:o + s.numel])
                o += s.numel
            parts.append(q)
        out = rp.compose_step_fp32(parts, [s.name for s in specs], [s.numel for s in specs],
                                   order, groups, rp.LarsHyper(0.001, 0.0, 5e-4, 0.9), 0.1,
                                   oloss, 1 << 20)
        assert res.applied == out.applied and pipe.loss_scale.scale == oloss.scale
        assert res.grad_norm == pytest.approx(out.grad_norm, rel=1e-12)
        for name, attr in (("master", "master"), ("velocity", "velocity")):
            got = pipe.registration_view(getattr(pipe, name)).cpu().numpy().view(np.uint32)
            want = np.concatenate([getattr(g, attr) for g in groups]).view(np.uint32)
            assert np.array_equal(got, want), f"p={p} step={step}: {name}"
        got = pipe.registration_view(pipe.working).cpu().numpy()
        assert np.array_equal(got, np.concatenate([g.working for g in groups]))
