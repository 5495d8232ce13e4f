"""Pipeline-level LARS v1 checkpoints (lars.py:184-237, pkg/README.md:167-173)
straight from the device arenas: byte-identical to a file the REFERENCE's
save_checkpoint wrote (tests/golden/checkpoint_golden.lars), loadable back,
and a bitwise resume (test_lars.py:248-279) — also from a sharded (ZeRO-1)
pipeline, whose masters / velocities are gathered first."""

import json

import numpy as np
import pytest
import torch

import paper_1807_11205_b200 as gs
from paper_1807_11205_b200 import _device as dev
from paper_1807_11205_b200 import shapes as sh
from paper_1807_11205_b200.emulation import LocalWorld

pytestmark = pytest.mark.gpu


def golden_specs(golden):
    g = golden.npz("checkpoint_golden.npz")
    specs = [gs.ParamSpec(str(n), tuple(json.loads(str(s))), str(k))
             for n, s, k in zip(g["names"], g["shapes"], g["kinds"])]
    return g, specs


def cfg():
    return gs.LarsConfig(gs.Schedule(0.1), eta=0.001, weight_decay=5e-4, momentum=0.9)


def test_save_is_byte_identical_to_reference(golden, tmp_path):
    g, specs = golden_specs(golden)
    n = len(specs)
    pipe = gs.GradientPipeline(specs, cfg(), threshold_bytes=4096,
                               init_master=np.concatenate([g[f"w_{i}"] for i in range(n)]))
    for i, grp in enumerate(pipe.groups):
        grp.velocity.copy_(torch.from_numpy(g[f"v_{i}"]))
        grp.working_w16.copy_(torch.from_numpy(g[f"h_{i}"]))
    out = tmp_path / "mine.lars"
    pipe.save_checkpoint(out, step=2)
    from pathlib import Path
    want = (Path(__file__).parent / "golden" / "checkpoint_golden.lars").read_bytes()
    assert out.read_bytes() == want


def test_load_restores_every_arena(golden):
    g, specs = golden_specs(golden)
    from pathlib import Path
    path = Path(__file__).parent / "golden" / "checkpoint_golden.lars"
    pipe = gs.GradientPipeline(specs, cfg(), threshold_bytes=4096)
    assert pipe.load_checkpoint(path) == 2
    for i, grp in enumerate(pipe.groups):
        assert np.array_equal(dev.to_host(grp.master_w).view(np.uint32), g[f"w_{i}"].view(np.uint32))
        assert np.array_equal(dev.to_host(grp.velocity).view(np.uint32), g[f"v_{i}"].view(np.uint32))
        assert np.array_equal(dev.to_host(grp.working_w16), g[f"h_{i}"])
    # a mismatched pipeline is refused with the reason
    bad = [gs.ParamSpec(s.name, s.shape, "bias" if s.kind == "weight" else s.kind) for s in specs]
    with pytest.raises(ValueError, match="does not match"):
        gs.GradientPipeline(bad, cfg(), threshold_bytes=4096).load_checkpoint(path)


def _grads(specs, step, p=1):
    return [torch.from_numpy(sh.synth_wire_grads(specs, rank=r, seed=step)).cuda()
            for r in range(p)]


def test_bitwise_resume(tmp_path):
    """4 steps straight == 2 steps, save, a fresh pipeline loads, 2 steps."""
    specs = sh.load_shapes("shufflenet_v2_x0_5")
    master = sh.synth_master(specs, seed=0)
    a = gs.GradientPipeline(specs, cfg(), threshold_bytes=256 << 10, init_master=master)
    b = gs.GradientPipeline(specs, cfg(), threshold_bytes=256 << 10, init_master=master)
    for step in range(4):
        a.step(_grads(specs, step)[0], step)
    for step in range(2):
        b.step(_grads(specs, step)[0], step)
    b.save_checkpoint(tmp_path / "b.lars", step=2)
    c = gs.GradientPipeline(specs, cfg(), threshold_bytes=256 << 10,
                            init_master=sh.synth_master(specs, seed=9),
                            loss_scale=gs.LossScale(b.loss_scale.scale,
                                                    clean_steps=b.loss_scale.clean_steps))
    assert c.load_checkpoint(tmp_path / "b.lars") == 2
    for step in range(2, 4):
        c.step(_grads(specs, step)[0], step)
    for name in ("master", "velocity", "working"):
        assert torch.equal(getattr(a, name), getattr(c, name)), name
    a.save_checkpoint(tmp_path / "a.lars", step=4)
    c.save_checkpoint(tmp_path / "c.lars", step=4)
    assert (tmp_path / "a.lars").read_bytes() == (tmp_path / "c.lars").read_bytes()


@pytest.mark.parametrize("p", [2, 4])
def test_sharded_checkpoint_matches_replicated(p, tmp_path):
    """Every rank of an emulated ZeRO-1 job writes the same file, equal to
    the file of the single-process reference-order fold after the same steps."""
    d = dev.require_cuda()
    specs = sh.load_shapes("shufflenet_v2_x0_5")
    master = sh.synth_master(specs, seed=0)
    world = LocalWorld(gs.Topology(p, 1), d, peer_ctas=8)
    pipes = [gs.GradientPipeline(specs, cfg(), threshold_bytes=256 << 10, comm=c,
                                 sharded_update=True, init_master=master, device=d)
             for c in world.comms]
    ref = gs.GradientPipeline(specs, cfg(), threshold_bytes=256 << 10, local_workers=p,
                              init_master=master)
    for step in range(2):
        g = _grads(specs, step, p)
        world.step(pipes, g, step)
        ref.step(g, step)
    world.gather_state(pipes)
    files = []
    for r, pp in enumerate(pipes):
        # the gather already ran: save the groups directly (no second collective)
        gs.save_checkpoint(tmp_path / f"r{r}.lars", pp.groups, 2)
        files.append((tmp_path / f"r{r}.lars").read_bytes())
    ref.save_checkpoint(tmp_path / "ref.lars", step=2)
    assert all(f == files[0] for f in files)
    assert files[0] == (tmp_path / "ref.lars").read_bytes()
