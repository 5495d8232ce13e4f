"""Backward-overlap driver (overlap.py): buckets launched from
autograd hooks during backward must give bit-for-bit the state the CPU oracle
(the reference's step composition, experiment.py:368-413 on the fp16 wire)
computes from the same hooked gradients, including a skipped (overflow) step,
and the model's fp16 weights must be the working arena."""

import numpy as np
import pytest
import torch

from oracle import reference_port as rp
import paper_1807_11205_b200 as gs

pytestmark = pytest.mark.gpu


class Net(torch.nn.Module):
    def __init__(self):
        super().__init__()
        self.c1 = torch.nn.Conv2d(3, 16, 3, padding=1, bias=False)
        self.b1 = torch.nn.BatchNorm2d(16)
        self.c2 = torch.nn.Conv2d(16, 32, 3, stride=2, padding=1, bias=False)
        self.b2 = torch.nn.BatchNorm2d(32)
        self.fc = torch.nn.Linear(32, 10)

    def forward(self, x):
        x = torch.relu(self.b1(self.c1(x)))
        x = torch.relu(self.b2(self.c2(x)))
        return self.fc(x.mean(dim=(2, 3)))


def _setup(theta):
    torch.manual_seed(0)
    net = Net().cuda()
    cfg = gs.LarsConfig(gs.Schedule(0.1), eta=0.001, weight_decay=5e-4, momentum=0.9)
    drv = gs.BackwardOverlap.for_module(net, cfg, threshold_bytes=theta,
                                        loss_scale=gs.LossScale(1024.0))
    master = drv.pipe.registration_view(drv.pipe.master).cpu().numpy()
    groups, o = [], 0
    for s in drv.pipe.specs:
        w = master[o:o + s.numel].copy()
        groups.append(rp.Group(s.name, s.kind, w, np.zeros(s.numel, np.float32),
                               np.zeros(s.numel, np.float32), rp.narrow(w)))
        o += s.numel
    return net, drv, groups


def _bits(t):
    return t.cpu().numpy().view(np.uint16 if t.dtype == torch.uint16 else np.uint32)


@pytest.mark.parametrize("theta", [0, 2048, 1 << 30])
def test_overlap_matches_oracle(theta):
    net, drv, groups = _setup(theta)
    specs = drv.pipe.specs
    oloss = rp.LossScaleState(1024.0)
    assert drv.pipe.specs[0].kind == "weight" and drv.pipe.specs[1].kind == "bn_gamma"
    assert drv.pipe.specs[2].kind == "bn_beta" and drv.pipe.specs[-1].kind == "bias"
    seen = {}
    for i, p in enumerate(drv.params):
        p.register_post_accumulate_grad_hook(
            lambda q, i=i: seen.__setitem__(i, q.grad.detach().clone().view(torch.uint16)))
    inf_hook = None
    for step in range(4):
        x = torch.randn(8, 3, 16, 16, device="cuda", generator=None).half()
        y = torch.randint(0, 10, (8,), device="cuda")
        if step == 2:  # forced overflow on one gradient: the step must be skipped
            inf_hook = drv.params[0].register_hook(
                lambda g: g.flatten().index_fill(0, torch.tensor([3], device=g.device),
                                                 float("inf")).view_as(g))
        drv.begin(step)
        loss = torch.nn.functional.cross_entropy(net(x).float(), y)
        (loss * drv.loss_scale).backward()
        res = drv.finish()
        if inf_hook is not None:
            inf_hook.remove()
            inf_hook = None
        grads = [seen[i].cpu().numpy().reshape(-1) for i in range(len(drv.params))]
        want = rp.compose_step_fp16([grads], [s.name for s in specs], [s.numel for s in specs],
                                    list(reversed(range(len(specs)))), groups,
                                    rp.LarsHyper(0.001, 0.0, 5e-4, 0.9), 0.1, oloss, theta, 0)
        assert (res.applied, res.scale) == (want.applied, want.scale_used)
        assert drv.pipe.loss_scale.scale == oloss.scale
        assert res.grad_norm == pytest.approx(want.grad_norm, rel=1e-12)
        assert res.applied == (step != 2)
        for name, attr in (("master", "master"), ("velocity", "velocity"),
                           ("working", "working")):
            a = np.concatenate([getattr(g, attr) for g in groups])
            b = _bits(drv.pipe.registration_view(getattr(drv.pipe, name)))
            assert np.array_equal(a.view(b.dtype), b), f"step {step}: {name} differs"
        # the model's weights ARE the working arena
        flat = torch.cat([p.detach().reshape(-1) for p in drv.params]).view(torch.uint16)
        assert torch.equal(flat, drv.pipe.registration_view(drv.pipe.working))
        assert all(p.grad is None for p in drv.params)
    assert drv.pipe.loss_scale.scale == 512.0


def test_overlap_missing_gradient_raises():
    net, drv, _ = _setup(4096)
    drv.begin(0)
    x = torch.randn(2, 3, 8, 8, device="cuda").half()
    out = torch.relu(net.b1(net.c1(x))).sum()  # c2/b2/fc get no gradient
    out.backward()
    with pytest.raises(RuntimeError, match="no gradient arrived"):
        drv.finish()
