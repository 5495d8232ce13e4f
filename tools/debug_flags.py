import numpy as np, torch
import paper_1807_11205_b200 as gs
from paper_1807_11205_b200 import _native, _device as dev
from paper_1807_11205_b200.lars import _plan_for
from paper_1807_11205_b200._plan import step_params
cfg = gs.LarsConfig(gs.Schedule(base_lr=0.1))
a = gs.make_param_group("a", "weight", np.ones(4))
b = gs.make_param_group("b", "bias", np.ones(4))
a.grad.fill_(0.5)
b.grad.copy_(torch.tensor([0.1, float("nan"), 0.1, 0.1]))
plan = _plan_for([a, b])
print("segs", plan.host_segs)
print("chunks", plan.host_chunks)
plan.set_params(step_params(eta=0.001, epsilon=0.0, gamma=0.1, weight_decay=1e-4, momentum=0.9))
sh = dev.stream_of()
plan.reset_flags(sh); torch.cuda.synchronize(); print("after reset", plan.flags.item())
plan.pass1(sh, False); torch.cuda.synchronize(); print("after pass1", plan.flags.item(), plan.partials.cpu().numpy())
plan.trust(sh); torch.cuda.synchronize(); print("after trust", plan.flags.item(), plan.seg_out.cpu().numpy())
plan.pass2(sh, False, 2); torch.cuda.synchronize(); print("after pass2", plan.flags.item())
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
x = torch.tensor([1.0, float('inf')], device='cuda')
print("any_nonfinite", gs.halfprec.any_nonfinite([x]))
