import numpy as np, torch
import paper_1807_11205_b200 as gs
from paper_1807_11205_b200 import _native, _device as dev
from paper_1807_11205_b200._plan import LarsPlan, SegmentSpec, step_params
sh = dev.stream_of()
def trial(kind_flags, n, pos, val, gnorm=False, mode_decay=True):
    w = torch.ones(n, device='cuda'); g = torch.full((n,), 0.5, device='cuda'); g[pos] = val
    v = torch.zeros(n, device='cuda'); h = torch.zeros(n, dtype=torch.uint16, device='cuda')
    plan = LarsPlan([SegmentSpec(g.data_ptr(), w.data_ptr(), v.data_ptr(), h.data_ptr(), n, kind_flags)], g.device)
    plan.set_params(step_params(eta=0.001, epsilon=0.0, gamma=0.1, weight_decay=1e-4 if mode_decay else 0.0, momentum=0.9, grad_norm=gnorm))
    plan.reset_flags(sh); plan.pass1(sh, False); torch.cuda.synchronize()
    return plan.flags.item()
for flags in (0, 1, 2, 3):
    for n, pos in ((4, 1), (16, 9), (8192, 5000), (20000, 19999)):
        for gnorm in (False, True):
            print(f"segflags={flags} n={n} pos={pos} gnorm={gnorm}: nan->{trial(flags, n, pos, float('nan'), gnorm)} inf->{trial(flags, n, pos, float('inf'), gnorm)}")
