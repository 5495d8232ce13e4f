"""Time gs_lars_pass1 / gs_lars_pass1_trust variants on ResNet-50 shapes.

python tools/pass1_variants.py   (GPU)
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1807_11205_b200 import _native, _device as dev, shapes as sh  # noqa: E402
from paper_1807_11205_b200._plan import LarsPlan, SegmentSpec, step_params  # noqa: E402
from paper_1807_11205_b200.lars import KINDS  # noqa: E402


def main():
    d = torch.device("cuda")
    specs = sh.load_shapes("resnet50")
    n = sh.total_params(specs)
    g = torch.from_numpy(sh.synth_wire_grads(specs, 0)).to(d)
    w = torch.from_numpy(sh.synth_master(specs)).to(d)
    v = torch.zeros_like(w)
    h = torch.zeros_like(g)
    wire = torch.zeros_like(g)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=d)
    offs = np.cumsum([0] + [s.numel for s in specs])
    order = list(reversed(range(len(specs))))
    base = lambda t, i, es: t.data_ptr() + es * int(offs[i])
    flags = lambda s: (0 if s.kind == "weight" else 1) | (2 if s.kind == "weight" else 0)
    results = {}
    import os
    gc = os.environ.get("P1_GCOPY", "0") == "1"
    combos = ((8192, gc),) if os.environ.get("GRADSYNC_B200_LIB") else \
        ((8192, True), (16384, True), (8192, False))
    for ce, gcopy in combos:
        segs = [SegmentSpec(base(g, i, 2), base(w, i, 4), base(v, i, 4), base(h, i, 2), s.numel,
                            flags(s), base(wire, i, 2) if gcopy else 0)
                for i, s in enumerate(specs)]
        plan = LarsPlan(segs, d, order=order, chunk_elems=ce)
        for gn in (True,):
            prm = step_params(eta=0.001, epsilon=0.0, gamma=0.1, weight_decay=5e-4, momentum=0.9,
                              unscale_divisor=1024.0, grad_norm=gn)
            for bulk in ((False,) if os.environ.get("GRADSYNC_B200_LIB") else (True, False)):
                for fuse in (False,):
                    plan.extra_hint = 0 if bulk else _native.HINT_NO_BULK
                    plan.set_params(prm.copy(), g_is_f16=True)
                    sh_ = dev.stream_of()
                    ts, t2, tt, t3 = [], [], [], []
                    for it in range(12):
                        _native.call("gs_fill_zero", flush.data_ptr(), flush.numel(), sh_)
                        plan.reset_flags(sh_)
                        a = torch.cuda.Event(enable_timing=True)
                        b = torch.cuda.Event(enable_timing=True)
                        torch.cuda._sleep(2_000_000)
                        a.record()
                        plan.pass1(sh_, True, fuse=fuse)
                        b.record()
                        t0 = torch.cuda.Event(enable_timing=True)
                        t0.record()
                        plan.trust(sh_)
                        _native.call("gs_fill_zero", flush.data_ptr(), flush.numel(), sh_)
                        torch.cuda._sleep(1_000_000)
                        c2 = torch.cuda.Event(enable_timing=True)
                        c2.record()
                        plan.pass2(sh_, True, 3)
                        e2 = torch.cuda.Event(enable_timing=True)
                        e2.record()
                        _native.call("gs_fill_zero", flush.data_ptr(), flush.numel(), sh_)
                        torch.cuda._sleep(1_000_000)
                        e2 = torch.cuda.Event(enable_timing=True)
                        e2.record()
                        plan.pass2(sh_, True, 3, trust=True)
                        e3 = torch.cuda.Event(enable_timing=True)
                        e3.record()
                        e3.synchronize()
                        if it >= 2:
                            ts.append(a.elapsed_time(b) * 1e3)
                            t2.append(c2.elapsed_time(e2) * 1e3)
                            tt.append(t0.elapsed_time(c2) * 1e3)
                            t3.append(e2.elapsed_time(e3) * 1e3)
                    key = f"chunk={ce} gcopy={int(gcopy)} gnorm={int(gn)} bulk={int(bulk)} fuse={int(fuse)}"
                    results[key] = float(np.median(ts))
                    p2 = float(np.median(t2))
                    print(f"{key}: pass1 {results[key]:8.1f} us  ({(6 + 2 * gcopy) * n / results[key] / 1e3:7.0f} GB/s)"
                          f"   trust {float(np.median(tt)):6.1f} us   pass2 {p2:7.1f} us ({20 * n / p2 / 1e3:7.0f} GB/s)"
                          f"   pass2+trust {float(np.median(t3)):7.1f} us",
                          flush=True)


if __name__ == "__main__":
    main()
