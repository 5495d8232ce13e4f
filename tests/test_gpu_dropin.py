"""The reference's hot-path tests, run against the drop-in API on the GPU.

Mirrors pkg/tests/test_halfprec.py, test_fusion.py, test_collectives.py and
test_lars.py (file:line cited per test) with numpy in / numpy out, plus the
golden vectors the reference produced (tests/golden/).
"""

import math

import numpy as np
import pytest
import torch

import paper_1807_11205_b200 as gs
from oracle import reference_port as rp
from paper_1807_11205_b200 import halfprec as hp
from test_oracle import BOUNDARY_CASES

pytestmark = pytest.mark.gpu


# ------------------------------------------------------------ halfprec

@pytest.mark.parametrize("value,bits", BOUNDARY_CASES)
def test_narrow_boundaries(value, bits):            # test_halfprec.py:74-77
    assert int(hp.f32_to_f16(value)) == bits


def test_narrow_golden_and_sticky(golden):
    g = golden.npz("halfprec_golden.npz")
    assert np.array_equal(hp.f32_to_f16(g["narrow_in"].view(np.float32)), g["narrow_out"])
    x = np.nextafter(np.float32(2.0**-25), np.float32(1))  # test_halfprec.py:80-85
    assert int(hp.f32_to_f16(x)) == 0x0001


def torch_narrow_ref(u: torch.Tensor) -> torch.Tensor:
    """The oracle's integer narrowing (oracle/reference_port.py:narrow) restated
    with torch int64 ops, so all 2^32 patterns can be checked on the device
    independently of the kernel's cvt.rn.f16.f32."""
    sign = (u >> 16) & 0x8000
    a = u & 0x7FFFFFFF
    out = torch.zeros_like(u)
    nrm = (a >= 0x38800000) & (a < 0x477FF000)
    out = torch.where(nrm, (a - 0x38000000 + 0xFFF + ((a >> 13) & 1)) >> 13, out)
    sub = (a >= 0x33000000) & (a < 0x38800000)
    e = a >> 23
    mant = (a & 0x7FFFFF) | 0x800000
    sh = torch.clamp(126 - e, 1, 40)
    q = mant >> sh
    rem = mant & ((torch.ones_like(sh) << sh) - 1)
    half = torch.ones_like(sh) << (sh - 1)
    q = q + ((rem > half) | ((rem == half) & ((q & 1) == 1))).to(torch.int64)
    out = torch.where(sub, q, out)
    out = torch.where((a >= 0x477FF000) & (a <= 0x7F800000), torch.full_like(out, 0x7C00), out)
    out = out | sign
    out = torch.where(a > 0x7F800000, torch.full_like(out, 0x7E00), out)
    return out


def test_narrow_exhaustive_all_float32_patterns():
    """All 2^32 float32 bit patterns through gs_f32_to_f16 against the
    oracle's integer rounding rule evaluated on the device."""
    chunk = 1 << 27
    dev = torch.device("cuda")
    for base in range(0, 1 << 32, chunk):
        u = torch.arange(base, base + chunk, dtype=torch.int64, device=dev)
        bits32 = torch.where(u >= (1 << 31), u - (1 << 32), u).to(torch.int32)
        out = hp.f32_to_f16(bits32.view(torch.float32))
        ref = torch_narrow_ref(u)
        assert torch.equal(out.to(torch.int32).to(torch.int64) & 0xFFFF, ref), hex(base)
    # and the device restatement against the numpy oracle on a sample
    rng = np.random.default_rng(5)
    u = rng.integers(0, 2**32, size=1 << 20, dtype=np.uint64)
    got = torch_narrow_ref(torch.from_numpy(u.astype(np.int64)).cuda()).cpu().numpy()
    assert np.array_equal(got.astype(np.uint16), rp.narrow(u.astype(np.uint32).view(np.float32)))


def test_widen_exhaustive(golden):                      # test_halfprec.py:104-110
    g = golden.npz("halfprec_golden.npz")
    mine = hp.f16_to_f32(np.arange(65536, dtype=np.uint16))
    # bitwise, NaNs included: every NaN pattern widens to numpy's 0x7FC00000
    assert np.array_equal(mine.view(np.uint32), g["widen_out"])


def test_roundtrip_exhaustive():                        # test_halfprec.py:113-118
    allbits = np.arange(65536, dtype=np.uint16)
    finite = allbits[((allbits >> 10) & 0x1F) != 31]
    assert np.array_equal(hp.f32_to_f16(hp.f16_to_f32(finite)), finite)


def test_nan_canonical_and_inf():                       # test_halfprec.py:121-128
    assert int(hp.f32_to_f16(np.float32(np.inf))) == 0x7C00
    assert int(hp.f32_to_f16(np.float32(-np.inf))) == 0xFC00
    payloads = np.array([0x7FC00000, 0x7F800001, 0xFFC00000, 0x7FABCDEF], dtype=np.uint32)
    assert np.all(hp.f32_to_f16(payloads.view(np.float32)) == 0x7E00)
    assert math.isnan(hp.f16_to_f32(np.uint16(0x7E01)))


def test_quantize_unscale_golden(golden):
    g = golden.npz("halfprec_golden.npz")
    assert np.array_equal(hp.quantize_tensor(g["q_in"]).view(np.uint32), g["q_out"].view(np.uint32))
    for i, s in enumerate(g["unscale_scales"]):
        got = hp.unscale_gradients(g["g"], float(s))
        assert np.array_equal(got.view(np.uint32), g[f"unscale_{i}"].view(np.uint32))


def test_loss_scale_rescue_and_policy():                # test_halfprec.py:202-255
    g = np.array([2.0**-30], dtype=np.float32)
    ls = hp.LossScale(scale=2.0**10)
    through = hp.f16_to_f32(hp.f32_to_f16(g * np.float32(ls.scale)))
    assert hp.unscale_gradients(through, ls)[0] == np.float32(2.0**-30)
    assert hp.quantize_tensor(g)[0] == 0.0
    ls = hp.LossScale(scale=1024.0, growth_interval=3)
    bad = np.array([np.inf], dtype=np.float32)
    good = np.array([1.0], dtype=np.float32)
    assert ls.update(bad) is False and ls.scale == 512.0
    assert ls.update(good) and ls.update(good) and ls.scale == 512.0
    assert ls.update(good) and ls.scale == 1024.0
    assert ls.update([good, bad]) is False and ls.scale == 512.0
    fixed = hp.LossScale(scale=256.0, policy="fixed")
    assert fixed.update(np.array([np.nan], np.float32)) is False and fixed.scale == 256.0


def test_fused_scale_narrow_flag():
    x = torch.tensor([1.0, 64.0, 100.0], device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = hp.f32_to_f16(x, scale=1024.0, nonfinite=flag)
    assert out.cpu().numpy().tolist() == [0x6400, 0x7C00, 0x7C00]
    assert flag.item() == 1


# ------------------------------------------------------------ fusion

def f32(n, start=0.0):
    return np.arange(start, start + n, dtype=np.float32)


def test_fusion_threshold_rules():                      # test_fusion.py:16-53
    buf = gs.FusionBuffer(1000)
    assert buf.enqueue("a", f32(75)) is None
    assert buf.enqueue("b", f32(75)) is None
    assert buf.pending_bytes == 600
    batch = buf.enqueue("c", f32(125))
    assert batch.nbytes == 1100 and batch.tensor_ids == ["a", "b", "c"]
    assert np.array_equal(batch.payload, np.concatenate([f32(75), f32(75), f32(125)]))
    buf = gs.FusionBuffer(10_000)
    buf.enqueue("a", f32(4))
    buf.enqueue("b", f32(6))
    batch = buf.flush()
    assert batch.unpack_map == (("a", 0, 4), ("b", 4, 6))
    with pytest.raises(ValueError, match="mixed dtypes"):
        buf.enqueue("x", f32(2))
        buf.enqueue("y", np.arange(2, dtype=np.uint16))


def test_fusion_fuzz_payload_bitwise(golden):
    """Golden fuzz maps + bitwise conservation through gs_batched_copy with
    device tensors of odd sizes (unaligned pieces)."""
    rng = np.random.default_rng(0)
    for case in golden.json("fusion_golden.json")["fuzz"]:
        dt = np.uint16 if case["dtype"] == "uint16" else np.float32
        host = [(rng.integers(0, 60000, size=n).astype(dt)) for n in case["sizes"]]
        buf = gs.FusionBuffer(case["theta"])
        batches = []
        for i, t in enumerate(host):
            b = buf.enqueue(f"t{i}", torch.from_numpy(t).cuda())
            if b is not None:
                batches.append(b)
        t = buf.flush()
        if t is not None:
            batches.append(t)
        assert [[list(m) for m in b.unpack_map] for b in batches] == case["maps"]
        got = np.concatenate([b.payload.cpu().numpy() for b in batches]) if batches else \
            np.empty(0, dt)
        assert np.array_equal(got, np.concatenate(host) if host else np.empty(0, dt))
        for b in batches:
            for tid, view in gs.unpack(b):
                assert np.array_equal(view.cpu().numpy(), host[int(tid[1:])])


def test_fusion_large_skewed_copy():
    sizes = [64, 2_359_296, 1, 3, 1_048_583, 0, 17]
    ts = [torch.randint(0, 65535, (n,), dtype=torch.int32, device="cuda").to(torch.uint16)
          for n in sizes]
    buf = gs.FusionBuffer(1 << 40)
    for i, t in enumerate(ts):
        buf.enqueue(f"t{i}", t[1:] if i == 1 else t)   # an unaligned view too
    b = buf.flush()
    want = torch.cat([ts[0], ts[1][1:], *ts[2:]])
    assert torch.equal(b.payload, want)


# ------------------------------------------------------------ collectives

def test_folds_match_reference_golden(golden):
    g = golden.npz("folds_golden.npz")
    for key in g.files:
        if key.startswith("f32_in_"):
            p = key.rsplit("_", 1)[1]
            out, sched = gs.ring_allreduce(list(g[key]))
            assert np.array_equal(out[0].view(np.uint32), g[f"f32_sum_{p}"].view(np.uint32))
            out, _ = gs.ring_allreduce(list(g[key]), op="mean")
            assert np.array_equal(out[-1].view(np.uint32), g[f"f32_mean_{p}"].view(np.uint32))
        if key.startswith("f16_in_"):
            p = key.rsplit("_", 1)[1]
            out, _ = gs.allreduce_f16(list(g[key]))
            assert np.array_equal(out[0], g[f"f16_tree_{p}"]), p


def test_fold_nonfinite_flag():
    a = torch.tensor([0x7BFF, 0x3C00], dtype=torch.int32).to(torch.uint16).cuda()
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = gs.collectives.fold_f16_tree([a, a], nonfinite=flag)
    assert out.cpu().numpy().tolist() == [0x7C00, 0x4000] and flag.item() == 1
    flag.zero_()
    gs.collectives.fold_f16_tree([a[1:], a[1:], a[1:]], nonfinite=flag)
    assert flag.item() == 0


def test_allreduce_api_semantics():                      # test_collectives.py:168-231
    rng = np.random.default_rng(2)
    bufs = [rng.standard_normal(200).astype(np.float32) for _ in range(8)]
    ring, s1 = gs.ring_allreduce(bufs)
    hier, s2 = gs.hierarchical_allreduce(bufs, gs.Topology(8, 2))
    assert np.array_equal(ring[0], hier[0]) and s2.algorithm == "hierarchical"
    out, _ = gs.ring_allreduce([np.full(4, float(i + 1), np.float32) for i in range(4)], op="mean")
    assert np.array_equal(out[0], np.full(4, 2.5, np.float32))
    buf = np.arange(5, dtype=np.float32)
    out, sched = gs.ring_allreduce([buf])
    out[0][0] = -1
    assert buf[0] == 0 and sched.total_steps == 0
    _, sched = gs.hybrid_allreduce([np.ones(25, np.float32)] * 4, gs.Topology(4, 2), 101)
    assert sched.algorithm == "hierarchical"
    tb = [torch.from_numpy(b).cuda() for b in bufs]
    tout, _ = gs.ring_allreduce(tb)
    assert torch.equal(tout[3].cpu(), torch.from_numpy(ring[0]))


def test_f16_allreduce_error_bound():                    # test_collectives.py:237-261
    rng = np.random.default_rng(5)
    for p in (2, 5, 16):
        b32 = [rng.uniform(0.5, 1.5, 2048).astype(np.float32) for _ in range(p)]
        b16 = [hp.f32_to_f16(b) for b in b32]
        out, sched = gs.allreduce_f16(b16)
        ref = rp.fold_ascending(b32)
        assert np.max(np.abs(hp.f16_to_f32(out[0]) - ref) / np.abs(ref)) <= 2.0**-9
        assert sched.bytes_on_wire == 2 * (p - 1) * 2048 * 2


# ------------------------------------------------------------ lars

def test_two_step_momentum_reference():                  # test_lars.py:138-169
    rng = np.random.default_rng(3)
    w0 = rng.uniform(0.5, 1.5, 32).astype(np.float32)
    g1 = rng.standard_normal(32).astype(np.float32) * np.float32(0.1)
    g2 = rng.standard_normal(32).astype(np.float32) * np.float32(0.1)
    cfg = gs.LarsConfig(gs.Schedule(base_lr=0.5), eta=0.001, weight_decay=0.01, momentum=0.9)
    group = gs.make_param_group("w", "weight", w0)

    def norm64(x):
        return float(np.linalg.norm(x.astype(np.float64)))
    wd, m = np.float32(0.01), np.float32(0.9)
    eff1 = g1 + wd * w0
    s1 = np.float32((0.001 * norm64(w0) / norm64(eff1)) * 0.5)
    v1 = s1 * eff1
    w1 = w0 - v1
    eff2 = g2 + wd * w1
    s2 = np.float32((0.001 * norm64(w1) / norm64(eff2)) * 0.5)
    v2 = m * v1 + s2 * eff2
    w2 = w1 - v2
    group.grad.copy_(torch.from_numpy(g1))
    assert gs.lars_step([group], cfg, step=0)
    group.grad.copy_(torch.from_numpy(g2))
    assert gs.lars_step([group], cfg, step=1)
    assert np.array_equal(group.velocity.cpu().numpy(), v2)
    assert np.array_equal(group.master_w.cpu().numpy(), w2)
    assert np.array_equal(group.working_w16.cpu().numpy(), hp.f32_to_f16(w2))


def test_rejects_nonfinite_without_mutation():           # test_lars.py:184-200
    cfg = gs.LarsConfig(gs.Schedule(base_lr=0.1))
    a = gs.make_param_group("a", "weight", np.ones(4))
    b = gs.make_param_group("b", "bias", np.ones(4))
    a.grad.fill_(0.5)
    b.grad.copy_(torch.tensor([0.1, float("nan"), 0.1, 0.1]))
    before = [t.clone() for t in (a.master_w, a.velocity, a.working_w16, b.master_w)]
    assert gs.lars_step([a, b], cfg, step=0) is False
    for x, y in zip(before, (a.master_w, a.velocity, a.working_w16, b.master_w)):
        assert torch.equal(x, y)


def test_local_lr_known_answers(golden):                  # test_lars.py:25-49
    g = golden.npz("lars_golden.npz")
    for i in range(int(g["llr_count"])):
        got = gs.lars_local_lr(g[f"llr_w_{i}"], g[f"llr_g_{i}"], 0.001, float(g[f"llr_eps_{i}"]))
        assert got == pytest.approx(float(g[f"llr_out_{i}"]), rel=1e-12)
    assert gs.lars_local_lr(np.zeros(8, np.float32), np.ones(8, np.float32), 0.001) == 1.0
    assert gs.lars_local_lr(np.ones(8, np.float32), np.zeros(8, np.float32), 0.001) == 1.0


def test_master_accumulation_survives_tiny_updates():    # test_lars.py:223-238
    cfg = gs.LarsConfig(gs.Schedule(base_lr=1.0), weight_decay=0.0, momentum=0.9)
    g = gs.make_param_group("b", "bias", np.ones(512))
    for step in range(200):
        g.grad.fill_(1e-8)
        assert gs.lars_step([g], cfg, step)
    assert bool((g.master_w < 1.0 - 5e-6).all())
    assert bool((hp.f16_to_f32(g.working_w16) == 1.0).all())


def test_checkpoint_roundtrip(tmp_path):                  # test_lars.py:248-279
    cfg = gs.LarsConfig(gs.Schedule(base_lr=0.5))
    groups = [gs.make_param_group("w", "weight", np.linspace(-1, 1, 33)),
              gs.make_param_group("b", "bias", np.ones(5), decay_exempt=False)]
    for g in groups:
        g.grad.fill_(0.25)
    gs.lars_step(groups, cfg, 0)
    gs.save_checkpoint(tmp_path / "c.lars", groups, step=7)
    loaded, step = gs.load_checkpoint(tmp_path / "c.lars")
    assert step == 7 and loaded[1].decay_exempt is False and loaded[0].lars_enabled
    for a, b in zip(groups, loaded):
        assert torch.equal(a.master_w, b.master_w) and torch.equal(a.velocity, b.velocity)
        assert torch.equal(a.working_w16, b.working_w16)
