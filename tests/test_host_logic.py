"""Host-side logic of the drop-in package against the reference's goldens (CPU)."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_1807_11205_b200 as gs
from paper_1807_11205_b200 import _native, shapes as sh
from paper_1807_11205_b200._plan import _pow2_rcp, build_chunks, step_params
from paper_1807_11205_b200.collectives import ReduceSchedule, _validated
from paper_1807_11205_b200.pipeline import BUCKET_ALIGN, plan_layout

ROOT = Path(__file__).resolve().parent.parent


def test_schedules_match_reference_golden(golden):
    for case in golden.json("schedules_golden.json"):
        topo = gs.Topology(case["p"], case["k"])
        ring = gs.ring_schedule(case["p"], case["n"], case["itemsize"], k=case["k"])
        hier = gs.hierarchical_schedule(topo, case["n"], case["itemsize"])
        assert ring.to_json() == case["ring"], case
        assert hier.to_json() == case["hier"], case
        assert ReduceSchedule.from_json(case["hier"]).to_json() == case["hier"]


@pytest.mark.parametrize("p,k", [(1024, 16), (16, 4), (64, 8)])
def test_step_counts(p, k):                        # test_collectives.py:56-69
    assert gs.ring_schedule(p, 64).total_steps == 2 * (p - 1)
    assert gs.hierarchical_schedule(gs.Topology(p, k), 64).total_steps == \
        4 * (k - 1) + 2 * (p // k - 1)


def test_topology_and_selector():                  # test_collectives.py:33-50, 207-215
    t = gs.Topology(8, 2)
    assert t.group_count == 4 and t.masters() == [0, 2, 4, 6]
    assert list(t.members(1)) == [2, 3] and t.group_of(5) == 2
    for p, k in [(0, 1), (4, 3), (4, 0), (2, 4)]:
        with pytest.raises(ValueError):
            gs.Topology(p, k)
    assert gs.choose_algorithm(100, 101) == "hierarchical"
    assert gs.choose_algorithm(100, 100) == "ring"
    assert gs.choose_algorithm(100, 0) == "ring"
    assert gs.chunk_sizes(7, 4).tolist() == [2, 2, 2, 1]
    assert gs.chunk_sizes(3, 8).tolist() == [1, 1, 1, 0, 0, 0, 0, 0]


def test_validation_messages():                    # test_collectives.py:218-231
    good = np.ones(4, np.float32)
    with pytest.raises(ValueError, match="at least one"):
        gs.ring_allreduce([])
    with pytest.raises(ValueError, match="expected float32"):
        gs.ring_allreduce([good.astype(np.float64)] * 2)
    with pytest.raises(ValueError, match="shape"):
        gs.ring_allreduce([good, np.ones(5, np.float32)])
    with pytest.raises(ValueError, match="expected uint16"):
        gs.allreduce_f16([good, good])


def test_fusion_plan_matches_reference_golden(golden):
    doc = golden.json("fusion_golden.json")
    for case in doc["models"]:
        specs = sh.load_shapes(case["model"])
        order = list(reversed(range(len(specs))))
        itemsize = 2 if case["dtype"] == "uint16" else 4
        plan = gs.plan_buckets([specs[i].numel for i in order], itemsize, case["theta"])
        maps = []
        for b in plan:
            off, m = 0, []
            for q in b:
                s = specs[order[q]]
                m.append([s.name, off, s.numel])
                off += s.numel
            maps.append(m)
        assert maps == case["maps"]
        # the pipeline's wire layout: binary16 and the fp32 wire alike
        wire_off, buckets, total = plan_layout(specs, order, case["theta"], itemsize)
        assert [[list(x) for x in b.unpack_map] for b in buckets] == case["maps"]
        assert [b.nbytes for b in buckets] == case["bytes"]
        for b in buckets:
            assert b.start % BUCKET_ALIGN == 0 and b.padded >= b.length
    for case in doc["fuzz"]:
        itemsize = 2 if case["dtype"] == "uint16" else 4
        plan = gs.plan_buckets(case["sizes"], itemsize, case["theta"])
        maps = [[[f"t{i}", sum(case["sizes"][j] for j in b[:b.index(i)]), case["sizes"][i]]
                 for i in b] for b in plan]
        assert maps == case["maps"]


def test_fusion_validation_and_unpack():           # test_fusion.py:95-120
    with pytest.raises(ValueError):
        gs.FusionBuffer(-1)
    batch = gs.FusedBatch(payload=np.arange(10, dtype=np.float32),
                          unpack_map=(("a", 0, 4), ("b", 5, 5)))
    with pytest.raises(ValueError, match="corrupt unpack map"):
        gs.unpack(batch)
    short = gs.FusedBatch(payload=np.arange(10, dtype=np.float32), unpack_map=(("a", 0, 4),))
    with pytest.raises(ValueError, match="covers 4 of 10"):
        gs.unpack(short)
    ok = gs.FusedBatch(payload=np.arange(10, dtype=np.float32),
                       unpack_map=(("a", 0, 4), ("b", 4, 6)))
    parts = gs.unpack(ok)
    assert parts[1][1].tolist() == list(range(4, 10))
    rec = gs.trace_record(3, 0, ok)
    assert rec == {"step": 3, "batch_index": 0, "tensor_ids": ["a", "b"], "bytes": 40}


def test_loss_scale_state_machine():               # test_halfprec.py:225-255
    ls = gs.LossScale(scale=1024.0, growth_interval=3)
    assert ls.update_from_flag(True) is False and ls.scale == 512.0
    assert ls.update_from_flag(False) and ls.update_from_flag(False) and ls.scale == 512.0
    assert ls.update_from_flag(False) and ls.scale == 1024.0 and ls.clean_steps == 0
    ls = gs.LossScale()
    for _ in range(199):
        ls.update_from_flag(False)
    assert ls.scale == 1024.0
    ls.update_from_flag(False)
    assert ls.scale == 2048.0
    fixed = gs.LossScale(scale=256.0, policy="fixed", growth_interval=1)
    assert fixed.update_from_flag(True) is False and fixed.update_from_flag(False)
    assert fixed.scale == 256.0
    for bad in (dict(scale=0.0), dict(policy="x"), dict(growth_factor=1.0),
                dict(backoff_factor=1.0), dict(growth_interval=0)):
        with pytest.raises(ValueError):
            gs.LossScale(**bad)
    assert gs.apply_loss_scale(0.5, gs.LossScale(scale=1024.0)) == 512.0


def test_describe_half():
    d = gs.describe_half(0x3C00)
    assert d["category"] == "normal" and d["value"] == 1.0 and d["bits"] == "0x3C00"
    assert gs.describe_half(0x0001)["value"] == 2.0 ** -24
    assert gs.describe_half(0x7E00)["category"] == "nan"
    assert gs.describe_half(0xFC00)["value"] == float("-inf")
    with pytest.raises(ValueError):
        gs.describe_half(0x10000)


def test_schedule_and_config():                    # test_lars.py:63-129
    s = gs.Schedule(base_lr=0.8, warmup_steps=10)
    assert s.lr(0) == 0.0 and s.lr(5) == pytest.approx(0.4) and s.lr(10) == 0.8
    s = gs.Schedule(base_lr=1.0, kind="poly", total_steps=100)
    assert s.lr(50) == pytest.approx(0.25) and s.lr(150) == 0.0
    with pytest.raises(ValueError, match="base_lr"):
        gs.Schedule(base_lr=0.0)
    with pytest.raises(ValueError, match="kind"):
        gs.Schedule(base_lr=1.0, kind="cosine")
    with pytest.raises(ValueError, match="total_steps"):
        gs.Schedule(base_lr=1.0, kind="poly", warmup_steps=10, total_steps=10)
    with pytest.raises(ValueError, match="end_lr"):
        gs.Schedule(base_lr=1.0, kind="poly", total_steps=10, end_lr=2.0)
    with pytest.raises(ValueError, match="eta"):
        gs.LarsConfig(gs.Schedule(1.0), eta=0.0)
    with pytest.raises(ValueError, match="momentum"):
        gs.LarsConfig(gs.Schedule(1.0), momentum=1.0)
    with pytest.raises(ValueError, match="weight_decay"):
        gs.LarsConfig(gs.Schedule(1.0), weight_decay=-0.1)


def test_param_group_validation():                 # test_lars.py:109-129
    ok = np.zeros(3, dtype=np.float32)
    with pytest.raises(ValueError, match="kind"):
        gs.ParamGroup("x", "conv", ok, ok, ok, np.zeros(3, np.uint16))
    with pytest.raises(TypeError, match="grad"):
        gs.ParamGroup("x", "weight", ok, ok.astype(np.float64), ok.copy(),
                      np.zeros(3, np.uint16))
    with pytest.raises(ValueError, match="velocity"):
        gs.ParamGroup("x", "weight", ok, ok.copy(), np.zeros(5, np.float32),
                      np.zeros(3, np.uint16))


def test_chunk_table_and_params():
    chunks, begin, count = build_chunks([10, 0, 20000, 8192], order=[3, 2, 1, 0],
                                        chunk_elems=8192)
    assert count.tolist() == [1, 0, 3, 1]
    assert begin.tolist()[3] == 0 and begin.tolist()[2] == 1 and begin.tolist()[0] == 4
    assert chunks["len"].tolist() == [8192, 8192, 8192, 20000 - 16384, 10]
    assert chunks["seg"].tolist() == [3, 2, 2, 2, 0]
    assert _pow2_rcp(np.float32(1024.0)) == (True, np.float32(1 / 1024))
    assert _pow2_rcp(np.float32(1000.0))[0] is False
    assert _pow2_rcp(np.float32(2.0 ** -3))[0] is True
    p = step_params(eta=0.001, epsilon=0.0, gamma=0.1, weight_decay=5e-4, momentum=0.9,
                    mean_divisor=8, unscale_divisor=1024.0, grad_norm=True)
    m = int(p["mode"][0])
    assert m & _native.MODE_DIV1 and m & _native.MODE_DIV1_POW2 and m & _native.MODE_DIV2_POW2
    assert m & _native.MODE_DECAY and m & _native.MODE_GRADNORM
    p = step_params(eta=0.001, epsilon=0.0, gamma=0.1, weight_decay=0.0, momentum=0.9,
                    mean_divisor=3)
    assert not int(p["mode"][0]) & _native.MODE_DECAY
    assert not int(p["mode"][0]) & _native.MODE_DIV1_POW2


def test_shapes_frozen():
    assert len(sh.load_shapes("resnet50")) == 161
    assert sh.total_params(sh.load_shapes("resnet50")) == 25_557_032
    assert sh.total_params(sh.load_shapes("alexnet")) == 61_100_840
    assert sh.total_params(sh.load_shapes("shufflenet_v2_x0_5")) == 1_366_792
    kinds = [s.kind for s in sh.load_shapes("resnet50")]
    assert kinds.count("weight") == 54 and kinds.count("bias") == 1


def test_specs_from_module_kind_map():
    """overlap.specs_from_module follows the shapes.json kind map:
    BN weight/bias -> bn_gamma/bn_beta, dim > 1 -> weight, other 1-D -> bias."""
    import torch
    from paper_1807_11205_b200.overlap import specs_from_module

    net = torch.nn.Sequential(torch.nn.Conv2d(3, 4, 3), torch.nn.BatchNorm2d(4),
                              torch.nn.Flatten(), torch.nn.Linear(4, 2))
    specs = specs_from_module(net)
    assert [(s.name, s.kind) for s in specs] == [
        ("0.weight", "weight"), ("0.bias", "bias"), ("1.weight", "bn_gamma"),
        ("1.bias", "bn_beta"), ("3.weight", "weight"), ("3.bias", "bias")]
    assert [s.shape for s in specs][0] == (4, 3, 3, 3)
    # same map as the frozen torchvision shape lists
    r50 = sh.load_shapes("resnet50")
    assert sum(s.kind == "bn_gamma" for s in r50) == 53


@pytest.mark.parametrize("model,theta,p", [("resnet50", 16 << 20, 2), ("resnet50", 256 << 10, 4),
                                           ("alexnet", 4 << 20, 8),
                                           ("shufflenet_v2_x0_5", 256 << 10, 8)])
def test_shard_buckets_cover_every_chunk_once(model, theta, p):
    """Sharded-update ownership (pipeline.shard_buckets): per bucket the p
    chunk ranges tile the bucket's chunks, the element bounds tile the padded
    bucket and agree with the chunk starts, and the split is balanced to
    within one chunk."""
    from paper_1807_11205_b200.pipeline import shard_buckets
    specs = sh.load_shapes(model)
    order = list(reversed(range(len(specs))))
    wire_off, buckets, _ = plan_layout(specs, order, theta)
    chunks, begin, count = build_chunks([s.numel for s in specs], order)
    c = 0
    for bk in buckets:
        bk.chunk0, bk.nchunk = c, int(sum(int(count[i]) for i in bk.params))
        c += bk.nchunk
    abs_start = np.array([wire_off[int(x["seg"])] + int(x["start"]) for x in chunks])
    Cs, Es = shard_buckets(buckets, abs_start, p)
    owned = np.zeros(len(chunks), dtype=int)
    for bk, C, E in zip(buckets, Cs, Es):
        assert C[0] == bk.chunk0 and C[-1] == bk.chunk0 + bk.nchunk and C == sorted(C)
        assert E[0] == bk.start and E[-1] == bk.start + bk.padded and E == sorted(E)
        for q in range(p):
            owned[C[q]:C[q + 1]] += 1
            if C[q] < C[q + 1]:
                assert E[q] == abs_start[C[q]]
                last = C[q + 1] - 1
                assert abs_start[last] + int(chunks[last]["len"]) <= E[q + 1]
            share = sum(int(chunks[k]["len"]) for k in range(C[q], C[q + 1]))
            assert share <= bk.length // p + 8192 + 1
    assert (owned == 1).all()
