"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the dev container (where /root/reference exists):
    python tests/golden/make_golden.py
The reference package (pure Python + numpy) is imported from
/root/reference/pkg/src under the name `gradsync_ref`; nothing here is
needed at test time — the tests read only the committed fixture files.

Fixtures:
  halfprec_golden.npz   narrow/widen/quantize/unscale outputs of the reference
  fusion_golden.json    unpack maps (resnet50/alexnet/shufflenet shapes, several
                        thetas, fp16 + fp32) and a random-size fuzz set
  schedules_golden.json ring / hierarchical schedules (reference to_json)
  folds_golden.npz      fold_ascending / fold_f16_tree results for small p
  lars_golden.npz       multi-group, multi-step lars_step trajectories
  step_golden.json      the fp16-wire step composed from reference primitives
                        on config 1 (shufflenet shapes, p=4, Topology(4,2),
                        theta=256 KiB, eta=inf): hashes of master/velocity/
                        working after each step, per-group fp32 scales, flags
  netsim_golden.json    simulate() reports and crossover sweeps of the α-β model
                        (`python tests/golden/make_golden.py make_netsim` alone)
  step32_golden.json    the reference's OWN fp32-wire step body (run_experiment,
                        experiment.py:368-413, with its _fused_allreduce
                        op="mean", experiment.py:282-301) on config-1 shapes
                        with fp32 gradients: hashes per step (`make_step32`)
  checkpoint_golden.lars  a LARS v1 checkpoint written by the reference's
                        save_checkpoint (lars.py:197-207) after two lars_step
                        calls on the first 14 shufflenet tensors, and
  checkpoint_golden.npz the groups' arrays it holds (`make_checkpoint`)
"""

from __future__ import annotations

import hashlib
import importlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
REF_SRC = Path("/root/reference/pkg/src")


def load_reference():
    if "gradsync_ref" in sys.modules:
        return sys.modules["gradsync_ref"]
    spec = importlib.util.spec_from_file_location(
        "gradsync_ref", REF_SRC / "gradsync" / "__init__.py",
        submodule_search_locations=[str(REF_SRC / "gradsync")])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["gradsync_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_halfprec(ref):
    hp = importlib.import_module("gradsync_ref.halfprec")
    rng = np.random.default_rng(1234)
    bits = rng.integers(0, 2**32, size=60_000, dtype=np.uint64).astype(np.uint32)
    # dense coverage of the subnormal / flush / overflow boundaries
    sub = rng.integers(0x32F00000, 0x38900000, size=20_000, dtype=np.uint64).astype(np.uint32)
    ovf = rng.integers(0x477F0000, 0x47810000, size=10_000, dtype=np.uint64).astype(np.uint32)
    special = np.array([0, 0x80000000, 0x3F800000, 0x477FE000, 0x477FF000, 0x477FEFFF,
                        0x33000000, 0x33000001, 0xB3000000, 0x38800000, 0x387FFFFF,
                        0x7F800000, 0xFF800000, 0x7FC00000, 0x7F800001, 0xFFC00000,
                        0x7FABCDEF, 0x00000001, 0x807FFFFF], dtype=np.uint32)
    sign = rng.integers(0, 2, size=sub.size + ovf.size, dtype=np.uint32) << 31
    allbits = np.concatenate([bits, np.concatenate([sub, ovf]) | sign, special])
    x = allbits.view(np.float32)
    narrow_out = hp.f32_to_f16(x)
    h = np.arange(65536, dtype=np.uint16)
    widen_out = hp.f16_to_f32(h).view(np.uint32)
    q_in = (rng.standard_normal(20_000) * 10.0 ** rng.integers(-9, 5, size=20_000)).astype(np.float32)
    q_out = hp.quantize_tensor(q_in)
    g = rng.standard_normal(20_000).astype(np.float32)
    unscale = {s: hp.unscale_gradients(g, s) for s in (1024.0, 3.0, 2.0 ** -3, 65536.0)}
    np.savez_compressed(HERE / "halfprec_golden.npz", narrow_in=allbits, narrow_out=narrow_out,
                        widen_out=widen_out, q_in=q_in, q_out=q_out, g=g,
                        **{f"unscale_{i}": v for i, v in enumerate(unscale.values())},
                        unscale_scales=np.array(list(unscale), dtype=np.float64))


def shapes():
    return json.loads((ROOT / "paper_1807_11205_b200" / "shapes.json").read_text())


def make_fusion(ref):
    fusion = importlib.import_module("gradsync_ref.fusion")
    out = {"models": [], "fuzz": []}
    for model, rows in shapes().items():
        names = [r[0] for r in rows]
        sizes = [int(np.prod(r[1])) for r in rows]
        order = list(reversed(range(len(rows))))
        for dtype in (np.uint16, np.float32):
            thetas = [0, 256 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20, 1 << 40]
            if dtype is np.float32:
                thetas = [4 << 20]
            for theta in thetas:
                buf = fusion.FusionBuffer(theta)
                batches = []
                for i in order:
                    b = buf.enqueue(names[i], np.zeros(sizes[i], dtype=dtype))
                    if b is not None:
                        batches.append(b)
                t = buf.flush()
                if t is not None:
                    batches.append(t)
                out["models"].append({"model": model, "dtype": np.dtype(dtype).name,
                                      "theta": theta, "order": "backward",
                                      "maps": [list(map(list, b.unpack_map)) for b in batches],
                                      "bytes": [b.nbytes for b in batches]})
    rng = np.random.default_rng(99)
    for case in range(300):
        n = int(rng.integers(1, 25))
        sizes = [int(s) for s in rng.integers(0, 60, size=n)]
        theta = int(rng.integers(0, 500))
        dtype = np.uint16 if case % 2 else np.float32
        buf = fusion.FusionBuffer(theta)
        maps = []
        for i, s in enumerate(sizes):
            b = buf.enqueue(f"t{i}", np.zeros(s, dtype=dtype))
            if b is not None:
                maps.append(list(map(list, b.unpack_map)))
        t = buf.flush()
        if t is not None:
            maps.append(list(map(list, t.unpack_map)))
        out["fuzz"].append({"sizes": sizes, "theta": theta, "dtype": np.dtype(dtype).name,
                            "maps": maps})
    (HERE / "fusion_golden.json").write_text(json.dumps(out))


def make_schedules(ref):
    col = importlib.import_module("gradsync_ref.collectives")
    cases = []
    for p, k, n, itemsize in [(1, 1, 10, 4), (2, 1, 7, 4), (2, 2, 7, 2), (3, 1, 10, 4),
                              (4, 2, 1000, 2), (4, 4, 33, 4), (6, 3, 100, 4), (8, 2, 513, 2),
                              (8, 4, 513, 2), (8, 8, 64, 4), (12, 4, 97, 4), (16, 4, 5, 2),
                              (24, 6, 1001, 4), (8, 1, 25557032, 2)]:
        topo = col.Topology(p, k)
        cases.append({"p": p, "k": k, "n": n, "itemsize": itemsize,
                      "ring": col.ring_schedule(p, n, itemsize, k=k).to_json(),
                      "hier": col.hierarchical_schedule(topo, n, itemsize).to_json()})
    (HERE / "schedules_golden.json").write_text(json.dumps(cases))


def make_folds(ref):
    col = importlib.import_module("gradsync_ref.collectives")
    hp = importlib.import_module("gradsync_ref.halfprec")
    rng = np.random.default_rng(7)
    out = {}
    for p in (1, 2, 3, 5, 8, 13):
        bufs = np.stack([(rng.standard_normal(1031) * 10).astype(np.float32) for _ in range(p)])
        out[f"f32_in_{p}"] = bufs
        out[f"f32_sum_{p}"] = col.fold_ascending(list(bufs), "sum")
        out[f"f32_mean_{p}"] = col.fold_ascending(list(bufs), "mean")
    for p in (1, 2, 3, 4, 5, 6, 7, 8, 9, 16, 24, 70):
        vals = rng.standard_normal((p, 1029)).astype(np.float32) * np.float32(3000.0)
        vals[:, :8] = 65504.0 / max(1, p // 2)          # near-overflow sums
        bits = np.stack([hp.f32_to_f16(v) for v in vals])
        bits[0, 10] = 0x7C00                             # +Inf
        bits[p - 1, 11] = 0xFC00                         # -Inf (Inf - Inf -> NaN if p == 1? no)
        bits[0, 12] = 0x7E01                             # NaN payload
        bits[:, 13] = 0x0001                             # subnormals
        out[f"f16_in_{p}"] = bits
        out[f"f16_tree_{p}"] = col.fold_f16_tree(list(bits))
    np.savez_compressed(HERE / "folds_golden.npz", **out)


def make_lars(ref):
    lars = importlib.import_module("gradsync_ref.lars")
    rng = np.random.default_rng(21)
    kinds = ["weight", "bias", "bn_gamma", "bn_beta", "weight", "weight", "bias"]
    sizes = [300, 17, 64, 64, 1, 2049, 0]
    cfgs = [dict(base_lr=0.5, eta=0.001, epsilon=0.0, weight_decay=0.01, momentum=0.9),
            dict(base_lr=0.1, eta=0.002, epsilon=1e-6, weight_decay=0.0, momentum=0.0),
            dict(base_lr=3.0, eta=0.001, epsilon=0.5, weight_decay=5e-4, momentum=0.95,
                 kind="poly", warmup_steps=2, total_steps=6, end_lr=0.1)]
    out = {"sizes": np.array(sizes), "ncfg": np.array(len(cfgs))}
    meta = []
    for ci, c in enumerate(cfgs):
        sched = lars.Schedule(base_lr=c["base_lr"], kind=c.get("kind", "constant"),
                              warmup_steps=c.get("warmup_steps", 0),
                              total_steps=c.get("total_steps", 1), end_lr=c.get("end_lr", 0.0))
        cfg = lars.LarsConfig(schedule=sched, eta=c["eta"], epsilon=c["epsilon"],
                              weight_decay=c["weight_decay"], momentum=c["momentum"])
        groups = []
        for gi, (k, n) in enumerate(zip(kinds, sizes)):
            w0 = (rng.standard_normal(n) * rng.uniform(0.05, 2.0)).astype(np.float32)
            if gi == 4:
                w0[:] = 0.0  # degenerate ||w|| = 0 -> local 1.0
            out[f"c{ci}_w0_{gi}"] = w0
            groups.append(lars.make_param_group(f"g{gi}", k, w0))
        for step in range(4):
            for gi, g in enumerate(groups):
                gr = (rng.standard_normal(g.size) * rng.uniform(1e-4, 1.0)).astype(np.float32)
                if step == 2 and gi == 2 and g.size:
                    gr[3] = np.inf  # rejected step: no mutation
                g.grad[:] = gr
                out[f"c{ci}_s{step}_g_{gi}"] = gr
            ok = lars.lars_step(groups, cfg, step)
            out[f"c{ci}_s{step}_ok"] = np.array(ok)
            for gi, g in enumerate(groups):
                out[f"c{ci}_s{step}_w_{gi}"] = g.master_w.copy()
                out[f"c{ci}_s{step}_v_{gi}"] = g.velocity.copy()
                out[f"c{ci}_s{step}_h_{gi}"] = g.working_w16.copy()
        meta.append(c)
    # lars_local_lr known answers
    llr = []
    for _ in range(30):
        n = int(rng.integers(1, 500))
        w = (rng.standard_normal(n) * rng.uniform(0.01, 10)).astype(np.float32)
        g = (rng.standard_normal(n) * rng.uniform(0.001, 5)).astype(np.float32)
        for eps in (0.0, 1e-6, 0.5):
            llr.append((w, g, eps, lars.lars_local_lr(w, g, 0.001, eps)))
    for i, (w, g, eps, v) in enumerate(llr):
        out[f"llr_w_{i}"], out[f"llr_g_{i}"] = w, g
        out[f"llr_eps_{i}"], out[f"llr_out_{i}"] = np.array(eps), np.array(v)
    out["llr_count"] = np.array(len(llr))
    np.savez_compressed(HERE / "lars_golden.npz", **out)
    (HERE / "lars_golden_meta.json").write_text(json.dumps(meta))


def compose_reference_step(ref, specs, wire, groups, cfg, loss, topo, theta, eta, step):
    """The fp16-wire step from reference primitives."""
    fusion = importlib.import_module("gradsync_ref.fusion")
    col = importlib.import_module("gradsync_ref.collectives")
    hp = importlib.import_module("gradsync_ref.halfprec")
    lars = importlib.import_module("gradsync_ref.lars")
    p = len(wire)
    order = list(reversed(range(len(specs))))
    bufs = [fusion.FusionBuffer(theta) for _ in range(p)]
    batches = [[] for _ in range(p)]
    for i in order:
        for r in range(p):
            b = bufs[r].enqueue(specs[i][0], wire[r][i])
            if b is not None:
                batches[r].append(b)
    for r in range(p):
        t = bufs[r].flush()
        if t is not None:
            batches[r].append(t)
    merged, maps, algos = {}, [], []
    for bi in range(len(batches[0])):
        aligned = [batches[r][bi] for r in range(p)]
        algo = col.choose_algorithm(aligned[0].nbytes, eta)
        res, _ = col.allreduce_f16([a.payload for a in aligned], topo, algorithm=algo)
        algos.append(algo)
        maps.append([list(m) for m in aligned[0].unpack_map])
        for name, t in fusion.unpack(fusion.FusedBatch(res[0], aligned[0].unpack_map)):
            merged[name] = t
    step_scale = loss.scale
    with np.errstate(over="ignore", invalid="ignore"):
        for g in groups:
            g.grad[:] = hp.f16_to_f32(merged[g.name]) / np.float32(p)
        applied = loss.update([g.grad for g in groups])
        grad_norm = 0.0
        if applied:
            for g in groups:
                g.grad[:] = hp.unscale_gradients(g.grad, step_scale)
            grad_norm = float(np.sqrt(sum(float(np.dot(g.grad.astype(np.float64),
                                                       g.grad.astype(np.float64)))
                                          for g in groups)))
            applied = lars.lars_step(groups, cfg, step)
    return {"applied": bool(applied), "scale_used": step_scale, "scale_after": loss.scale,
            "grad_norm": grad_norm, "maps": maps, "algorithms": algos}


def make_step(ref):
    sys.path.insert(0, str(ROOT))
    from paper_1807_11205_b200 import shapes as sh
    lars = importlib.import_module("gradsync_ref.lars")
    hp = importlib.import_module("gradsync_ref.halfprec")
    col = importlib.import_module("gradsync_ref.collectives")
    model, p, k, theta = "shufflenet_v2_x0_5", 4, 2, 256 << 10
    specs_obj = sh.load_shapes(model)
    specs = [(s.name, s.numel, s.kind) for s in specs_obj]
    master = sh.synth_master(specs_obj, seed=0)
    groups, o = [], 0
    for name, n, kind in specs:
        groups.append(lars.make_param_group(name, kind, master[o:o + n]))
        o += n
    sched = lars.Schedule(base_lr=0.1)
    cfg = lars.LarsConfig(schedule=sched, eta=0.001, epsilon=0.0, weight_decay=5e-4,
                          momentum=0.9)
    loss = hp.LossScale(scale=1024.0)
    topo = col.Topology(p, k)
    steps = []
    for step in range(3):
        wire = []
        for r in range(p):
            flat = sh.synth_wire_grads(specs_obj, rank=r, seed=step, loss_scale=loss.scale)
            if step == 2 and r == 1:
                flat[12345] = 0x7C00  # injected overflow -> skip, scale halves
            parts, o = [], 0
            for _, n, _ in specs:
                parts.append(flat[o:o + n])
                o += n
            wire.append(parts)
        res = compose_reference_step(ref, specs, wire, groups, cfg, loss, topo, theta,
                                     1 << 40, step)
        res["master_sha"] = sha(np.concatenate([g.master_w for g in groups]))
        res["velocity_sha"] = sha(np.concatenate([g.velocity for g in groups]))
        res["working_sha"] = sha(np.concatenate([g.working_w16 for g in groups]))
        res["master_probe"] = [float(x) for x in np.concatenate([g.master_w for g in groups])[::9973]]
        steps.append(res)
    doc = {"model": model, "p": p, "k": k, "theta": theta, "eta_bytes": 1 << 40,
           "lr": 0.1, "eta": 0.001, "epsilon": 0.0, "weight_decay": 5e-4, "momentum": 0.9,
           "loss_scale": 1024.0, "grad_seed_is_step": True, "inject": {"step": 2, "rank": 1,
                                                                      "index": 12345},
           "steps": steps}
    (HERE / "step_golden.json").write_text(json.dumps(doc))


def make_netsim(ref):
    """netsim_golden.json: reference simulate() reports and crossover sweeps
    (pkg/src/gradsync/netsim.py:77-170) over ring / hierarchical schedules
    and several link models, floats stored as repr so the check is bitwise."""
    col = importlib.import_module("gradsync_ref.collectives")
    ns = importlib.import_module("gradsync_ref.netsim")
    links = [dict(alpha=1e-5, beta_inv=1e9),
             dict(alpha=2.5e-6, beta_inv=3.7e11, intra_group_alpha=1.1e-6,
                  intra_group_beta_inv=8.9e11),
             dict(alpha=0.0, beta_inv=1e9, intra_group_beta_inv=7e10),
             dict(alpha=1.3e-5, beta_inv=2.2e10, intra_group_alpha=0.0)]
    sims = []
    for (p, k, n, itemsize) in [(2, 1, 1000, 4), (4, 2, 200, 4), (8, 4, 12345, 2),
                                (16, 4, 1_000_003, 2), (64, 8, 25_557_032, 2),
                                (6, 3, 7, 4), (1, 1, 100, 4)]:
        for li, lk in enumerate(links):
            link = ns.LinkModel(**lk)
            for name, sched in (("ring", col.ring_schedule(p, n, itemsize, k=k)),
                                ("hierarchical", col.hierarchical_schedule(
                                    col.Topology(p, k), n, itemsize))):
                rep = ns.simulate(sched, link)
                sims.append({"p": p, "k": k, "n": n, "itemsize": itemsize, "link": li,
                             "schedule": name, "total_time": repr(rep.total_time),
                             "per_phase": {ph: repr(t) for ph, t in rep.per_phase_time.items()},
                             "total_steps": rep.total_steps, "bytes_on_wire": rep.bytes_on_wire})
    sweeps = []
    for (p, k, li) in [(64, 8, 0), (16, 4, 1), (8, 2, 3), (4, 2, 1)]:
        sizes = [4 * 10**i for i in range(9)] + [1 << s for s in range(10, 31, 4)]
        rows = ns.crossover_sweep(p, k, ns.LinkModel(**links[li]), sizes)
        sweeps.append({"p": p, "k": k, "link": li, "sizes": sizes,
                       "rows": [{"bytes": r["bytes"], "ring_time": repr(r["ring_time"]),
                                 "hierarchical_time": repr(r["hierarchical_time"]),
                                 "faster": r["faster"]} for r in rows],
                       "crossover": ns.find_crossover(rows)})
    (HERE / "netsim_golden.json").write_text(json.dumps({"links": links, "simulate": sims,
                                                         "sweeps": sweeps}))


def make_step32(ref):
    """run_experiment's step body verbatim in structure, minus the toy
    model: per-worker FusionBuffer over fp32 gradients in registration order
    (experiment.py:369-379), experiment._fused_allreduce per bucket (hybrid
    choice, op="mean"), unpack, LossScale.update on the scaled mean,
    unscale_gradients, grad norm, lars_step (experiment.py:395-412)."""
    sys.path.insert(0, str(ROOT))
    from paper_1807_11205_b200 import shapes as sh
    fusion = importlib.import_module("gradsync_ref.fusion")
    col = importlib.import_module("gradsync_ref.collectives")
    hp = importlib.import_module("gradsync_ref.halfprec")
    lars = importlib.import_module("gradsync_ref.lars")
    exp = importlib.import_module("gradsync_ref.experiment")
    netsim = importlib.import_module("gradsync_ref.netsim")
    model, p, k, theta, eta = "shufflenet_v2_x0_5", 4, 2, 256 << 10, 1 << 40
    specs_obj = sh.load_shapes(model)
    master = sh.synth_master(specs_obj, seed=0)
    groups, o = [], 0
    for s in specs_obj:
        groups.append(lars.make_param_group(s.name, s.kind, master[o:o + s.numel]))
        o += s.numel
    cfg = lars.LarsConfig(schedule=lars.Schedule(base_lr=0.1), eta=0.001, epsilon=0.0,
                          weight_decay=5e-4, momentum=0.9)
    scale = hp.LossScale(scale=1024.0)
    topo = col.Topology(p, k)
    link = netsim.LinkModel()
    steps = []
    for step in range(3):
        step_scale = scale.scale
        worker_grads = []
        for r in range(p):
            flat = sh.synth_grads_f32(specs_obj, rank=r, seed=step) * np.float32(step_scale)
            if step == 2 and r == 1:
                flat[12345] = np.inf
            d, o = {}, 0
            for s in specs_obj:
                d[s.name] = flat[o:o + s.numel]
                o += s.numel
            worker_grads.append(d)
        buffers = [fusion.FusionBuffer(theta) for _ in range(p)]
        step_batches = [[] for _ in range(p)]
        for g in groups:
            for w in range(p):
                emitted = buffers[w].enqueue(g.name, worker_grads[w][g.name])
                if emitted is not None:
                    step_batches[w].append(emitted)
        for w in range(p):
            tail = buffers[w].flush()
            if tail is not None:
                step_batches[w].append(tail)
        merged, algos, maps = {}, [], []
        for b_idx in range(len(step_batches[0])):
            aligned = [step_batches[w][b_idx] for w in range(p)]
            mean_payload, algorithm, _, _ = exp._fused_allreduce(aligned, topo, link, eta, None)
            algos.append(algorithm)
            maps.append([list(m) for m in aligned[0].unpack_map])
            for name, tensor in fusion.unpack(fusion.FusedBatch(mean_payload,
                                                                aligned[0].unpack_map)):
                merged[name] = tensor
        for g in groups:
            g.grad[:] = merged[g.name]
        with np.errstate(over="ignore", invalid="ignore"):
            applied = scale.update([g.grad for g in groups])
            grad_norm = 0.0
            if applied:
                for g in groups:
                    g.grad[:] = hp.unscale_gradients(g.grad, step_scale)
                grad_norm = float(np.sqrt(sum(float(np.dot(g.grad.astype(np.float64),
                                                           g.grad.astype(np.float64)))
                                              for g in groups)))
                applied = lars.lars_step(groups, cfg, step)
        steps.append({"applied": bool(applied), "scale_used": step_scale,
                      "scale_after": scale.scale, "grad_norm": grad_norm, "maps": maps,
                      "algorithms": algos,
                      "master_sha": sha(np.concatenate([g.master_w for g in groups])),
                      "velocity_sha": sha(np.concatenate([g.velocity for g in groups])),
                      "working_sha": sha(np.concatenate([g.working_w16 for g in groups]))})
    doc = {"model": model, "p": p, "k": k, "theta": theta, "eta_bytes": eta, "lr": 0.1,
           "eta": 0.001, "epsilon": 0.0, "weight_decay": 5e-4, "momentum": 0.9,
           "loss_scale": 1024.0, "inject": {"step": 2, "rank": 1, "index": 12345},
           "grads": "shapes.synth_grads_f32(rank, seed=step) * scale (fp32)",
           "order": "registration (experiment.py:371)", "steps": steps}
    (HERE / "step32_golden.json").write_text(json.dumps(doc))


def make_checkpoint(ref):
    lars = importlib.import_module("gradsync_ref.lars")
    spec = json.loads((ROOT / "paper_1807_11205_b200" / "shapes.json").read_text())
    rows = spec["shufflenet_v2_x0_5"][:14]
    rng = np.random.default_rng(77)
    groups = []
    for name, shape, kind in rows:
        n = int(np.prod(shape)) if shape else 1
        w0 = (rng.standard_normal(n) * 0.1).astype(np.float32)
        groups.append(lars.make_param_group(name, kind, w0))
    cfg = lars.LarsConfig(schedule=lars.Schedule(base_lr=0.1), eta=0.001, epsilon=0.0,
                          weight_decay=5e-4, momentum=0.9)
    for step in range(2):
        for g in groups:
            g.grad[:] = (rng.standard_normal(g.size) * 1e-3).astype(np.float32)
        assert lars.lars_step(groups, cfg, step)
    lars.save_checkpoint(HERE / "checkpoint_golden.lars", groups, step=2)
    out = {"names": np.array([g.name for g in groups]), "kinds": np.array([g.kind for g in groups]),
           "shapes": np.array([json.dumps(r[1]) for r in rows])}
    for i, g in enumerate(groups):
        out[f"w_{i}"], out[f"v_{i}"], out[f"h_{i}"] = g.master_w, g.velocity, g.working_w16
    np.savez_compressed(HERE / "checkpoint_golden.npz", **out)


def main():
    ref = load_reference()
    fns = (make_halfprec, make_fusion, make_schedules, make_folds, make_lars, make_step,
           make_netsim, make_checkpoint, make_step32)
    only = set(sys.argv[1:])
    for fn in fns:
        if only and fn.__name__ not in only:
            continue
        fn(ref)
        print("wrote", fn.__name__)


if __name__ == "__main__":
    main()
