#!/usr/bin/env python
"""Benchmark: fused MP-LARS step time + all-reduce bus bandwidth on ResNet-50
gradients (BASELINE.json), 1..8 B200, one process per GPU.

  python bench.py [--gpus N --steps K --warmup W]          # our arm
  python bench.py --impl reference [...]                   # the reference's
                                                           # CPU path (oracle)

One step = pack the rank's 161 fp16 gradient tensors into theta-buckets ->
all-reduce every bucket over NCCL (N > 1) -> pass 1 (mean, overflow flags,
unscale, fp64 segment norms) -> trust ratios -> pass 2 (momentum / master /
working-copy update) -> read the flags (the one host sync).  Inputs are
resident in HBM; L2 is flushed (256 MiB written, then read back so it is
left clean) before every timed step and each step is timed alone with CUDA events on the launching stream; the value
is the mean step time, max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fused MP-LARS step time (ms) + allreduce bus GB/s, ResNet-50 grads, 1/2/4/8 B200"
PIECE = "pass2"   # dominant kernel for the roofline line


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--theta", type=int, default=16 << 20, help="fusion threshold (bytes)")
    ap.add_argument("--algorithm", default="zero",
                    choices=["ring", "hierarchical", "sharded", "ordered", "zero", "zero_unfused"],
                    help="gradient exchange at N > 1: zero (default) = sharded ZeRO-1 step in "
                         "fused kernels (reduce-scatter + pass 1, pass 2 + working-weight push); "
                         "zero_unfused = the same with separate collective kernels; ordered = "
                         "own bit-exact NVLink all-reduce + replicated update; "
                         "ring/hierarchical/sharded = NCCL all-reduce + replicated update")
    ap.add_argument("--group-size", type=int, default=4, help="k of Topology(p, k)")
    ap.add_argument("--eta-bytes", type=int, default=None,
                    help="hybrid threshold; default: 0 for ring, inf otherwise")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-allreduce-sweep", action="store_true")
    ap.add_argument("--overflow", action="store_true",
                    help="forced overflow: rank 0's gradient carries +Inf, every step takes "
                         "the skip path (fixed loss-scale policy so the scale stays put)")
    ap.add_argument("--no-soak", action="store_true", help="skip the clock soak (profiling runs)")
    ap.add_argument("--loss-scale", type=float, default=1024.0,
                    help="initial loss scale (a non-power-of-two value takes the IEEE-division "
                         "kernels)")
    ap.add_argument("--wire", default="f16", choices=["f16", "f32"],
                    help="f32: the reference's own run_experiment path (fp32 gradients fused at "
                         "4 B/element, mean all-reduce); replicated update only")
    ap.add_argument("--no-grad-norm", action="store_true",
                    help="A/B only: do not compute the grad-norm metric (experiment.py:408-411)")
    return ap.parse_args(argv)


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ shared

def workload_config(args, world: int) -> dict:
    """The config object both arms print (same keys, same values)."""
    from paper_1807_11205_b200 import shapes as sh
    from paper_1807_11205_b200.fusion import plan_buckets

    specs = sh.load_shapes(args.model)
    sizes = [s.numel for s in specs]
    nb = len(plan_buckets([sizes[i] for i in reversed(range(len(sizes)))], 2, args.theta))
    algo = args.algorithm if world > 1 else "none"
    k = args.group_size if algo in ("hierarchical", "sharded") and world % args.group_size == 0 \
        else 1
    extra = {} if getattr(args, "loss_scale", 1024.0) == 1024.0 else {"loss_scale": args.loss_scale}
    if getattr(args, "wire", "f16") != "f16":
        extra["wire"] = args.wire
    wire = "fp16" if getattr(args, "wire", "f16") == "f16" else "fp32"
    return {**extra, "workload": f"{args.model} fused MP-LARS step, {wire} wire, p={world}",
            "model": args.model, "params": sum(sizes), "tensors": len(specs),
            "theta": args.theta, "buckets": nb, "algorithm": algo,
            "topology": f"Topology({world},{k})" if world > 1 else "1 GPU",
            "forced_overflow": bool(args.overflow), "parallelism": f"dp{world}"}


def host_info() -> dict:
    """CPU model, core count and the numpy / BLAS build of this host."""
    import platform

    import numpy as np
    model = platform.processor() or ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = f"{b.get('name', '?')} {b.get('version', '')}".strip()
    except Exception:  # noqa: BLE001 - informational only
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "numpy": np.__version__, "blas": blas,
            "openblas_num_threads": os.environ.get("OPENBLAS_NUM_THREADS")}


# ------------------------------------------------------------------ reference arm

def cpu_reference(model: str, p: int, theta: int, eta_bytes: int, steps: int, warmup: int,
                  budget_s: float = 150.0) -> dict:
    """The reference's CPU implementation of the path (the oracle port of
    pkg/src/gradsync composed per SURVEY.md §8a-14), p workers simulated in one
    process as the reference does, on this host's cores."""
    import numpy as np
    from oracle import reference_port as rp
    from paper_1807_11205_b200 import shapes as sh

    specs = sh.load_shapes(model)
    names = [s.name for s in specs]
    sizes = [s.numel for s in specs]
    order = list(reversed(range(len(specs))))
    master = sh.synth_master(specs, seed=0)
    groups, o = [], 0
    for s in specs:
        w = master[o:o + s.numel].copy()
        groups.append(rp.Group(s.name, s.kind, w, np.zeros(s.numel, np.float32),
                               np.zeros(s.numel, np.float32), rp.narrow(w)))
        o += s.numel
    wires = []
    for r in range(p):
        flat = sh.synth_wire_grads(specs, rank=r, seed=0)
        parts, o = [], 0
        for s in specs:
            parts.append(flat[o:o + s.numel])
            o += s.numel
        wires.append(parts)
    hp = rp.LarsHyper(0.001, 0.0, 5e-4, 0.9)
    threads = rp.default_threads()
    # first (untimed) step sizes the sample
    t0 = time.perf_counter()
    rp.compose_step_fp16(wires, names, sizes, order, groups, hp, 0.1,
                         rp.LossScaleState(1024.0), theta, eta_bytes, threads=threads)
    t_full = time.perf_counter() - t0
    total = steps + max(0, warmup - 1)
    frac = 1.0
    if t_full * total > budget_s:
        frac = max(0.02, budget_s / (t_full * total))
    # sample = the first `frac` of the wire (backward order), whole tensors
    if frac < 1.0:
        keep, acc, target = [], 0, frac * sum(sizes)
        for i in order:
            if acc >= target:
                break
            keep.append(i)
            acc += sizes[i]
        frac = acc / sum(sizes)
        sub = sorted(keep)
        remap = {old: new for new, old in enumerate(sub)}
        s_names = [names[i] for i in sub]
        s_sizes = [sizes[i] for i in sub]
        s_groups = [groups[i] for i in sub]
        s_wires = [[w[i] for i in sub] for w in wires]
        s_order = [remap[i] for i in order if i in remap]
    else:
        s_names, s_sizes, s_groups, s_wires, s_order = names, sizes, groups, wires, order
    for _ in range(max(0, warmup - 1)):
        rp.compose_step_fp16(s_wires, s_names, s_sizes, s_order, s_groups, hp, 0.1,
                             rp.LossScaleState(1024.0), theta, eta_bytes, threads=threads)
    times = []
    stages: dict = {}
    for _ in range(steps):
        marks = []
        t0 = time.perf_counter()
        rp.compose_step_fp16(s_wires, s_names, s_sizes, s_order, s_groups, hp, 0.1,
                             rp.LossScaleState(1024.0), theta, eta_bytes, threads=threads,
                             timer=lambda name: marks.append((name, time.perf_counter())))
        times.append((time.perf_counter() - t0) / frac)
        for (a, ta), (_, tb) in zip(marks, marks[1:]):
            stages.setdefault(a, []).append((tb - ta) / frac)
    ms = 1e3 * statistics.mean(times)
    return {"ms": ms, "threads": threads, "frac": frac, "t_full_s": t_full, "params": sum(sizes),
            "stages_ms": {k: round(1e3 * statistics.median(v), 2) for k, v in stages.items()},
            "sample": (f"{model} p={p} theta={theta}: "
                       + ("full workload" if frac == 1.0 else
                          f"first {frac:.3f} of the parameters (wire order), time scaled by 1/frac")
                       + f", {steps} timed steps")}


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    flat = args.algorithm in ("ring", "ordered", "zero", "zero_unfused")
    eta = args.eta_bytes if args.eta_bytes is not None else (0 if flat else 1 << 62)
    r = cpu_reference(args.model, world, args.theta, eta, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(r["ms"], 3), "unit": "ms",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(r["ms"], 3), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": round(r["ms"], 3), "unit": "ms", "cores": r["threads"],
                         "kind": "port", "sample": r["sample"] + f"; p={world} workers simulated "
                         "in one process as the reference does", "stages_ms": r["stages_ms"],
                         **host_info()},
        "e2e": {"value": round(r["ms"], 3), "unit": "ms", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm

def run_ours(args, rank: int, world: int, local: int) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1807_11205_b200 as gs
    from paper_1807_11205_b200 import _native, shapes as sh
    from paper_1807_11205_b200.dist import Communicator

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    specs = sh.load_shapes(args.model)
    n_params = sh.total_params(specs)
    comm = None
    if world > 1:
        k = args.group_size if args.algorithm in ("hierarchical", "sharded") else 1
        comm = Communicator(gs.Topology(world, k if world % k == 0 else 1))
    flat = args.algorithm in ("ring", "ordered", "zero", "zero_unfused")
    eta = args.eta_bytes if args.eta_bytes is not None else (0 if flat else 1 << 62)
    cfg = gs.LarsConfig(gs.Schedule(base_lr=0.1), eta=0.001, epsilon=0.0, weight_decay=5e-4,
                        momentum=0.9)
    pipe = gs.GradientPipeline(specs, cfg, threshold_bytes=args.theta, comm=comm, eta_bytes=eta,
                               hier_variant=args.algorithm if not flat else "hierarchical",
                               flat_variant="ordered" if args.algorithm == "ordered" else "ring",
                               sharded_update=(args.algorithm.startswith("zero") and world > 1
                                               and args.wire == "f16"),
                               fused_collective=args.algorithm == "zero",
                               wire_dtype=args.wire,
                               init_master=sh.synth_master(specs, seed=0),
                               loss_scale=gs.LossScale(args.loss_scale, policy="fixed" if args.overflow
                                                       else "dynamic"), device=dev,
                               grad_norm=not args.no_grad_norm)
    wire_np = sh.synth_wire_grads(specs, rank=rank, seed=0)
    if args.overflow and rank == 0:
        wire_np[len(wire_np) // 2] = 0x7C00  # +Inf: every step is skipped
    grads_host = torch.from_numpy(wire_np).pin_memory()
    if args.wire == "f32":  # the same values as fp32 gradients
        grads_host = grads_host.view(torch.float16).float().pin_memory()
    grads = grads_host.to(dev)
    if pipe.sharded and pipe.fused_collective:
        # the gradients live in their bucket slots of the raw wire (DDP's
        # gradient-as-bucket-view): the fused step reads them in place and
        # never modifies them, so no pack runs inside the step
        o = 0
        views = pipe.grad_views()
        for v, spec in zip(views, specs):
            v.copy_(grads[o:o + spec.numel])
            o += spec.numel
        grads = views
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    s0 = torch.cuda.current_stream(dev)

    flush_sink = torch.zeros(1, dtype=torch.int64, device=dev)

    def flush_l2():
        # write 256 MiB (> 126 MB L2), then read it back: every line of the
        # step's data is evicted AND the L2 is left clean, so the write-back of
        # the flush buffer's dirty lines is not charged to the timed step
        _native.call("gs_fill_zero", flush.data_ptr(), flush.numel(), int(s0.cuda_stream))
        flush_sink.add_(flush.view(torch.int64).sum())

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    tok = torch.zeros(1, dtype=torch.float32, device=dev)

    def device_barrier():
        """Untimed, on the launching stream: a 4-byte all-reduce that every
        rank's stream leaves at (nearly) the same moment, so a timed step
        starts together on all ranks instead of absorbing host launch skew."""
        if world > 1:
            dist.all_reduce(tok)

    barrier()  # ranks start the first step together
    # ---- warmup (the first two calls also capture the CUDA graph at p = 1)
    for i in range(args.warmup):
        pipe.step(grads, i)

    clocks = ClockSampler(local)
    clocks.start()
    # clock soak: keep the GPU busy with real steps for ~1.5 s so the sampler
    # sees the clocks this workload runs at (untimed)
    t_end = time.perf_counter() + (0.0 if args.no_soak else 1.5)
    while time.perf_counter() < t_end:
        for _ in range(20):
            pipe.step(grads, args.warmup)

    # ---- timed region: K steps, each alone between an L2 flush and its flag
    # read; device time by CUDA events on the launching stream
    barrier()
    launches0 = _native.kernel_launches()
    step_ms = []
    for i in range(args.steps):
        flush_l2()
        pipe.prepare(args.warmup + i)  # host-only: schedule, loss scale, hint
        # the stream sleeps while the host enqueues the step (as in training,
        # where the host runs ahead of the device): the events time the
        # device, not the host prologue; at N > 1 the barrier after the sleep
        # starts every rank's step together
        torch.cuda._sleep(4_000_000)
        device_barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s0)
        pipe.enqueue(grads, args.warmup + i)
        b.record(s0)
        res = pipe.finish()
        step_ms.append(a.elapsed_time(b))
    launches = _native.kernel_launches() - launches0 - args.steps  # minus the L2 flushes
    barrier()
    clk = clocks.stop()

    # ---- per-kernel breakdown: the same step launched eagerly behind a
    # device-side sleep, so every kernel runs back to back and the events
    # between launches time kernels, not host launch gaps
    phase_ms = {}
    wanted = None  # every phase the step reports
    for i in range(max(3, min(args.steps, 10))):
        flush_l2()
        torch.cuda._sleep(4_000_000)
        device_barrier()
        ev = {}

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record(s0)
            ev[name] = e
        mark("begin")
        pipe.enqueue(grads, args.warmup + i, timer=mark)
        pipe.finish()
        names = list(ev)  # insertion order = launch order
        for x, y in zip(names, names[1:]):
            phase_ms.setdefault(x, []).append(ev[x].elapsed_time(ev[y]))

    mean_ms = statistics.mean(step_ms)
    # every rank's mean phase times (rank skew shows up as a fence / wait
    # phase that is long on the early ranks only)
    phase_spread = None
    if world > 1:
        names = list(phase_ms)
        loc = torch.tensor([statistics.mean(phase_ms[k]) for k in names], dtype=torch.float64,
                           device=dev)
        lo, hi = loc.clone(), loc.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        phase_spread = {k: [round(float(a), 4), round(float(b), 4)]
                        for k, a, b in zip(names, lo.tolist(), hi.tolist())}
    # the dominant kernel: pass 2 (gs_pass2_push in the fused sharded step,
    # over this rank's owned elements only); its achieved bandwidth is taken
    # per rank and the slowest rank reported
    # (gs_zero_update = fence + trust + pass 2 push in one launch: its time
    # includes the fence and the trust CTAs, so the figure is conservative)
    p2_name = "update" if "update" in phase_ms else \
        "pass2_push" if "pass2_push" in phase_ms else "pass2"
    p2_elems = pipe.owned_elems if pipe.sharded else n_params
    p2_ms_local = statistics.median(phase_ms[p2_name])
    # pass 2 per element: r g (2 or 4) w 4 v 4, w v 4 w 4 w16 2
    p2_bpe = 20 if args.wire == "f16" else 22
    t = torch.tensor([mean_ms, -p2_bpe * p2_elems / (p2_ms_local * 1e-3) / 1e9],
                     dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    mean_ms, achieved = float(t[0]), -float(t[1])
    pass2_bytes = p2_bpe * p2_elems
    pass2_ms = p2_ms_local

    # ---- all-reduce bus bandwidth on the whole fp16 gradient (S = 2N bytes)
    allreduce = None
    if world > 1 and not args.no_allreduce_sweep:
        allreduce = allreduce_busbw(pipe, world, local, dev)

    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e_ms = []
        for i in range(max(2, min(args.steps, 10))):
            flush_l2()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            pipe.prepare(1000 + i)
            device_barrier()
            a.record(s0)
            pipe.enqueue_host(grads_host, 1000 + i)  # H2D per bucket, overlapped
            pipe.finish()
            b.record(s0)
            b.synchronize()
            e2e_ms.append(a.elapsed_time(b))
        te = torch.tensor([statistics.mean(e2e_ms[1:])], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": round(float(te[0]), 4), "unit": "ms",
               "h2d_bytes_per_step": (2 if args.wire == "f16" else 4) * n_params,
               "d2h_bytes_per_step": 4 + 8}

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        r = cpu_reference(args.model, 1, args.theta, eta, steps=3, warmup=1, budget_s=30.0)
        cpu = {"value": round(r["ms"], 2), "unit": "ms", "cores": r["threads"], "kind": "port",
               "sample": r["sample"], "stages_ms": r["stages_ms"], **host_info(),
               "note": "numpy restatement of the reference (oracle/reference_port.py) on a "
                       "thread pool; the reference's own single-threaded code measured ~2.4 s "
                       "per ResNet-50 step in the survey, so this baseline is conservative"}

    nvlink = None
    if pipe.sharded and pipe.fused_collective and world > 1:
        # the sharded kernels also move (p-1)/p of their slice over NVLink:
        # rs_pass1 pulls p-1 peer copies of the rank's slice (2 B/elem each),
        # pass2_push stores the updated binary16 slice into p-1 peers (a
        # collective: every rank takes part before rank 0 alone reports)
        nv_bytes = (world - 1) * 2 * pipe.owned_elems
        rs_ms = sum(statistics.median(v) for k, v in phase_ms.items() if k.startswith("rs_pass1"))
        t_nv = torch.tensor([rs_ms, p2_ms_local], dtype=torch.float64, device=dev)
        dist.all_reduce(t_nv, op=dist.ReduceOp.MAX)
        nvlink = {"peak_gbs": 900.0, "peak_kind": "NVLink 5 per direction (nominal)",
                  "rs_pass1_in_gbs": round(nv_bytes / (float(t_nv[0]) * 1e-3) / 1e9, 1),
                  "pass2_push_out_gbs": round(nv_bytes / (float(t_nv[1]) * 1e-3) / 1e9, 1),
                  "pass2_push_phase": p2_name,
                  "bytes_per_rank": nv_bytes}
    if rank != 0:
        return
    peak, peak_kind = load_peaks()
    traffic = None
    tfile = ROOT / "profiles" / "pass2_traffic.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get(args.model)
    # algorithmic bytes of the update kernels per element: pass 1 reads g (2)
    # and w (4); pass 2 reads g w v (10) and writes v w w16 (10); a pack adds
    # 4 (p = 1 lazy wire and the in-place sharded step: no pack at all)
    packs = world > 1 and not (pipe.sharded and pipe.fused_collective)
    # (26 B/elem for fp16 gradients, 30 for the fp32 wire)
    update_bytes = ((26 if args.wire == "f16" else 30) +
                    ((4 if args.wire == "f16" else 8) if packs or pipe.snapshot_wire else 0)
                    ) * n_params
    roofline = {"bound": "hbm",
                "kernel": {"update": "gs_zero_update (fence + trust + pass 2 with the w16 push)",
                           "pass2_push": "gs_pass2_push"}.get(p2_name, "gs_lars_pass2"),
                "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": pass2_bytes}
    if nvlink is not None:
        roofline["nvlink"] = nvlink
    if args.overflow:
        # every step is skipped: pass 2 only reads the flag and exits, so its
        # bandwidth is not a roofline figure
        roofline["frac"] = None
        roofline["note"] = "forced-overflow run: pass 2 takes the skip exit"
    line = {
        "metric": METRIC, "value": round(mean_ms, 4), "unit": "ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(mean_ms, 4),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "wire_dtype": args.wire, "data": "synthetic",
        "config": workload_config(args, world),
        "kernels": (
            "pass1 -> trust -> pass2 (lazy wire: the kernels read the gradients in place; the "
            "FusedBatch payloads are packed only on request)" if world == 1 else
            "gs_rs_pass1 [reduce-scatter+pass1, partials pushed] -> gs_zero_update [fence + trust "
            "+ pass2 with the w16 push] -> fence (gradients in their wire slots: no pack)"
            if args.algorithm == "zero" else
            "pack -> reduce-scatter -> pass1(shard) -> gather partials -> trust -> "
            "pass2(shard) -> all-gather w16" if args.algorithm == "zero_unfused" else
            "pack -> allreduce -> pass1 -> trust -> pass2"),
        "l2": "flushed before every step (256 MiB write, then read: no step data resident, "
              "L2 clean)",
        "phases_ms": {k: round(statistics.mean(v), 4) for k, v in phase_ms.items() if v},
        "phases_ms_min_max_over_ranks": phase_spread,
        "update_roofline_ms": round(update_bytes / (peak * 1e9) * 1e3, 4),
        "roofline": roofline,
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": launches,
        "allreduce": allreduce,
        "cpu_baseline": cpu,
        "last_step": {"applied": res.applied, "scale": res.scale, "grad_norm": res.grad_norm},
    }
    print(json.dumps(line), flush=True)


def allreduce_busbw(pipe, world, local, dev) -> dict:
    """busBW = S/t * 2(p-1)/p for the flat ring, the literal master hierarchy
    and the sharded hierarchy on the whole fp16 gradient buffer."""
    import torch
    import torch.distributed as dist
    import paper_1807_11205_b200 as gs
    from paper_1807_11205_b200.dist import Communicator

    buf = torch.zeros(pipe.total, dtype=torch.uint16, device=dev).view(torch.float16)
    S = 2 * sum(pipe.sizes)
    out = {"bytes": S}
    variants = [("ring", 1)]
    for k in (4, 2):
        if world % k == 0 and k < world:
            variants += [(f"hierarchical_{world // k}x{k}", k), (f"sharded_{world // k}x{k}", k),
                         (f"ordered_hier_{world // k}x{k}", k),
                         (f"ordered_hier_push_{world // k}x{k}", k)]
    comms = {}
    s0 = torch.cuda.current_stream(dev)
    variants += [("ordered", 1), ("ordered_push", 1)]
    ow = None
    for name, k in variants:
        if k not in comms:
            comms[k] = Communicator(gs.Topology(world, k))
        comm = comms[k]
        algo = "ordered" if name.startswith("ordered") else name.split("_")[0]
        hier_k = k if name.startswith("ordered_hier") else 0
        n = buf.numel() - buf.numel() % (k * 8)
        t = buf[:n]
        if algo == "ordered":
            from paper_1807_11205_b200.dist import OrderedWire
            ow = ow or OrderedWire(comm, pipe.total, dev)
            half = [0]

            def run_ordered(_t=None, _push="push" in name, _k=hier_k):
                from paper_1807_11205_b200._peer import launch
                ow.push = _push
                if _k:  # the bit-exact two-level kernel over Topology(p, k)
                    launch([ow.hier_op(half[0], 0, n, _k, int(s0.cuda_stream))])
                else:
                    ow.allreduce(half[0], 0, n, int(s0.cuda_stream))
                ow.advance(1, int(s0.cuda_stream))
                half[0] ^= 1
            comm_allreduce = run_ordered
        else:
            comm_allreduce = (lambda _t, _c=comm, _a=algo: _c.allreduce(_t, _a))
        for _ in range(3):
            comm_allreduce(t)
        torch.cuda.synchronize(dev)
        dist.barrier(device_ids=[local])
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        iters = 10
        a.record(s0)
        for _ in range(iters):
            comm_allreduce(t)
        b.record(s0)
        b.synchronize()
        ms = torch.tensor([a.elapsed_time(b) / iters], dtype=torch.float64, device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        sec = float(ms) * 1e-3
        out[name] = {"us": round(sec * 1e6, 2),
                     "busbw_gbs": round(S / sec * 2 * (world - 1) / world / 1e9, 1),
                     "algbw_gbs": round(S / sec / 1e9, 1)}
    return out


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        from paper_1807_11205_b200.dist import init_from_env
        init_from_env("nccl")
    run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
