"""α-β cost model over reduce schedules, calibrated on measured B200 sweeps.

Drop-in for the reference's `gradsync.netsim` (pkg/src/gradsync/netsim.py:16-26):
`LinkModel`, `SimReport`, `simulate`, `EfficiencyInput`, `EfficiencyReport`,
`scaling_efficiency`, `implied_system_throughput`, `crossover_sweep`,
`find_crossover` keep the reference's names, argument meaning, validation
errors and arithmetic (a round of concurrent transfers costs
`alpha + max_bytes / bandwidth`, rounds serialise; netsim.py:77-94), so the
reference's test_netsim.py reads unchanged against this module.

What is new here is SURVEY.md §8f row 4: the model is CALIBRATED with the
all-reduce sweeps measured on the B200 box (`tools/allreduce_sweep.py`,
`profiles/*/sweep_*.jsonl`) instead of hand-set α/β, and the calibrated model
seeds the hybrid threshold η (`calibrated_eta`, the reference's
crossover_sweep → find_crossover route, netsim.py:139-170).  `fit_link` solves
the per-phase α/β by non-negative least squares on relative error over the
schedule's round counts and per-round byte sums, so one fit covers 1 KB-1 GB.

Host-side arithmetic only: no device work, nothing on the step's hot path.
"""

from __future__ import annotations

import itertools
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .collectives import ReduceSchedule, Topology, hierarchical_schedule, ring_schedule

__all__ = [
    "LinkModel",
    "SimReport",
    "simulate",
    "EfficiencyInput",
    "EfficiencyReport",
    "scaling_efficiency",
    "implied_system_throughput",
    "crossover_sweep",
    "find_crossover",
    "schedule_features",
    "fit_link",
    "load_sweep",
    "calibrate_from_sweep",
    "calibrated_eta",
]


@dataclass(frozen=True)
class LinkModel:
    """Per-round latency `alpha` (s) and bandwidth `beta_inv` (bytes/s), with
    optional separate parameters for the intra-group phases
    (netsim.py:29-54).  An unset intra parameter falls back to the flat one
    independently of the other."""

    alpha: float = 1e-5
    beta_inv: float = 1e9
    intra_group_alpha: float | None = None
    intra_group_beta_inv: float | None = None

    def __post_init__(self):
        checks = (
            (self.alpha < 0, f"latency must be >= 0, got {self.alpha}"),
            (self.beta_inv <= 0, f"bandwidth must be > 0, got {self.beta_inv}"),
            (self.intra_group_alpha is not None and self.intra_group_alpha < 0,
             "intra-group latency must be >= 0"),
            (self.intra_group_beta_inv is not None and self.intra_group_beta_inv <= 0,
             "intra-group bandwidth must be > 0"),
        )
        for bad, msg in checks:
            if bad:
                raise ValueError(msg)

    def params_for(self, phase: str) -> tuple[float, float]:
        """(alpha, bandwidth) of a round of `phase`; phases named `intra*`
        use the intra-group link."""
        if not phase.startswith("intra"):
            return self.alpha, self.beta_inv
        a = self.alpha if self.intra_group_alpha is None else self.intra_group_alpha
        b = self.beta_inv if self.intra_group_beta_inv is None else self.intra_group_beta_inv
        return a, b

    def to_dict(self) -> dict:
        return {"alpha": self.alpha, "beta_inv": self.beta_inv,
                "intra_group_alpha": self.intra_group_alpha,
                "intra_group_beta_inv": self.intra_group_beta_inv}


@dataclass
class SimReport:
    """Modelled cost of one schedule under one link model (netsim.py:57-74)."""

    algorithm: str
    total_time: float
    per_phase_time: dict
    total_steps: int
    bytes_on_wire: int

    def to_dict(self) -> dict:
        return {
            "algorithm": self.algorithm,
            "total_time": self.total_time,
            "per_phase_time": dict(self.per_phase_time),
            "total_steps": self.total_steps,
            "bytes_on_wire": self.bytes_on_wire,
        }


def simulate(schedule: ReduceSchedule, link: LinkModel) -> SimReport:
    """Serialise the schedule's rounds through `link` (netsim.py:77-94).

    Round times are summed in round order, per phase and in total, so the
    floating-point result is the reference's to the bit."""
    per_phase: dict = {}
    total = 0.0
    wire = 0
    for rnd in schedule.rounds:
        a, bw = link.params_for(rnd.phase)
        t = a + rnd.max_bytes / bw
        per_phase[rnd.phase] = per_phase.get(rnd.phase, 0.0) + t
        total += t
        wire += rnd.total_bytes
    return SimReport(algorithm=schedule.algorithm, total_time=total,
                     per_phase_time=per_phase, total_steps=schedule.total_steps,
                     bytes_on_wire=wire)


@dataclass(frozen=True)
class EfficiencyInput:
    """S (samples/s of one worker), N (workers), T (samples/s of the system)
    for the identity e = T / (S·N) (netsim.py:97-111)."""

    single_worker_throughput: float
    worker_count: int
    system_throughput: float

    def __post_init__(self):
        if self.single_worker_throughput <= 0:
            raise ValueError("single-worker throughput must be > 0")
        if self.worker_count < 1:
            raise ValueError("worker count must be >= 1")
        if self.system_throughput < 0:
            raise ValueError("system throughput must be >= 0")


@dataclass(frozen=True)
class EfficiencyReport:
    """Raw efficiency, its headline clamp at 1, and a flag instead of hiding
    super-ideal values (netsim.py:114-125)."""

    efficiency: float
    clamped: float
    exceeds_ideal: bool

    def to_dict(self) -> dict:
        return {"efficiency": self.efficiency, "clamped": self.clamped,
                "exceeds_ideal": self.exceeds_ideal}


def scaling_efficiency(inp: EfficiencyInput) -> EfficiencyReport:
    """e = T / (S·N) (netsim.py:128-131)."""
    e = inp.system_throughput / (inp.single_worker_throughput * inp.worker_count)
    return EfficiencyReport(efficiency=e, clamped=min(e, 1.0), exceeds_ideal=e > 1.0)


def implied_system_throughput(single: float, workers: int, efficiency: float) -> float:
    """T = S·N·e, the inverse of `scaling_efficiency` (netsim.py:134-136)."""
    return single * workers * efficiency


def crossover_sweep(p: int, k: int, link: LinkModel, sizes_bytes, itemsize: int = 4) -> list:
    """Modelled ring vs hierarchical time per payload size; ties go to ring,
    as in the hybrid selector (netsim.py:139-158)."""
    topo = Topology(p, k)
    rows = []
    for nbytes in sizes_bytes:
        n = max(int(nbytes) // itemsize, 0)
        t_ring = simulate(ring_schedule(p, n, itemsize, k=k), link).total_time
        t_hier = simulate(hierarchical_schedule(topo, n, itemsize), link).total_time
        rows.append({"bytes": n * itemsize, "ring_time": t_ring,
                     "hierarchical_time": t_hier,
                     "faster": "hierarchical" if t_hier < t_ring else "ring"})
    return rows


def find_crossover(rows) -> int | None:
    """First sampled size at which ring is no longer slower; payloads below
    it go hierarchical.  None when ring never wins (netsim.py:161-170)."""
    return next((row["bytes"] for row in rows if row["faster"] == "ring"), None)


# --------------------------------------------------------------------------
# calibration on measured sweeps
# --------------------------------------------------------------------------

def schedule_features(schedule: ReduceSchedule) -> np.ndarray:
    """[inter rounds, inter Σ max_bytes, intra rounds, intra Σ max_bytes]:
    the schedule's modelled time is exactly the dot product of this vector
    with [α, 1/β, α_intra, 1/β_intra]."""
    f = np.zeros(4)
    for rnd in schedule.rounds:
        o = 2 if rnd.phase.startswith("intra") else 0
        f[o] += 1.0
        f[o + 1] += rnd.max_bytes
    return f


def _nnls_small(A: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Non-negative least squares for a handful of unknowns by enumerating
    the passive sets (2^m ≤ 16 unconstrained solves)."""
    m = A.shape[1]
    best, best_r = np.zeros(m), float(b @ b)
    for r in range(1, m + 1):
        for cols in itertools.combinations(range(m), r):
            sub = A[:, cols]
            if np.linalg.matrix_rank(sub) < r:
                continue
            x, *_ = np.linalg.lstsq(sub, b, rcond=None)
            if np.any(x < 0):
                continue
            full = np.zeros(m)
            full[list(cols)] = x
            res = b - A @ full
            rr = float(res @ res)
            if rr < best_r:
                best, best_r = full, rr
    return best


def fit_link(samples, p: int, k: int = 1, itemsize: int = 2) -> LinkModel:
    """Fit a `LinkModel` to measured all-reduce times.

    samples: iterable of (algorithm, nbytes, seconds), algorithm "ring" or
    "hierarchical" (the schedule the measured collective executes, on
    Topology(p, k)).  Each sample contributes one row
    features(schedule(nbytes)) · [α, 1/β, α_i, 1/β_i] = seconds, weighted by
    1/seconds so a 1 KB latency point counts as much as a 1 GB bandwidth
    point.  Intra-group parameters are fitted only when some sample has
    intra-group rounds; a zero inverse bandwidth (infinitely fast link) is
    reported as bandwidth 1e30."""
    topo = Topology(p, k)
    rows, rhs = [], []
    for algorithm, nbytes, seconds in samples:
        n = int(nbytes) // itemsize
        if algorithm == "ring":
            sched = ring_schedule(p, n, itemsize, k=k)
        elif algorithm == "hierarchical":
            sched = hierarchical_schedule(topo, n, itemsize)
        else:
            raise ValueError(f"unknown algorithm {algorithm!r}")
        if seconds <= 0:
            raise ValueError(f"measured time must be > 0, got {seconds}")
        rows.append(schedule_features(sched) / seconds)
        rhs.append(1.0)
    if not rows:
        raise ValueError("no samples to fit")
    A, b = np.asarray(rows), np.asarray(rhs)
    has_intra = bool(np.any(A[:, 2:] > 0))
    x = _nnls_small(A if has_intra else A[:, :2], b)

    def bw(inv):
        return 1e30 if inv <= 0 else 1.0 / inv

    if not has_intra:
        return LinkModel(alpha=float(x[0]), beta_inv=bw(float(x[1])))
    return LinkModel(alpha=float(x[0]), beta_inv=bw(float(x[1])),
                     intra_group_alpha=float(x[2]), intra_group_beta_inv=bw(float(x[3])))


def load_sweep(path, variants=None) -> list:
    """Rows of a `tools/allreduce_sweep.py` JSONL file (bytes, variant, p, us)."""
    out = []
    for line in Path(path).read_text().splitlines():
        line = line.strip()
        if not line:
            continue
        row = json.loads(line)
        if "variant" in row and (variants is None or row["variant"] in variants):
            out.append(row)
    return out


def calibrate_from_sweep(rows, p: int, k: int, *, ring_variant: str = "ring",
                         hier_variant: str | None = None, itemsize: int = 2) -> LinkModel:
    """Calibrate on one sweep: the flat ring rows give (α, β); the literal
    hierarchy rows (variant `hierarchical_{k}x{p//k}` by default) add the
    intra-group (α_i, β_i)."""
    hier_variant = hier_variant or f"hierarchical_{k}x{p // k}"
    samples = []
    for row in rows:
        if row.get("p", p) != p:
            continue
        if row["variant"] == ring_variant:
            samples.append(("ring", row["bytes"], row["us"] * 1e-6))
        elif row["variant"] == hier_variant and k > 1:
            samples.append(("hierarchical", row["bytes"], row["us"] * 1e-6))
    return fit_link(samples, p, k, itemsize)


def calibrated_eta(p: int, k: int, link: LinkModel, sizes_bytes=None, itemsize: int = 2):
    """Hybrid threshold η seeded from the calibrated model (netsim.py:161-170):
    returns (eta_bytes, rows).  η = 0 when ring already wins at the smallest
    sampled size (every payload goes ring); η = ∞ when it never wins."""
    sizes = list(sizes_bytes) if sizes_bytes is not None else [1 << s for s in range(10, 31)]
    rows = crossover_sweep(p, k, link, sizes, itemsize=itemsize)
    x = find_crossover(rows)
    if x is None:
        return float("inf"), rows
    return (0 if x == rows[0]["bytes"] else x), rows


def eta_from_sweep(path, p: int, k: int, itemsize: int = 2):
    """The hybrid threshold η for Topology(p, k) seeded from a measured
    all-reduce sweep file (`tools/allreduce_sweep.py` JSONL): calibrate the
    link model on the file's flat-ring (and literal-hierarchy) rows, then
    `calibrated_eta`.  Returns bytes (int), or float("inf")."""
    link = calibrate_from_sweep(load_sweep(path), p, k, itemsize=itemsize)
    eta, _ = calibrated_eta(p, k, link, itemsize=itemsize)
    return eta
