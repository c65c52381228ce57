"""Virtual-time schedule simulator + throughput model, calibrated on B200.

Drop-in for the reference `biflow.costsim` (costsim.py:29-249): the same
`CostModel` / `simulate` / `SimReport` / `throughput_model` / `fit_two_point`
API and semantics -- every lane is a serial queue ordered by readiness time
(ties broken by graph insertion order), readiness is the dispatcher's own
`ReadinessState`, each graph of a sequence starts when the previous one has
finished, and a run is exactly reproducible.

B200 additions ("cost simulator calibrated with measured
B200 per-kernel times"):

* `measured_costs(path)` turns the per-operator device times written by
  ``bench.py --op-table`` (a traced replay of the captured GoogLeNet / NIN
  iteration) into a `CostModel` keyed by operator name;
* `exchange_cost(bytes, world, ...)` models one lowered bucket exchange
  (reduce-scatter + sharded update + all-gather) from the latency / bus
  bandwidth a `tools/exchange_sweep.py` run measures;
* `predict_scaling(net, worlds, op_times)` simulates the exchange-lowered
  rank sequence of `exchange.build_rank_sequence` for each world size and
  reports predicted images/s, scaling efficiency and exposed communication.
"""

from __future__ import annotations

import heapq
import math
from collections.abc import Callable, Mapping
from dataclasses import dataclass, field
from typing import NamedTuple

from .dispatcher import ReadinessState, TraceRecord, WorkerLane, lane_of
from .graph import BiGraph, GraphSequence, OperatorVertex

__all__ = ["CostModel", "FitResult", "ScalingPoint", "SimError", "SimReport", "exchange_cost",
           "fit_two_point", "measured_costs", "predict_scaling", "simulate", "throughput_model"]

_TRANSFER_KINDS = ("copy", "send", "recv", "gate")  # bandwidth/latency fallback (costsim.py:23)


class SimError(ValueError):
    """Bad cost model, operator kind without a cost, or invalid fit input."""


@dataclass(frozen=True)
class CostModel:
    """Operator durations in virtual seconds (reference costsim.py:29-90).

    Lookup order for an operator: its ``delay_s`` attribute; ``op_costs`` by
    operator name (measured tables); ``kind_costs`` by kind (a constant or
    ``f(in_shapes, out_shapes) -> seconds``); for transfer kinds
    ``latency + bytes / bandwidth``.  ``per_image_compute`` / ``overhead``
    are the closed-form model's (a, c) and are not read by `simulate`."""

    kind_costs: Mapping[str, float | Callable] = field(default_factory=dict)
    bandwidth: float = math.inf
    latency: float = 0.0
    per_image_compute: float = 0.0
    overhead: float = 0.0
    op_costs: Mapping[str, float] = field(default_factory=dict)

    def __post_init__(self) -> None:
        if not self.bandwidth > 0:
            raise SimError(f"bandwidth must be > 0, got {self.bandwidth}")
        for name in ("latency", "per_image_compute", "overhead"):
            if getattr(self, name) < 0:
                raise SimError(f"{name} must be >= 0, got {getattr(self, name)}")

    def duration_of(self, op: OperatorVertex, graph: BiGraph) -> float:
        if "delay_s" in op.attrs:
            dur = float(op.attrs["delay_s"])
        elif op.name in self.op_costs:
            dur = float(self.op_costs[op.name])
        elif op.kind in self.kind_costs:
            entry = self.kind_costs[op.kind]
            if callable(entry):
                dur = float(entry([graph.tensors[t].shape for t in op.inputs],
                                  [graph.tensors[t].shape for t in op.outputs]))
            else:
                dur = float(entry)
        elif op.kind in _TRANSFER_KINDS:
            tid = (op.outputs or op.inputs)[0]
            dur = self.latency + 4 * math.prod(graph.tensors[tid].shape) / self.bandwidth
        else:
            raise SimError(f"no cost entry for operator kind {op.kind!r} (op {op.name!r})")
        if not (dur >= 0 and math.isfinite(dur)):
            raise SimError(f"operator {op.name!r} has invalid duration {dur}")
        return dur


@dataclass
class SimReport:
    makespan: float
    trace: list[TraceRecord]
    throughput: float | None = None


def _sequence(obj, iterations) -> GraphSequence:
    if isinstance(obj, GraphSequence):
        return obj if iterations is None else GraphSequence(obj.graphs, iterations=iterations,
                                                            layout=obj.layout)
    return GraphSequence([obj], iterations=1 if iterations is None else iterations)


def simulate(graph_or_sequence, costs: CostModel, iterations: int | None = None, *,
             images_per_iteration: float | None = None) -> SimReport:
    """Event-driven virtual-time execution (reference costsim.py:100-196)."""
    seq = _sequence(graph_or_sequence, iterations)
    for g in seq.graphs:
        rep = g.validate()
        if not rep.ok:
            raise SimError("graph failed validation: " + "; ".join(rep.violations))
    plans = []
    for g in seq.graphs:
        rank = {oid: i for i, oid in enumerate(g.insertion_order)}
        dur = {op.id: costs.duration_of(op, g) for op in g.operators_in_order()}
        plans.append((ReadinessState(g), dur, rank))

    trace: list[TraceRecord] = []
    lane_free: dict[WorkerLane, float] = {}
    floor = 0.0
    for it in range(seq.iterations):
        for g, (state, dur, rank) in zip(seq.graphs, plans):
            state.reset()
            armed = state.arm()
            if not g.operators:
                continue
            queues: dict[WorkerLane, list] = {}  # lane -> heap of (ready time, rank, op)
            busy: set[WorkerLane] = set()
            running: list = []  # heap of (end, rank, op, start)

            def push(oid: int, t: float) -> None:
                heapq.heappush(queues.setdefault(lane_of(g.operators[oid]), []),
                               (t, rank[oid], oid))

            def dispatch() -> None:
                for lane, q in queues.items():
                    if lane in busy or not q:
                        continue
                    t, r, oid = heapq.heappop(q)
                    start = max(t, lane_free.get(lane, 0.0))
                    busy.add(lane)
                    heapq.heappush(running, (start + dur[oid], r, oid, start))

            for oid in armed:
                push(oid, floor)
            dispatch()
            end_of_graph = floor
            while running:
                now = running[0][0]
                while running and running[0][0] == now:
                    end, _r, oid, start = heapq.heappop(running)
                    op = g.operators[oid]
                    lane = lane_of(op)
                    busy.discard(lane)
                    lane_free[lane] = end
                    trace.append(TraceRecord(oid, op.name, lane, int(round(start * 1e9)),
                                             int(round(end * 1e9)), it))
                    for nxt in state.complete(oid):
                        push(nxt, end)
                dispatch()
                end_of_graph = now
            floor = max(floor, end_of_graph)
    thr = None
    if images_per_iteration is not None and floor > 0:
        thr = images_per_iteration * seq.iterations / floor
    return SimReport(makespan=floor, trace=trace, throughput=thr)


# ---------------------------------------------------------------------------
# closed-form model (reference costsim.py:203-249)


def throughput_model(peers: int, batch: float, a: float, c: float) -> float:
    """Images/s of ``peers`` workers at ``batch`` images each: compute scales,
    only a constant ``c`` per iteration is not overlapped."""
    if peers < 1 or batch < 1:
        raise SimError(f"need peers >= 1 and batch >= 1, got {peers}, {batch}")
    if a <= 0 or c < 0:
        raise SimError(f"need a > 0 and c >= 0, got a={a}, c={c}")
    return peers * batch / (a * batch + c)


class FitResult(NamedTuple):
    a: float
    c: float
    residuals: dict[float, float]


def fit_two_point(table, peers: int) -> FitResult:
    """(a, c) from the smallest- and largest-batch rows of (batch, img/s)
    measurements at ``peers`` workers; the other rows become residuals."""
    rows = [(float(b), float(r)) for b, r in table]
    if len(rows) < 2:
        raise SimError("fit_two_point: need at least two (batch, rate) rows")
    if len({b for b, _ in rows}) != len(rows):
        raise SimError("fit_two_point: duplicate batch values")
    (b0, r0), (b1, r1) = min(rows), max(rows)
    t0, t1 = peers * b0 / r0, peers * b1 / r1  # a*B + c per extreme row
    a = (t1 - t0) / (b1 - b0)
    c = t0 - a * b0
    if a <= 0:
        raise SimError(f"fit_two_point: non-positive compute cost a={a}")
    res = {b: (throughput_model(peers, b, a, c) - r) / r for b, r in rows if b not in (b0, b1)}
    return FitResult(a, c, res)


# ---------------------------------------------------------------------------
# B200 calibration


def measured_costs(path) -> dict[str, float]:
    """Per-operator device seconds from a ``bench.py --op-table`` TSV
    (op, kind, ms, gflop, mbytes)."""
    out: dict[str, float] = {}
    with open(path) as f:
        header = f.readline().rstrip("\n").split("\t")
        if header[:3] != ["op", "kind", "ms"]:
            raise SimError(f"{path}: not an op table (header {header})")
        for line in f:
            cols = line.rstrip("\n").split("\t")
            if len(cols) >= 3:
                out[cols[0]] = float(cols[2]) * 1e-3
    return out


def exchange_cost(nbytes: float, world: int, latency_s: float = 10e-6,
                  busbw_gbs: float = 700.0, update_gbs: float = 5000.0) -> float:
    """Seconds for one lowered bucket exchange: reduce-scatter + all-gather of
    ``nbytes`` (ring bus-bandwidth model, 2(N-1)/N of the bytes cross the
    fabric) plus the fused mean+SGD over the 1/N shard (12 bytes per element
    through HBM).  Defaults: NVLink 5 / NVSwitch bus bandwidth at the sizes
    the buckets use and the B200 HBM rate; measure with tools/exchange_sweep.py."""
    if world < 1 or nbytes < 0:
        raise SimError(f"exchange_cost: bad arguments bytes={nbytes}, world={world}")
    wire = 0.0 if world == 1 else 2 * latency_s + nbytes * 2 * (world - 1) / world / (busbw_gbs * 1e9)
    update = 3 * nbytes / world / (update_gbs * 1e9)
    return wire + update


class ScalingPoint(NamedTuple):
    world: int
    iteration_s: float
    images_per_s: float
    efficiency: float
    exposed_comm: float


def predict_scaling(net, worlds, op_times: Mapping[str, float], *, batch: int | None = None,
                    exchange=exchange_cost, bucket_bytes: int = 4 << 20,
                    compute_scale: float = 1.0,
                    exchange_slowdown: float = 1.5) -> list[ScalingPoint]:
    """Simulate the exchange-lowered rank sequence (exchange.py) at each world
    size with measured compute times (`measured_costs`, keyed by the rank-0
    operator names the bench traces) and a modelled bucket exchange; returns
    predicted images/s, efficiency vs world 1 and exposed-exchange fraction
    (profiler.exposed_ns over the simulated trace).

    ``compute_scale`` rescales the measured (serialised) operator times to the
    measured step (branch streams overlap them on the device);
    ``exchange_slowdown`` is the bucket exchange's slowdown while it overlaps
    backward GEMMs (1.5x at the 4 MB buckets, profiles/r01_exchange_sweep_1gpu.md)."""
    from .exchange import lower_data_parallel, plan_buckets
    from .builders import ParallelPlan, build_data_parallel, param_names
    from .graph import Location
    from .profiler import exposed_ns

    batch = batch or net.batch
    points: list[ScalingPoint] = []
    base = None
    for world in worlds:
        plan = ParallelPlan("data", peers=tuple(Location("local", k) for k in range(world)),
                            server=Location("local", world))
        full = build_data_parallel(net, plan)
        xplan = plan_buckets(param_names(net), world, bucket_bytes)
        seq = lower_data_parallel(full, 0, xplan, net)
        g = seq.graphs[0]
        costs: dict[str, float] = {}
        for op in g.operators.values():
            if op.kind == "dp_exchange":
                nbytes = 4 * sum(math.prod(g.tensors[t].shape) for t in op.inputs)
                costs[op.name] = exchange(nbytes, world) * (exchange_slowdown if world > 1 else 1.0)
            elif op.name in op_times:
                costs[op.name] = op_times[op.name] * compute_scale
            elif op.kind in ("swap", "flatten_forward", "flatten_backward"):
                costs[op.name] = 0.0
        missing = [op.name for op in g.operators.values() if op.name not in costs]
        if missing:
            raise SimError(f"predict_scaling: no measured time for {len(missing)} operators, "
                           f"e.g. {missing[:3]}")
        rep = simulate(GraphSequence([g], iterations=1), CostModel(op_costs=costs))
        comm = [(r.start, r.end) for r in rep.trace if g.operators[r.op].kind == "dp_exchange"]
        comp = [(r.start, r.end) for r in rep.trace if g.operators[r.op].kind != "dp_exchange"]
        t = rep.makespan
        ips = world * batch / t
        if base is None:
            base = ips
        points.append(ScalingPoint(world, t, ips, ips / (world * base / worlds[0]) if base else 0.0,
                                   exposed_ns(comm, comp) / max(1, int(round(t * 1e9)))))
    return points
