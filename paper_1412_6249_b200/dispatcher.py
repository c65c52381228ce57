"""Event-driven graph execution on CUDA streams.

Drop-in for the reference dispatcher (`pkg/src/biflow/dispatcher.py`):
same `run` / `run_sequence` signatures and hooks, same `ReadinessState`
bookkeeping, `TraceRecord` / `RunReport` / `merged_trace`, `DispatchError`
with first-error-wins, `BIFLOW_LANES` lane cap.

B200 design.  The reference runs one OS thread per lane, each pulling ready
operators from a FIFO and executing numpy kernels synchronously.  Here a
lane ``(host, device, thread)`` is a CUDA stream of the store's device and
readiness is enforced ON THE DEVICE: every tensor carries the CUDA event its
producer recorded, and an operator is enqueued behind
``cudaStreamWaitEvent`` on each input produced on another stream.  The host
therefore never waits for kernels; it walks the graph once, in the
reference's serial-mode order (the `ReadinessState` arm/complete FIFO,
dispatcher.py:144-191), which is topological, so FIFO streams cannot
deadlock even when lanes share a stream, and every rank enqueues collectives
in the same order.  Streams run concurrently, giving the reference's
lane-level overlap (compute lanes vs. copy lanes) on the GPU.

Inside a compute lane, independent operators (Inception branches; weight vs.
data gradients) are further spread over up to ``PURINE_B200_BRANCH_STREAMS``
(default 8) streams by greedy chain decomposition, with event waits on every
cross-stream input: an operator starts when its inputs' events fire.  Lanes
that carry collectives keep one stream, created at high priority so the block
scheduler starts exchange CTAs ahead of queued compute CTAs.

Lane cap: ``max_workers`` / ``BIFLOW_LANES`` bounds the number of streams;
sorted lanes map round-robin onto them exactly as lanes map onto worker
threads in the reference (dispatcher.py:261-267).  ``1`` is the fully serial
mode: one stream (no branch streams), device execution order == dispatch order.

Timing: with ``trace=True`` each operator is bracketed by CUDA events on its
stream; `TraceRecord` start/end are ns since the sequence's zero event, so
the reference's interval arithmetic (profiler.py) applies unchanged.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import torch

from .graph import BiGraph, GraphSequence, OperatorVertex
from .kinds import KINDS, KernelError
from .store import TensorStore

__all__ = [
    "DispatchError",
    "LANES_ENV",
    "ReadinessState",
    "RunContext",
    "RunReport",
    "TraceRecord",
    "WorkerLane",
    "lane_of",
    "merged_trace",
    "raise_if_nonfinite",
    "run",
    "run_sequence",
    "serial_order",
]

LANES_ENV = "BIFLOW_LANES"


class DispatchError(RuntimeError):
    """A run could not start or finish; carries the offending operator's name."""


@dataclass(frozen=True, order=True)
class WorkerLane:
    """A serial execution queue (here: one CUDA stream)."""

    host: str
    device: int
    thread: int


def lane_of(op: OperatorVertex) -> WorkerLane:
    return WorkerLane(op.location.host, op.location.device, op.thread)


@dataclass(frozen=True)
class TraceRecord:
    """One operator execution; times are ns since the run's zero event."""

    op: int
    name: str
    lane: WorkerLane
    start: int
    end: int
    iteration: int = 0


@dataclass
class RunReport:
    trace: list[TraceRecord]
    elapsed: int
    iteration: int = 0
    graph_index: int = 0
    dispatch_order: list[str] = field(default_factory=list)


def merged_trace(reports: list[RunReport]) -> list[TraceRecord]:
    recs = [r for rep in reports for r in rep.trace]
    recs.sort(key=lambda r: (r.start, r.end))
    return recs


# ---------------------------------------------------------------------------
# readiness bookkeeping (dispatcher.py:96-206)


class ReadinessState:
    """Pending-count bookkeeping for one graph (same contract as the reference).

    ``pending_inputs``: operator id -> unsatisfied input edges;
    ``pending_producers``: tensor id -> producers not yet completed.
    `arm` returns the initially ready operators and `complete` the newly
    ready ones, both in graph-insertion order.
    """

    def __init__(self, graph: BiGraph) -> None:
        self.graph = graph
        self._rank = {oid: i for i, oid in enumerate(graph.insertion_order)}
        self._tensor_sinks = {t for t in graph.tensors if not graph.consumers_of(t)}
        self._op_sinks = {o for o, op in graph.operators.items() if not op.outputs}
        self.sink_count = len(self._tensor_sinks) + len(self._op_sinks)
        self._in_flight = 0
        self.reset()

    def reset(self) -> None:
        if self._in_flight:
            raise DispatchError("reset() while operators are in flight")
        g = self.graph
        self.pending_inputs = {o: len(op.inputs) for o, op in g.operators.items()}
        self.pending_producers = {t: int(g.producer_of(t) is not None) for t in g.tensors}
        self.completed_sinks = 0
        self._executed = 0
        self._armed = False

    def _release(self, tid: int, out: list[int]) -> None:
        if tid in self._tensor_sinks:
            self.completed_sinks += 1
        for oid, _pos in self.graph.consumers_of(tid):
            self.pending_inputs[oid] -= 1
            if self.pending_inputs[oid] == 0:
                out.append(oid)

    def arm(self) -> list[int]:
        if self._armed:
            raise DispatchError("arm() on an already armed state")
        self._armed = True
        ready = [o for o in self.graph.insertion_order if self.pending_inputs[o] == 0]
        for tid in sorted(self.graph.tensors):
            if self.pending_producers[tid] == 0:
                self._release(tid, ready)
        ordered = sorted(dict.fromkeys(ready), key=self._rank.__getitem__)
        self._in_flight += len(ordered)
        return ordered

    def complete(self, op_id: int) -> list[int]:
        op = self.graph.operators[op_id]
        self._executed += 1
        self._in_flight -= 1
        if op_id in self._op_sinks:
            self.completed_sinks += 1
        fresh: list[int] = []
        for tid in op.outputs:
            self.pending_producers[tid] -= 1
            if self.pending_producers[tid] == 0:
                self._release(tid, fresh)
        fresh.sort(key=self._rank.__getitem__)
        self._in_flight += len(fresh)
        return fresh

    def abandon(self, count: int = 1) -> None:
        self._in_flight -= count

    @property
    def in_flight(self) -> int:
        return self._in_flight

    @property
    def done(self) -> bool:
        return self._executed == len(self.graph.operators) and self.completed_sinks == self.sink_count




def serial_order(graph: BiGraph) -> list[int]:
    """Reference serial-mode (one worker) dispatch order of ``graph``."""
    # cached on the graph object (an id()-keyed cache can serve a dead graph's
    # order to a new graph allocated at the same address)
    stamp = len(graph.insertion_order) * 1_000_003 + len(graph.tensors)
    hit = graph.__dict__.get("_serial_order")
    if hit is not None and hit[0] == stamp:
        return hit[1]
    st = ReadinessState(graph)
    queue = st.arm()
    head = 0
    while head < len(queue):
        queue.extend(st.complete(queue[head]))
        head += 1
    if len(queue) != len(graph.operators):
        raise DispatchError("graph cannot complete: some operators never become ready")
    graph.__dict__["_serial_order"] = (stamp, queue)
    return queue


# ---------------------------------------------------------------------------
# run context and stream/workspace pools


@dataclass
class RunContext:
    """Everything a kernel execution hook may touch (dispatcher.py:209-217),
    plus the lane's CUDA stream handle and split-K workspace."""

    store: TensorStore
    graph: BiGraph
    iteration: int = 0
    transport: object | None = None
    copy_latency_s: float = 0.0
    stream: int = 0
    workspace: object | None = None  # _Workspace: .data_ptr() / .numel(), lazily allocated
    lane: WorkerLane | None = None
    fused: dict | None = None  # epilogue-fusion instructions for this operator (see _Plan)


WORKSPACE_FLOATS = int(os.environ.get("PURINE_B200_WORKSPACE_MB", "1024")) << 18  # 1 GiB


class _Workspace:
    """Per-stream scratch (split-K partials, pre-packed GEMM operands),
    allocated on first use so lanes that never run a contraction cost nothing."""

    def __init__(self, device) -> None:
        self.device = device
        self.buf: torch.Tensor | None = None

    def tensor(self) -> torch.Tensor:
        if self.buf is None:
            self.buf = torch.empty(WORKSPACE_FLOATS, dtype=torch.float32, device=self.device)
        return self.buf

    def data_ptr(self) -> int:
        return self.tensor().data_ptr()

    def numel(self) -> int:
        return WORKSPACE_FLOATS


class _Lanes:
    """Per-store pool of CUDA streams (one per lane slot) and workspaces."""

    def __init__(self, store: TensorStore) -> None:
        self.device = store.device
        self.streams: list[torch.cuda.Stream] = []
        self.workspaces: list[_Workspace] = []
        self.high: dict[int, tuple[torch.cuda.Stream, _Workspace]] = {}

    def get(self, idx: int, high: bool = False) -> tuple[torch.cuda.Stream, _Workspace]:
        """Stream + workspace of slot ``idx``; ``high`` selects a separate
        high-priority stream (the exchange lane: the block scheduler then
        starts its collective / update CTAs ahead of queued compute CTAs)."""
        if high:
            if idx not in self.high:
                self.high[idx] = (torch.cuda.Stream(device=self.device, priority=-1),
                                  _Workspace(self.device))
            return self.high[idx]
        while len(self.streams) <= idx:
            self.streams.append(torch.cuda.Stream(device=self.device))
            self.workspaces.append(_Workspace(self.device))
        return self.streams[idx], self.workspaces[idx]


def lanes_of(store: TensorStore) -> _Lanes:
    pool = getattr(store, "_lane_pool", None)
    if pool is None:
        pool = _Lanes(store)
        store._lane_pool = pool
        if store.device.type == "cuda":
            from . import _native

            _native.lib()("bf_set_device", store.device.index or 0)
    return pool


def _env_lane_cap() -> int:
    raw = os.environ.get(LANES_ENV)
    if not raw:
        return 1 << 16
    try:
        cap = int(raw)
    except ValueError:
        raise DispatchError(f"{LANES_ENV} must be an integer, got {raw!r}") from None
    if cap < 1:
        raise DispatchError(f"{LANES_ENV} must be >= 1, got {cap}")
    return cap


def _check_sources(graph: BiGraph, store: TensorStore) -> None:
    for tid, t in graph.tensors.items():
        if graph.producer_of(tid) is None and graph.consumers_of(tid):
            if not store.has(t.name):
                raise DispatchError(f"source tensor {t.name!r} has no buffer in the store")
            if store.get(t.name).shape != t.shape:
                raise DispatchError(f"source tensor {t.name!r}: store shape "
                                    f"{store.get(t.name).shape} != graph shape {t.shape}")


class _Plan:
    """Static per-(graph, lane cap) launch plan: order, lane slots, cross-stream edges."""

    def __init__(self, graph: BiGraph, cap: int, branches: int = 1) -> None:
        self.order = serial_order(graph)
        lanes = sorted({lane_of(op) for op in graph.operators.values()})
        n = max(1, min(len(lanes), cap)) if lanes else 0
        self.slot_of_lane = {ln: i % n for i, ln in enumerate(lanes)} if n else {}
        self.slot = {oid: self.slot_of_lane[lane_of(op)] for oid, op in graph.operators.items()}
        self.n_slots = n
        # slots running the parameter exchange get a high-priority stream
        self.high_priority = {self.slot[oid] for oid, op in graph.operators.items()
                              if op.kind == "dp_exchange"}
        if branches > 1 and cap > 1 and n:
            self._split_branches(graph, branches)
        # inputs produced by an op on a different slot -> that producer must record an event
        self.waits: dict[int, list[int]] = {}
        self.signals: set[int] = set()
        for oid, op in graph.operators.items():
            deps = []
            for tid in op.inputs:
                p = graph.producer_of(tid)
                if p is not None and self.slot[p] != self.slot[oid] and p not in deps:
                    deps.append(p)
                    self.signals.add(p)
            self.waits[oid] = deps
        # epilogue fusion: a relu_forward on the same stream directly after the
        # conv2d_forward producing its input is computed by the conv epilogue
        # (the relu operator is still dispatched, as a no-op, so dispatch order,
        # readiness events and traces are unchanged; results are bit-identical)
        self.fusion: dict[int, dict] = {}
        self.fused_away: set[int] = set()
        for oid, op in graph.operators.items():
            if op.kind != "relu_forward":
                continue
            p = graph.producer_of(op.inputs[0])
            if p is None or graph.operators[p].kind != "conv2d_forward":
                continue
            if self.slot[p] != self.slot[oid]:
                continue
            self.fusion[p] = {"relu_out": graph.tensors[op.outputs[0]].name}
            self.fused_away.add(oid)
        # bias gradient: a conv2d_backward_bias on the same stream after the
        # conv2d_backward_weight reading the same dy takes its sums from the
        # weight gradient's pass over dy (within tolerance, not bit-identical to
        # the stand-alone bias kernel: different summation blocking)
        pos = {oid: i for i, oid in enumerate(self.order)}
        for oid, op in graph.operators.items():
            if op.kind != "conv2d_backward_bias":
                continue
            sib = [c for c, _ in graph.consumers_of(op.inputs[0])
                   if graph.operators[c].kind == "conv2d_backward_weight"
                   and self.slot[c] == self.slot[oid] and pos[c] < pos[oid] and c not in self.fusion]
            if sib:
                self.fusion[sib[0]] = {"db": graph.tensors[op.outputs[0]].name}
                self.fused_away.add(oid)
        # concat elision (Inception): when every part of a concat_forward is a
        # fused conv+ReLU output consumed by nothing else, each conv epilogue
        # writes its ReLU straight into its channel slice of the concat output;
        # when every part of a concat_backward feeds exactly one relu_backward,
        # each relu_backward reads its slice of the concatenated gradient.  The
        # concat operators become no-ops and their per-branch tensors are never
        # materialised (``elided``); every other tensor is bit-identical.
        self.elided: set[str] = set()
        relu_src = {f["relu_out"]: p for p, f in self.fusion.items() if "relu_out" in f}
        for oid, op in graph.operators.items():
            if op.kind == "concat_forward":
                parts = [graph.tensors[t] for t in op.inputs]
                convs = [relu_src.get(t.name) for t in parts]
                if any(c is None for c in convs) or any(
                        len(graph.consumers_of(t)) != 1 for t in op.inputs):
                    continue
                out = graph.tensors[op.outputs[0]]
                c0 = 0
                for conv, t in zip(convs, parts):
                    self.fusion[conv]["relu_slice"] = (out.name, out.shape, c0)
                    self.elided.add(t.name)
                    c0 += t.shape[1]
                self.fused_away.add(oid)
            elif op.kind == "concat_backward":
                dy = graph.tensors[op.inputs[0]]
                users = []
                for t in op.outputs:
                    cons = graph.consumers_of(t)
                    ok = (len(cons) == 1 and graph.operators[cons[0][0]].kind == "relu_backward"
                          and graph.operators[cons[0][0]].inputs[1] == t)
                    users.append(cons[0][0] if ok else None)
                if any(u is None for u in users):
                    continue
                # a rank-ordered sum feeding only this concat_backward (the gradient
                # of an Inception module's input) is folded in as well
                agg = graph.producer_of(op.inputs[0])
                parts = None
                if (agg is not None and graph.operators[agg].kind == "aggregate"
                        and graph.operators[agg].attrs.get("mode", "mean") == "sum"
                        and len(graph.consumers_of(op.inputs[0])) == 1
                        and len(graph.operators[agg].inputs) <= 32):
                    parts = [graph.tensors[t].name for t in graph.operators[agg].inputs]
                    self.fused_away.add(agg)
                    self.elided.add(dy.name)
                c0 = 0
                for u, t in zip(users, op.outputs):
                    self.fusion[u] = ({"dy_parts": (parts, c0, dy.shape[1])} if parts else
                                      {"dy_slice": (dy.name, c0, dy.shape[1])})
                    self.elided.add(graph.tensors[t].name)
                    c0 += graph.tensors[t].shape[1]
                self.fused_away.add(oid)

        foldable = tuple(k for k in os.environ.get(RELU_FOLD_ENV, RELU_FOLD_DEFAULT).split(",") if k)
        # max-pool mask elision: when a maxpool_forward's argmax mask feeds only
        # maxpool_backward operators of the same x and attributes, the backward
        # also absorbs the relu_backward of the ReLU that produced x, and the
        # shared-memory staged kernels fit the shape, the graph's float mask is
        # never stored: the forward writes a signed mask instead (argmax, with
        # the sign of the window's maximum = the ReLU mask at that pixel), so
        # the backward reads neither x nor a (pool1: 0.23 -> 0.12 ms); with
        # PURINE_B200_POOL_SMASK=0 the backward recomputes every argmax from x
        # (the forward's own scan: bit-identical).  Elsewhere the staged
        # backward reads the graph's mask (a quarter of x at stride 2)
        for oid, op in graph.operators.items():
            if op.kind != "maxpool_forward" or len(op.outputs) != 2:
                continue
            mk = op.outputs[1]
            cons = graph.consumers_of(mk)
            if not cons or any(
                    graph.operators[c].kind != "maxpool_backward" or
                    graph.operators[c].inputs[0] != op.inputs[0] or
                    graph.operators[c].inputs[1] != mk or
                    graph.operators[c].attrs != op.attrs for c, _ in cons):
                continue
            if not _pool_relu_foldable(graph, cons, foldable):
                continue
            if os.environ.get(POOL_SMASK_ENV, "1") != "0" and _pool_staged(graph, op, 3):
                # the signed mask: each window's argmax with the sign of its
                # maximum, which is the folded ReLU's mask at that pixel -- the
                # backward reads neither x nor the graph's float mask
                name = graph.tensors[mk].name + "#signed"
                self.fusion.setdefault(oid, {})["pool_smask"] = name
                for c, _ in cons:
                    self.fusion.setdefault(c, {})["pool_smask"] = name
                self.elided.add(graph.tensors[mk].name)
                continue
            if not _pool_staged(graph, op):
                continue
            self.fusion.setdefault(oid, {})["pool_no_mask"] = True
            for c, _ in cons:
                self.fusion.setdefault(c, {})["pool_recompute"] = True
            self.elided.add(graph.tensors[mk].name)

        # relu_backward folded into the operator producing its dy (a data
        # gradient epilogue, the max-pool or LRN backward kernel) when that dy
        # has no other consumer: the producer writes relu_backward's dx directly
        # (bit-identical: the same x > 0 ? g : 0 select), dy is never stored
        for oid, op in graph.operators.items():
            if op.kind != "relu_backward" or oid in self.fusion or len(op.inputs) != 2:
                continue
            g = op.inputs[1]
            p = graph.producer_of(g)
            if (p is None or graph.operators[p].kind not in foldable
                    or (p in self.fusion
                        and set(self.fusion[p]) not in ({"pool_recompute"}, {"pool_smask"}))
                    or len(graph.consumers_of(g)) != 1 or p in self.fused_away):
                continue
            rx = graph.tensors[op.inputs[0]].name
            pk = graph.operators[p]
            if pk.kind == "maxpool_backward":
                # staged backward only, and only when the pool's own input is this
                # ReLU's output: relu(a) > 0 <=> a > 0, so x is the mask
                if p not in self.fusion or not any(
                        graph.operators[c].kind == "relu_forward"
                        and graph.operators[c].outputs[0] == pk.inputs[0]
                        for c, _ in graph.consumers_of(op.inputs[0])):
                    continue
                self.fusion[p].update({"relu_from_x": True,
                                       "relu_dx": graph.tensors[op.outputs[0]].name})
                self.fused_away.add(oid)
                self.elided.add(graph.tensors[g].name)
                continue
            if pk.kind == "lrn_backward":
                # the LRN's own input is the ReLU's output: its sign is the
                # same mask (relu(a) > 0 <=> a > 0) and the kernel already
                # reads it -- the pre-activation is not read again
                for c, _ in graph.consumers_of(op.inputs[0]):
                    cop = graph.operators[c]
                    if cop.kind == "relu_forward" and cop.outputs[0] == pk.inputs[0]:
                        rx = graph.tensors[pk.inputs[0]].name
            elif os.environ.get(PREACT_ENV, "1") != "0":
                # the ReLU's own output as the mask (relu(a) > 0 <=> a > 0, the
                # same select bit for bit) when it is materialised as itself:
                # the pre-activation is then left without a reader
                ro = self._relu_output_of(graph, op.inputs[0])
                if ro is not None:
                    rx = ro
            self.fusion[p] = {"relu_x": rx, "relu_dx": graph.tensors[op.outputs[0]].name}
            self.fused_away.add(oid)
            self.elided.add(graph.tensors[g].name)

        # LRN scale elision: when an lrn_forward's scale feeds only lrn_backward
        # operators of the same (x, y) and attributes, the backward recomputes
        # scale and y from x (the forward's exact operation sequence, so
        # bit-identical) and the forward never stores scale
        for oid, op in graph.operators.items():
            if op.kind != "lrn_forward" or len(op.outputs) != 2 or op.attrs.get("size", 5) != 5:
                continue
            sc = op.outputs[1]
            cons = graph.consumers_of(sc)
            if not cons or any(
                    graph.operators[c].kind != "lrn_backward" or
                    tuple(graph.operators[c].inputs[:3]) != (op.inputs[0], op.outputs[0], sc) or
                    graph.operators[c].attrs != op.attrs for c, _ in cons):
                continue
            self.fusion.setdefault(oid, {})["lrn_no_scale"] = True
            for c, _ in cons:
                self.fusion.setdefault(c, {})["lrn_recompute"] = True
            self.elided.add(graph.tensors[sc].name)

        self._preact_elision(graph)
        self._group_1x1(graph)
        self._group_1x1_dgrad(graph)
        self.finite_mode = _finite_mode()
        self.finite_watch = _finite_watch(graph, self, self.finite_mode)

    def _relu_output_of(self, graph: BiGraph, a: int) -> str | None:
        """Name of relu(a) when a is a conv pre-activation whose ReLU the conv
        epilogue writes as a tensor of its own (not into a concat slice)."""
        pa = graph.producer_of(a)
        f = self.fusion.get(pa) if pa is not None else None
        if not f or "relu_out" not in f or "relu_slice" in f or f["relu_out"] in self.elided:
            return None
        return f["relu_out"]

    def _preact_elision(self, graph: BiGraph) -> None:
        """Pre-activation elision: a fused conv+ReLU whose pre-activation y has
        no reader left stores only relu(y) (``no_y``; y joins ``elided``).  The
        relu_backward of such a ReLU takes relu(y) as its mask -- relu(a) > 0
        <=> a > 0, so every select is bit-identical: folded into a data
        gradient it reads the ReLU output (the fold above), folded into the
        max-pool / LRN backward it reads their x, and reading a slice of an
        elided concat gradient it reads the ReLU's slice of the concat output
        (``x_slice``).  Saves one store of every conv output (1.65 GB per
        GoogLeNet step at batch 128)."""
        if os.environ.get(PREACT_ENV, "1") == "0":
            return
        relu_slice = {}
        for p, f in self.fusion.items():
            if "relu_slice" in f:
                relu_slice[graph.operators[p].outputs[0]] = f["relu_slice"]
        for oid, op in graph.operators.items():
            f = self.fusion.get(oid)
            if (op.kind == "relu_backward" and f and ("dy_slice" in f or "dy_parts" in f)
                    and op.inputs[0] in relu_slice):
                name, shape, c0 = relu_slice[op.inputs[0]]
                f["x_slice"] = (name, c0, shape[1])
        readers = {f["relu_x"] for f in self.fusion.values() if "relu_x" in f}
        for oid, op in graph.operators.items():
            f = self.fusion.get(oid)
            if op.kind != "conv2d_forward" or not f or not ("relu_out" in f or "relu_slice" in f):
                continue
            y = op.outputs[0]
            yname = graph.tensors[y].name
            if yname in readers:
                continue
            ok = True
            for c, _ in graph.consumers_of(y):
                cop, cf = graph.operators[c], self.fusion.get(c, {})
                if cop.kind == "relu_forward" and c in self.fused_away:
                    continue  # computed by this conv's epilogue
                if cop.kind == "relu_backward" and (c in self.fused_away or "x_slice" in cf):
                    continue  # folded (its mask is read elsewhere) or reads the slice
                ok = False
                break
            if ok:
                f["no_y"] = True
                self.elided.add(yname)

    def _group_1x1_dgrad(self, graph: BiGraph) -> None:
        """The backward half of the Inception 1x1 grouping: the data gradients
        of sibling 1x1 convolutions (same x) whose outputs only feed the same
        aggregate(sum) -- the module's input gradient -- are computed as ONE
        GEMM over their K-concatenated dy, which IS their sum
        (bf_conv1x1_dgrad_group): one launch and one dx write instead of three,
        and the aggregate (or the ReLU-backward slice sums it is folded into)
        adds two parts instead of four.  The GEMM runs at the LAST member in
        serial order (every member's dy is ready there) into that member's
        output buffer; the earlier members become no-ops.  The member outputs
        are listed in ``elided`` (none holds its own part any more); the sum
        is reassociated, so it agrees at the contraction tolerance."""
        if os.environ.get(GROUP_ENV, "1") == "0":
            return
        from .kinds import conv_attrs

        pos = {oid: i for i, oid in enumerate(self.order)}
        for aid, agg in graph.operators.items():
            if agg.kind != "aggregate" or agg.attrs.get("mode", "mean") != "sum":
                continue
            cand: dict[int, list[int]] = {}
            for t in agg.inputs:
                p = graph.producer_of(t)
                if p is None or p in self.fusion or p in self.fused_away:
                    continue
                op = graph.operators[p]
                if op.kind != "conv2d_backward_data" or len(graph.consumers_of(t)) != 1:
                    continue
                w = graph.tensors[op.inputs[1]]
                x = graph.tensors[op.inputs[0]]
                stride, pad, _floor = conv_attrs(op.attrs)
                if (len(w.shape) != 4 or w.shape[2:] != (1, 1) or stride != 1 or pad != 0
                        or (x.shape[2] * x.shape[3]) % 4):
                    continue
                cand.setdefault(op.inputs[0], []).append(p)
            for members in cand.values():
                if len(members) < 2:
                    continue
                members = sorted(members, key=pos.__getitem__)[-4:]
                lead = members[-1]
                self.fusion[lead] = {"group_dgrad": [graph.operators[m] for m in members]}
                for m in members[:-1]:
                    self.fused_away.add(m)
                    self.fusion[m] = {"group_member": lead}
                    # the lead reads every member's dy: wait for their producers
                    for t in graph.operators[m].inputs:
                        pr = graph.producer_of(t)
                        if pr is not None and self.slot[pr] != self.slot[lead] \
                                and pr not in self.waits[lead]:
                            self.waits[lead].append(pr)
                            self.signals.add(pr)
                gone = {graph.tensors[graph.operators[m].outputs[0]].name for m in members[:-1]}
                lead_out = graph.tensors[graph.operators[lead].outputs[0]].name
                for m in members:
                    self.elided.add(graph.tensors[graph.operators[m].outputs[0]].name)
                # the aggregate (or the slice sums it is folded into) now adds the
                # group's sum once, in the lead's place, and skips the others
                names = [graph.tensors[t].name for t in agg.inputs]
                kept = [n for n in names if n not in gone]
                self.fusion.setdefault(aid, {})["agg_parts"] = kept
                for f in self.fusion.values():
                    if "dy_parts" in f and f["dy_parts"][0] == names:
                        _names, c0, ctot = f["dy_parts"]
                        f["dy_parts"] = (kept, c0, ctot)
                assert lead_out in kept

    def _group_1x1(self, graph: BiGraph) -> None:
        """Horizontal fusion (Inception): the 1x1 stride-1 conv2d_forward
        operators reading the same x -- 1x1, 3x3_reduce, 5x5_reduce -- run as
        ONE GEMM over their concatenated output channels (x read once, one
        launch, a wider N tile), executed by the first of them in serial order
        with each member's epilogue fusion (ReLU, concat slice) kept.  The
        other members become no-ops whose streams wait for that leader, so
        everything downstream of a member still follows its producer.  The
        wider GEMM tile may change the tensor-core accumulation scheme (the
        separate small-term accumulator needs BN <= 128), so results agree with
        the ungrouped kernels at the contraction tolerance, not bit for bit."""
        if os.environ.get(GROUP_ENV, "1") == "0":
            return
        from .kinds import conv_attrs

        pos = {oid: i for i, oid in enumerate(self.order)}
        by_x: dict[int, list[int]] = {}
        for oid, op in graph.operators.items():
            if op.kind != "conv2d_forward" or oid in self.fused_away:
                continue
            w = graph.tensors[op.inputs[1]]
            x = graph.tensors[op.inputs[0]]
            if len(w.shape) != 4 or w.shape[2:] != (1, 1) or len(x.shape) != 4:
                continue
            stride, pad, _floor = conv_attrs(op.attrs)
            if stride != 1 or pad != 0 or (x.shape[2] * x.shape[3]) % 4:
                continue
            if set(self.fusion.get(oid, {})) - {"relu_out", "relu_slice", "no_y"}:
                continue
            by_x.setdefault(op.inputs[0], []).append(oid)
        for members in by_x.values():
            if len(members) < 2:
                continue
            members = sorted(members, key=pos.__getitem__)[:4]
            lead = members[0]
            self.fusion.setdefault(lead, {})["group_fwd"] = [
                (graph.operators[m], dict(self.fusion.get(m, {}))) for m in members]
            for m in members[1:]:
                self.fused_away.add(m)
                self.fusion.setdefault(m, {})["group_member"] = lead
                if lead not in self.waits[m]:
                    self.waits[m].append(lead)
                self.signals.add(lead)

    def _split_branches(self, graph: BiGraph, branches: int) -> None:
        """Event-driven device concurrency inside a lane: the lane's operators
        are spread over up to ``branches`` CUDA streams by greedy chain
        decomposition in serial order (an operator continues the stream whose
        last operator produced one of its inputs, else takes a new or the
        least recently used stream), so independent Inception branches run
        concurrently; every cross-stream input becomes an event wait (``waits``).
        Host dispatch order is unchanged.  Lanes carrying collectives or copies
        keep one stream (NCCL calls must stay ordered per communicator)."""
        serial_kinds = {"dp_exchange", "copy", "swap"}
        keep = {self.slot[oid] for oid, op in graph.operators.items() if op.kind in serial_kinds}
        subs: dict[int, list[int]] = {}
        last_op: dict[int, int] = {}
        last_use: dict[int, int] = {}
        done: set[int] = set()
        for i, oid in enumerate(self.order):
            base = self.slot[oid]
            if base in keep:
                continue
            pool = subs.setdefault(base, [base])
            chosen = None
            op = graph.operators[oid]
            if op.kind == "conv2d_backward_bias":  # stays with its weight gradient (fusion)
                for c, _ in graph.consumers_of(op.inputs[0]):
                    if graph.operators[c].kind == "conv2d_backward_weight" and c in done:
                        chosen = self.slot[c]
            for tid in (op.inputs if chosen is None else ()):
                p = graph.producer_of(tid)
                if p is not None and self.slot.get(p) in pool and last_op.get(self.slot[p]) == p:
                    chosen = self.slot[p]
                    break
            if chosen is None:
                if len(pool) < branches and all(s in last_op for s in pool):
                    chosen = self.n_slots
                    self.n_slots += 1
                    pool.append(chosen)
                else:
                    chosen = min(pool, key=lambda s: last_use.get(s, -1))
            self.slot[oid] = chosen
            last_op[chosen] = oid
            last_use[chosen] = i
            done.add(oid)


FINITE_ENV = "PURINE_B200_CHECK_FINITE"  # "sinks" (default) | "all" | "0"
# kinds whose outputs the reference checks for non-finite values (ops.py:61-64 and
# its call sites ops.py:175-456), plus this library's extension kinds
FINITE_KINDS = frozenset({
    "fc_forward", "fc_backward", "fc_backward_data", "fc_backward_weight", "fc_backward_bias",
    "conv2d_forward", "conv2d_backward", "conv2d_backward_data", "conv2d_backward_weight",
    "conv2d_backward_bias", "relu_forward", "relu_backward", "softmax_xent", "sgd_update",
    "aggregate", "sgd_momentum", "dp_exchange", "maxpool_forward", "maxpool_backward",
    "avgpool_forward", "avgpool_backward", "lrn_forward", "lrn_backward", "concat_forward",
    "concat_backward"})


def _finite_mode() -> str:
    raw = os.environ.get(FINITE_ENV, "sinks").strip().lower()
    if raw in ("0", "off", "none", "false"):
        return "off"
    if raw not in ("sinks", "all"):
        raise DispatchError(f"{FINITE_ENV} must be sinks, all or 0, got {raw!r}")
    return raw


def _finite_watch(graph: BiGraph, plan, mode: str) -> list[str]:
    """Tensors checked for non-finite values after the graph's last kernel.

    The reference checks every kernel output on the host (ops.py:61-64).  Here
    the check is one device pass per graph into a sticky flag: ``sinks`` (default)
    covers the outputs nothing in the graph consumes -- the loss and the updated
    parameters, which every forward / gradient value flows into -- and ``all``
    every materialised output of a checked kind (the reference's coverage, at
    the cost of re-reading every activation).  When the flag fires, the first
    offending operator in serial order is located on the host and reported as
    the reference reports it (`raise_if_nonfinite`)."""
    if mode == "off":
        return []
    out: list[str] = []
    seen: set[str] = set()
    for oid in plan.order:
        op = graph.operators[oid]
        if op.kind not in FINITE_KINDS:
            continue
        for tid in op.outputs:
            name = graph.tensors[tid].name
            if name in seen or name in plan.elided:
                continue
            if mode == "sinks" and graph.consumers_of(tid):
                continue
            seen.add(name)
            out.append(name)
    return out


def _launch_finite_check(store: TensorStore, names: list[str], stream) -> None:
    if not names:
        return
    import ctypes as C

    from . import _native

    flag = store.finite_flag()
    ts = [store.get(n) for n in names]
    ptrs = (C.c_void_p * len(ts))(*[t.ptr for t in ts])
    lens = (C.c_int64 * len(ts))(*[t.numel for t in ts])
    _native.lib()("bf_check_finite_list", ptrs, lens, len(ts), flag.data_ptr(), stream.cuda_stream)


def raise_if_nonfinite(store: TensorStore, graphs, *, sync: bool = True,
                       cap: int | None = None) -> None:
    """Read the store's sticky non-finite flag; if set, name the first operator
    (serial order over ``graphs``) holding a non-finite output and raise
    ``DispatchError("operator 'x' failed: <kind>: non-finite value in output")``
    -- the reference's first-error report of ops.py:61-64 (dispatcher.py:344-346)."""
    if not store.has_finite_flag():
        return
    if sync:
        torch.cuda.synchronize(store.device)
    if not store.finite_flag_set():
        return
    store.reset_finite_flag()
    for g in graphs:
        plan = _plan(g, _env_lane_cap() if cap is None else cap)
        for oid in plan.order:
            op = g.operators[oid]
            if op.kind not in FINITE_KINDS:
                continue
            if op.kind == "softmax_xent":  # the kernel turns a bad label into a NaN loss
                lab = store.tensor(g.tensors[op.inputs[1]].name)
                k = g.tensors[op.inputs[0]].shape[1]
                if not bool(((lab == lab.floor()) & (lab >= 0) & (lab < k)).all()):
                    raise DispatchError(f"operator {op.name!r} failed: softmax_xent: labels "
                                        f"must be integral and in [0, {k})")
            for tid in op.outputs:
                name = g.tensors[tid].name
                if name in plan.elided or not store.has(name):
                    continue
                if not bool(torch.isfinite(store.tensor(name)).all()):
                    raise DispatchError(f"operator {op.name!r} failed: "
                                        f"{op.kind}: non-finite value in output")
    raise DispatchError("non-finite value in a graph output (the producing operator's "
                        "buffers were overwritten before it could be located)")


BRANCH_ENV = "PURINE_B200_BRANCH_STREAMS"  # device streams per compute lane (1 = lane-exclusive)


def _branch_streams() -> int:
    raw = os.environ.get(BRANCH_ENV, "8")
    try:
        k = int(raw)
    except ValueError:
        raise DispatchError(f"{BRANCH_ENV} must be an integer, got {raw!r}") from None
    if k < 1:
        raise DispatchError(f"{BRANCH_ENV} must be >= 1, got {k}")
    return k


FUSE_ENV = "PURINE_B200_FUSE"  # "0" disables epilogue fusion (A/B and debugging)
GROUP_ENV = "PURINE_B200_GROUP_1X1"  # "0" disables the Inception 1x1 horizontal fusion
PREACT_ENV = "PURINE_B200_PREACT_ELISION"  # "0" keeps every conv pre-activation stored
# producer kinds that may absorb the relu_backward after them (all three have the
# kernel support; measured net gains decide the default)
POOL_SMASK_ENV = "PURINE_B200_POOL_SMASK"  # "0": recompute the argmax from x instead
RELU_FOLD_ENV = "PURINE_B200_RELU_FOLD"
RELU_FOLD_DEFAULT = "conv2d_backward_data,lrn_backward,maxpool_backward"


def _pool_relu_foldable(graph: BiGraph, cons, foldable) -> bool:
    """The single maxpool_backward in ``cons`` feeds exactly one relu_backward
    whose ReLU produced the pool's input (the fold through x, see _Plan)."""
    if "maxpool_backward" not in foldable or len(cons) != 1:
        return False
    pb = graph.operators[cons[0][0]]
    users = graph.consumers_of(pb.outputs[0])
    if len(users) != 1:
        return False
    rb = graph.operators[users[0][0]]
    if rb.kind != "relu_backward" or len(rb.inputs) != 2 or rb.inputs[1] != pb.outputs[0]:
        return False
    return any(graph.operators[c].kind == "relu_forward"
               and graph.operators[c].outputs[0] == pb.inputs[0]
               for c, _ in graph.consumers_of(rb.inputs[0]))


def _pool_staged(graph: BiGraph, op, mode: int = 1) -> bool:
    """Whether the shared-memory staged max-pool kernels take this shape (both
    directions; mode 1: the backward recomputing the argmax from x, 3: the
    signed-mask pair): the condition for eliding the float argmax mask."""
    from .kinds import pool_attrs

    try:
        from . import _native

        k, s, p = pool_attrs(op.attrs)
        n, c, h, w = graph.tensors[op.inputs[0]].shape
        _, _, ph, pw = graph.tensors[op.outputs[0]].shape
        ok = _native.lib().raw("bf_maxpool_staged_ok")
        if mode == 3:
            return bool(ok(n, c, h, w, ph, pw, k, s, p, 3))
        return bool(ok(n, c, h, w, ph, pw, k, s, p, 0) and ok(n, c, h, w, ph, pw, k, s, p, 1))
    except Exception:  # noqa: BLE001 - no library: the plain kernels run (and fail loudly)
        return False


def _fusion_enabled(registry) -> bool:
    if os.environ.get(FUSE_ENV, "1") == "0":
        return False
    # only when both kinds run the product kernels (a user-registered kind is
    # never bypassed)
    return all(registry.get(k) is KINDS[k] for k in ("conv2d_forward", "relu_forward",
                                                      "conv2d_backward_weight",
                                                      "conv2d_backward_bias", "concat_forward",
                                                      "concat_backward", "relu_backward",
                                                      "aggregate", "conv2d_backward_data",
                                                      "maxpool_forward", "maxpool_backward",
                                                      "lrn_forward", "lrn_backward"))


def _plan(graph: BiGraph, cap: int) -> _Plan:
    """The graph's launch plan, cached on the graph object itself (keyed by the
    lane cap, branch streams and non-finite mode; rebuilt when the graph grew).
    An id()-keyed global cache would hand a dead graph's plan to a new graph
    that happens to reuse its address."""
    branches = _branch_streams()
    key = (cap, branches, _finite_mode(), os.environ.get(GROUP_ENV, "1"),
           os.environ.get(RELU_FOLD_ENV, RELU_FOLD_DEFAULT), os.environ.get(PREACT_ENV, "1"),
           os.environ.get(POOL_SMASK_ENV, "1"))
    stamp = len(graph.insertion_order) * 1_000_003 + len(graph.tensors)
    cache = graph.__dict__.setdefault("_launch_plans", {})
    hit = cache.get(key)
    if hit is not None and hit[0] == stamp:
        return hit[1]
    p = _Plan(graph, cap, branches)
    cache[key] = (stamp, p)
    return p


# ---------------------------------------------------------------------------
# one graph run


class _TimeBase:
    def __init__(self) -> None:
        self.event = torch.cuda.Event(enable_timing=True)
        self.event.record()

    def ns(self, ev: torch.cuda.Event) -> int:
        return int(round(self.event.elapsed_time(ev) * 1e6))


def _enqueue(graph, store, registry, cap, ctx, trace, base):
    """Launch every operator of ``graph``; returns (dispatch names, timing events)."""
    plan = _plan(graph, cap)
    pool = lanes_of(store)
    cur = torch.cuda.current_stream(store.device)
    fork = torch.cuda.Event()
    fork.record(cur)
    slots = [pool.get(i, i in plan.high_priority) for i in range(plan.n_slots)]
    for s, _ in slots:
        s.wait_event(fork)
    done_ev: dict[int, torch.cuda.Event] = {}
    timing: list[tuple[int, torch.cuda.Event, torch.cuda.Event]] = []
    names: list[str] = []
    from . import _native

    failure = None
    fuse = _fusion_enabled(registry)
    for oid in plan.order:
        op = graph.operators[oid]
        spec = registry.get(op.kind)
        if spec is None:
            failure = (op.name, DispatchError(
                f"operator kind {op.kind!r} unknown to registry (op {op.name!r})"))
            break
        stream, ws = slots[plan.slot[oid]]
        for p in plan.waits[oid]:
            stream.wait_event(done_ev[p])
        ctx.stream = stream.cuda_stream
        ctx.workspace = ws
        ctx.lane = lane_of(op)
        ctx.fused = plan.fusion.get(oid) if fuse else None
        try:
            with torch.cuda.stream(stream):
                if trace:
                    t_start = torch.cuda.Event(enable_timing=True, external=True)
                    t_start.record(stream)
                delay = float(op.attrs.get("delay_s", 0.0) or 0.0)
                if delay > 0:
                    _native.lib()("bf_delay_ns", int(delay * 1e9), ctx.stream)
                if not (fuse and oid in plan.fused_away):
                    spec.execute(ctx, op)
                else:  # computed by a neighbour (see _Plan); still owns its output buffers
                    for tid in op.outputs:
                        t = graph.tensors[tid]
                        store.ensure(t.name, t.shape)
                if trace:
                    t_end = torch.cuda.Event(enable_timing=True, external=True)
                    t_end.record(stream)
                    timing.append((oid, t_start, t_end))
        except BaseException as exc:  # noqa: BLE001 - first error wins
            failure = (op.name, exc)
            break
        if oid in plan.signals:
            ev = torch.cuda.Event()
            ev.record(stream)
            done_ev[oid] = ev
        names.append(op.name)
    for s, _ in slots:
        join = torch.cuda.Event()
        join.record(s)
        cur.wait_event(join)
    if failure is None:
        _launch_finite_check(store, plan.finite_watch, cur)
    if failure is not None:
        for s, _ in slots:  # drain what was already enqueued
            s.synchronize()
        name, exc = failure
        if isinstance(exc, DispatchError) and "unknown to registry" in str(exc):
            raise exc
        raise DispatchError(f"operator {name!r} failed: {exc}") from exc
    return names, timing


CAPTURE_ENV = "PURINE_B200_CAPTURE"  # "0": run() walks the graph every call
_REPLAY_CACHE_MAX = 8  # bindings remembered per graph (a training sequence uses two)


def _replayable(graph, store, registry, trace, transport, copy_latency_s) -> bool:
    """An untraced run of a device graph through the product kinds can be a
    CUDA-graph replay: the launch walk is deterministic and its arguments
    depend only on the store's buffer bindings (and the plan)."""
    if trace or transport is not None or copy_latency_s or registry is not KINDS:
        return False
    if store.device.type != "cuda" or os.environ.get(CAPTURE_ENV, "1") == "0":
        return False
    from .gpu_ops import HOST_ONLY

    return not all(op.kind in HOST_ONLY for op in graph.operators.values())


def _run_replayed(graph, store, registry, cap, ctx) -> list[str]:
    """run(trace=False) through a replay cache: the first call with a given
    buffer binding walks the graph (allocating outputs and workspaces), the
    second captures the same walk into a CUDA graph, later ones replay it.
    The key is the store's binding signature (serial, allocation epoch, swap
    parity -- a training sequence alternates between two), the lane cap and
    the launch plan (which carries the fusion / stream environment)."""
    plan = _plan(graph, cap)
    key = (store.binding_sig(), cap, id(plan))
    cache = graph.__dict__.setdefault("_replays", {})
    ent = cache.get(key)
    if ent is not None and ent[0] is not None:
        cache[key] = cache.pop(key)  # most recently used last
        ent[0].replay()
        return ent[1]
    if ent is None:
        names, _ = _enqueue(graph, store, registry, cap, ctx, False, None)
        while len(cache) >= _REPLAY_CACHE_MAX:  # bindings that never recur: evict the oldest
            cache.pop(next(iter(cache)))
        cache[key] = (None, names)
        return names
    pool = getattr(store, "_replay_pool", None)
    if pool is None:
        pool = torch.cuda.graph_pool_handle()
        store._replay_pool = pool
    cg = torch.cuda.CUDAGraph()
    cap_stream = torch.cuda.Stream(device=store.device)
    cap_stream.wait_stream(torch.cuda.current_stream(store.device))
    with torch.cuda.graph(cg, pool=pool, stream=cap_stream):
        names, _ = _enqueue(graph, store, registry, cap, ctx, False, None)
    cache[key] = (cg, names)
    cg.replay()
    return names


def run(graph: BiGraph, store: TensorStore, registry: dict | None = None, *,
        max_workers: int | None = None, iteration: int = 0, t0=None,
        transport: object | None = None, copy_latency_s: float = 0.0,
        validated: bool = False, trace: bool = True) -> RunReport:
    """Execute one graph to completion (dispatcher.py:378-417).

    With ``trace=True`` (default, as in the reference) the call returns after
    the device finished the graph and the report carries per-operator device
    times.  With ``trace=False`` it returns as soon as everything is enqueued.
    """
    if not validated:
        rep = graph.validate()
        if not rep.ok:
            raise DispatchError("graph failed validation: " + "; ".join(rep.violations))
    _check_sources(graph, store)
    registry = KINDS if registry is None else registry
    cap = max_workers if max_workers is not None else _env_lane_cap()
    base = t0 if isinstance(t0, _TimeBase) else None
    host0 = time.monotonic_ns()
    if trace and base is None:
        base = _TimeBase()
    ctx = RunContext(store=store, graph=graph, iteration=iteration, transport=transport,
                     copy_latency_s=copy_latency_s)
    if _replayable(graph, store, registry, trace, transport, copy_latency_s):
        names = _run_replayed(graph, store, registry, cap, ctx)
        return RunReport(trace=[], elapsed=time.monotonic_ns() - host0, iteration=iteration,
                         dispatch_order=names)
    names, timing = _enqueue(graph, store, registry, cap, ctx, trace, base)
    records: list[TraceRecord] = []
    if trace:
        end = torch.cuda.Event(enable_timing=True)
        end.record(torch.cuda.current_stream(store.device))
        end.synchronize()
        for oid, a, b in timing:
            op = graph.operators[oid]
            s, e = base.ns(a), base.ns(b)
            records.append(TraceRecord(oid, op.name, lane_of(op), s, max(e, s + 1), iteration))
        records.sort(key=lambda r: (r.start, r.end))
        raise_if_nonfinite(store, [graph], sync=False, cap=cap)
    return RunReport(trace=records, elapsed=time.monotonic_ns() - host0, iteration=iteration,
                     dispatch_order=names)


def run_sequence(seq: GraphSequence, store: TensorStore, registry: dict | None = None, *,
                 max_workers: int | None = None, transport: object | None = None,
                 copy_latency_s: float = 0.0, before_iteration=None, after_graph=None,
                 iterations: int | None = None, trace: bool = True) -> list[RunReport]:
    """Run every graph of ``seq`` in order, ``iterations`` times (dispatcher.py:420-469).

    Graph completion is the synchronisation point: graph i+1's streams wait
    on an event joined from all of graph i's streams.  ``before_iteration``
    and ``after_graph`` hooks behave as in the reference.
    """
    for g in seq.graphs:
        rep = g.validate()
        if not rep.ok:
            raise DispatchError("graph failed validation: " + "; ".join(rep.violations))
    base = _TimeBase() if trace else None
    reports: list[RunReport] = []
    rounds = seq.iterations if iterations is None else iterations
    for it in range(rounds):
        if before_iteration is not None:
            before_iteration(it, store)
        for gi, g in enumerate(seq.graphs):
            rep = run(g, store, registry, max_workers=max_workers, iteration=it, t0=base,
                      transport=transport, copy_latency_s=copy_latency_s, validated=True,
                      trace=trace)
            rep.graph_index = gi
            reports.append(rep)
            if after_graph is not None:
                after_graph(rep, store)
    if not trace:  # traced runs checked after every graph; here once, at the end
        raise_if_nonfinite(store, seq.graphs, cap=max_workers)
    return reports
