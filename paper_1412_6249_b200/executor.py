"""CUDA-graph replay of a graph sequence (launch-overhead removal).

An iteration of GoogLeNet enqueues ~520 operators (~1k kernels); walking the
graph in Python every iteration would cost more host time than the device
needs.  The dispatcher's launch walk is deterministic, so it is captured once
into a `torch.cuda.CUDAGraph` per graph of the sequence and replayed.

Buffer bindings change every iteration: the swap graph exchanges
``w`` <-> ``w_new`` handles (ops.py:93-102).  A swap graph is an involution,
so there are exactly two bindings; each graph is captured once per binding
parity and the replays alternate (ping-pong).  Host-only graphs (pure swap
graphs) are not captured: their handle exchanges run on the host each
iteration so `TensorStore` lookups stay truthful.
"""

from __future__ import annotations

import torch

from .dispatcher import (DispatchError, RunContext, RunReport, _check_sources, _enqueue,
                         _env_lane_cap, lanes_of, raise_if_nonfinite)
from .gpu_ops import HOST_ONLY
from .graph import GraphSequence
from .kinds import KINDS

__all__ = ["CapturedSequence"]


def _binding(store) -> dict[str, int]:
    return {n: store.get(n).ptr for n in store.names()}


class CapturedSequence:
    """Captured replay of ``seq`` on ``store``'s device.

    Call `prepare()` after the store holds every source tensor (parameters,
    data, labels); it runs one eager iteration (which allocates every
    buffer and advances the parameters by one step, like any iteration) and
    then captures.  `step()` replays one full iteration."""

    def __init__(self, seq: GraphSequence, store, registry: dict | None = None,
                 max_workers: int | None = None, trace: bool = False) -> None:
        self.seq = seq
        self.store = store
        self.registry = KINDS if registry is None else registry
        self.cap = max_workers if max_workers is not None else _env_lane_cap()
        self.parity = 0
        self.graphs: list[list[torch.cuda.CUDAGraph | None]] = [[], []]
        self.host_only = [all(op.kind in HOST_ONLY for op in g.operators.values())
                          for g in seq.graphs]
        self.ready = False
        self.trace = trace
        # per parity, per graph: [(op id, start event, end event)] recorded by the replays
        self.timing: list[list[list]] = [[], []]
        self.launches_per_step = 0
        self._copy_stream = None  # prefetch(): host->device copies of the next step's inputs
        self._staging: dict[tuple[int, str], torch.Tensor] = {}
        self._pending = None
        self._slot = 0
        self._consumed: list = [None, None]
        self._flag_host = None  # pinned mirror of the store's non-finite flag

    def _ctx(self, g, it=0):
        return RunContext(store=self.store, graph=g, iteration=it)

    def _run_eager(self, gi: int, it: int = 0, trace: bool = False):
        g = self.seq.graphs[gi]
        return _enqueue(g, self.store, self.registry, self.cap, self._ctx(g, it), trace, None)[1]

    def prepare(self) -> None:
        for g in self.seq.graphs:
            rep = g.validate()
            if not rep.ok:
                raise DispatchError("graph failed validation: " + "; ".join(rep.violations))
            _check_sources(g, self.store)
        lanes_of(self.store)
        for gi in range(len(self.seq.graphs)):  # warm-up: allocates every output buffer
            self._run_eager(gi)
        torch.cuda.synchronize(self.store.device)
        start = _binding(self.store)
        pool = torch.cuda.graph_pool_handle()
        cap_stream = torch.cuda.Stream(device=self.store.device)
        from . import _native

        count = _native.lib().raw("bf_launch_count")
        for par in (0, 1):
            per, times = [], []
            before = count()
            for gi, g in enumerate(self.seq.graphs):
                if self.host_only[gi]:
                    self._run_eager(gi)
                    per.append(None)
                    times.append([])
                    continue
                cg = torch.cuda.CUDAGraph()
                with torch.cuda.graph(cg, pool=pool, stream=cap_stream):
                    times.append(self._run_eager(gi, trace=self.trace))
                per.append(cg)
            self.launches_per_step = count() - before
            self.graphs[par] = per
            self.timing[par] = times
        if _binding(self.store) != start:
            raise DispatchError("graph capture needs a period-2 buffer binding "
                                "(swap graphs must be involutions)")
        self.ready = True

    def op_times_ms(self, parity: int) -> list[tuple[int, object, float]]:
        """(graph index, operator, device ms) of the last replay of ``parity``
        (needs ``trace=True``; call after synchronising)."""
        out = []
        for gi, recs in enumerate(self.timing[parity]):
            g = self.seq.graphs[gi]
            for oid, a, b in recs:
                out.append((gi, g.operators[oid], a.elapsed_time(b)))
        return out

    def op_intervals_ns(self, parity: int) -> list[tuple[int, object, int, int]]:
        """(graph index, operator, start ns, end ns) of the last replay of
        ``parity``, relative to the first operator start of graph 0 (needs
        ``trace=True``; call after synchronising)."""
        base = None
        out = []
        for gi, recs in enumerate(self.timing[parity]):
            g = self.seq.graphs[gi]
            for oid, a, b in recs:
                if base is None:
                    base = a
                s = int(round(base.elapsed_time(a) * 1e6))
                out.append((gi, g.operators[oid], s, s + int(round(a.elapsed_time(b) * 1e6))))
        return out

    def prefetch(self, inputs: dict) -> None:
        """Start copying the NEXT step's source tensors (name -> pinned host
        torch tensor, e.g. the data batch and labels) on a side stream into
        device staging buffers; the following `step()` waits for the copy and
        moves the staged data into the bound tensors with one device-to-device
        copy each.  Issued right after `step()`, the host->device transfer of
        batch i+1 overlaps the compute of batch i (the reference's feeder
        writes the store synchronously before each iteration, builders.py:
        284-365)."""
        dev = self.store.device
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(device=dev)
        cs = self._copy_stream
        # two staging sets: this copy may only overwrite the set whose previous
        # contents were already moved into the bound tensors (event recorded
        # right after those device-to-device copies, not after the whole step)
        slot = self._slot
        self._slot ^= 1
        if self._consumed[slot] is not None:
            cs.wait_event(self._consumed[slot])
        else:
            cs.wait_stream(torch.cuda.current_stream(dev))
        staged = {}
        with torch.cuda.stream(cs):
            for name, src in inputs.items():
                key = (slot, name)
                buf = self._staging.get(key)
                if buf is None or buf.shape != src.shape:
                    buf = torch.empty(src.shape, dtype=torch.float32, device=dev)
                    self._staging[key] = buf
                buf.copy_(src, non_blocking=True)
                staged[name] = buf
            ev = torch.cuda.Event()
            ev.record(cs)
        self._pending = (staged, ev, slot)

    def sync(self) -> None:
        """Wait for every enqueued step and raise `DispatchError` if any of them
        produced a non-finite value (the dispatcher's per-graph device check)."""
        raise_if_nonfinite(self.store, self.seq.graphs, sync=True, cap=self.cap)

    def step(self, after_graph=None, iteration: int = 0) -> None:
        if not self.ready:
            raise DispatchError("CapturedSequence.step() before prepare()")
        # the non-finite flag of earlier steps, copied to pinned memory behind
        # them: read without waiting (a step or two late), located and raised
        # like the reference's per-kernel check once it shows up
        if self._flag_host is not None and int(self._flag_host[0]) != 0:
            self._flag_host.zero_()
            self.sync()
        if self._pending is not None:  # inputs staged by prefetch()
            staged, ev, slot = self._pending
            self._pending = None
            cur = torch.cuda.current_stream(self.store.device)
            cur.wait_event(ev)
            for name, buf in staged.items():
                self.store.get(name).data.copy_(buf.reshape(self.store.get(name).data.shape))
            done = torch.cuda.Event()
            done.record(cur)
            self._consumed[slot] = done
        for gi, cg in enumerate(self.graphs[self.parity]):
            if cg is None:
                self._run_eager(gi, iteration)
            else:
                cg.replay()
            if after_graph is not None:
                after_graph(RunReport(trace=[], elapsed=0, iteration=iteration, graph_index=gi),
                            self.store)
        if self.store.has_finite_flag():
            if self._flag_host is None:
                self._flag_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
            self._flag_host.copy_(self.store.finite_flag(), non_blocking=True)
        self.parity ^= 1


class PrefetchFeed:
    """A ``run_sequence`` ``before_iteration`` hook that overlaps each
    iteration's host->device input copy with the previous iteration's compute.

    ``batches(it)`` returns ``{name: pinned host float32 tensor}`` for
    iteration ``it``.  Iteration ``it``'s copy runs on a side stream into one
    of two device staging sets while iteration ``it - 1`` computes; the hook
    then waits for it on the current stream and writes the staged tensors into
    the store with one device-to-device copy each (`TensorStore.set`, in
    place, so run()'s replay cache keeps its binding).  The reference's feeder
    writes the store synchronously before each iteration (builders.py:284-365);
    this is the same data flow with the transfer off the critical path.
    ``iterations`` (optional) stops the look-ahead after the last iteration."""

    def __init__(self, batches, device, iterations: int | None = None):
        self.batches = batches
        self.device = torch.device(device)
        self.iterations = iterations
        self._cs = None
        self._staging: dict = {}
        self._consumed = [None, None]
        self._pending = None  # (iteration, staged, event, slot)

    def _issue(self, it: int) -> None:
        if self._cs is None:
            self._cs = torch.cuda.Stream(device=self.device)
        slot = it & 1
        if self._consumed[slot] is not None:  # the set's previous contents are in the store
            self._cs.wait_event(self._consumed[slot])
        else:
            self._cs.wait_stream(torch.cuda.current_stream(self.device))
        staged = {}
        with torch.cuda.stream(self._cs):
            for name, src in self.batches(it).items():
                buf = self._staging.get((slot, name))
                if buf is None or buf.shape != src.shape:
                    buf = torch.empty(src.shape, dtype=torch.float32, device=self.device)
                    self._staging[(slot, name)] = buf
                buf.copy_(src, non_blocking=True)
                staged[name] = buf
            ev = torch.cuda.Event()
            ev.record(self._cs)
        self._pending = (it, staged, ev, slot)

    def __call__(self, it: int, store) -> None:
        if self._pending is None or self._pending[0] != it:
            self._issue(it)  # first iteration (or a restart): nothing to overlap with
        _, staged, ev, slot = self._pending
        cur = torch.cuda.current_stream(self.device)
        cur.wait_event(ev)
        for name, buf in staged.items():
            store.set(name, buf)
        done = torch.cuda.Event()
        done.record(cur)
        self._consumed[slot] = done
        if self.iterations is None or it + 1 < self.iterations:
            self._issue(it + 1)
