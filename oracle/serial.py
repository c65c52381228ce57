"""Serial-mode graph execution on the CPU (TEST INFRASTRUCTURE ONLY).

Restates the reference dispatcher's readiness bookkeeping
(`pkg/src/biflow/dispatcher.py:96-206`) in its fully serial mode
(one worker, `BIFLOW_LANES=1`, `dispatcher.py:261-267`): the initially
ready operators in graph-insertion order, then a single FIFO queue to which
each completion appends its newly ready operators sorted by insertion
index.  That order is the dispatch-order contract.

The graph argument is duck-typed: anything with ``operators`` (id -> op with
``name, kind, inputs, outputs, attrs``), ``tensors`` (id -> t with ``name``)
and ``insertion_order`` works, so both the reference's BiGraph and the
product package's BiGraph can be checked.
"""

from __future__ import annotations

from collections import deque

import numpy as np

from .kernels import KERNELS, OracleError


def _consumers(graph):
    cons = {tid: [] for tid in graph.tensors}
    for oid in graph.insertion_order:
        for tid in graph.operators[oid].inputs:
            cons[tid].append(oid)
    return cons


def serial_order(graph) -> list[int]:
    """Operator ids in reference serial-mode dispatch order."""
    rank = {oid: i for i, oid in enumerate(graph.insertion_order)}
    cons = _consumers(graph)
    produced = set()
    for op in graph.operators.values():
        produced.update(op.outputs)
    waiting = {oid: len(op.inputs) for oid, op in graph.operators.items()}

    def release(tid, out):
        for oid in cons[tid]:
            waiting[oid] -= 1
            if waiting[oid] == 0:
                out.append(oid)

    first = [oid for oid in graph.insertion_order if waiting[oid] == 0]
    for tid in sorted(graph.tensors):
        if tid not in produced:
            release(tid, first)
    queue = deque(sorted(dict.fromkeys(first), key=rank.__getitem__))
    order = []
    while queue:
        oid = queue.popleft()
        order.append(oid)
        fresh = []
        for tid in graph.operators[oid].outputs:
            release(tid, fresh)
        queue.extend(sorted(fresh, key=rank.__getitem__))
    if len(order) != len(graph.operators):
        raise OracleError("graph cannot complete: some operators never become ready")
    return order


def run_graph_serial(graph, store: dict, kernels=None) -> list[str]:
    """Execute one graph over a name -> ndarray dict; returns op names in order."""
    kernels = KERNELS if kernels is None else kernels
    names = []
    for oid in serial_order(graph):
        op = graph.operators[oid]
        ins = [graph.tensors[t].name for t in op.inputs]
        outs = [graph.tensors[t].name for t in op.outputs]
        if op.kind == "swap":
            a, b = outs
            store[a], store[b] = store[b], store[a]
        elif op.kind == "copy":
            store[outs[0]] = np.array(store[ins[0]], dtype=np.float32, copy=True)
        else:
            fn = kernels.get(op.kind)
            if fn is None:
                raise OracleError(f"oracle has no kernel for kind {op.kind!r}")
            results = fn([store[n] for n in ins], dict(op.attrs))
            for name, arr in zip(outs, results):
                store[name] = np.ascontiguousarray(arr, dtype=np.float32)
        names.append(op.name)
    return names


def run_sequence_serial(graphs, store: dict, iterations: int, before_iteration=None,
                        kernels=None) -> list[list[str]]:
    """Iterate a graph sequence serially; returns per-graph op-name orders."""
    orders = []
    for it in range(iterations):
        if before_iteration is not None:
            before_iteration(it, store)
        for g in graphs:
            orders.append(run_graph_serial(g, store, kernels))
    return orders


def _lane(op) -> tuple:
    loc = op.location
    return (loc.host, loc.device, int(getattr(op, "thread", 0) or 0))


def run_graph_lanes(graph, store: dict, kernels=None) -> list[str]:
    """Multi-worker mode of the reference dispatcher (dispatcher.py:209-375):
    one worker thread per lane ``(host, device, thread)``, each taking its
    lane's ready operators in FIFO order; a completion releases its consumers
    into their lanes' queues.  numpy releases the GIL inside its kernels, so
    replicas on different lanes run concurrently -- the reference's
    data-parallel CPU execution, used as the bench's CPU baseline.  Returns the
    completion order (not a contract: lanes interleave)."""
    import threading

    kernels = KERNELS if kernels is None else kernels
    rank = {oid: i for i, oid in enumerate(graph.insertion_order)}
    cons = _consumers(graph)
    produced = set()
    for op in graph.operators.values():
        produced.update(op.outputs)
    waiting = {oid: len(op.inputs) for oid, op in graph.operators.items()}
    for tid in graph.tensors:
        if tid not in produced:
            for oid in cons[tid]:
                waiting[oid] -= 1
    lanes = sorted({_lane(op) for op in graph.operators.values()})
    queues = {ln: deque() for ln in lanes}
    cv = threading.Condition()
    for oid in sorted((o for o, w in waiting.items() if w == 0), key=rank.__getitem__):
        queues[_lane(graph.operators[oid])].append(oid)
    done: list[str] = []
    errors: list[BaseException] = []
    remaining = [len(graph.operators)]

    def execute(oid):
        op = graph.operators[oid]
        ins = [graph.tensors[t].name for t in op.inputs]
        outs = [graph.tensors[t].name for t in op.outputs]
        if op.kind == "swap":
            a, b = outs
            store[a], store[b] = store[b], store[a]
        elif op.kind == "copy":
            store[outs[0]] = np.array(store[ins[0]], dtype=np.float32, copy=True)
        else:
            fn = kernels.get(op.kind)
            if fn is None:
                raise OracleError(f"oracle has no kernel for kind {op.kind!r}")
            results = fn([store[n] for n in ins], dict(op.attrs))
            for name, arr in zip(outs, results):
                store[name] = np.ascontiguousarray(arr, dtype=np.float32)

    def worker(ln):
        q = queues[ln]
        while True:
            with cv:
                while not q and remaining[0] > 0 and not errors:
                    cv.wait()
                if errors or remaining[0] == 0:
                    return
                oid = q.popleft()
            try:
                execute(oid)
            except BaseException as exc:  # noqa: BLE001 - first error wins
                with cv:
                    errors.append(exc)
                    cv.notify_all()
                return
            with cv:
                done.append(graph.operators[oid].name)
                remaining[0] -= 1
                fresh = []
                for tid in graph.operators[oid].outputs:
                    for c in cons[tid]:
                        waiting[c] -= 1
                        if waiting[c] == 0:
                            fresh.append(c)
                for c in sorted(fresh, key=rank.__getitem__):
                    queues[_lane(graph.operators[c])].append(c)
                cv.notify_all()

    threads = [threading.Thread(target=worker, args=(ln,), daemon=True) for ln in lanes]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    if remaining[0]:
        raise OracleError("graph cannot complete: some operators never become ready")
    return done
