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
