"""Scheduler soundness on the CUDA-stream dispatcher, checked on its CUDA-event
traces (the reference's C1 and first-error-wins tests re-pointed at
device timestamps).

* C1 (ref `pkg/tests/test_acceptance.py:84-169`, `test_dispatcher.py:206-261`):
  over random acyclic bi-graphs every operator runs exactly once, no operator
  starts before the producers of its inputs ended (device timestamps), every
  sink tensor is produced, and -- with one stream per lane
  (``PURINE_B200_BRANCH_STREAMS=1``) -- a lane's intervals never overlap.  With
  branch streams a compute lane spreads over several streams by design, so
  only exactly-once and causality are required there.
* first error wins (ref `test_dispatcher.py:166-198`): a failing operator is
  reported by name and the operators queued behind it are not reported as
  failures.

The random graphs use one device (the GPU box has one), copies between lanes
of that device, and device-side sleeps for the ``delay_s`` attribute (scaled
to <= 0.5 ms to keep the suite short).
"""

import random
from collections import defaultdict

import numpy as np
import pytest

from paper_1412_6249_b200 import BiGraph, DispatchError, Location, TensorStore, run

pytestmark = pytest.mark.gpu

LOC = Location("local", 0)


def random_bigraph(rng):
    g = BiGraph()
    target = int(rng.integers(10, 51))
    tensors = [g.add_tensor(f"t{i}", (4,), LOC) for i in range(int(rng.integers(1, 4)))]
    n_vertices, n_ops = len(tensors), 0
    while n_vertices + 2 <= target:
        attrs = {}
        if rng.random() < 0.25:
            attrs["delay_s"] = float(rng.uniform(0.0, 0.0005))
        thread = int(rng.integers(0, 3))
        src = tensors[int(rng.integers(len(tensors)))]
        out = g.add_tensor(f"t{len(tensors)}", (4,), LOC)
        if rng.random() < 0.2:
            g.add_operator(f"op{n_ops}", "copy", [src], [out], LOC, thread=thread, attrs=attrs)
        else:
            k = min(len(tensors), int(rng.integers(1, 4)))
            ins = [int(t) for t in rng.choice(tensors, size=k, replace=False)]
            kind = "relu_forward" if k == 1 else "aggregate"
            g.add_operator(f"op{n_ops}", kind, ins, [out], LOC, thread=thread, attrs=attrs)
        tensors.append(out)
        n_vertices += 2
        n_ops += 1
    return g


def check_schedule(g, rng, lane_exclusive: bool, workers=None):
    store = TensorStore("cuda:0")
    producer = {tid: oid for oid, op in g.operators.items() for tid in op.outputs}
    for tid, t in g.tensors.items():
        if tid not in producer:
            store.set(t.name, rng.standard_normal(t.shape).astype(np.float32))
    trace = run(g, store, max_workers=workers).trace
    executed = [rec.op for rec in trace]
    assert len(executed) == len(g.operators), "some operator never ran"
    assert len(set(executed)) == len(executed), "some operator ran twice"
    start = {rec.op: rec.start for rec in trace}
    end = {rec.op: rec.end for rec in trace}
    for oid, op in g.operators.items():
        for tid in op.inputs:
            if tid in producer:
                assert start[oid] >= end[producer[tid]], \
                    f"{op.name} started before its input was produced"
    if lane_exclusive:
        by_lane = defaultdict(list)
        for rec in trace:
            by_lane[rec.lane].append((rec.start, rec.end))
        for lane, spans in by_lane.items():
            spans.sort()
            for (_, e1), (s2, _) in zip(spans, spans[1:]):
                assert s2 >= e1, f"two operators overlapped on lane {lane}"
    for t in g.tensors.values():
        assert t.name in store, f"sink tensor {t.name} never produced"


@pytest.mark.parametrize("branches", ["1", "8"])
def test_c1_scheduling_soundness(monkeypatch, branches):
    monkeypatch.setenv("PURINE_B200_BRANCH_STREAMS", branches)
    rng = np.random.default_rng(2024)
    for i in range(150):
        g = random_bigraph(rng)
        check_schedule(g, rng, lane_exclusive=branches == "1",
                       workers=None if i % 3 else (1 if i % 2 else 4))


def random_dag(rng):
    g = BiGraph()
    avail = [g.add_tensor(f"src{i}", (4, 4), LOC) for i in range(2)]
    for i in range(rng.randrange(4, 9)):
        thread = rng.randrange(3)
        delay = rng.choice([0.0, 0.0, 0.0001, 0.0002])
        attrs = {"delay_s": delay} if delay else {}
        if rng.random() < 0.5 and len(avail) >= 2:
            ins, kind = rng.sample(avail, 2), "relu_backward"
        else:
            ins, kind = [rng.choice(avail)], "relu_forward"
        out = g.add_tensor(f"t{i}", (4, 4), LOC)
        g.add_operator(f"op{i}", kind, ins, [out], LOC, thread=thread, attrs=attrs)
        avail.append(out)
    return g


def test_random_dags_hold_invariants_and_values(monkeypatch):
    """ref test_dispatcher.py:206-261, plus: the results equal the oracle's."""
    from oracle.serial import run_graph_serial

    monkeypatch.setenv("PURINE_B200_BRANCH_STREAMS", "1")
    rng = random.Random(1234)
    for trial in range(12):
        g = random_dag(rng)
        arr = np.random.default_rng(trial).standard_normal((4, 4)).astype(np.float32)
        for workers in (1, 4):
            store = TensorStore("cuda:0")
            store.set("src0", arr)
            store.set("src1", -arr)
            rep = run(g, store, max_workers=workers)
            assert sorted(r.name for r in rep.trace) == sorted(op.name for op in
                                                                g.operators.values())
            by_op = {r.op: r for r in rep.trace}
            for op in g.operators.values():
                for tid in op.inputs:
                    pid = g.producer_of(tid)
                    if pid is not None:
                        assert by_op[op.id].start >= by_op[pid].end
            lanes = defaultdict(list)
            for r in rep.trace:
                lanes[r.lane].append(r)
            for recs in lanes.values():
                recs.sort(key=lambda r: r.start)
                for a, b in zip(recs, recs[1:]):
                    assert a.end <= b.start
            ref = {"src0": arr, "src1": -arr}
            run_graph_serial(g, ref)
            for t in g.tensors.values():
                assert np.array_equal(store.array(t.name), ref[t.name]), t.name


def _xent_graph(tail: int):
    g = BiGraph()
    logits = g.add_tensor("logits", (2, 3), LOC)
    labels = g.add_tensor("labels", (2,), LOC)
    loss = g.add_tensor("loss", (1,), LOC)
    dl = g.add_tensor("dlogits", (2, 3), LOC)
    g.add_operator("bad", "softmax_xent", [logits, labels], [loss, dl], LOC, thread=0)
    prev = dl
    for i in range(tail):
        nxt = g.add_tensor(f"t{i}", (2, 3), LOC)
        g.add_operator(f"tail{i}", "relu_forward", [prev], [nxt], LOC, thread=0)
        prev = nxt
    return g


@pytest.mark.parametrize("tail", [0, 6])
def test_bad_label_is_reported_first_error_wins(tail):
    """ref test_dispatcher.py:166-198: the failing operator is named; the
    tail queued behind it is not blamed."""
    store = TensorStore("cuda:0")
    store.set("logits", np.zeros((2, 3), dtype=np.float32))
    store.set("labels", np.array([0.0, 9.0], dtype=np.float32))
    with pytest.raises(DispatchError) as ei:
        run(_xent_graph(tail), store)
    assert str(ei.value) == ("operator 'bad' failed: softmax_xent: labels must be integral "
                             "and in [0, 3)")


def test_unknown_kind_is_reported_before_launch():
    g = BiGraph()
    a = g.add_tensor("a", (4,), LOC)
    b = g.add_tensor("b", (4,), LOC)
    c = g.add_tensor("c", (4,), LOC)
    g.add_operator("ok", "copy", [a], [b], LOC)
    g.add_operator("mystery", "relu_forward", [b], [c], LOC)
    store = TensorStore("cuda:0")
    store.set("a", np.ones(4, np.float32))
    from paper_1412_6249_b200 import KINDS

    reg = {k: v for k, v in KINDS.items() if k != "relu_forward"}
    with pytest.raises(DispatchError, match="unknown to registry"):
        run(g, store, registry=reg)
