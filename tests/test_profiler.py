"""Profiler interval arithmetic against the reference's frozen cases
(`pkg/tests/test_profiler.py:33-219`): overlap fraction, iteration gaps,
Chrome-trace export with its microsecond rounding -- and the exposed-comm
figure the bench derives from the same unions."""

import json

import pytest

from paper_1412_6249_b200.dispatcher import TraceRecord, WorkerLane
from paper_1412_6249_b200.profiler import (COMPUTE, COPY, TRANSPORT, LaneClass, exposed_fraction,
                                           exposed_ns, export_trace, iteration_gap,
                                           overlap_fraction)

CPU = WorkerLane("local", 0, 0)
MOVER = WorkerLane("local", 0, 1)
WIRE = WorkerLane("local", 0, 2)
CLASSES = {CPU: COMPUTE, MOVER: COPY, WIRE: TRANSPORT}


def rec(name, lane, start, end, iteration=0):
    return TraceRecord(op=0, name=name, lane=lane, start=start, end=end, iteration=iteration)


@pytest.mark.parametrize("trace,want", [
    ([rec("c", CPU, 0, 100), rec("m", MOVER, 10, 20)], 1.0),          # copy inside compute
    ([rec("c", CPU, 0, 50), rec("m", MOVER, 100, 110)], 0.0),         # disjoint
    ([rec("c", CPU, 5, 30), rec("m", MOVER, 0, 10)], 0.5),            # intersection ratio
    ([rec("c1", CPU, 0, 3), rec("c2", CPU, 8, 20), rec("m", MOVER, 0, 10)], 0.5),
    ([rec("c1", CPU, 0, 4), rec("c2", CPU, 0, 4), rec("m", MOVER, 0, 10)], 0.4),  # union
    ([rec("w", WIRE, 0, 100), rec("m", MOVER, 10, 20)], 0.0),         # transport != compute
])
def test_overlap_fraction_cases(trace, want):
    assert overlap_fraction(trace, CLASSES) == want


def test_overlap_invariant_under_translation_and_splitting():
    base = [rec("c", CPU, 5, 30), rec("m", MOVER, 0, 10)]
    split = [rec("c1", CPU, 5, 17), rec("c2", CPU, 17, 30), rec("m", MOVER, 0, 10)]
    shifted = [rec(r.name, r.lane, r.start + 10**6, r.end + 10**6) for r in base]
    want = overlap_fraction(base, CLASSES)
    assert overlap_fraction(split, CLASSES) == want == overlap_fraction(shifted, CLASSES)


def test_overlap_monotone_in_compute():
    trace = [rec("m", MOVER, 0, 100)]
    prev = 0.0
    for i, (s, e) in enumerate([(0, 10), (50, 60), (5, 55), (90, 200)]):
        trace.append(rec(f"c{i}", CPU, s, e))
        cur = overlap_fraction(trace, CLASSES)
        assert 0.0 <= prev <= cur <= 1.0
        prev = cur


def test_overlap_errors():
    with pytest.raises(ValueError):  # no copy records
        overlap_fraction([rec("c", CPU, 0, 10)], CLASSES)
    with pytest.raises(ValueError):  # classification must be total
        overlap_fraction([rec("x", WorkerLane("elsewhere", 0, 0), 0, 5), rec("m", MOVER, 0, 5)],
                         CLASSES)
    with pytest.raises(ValueError):  # unknown class
        overlap_fraction([rec("m", MOVER, 0, 5)], LaneClass(lambda lane: "banana"))
    by_thread = LaneClass.of(lambda ln: COPY if ln.thread == 1 else COMPUTE)
    assert overlap_fraction([rec("c", CPU, 0, 10), rec("m", MOVER, 2, 4)], by_thread) == 1.0


@pytest.mark.parametrize("trace,want", [
    ([rec("c", CPU, 0, 100, 0), rec("c", CPU, 107, 200, 1), rec("c", CPU, 230, 300, 2)], [7, 30]),
    ([rec("c", CPU, 0, 100, 0), rec("c", CPU, 100, 180, 1)], [0]),
    ([rec("c", CPU, 0, 100, 0), rec("m", MOVER, 90, 140, 0), rec("w", WIRE, 100, 150, 1),
      rec("c", CPU, 150, 220, 1)], [50]),                              # copies ignored
    ([rec("c1", CPU, 0, 40, 0), rec("c2", CPU, 10, 90, 0), rec("c1", CPU, 95, 130, 1),
      rec("c2", CPU, 97, 160, 1)], [5]),                               # extreme records
])
def test_iteration_gap_cases(trace, want):
    assert iteration_gap(trace, CLASSES) == want


def test_iteration_gap_needs_two_iterations():
    with pytest.raises(ValueError):
        iteration_gap([rec("c", CPU, 0, 10, iteration=0)], CLASSES)


def test_export_golden_single_record(tmp_path):
    path = tmp_path / "trace.json"
    export_trace([rec("fc1", CPU, 0, 1500)], path)
    assert json.loads(path.read_text()) == [
        {"name": "fc1", "ph": "X", "ts": 0, "dur": 1, "pid": 0, "tid": 0, "args": {"iteration": 0}}]
    export_trace([], path)
    assert json.loads(path.read_text()) == []


def test_export_microsecond_rounding(tmp_path):
    path = tmp_path / "trace.json"
    for ns, us in {499: 0, 500: 0, 501: 1, 1499: 1, 1500: 1, 1501: 2, 2500: 2}.items():
        assert export_trace([rec("op", CPU, 0, ns)], path)[0]["dur"] == us, ns
    ev = export_trace([rec("op", CPU, 700, 2200)], path)[0]  # ts and dur round independently
    assert ev["ts"] == 1 and ev["dur"] == 1


def test_export_pid_per_host_tid_per_lane(tmp_path):
    trace = [rec("a", WorkerLane("h1", 0, 0), 0, 1000), rec("b", WorkerLane("h0", 1, 2), 1000, 2000),
             rec("c", WorkerLane("h0", 0, 5), 2000, 3000), rec("d", WorkerLane("h0", 1, 2), 3000, 4000)]
    by = {e["name"]: e for e in export_trace(trace, tmp_path / "t.json")}
    assert (by["a"]["pid"], by["b"]["pid"]) == (1, 0)
    assert (by["c"]["tid"], by["b"]["tid"], by["d"]["tid"]) == (0, 1, 1)


def test_export_round_trip_sorted(tmp_path):
    trace = [rec(f"op{i}", CPU, 1000 * (10 - i), 1000 * (10 - i) + 500) for i in range(10)]
    path = tmp_path / "t.json"
    events = export_trace(trace, path)
    parsed = json.loads(path.read_text())
    assert parsed == events and len(parsed) == 10
    assert [e["ts"] for e in parsed] == sorted(e["ts"] for e in parsed)


@pytest.mark.parametrize("comm,compute,want", [
    ([(0, 10)], [(0, 100)], 0),
    ([(0, 10)], [], 10),
    ([(0, 10)], [(5, 30)], 5),
    ([(0, 10), (5, 20)], [(8, 12)], 16),            # comm union [0,20) minus [8,12)
    ([(0, 100)], [(10, 20), (30, 40), (15, 35)], 70),
    ([(50, 60)], [(0, 10), (70, 80)], 10),
    ([], [(0, 10)], 0),
])
def test_exposed_ns_cases(comm, compute, want):
    assert exposed_ns(comm, compute) == want


def test_exposed_fraction_over_iteration_span():
    trace = [rec("c", CPU, 0, 80), rec("m", MOVER, 70, 100)]
    assert exposed_fraction(trace, CLASSES) == pytest.approx(20 / 100)
    assert exposed_fraction(trace, CLASSES, iteration_ns=200) == pytest.approx(0.1)
