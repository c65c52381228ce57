"""Cost simulator (costsim.py): the reference's schedule semantics, pinned
against schedules the reference simulator produced (golden/costsim.json),
and the B200 calibration helpers."""

import json
import math
from pathlib import Path

import pytest

from paper_1412_6249_b200 import BiGraph, GraphSequence, Location, graph_from_json
from paper_1412_6249_b200.costsim import (CostModel, SimError, exchange_cost, fit_two_point,
                                          measured_costs, predict_scaling, simulate,
                                          throughput_model)

GOLDEN = Path(__file__).resolve().parent / "golden"
LOC = Location("local", 0)


def chain(costs, threads=None, shape=(4,)):
    """t0 -> copy -> t1 -> copy -> ... with delay_s costs on given threads."""
    g = BiGraph()
    prev = g.add_tensor("t0", shape, LOC)
    for i, c in enumerate(costs):
        nxt = g.add_tensor(f"t{i + 1}", shape, LOC)
        g.add_operator(f"op{i}", "copy", [prev], [nxt], LOC,
                       thread=(threads[i] if threads else 0), attrs={"delay_s": c})
        prev = nxt
    return g


def test_matches_reference_schedules():
    """Makespan, start/end of every operator and iteration tags equal the
    reference simulator's on the reference-built graphs (2 iterations)."""
    gold = json.loads((GOLDEN / "costsim.json").read_text())
    graphs = json.loads((GOLDEN / "graphs.json").read_text())
    model = CostModel(kind_costs={k: v * 1e-6 for k, v in gold["kind_cost_us"].items()},
                      bandwidth=gold["bandwidth"], latency=gold["latency"])
    for tag, case in gold["cases"].items():
        seq = GraphSequence([graph_from_json(g) for g in graphs[tag]["graphs"]], iterations=2)
        rep = simulate(seq, model, images_per_iteration=16)
        assert rep.makespan == pytest.approx(case["makespan"], rel=1e-12), tag
        assert rep.throughput == pytest.approx(case["throughput"], rel=1e-12), tag
        got = [[r.name, r.lane.thread, r.start, r.end, r.iteration] for r in rep.trace]
        assert got == case["trace"], tag


def test_single_lane_chain_is_the_sum():
    rep = simulate(chain([1.0, 2.0, 0.5]), CostModel())
    assert rep.makespan == pytest.approx(3.5)
    assert [r.name for r in rep.trace] == ["op0", "op1", "op2"]


def test_independent_lanes_overlap_and_shared_lane_serialises():
    g = BiGraph()
    src = g.add_tensor("x", (4,), LOC)
    a, b = g.add_tensor("a", (4,), LOC), g.add_tensor("b", (4,), LOC)
    g.add_operator("left", "copy", [src], [a], LOC, thread=1, attrs={"delay_s": 2.0})
    g.add_operator("right", "copy", [src], [b], LOC, thread=2, attrs={"delay_s": 3.0})
    assert simulate(g, CostModel()).makespan == pytest.approx(3.0)
    g2 = BiGraph()
    src = g2.add_tensor("x", (4,), LOC)
    a, b = g2.add_tensor("a", (4,), LOC), g2.add_tensor("b", (4,), LOC)
    g2.add_operator("left", "copy", [src], [a], LOC, thread=1, attrs={"delay_s": 2.0})
    g2.add_operator("right", "copy", [src], [b], LOC, thread=1, attrs={"delay_s": 3.0})
    rep = simulate(g2, CostModel())
    assert rep.makespan == pytest.approx(5.0)
    assert [r.name for r in rep.trace] == ["left", "right"]  # insertion order breaks ties


def test_sequence_graphs_start_after_the_previous_and_iterate():
    seq = GraphSequence([chain([1.0]), chain([2.0])], iterations=3)
    rep = simulate(seq, CostModel())
    assert rep.makespan == pytest.approx(9.0)
    assert [r.iteration for r in rep.trace] == [0, 0, 1, 1, 2, 2]


def test_deterministic():
    g = chain([0.1, 0.2, 0.3], threads=[0, 1, 0])
    assert simulate(g, CostModel()).trace == simulate(g, CostModel()).trace


def test_costs_by_kind_name_and_transfer_model():
    g = chain([0.0])  # delay 0 still wins over every table
    assert simulate(g, CostModel(kind_costs={"copy": 5.0})).makespan == 0.0
    g = BiGraph()
    x, y = g.add_tensor("x", (1000,), LOC), g.add_tensor("y", (1000,), LOC)
    g.add_operator("mv", "copy", [x], [y], LOC)
    assert simulate(g, CostModel(bandwidth=4000.0, latency=0.5)).makespan == pytest.approx(1.5)
    assert simulate(g, CostModel(op_costs={"mv": 7.0})).makespan == pytest.approx(7.0)
    assert simulate(g, CostModel(kind_costs={"copy": lambda i, o: len(i) + 1})).makespan == 2.0


def test_errors():
    g = BiGraph()
    x, y = g.add_tensor("x", (4,), LOC), g.add_tensor("y", (4,), LOC)
    g.add_operator("r", "relu_forward", [x], [y], LOC)
    with pytest.raises(SimError, match="no cost entry"):
        simulate(g, CostModel())
    with pytest.raises(SimError):
        CostModel(bandwidth=0)
    with pytest.raises(SimError):
        CostModel(latency=-1)
    with pytest.raises(SimError):
        throughput_model(0, 1, 1.0, 0.0)


def test_throughput_model_and_fit_round_trip():
    a, c = 2e-3, 0.05
    table = [(b, throughput_model(8, b, a, c)) for b in (16, 32, 64, 128)]
    fit = fit_two_point(table, 8)
    assert fit.a == pytest.approx(a) and fit.c == pytest.approx(c)
    assert all(abs(r) < 1e-12 for r in fit.residuals.values())
    assert throughput_model(4, 32, a, 0.0) == pytest.approx(4 * 32 / (a * 32))
    with pytest.raises(SimError):
        fit_two_point([(32, 100.0)], 1)


def test_exchange_cost_model():
    assert exchange_cost(1 << 20, 1) < exchange_cost(1 << 20, 2) < exchange_cost(1 << 20, 8)
    per_byte = exchange_cost(2 << 30, 8) / (2 << 30)
    assert per_byte == pytest.approx((2 * 7 / 8) / 700e9 + 3 / 8 / 5000e9, rel=1e-3)


def test_measured_costs_and_scaling_prediction(tmp_path):
    """A measured op table drives the exchange-lowered rank sequence: world 1
    = the compute sum plus the local update, larger worlds add overlapped
    exchanges (efficiency <= 1, exposed fraction in [0, 1))."""
    from paper_1412_6249_b200.exchange import lower_data_parallel, plan_buckets
    from paper_1412_6249_b200.builders import ParallelPlan, build_data_parallel, param_names
    from paper_1412_6249_b200.nets import cifar_convnet

    net = cifar_convnet(batch=16)
    plan = ParallelPlan("data", peers=(Location("local", 0),), server=Location("local", 1))
    seq = lower_data_parallel(build_data_parallel(net, plan), 0, plan_buckets(param_names(net), 1,
                                                                               4 << 20), net)
    path = tmp_path / "ops.tsv"
    with open(path, "w") as f:
        f.write("op\tkind\tms\tgflop\tmbytes\n")
        for op in seq.graphs[0].operators.values():
            if op.kind not in ("dp_exchange", "swap"):
                f.write(f"{op.name}\t{op.kind}\t0.05\t0\t0\n")
    times = measured_costs(path)
    pts = predict_scaling(net, [1, 2, 4, 8], times)
    assert [p.world for p in pts] == [1, 2, 4, 8]
    assert pts[0].efficiency == pytest.approx(1.0)
    for p in pts:
        assert 0 < p.efficiency <= 1.0 + 1e-9 and 0 <= p.exposed_comm < 1
        assert p.images_per_s == pytest.approx(p.world * 16 / p.iteration_s)
    assert math.isfinite(pts[-1].iteration_s)
