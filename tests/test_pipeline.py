"""Model-parallel pipeline (reference builders.py:650-785,
tests test_builders.py:266-367 and acceptance criterion 8).

CPU: the product builder emits the reference's graphs exactly (golden JSON +
serial dispatch order from tests/golden/make_pipeline_golden.py), the oracle
running them reproduces the reference's outputs bit for bit, and the
virtual-time simulator gives the staircase makespan (S + R - 1) x stage cost.
GPU: the same graphs through the CUDA-stream dispatcher (one lane per stage
location, gates and boundary copies on the copy lanes) match the reference
outputs within the NS tolerance and the unpipelined GPU chain bit for bit.
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1412_6249_b200 import (GraphError, Location, ParallelPlan, Stage,
                                  build_model_parallel_pipeline, fill_tokens, graph_to_json,
                                  serial_order)
from paper_1412_6249_b200.builders import LayerSpec, NetSpec
from paper_1412_6249_b200.costsim import CostModel, simulate

CASES = {
    "mlp3x3": (NetSpec((8,), (LayerSpec("fc", 8), LayerSpec("fc", 8), LayerSpec("fc", 4)),
                       batch=4), ((0, 1), (1, 2), (2, 3)), 3, 21),
    "conv2x4": (NetSpec((3, 32, 32), (LayerSpec("conv", 32, 5, 1, 2), LayerSpec("relu"),
                                      LayerSpec("fc", 10)), batch=16, lr=1e-3),
                ((0, 2), (2, 3)), 4, 7),
}


@pytest.fixture(scope="module")
def golden():
    return (json.loads((GOLDEN / "pipeline.json").read_text()),
            dict(np.load(GOLDEN / "pipeline.npz")))


def _build(tag):
    net, spans, replicas, seed = CASES[tag]
    plan = ParallelPlan("model", stages=tuple(Stage(s, Location("local", k))
                                              for k, s in enumerate(spans)),
                        replicas=replicas)
    return net, build_model_parallel_pipeline(net, plan), seed


@pytest.mark.parametrize("tag", sorted(CASES))
def test_pipeline_graph_identical_to_reference(golden, tag):
    _net, seq, _seed = _build(tag)
    ref = golden[0][tag]
    assert [graph_to_json(g) for g in seq.graphs] == ref["graphs"]
    for g, order in zip(seq.graphs, ref["serial"]):
        assert [g.operators[o].name for o in serial_order(g)] == order
    lay = seq.layout
    assert list(lay.data_names) == ref["layout"]["data"]
    assert list(lay.token_names) == ref["layout"]["tokens"]
    assert list(lay.output_names) == ref["layout"]["outputs"]
    assert list(lay.canonical_params) == ref["layout"]["params"]
    assert seq.graphs[0].validate().ok


@pytest.mark.parametrize("tag", sorted(CASES))
def test_pipeline_oracle_matches_reference_outputs_bitwise(golden, tag):
    from oracle.serial import run_graph_serial

    net, seq, _seed = _build(tag)
    arrs = golden[1]
    store = {n: arrs[f"{tag}_{n}"] for n in seq.layout.canonical_params}
    for r, n in enumerate(seq.layout.data_names):
        store[n] = arrs[f"{tag}_x_r{r}"]

    class _S(dict):
        def set(self, name, arr):
            self[name] = arr

    tokens = _S()
    fill_tokens(tokens, seq)
    store.update(tokens)
    run_graph_serial(seq.graphs[0], store)
    for n in seq.layout.output_names:
        assert np.array_equal(store[n], arrs[f"{tag}_{n}"]), n


@pytest.mark.parametrize("tag", sorted(CASES))
def test_pipeline_staircase_makespan(golden, tag):
    """Unit cost per compute op: (S + R - 1) x (ops per stage), the
    reference simulator's own number."""
    _net, seq, _seed = _build(tag)
    for op in seq.graphs[0].operators.values():
        if op.kind not in ("copy", "gate"):
            op.attrs["delay_s"] = 1.0
    rep = simulate(seq, CostModel(kind_costs={}))
    assert rep.makespan == golden[0][tag]["unit_cost_makespan"]


def test_pipeline_gates_serialise_each_stage_across_replicas():
    _net, seq, _seed = _build("mlp3x3")
    for op in seq.graphs[0].operators.values():
        if op.kind == "fc_forward":
            op.attrs["delay_s"] = 1.0
    rep = simulate(seq, CostModel(kind_costs={}))
    win = {r.name: (r.start, r.end) for r in rep.trace if r.name.startswith("fc")}
    for pos in (1, 2, 3):
        for r in (1, 2):
            assert win[f"fc{pos}_r{r}"][0] >= win[f"fc{pos}_r{r - 1}"][1]


def test_pipeline_rejects_bad_stage_plans():
    net = CASES["mlp3x3"][0]
    L = Location("local", 0)
    for spans in (((0, 1), (2, 3)), ((1, 3),), ((0, 2),), ((0, 0), (0, 3))):
        plan = ParallelPlan("model", stages=tuple(Stage(s, L) for s in spans), replicas=2)
        with pytest.raises(GraphError):
            build_model_parallel_pipeline(net, plan)
    with pytest.raises(GraphError):
        build_model_parallel_pipeline(net, ParallelPlan("data", peers=(L,), server=L))


# ---------------------------------------------------------------------------
# GPU: the CUDA-stream dispatcher and the sm_100a kernels


def _gpu_run(seq, net, inputs, params):
    from paper_1412_6249_b200 import TensorStore, run_sequence

    store = TensorStore("cuda:0")
    for n, a in params.items():
        store.set(n, a)
    fill_tokens(store, seq)
    for n, a in zip(seq.layout.data_names, inputs):
        store.set(n, a)
    run_sequence(seq, store)
    return store


@pytest.mark.gpu
@pytest.mark.parametrize("tag", sorted(CASES))
def test_pipeline_gpu_matches_reference(golden, tag):
    from gpu_util import ATOL, RTOL, assert_close

    net, seq, _seed = _build(tag)
    arrs = golden[1]
    params = {n: arrs[f"{tag}_{n}"] for n in seq.layout.canonical_params}
    xs = [arrs[f"{tag}_x_r{r}"] for r in range(len(seq.layout.data_names))]
    store = _gpu_run(seq, net, xs, params)
    for n in seq.layout.output_names:
        want = arrs[f"{tag}_{n}"]
        assert_close(store.array(n), want, RTOL, ATOL * max(1.0, float(np.abs(want).max())), n)

    # the unpipelined chain (one stage, one replica) on the same kernels: bitwise
    one = ParallelPlan("model", stages=(Stage((0, len(net.layers)), Location("local", 0)),),
                       replicas=1)
    flat = build_model_parallel_pipeline(net, one)
    for r, n in enumerate(seq.layout.output_names):
        s1 = _gpu_run(flat, net, [xs[r]], params)
        assert np.array_equal(store.array(n), s1.array(flat.layout.output_names[0])), n
