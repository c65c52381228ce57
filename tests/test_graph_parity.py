"""The product builders emit the reference's graphs exactly, and the product
dispatcher's host order is the reference's serial-mode order."""

import pytest

from paper_1412_6249_b200 import (BiGraph, GraphError, Location, ParallelPlan, build_data_parallel,
                                  build_sgd_iteration, graph_from_json, graph_to_json,
                                  serial_order)
from paper_1412_6249_b200.builders import LayerSpec, NetSpec
from paper_1412_6249_b200.nets import cifar_convnet, conv_relu_fc, googlenet, nin


def _mlp():
    return NetSpec((20,), (LayerSpec("fc", 16), LayerSpec("relu"), LayerSpec("fc", 4)), batch=8,
                   lr=0.05)


def _plan(n):
    return ParallelPlan("data", peers=tuple(Location("local", k) for k in range(n)),
                        server=Location("local", n))


def test_cfg1_graphs_identical_to_reference(golden_graphs):
    seq = build_sgd_iteration(conv_relu_fc())
    ref = golden_graphs["cfg1"]
    assert [graph_to_json(g) for g in seq.graphs] == ref["graphs"]
    for g, order in zip(seq.graphs, ref["serial"]):
        assert [g.operators[o].name for o in serial_order(g)] == order


@pytest.mark.parametrize("split", [False, True])
def test_dp_graphs_identical_to_reference(golden_graphs, split):
    seq = build_data_parallel(_mlp(), _plan(2), split_backward=split)
    ref = golden_graphs[f"mlp_dp2_{'split' if split else 'fused'}"]
    assert [graph_to_json(g) for g in seq.graphs] == ref["graphs"]
    for g, order in zip(seq.graphs, ref["serial"]):
        assert [g.operators[o].name for o in serial_order(g)] == order


def test_json_round_trip_preserves_order():
    seq = build_data_parallel(cifar_convnet(), _plan(2))
    g = seq.graphs[0]
    g2 = graph_from_json(graph_to_json(g))
    assert graph_to_json(g2) == graph_to_json(g)
    assert [g.operators[o].name for o in serial_order(g)] == \
        [g2.operators[o].name for o in serial_order(g2)]


@pytest.mark.parametrize("factory", [googlenet, nin, cifar_convnet])
def test_dag_nets_build_valid_graphs(factory):
    net = factory(batch=2)
    for seq in (build_sgd_iteration(net), build_data_parallel(net, _plan(2))):
        for g in seq.graphs:
            rep = g.validate()
            assert rep.ok, rep.violations
            assert len(serial_order(g)) == len(g.operators)


def test_googlenet_structure():
    seq = build_sgd_iteration(googlenet(batch=2))
    g = seq.graphs[0]
    kinds = [op.kind for op in g.operators.values()]
    assert kinds.count("conv2d_forward") == 57
    assert kinds.count("maxpool_forward") == 13
    assert kinds.count("avgpool_forward") == 1
    assert kinds.count("lrn_forward") == 2
    assert kinds.count("concat_forward") == 9
    assert kinds.count("conv2d_backward_weight") == 57
    assert kinds.count("conv2d_backward_data") == 56  # no data gradient for the image
    assert kinds.count("sgd_update") == 116
    # inception inputs fan out to 4 branches -> summed gradients
    assert kinds.count("aggregate") == 9
    assert len(seq.graphs[1].operators) == 116


def test_graph_invariants_enforced():
    g = BiGraph()
    loc = Location("local", 0)
    a = g.add_tensor("a", (2, 3), loc)
    b = g.add_tensor("b", (2, 3), loc)
    g.add_operator("r", "relu_forward", [a], [b], loc)
    with pytest.raises(GraphError):
        g.add_operator("r2", "relu_forward", [a], [b], loc)  # second producer
    with pytest.raises(GraphError):
        g.add_operator("r3", "relu_forward", [b], [a], loc)  # cycle
    c = g.add_tensor("c", (2, 3), Location("local", 1))
    with pytest.raises(GraphError):
        g.add_operator("r4", "relu_forward", [b], [c], loc)  # only copy crosses
    g.add_operator("cp", "copy", [b], [c], loc, thread=1)
    d = g.add_tensor("d", (3, 3), loc)
    with pytest.raises(GraphError):
        g.add_operator("bad", "relu_forward", [a], [d], loc)  # shape rule
