"""The dispatcher's static fusion plan (_Plan) on CPU: which operators become
no-ops, which tensors are never materialised, and that a rule does not fire
when its preconditions fail."""

from paper_1412_6249_b200 import BiGraph, Location, build_sgd_iteration
from paper_1412_6249_b200.dispatcher import _Plan
from paper_1412_6249_b200.nets import googlenet

LOC = Location("local", 0)
LRN = {"size": 5, "alpha": 1e-4, "beta": 0.75, "k": 1.0}


def test_googlenet_plan():
    g = build_sgd_iteration(googlenet(batch=2)).graphs[0]
    plan = _Plan(g, 4, 4)
    name = {oid: op.name for oid, op in g.operators.items()}
    kinds = {oid: op.kind for oid, op in g.operators.items()}
    away = [kinds[o] for o in plan.fused_away]
    # every conv's ReLU is computed by its epilogue; all 9 concats elided both ways
    assert away.count("relu_forward") == 57
    assert away.count("concat_forward") == 9 and away.count("concat_backward") == 9
    # LRN: both forwards drop scale, both backwards recompute it
    lrn = {name[o]: f for o, f in plan.fusion.items() if kinds[o].startswith("lrn")}
    assert lrn["lrn4"] == {"lrn_no_scale": True} and lrn["lrn9"] == {"lrn_no_scale": True}
    assert lrn["bwd_lrn4"]["lrn_recompute"] and lrn["bwd_lrn9"]["lrn_recompute"]
    assert {"scale4", "scale9"} <= plan.elided
    # no tensor a non-no-op operator reads is elided unless its reader is fused for it
    for oid, op in g.operators.items():
        if oid in plan.fused_away:
            continue
        for t in op.inputs:
            tn = g.tensors[t].name
            if tn in plan.elided:
                assert oid in plan.fusion, (op.name, tn)


def _lrn_graph(extra_reader: bool):
    g = BiGraph()
    x, y, s = (g.add_tensor(n, (2, 8, 4, 4), LOC) for n in ("x", "y", "s"))
    dy, dx = g.add_tensor("dy", (2, 8, 4, 4), LOC), g.add_tensor("dx", (2, 8, 4, 4), LOC)
    g.add_operator("f", "lrn_forward", [x], [y, s], LOC, attrs=LRN)
    g.add_operator("b", "lrn_backward", [x, y, s, dy], [dx], LOC, attrs=LRN)
    if extra_reader:
        c = g.add_tensor("c", (2, 8, 4, 4), LOC)
        g.add_operator("cp", "copy", [s], [c], LOC)
    return g


def test_lrn_scale_elision_preconditions():
    plan = _Plan(_lrn_graph(False), 1)
    assert "s" in plan.elided
    plan = _Plan(_lrn_graph(True), 1)  # scale read by another operator: stored
    assert "s" not in plan.elided and not plan.fusion
