"""Generate golden fixtures from the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``biflow`` from /root/reference/pkg/src (read-only, no bytecode
written) and records, with fixed seeds:
  * op-level vectors of every reference kernel on the DP path
    (ops.py:164-457) -> ops.npz
  * graph JSON of reference-built sequences (builders.py:496-647) and their
    serial-mode dispatch order (dispatcher.py, BIFLOW_LANES=1) -> graphs.json
  * end-to-end training results (losses, final parameters) of
      - config 1: conv(32,k5,p2)+relu+fc10, batch 16, build_sgd_iteration
      - a 2-peer data-parallel MLP (build_data_parallel, fused and split)
      - config 2 (conv-pool-conv-pool-fc, 2 peers + server) built by the
        product builder, executed by the REFERENCE dispatcher with the
        oracle's pooling kernels registered through the reference's own
        extension hook (default_registry(), ops.py:807-809)
    -> train.npz / train.json
The GPU box never runs this script; the fixtures it writes are committed.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import biflow  # noqa: E402
from biflow import builders as rb  # noqa: E402
from biflow import ops as rops  # noqa: E402
from biflow.dispatcher import run_sequence as ref_run_sequence  # noqa: E402
from biflow.graph import graph_from_json as ref_graph_from_json  # noqa: E402
from biflow.graph import graph_to_json as ref_graph_to_json  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32)


def op_vectors() -> dict[str, np.ndarray]:
    rng = np.random.default_rng(2024)
    out: dict[str, np.ndarray] = {}
    x = f32(rng.standard_normal((6, 20)))
    w = f32(rng.standard_normal((20, 7)))
    b = f32(rng.standard_normal(7))
    dy = f32(rng.standard_normal((6, 7)))
    out.update(fc_x=x, fc_w=w, fc_b=b, fc_dy=dy, fc_y=rops.fc_forward(x, w, b))
    dx, dw, db = rops.fc_backward(x, w, dy)
    out.update(fc_dx=dx, fc_dw=dw, fc_db=db)
    for tag, (n, c, h, wd, k, r, stride, pad) in {
        "c1": (2, 3, 9, 9, 4, 3, 1, 1),
        "c2": (2, 5, 8, 8, 6, 1, 1, 0),
        "c3": (1, 2, 11, 11, 3, 5, 2, 2),
        "c4": (3, 4, 7, 7, 5, 5, 1, 2),
    }.items():
        xx = f32(rng.standard_normal((n, c, h, wd)))
        ww = f32(rng.standard_normal((k, c, r, r)))
        bb = f32(rng.standard_normal(k))
        y = rops.conv2d_forward(xx, ww, bb, stride=stride, pad=pad)
        gy = f32(rng.standard_normal(y.shape))
        gx, gw, gb = rops.conv2d_backward(xx, ww, gy, stride=stride, pad=pad)
        out.update({f"{tag}_x": xx, f"{tag}_w": ww, f"{tag}_b": bb, f"{tag}_y": y,
                    f"{tag}_dy": gy, f"{tag}_dx": gx, f"{tag}_dw": gw, f"{tag}_db": gb,
                    f"{tag}_geom": np.array([stride, pad], dtype=np.int64)})
    rx = f32(rng.standard_normal((4, 33)))
    rx[0, :3] = [0.0, -0.0, 1e-30]
    rdy = f32(rng.standard_normal((4, 33)))
    out.update(relu_x=rx, relu_y=rops.relu_forward(rx), relu_dy=rdy,
               relu_dx=rops.relu_backward(rx, rdy))
    logits = f32(rng.standard_normal((16, 10)) * 3)
    labels = f32(rng.integers(0, 10, 16))
    loss, dl = rops.softmax_xent(logits, labels)
    out.update(sm_logits=logits, sm_labels=labels, sm_loss=loss, sm_dlogits=dl)
    sw = f32(rng.standard_normal(1001))
    sg = f32(rng.standard_normal(1001))
    out.update(sgd_w=sw, sgd_g=sg, sgd_out=rops.sgd_update(sw, sg, 0.0123))
    parts = [f32(rng.standard_normal(777)) for _ in range(3)]
    out.update(agg_p0=parts[0], agg_p1=parts[1], agg_p2=parts[2],
               agg_mean=rops.aggregate(parts, "mean"), agg_sum=rops.aggregate(parts, "sum"))
    return out


def serial_order(reports) -> list[list[str]]:
    return [[r.name for r in sorted(rep.trace, key=lambda r: (r.start, r.end))] for rep in reports]


def train(seq, net, feed, seed, iterations, registry=None):
    store = rops.TensorStore()
    rb.init_params(net, store, seed, seq.layout)
    losses = []

    def after(rep, st):
        if rep.graph_index == 0:
            losses.append([float(st.array(n)[0]) for n in seq.layout.loss_names])

    reps = ref_run_sequence(seq, store, registry, max_workers=1,
                            before_iteration=rb.feeder(feed, seq.layout), after_graph=after,
                            iterations=iterations)
    return store, losses, serial_order(reps[:len(seq.graphs)])


def peers_plan(n):
    return rb.ParallelPlan(scheme="data", peers=tuple(biflow.Location("local", k) for k in range(n)),
                           server=biflow.Location("local", n))


def main() -> None:
    np.savez_compressed(HERE / "ops.npz", **op_vectors())

    graphs: dict[str, object] = {}
    arrays: dict[str, np.ndarray] = {}
    meta: dict[str, object] = {}

    # config 1 through build_sgd_iteration
    cfg1 = rb.NetSpec((3, 32, 32), (rb.LayerSpec("conv", 32, 5, 1, 2), rb.LayerSpec("relu"),
                                    rb.LayerSpec("fc", 10)), batch=16, lr=1e-3)
    seq = rb.build_sgd_iteration(cfg1)
    feed = rb.SyntheticFeed.for_net(cfg1, 7)
    feed = rb.SyntheticFeed(feed.seed, feed.input_shape, feed.classes, feed.batch, spread=0.0)
    store, losses, order = train(seq, cfg1, feed, 7, 2)
    graphs["cfg1"] = {"graphs": [ref_graph_to_json(g) for g in seq.graphs], "serial": order}
    meta["cfg1_losses"] = losses
    for name in seq.layout.canonical_params:
        arrays[f"cfg1_{name}"] = store.array(name)

    # 2-peer data-parallel MLP, fused and split backward
    mlp = rb.NetSpec((20,), (rb.LayerSpec("fc", 16), rb.LayerSpec("relu"), rb.LayerSpec("fc", 4)),
                     batch=8, lr=0.05)
    for split in (False, True):
        tag = f"mlp_dp2_{'split' if split else 'fused'}"
        seq = rb.build_data_parallel(mlp, peers_plan(2), split_backward=split)
        feed = rb.SyntheticFeed.for_net(mlp, 13, peers=2)
        store, losses, order = train(seq, mlp, feed, 13, 3)
        graphs[tag] = {"graphs": [ref_graph_to_json(g) for g in seq.graphs], "serial": order}
        meta[f"{tag}_losses"] = losses
        for name in seq.layout.canonical_params:
            arrays[f"{tag}_{name}"] = store.array(name)

    # config 2: product builder graph, reference dispatcher + oracle pooling kinds
    import oracle
    from paper_1412_6249_b200 import builders as pb
    from paper_1412_6249_b200 import graph as pg
    from paper_1412_6249_b200.nets import cifar_convnet

    net2 = cifar_convnet(batch=16, lr=1e-3)
    plan = pb.ParallelPlan("data", peers=(pg.Location("local", 0), pg.Location("local", 1)),
                           server=pg.Location("local", 2))
    pseq = pb.build_data_parallel(net2, plan)
    ref_graphs = [ref_graph_from_json(pg.graph_to_json(g)) for g in pseq.graphs]
    rseq = biflow.GraphSequence(ref_graphs, layout=pseq.layout)
    registry = rops.default_registry()

    def plain(kind):
        fn = oracle.KERNELS[kind]

        def execute(ctx, op):
            ins = [ctx.store.array(ctx.graph.tensors[t].name) for t in op.inputs]
            for t, arr in zip(op.outputs, fn(ins, op.attrs)):
                ctx.store.set(ctx.graph.tensors[t].name, arr)

        return execute

    for kind in ("maxpool_forward", "maxpool_backward"):
        registry[kind] = rops.OpKindSpec(kind, 1, None, None, lambda *a: None, plain(kind))
    store = rops.TensorStore()
    pb.init_params(net2, store, 7, pseq.layout)
    feed2 = pb.SyntheticFeed.for_net(net2, 7, peers=2, spread=0.0)
    losses = []

    def after(rep, st):
        if rep.graph_index == 0:
            losses.append([float(st.array(n)[0]) for n in pseq.layout.loss_names])

    reps = ref_run_sequence(rseq, store, registry, max_workers=1,
                            before_iteration=pb.feeder(feed2, pseq.layout), after_graph=after,
                            iterations=2)
    graphs["cfg2_dp2"] = {"serial": serial_order(reps[:2])}
    meta["cfg2_dp2_losses"] = losses
    for name in pseq.layout.canonical_params:
        arrays[f"cfg2_dp2_{name}"] = store.array(name)

    np.savez_compressed(HERE / "train.npz", **arrays)
    (HERE / "graphs.json").write_text(json.dumps(graphs, sort_keys=True) + "\n")
    (HERE / "train.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print("wrote", sorted(p.name for p in HERE.iterdir()))


if __name__ == "__main__":
    os.environ["BIFLOW_LANES"] = "1"
    main()
