"""Diagnostic (not collected by pytest): GoogLeNet/NIN one-iteration gradient
agreement of GPU and CPU-oracle float32 results, each measured against a
float64 ground truth.  Prints one line per parameter tensor.

    python tests/diag_parity.py [googlenet|nin] [batch]
"""

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))

from fp64_reference import dag_grads_fp64  # noqa: E402
from oracle.serial import run_graph_serial  # noqa: E402
from paper_1412_6249_b200 import (SyntheticFeed, TensorStore, build_sgd_iteration, feeder,  # noqa: E402
                                  init_params, run_sequence)
from paper_1412_6249_b200.nets import googlenet, nin  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "googlenet"
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    net = (googlenet if name == "googlenet" else nin)(batch=batch, lr=0.01)
    seq = build_sgd_iteration(net)
    feed = SyntheticFeed.for_net(net, 7, spread=0.0)

    class _S(dict):
        def set(self, n, a):
            self[n] = np.array(a, dtype=np.float32, copy=True)

    ref = _S()
    init_params(net, ref, 7, seq.layout)
    feeder(feed, seq.layout)(0, ref)
    params = {p: ref[p].copy() for p, _ in net.param_shapes()}
    x, labels = ref["x"].copy(), ref["labels"].copy()
    run_graph_serial(seq.graphs[0], ref)

    store = TensorStore("cuda:0")
    init_params(net, store, 7, seq.layout)
    run_sequence(seq, store, before_iteration=feeder(feed, seq.layout), iterations=1)

    acts = {}
    loss64, g64 = dag_grads_fp64(net, params, x, labels, acts)
    print(f"loss fp64 {loss64:.8f} oracle {float(ref['loss'][0]):.8f} "
          f"gpu {float(store.array('loss')[0]):.8f}")
    for i, nd in enumerate(net.nodes[:40]):
        a = f"a{i + 1}"
        t64, d64 = acts[a]
        line = (f"{a:5s} {nd.kind:8s} {nd.name:28s} fwd gpu {rel(store.array(a), t64):8.2e} "
                f"oracle {rel(ref[a], t64):8.2e}")
        if d64 is not None and store.has("d" + a) and ("d" + a) in ref:
            line += (f" | bwd gpu {rel(store.array('d' + a), d64):8.2e} "
                     f"oracle {rel(ref['d' + a], d64):8.2e}")
        print(line)
    worst_gpu = worst_orc = 0.0
    for p, _ in net.param_shapes():
        gg, go, gt = store.array(f"d{p}"), ref[f"d{p}"], g64[p]
        scale = max(float(np.abs(gt).max()), 1e-30)
        eg = float(np.abs(gg - gt).max()) / scale
        eo = float(np.abs(go - gt).max()) / scale
        ego = float(np.abs(gg - go).max()) / scale
        bad = int((~np.isclose(gg, go, rtol=1e-4, atol=1e-5 * max(1.0, scale))).sum())
        worst_gpu, worst_orc = max(worst_gpu, eg), max(worst_orc, eo)
        print(f"d{p:6s} max|.|={scale:9.3e} gpu-vs-fp64 {eg:8.2e} (norm {rel(gg, gt):8.2e}) "
              f"oracle-vs-fp64 {eo:8.2e} (norm {rel(go, gt):8.2e}) gpu-vs-oracle {ego:8.2e} "
              f"fails(1e-4/1e-5*max)={bad}")
    print(f"worst scaled max error vs fp64: gpu {worst_gpu:.2e} oracle {worst_orc:.2e}")


if __name__ == "__main__":
    main()
