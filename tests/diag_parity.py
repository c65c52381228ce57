"""Diagnostic (not collected by pytest): one GoogLeNet/NIN training iteration
on the GPU product path (fusion plan, branch streams) and on the CPU oracle,
each measured against a float64 ground truth (torch autograd on the CPU).

Prints, per parameter gradient, the max error scaled by max|fp64| and the
norm-relative error of GPU and oracle against fp64, their ratio, and the
elementwise NS check (rel 1e-4 / abs 1e-5, unscaled) of GPU vs oracle.

    python tests/diag_parity.py [googlenet|nin] [batch] [--md OUT.md]
"""

import argparse
import os
import sys
import time
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
    ap = argparse.ArgumentParser()
    ap.add_argument("net", nargs="?", default="googlenet")
    ap.add_argument("batch", nargs="?", type=int, default=8)
    ap.add_argument("--md", default=None)
    a = ap.parse_args()
    net = (googlenet if a.net == "googlenet" else nin)(batch=a.batch, lr=0.01)
    seq = build_sgd_iteration(net)
    feed = SyntheticFeed.for_net(net, 7, spread=0.0)

    class _S(dict):
        def set(self, n, arr):
            self[n] = np.array(arr, dtype=np.float32, copy=True)

    ref = _S()
    init_params(net, ref, 7, seq.layout)
    feeder(feed, seq.layout)(0, ref)
    params = {p: ref[p].copy() for p, _ in net.param_shapes()}
    x, labels = ref["x"].copy(), ref["labels"].copy()
    t = time.perf_counter()
    run_graph_serial(seq.graphs[0], ref)
    t_orc = time.perf_counter() - t

    store = TensorStore("cuda:0")
    init_params(net, store, 7, seq.layout)
    run(seq, store, feed)

    t = time.perf_counter()
    loss64, g64 = dag_grads_fp64(net, params, x, labels)
    t_64 = time.perf_counter() - t
    lg, lo = float(store.array("loss")[0]), float(ref["loss"][0])
    lib = os.environ.get("PURINE_B200_LIB", "lib/libpurine_b200.so (default)")
    out = [f"# fp64 parity: {a.net} batch {a.batch}, one training iteration", "",
           f"library: `{lib}`; oracle {t_orc:.1f} s, fp64 {t_64:.1f} s", "",
           f"loss fp64 {loss64:.9f} | oracle {lo:.9f} (|d| {abs(lo - loss64):.2e}) | "
           f"gpu {lg:.9f} (|d| {abs(lg - loss64):.2e})", "",
           "| grad | max abs fp64 | gpu vs fp64 (max/scale) | oracle vs fp64 | ratio | "
           "gpu norm-rel | oracle norm-rel | gpu-vs-oracle max abs | NS fails (unscaled) |",
           "|---|---|---|---|---|---|---|---|---|"]
    worst_gpu = worst_orc = 0.0
    ratios = []
    fails_total = 0
    for p, _ in net.param_shapes():
        gg, go, gt = store.array(f"d{p}"), ref[f"d{p}"], g64[p]
        scale = max(float(np.abs(gt).max()), 1e-30)
        eg = float(np.abs(gg - gt).max()) / scale
        eo = float(np.abs(go - gt).max()) / scale
        r = eg / max(eo, 1e-30)
        ratios.append(r)
        bad = int((~np.isclose(gg, go, rtol=1e-4, atol=1e-5)).sum())
        fails_total += bad
        worst_gpu, worst_orc = max(worst_gpu, eg), max(worst_orc, eo)
        out.append(f"| d{p} | {scale:.3e} | {eg:.2e} | {eo:.2e} | {r:.2f} | {rel(gg, gt):.2e} | "
                   f"{rel(go, gt):.2e} | {float(np.abs(gg - go).max()):.2e} | {bad} |")
    out += ["", f"worst scaled max error vs fp64: gpu {worst_gpu:.2e}, oracle {worst_orc:.2e}; "
                f"median ratio {float(np.median(ratios)):.2f}, max ratio {max(ratios):.2f}; "
                f"elements outside rel 1e-4 / abs 1e-5 of the oracle: {fails_total}"]
    text = "\n".join(out)
    print(text)
    if a.md:
        Path(a.md).write_text(text + "\n")


def run(seq, store, feed):
    run_sequence(seq, store, before_iteration=feeder(feed, seq.layout), iterations=1)


if __name__ == "__main__":
    main()
