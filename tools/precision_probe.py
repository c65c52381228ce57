"""Contraction precision vs float64 as a function of the reduction length K.

For each case one contraction runs through the product boundary (graph ->
dispatcher -> C ABI) on cuda:0; the float64 answer comes from torch on the
GPU in float64.  Prints max |err| / max |ref|, the mean signed error
relative to |ref| (sign(ref) * (got - ref) / |ref| averaged: negative means
magnitudes shrink, the signature of round-toward-zero accumulation), and the
count of elements outside the NS bound |d| <= 1e-5 + 1e-4 |ref| (unscaled).

    python tools/precision_probe.py [--dist normal|uniform] [--md OUT]
"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))

from gpu_util import run_op  # noqa: E402


def stats(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    d = got - ref
    scale = float(np.abs(ref).max())
    nz = np.abs(ref) > 1e-3 * scale
    signed = float(np.mean(np.sign(ref[nz]) * d[nz] / np.abs(ref[nz])))
    fails = int((np.abs(d) > 1e-5 + 1e-4 * np.abs(ref)).sum())
    return float(np.abs(d).max()) / scale, signed, fails, scale


def gen(shape, dist, rng):
    if dist == "uniform":
        return rng.uniform(0.0, 1.0, shape).astype(np.float32)
    return rng.standard_normal(shape).astype(np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dist", default="normal")
    ap.add_argument("--md", default=None)
    a = ap.parse_args()
    rng = np.random.default_rng(1)
    rows = []

    def rec(name, k, got, ref):
        e, s, f, sc = stats(got, ref)
        rows.append(f"| {name} | {k} | {sc:.3e} | {e:.2e} | {s:+.2e} | {f} / {np.asarray(ref).size} |")
        print(rows[-1], flush=True)

    dev = torch.device("cuda:0")
    # fc forward: y = x @ w + b, K = d
    for d in (256, 1024, 4096, 16384, 65536):
        x, w = gen((128, d), a.dist, rng), gen((d, 256), a.dist, rng) / np.float32(np.sqrt(d))
        b = np.zeros(256, np.float32)
        got = run_op("fc_forward", {"x": x, "w": w, "b": b}, {"y": (128, 256)})["y"]
        ref = (torch.tensor(x, dtype=torch.float64, device=dev) @
               torch.tensor(w, dtype=torch.float64, device=dev)).cpu().numpy()
        rec("fc_forward", d, got, ref)
    # conv forward 3x3 (K = C*9) and 1x1 (K = C)
    for c, r in ((64, 3), (256, 3), (512, 3), (256, 1), (832, 1)):
        x = gen((8, c, 14, 14), a.dist, rng)
        w = gen((64, c, r, r), a.dist, rng) / np.float32(np.sqrt(c * r * r))
        b = np.zeros(64, np.float32)
        got = run_op("conv2d_forward", {"x": x, "w": w, "b": b}, {"y": (8, 64, 14, 14)},
                     {"stride": 1, "pad": r // 2})["y"]
        ref = F.conv2d(torch.tensor(x, dtype=torch.float64, device=dev),
                       torch.tensor(w, dtype=torch.float64, device=dev), padding=r // 2).cpu().numpy()
        rec(f"conv2d_forward {r}x{r}", c * r * r, got, ref)
    # conv weight gradient: K = N*P*Q
    for n, hw in ((8, 14), (32, 28), (128, 28), (128, 56)):
        x = gen((n, 64, hw, hw), a.dist, rng)
        dy = gen((n, 64, hw, hw), a.dist, rng) / np.float32(np.sqrt(n * hw * hw))
        w = np.zeros((64, 64, 3, 3), np.float32)
        got = run_op("conv2d_backward_weight", {"x": x, "w": w, "dy": dy}, {"dw": (64, 64, 3, 3)},
                     {"stride": 1, "pad": 1})["dw"]
        xt = torch.tensor(x, dtype=torch.float64, device=dev)
        dyt = torch.tensor(dy, dtype=torch.float64, device=dev)
        ref = torch.nn.grad.conv2d_weight(xt, (64, 64, 3, 3), dyt, padding=1).cpu().numpy()
        rec("conv2d_backward_weight 3x3", n * hw * hw, got, ref)
    out = ["| case | K | max abs ref | max err / max ref | mean signed rel err | NS fails |",
           "|---|---|---|---|---|---|"] + rows
    if a.md:
        Path(a.md).write_text(f"# contraction precision vs fp64 ({a.dist} inputs)\n\n" +
                              "\n".join(out) + "\n")


if __name__ == "__main__":
    main()
