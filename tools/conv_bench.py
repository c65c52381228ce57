"""Per-layer timing of the conv contractions at GoogLeNet shapes (batch 128).

    python tools/conv_bench.py [--net googlenet] [--batch 128] [--pass fwd,dgrad,wgrad]
                               [--engine 0|1] [--only N] [--reps 5]

Launches the C-ABI entry points directly on device buffers and times each
with CUDA events; prints one line per (layer, pass) and per-pass totals.
"""

import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1412_6249_b200 import _native  # noqa: E402
from paper_1412_6249_b200.kinds import conv_out_dim  # noqa: E402
from paper_1412_6249_b200.nets import googlenet, nin  # noqa: E402


def conv_layers(net):
    r = net._resolved()
    out = []
    for i, nd in enumerate(net.nodes):
        if nd.kind != "conv":
            continue
        x = r["shapes"][nd.inputs[0]]
        n, c, h, w = x
        p = conv_out_dim(h, nd.kernel, nd.stride, nd.pad, nd.floor)
        q = conv_out_dim(w, nd.kernel, nd.stride, nd.pad, nd.floor)
        out.append((nd.name, n, c, h, w, nd.out, nd.kernel, nd.kernel, p, q, nd.stride, nd.pad,
                    nd.inputs[0] == "data"))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="googlenet")
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--passes", default="fwd,dgrad,wgrad")
    ap.add_argument("--engine", type=int, default=0)
    ap.add_argument("--only", type=int, default=-1)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--quiet", action="store_true")
    a = ap.parse_args()
    lib = _native.lib()
    lib("bf_set_device", 0)
    lib("bf_set_gemm_engine", a.engine)
    net = (googlenet if a.net == "googlenet" else nin)(batch=a.batch)
    ws = torch.empty(256 << 20, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    totals = {}
    layers = conv_layers(net)
    if a.only >= 0:
        layers = [layers[a.only]]
    for (name, n, c, h, w, k, r, s, p, q, st, pad, bottom) in layers:
        x = torch.randn(n, c, h, w, device="cuda")
        wt = torch.randn(k, c, r, s, device="cuda") / (c * r * s) ** 0.5
        b = torch.randn(k, device="cuda")
        y = torch.empty(n, k, p, q, device="cuda")
        dy = torch.randn(n, k, p, q, device="cuda")
        dx = torch.empty_like(x)
        dw = torch.empty_like(wt)
        flops = 2.0 * n * k * p * q * c * r * s
        geo = (n, c, h, w, k, r, s, p, q, st, pad)
        calls = {
            "fwd": ("bf_conv2d_fwd", (x.data_ptr(), wt.data_ptr(), b.data_ptr(), y.data_ptr())),
            "dgrad": ("bf_conv2d_bwd_data", (wt.data_ptr(), dy.data_ptr(), dx.data_ptr())),
            "wgrad": ("bf_conv2d_bwd_weight", (x.data_ptr(), dy.data_ptr(), dw.data_ptr())),
        }
        line = f"{name:28s} {n:4d}x{c:4d}x{h:3d}x{w:3d} -> {k:4d} {r}x{s}/{st}"
        for ps in a.passes.split(","):
            if ps == "dgrad" and bottom:
                continue
            fn, ptrs = calls[ps]
            args = (*ptrs, *geo, ws.data_ptr(), ws.numel() * 4, stream)
            lib(fn, *args)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                lib(fn, *args)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            totals.setdefault(ps, [0.0, 0.0])
            totals[ps][0] += ms
            totals[ps][1] += flops
            line += f" | {ps} {ms:7.3f} ms {flops / ms / 1e9:6.1f} TF/s"
        if not a.quiet:
            print(line, flush=True)
    allms = sum(v[0] for v in totals.values())
    allfl = sum(v[1] for v in totals.values())
    for ps, (ms, fl) in totals.items():
        print(f"TOTAL {ps:6s} {ms:8.2f} ms  {fl / ms / 1e9:6.1f} TF/s")
    print(f"TOTAL all    {allms:8.2f} ms  {allfl / allms / 1e9:6.1f} TF/s")


if __name__ == "__main__":
    main()
