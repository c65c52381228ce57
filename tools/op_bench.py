"""Time one memory-bound kernel family at GoogLeNet shapes (batch 128).

    python tools/op_bench.py maxpool_fwd|maxpool_bwd|maxpool_fwd_staged|maxpool_bwd_x|lrn_fwd|lrn_fwd_noscale|lrn_bwd|lrn_bwd_rc [--reps 5]

Prints per-shape time and achieved GB/s (algorithmic bytes).
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1412_6249_b200 import _native  # noqa: E402
from paper_1412_6249_b200.kinds import pool_out_dim  # noqa: E402
from paper_1412_6249_b200.nets import googlenet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("op")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    lib = _native.lib()
    lib("bf_set_device", 0)
    net = googlenet(batch=128)
    r = net._resolved()
    st = torch.cuda.current_stream().cuda_stream
    tot_ms = tot_b = 0.0
    for nd in net.nodes:
        if not nd.kind.startswith("maxpool") or not a.op.startswith("maxpool"):
            if not (a.op.startswith("lrn") and nd.kind == "lrn"):
                continue
        n, c, h, w = r["shapes"][nd.inputs[0]]
        x = torch.randn(n, c, h, w, device="cuda")
        if nd.kind == "maxpool":
            p = pool_out_dim(h, nd.kernel, nd.stride, nd.pad)
            q = pool_out_dim(w, nd.kernel, nd.stride, nd.pad)
            y = torch.empty(n, c, p, q, device="cuda")
            m = torch.empty_like(y)
            dx = torch.empty_like(x)
            if a.op == "maxpool_fwd_staged":  # no mask (elided in the product pairing)
                fn = lambda: lib("bf_maxpool_fwd_staged", x.data_ptr(), y.data_ptr(), None, n, c,
                                 h, w, p, q, nd.kernel, nd.stride, nd.pad, st)
                nbytes = 4 * x.numel() + 4 * y.numel()
            elif a.op in ("maxpool_bwd_x", "maxpool_bwd_xr"):  # argmax recomputed from x
                rf = 1 if a.op == "maxpool_bwd_xr" else 0  # + the folded ReLU backward
                fn = lambda: lib("bf_maxpool_bwd_x", x.data_ptr(), y.data_ptr(), dx.data_ptr(), rf,
                                 n, c, h, w, p, q, nd.kernel, nd.stride, nd.pad, st)
                nbytes = 8 * x.numel() + 4 * y.numel()
            elif a.op == "maxpool_fwd":
                fn = lambda: lib("bf_maxpool_fwd", x.data_ptr(), y.data_ptr(), m.data_ptr(), n, c, h,
                                 w, p, q, nd.kernel, nd.stride, nd.pad, st)
                nbytes = 4 * x.numel() + 8 * y.numel()
            else:
                lib("bf_maxpool_fwd", x.data_ptr(), y.data_ptr(), m.data_ptr(), n, c, h, w, p, q,
                    nd.kernel, nd.stride, nd.pad, st)
                fn = lambda: lib("bf_maxpool_bwd", m.data_ptr(), y.data_ptr(), dx.data_ptr(), n, c,
                                 h, w, p, q, nd.kernel, nd.stride, nd.pad, st)
                nbytes = 8 * y.numel() + 4 * x.numel()
        else:
            yy, sc, dx = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
            if a.op == "lrn_fwd":
                fn = lambda: lib("bf_lrn_fwd", x.data_ptr(), yy.data_ptr(), sc.data_ptr(), n, c, h, w,
                                 5, 1e-4, 0.75, 1.0, st)
                nbytes = 12 * x.numel()
            elif a.op == "lrn_fwd_noscale":
                fn = lambda: lib("bf_lrn_fwd", x.data_ptr(), yy.data_ptr(), None, n, c, h, w,
                                 5, 1e-4, 0.75, 1.0, st)
                nbytes = 8 * x.numel()
            elif a.op == "lrn_bwd_rc":
                fn = lambda: lib("bf_lrn_bwd_recompute", x.data_ptr(), sc.data_ptr(), dx.data_ptr(),
                                 None, n, c, h, w, 5, 1e-4, 0.75, 1.0, st)
                nbytes = 12 * x.numel()
            else:
                lib("bf_lrn_fwd", x.data_ptr(), yy.data_ptr(), sc.data_ptr(), n, c, h, w, 5, 1e-4,
                    0.75, 1.0, st)
                fn = lambda: lib("bf_lrn_bwd", x.data_ptr(), yy.data_ptr(), sc.data_ptr(),
                                 x.data_ptr(), dx.data_ptr(), n, c, h, w, 5, 1e-4, 0.75, 1.0, st)
                nbytes = 20 * x.numel()
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        tot_ms += ms
        tot_b += nbytes
        print(f"{nd.name:28s} {n}x{c}x{h}x{w} k{nd.kernel}/s{nd.stride}: {ms:7.3f} ms "
              f"{nbytes / ms / 1e6:7.1f} GB/s")
    print(f"TOTAL {a.op}: {tot_ms:.3f} ms {tot_b / tot_ms / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
