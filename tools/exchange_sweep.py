"""BASELINE config 5: per-layer gradient reduce + parameter broadcast sweep.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port 29511 tools/exchange_sweep.py [--min-kb 4] [--max-mb 256] [--overlap]

For message sizes S = 4 KB .. 256 MB (powers of two, 17 points) every rank runs
the lowered exchange step of exchange.py on one S-byte bucket through the
library's C ABI: in-place ncclReduceScatter(sum) -> bf_sgd_mean_update on the
owned 1/N shard -> in-place ncclAllGather.  Device time per
exchange is taken with CUDA events on the exchange stream, max over ranks.
Reported: algbw = S / t and busbw = algbw * 2 (N - 1) / N (reduce-scatter +
all-gather), as nccl-tests does.

``--overlap`` repeats the sweep while a GoogLeNet backward-sized load (conv
weight gradients, the batch-128 conv2/3x3 shape) runs on a second stream, and
reports the exchange's slowdown: the cost of overlapping gradient transfer
with backward layers (the paper's central claim).

One JSON line per size on rank 0.  At N = 1 the collectives are 1-rank NCCL
calls (a local copy), which checks the plumbing, not NVLink.
"""

import argparse
import ctypes
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def sizes(min_kb: int, max_mb: int) -> list[int]:
    out, s = [], min_kb << 10
    while s <= max_mb << 20:
        out.append(s)
        s <<= 1
    return out


def bus_bw(nbytes: int, seconds: float, world: int) -> tuple[float, float]:
    """(algbw, busbw) in GB/s for one reduce-scatter + all-gather of nbytes."""
    alg = nbytes / seconds / 1e9 if seconds > 0 else 0.0
    return alg, alg * (2 * (world - 1) / world if world > 1 else 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-kb", type=int, default=4)
    ap.add_argument("--max-mb", type=int, default=256)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--overlap", action="store_true")
    ap.add_argument("--sm-reserve", type=int, default=None,
                    help="SMs kept free of GEMM CTAs (default: the library's, 8 when N > 1)")
    a = ap.parse_args()

    import torch
    import torch.distributed as dist

    from paper_1412_6249_b200 import TensorStore, _native
    from paper_1412_6249_b200.exchange import setup_nccl

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    store = TensorStore(dev)
    setup_nccl(store, world, rank)
    lib = _native.lib()
    if a.sm_reserve is not None:
        lib("bf_set_sm_reserve", a.sm_reserve)
    comm = ctypes.c_void_p(store._nccl)
    xs = torch.cuda.Stream(device=dev, priority=-1)  # as the dispatcher's exchange lane
    bg = torch.cuda.Stream(device=dev)
    ws = torch.empty(64 << 20, device=dev)

    # background load for --overlap: repeated conv2/3x3 weight gradients (batch 128)
    if a.overlap:
        g = (128, 64, 56, 56, 192, 3, 3, 56, 56, 1, 1)
        bx = torch.randn(128, 64, 56, 56, device=dev)
        bdy = torch.randn(128, 192, 56, 56, device=dev)
        bdw = torch.empty(192, 64, 3, 3, device=dev)

    def background(n):
        with torch.cuda.stream(bg):
            for _ in range(n):
                lib("bf_conv2d_bwd_weight", bx.data_ptr(), bdy.data_ptr(), bdw.data_ptr(), *g,
                    ws.data_ptr(), ws.numel() * 4, bg.cuda_stream)

    for nbytes in sizes(a.min_kb, a.max_mb):
        n = nbytes // 4
        n = (n + world - 1) // world * world
        shard = n // world
        grad = torch.randn(n, device=dev)
        w = torch.randn(n, device=dev)
        out = torch.empty(n, device=dev)

        def one():
            s = xs.cuda_stream
            off = rank * shard
            lib("bf_nccl_reduce_scatter", comm, grad.data_ptr(), grad.data_ptr() + off * 4, shard, s)
            lib("bf_sgd_mean_update", w.data_ptr() + off * 4, grad.data_ptr() + off * 4,
                out.data_ptr() + off * 4, 0.01, world, shard, s)
            lib("bf_nccl_all_gather", comm, out.data_ptr() + off * 4, out.data_ptr(), shard, s)

        res = {}
        for mode in (["alone", "overlap"] if a.overlap else ["alone"]):
            torch.cuda.synchronize()
            dist.barrier()
            with torch.cuda.stream(xs):
                for _ in range(a.warmup):
                    one()
            torch.cuda.synchronize()
            if mode == "overlap":
                background(4 * a.iters)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(xs):
                e0.record(xs)
                for _ in range(a.iters):
                    one()
                e1.record(xs)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / a.iters], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sec = float(t.item()) / 1e3
            alg, bus = bus_bw(nbytes, sec, world)
            res[mode] = {"us": sec * 1e6, "algbw_gbs": alg, "busbw_gbs": bus}
        if rank == 0:
            line = {"bytes": nbytes, "n_gpus": world, **res}
            if "overlap" in res:
                line["overlap_slowdown"] = res["overlap"]["us"] / res["alone"]["us"]
            print(json.dumps(line), flush=True)
    lib("bf_nccl_destroy", comm)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
