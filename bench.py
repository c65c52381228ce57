#!/usr/bin/env python
"""Benchmark: GoogLeNet data-parallel SGD training throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--net googlenet|nin] [--batch 128]

A step is one full Purine iteration — the training graph (forward, loss,
backward, parameter exchange + SGD update) plus the swap graph — of
GoogLeNet at batch 128 per GPU on synthetic 224x224 data (BASELINE.json
config 4; metric "GoogLeNet train images/sec").  One process per GPU; for
N > 1 launch under torchrun (the exchange runs over NCCL/NVLink).

`value`: img/s with inputs resident in HBM (K replays of the captured
iteration, CUDA events, max over ranks).  `e2e`: the same metric through
the public API with the batch copied in from pinned host memory and the loss
read back every step.  `roofline`: the dominant kernel family (the conv /
fc contractions) from a traced replay of the same captured iteration.
`cpu_baseline`: the CPU oracle (numpy port of the reference kernels) on a
bounded sample.  `--impl reference` times that CPU path alone.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--net", default="googlenet", choices=["googlenet", "nin"])
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--force-nccl", action="store_true",
                    help="route the exchange through NCCL even on one GPU (plumbing test)")
    ap.add_argument("--op-table", default=None,
                    help="write the traced replay's per-operator device times (TSV) here")
    ap.add_argument("--intervals", default=None,
                    help="write the branch-concurrent traced replay's operator intervals (TSV)")
    ap.add_argument("--profile-steps", type=int, default=0,
                    help="extra replays for an external profiler (ncu); no timing")
    return ap.parse_args()


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def _tf32_peak(peaks):
    """Effective fp32-accurate (3xTF32) tensor peak, TFLOP/s, and its basis."""
    p = ROOT / "profiles" / "tf32_peak.json"
    if p.exists():
        try:
            rec = json.loads(p.read_text())
            tf = rec.get("tf32_tflops_sustained") or rec["tf32_tflops"]
            return tf / 3.0, ("measured cuBLAS TF32 sustained (profiles/tf32_peak.json) / 3 "
                              "passes (kernels timed inside a long step)")
        except Exception:
            pass
    bf = peaks.get("bf16_tflops_sustained") or peaks.get("bf16_tflops") or 1398.2
    return bf / 2.0 / 3.0, "measured bf16 sustained (MEASURED_PEAKS.json) / 2 (tf32 rate) / 3 passes"


def _step_traffic(net):
    """DRAM bytes per step of the contraction family and of the HBM-bound kernels,
    from the newest committed ncu capture of one captured step
    (profiles/*_step_traffic_*.json, tools/summarize_ncu.py traffic): ncu
    replays each kernel cold-cache, so this bounds the real (L2-warm) traffic
    from above."""
    if net != "googlenet":
        return None
    import re

    files = sorted((ROOT / "profiles").glob("*_step_traffic_v*.json"),
                   key=lambda f: int(re.search(r"_v(\d+)\.json$", f.name).group(1)))
    if not files:
        return None
    try:
        rec = json.loads(files[-1].read_text())
        rec["file"] = "profiles/" + files[-1].name
        return rec
    except Exception:
        return None


class _Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
            # nvidia-smi takes a moment to start: only enter the timed region once
            # it is sampling, and keep only the samples taken inside it
            t_end = time.monotonic() + 5.0
            while not self.lines and time.monotonic() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.first = len(self.lines)
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            # a region shorter than the sampling period: take the first sample
            # after it (the clocks it ended at)
            t_end = time.monotonic() + 0.3
            while len(self.lines) <= self.first and time.monotonic() < t_end:
                time.sleep(0.005)
            self.last = len(self.lines)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[self.first:getattr(self, "last", len(self.lines))]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline (oracle port of the reference kernels)


def _cpu_sample(net_name: str, batch: int, seed: int = 7):
    """One CPU training iteration (forward, backward, SGD) of ``net`` at
    ``batch`` images through the oracle's serial executor."""
    from oracle.serial import run_graph_serial

    from paper_1412_6249_b200 import SyntheticFeed, build_sgd_iteration, feeder, init_params
    from paper_1412_6249_b200.nets import googlenet, nin

    net = (googlenet if net_name == "googlenet" else nin)(batch=batch)
    seq = build_sgd_iteration(net)

    class _S(dict):
        def set(self, name, arr):
            self[name] = np.array(arr, dtype=np.float32, copy=True)

    st = _S()
    init_params(net, st, seed, seq.layout)
    feeder(SyntheticFeed.for_net(net, seed, spread=0.0), seq.layout)(0, st)

    def one():
        t = time.perf_counter()
        for g in seq.graphs:
            run_graph_serial(g, st)
        return time.perf_counter() - t

    return one


def cpu_throughput(net_name: str, sample_batch: int, workers: int, steps: int):
    """Replicas as threads (the reference's lane-per-peer model; numpy
    releases the GIL in its kernels).  Returns (img/s, per-step seconds)."""
    from concurrent.futures import ThreadPoolExecutor

    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=1):
        runners = [_cpu_sample(net_name, sample_batch, seed=7 + i) for i in range(workers)]
        times = []
        with ThreadPoolExecutor(max_workers=workers) as ex:
            for _ in range(steps):
                t = time.perf_counter()
                list(ex.map(lambda f: f(), runners))
                times.append(time.perf_counter() - t)
    return workers * sample_batch / float(np.mean(times)), times


def _reference_dp(net_name: str, peers: int, batch: int, seed: int = 7):
    """The reference's data-parallel CPU execution: the
    bi-graph of ``build_data_parallel`` with ``peers`` replicas + the server
    subgraph, fused backward, run by the oracle's restatement of the
    reference dispatcher's multi-worker mode (one thread per lane) on the
    oracle's numpy kernels.  Returns a callable timing one iteration (G_dnn +
    G_swap) in seconds."""
    from oracle.serial import run_graph_lanes

    from paper_1412_6249_b200 import (Location, ParallelPlan, SyntheticFeed, build_data_parallel,
                                      feeder, init_params)
    from paper_1412_6249_b200.nets import googlenet, nin

    net = (googlenet if net_name == "googlenet" else nin)(batch=batch)
    plan = ParallelPlan("data", peers=tuple(Location("local", k) for k in range(peers)),
                        server=Location("local", peers))
    seq = build_data_parallel(net, plan, split_backward=False)

    class _S(dict):
        def set(self, name, arr):
            self[name] = np.array(arr, dtype=np.float32, copy=True)

    st = _S()
    init_params(net, st, seed, seq.layout)
    feed = feeder(SyntheticFeed.for_net(net, seed, peers=peers, spread=0.0), seq.layout)
    it = [0]

    def one():
        feed(it[0], st)
        it[0] += 1
        t = time.perf_counter()
        for g in seq.graphs:
            run_graph_lanes(g, st)
        return time.perf_counter() - t

    return one, st, seq.layout


def run_reference(args):
    """CPU reference arm: BASELINE.md section 4's plan -- P = --gpus peers at
    batch 8 per peer through the reference's data-parallel graph (replicas on
    their own lane threads, numpy single-threaded per lane), 1 warm-up and at
    most 2 timed iterations (a GoogLeNet iteration is ~10 s of CPU per peer)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits

    peers = max(1, args.gpus)
    batch = 8
    steps = max(1, min(args.steps, 2))
    warm = max(0, min(args.warmup, 1))
    with threadpool_limits(limits=1):
        one, st, layout = _reference_dp(args.net, peers, batch)
        for _ in range(warm):
            one()
        times = [one() for _ in range(steps)]
    loss = float(np.mean([st[n][0] for n in layout.loss_names]))
    value = peers * batch / float(np.mean(times))
    affinity = len(os.sched_getaffinity(0))
    cores = min(peers + 1, affinity)  # one lane thread per peer + the server lane
    metric = "GoogLeNet train images/sec" if args.net == "googlenet" else "NIN train images/sec"
    sample = (f"{steps} timed iteration(s) after {warm} warm-up of {args.net} data-parallel SGD, "
              f"{peers} peer(s) x batch {batch} + server subgraph (build_data_parallel, fused "
              f"backward), oracle numpy port on the reference's lane-per-thread dispatcher")
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": "img/s",
        "n_gpus": args.gpus, "steps": steps, "steps_requested": args.steps, "warmup": warm,
        "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (SyntheticFeed seed 7, spread 0)",
        "config": {"workload": f"{args.net} data-parallel SGD iteration (G_dnn + G_swap), 224x224, "
                               f"CPU: {peers} peers x batch {batch} (BASELINE.md section 4)",
                   "global_batch": peers * batch, "per_peer_batch": batch, "peers": peers,
                   "parallelism": f"dp{peers} (CPU lanes)"},
        "cpu_baseline": {"value": value, "unit": "img/s", "cores": cores, "kind": "port",
                         "sample": sample, "os_cpu_count": os.cpu_count(),
                         "affinity_cores": affinity},
        "e2e": {"value": value, "unit": "img/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "final_loss": loss,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU path


def run_ours(args):
    import torch

    from paper_1412_6249_b200 import (Location, ParallelPlan, SyntheticFeed, TensorStore,
                                      build_data_parallel, init_params)
    from paper_1412_6249_b200 import _native
    from paper_1412_6249_b200.executor import CapturedSequence
    from paper_1412_6249_b200.nets import googlenet, nin
    from paper_1412_6249_b200.perf import CONTRACTION_KINDS, op_bytes, op_flops

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1 or args.force_nccl:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    net = (googlenet if args.net == "googlenet" else nin)(batch=args.batch, lr=0.01)
    store = TensorStore(dev)
    from paper_1412_6249_b200.exchange import build_rank_sequence

    seq, exch = build_rank_sequence(net, world, rank, store,
                                    nccl=True if args.force_nccl else None)
    layout = seq.layout
    init_params(net, store, 7, layout)
    feed = SyntheticFeed.for_net(net, 7, peers=world, spread=0.0)
    x_host, lab_host = feed.batch_for(0, rank)
    xname, lname = layout.data_names[0], layout.label_names[0]
    store.set(xname, x_host)
    store.set(lname, lab_host)
    loss_name = layout.loss_names[0]

    exe = CapturedSequence(seq, store)
    exe.prepare()
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        exe.step()
    barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with _Clocks(local) as clocks:
        start.record()
        for _ in range(args.steps):
            exe.step()
        end.record()
        end.synchronize()
    ms = start.elapsed_time(end)
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    img_s = world * args.batch * args.steps / (ms / 1e3)
    loss = float(store.array(loss_name)[0])
    finite = bool(np.isfinite(loss))

    for _ in range(args.profile_steps):
        exe.step()
    torch.cuda.synchronize()

    # e2e through the public API: pinned host batch in, loss out, every step
    e2e = None
    if not args.no_e2e:
        x_pin = torch.from_numpy(x_host).pin_memory()
        l_pin = torch.from_numpy(lab_host).pin_memory()

        def e2e_pass(n):
            exe.prefetch({xname: x_pin, lname: l_pin})
            rs = []
            for s in range(n):
                exe.step()
                rs.append(store.read_async(loss_name))
                if s + 1 < n:
                    exe.prefetch({xname: x_pin, lname: l_pin})
            return rs

        # untimed warm-up of the same loop: the first DMA from freshly pinned
        # pages and the host allocator's first pinned loss buffers (one per
        # pending read) are set up here, not inside the timed steps
        for r in e2e_pass(args.steps):
            r.value()
        barrier()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        # every step: its batch is copied host->device inside the timed region
        # (prefetched on a side stream while the previous step computes) and
        # its loss is read back
        exe.prefetch({xname: x_pin, lname: l_pin})
        reads = []
        for s in range(args.steps):
            exe.step()
            reads.append(store.read_async(loss_name))  # this step's loss, device -> host
            if s + 1 < args.steps:
                exe.prefetch({xname: x_pin, lname: l_pin})
        e1.record()
        e2e_losses = [float(r.value()[0]) for r in reads]
        e1.synchronize()
        e2e_ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": world * args.batch * args.steps / (e2e_ms / 1e3), "unit": "img/s",
               "h2d_bytes_per_step": int(x_pin.numel() * 4 + l_pin.numel() * 4),
               "d2h_bytes_per_step": 4, "wall_s": time.perf_counter() - t0,
               "api": "CapturedSequence.prefetch(pinned batch) -> .step() -> "
                      "TensorStore.read_async(loss)",
               "overlap": "batch i+1's host->device copy runs on a side stream during step i; "
                          "each step's loss is copied to pinned host memory behind it",
               "losses_finite": bool(np.all(np.isfinite(e2e_losses)))}
        exe.sync()  # raises if any step produced a non-finite value

        # the same through the drop-in API itself, feeding the pinned batch with
        # before_iteration and reading each loss in after_graph.  run() keeps a
        # replay cache (dispatcher._run_replayed): a graph's first call with a
        # given buffer binding walks it, the second captures the walk, later
        # ones replay it -- the 4 untimed iterations cover both swap parities
        from paper_1412_6249_b200 import run_sequence
        from paper_1412_6249_b200.executor import PrefetchFeed

        rs_reads = []
        # each iteration's pinned batch is copied host->device on a side stream
        # while the previous iteration computes (PrefetchFeed, a
        # before_iteration hook writing the store through TensorStore.set)
        # (one feed object for the warm-up and the timed run: its staging
        # buffers and copy stream are allocated outside the timed region)
        before = PrefetchFeed(lambda it: {xname: x_pin, lname: l_pin}, dev, iterations=4)

        def after(rep, st):
            if rep.graph_index == 0:
                rs_reads.append(st.read_async(loss_name))

        run_sequence(seq, store, before_iteration=before, after_graph=after, iterations=4,
                     trace=False)
        barrier()
        rs_reads.clear()
        before.iterations = args.steps
        e0.record()
        run_sequence(seq, store, before_iteration=before, after_graph=after,
                     iterations=args.steps, trace=False)
        e1.record()
        rs_losses = [float(r.value()[0]) for r in rs_reads]
        e1.synchronize()
        rs_ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([rs_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            rs_ms = float(t.item())
        # the headline e2e is the drop-in API's; CapturedSequence (the same
        # schedule driven without the per-graph Python dispatch) rides along
        captured = e2e
        e2e = {"value": world * args.batch * args.steps / (rs_ms / 1e3), "unit": "img/s",
               "h2d_bytes_per_step": captured["h2d_bytes_per_step"],
               "d2h_bytes_per_step": captured["d2h_bytes_per_step"],
               "api": "run_sequence(seq, store, before_iteration=PrefetchFeed(<pinned batch>), "
                      "after_graph=<TensorStore.read_async(loss)>, trace=False)",
               "overlap": "PrefetchFeed copies iteration i+1's batch host->device on a side "
                          "stream during iteration i; each iteration's loss is copied to pinned "
                          "host memory behind it",
               "note": "run() walks each graph once per buffer binding, captures the walk on "
                       "the second call and replays it afterwards (PURINE_B200_CAPTURE=0: walk "
                       "every call)",
               "losses_finite": bool(np.all(np.isfinite(rs_losses))),
               "captured_sequence": {k: captured[k] for k in
                                     ("value", "unit", "api", "overlap", "losses_finite")}}

    # traced replay of the same schedule, serialised on one stream per lane
    # (branch streams off) so each operator's interval is its own kernels'
    # device time, not time shared with concurrent branches
    texe = CapturedSequence(seq, store, trace=True)
    prev = os.environ.get("PURINE_B200_BRANCH_STREAMS")
    os.environ["PURINE_B200_BRANCH_STREAMS"] = "1"
    try:
        texe.prepare()
    finally:
        if prev is None:
            del os.environ["PURINE_B200_BRANCH_STREAMS"]
        else:
            os.environ["PURINE_B200_BRANCH_STREAMS"] = prev
    from paper_1412_6249_b200.dispatcher import _Plan

    # operators the fusion plan turns into no-ops launch nothing: their bytes
    # are moved (or never moved) by the kernel that absorbed them
    fused_away = [_Plan(g, texe.cap, 1).fused_away for g in seq.graphs]
    reps = 3
    per_kind: dict[str, float] = {}
    contraction_ms = contraction_flops = 0.0
    hbm_ms = hbm_bytes = 0.0
    rows: dict[str, list] = {}
    for r in range(reps):
        par = texe.parity
        texe.step()
        torch.cuda.synchronize()
        if r == 0:
            continue
        for gi, op, t in texe.op_times_ms(par):
            per_kind[op.kind] = per_kind.get(op.kind, 0.0) + t / (reps - 1)
            g = seq.graphs[gi]
            row = rows.setdefault(op.name, [op.kind, 0.0, op_flops(g, op), op_bytes(g, op)])
            row[1] += t / (reps - 1)
            if op.kind in CONTRACTION_KINDS:
                contraction_ms += t / (reps - 1)
                contraction_flops += op_flops(g, op) / (reps - 1)
            elif (op.kind not in ("swap", "flatten_forward", "flatten_backward", "copy",
                                  "dp_exchange") and op.id not in fused_away[gi]):
                hbm_ms += t / (reps - 1)
                hbm_bytes += op_bytes(g, op) / (reps - 1)
    # exposed communication: |union(exchange) minus union(compute)| / T_iter
    # on the traced replay's device intervals (profiler.exposed_ns, the reference's
    # interval arithmetic, profiler.py:58-102)
    from paper_1412_6249_b200.profiler import _union, exposed_ns

    # ... on the schedule that is timed: a traced replay with the branch streams on
    cexe = CapturedSequence(seq, store, trace=True)
    cexe.prepare()
    for _ in range(3):
        cpar = cexe.parity
        cexe.step()
    torch.cuda.synchronize()
    iv = cexe.op_intervals_ns(cpar)
    if args.intervals and rank == 0:
        with open(args.intervals, "w") as f:
            f.write("op\tkind\tstart_ns\tend_ns\n")
            for _gi, op, s0, s1 in iv:
                f.write(f"{op.name}\t{op.kind}\t{s0}\t{s1}\n")
    comm_sp = [(s0, s1) for _, op, s0, s1 in iv if op.kind in ("dp_exchange", "copy")]
    comp_sp = [(s0, s1) for _, op, s0, s1 in iv if op.kind not in ("dp_exchange", "copy", "swap")]
    t_iter = (max(s1 for *_, s1 in iv) - min(s0 for _, _, s0, _ in iv)) if iv else 0
    exposed = {"fraction": exposed_ns(comm_sp, comp_sp) / t_iter if t_iter else None,
               "exchange_ms": sum(b - a for a, b in _union(comm_sp)) / 1e6,
               "traced_iteration_ms": t_iter / 1e6,
               "basis": ("dp_exchange ops on the exchange stream vs compute ops, device "
                         "intervals of a traced replay with the timed schedule's branch "
                         "streams" + ("" if world > 1 else
                                                           "; world 1: the exchange is the "
                                                           "local fused mean+SGD, no NCCL"))}
    # the virtual-time simulator calibrated with this run's
    # per-operator device times predicts the 1..8-GPU scaling of this config
    predicted = None
    if rank == 0 and world == 1:
        from paper_1412_6249_b200.costsim import predict_scaling

        op_s = {name: t / 1e3 for name, (kind, t, _f, _b) in rows.items()}
        try:
            first = predict_scaling(net, [1], op_s)[0]
            scale = (ms / args.steps / 1e3) / first.iteration_s
            pts = predict_scaling(net, [1, 2, 4, 8], op_s, compute_scale=scale)
            predicted = {"basis": "costsim.predict_scaling: measured op times (scaled to the "
                                  "measured step), NVLink bucket-exchange model x1.5 overlap "
                                  "slowdown; a prediction, not a measurement",
                         "points": [{"n_gpus": p.world, "img_s": round(p.images_per_s, 1),
                                     "efficiency": round(p.efficiency, 4),
                                     "exposed_comm": round(p.exposed_comm, 4)} for p in pts]}
        except Exception as exc:  # noqa: BLE001 - the prediction is optional
            predicted = {"error": str(exc)}
    if args.op_table and rank == 0:
        with open(args.op_table, "w") as f:
            f.write("op\tkind\tms\tgflop\tmbytes\n")
            for name, (kind, t, fl, by) in sorted(rows.items(), key=lambda kv: -kv[1][1]):
                f.write(f"{name}\t{kind}\t{t:.4f}\t{fl / 1e9:.3f}\t{by / 1e6:.2f}\n")
    peaks = _peaks()
    tpeak, basis = _tf32_peak(peaks)
    traffic = _step_traffic(args.net)
    achieved = contraction_flops / (contraction_ms / 1e3) / 1e12 if contraction_ms else 0.0
    roofline = {"bound": "tensor", "achieved": achieved, "peak": tpeak, "unit": "TFLOP/s",
                "frac": achieved / tpeak if tpeak else None,
                "traffic": (traffic or {}).get("contraction", {}).get("dram_bytes"),
                "traffic_basis": (f"dram__bytes_read.sum + dram__bytes_write.sum of the "
                                  f"contraction family's launches in one step, bytes per step "
                                  f"({traffic['file']}, ncu, cold-cache per launch)")
                                 if traffic else None,
                "kernel": "conv/fc implicit-GEMM family (fwd+dgrad+wgrad), per step",
                "peak_basis": basis,
                "share_of_step": contraction_ms / (ms / args.steps),
                "timing_basis": "per-operator CUDA events of a serialised traced replay",
                "algorithmic_tflop_per_step": contraction_flops / 1e12,
                "hbm_kernels": {"basis": "algorithmic bytes (SURVEY 8d) of the launched "
                                         "non-contraction operators (fused-away no-ops "
                                         "excluded) / their serialised device time",
                                "achieved_gbs": hbm_bytes / (hbm_ms / 1e3) / 1e9 if hbm_ms else None,
                                "peak_gbs": peaks.get("hbm_gbs", 6533.8),
                                "ms_per_step": hbm_ms,
                                "algorithmic_bytes_per_step": hbm_bytes,
                                "traffic": (traffic or {}).get("hbm_kernels", {}).get("dram_bytes")},
                # whole iteration = (FLOP / tensor peak + bytes / HBM peak) / T_step
                "iteration": {"ideal_ms": 1e3 * (contraction_flops / (tpeak * 1e12) +
                                                 hbm_bytes / (peaks.get("hbm_gbs", 6533.8) * 1e9)),
                              "frac": 1e3 * (contraction_flops / (tpeak * 1e12) +
                                             hbm_bytes / (peaks.get("hbm_gbs", 6533.8) * 1e9))
                              / (ms / args.steps)}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sample = 2
        val, _t = cpu_throughput(args.net, sample, 1, 1)
        cpu = {"value": val, "unit": "img/s", "cores": 1, "kind": "port",
               "sample": f"one {sample}-image {args.net} training iteration, oracle numpy port, "
                         "1 thread"}

    lib = _native.lib()
    line = {
        "metric": "GoogLeNet train images/sec" if args.net == "googlenet" else "NIN train images/sec",
        "value": img_s, "unit": "img/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (3xTF32 tensor-core / fp32 SIMT)",
        "data": "synthetic (SyntheticFeed spread=0: N(0,1) images, uniform labels; one batch "
                "reused per step, resident in HBM)",
        "config": {"workload": f"{args.net} v1 data-parallel SGD iteration (G_dnn + G_swap), "
                               f"224x224, batch {args.batch}/GPU",
                   "model": args.net, "global_batch": world * args.batch, "per_gpu_batch": args.batch,
                   "image": 224, "parallelism": f"dp{world}",
                   "l2": "inputs (77 MB/batch) and activations (~3.4 GB) exceed the 126 MB L2"},
        "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "exposed_comm": exposed,
        "predicted_scaling": predicted,
        "clocks": clocks.summary(),
        "gpu_launches": int(exe.launches_per_step) * args.steps,
        "launches_per_step": int(exe.launches_per_step),
        "final_loss": loss, "loss_finite": finite,
        "tcgen05": bool(lib.raw("bf_has_tcgen05")()),
        "kernel_ms_per_step": {k: round(v, 4) for k, v in sorted(per_kind.items(),
                                                                   key=lambda kv: -kv[1])},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def _launch_ranks(args) -> int:
    """``--gpus N`` (N > 1) started without torchrun: re-launch this script as
    N ranks, one process per GPU, through torch.distributed.run on 127.0.0.1.
    Fails loudly when fewer than N GPUs are visible."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} needs {args.gpus} visible CUDA devices, "
                                   f"found {have}"}), flush=True)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = _args()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_launch_ranks(args))
    if args.impl == "ours" and "WORLD_SIZE" in os.environ and \
            int(os.environ["WORLD_SIZE"]) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
