"""Lowering of the parameter-server subgraph to NCCL for one process per GPU.

The reference's data-parallel scheme (builders.py:581-611) moves every
gradient to a server location (``up_`` copies), averages in rank order
(``agg_``), updates once (``upd_``) and broadcasts back (``down_`` copies).
On one 8xB200 NVSwitch box that topology would funnel 8x28 MB through one
GPU.  Lowering keeps the graph and its semantics but replaces, per rank, the
server subgraph by ``dp_exchange`` operators on the rank's upload lane, one
per gradient *bucket*:

    ncclReduceScatter(sum, in place)  ->  fused mean + SGD on the owned shard
    (bf_sgd_mean_update: w - lr * (g_sum / f32(world)), or with momentum
    bf_sgd_mean_momentum: v' = mu*v + lr*(g_sum / f32(world)); w - v')
    ->  ncclAllGather

so each GPU is the parameter server for 1/world of every bucket ("gradient
reduce and parameter broadcast sharded across the box", NS).  Buckets are
formed in backward order, so the dispatcher issues each bucket's exchange as
soon as its last weight gradient exists and it overlaps the remaining
backward layers on its own CUDA stream.  Every rank builds the same graph,
so every rank enqueues collectives in the same (serial-mode) order.

Memory: parameters, their ``_new`` twins and gradients live in three flat
HBM arenas laid out in bucket order (each tensor padded to 16 floats, each
bucket to a multiple of 16*world), so a bucket is one contiguous range for
NCCL and one launch for the update.  Swapping ``w`` <-> ``w_new`` views keeps
the layout, so both CUDA-graph bindings see contiguous buckets.

Momentum (the server's ``sgd_momentum`` + velocity swaps, builders.py
581-611 with SPEC.md:312's extension): each rank keeps only the velocity of
the shards it owns, one ``vxch_b{i}`` tensor per bucket (length
flat_len / world) in a fourth and fifth flat arena, ping-ponged with
``vxch_b{i}_new`` by the swap graph exactly like the parameters.

Collectives go through ``store._collective`` (`NcclCollective` over an
NCCL communicator, or `LocalGroup`: several ranks' stores on ONE device with
the reduce-scatter / all-gather done by this library's own rank-ordered
aggregate and copy kernels -- the single-GPU stand-in the tests use to run
world-2 product code).

Numerics: at world=1 the result is bitwise the reference's aggregate(mean)
+ sgd_update (or sgd_momentum); `LocalGroup` sums in rank order, so it is
bitwise the reference-shaped server graph at any world; over NCCL the
summation order is NCCL's, so parity is tolerance-based.
"""

from __future__ import annotations

import os

from dataclasses import dataclass, field
from math import prod

from .builders import Layout, ParallelPlan, build_data_parallel, param_names
from .graph import BiGraph, GraphError, GraphSequence, Location
from .kinds import KernelError

__all__ = ["Bucket", "ExchangePlan", "plan_buckets", "lower_data_parallel", "materialize",
           "setup_nccl", "build_rank_sequence", "NcclCollective", "LocalGroup",
           "velocity_name"]

ALIGN = 16  # floats (64 B)


def _pad(n: int, a: int) -> int:
    return -(-n // a) * a


@dataclass
class Bucket:
    params: list[str]                    # canonical names, arena order
    offsets: dict[str, int] = field(default_factory=dict)  # element offsets in the arena
    start: int = 0
    length: int = 0                      # padded, multiple of ALIGN * world


@dataclass
class ExchangePlan:
    world: int
    buckets: list[Bucket]
    total: int
    shapes: dict[str, tuple[int, ...]]

    def bucket_of(self, name: str) -> Bucket:
        for b in self.buckets:
            if name in b.offsets:
                return b
        raise KeyError(name)


def plan_buckets(param_shapes, world: int, bucket_bytes: int = 4 << 20) -> ExchangePlan:
    """Group parameters into contiguous buckets in backward (reverse layer) order."""
    if world < 1:
        raise GraphError(f"world must be >= 1, got {world}")
    shapes = dict(param_shapes)
    order = [n for n, _ in reversed(list(param_shapes))]
    buckets: list[Bucket] = []
    cur: list[str] = []
    size = 0
    for name in order:
        cur.append(name)
        size += _pad(prod(shapes[name]), ALIGN)
        if size * 4 >= bucket_bytes:
            buckets.append(Bucket(cur))
            cur, size = [], 0
    if cur:
        buckets.append(Bucket(cur))
    pos = 0
    for b in buckets:
        b.start = pos
        off = pos
        for name in b.params:
            b.offsets[name] = off
            off += _pad(prod(shapes[name]), ALIGN)
        b.length = _pad(off - pos, ALIGN * world)
        pos += b.length
    return ExchangePlan(world, buckets, pos, shapes)


def lower_data_parallel(seq: GraphSequence, rank: int, plan: ExchangePlan, net) -> GraphSequence:
    """Rank ``rank``'s partition of a `build_data_parallel` sequence with the
    server subgraph replaced by per-bucket ``dp_exchange`` operators."""
    layout = seq.layout
    if layout is None or layout.scheme != "data":
        raise GraphError("lower_data_parallel needs a data-parallel sequence")
    g = seq.graphs[0]
    sfx = f"_p{rank}"
    peer = g.tensor_named(f"x{sfx}").location
    base = min(layout.copy_threads)
    keep = [g.operators[o] for o in g.insertion_order
            if g.operators[o].location == peer and g.operators[o].kind != "copy"]
    used: set[int] = set()
    for op in keep:
        used.update(op.inputs)
        used.update(op.outputs)
    new_names = {f"{c}_new{sfx}" for c, _ in plan.shapes.items()}
    ng = BiGraph()
    for tid in sorted(g.tensors):
        t = g.tensors[tid]
        if tid in used or t.name in new_names:
            ng.add_tensor(t.name, t.shape, t.location)
    for op in keep:
        ng.add_operator(op.name, op.kind, [ng.tensor_id(g.tensors[t].name) for t in op.inputs],
                        [ng.tensor_id(g.tensors[t].name) for t in op.outputs], op.location,
                        op.thread, dict(op.attrs))
    grad_of = {}
    for c in plan.shapes:
        grad_of[c] = f"d{c}{sfx}"
        if not ng.has_tensor(grad_of[c]):
            raise GraphError(f"lowering: gradient {grad_of[c]!r} not found")
    mu = float(getattr(net, "momentum", 0.0) or 0.0)
    vel: list[tuple[str, int]] = []
    for i, b in enumerate(plan.buckets):
        ws = [ng.tensor_id(f"{c}{sfx}") for c in b.params]
        gs = [ng.tensor_id(grad_of[c]) for c in b.params]
        outs = [ng.tensor_id(f"{c}_new{sfx}") for c in b.params]
        attrs = {"lr": net.lr, "world": plan.world, "rank": rank, "flat_len": b.length,
                 "offsets": [b.offsets[c] - b.start for c in b.params]}
        if mu > 0:  # the rank's velocity shard of this bucket: one more input / output
            shard = b.length // plan.world
            vname = velocity_name(i, rank)
            ws.append(ng.add_tensor(vname, (shard,), peer))
            outs.append(ng.add_tensor(f"{vname[:-len(sfx)]}_new{sfx}", (shard,), peer))
            attrs["momentum"] = mu
            vel.append((vname, shard))
        ng.add_operator(f"xch_b{i}{sfx}", "dp_exchange", ws + gs, outs, peer, thread=base + 2 * rank,
                        attrs=attrs)
    sw = seq.graphs[1]
    nsw = BiGraph()
    for o in sw.insertion_order:
        op = sw.operators[o]
        if op.location != peer:
            continue
        ids = []
        for t in op.outputs:
            tv = sw.tensors[t]
            ids.append(nsw.tensor_id(tv.name) if nsw.has_tensor(tv.name)
                       else nsw.add_tensor(tv.name, tv.shape, tv.location))
        nsw.add_operator(op.name, op.kind, [], ids, op.location, op.thread, dict(op.attrs))
        swap_thread = op.thread
    for vname, shard in vel:  # velocity ping-pong, next to the parameter swaps
        vnew = f"{vname[:-len(sfx)]}_new{sfx}"
        a = nsw.add_tensor(vname, (shard,), peer)
        b = nsw.add_tensor(vnew, (shard,), peer)
        nsw.add_operator(f"swap_{vname}", "swap", [], [a, b], peer, swap_thread)
    canon = tuple(plan.shapes)
    lay = Layout(scheme="data", data_names=(f"x{sfx}",), label_names=(f"labels{sfx}",),
                 loss_names=(f"loss{sfx}",), canonical_params=canon,
                 peer_params=(tuple(f"{c}{sfx}" for c in canon),),
                 copy_threads=layout.copy_threads, classes=layout.classes, batch=layout.batch,
                 velocity_params=tuple(v for v, _ in vel), canonical_in_store=False,
                 first_rank=rank)
    return GraphSequence([ng, nsw], iterations=seq.iterations, layout=lay)


def velocity_name(bucket: int, rank: int) -> str:
    """The lowered graph's velocity shard of ``bucket`` on ``rank``."""
    return f"vxch_b{bucket}_p{rank}"


def materialize(store, plan: ExchangePlan, rank: int, momentum: bool = False) -> None:
    """Allocate the flat arenas on the store's device and bind the rank's
    parameter / new-parameter / gradient tensors (and, with momentum, its
    velocity shards) as views into them."""
    import torch

    sfx = f"_p{rank}"
    arenas = [torch.zeros(plan.total, dtype=torch.float32, device=store.device) for _ in range(3)]
    store._arenas = arenas
    for b in plan.buckets:
        for c in b.params:
            n = prod(plan.shapes[c])
            o = b.offsets[c]
            for arena, name in zip(arenas, (f"{c}{sfx}", f"{c}_new{sfx}", f"d{c}{sfx}")):
                store.place(name, arena[o:o + n].view(plan.shapes[c]))
    if momentum:  # this rank's velocity shards, bucket order (1/world of the parameters)
        vel = [torch.zeros(plan.total // plan.world, dtype=torch.float32, device=store.device)
               for _ in range(2)]
        store._arenas += vel
        for i, b in enumerate(plan.buckets):
            shard, o = b.length // plan.world, b.start // plan.world
            vname = velocity_name(i, rank)
            store.place(vname, vel[0][o:o + shard])
            store.place(f"{vname[:-len(sfx)]}_new{sfx}", vel[1][o:o + shard])


def setup_nccl(store, world: int, rank: int) -> None:
    """Create this rank's NCCL communicator (unique id broadcast over the
    default torch.distributed process group) and attach it to the store."""
    import ctypes

    import torch.distributed as dist

    from . import _native

    lib = _native.lib()
    buf = ctypes.create_string_buffer(128)
    if rank == 0:
        lib("bf_nccl_unique_id", ctypes.cast(buf, ctypes.c_void_p))
    box = [bytes(buf.raw) if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    uid = ctypes.create_string_buffer(box[0], 128)
    comm = ctypes.c_void_p()
    lib("bf_set_device", store.device.index or 0)
    lib("bf_nccl_init", ctypes.byref(comm), world, rank, ctypes.cast(uid, ctypes.c_void_p))
    # the exchange lane's stream is high-priority (dispatcher), which keeps
    # small-bucket collectives at their unloaded latency under a GEMM load
    # (tools/exchange_sweep.py --overlap); optionally also keep SMs free of
    # persistent GEMM CTAs
    reserve = int(os.environ.get("PURINE_B200_SM_RESERVE", "0"))
    if reserve:
        lib("bf_set_sm_reserve", reserve)
    store._nccl = comm.value
    store._nccl_rank = rank
    store._nccl_world = world
    store._collective = NcclCollective(comm.value, world, rank)


def build_rank_sequence(net, world: int, rank: int, store, bucket_bytes: int = 4 << 20,
                        nccl: bool | None = None):
    """Full DP graph for ``world`` peers (server on device ``world``), lowered
    for ``rank``; arenas materialised in ``store``; NCCL set up when world > 1."""
    plan = ParallelPlan("data", peers=tuple(Location("local", k) for k in range(world)),
                        server=Location("local", world))
    full = build_data_parallel(net, plan)
    xplan = plan_buckets(param_names(net), world, bucket_bytes)
    seq = lower_data_parallel(full, rank, xplan, net)
    materialize(store, xplan, rank, momentum=bool(seq.layout.velocity_params))
    if nccl is None:
        nccl = world > 1
    if nccl:  # world == 1 with nccl=True exercises the NCCL path on one GPU (tests)
        setup_nccl(store, world, rank)
    return seq, xplan


class NcclCollective:
    """In-place reduce-scatter(sum) / all-gather of one bucket over an NCCL
    communicator (csrc/nccl_ops.cu), enqueued on the exchange lane's stream."""

    def __init__(self, comm: int, world: int, rank: int) -> None:
        self.comm, self.world, self.rank = comm, world, rank

    def reduce_scatter(self, base: int, shard: int, stream: int) -> None:
        from . import _native

        _native.lib()("bf_nccl_reduce_scatter", self.comm, base, base + 4 * shard * self.rank,
                      shard, stream)

    def all_gather(self, base: int, shard: int, stream: int) -> None:
        from . import _native

        _native.lib()("bf_nccl_all_gather", self.comm, base + 4 * shard * self.rank, base, shard,
                      stream)


class LocalGroup:
    """``world`` ranks' stores on ONE CUDA device, each dispatched from its own
    host thread, exchanging through this library's kernels instead of NCCL.

    Each collective is a rendezvous: every rank records an event on its
    exchange stream and waits at a barrier; the last rank to arrive makes its
    stream wait on all the others' events, runs the collective there
    (reduce-scatter: `bf_aggregate` sum of every rank's shard in RANK order,
    written in place into the owner's shard -- the reference aggregate's
    order, ops.py:440-457; all-gather: `bf_copy` of every owned shard to every
    rank), records a completion event, and every rank's stream waits on it.
    Host order is the serial dispatch order, identical on every rank, so the
    rendezvous sequence matches.  Eager dispatch only (a captured CUDA graph
    cannot wait on another capture's events)."""

    def __init__(self, world: int, timeout_s: float = 120.0) -> None:
        import threading

        self.world = world
        self._barrier = threading.Barrier(world, timeout=timeout_s)
        self._lock = threading.Lock()
        self._slots: list = [None] * world
        self._done = None

    def member(self, rank: int) -> "_LocalMember":
        return _LocalMember(self, rank)

    def _rendezvous(self, rank: int, base: int, shard: int, stream: int, op: str) -> None:
        import torch

        ext = torch.cuda.ExternalStream(stream)
        ev = torch.cuda.Event()
        ev.record(ext)
        self._slots[rank] = (base, shard, ext, ev, op)
        import threading

        try:
            idx = self._barrier.wait()
            if idx == 0:  # exactly one thread runs the collective
                try:
                    self._run()
                except BaseException:
                    self._barrier.abort()
                    raise
            self._barrier.wait()
        except threading.BrokenBarrierError:
            raise KernelError("LocalGroup: a peer rank failed or never reached this "
                              "collective") from None
        ext.wait_event(self._done)
        self._barrier.wait()  # every rank has consumed `_done` before it is reused

    def _run(self) -> None:
        import torch

        from . import _native

        slots = list(self._slots)
        bases, shards, ops = [s[0] for s in slots], {s[1] for s in slots}, {s[4] for s in slots}
        if len(shards) != 1 or len(ops) != 1:
            raise KernelError(f"LocalGroup: ranks disagree on the collective ({ops}, {shards})")
        shard, op = shards.pop(), ops.pop()
        st = slots[0][2]
        for s in slots[1:]:
            st.wait_event(s[3])
        lib = _native.lib()
        h = st.cuda_stream
        if op == "reduce_scatter":
            for r in range(self.world):
                parts = _native.ptr_array([b + 4 * shard * r for b in bases])
                lib("bf_aggregate", parts, self.world, bases[r] + 4 * shard * r, shard, 0, h)
        else:  # all_gather: owner r's shard to every other rank
            dev = torch.cuda.current_device()
            for r in range(self.world):
                for q in range(self.world):
                    if q != r:
                        lib("bf_copy", bases[q] + 4 * shard * r, dev, bases[r] + 4 * shard * r,
                            dev, shard, h)
        done = torch.cuda.Event()
        done.record(st)
        self._done = done


class _LocalMember:
    def __init__(self, group: LocalGroup, rank: int) -> None:
        self.group, self.rank, self.world = group, rank, group.world

    def reduce_scatter(self, base: int, shard: int, stream: int) -> None:
        self.group._rendezvous(self.rank, base, shard, stream, "reduce_scatter")

    def all_gather(self, base: int, shard: int, stream: int) -> None:
        self.group._rendezvous(self.rank, base, shard, stream, "all_gather")


def shard_of(flat_len: int, world: int, rank: int) -> tuple[int, int]:
    """(shard length, element offset of ``rank``'s shard) of a bucket: the
    in-place reduce-scatter leaves the gradient sum of that range on ``rank``,
    which updates it and all-gathers it back (NCCL in-place convention
    recvbuff = sendbuff + rank * recvcount)."""
    if flat_len % world:
        raise KernelError(f"dp_exchange: bucket length {flat_len} not divisible by world {world}")
    shard = flat_len // world
    return shard, rank * shard


def check_bucket(ws, gs, outs, offsets) -> tuple[int, int, int]:
    """Verify a bucket's tensors are laid out contiguously as planned;
    returns the flat base pointers (w, g, w_new)."""
    w0, g0, o0 = ws[0].ptr, gs[0].ptr, outs[0].ptr
    for t, off in zip(ws, offsets):
        if t.ptr != w0 + 4 * off:
            raise KernelError("dp_exchange: parameters are not laid out in a flat arena "
                              "(call exchange.materialize before running)")
    for t, off in zip(gs, offsets):
        if t.ptr != g0 + 4 * off:
            raise KernelError("dp_exchange: gradients are not laid out in a flat arena")
    for t, off in zip(outs, offsets):
        if t.ptr != o0 + 4 * off:
            raise KernelError("dp_exchange: new parameters are not laid out in a flat arena")
    return w0, g0, o0
