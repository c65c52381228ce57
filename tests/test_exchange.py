"""Host-side logic of the lowered data-parallel exchange (exchange.py):
bucket planning, per-rank graph partition, collective issue order, and the
reduce-scatter -> shard update -> all-gather arithmetic across 2 gloo ranks."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1412_6249_b200 import (Location, ParallelPlan, build_data_parallel, param_names,
                                  serial_order)
from paper_1412_6249_b200.exchange import lower_data_parallel, plan_buckets, shard_of
from paper_1412_6249_b200.nets import cifar_convnet, googlenet


def _full(net, world):
    return build_data_parallel(net, ParallelPlan(
        "data", peers=tuple(Location("local", k) for k in range(world)),
        server=Location("local", world)))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_bucket_plan_is_contiguous_and_shardable(world):
    net = googlenet(batch=2)
    plan = plan_buckets(param_names(net), world, bucket_bytes=2 << 20)
    pos = 0
    seen = set()
    for b in plan.buckets:
        assert b.start == pos and b.length % (16 * world) == 0
        last = b.start
        for name in b.params:
            assert b.offsets[name] >= last and b.offsets[name] % 16 == 0
            last = b.offsets[name] + int(np.prod(plan.shapes[name]))
            seen.add(name)
        assert last <= b.start + b.length
        pos += b.length
        shard, first = shard_of(b.length, world, world - 1)
        assert shard * world == b.length and first + shard == b.length
    assert seen == {n for n, _ in param_names(net)} and plan.total == pos
    # backward order: the first bucket holds the classifier
    assert plan.buckets[0].params[0] == param_names(net)[-1][0]


@pytest.mark.parametrize("world", [2, 4])
def test_lowered_partition_replaces_server_subgraph(world):
    net = cifar_convnet(batch=4)
    full = _full(net, world)
    plan = plan_buckets(param_names(net), world, bucket_bytes=64 << 10)
    orders = []
    for rank in range(world):
        seq = lower_data_parallel(full, rank, plan, net)
        g = seq.graphs[0]
        assert g.validate().ok
        kinds = [op.kind for op in g.operators.values()]
        assert "copy" not in kinds and "aggregate" not in kinds and "sgd_update" not in kinds
        assert kinds.count("dp_exchange") == len(plan.buckets)
        for op in g.operators.values():
            assert op.location == Location("local", rank)
            if op.kind == "dp_exchange":
                assert op.thread == 1 + 2 * rank  # the rank's upload lane (builders.py:581-587)
        order = [g.operators[o].name for o in serial_order(g)]
        orders.append([n.rsplit("_p", 1)[0] for n in order])
        swaps = seq.graphs[1]
        assert len(swaps.operators) == len(param_names(net))
    # every rank enqueues its collectives in the same order
    assert all(o == orders[0] for o in orders)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, grads, w, lr, plan_len, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.from_numpy(grads[rank].copy())
    shard, first = shard_of(plan_len, world, rank)
    # reduce-scatter (sum), emulated on gloo by all_reduce + owning our shard
    dist.all_reduce(g)
    mine = g[first:first + shard].numpy()
    wn = np.float32(w[first:first + shard]) - np.float32(lr) * (mine / np.float32(world))
    pieces = [torch.empty(shard) for _ in range(world)]
    dist.all_gather(pieces, torch.from_numpy(wn.astype(np.float32)))
    out[rank] = torch.cat(pieces).numpy().copy()
    dist.destroy_process_group()


def test_gloo_two_ranks_match_aggregate_mean_sgd():
    world, n, lr = 2, 4 * 16 * 2, 0.05
    rng = np.random.default_rng(3)
    grads = [rng.standard_normal(n).astype(np.float32) for _ in range(world)]
    w = rng.standard_normal(n).astype(np.float32)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [mp.get_context("spawn").Process(target=_rank_main,
                                             args=(r, world, port, grads, w, lr, n, out))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    import oracle

    want = oracle.sgd_update(w, oracle.aggregate(grads, "mean"), lr)
    for r in range(world):
        got = np.asarray(out[r])
        assert np.array_equal(got, out[0])  # every rank holds identical parameters
        assert np.allclose(got, want, rtol=1e-6, atol=1e-7)


def test_exchange_sweep_sizes_and_bandwidth_math():
    """BASELINE config 5 sweep (tools/exchange_sweep.py): 17 message sizes from
    4 KB to 256 MB; busbw = algbw * 2(N-1)/N for reduce-scatter + all-gather."""
    import importlib.util
    from pathlib import Path

    spec = importlib.util.spec_from_file_location(
        "exchange_sweep", Path(__file__).resolve().parent.parent / "tools" / "exchange_sweep.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    s = mod.sizes(4, 256)
    assert len(s) == 17 and s[0] == 4096 and s[-1] == 256 << 20
    alg, bus = mod.bus_bw(1 << 30, 0.5, 8)
    assert abs(alg - 2.147483648) < 1e-9 and abs(bus - alg * 14 / 8) < 1e-9
    assert mod.bus_bw(1000, 1e-6, 1) == (1.0, 1.0)


@pytest.mark.parametrize("world", [1, 2, 4])
def test_lowered_partition_carries_momentum_shards(world):
    """With momentum the server's sgd_momentum + velocity swaps (builders.py
    581-611) become one velocity shard per bucket on each rank (length
    flat_len / world), an extra input/output of dp_exchange, and a swap."""
    net = cifar_convnet(batch=4, momentum=0.9)
    full = _full(net, world)
    assert any(op.kind == "sgd_momentum" for op in full.graphs[0].operators.values())
    plan = plan_buckets(param_names(net), world, bucket_bytes=64 << 10)
    for rank in range(world):
        seq = lower_data_parallel(full, rank, plan, net)
        g, sw = seq.graphs
        assert g.validate().ok and sw.validate().ok
        xch = [op for op in g.operators.values() if op.kind == "dp_exchange"]
        assert len(xch) == len(plan.buckets)
        for i, (op, b) in enumerate(zip(xch, plan.buckets)):
            assert op.attrs["momentum"] == 0.9
            nb = len(b.params)
            assert len(op.inputs) == 2 * nb + 1 and len(op.outputs) == nb + 1
            v = g.tensors[op.inputs[nb]]
            assert v.name == f"vxch_b{i}_p{rank}" and v.shape == (b.length // world,)
            assert g.tensors[op.outputs[nb]].name == f"vxch_b{i}_new_p{rank}"
        assert seq.layout.velocity_params == tuple(f"vxch_b{i}_p{rank}"
                                                   for i in range(len(plan.buckets)))
        swapped = {sw.tensors[op.outputs[0]].name for op in sw.operators.values()}
        assert set(seq.layout.velocity_params) <= swapped
        assert len(sw.operators) == len(param_names(net)) + len(plan.buckets)
        assert seq.layout.first_rank == rank


def test_dp_exchange_shape_check_rejects_bad_arity():
    from paper_1412_6249_b200 import BiGraph, GraphError
    from paper_1412_6249_b200.kinds import KernelError

    loc = Location("local", 0)
    g = BiGraph()
    w = g.add_tensor("w", (4,), loc)
    d = g.add_tensor("dw", (4,), loc)
    o = g.add_tensor("w_new", (4,), loc)
    with pytest.raises((GraphError, KernelError)):  # momentum needs the velocity pair
        g.add_operator("x", "dp_exchange", [w, d], [o], loc, attrs={"lr": 0.1, "world": 1,
                                                                     "momentum": 0.9})
    g.add_operator("x", "dp_exchange", [w, d], [o], loc, attrs={"lr": 0.1, "world": 1})
