"""The lowered data-parallel exchange (exchange.py) as product code at world 2
on one GPU, with and without momentum.

`LocalGroup` runs each rank's partition from its own host thread against
its own TensorStore on cuda:0; reduce-scatter / all-gather are this
library's rank-ordered aggregate and copy kernels, so both ranks must equal
the reference-shaped parameter-server graph (builders.py:543-647: up_
copies -> agg_ mean in rank order -> upd_ -> down_ copies) bit for bit, and
the reference's own 2-peer config-2 training results (golden) within the NS
tolerance.  The rank>0 offsets of `_dp_exchange` (shard = rank * flat_len /
world) and the velocity shards run here exactly as they do over NCCL."""

import threading

import numpy as np
import pytest
import torch

from gpu_util import ATOL, RTOL, assert_close
from paper_1412_6249_b200 import (Location, ParallelPlan, SyntheticFeed, TensorStore,
                                  build_data_parallel, feeder, init_params, run_sequence)
from paper_1412_6249_b200.exchange import LocalGroup, build_rank_sequence
from paper_1412_6249_b200.nets import cifar_convnet, googlenet

pytestmark = pytest.mark.gpu


def _plan(n):
    return ParallelPlan("data", peers=tuple(Location("local", k) for k in range(n)),
                        server=Location("local", n))


def _server_graph(net, feed, world, iters):
    seq = build_data_parallel(net, _plan(world))
    st = TensorStore("cuda:0")
    init_params(net, st, 7, seq.layout)
    run_sequence(seq, st, before_iteration=feeder(feed, seq.layout), iterations=iters, trace=False)
    return st


def _lowered_ranks(net, feed, world, iters, bucket_bytes=64 << 10):
    group = LocalGroup(world)
    stores, errors = [None] * world, []

    def rank_main(rank):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                st = TensorStore("cuda:0")
                seq, _ = build_rank_sequence(net, world, rank, st, bucket_bytes=bucket_bytes,
                                             nccl=False)
                st._collective = group.member(rank)
                init_params(net, st, 7, seq.layout)
                run_sequence(seq, st, before_iteration=feeder(feed, seq.layout),
                             iterations=iters, trace=False)
                torch.cuda.synchronize()
                stores[rank] = st
        except BaseException as exc:  # noqa: BLE001 - re-raised below
            errors.append(exc)

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(600)
    if errors:
        raise errors[0]
    return stores


@pytest.mark.parametrize("momentum", [0.0, 0.9])
@pytest.mark.parametrize("world", [2, 3])
def test_local_group_ranks_equal_the_server_graph(world, momentum):
    net = cifar_convnet(batch=4, lr=0.01, momentum=momentum)
    feed = SyntheticFeed.for_net(net, 7, peers=world, spread=0.0)
    iters = 3
    full = _server_graph(net, feed, world, iters)
    ranks = _lowered_ranks(net, feed, world, iters)
    for pname, _ in net.param_shapes():
        want = full.array(pname)
        for r, st in enumerate(ranks):
            assert np.array_equal(st.array(f"{pname}_p{r}"), want), (pname, r)
    if momentum:  # every rank's velocity shards are the server's velocity, sliced
        for r, st in enumerate(ranks):
            assert any(n.startswith("vxch_") for n in st.names())


def test_local_group_world2_matches_reference_cfg2(golden_train):
    """Config 2 (2 replicas + parameter aggregation) through the lowered
    world-2 product path reproduces the reference's own training results."""
    arrays, meta = golden_train
    net = cifar_convnet(batch=16, lr=1e-3)
    feed = SyntheticFeed.for_net(net, 7, peers=2, spread=0.0)
    ranks = _lowered_ranks(net, feed, 2, 2)
    for name, _ in net.param_shapes():
        for r, st in enumerate(ranks):
            assert_close(st.array(f"{name}_p{r}"), arrays[f"cfg2_dp2_{name}"], rtol=RTOL, atol=ATOL,
                         what=f"{name} rank {r}")
    losses = [float(st.array(f"loss_p{r}")[0]) for r, st in enumerate(ranks)]
    assert np.allclose(losses, meta["cfg2_dp2_losses"][-1], rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("momentum", [0.0, 0.9])
def test_lowered_world1_momentum_bitwise_and_captured(momentum):
    """World 1: the lowered exchange with momentum is bitwise the server
    graph's sgd_momentum (+ velocity swaps), eagerly and from captured CUDA
    graphs (velocity shards ping-pong like the parameters)."""
    from paper_1412_6249_b200.executor import CapturedSequence

    net = cifar_convnet(batch=2, lr=0.01, momentum=momentum)
    feed = SyntheticFeed.for_net(net, 7, spread=0.0)
    fixed = lambda seq: (lambda it, s: feeder(feed, seq.layout)(0, s))  # noqa: E731
    full_seq = build_data_parallel(net, _plan(1))
    full = TensorStore("cuda:0")
    init_params(net, full, 7, full_seq.layout)
    run_sequence(full_seq, full, before_iteration=fixed(full_seq), iterations=4, trace=False)
    st = TensorStore("cuda:0")
    seq, _ = build_rank_sequence(net, 1, 0, st, bucket_bytes=32 << 10)
    assert bool(seq.layout.velocity_params) == (momentum > 0)
    init_params(net, st, 7, seq.layout)
    feeder(feed, seq.layout)(0, st)
    exe = CapturedSequence(seq, st)
    exe.prepare()  # one eager iteration
    for _ in range(3):
        exe.step()
    for pname, _ in net.param_shapes():
        assert np.array_equal(st.array(f"{pname}_p0"), full.array(pname)), pname
    if momentum:
        torch.cuda.synchronize()
        v_full = np.concatenate([full.array(f"v{p}").ravel() for p, _ in net.param_shapes()])
        v_low = np.concatenate([st.array(v).ravel() for v in seq.layout.velocity_params])
        assert np.count_nonzero(v_low) == np.count_nonzero(v_full)
        assert np.array_equal(np.sort(v_low[v_low != 0]), np.sort(v_full[v_full != 0]))


def test_googlenet_lowered_world2_equals_server_graph():
    """GoogLeNet (116 parameter tensors, multi-MB buckets) at world 2: both
    ranks equal the server graph bit for bit after 2 iterations."""
    net = googlenet(batch=2, lr=0.01, momentum=0.9)
    feed = SyntheticFeed.for_net(net, 7, peers=2, spread=0.0)
    full = _server_graph(net, feed, 2, 2)
    ranks = _lowered_ranks(net, feed, 2, 2, bucket_bytes=4 << 20)
    for pname, _ in net.param_shapes():
        want = full.array(pname)
        for r, st in enumerate(ranks):
            assert np.array_equal(st.array(f"{pname}_p{r}"), want), (pname, r)
