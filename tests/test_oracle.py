"""Pin the CPU oracle: against golden vectors produced by the reference itself
(tests/golden/make_golden.py), the reference's frozen scalars
(pkg/tests/test_ops.py), and brute-force / finite-difference checks for the
extension kinds the reference does not implement."""

import math

import numpy as np
import pytest

import oracle as O
from paper_1412_6249_b200 import (Location, ParallelPlan, SyntheticFeed, build_data_parallel,
                                  build_sgd_iteration, feeder, init_params)
from paper_1412_6249_b200.builders import LayerSpec, NetSpec
from paper_1412_6249_b200.nets import cifar_convnet, conv_relu_fc, googlenet, nin


def f32(a):
    return np.asarray(a, dtype=np.float32)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(a), np.linalg.norm(b), 1e-12))


# ---------------------------------------------------------------------------
# reference golden vectors


def test_fc_matches_reference_golden(golden_ops):
    g = golden_ops
    assert np.array_equal(O.fc_forward(g["fc_x"], g["fc_w"], g["fc_b"]), g["fc_y"])
    dx, dw, db = O.fc_backward(g["fc_x"], g["fc_w"], g["fc_dy"])
    assert np.array_equal(dx, g["fc_dx"]) and np.array_equal(dw, g["fc_dw"])
    assert np.array_equal(db, g["fc_db"])


@pytest.mark.parametrize("tag", ["c1", "c2", "c3", "c4"])
def test_conv_matches_reference_golden(golden_ops, tag):
    g = golden_ops
    stride, pad = (int(v) for v in g[f"{tag}_geom"])
    y = O.conv2d_forward(g[f"{tag}_x"], g[f"{tag}_w"], g[f"{tag}_b"], stride, pad)
    assert np.allclose(y, g[f"{tag}_y"], rtol=1e-6, atol=1e-6)
    dx, dw, db = O.conv2d_backward(g[f"{tag}_x"], g[f"{tag}_w"], g[f"{tag}_dy"], stride, pad)
    for got, key in ((dx, "dx"), (dw, "dw"), (db, "db")):
        assert np.allclose(got, g[f"{tag}_{key}"], rtol=1e-6, atol=1e-6), key


def test_elementwise_match_reference_golden_bitwise(golden_ops):
    g = golden_ops
    y = O.relu_forward(g["relu_x"])
    assert np.array_equal(y.view(np.uint32), g["relu_y"].view(np.uint32))  # keeps -0.0
    assert np.array_equal(O.relu_backward(g["relu_x"], g["relu_dy"]), g["relu_dx"])
    assert np.array_equal(O.sgd_update(g["sgd_w"], g["sgd_g"], 0.0123), g["sgd_out"])
    parts = [g["agg_p0"], g["agg_p1"], g["agg_p2"]]
    assert np.array_equal(O.aggregate(parts, "mean"), g["agg_mean"])
    assert np.array_equal(O.aggregate(parts, "sum"), g["agg_sum"])
    loss, dl = O.softmax_xent(g["sm_logits"], g["sm_labels"])
    assert np.array_equal(loss, g["sm_loss"]) and np.array_equal(dl, g["sm_dlogits"])


def test_reference_frozen_scalars():
    # pkg/tests/test_ops.py:52-62, 129-135, 200-205, 235-240, 295-306
    assert O.fc_forward(f32([[1, 2]]), f32([[3], [4]]), f32([1]))[0, 0] == 12.0
    dx, dw, db = O.fc_backward(f32([[2]]), f32([[3]]), f32([[5]]))
    assert (dx[0, 0], dw[0, 0], db[0]) == (15.0, 10.0, 5.0)
    y = O.conv2d_forward(np.ones((1, 1, 3, 3), np.float32), np.ones((1, 1, 3, 3), np.float32),
                         np.zeros(1, np.float32))
    assert y.shape == (1, 1, 1, 1) and y[0, 0, 0, 0] == 9.0
    assert np.array_equal(O.relu_backward(f32([[-2, 0, 3]]), f32([[1, 1, 7]])), f32([[0, 0, 7]]))
    loss, _ = O.softmax_xent(np.zeros((2, 4), np.float32), f32([0, 3]))
    assert abs(float(loss[0]) - math.log(4.0)) < 1e-6
    assert np.allclose(O.sgd_update(f32([1, 2]), f32([0.5, 0.5]), 0.1), [0.95, 1.95])
    assert np.array_equal(O.aggregate([f32([1, 2]), f32([3, 4])], "mean"), f32([2, 3]))


def test_conv_integral_rule_and_floor_mode():
    x = np.ones((1, 1, 5, 5), np.float32)
    with pytest.raises(O.OracleError):
        O.conv2d_forward(x, np.ones((1, 1, 2, 2), np.float32), np.zeros(1, np.float32), 2, 0)
    y = O.conv2d_forward(x, np.ones((1, 1, 2, 2), np.float32), np.zeros(1, np.float32), 2, 0, True)
    assert y.shape == (1, 1, 2, 2)
    # GoogLeNet conv1 / NIN conv1 at 224 (SURVEY.md finding 3)
    assert O.conv_out_dim(224, 7, 2, 3, floor=True) == 112
    assert O.conv_out_dim(224, 11, 4, 0, floor=True) == 54
    assert [O.pool_out_dim(s, 3, 2, 0) for s in (112, 56, 28, 14)] == [56, 28, 14, 7]
    assert O.pool_out_dim(54, 3, 2, 0) == 27 and O.pool_out_dim(13, 3, 2, 0) == 6


# ---------------------------------------------------------------------------
# extension kinds (parity unpinned by the reference): brute force + FD


def _maxpool_brute(x, k, s, p):
    n, c, h, w = x.shape
    P, Q = O.pool_out_dim(h, k, s, p), O.pool_out_dim(w, k, s, p)
    y = np.zeros((n, c, P, Q), np.float32)
    m = np.zeros((n, c, P, Q), np.float32)
    for a in range(n):
        for b in range(c):
            for i in range(P):
                for j in range(Q):
                    best, arg = -np.inf, -1
                    for hh in range(max(i * s - p, 0), min(i * s - p + k, h)):
                        for ww in range(max(j * s - p, 0), min(j * s - p + k, w)):
                            if x[a, b, hh, ww] > best:
                                best, arg = x[a, b, hh, ww], hh * w + ww
                    y[a, b, i, j], m[a, b, i, j] = best, arg
    return y, m


@pytest.mark.parametrize("k,s,p,h", [(3, 2, 0, 9), (3, 1, 1, 6), (2, 2, 0, 8), (3, 2, 0, 8)])
def test_maxpool_matches_bruteforce(k, s, p, h):
    rng = np.random.default_rng(5)
    x = f32(rng.standard_normal((2, 3, h, h)))
    x[0, 0, :2, :2] = 1.5  # ties: first maximum in row-major order wins
    y, m = O.maxpool_forward(x, k, s, p)
    by, bm = _maxpool_brute(x, k, s, p)
    assert np.array_equal(y, by) and np.array_equal(m, bm)
    dy = f32(rng.standard_normal(y.shape))
    dx = O.maxpool_backward(x, m, dy)
    ref = np.zeros_like(x)
    for idx in np.ndindex(*dy.shape):
        a, b, i, j = idx
        t = int(m[idx])
        ref[a, b, t // h, t % h] += dy[idx]
    assert np.array_equal(dx, ref)


def test_avgpool_and_fd_gradient():
    rng = np.random.default_rng(6)
    x = f32(rng.uniform(-1, 1, (1, 2, 7, 7)))
    y = O.avgpool_forward(x, 7, 1)
    assert np.allclose(y[..., 0, 0], x.mean(axis=(2, 3)), atol=1e-6)
    g = f32(rng.uniform(-1, 1, (1, 2, 3, 3)))

    def loss(xx):
        return float(np.sum(O.avgpool_forward(xx, 3, 2, 0).astype(np.float64) * g))

    base = f32(rng.uniform(-1, 1, (1, 2, 7, 7)))
    dx = O.avgpool_backward(base, g, 3, 2, 0)
    num = np.zeros_like(base, dtype=np.float64)
    for idx in np.ndindex(*base.shape):
        hi, lo = base.copy(), base.copy()
        hi[idx] += 1e-2
        lo[idx] -= 1e-2
        num[idx] = (loss(hi) - loss(lo)) / 2e-2
    assert rel(dx, num) < 1e-3


def test_lrn_forward_formula_and_fd_gradient():
    rng = np.random.default_rng(7)
    x = f32(rng.uniform(-2, 2, (2, 7, 3, 3)))
    y, scale = O.lrn_forward(x, 5, 1e-2, 0.75, 1.0)
    x64 = x.astype(np.float64)
    for c in range(7):
        lo, hi = max(c - 2, 0), min(c + 2, 6)
        sc = 1.0 + 1e-2 / 5 * np.sum(x64[:, lo:hi + 1] ** 2, axis=1)
        assert np.allclose(scale[:, c], sc, rtol=1e-6)
        assert np.allclose(y[:, c], x64[:, c] * sc ** -0.75, rtol=1e-5)
    g = f32(rng.uniform(-1, 1, x.shape))
    dx = O.lrn_backward(x, y, scale, g, 5, 1e-2, 0.75, 1.0)

    def loss(xx):
        return float(np.sum(O.lrn_forward(xx, 5, 1e-2, 0.75, 1.0)[0].astype(np.float64) * g))

    num = np.zeros(x.shape)
    for idx in np.ndindex(*x.shape):
        hi, lo = x.copy(), x.copy()
        hi[idx] += 1e-2
        lo[idx] -= 1e-2
        num[idx] = (loss(hi) - loss(lo)) / 2e-2
    assert rel(dx, num) < 1e-3


def test_concat_round_trip():
    rng = np.random.default_rng(8)
    parts = [f32(rng.standard_normal((2, c, 3, 3))) for c in (1, 4, 2)]
    y = O.concat_forward(parts)
    back = O.concat_backward(y, [1, 4, 2])
    assert all(np.array_equal(a, b) for a, b in zip(parts, back))


def test_momentum_zero_is_plain_sgd_bitwise():
    rng = np.random.default_rng(9)
    w, g, v = (f32(rng.standard_normal(513)) for _ in range(3))
    w_new, v_new = O.sgd_momentum(w, g, v, 0.01, 0.0)
    assert np.array_equal(w_new, O.sgd_update(w, g, 0.01))
    w2, v2 = O.sgd_momentum(w, g, v, 0.01, 0.9)
    assert np.array_equal(v2, f32(np.float32(0.9) * v) + f32(np.float32(0.01) * g))


# ---------------------------------------------------------------------------
# whole-iteration parity of the oracle executor with the reference


def _train_oracle(seq, net, feed, seed, iters):
    from oracle.serial import run_sequence_serial

    class _S(dict):
        def set(self, name, arr):
            self[name] = np.array(arr, dtype=np.float32, copy=True)

    store = _S()
    init_params(net, store, seed, seq.layout)
    fill = feeder(feed, seq.layout)
    losses, orders = [], []
    for it in range(iters):
        fill(it, store)
        for gi, g in enumerate(seq.graphs):
            from oracle.serial import run_graph_serial
            orders.append(run_graph_serial(g, store))
            if gi == 0:
                losses.append([float(store[n][0]) for n in seq.layout.loss_names])
    return store, losses, orders


def test_oracle_cfg1_training_matches_reference(golden_train, golden_graphs):
    arrays, meta = golden_train
    net = conv_relu_fc()
    seq = build_sgd_iteration(net)
    feed = SyntheticFeed.for_net(net, 7, spread=0.0)
    store, losses, orders = _train_oracle(seq, net, feed, 7, 2)
    assert np.allclose(losses, meta["cfg1_losses"], rtol=1e-6)
    for name in seq.layout.canonical_params:
        assert np.allclose(store[name], arrays[f"cfg1_{name}"], rtol=1e-6, atol=1e-7), name
    assert orders[:2] == golden_graphs["cfg1"]["serial"]


@pytest.mark.parametrize("split", [False, True])
def test_oracle_mlp_dp_matches_reference(golden_train, golden_graphs, split):
    arrays, meta = golden_train
    tag = f"mlp_dp2_{'split' if split else 'fused'}"
    net = NetSpec((20,), (LayerSpec("fc", 16), LayerSpec("relu"), LayerSpec("fc", 4)), batch=8,
                  lr=0.05)
    plan = ParallelPlan("data", peers=(Location("local", 0), Location("local", 1)),
                        server=Location("local", 2))
    seq = build_data_parallel(net, plan, split_backward=split)
    store, losses, orders = _train_oracle(seq, net, SyntheticFeed.for_net(net, 13, peers=2), 13, 3)
    assert losses == meta[f"{tag}_losses"]
    for name in seq.layout.canonical_params:
        assert np.array_equal(store[name], arrays[f"{tag}_{name}"]), name
    assert orders[:2] == golden_graphs[tag]["serial"]


def test_oracle_cfg2_dp_matches_reference_dispatcher(golden_train, golden_graphs):
    arrays, meta = golden_train
    net = cifar_convnet(batch=16, lr=1e-3)
    plan = ParallelPlan("data", peers=(Location("local", 0), Location("local", 1)),
                        server=Location("local", 2))
    seq = build_data_parallel(net, plan)
    feed = SyntheticFeed.for_net(net, 7, peers=2, spread=0.0)
    store, losses, orders = _train_oracle(seq, net, feed, 7, 2)
    assert losses == meta["cfg2_dp2_losses"]
    for name in seq.layout.canonical_params:
        assert np.array_equal(store[name], arrays[f"cfg2_dp2_{name}"]), name
    assert orders[:2] == golden_graphs["cfg2_dp2"]["serial"]


def test_network_sizes_match_survey():
    g = googlenet(batch=1)
    macs = g.macs_per_image()
    assert abs((macs["conv"] + macs["fc"]) / 1e9 - 1.583) < 2e-3
    assert len(g.param_shapes()) == 116
    assert sum(math.prod(s) for _, s in g.param_shapes()) == 6998552
    n = nin(batch=1)
    assert abs(n.macs_per_image()["conv"] / 1e9 - 1.100) < 2e-3
