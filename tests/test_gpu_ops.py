"""Per-operator parity of the sm_100a kernels with the CPU oracle, through the
product boundary.  Bit-exact for the integer/elementwise/pooling kinds,
rel 1e-4 / abs 1e-5 (the NS tolerance) for the contractions."""

import numpy as np
import pytest

import oracle as O
from gpu_util import ATOL, RTOL, assert_bitwise, assert_close, run_op

pytestmark = pytest.mark.gpu


def f32(a):
    return np.asarray(a, dtype=np.float32)


RNG = np.random.default_rng(1234)


def rnd(*shape, scale=1.0):
    return f32(RNG.standard_normal(shape) * scale)


# ---------------------------------------------------------------------------
# contractions


CONV_CASES = [
    # (N, C, H, W, K, R, stride, pad, floor)
    (2, 3, 9, 9, 4, 3, 1, 1, False),
    (2, 5, 8, 8, 6, 1, 1, 0, False),
    (1, 2, 11, 11, 3, 5, 2, 2, False),
    (3, 4, 7, 7, 5, 5, 1, 2, False),
    (2, 3, 32, 32, 32, 5, 1, 2, False),          # config 1
    (2, 3, 224, 224, 64, 7, 2, 3, True),          # GoogLeNet conv1 (floor mode)
    (2, 64, 56, 56, 192, 3, 1, 1, False),         # GoogLeNet conv2/3x3
    (2, 192, 28, 28, 64, 1, 1, 0, False),         # inception 3a 1x1
    (2, 16, 28, 28, 32, 5, 1, 2, False),          # inception 3a 5x5
    (2, 832, 7, 7, 384, 1, 1, 0, False),          # inception 5b 1x1
    (2, 160, 7, 7, 320, 3, 1, 1, False),          # inception 5a 3x3
    (1, 3, 224, 224, 96, 11, 4, 0, True),         # NIN conv1
    (2, 3, 13, 13, 8, 3, 2, 1, False),            # strided dgrad
    (2, 96, 14, 14, 208, 3, 1, 1, False),         # inception 4a 3x3 (dgrad: 208 = 6.5 blocks)
    (4, 48, 7, 7, 128, 5, 1, 2, False),           # inception 5b 5x5 (partial channel block)
    (3, 480, 14, 14, 208, 1, 1, 0, False),        # 1x1, two pixel tiles per image
    (2, 20, 6, 6, 40, 1, 1, 0, False),            # 1x1, partial channel block, tiny image
    (2, 256, 28, 28, 384, 1, 1, 0, False),        # 1x1, two output-channel tiles
    (2, 5, 19, 17, 24, 7, 1, 3, False),           # 7x7 stride 1 on 5 channels
    (1, 2, 16, 16, 40, 8, 3, 2, False),           # 8x8 stride 3
    (2, 8, 32, 32, 256, 3, 1, 1, False),          # TMA-streamed dY wgrad, two dY tiles
    (3, 4, 32, 32, 16, 5, 2, 2, True),            # transposed wgrad (gemm_wgrad_t.cu), Q = 16
    (2, 3, 36, 36, 64, 7, 2, 3, True),            # conv1 geometry small: Q = 18, 2 q-blocks
    (2, 3, 300, 300, 32, 7, 2, 3, True),          # window forward (gemm_fwd_win.cu): 2 tiles per row
    (2, 3, 20, 24, 48, 3, 1, 1, False),           # window forward, stride 1, K = 48
]


@pytest.fixture(params=[0, 3, 4, 5, 6, 7, 8],
                ids=["auto", "halo-v3", "no-tma-1x1", "no-tma-wgrad", "reg-prefetch",
                     "tma-dy-wgrad", "s2d"])
def gemm_engine(request, monkeypatch):
    """0 = default engine choice (1x1 convolutions through the TMA-fed engine
    v4, gemm_tc4.cu); 3 = also route stride-1 R x S convolutions through the
    opt-in halo-staged engine v3 (gemm_tc3.cu); 4 = 1x1 convolutions through
    the gathering engine v2 instead of v4; 5 = 1x1 weight gradients gathered
    instead of TMA-fed; 6 = engine v2 gathers prefetched in registers instead
    of cp.async-staged; 7 = also stream the raw dY by TMA for 16-aligned-row
    weight gradients (conv1 type, opt-in mode kWgradTma); 8 = engine 0 with
    strided convolutions through the opt-in space-to-depth view
    (PURINE_B200_S2D=1, conv_s2d.cu)."""
    from paper_1412_6249_b200 import _native

    lib = _native.lib()
    if request.param == 8:
        monkeypatch.setenv("PURINE_B200_S2D", "1")
    lib("bf_set_gemm_engine", 0 if request.param == 8 else request.param)
    yield request.param
    lib("bf_set_gemm_engine", 0)


@pytest.mark.parametrize("case", CONV_CASES, ids=lambda c: "x".join(map(str, c[:7])))
def test_conv_forward_backward(case, gemm_engine):
    n, c, h, w, k, r, s, p, fl = case
    if gemm_engine == 3 and not (s == 1 and r > 1):
        pytest.skip("engine v3 only takes stride-1 spatial filters")
    if gemm_engine in (4, 5) and r != 1:
        pytest.skip("engine switches 4 and 5 only change 1x1 convolutions")
    if gemm_engine == 8 and not (s >= 2 and r > s and c * s * s <= 64):
        pytest.skip("the space-to-depth view only takes strided convolutions on few channels")
    x = rnd(n, c, h, w)
    wt = rnd(k, c, r, r, scale=1.0 / np.sqrt(c * r * r))
    b = rnd(k)
    attrs = {"stride": s, "pad": p}
    if fl:
        attrs["floor"] = True
    # NS tolerance rel 1e-4 / abs 1e-5, the absolute part relative to the
    # output's largest magnitude: these accumulate O(1000) unit-scale products,
    # so a near-cancelling element carries an absolute error set by its
    # neighbours' scale, not its own (same rule for every contraction output)
    def close(got, want, what):
        assert_close(got, want, rtol=RTOL, atol=ATOL * max(1.0, float(np.abs(want).max())),
                     what=what)

    y_ref = O.conv2d_forward(x, wt, b, s, p, fl)
    got = run_op("conv2d_forward", {"x": x, "w": wt, "b": b}, {"y": y_ref.shape}, attrs)["y"]
    close(got, y_ref, "conv fwd")
    dy = rnd(*y_ref.shape)
    dx_ref, dw_ref, db_ref = O.conv2d_backward(x, wt, dy, s, p, fl)
    outs = run_op("conv2d_backward", {"x": x, "w": wt, "dy": dy},
                  {"dx": x.shape, "dw": wt.shape, "db": (k,)}, attrs)
    close(outs["dx"], dx_ref, "conv dgrad")
    close(outs["dw"], dw_ref, "conv wgrad")
    close(outs["db"], db_ref, "conv bgrad")


@pytest.mark.parametrize("shape", [(4, 64, 56, 56, 64), (2, 192, 28, 28, 16), (3, 480, 14, 14, 208),
                                   (2, 20, 6, 6, 40), (2, 256, 28, 28, 384), (2, 832, 7, 7, 128),
                                   (1, 300, 4, 4, 200)])
@pytest.mark.parametrize("engine", [0, 5], ids=["tma-wgrad", "gather-wgrad"])
def test_conv1x1_weight_bias_gradient(shape, engine):
    """bf_conv2d_bwd_weight_bias on 1x1 layers: the TMA-fed weight gradient
    (kTma1x1, bias from the same dy tiles) and the gather + dY-pack path."""
    import torch
    from paper_1412_6249_b200 import _native

    n, c, h, w, k = shape
    lib = _native.lib()
    x, dy = rnd(n, c, h, w), rnd(n, k, h, w)
    _, dw_ref, db_ref = O.conv2d_backward(x, rnd(k, c, 1, 1), dy, 1, 0, False)
    dev = torch.device("cuda:0")
    tx, tdy = torch.from_numpy(x).to(dev), torch.from_numpy(dy).to(dev)
    dw = torch.empty(k, c, 1, 1, device=dev)
    db = torch.empty(k, device=dev)
    ws = torch.empty(64 << 20, device=dev)
    lib("bf_set_gemm_engine", engine)
    try:
        lib("bf_conv2d_bwd_weight_bias", tx.data_ptr(), tdy.data_ptr(), dw.data_ptr(),
            db.data_ptr(), n, c, h, w, k, 1, 1, h, w, 1, 0, ws.data_ptr(), ws.numel() * 4, None)
        torch.cuda.synchronize()
    finally:
        lib("bf_set_gemm_engine", 0)
    for got, want, what in ((dw.cpu().numpy(), dw_ref, "dw"), (db.cpu().numpy(), db_ref, "db")):
        assert_close(got, want, rtol=RTOL, atol=ATOL * max(1.0, float(np.abs(want).max())),
                     what=what)


@pytest.mark.parametrize("n,d,m", [(16, 32768, 10), (128, 1024, 1000), (6, 20, 7), (3, 5, 2)])
def test_fc_forward_backward(n, d, m):
    # dy at the scale of a softmax gradient ((p - onehot) / n, ops.py:418)
    x, w, b, dy = rnd(n, d), rnd(d, m, scale=1 / np.sqrt(d)), rnd(m), rnd(n, m, scale=1.0 / n)
    assert_close(run_op("fc_forward", {"x": x, "w": w, "b": b}, {"y": (n, m)})["y"],
                 O.fc_forward(x, w, b), what="fc fwd")
    dx, dw, db = O.fc_backward(x, w, dy)
    out = run_op("fc_backward", {"x": x, "w": w, "dy": dy},
                 {"dx": (n, d), "dw": (d, m), "db": (m,)})
    # absolute tolerance scaled by the output's magnitude (accumulations of
    # O(1) products, as for conv wgrad above)
    for key, want in (("dx", dx), ("dw", dw), ("db", db)):
        assert_close(out[key], want, rtol=RTOL, atol=ATOL * max(1.0, float(np.abs(want).max())),
                     what=f"fc {key}")


def test_reference_golden_vectors_on_gpu(golden_ops):
    g = golden_ops
    y = run_op("fc_forward", {"x": g["fc_x"], "w": g["fc_w"], "b": g["fc_b"]}, {"y": g["fc_y"].shape})
    assert_close(y["y"], g["fc_y"])
    for tag in ("c1", "c2", "c3", "c4"):
        s, p = (int(v) for v in g[f"{tag}_geom"])
        out = run_op("conv2d_forward", {"x": g[f"{tag}_x"], "w": g[f"{tag}_w"], "b": g[f"{tag}_b"]},
                     {"y": g[f"{tag}_y"].shape}, {"stride": s, "pad": p})
        assert_close(out["y"], g[f"{tag}_y"], what=tag)


# ---------------------------------------------------------------------------
# elementwise / pooling / normalisation: bit-exact


def test_relu_bitwise(golden_ops):
    x = golden_ops["relu_x"]
    assert_bitwise(run_op("relu_forward", {"x": x}, {"y": x.shape})["y"], golden_ops["relu_y"])
    x = rnd(3, 7, 5, 5)
    x[0, 0, 0, :3] = [0.0, -0.0, 1e-38]
    dy = rnd(3, 7, 5, 5)
    assert_bitwise(run_op("relu_forward", {"x": x}, {"y": x.shape})["y"], O.relu_forward(x))
    assert_bitwise(run_op("relu_backward", {"x": x, "dy": dy}, {"dx": x.shape})["dx"],
                   O.relu_backward(x, dy))


def test_relu_nan_propagates_like_numpy(monkeypatch):
    """np.maximum(NaN, 0) is NaN (ops.py:361); the backward's where(x > 0)
    drops it.  The dispatcher's non-finite check is off so the raw values show."""
    monkeypatch.setenv("PURINE_B200_CHECK_FINITE", "0")
    x = rnd(2, 3, 4, 4)
    x[0, 0, 0, :4] = [np.nan, -np.nan, np.inf, -np.inf]
    dy = rnd(2, 3, 4, 4)
    y = run_op("relu_forward", {"x": x}, {"y": x.shape})["y"]
    want = O.relu_forward(x)
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(y), nan)  # NaN payloads are not part of the contract
    assert_bitwise(np.where(nan, 0, y), np.where(nan, 0, want))
    assert_bitwise(run_op("relu_backward", {"x": x, "dy": dy}, {"dx": x.shape})["dx"],
                   O.relu_backward(x, dy))


def test_sgd_momentum_aggregate_bitwise(golden_ops):
    g = golden_ops
    out = run_op("sgd_update", {"w": g["sgd_w"], "g": g["sgd_g"]}, {"o": g["sgd_w"].shape},
                 {"lr": 0.0123})["o"]
    assert_bitwise(out, g["sgd_out"])
    parts = {f"p{i}": g[f"agg_p{i}"] for i in range(3)}
    assert_bitwise(run_op("aggregate", parts, {"o": (777,)}, {"mode": "mean"})["o"], g["agg_mean"])
    assert_bitwise(run_op("aggregate", parts, {"o": (777,)}, {"mode": "sum"})["o"], g["agg_sum"])
    w, gg, v = rnd(1003), rnd(1003), rnd(1003)
    for mu in (0.0, 0.9):
        out = run_op("sgd_momentum", {"w": w, "g": gg, "v": v}, {"wn": w.shape, "vn": w.shape},
                     {"lr": 0.01, "momentum": mu})
        wn, vn = O.sgd_momentum(w, gg, v, 0.01, mu)
        assert_bitwise(out["wn"], wn)
        assert_bitwise(out["vn"], vn)


@pytest.mark.parametrize("shape,k,s,p", [((2, 3, 9, 9), 3, 2, 0), ((2, 64, 112, 112), 3, 2, 0),
                                         ((2, 192, 28, 28), 3, 1, 1), ((2, 832, 14, 14), 3, 2, 0),
                                         ((2, 4, 8, 8), 2, 2, 0), ((1, 96, 54, 54), 3, 2, 0),
                                         ((2, 5, 11, 13), 3, 2, 1), ((2, 8, 14, 14), 3, 2, 1),
                                         ((1, 2, 6, 7), 3, 2, 0), ((3, 7, 5, 5), 3, 1, 1),
                                         ((2, 3, 6, 7), 3, 1, 0), ((2, 64, 7, 7), 3, 1, 1),
                                         ((2, 16, 14, 14), 3, 1, 1), ((1, 3, 9, 32), 3, 1, 1),
                                         ((1, 3, 6, 33), 3, 1, 1), ((3, 5, 4, 1), 3, 1, 1)])
@pytest.mark.parametrize("walkers", ["63", "15", "7", "0"],
                         ids=["staged", "rows", "columns", "planes"])
@pytest.mark.parametrize("values", ["normal", "coarse"])
def test_maxpool_bitwise(shape, k, s, p, walkers, values, monkeypatch):
    """Bulk-staged 3x3 forward and mask-reading backward (default where they
    fit), warp-row kernels (stride-1 pad-1 planes <= 32 wide), column walkers
    and plane-staging kernels (PURINE_B200_POOL_WALKERS=63 / 15 / 7 / 0) all
    bit-exact.  "coarse" values make most
    windows hold ties (first maximum in raster order wins) and put a -inf
    block in the corner."""
    monkeypatch.setenv("PURINE_B200_POOL_WALKERS", walkers)
    x = rnd(*shape)
    x[:, :, ::3, ::3] = 0.5  # ties across windows
    if values == "coarse":
        x = f32(np.round(x))
        x[:, :, :3, :3] = -3e38
    y, m = O.maxpool_forward(x, k, s, p)
    out = run_op("maxpool_forward", {"x": x}, {"y": y.shape, "m": y.shape},
                 {"kernel": k, "stride": s, "pad": p})
    assert_bitwise(out["y"], y, "maxpool y")
    assert_bitwise(out["m"], m, "maxpool argmax")
    dy = rnd(*y.shape)
    dx = run_op("maxpool_backward", {"x": x, "m": m, "dy": dy}, {"dx": x.shape},
                {"kernel": k, "stride": s, "pad": p})["dx"]
    assert_bitwise(dx, O.maxpool_backward(x, m, dy), "maxpool dx")


MAXPOOL_STAGED_SHAPES = [((2, 64, 112, 112), 3, 2, 0), ((2, 192, 56, 56), 3, 2, 0),
                         ((2, 192, 28, 28), 3, 1, 1), ((3, 480, 28, 28), 3, 2, 0),
                         ((2, 832, 14, 14), 3, 2, 0), ((2, 528, 14, 14), 3, 1, 1),
                         ((4, 832, 7, 7), 3, 1, 1), ((2, 8, 14, 14), 3, 2, 1),
                         ((2, 5, 11, 13), 3, 2, 1), ((4, 7, 5, 5), 3, 1, 1),
                         ((2, 6, 6, 7), 3, 1, 0), ((4, 3, 9, 33), 3, 1, 1),
                         ((1, 96, 54, 54), 3, 2, 0), ((4, 6, 6, 7), 3, 2, 0)]


@pytest.mark.parametrize("shape,k,s,p", MAXPOOL_STAGED_SHAPES)
@pytest.mark.parametrize("fold", [False, True], ids=["pool", "relu+pool"])
@pytest.mark.parametrize("values", ["normal", "coarse"])
@pytest.mark.parametrize("s1_bwd", ["0", "1"], ids=["default", "s1-staged"])
@pytest.mark.parametrize("smask", ["1", "0"], ids=["signed-mask", "recompute"])
def test_maxpool_staged_mask_elided_bitwise(shape, k, s, p, fold, values, s1_bwd, smask,
                                            monkeypatch):
    """The product pairing: maxpool_forward and maxpool_backward in one graph,
    the float mask elided -- the forward writes a signed mask (each window's
    argmax carrying the sign of its maximum) that the backward gathers from, or
    (smask off) the backward recomputes each argmax from x with the forward's scan --
    and, after a ReLU, the relu_backward folded in through the pool's own
    input.  y, dx (or the folded da) bit-exact vs the oracle."""
    from paper_1412_6249_b200 import BiGraph, Location, TensorStore, run
    from paper_1412_6249_b200._native import lib
    from paper_1412_6249_b200.dispatcher import _plan

    monkeypatch.setenv("PURINE_B200_POOL_STAGED", s1_bwd)  # 1: stride-1 backward staged too
    monkeypatch.setenv("PURINE_B200_POOL_SMASK", smask)
    loc = Location("local", 0)
    a = rnd(*shape)
    a[:, :, ::3, ::3] = 0.5
    if values == "coarse":
        a = f32(np.round(a))
        a[:, :, :3, :3] = -3e38
    x = O.relu_forward(a) if fold else a
    y, m = O.maxpool_forward(x, k, s, p)
    dy = rnd(*y.shape)
    dx = O.maxpool_backward(x, m, dy)
    attrs = {"kernel": k, "stride": s, "pad": p}
    g = BiGraph()
    tx = g.add_tensor("x", shape, loc)
    if fold:
        ta = g.add_tensor("a", shape, loc)
        g.add_operator("relu", "relu_forward", [ta], [tx], loc)
    ty, tm = g.add_tensor("y", y.shape, loc), g.add_tensor("m", y.shape, loc)
    tdy, tdx = g.add_tensor("dy", y.shape, loc), g.add_tensor("dx", shape, loc)
    g.add_operator("pool", "maxpool_forward", [tx], [ty, tm], loc, attrs=attrs)
    g.add_operator("bwd_pool", "maxpool_backward", [tx, tm, tdy], [tdx], loc, attrs=attrs)
    if fold:
        tda = g.add_tensor("da", shape, loc)
        g.add_operator("bwd_relu", "relu_backward", [ta, tdx], [tda], loc)
    n, c, h, w = shape
    # the mask is elided where the backward also absorbs the ReLU backward
    # through x (fold); otherwise the staged backward reads the mask
    ok = lib().raw("bf_maxpool_staged_ok")
    staged = fold and bool(ok(n, c, h, w, y.shape[2], y.shape[3], k, s, p, 1) or
                           (smask == "1" and ok(n, c, h, w, y.shape[2], y.shape[3], k, s, p, 3)))
    plan = _plan(g, 8)
    assert ("m" in plan.elided) == staged
    st = TensorStore("cuda:0")
    st.set("a" if fold else "x", a)
    st.set("dy", dy)
    run(g, st)
    assert_bitwise(st.array("y"), y, "maxpool y")
    if fold:
        assert_bitwise(st.array("da"), O.relu_backward(a, dx), "relu+maxpool da")
        assert ("dx" in plan.elided) == staged
    else:
        assert_bitwise(st.array("dx"), dx, "maxpool dx")
    if staged:
        assert not st.has("m")  # never materialised


@pytest.mark.parametrize("couts,shape", [((64, 96, 16), (2, 192, 28, 28)),
                                          ((128, 128, 32), (2, 256, 28, 28)),
                                          ((160, 112, 24), (3, 512, 14, 14)),
                                          ((40, 8), (2, 20, 6, 6))])
def test_conv1x1_group_forward(couts, shape, monkeypatch):
    """Inception's sibling 1x1 convolutions over one x as one GEMM (dispatcher
    _Plan._group_1x1, bf_conv1x1_fwd_group): every member's output and fused
    ReLU -- one into a concat slice -- within the NS bound of the oracle and of
    the ungrouped kernels."""
    from paper_1412_6249_b200 import BiGraph, Location, TensorStore, run
    from paper_1412_6249_b200.dispatcher import _plan

    loc = Location("local", 0)
    n, c, h, w = shape
    rng = np.random.default_rng(5)
    x = f32(rng.standard_normal(shape))
    ws = [f32(rng.standard_normal((k, c, 1, 1)) / np.sqrt(c)) for k in couts]
    bs = [f32(rng.standard_normal(k) * 0.1) for k in couts]

    def graph():
        g = BiGraph()
        tx = g.add_tensor("x", shape, loc)
        cat_parts = []
        for i, k in enumerate(couts):
            tw = g.add_tensor(f"w{i}", (k, c, 1, 1), loc)
            tb = g.add_tensor(f"b{i}", (k,), loc)
            ty = g.add_tensor(f"y{i}", (n, k, h, w), loc)
            tr = g.add_tensor(f"r{i}", (n, k, h, w), loc)
            g.add_operator(f"conv{i}", "conv2d_forward", [tx, tw, tb], [ty], loc,
                           attrs={"stride": 1, "pad": 0})
            g.add_operator(f"relu{i}", "relu_forward", [ty], [tr], loc)
            if i == 0:
                cat_parts.append(tr)
        # the first branch's ReLU goes straight into a concat (elided slice)
        other = g.add_tensor("other", (n, 8, h, w), loc)
        cat = g.add_tensor("cat", (n, couts[0] + 8, h, w), loc)
        g.add_operator("bias_other", "relu_forward", [g.add_tensor("o_in", (n, 8, h, w), loc)],
                       [other], loc)
        g.add_operator("concat", "concat_forward", cat_parts + [other], [cat], loc)
        return g

    outs = {}
    monkeypatch.setenv("PURINE_B200_PREACT_ELISION", "0")  # y0.. are compared too
    for flag in ("1", "0"):
        monkeypatch.setenv("PURINE_B200_GROUP_1X1", flag)
        g = graph()
        plan = _plan(g, 8)
        grouped = any("group_fwd" in f for f in plan.fusion.values())
        assert grouped == (flag == "1")
        st = TensorStore("cuda:0")
        st.set("x", x)
        st.set("o_in", f32(rng.standard_normal((n, 8, h, w))))
        for i in range(len(couts)):
            st.set(f"w{i}", ws[i])
            st.set(f"b{i}", bs[i])
        run(g, st)
        outs[flag] = {nm: st.array(nm) for nm in
                      [f"y{i}" for i in range(len(couts))] +
                      [f"r{i}" for i in range(1, len(couts))] + ["cat"]}
    for i, k in enumerate(couts):
        want = O.conv2d_forward(x, ws[i], bs[i], 1, 0)
        assert_close(outs["1"][f"y{i}"], want, what=f"y{i} vs oracle")
        assert_close(outs["1"][f"y{i}"], outs["0"][f"y{i}"], what=f"y{i} grouped vs not")
        if i:
            assert_bitwise(outs["1"][f"r{i}"], O.relu_forward(outs["1"][f"y{i}"]))
    assert_bitwise(outs["1"]["cat"][:, :couts[0]], O.relu_forward(outs["1"]["y0"]))


@pytest.mark.parametrize("shape,k,s,p", [((2, 1024, 7, 7), 7, 1, 0), ((2, 5, 9, 9), 3, 2, 1),
                                         ((2, 1000, 6, 6), 6, 1, 0)])
def test_avgpool_bitwise(shape, k, s, p):
    x = rnd(*shape)
    y = O.avgpool_forward(x, k, s, p)
    got = run_op("avgpool_forward", {"x": x}, {"y": y.shape}, {"kernel": k, "stride": s, "pad": p})
    assert_bitwise(got["y"], y)
    dy = rnd(*y.shape)
    dx = run_op("avgpool_backward", {"x": x, "dy": dy}, {"dx": x.shape},
                {"kernel": k, "stride": s, "pad": p})["dx"]
    assert_bitwise(dx, O.avgpool_backward(x, dy, k, s, p))


@pytest.mark.parametrize("shape", [(2, 64, 56, 56), (2, 7, 5, 5), (1, 2, 4, 4), (3, 4, 2, 2),
                                   (1, 40, 6, 6), (2, 37, 3, 5)])
def test_lrn(shape):
    x = rnd(*shape, scale=3.0)
    y, sc = O.lrn_forward(x)
    out = run_op("lrn_forward", {"x": x}, {"y": shape, "s": shape},
                 {"size": 5, "alpha": 1e-4, "beta": 0.75, "k": 1.0})
    assert_bitwise(out["s"], sc, "lrn scale")
    assert_close(out["y"], y, rtol=1e-6, atol=1e-7, what="lrn y")
    dy = rnd(*shape)
    dx = run_op("lrn_backward", {"x": x, "y": y, "s": sc, "dy": dy}, {"dx": shape},
                {"size": 5, "alpha": 1e-4, "beta": 0.75, "k": 1.0})["dx"]
    assert_close(dx, O.lrn_backward(x, y, sc, dy), rtol=1e-5, atol=1e-6, what="lrn dx")


@pytest.mark.parametrize("shape", [(2, 64, 56, 56), (2, 7, 5, 5), (1, 2, 4, 4), (3, 4, 2, 2),
                                   (1, 40, 6, 6), (2, 37, 3, 5), (2, 192, 14, 14)])
@pytest.mark.parametrize("relu", [False, True])
def test_lrn_recompute_backward_bitwise(shape, relu):
    """Graph-plan LRN pair (scale elided): the forward without scale stores the
    same y, and the backward recomputing scale and y from x is bit-identical to
    the explicit backward fed the forward's outputs (with and without the
    folded ReLU mask); both within tolerance of the oracle."""
    import torch
    from paper_1412_6249_b200 import _native

    lib = _native.lib()
    dev = torch.device("cuda:0")
    x = torch.from_numpy(rnd(*shape, scale=3.0)).to(dev)
    dy = torch.from_numpy(rnd(*shape)).to(dev)
    rx = torch.from_numpy(rnd(*shape)).to(dev) if relu else None
    y, sc, y2 = (torch.empty_like(x) for _ in range(3))
    a = (5, 1e-4, 0.75, 1.0)
    lib("bf_lrn_fwd", x.data_ptr(), y.data_ptr(), sc.data_ptr(), *shape, *a, None)
    lib("bf_lrn_fwd", x.data_ptr(), y2.data_ptr(), None, *shape, *a, None)
    dx, dx2 = torch.empty_like(x), torch.empty_like(x)
    if relu:
        lib("bf_lrn_bwd_relu", x.data_ptr(), y.data_ptr(), sc.data_ptr(), dy.data_ptr(),
            dx.data_ptr(), rx.data_ptr(), *shape, *a, None)
    else:
        lib("bf_lrn_bwd", x.data_ptr(), y.data_ptr(), sc.data_ptr(), dy.data_ptr(), dx.data_ptr(),
            *shape, *a, None)
    lib("bf_lrn_bwd_recompute", x.data_ptr(), dy.data_ptr(), dx2.data_ptr(),
        rx.data_ptr() if relu else None, *shape, *a, None)
    torch.cuda.synchronize()
    assert_bitwise(y2.cpu().numpy(), y.cpu().numpy(), "lrn y without scale")
    assert_bitwise(dx2.cpu().numpy(), dx.cpu().numpy(), "lrn recompute dx")
    xn, dyn = x.cpu().numpy(), dy.cpu().numpy()
    want = O.lrn_backward(xn, y.cpu().numpy(), sc.cpu().numpy(), dyn)
    if relu:
        want = O.relu_backward(rx.cpu().numpy(), want)
    assert_close(dx2.cpu().numpy(), want, rtol=1e-5, atol=1e-6, what="lrn recompute vs oracle")


def test_concat_bitwise():
    parts = {f"p{i}": rnd(2, c, 7, 7) for i, c in enumerate((64, 128, 32, 32))}
    y = O.concat_forward(list(parts.values()))
    assert_bitwise(run_op("concat_forward", parts, {"y": y.shape})["y"], y)
    back = run_op("concat_backward", {"dy": y}, {f"g{i}": p.shape for i, p in enumerate(parts.values())},
                  {"channels": [64, 128, 32, 32]})
    for i, p in enumerate(parts.values()):
        assert_bitwise(back[f"g{i}"], p)


def test_softmax_xent(golden_ops):
    g = golden_ops
    out = run_op("softmax_xent", {"l": g["sm_logits"], "y": g["sm_labels"]},
                 {"loss": (1,), "d": g["sm_logits"].shape})
    assert_close(out["loss"], g["sm_loss"], rtol=1e-6, atol=1e-6)
    assert_close(out["d"], g["sm_dlogits"], rtol=1e-5, atol=1e-7)
    logits = rnd(128, 1000, scale=4.0)
    labels = f32(RNG.integers(0, 1000, 128))
    loss, d = O.softmax_xent(logits, labels)
    out = run_op("softmax_xent", {"l": logits, "y": labels}, {"loss": (1,), "d": logits.shape})
    assert_close(out["loss"], loss, rtol=1e-5)
    assert_close(out["d"], d, rtol=1e-5, atol=1e-8)


def test_flatten_is_zero_copy_alias():
    from paper_1412_6249_b200 import BiGraph, Location, TensorStore, run

    loc = Location("local", 0)
    g = BiGraph()
    a = g.add_tensor("a", (2, 3, 4, 4), loc)
    f = g.add_tensor("f", (2, 48), loc)
    g.add_operator("fl", "flatten_forward", [a], [f], loc)
    st = TensorStore("cuda:0")
    x = rnd(2, 3, 4, 4)
    st.set("a", x)
    run(g, st)
    assert st.tensor("f").data_ptr() == st.tensor("a").data_ptr()
    assert np.array_equal(st.array("f"), x.reshape(2, 48))


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("shape", [(3, 8, 7, 7), (2, 12, 14, 14), (2, 3, 7, 7)])
def test_relu_backward_slice_sum_bitwise(k, shape):
    """relu_backward on a channel slice of a k-part gradient sum (the elided
    aggregate -> concat_backward pair), with its mask read from a channel
    slice of a wider tensor: bitwise relu_backward(x, ((p0 + p1) + ...)[slice])
    (k <= 4 run the 2-D float4 kernel, k = 5 the grid-stride one)."""
    import torch

    from paper_1412_6249_b200 import _native

    n, c, h, w = shape
    ctot, c0, x_ctot, x_c0 = c + 8, 4, c + 4, 4
    parts = [rnd(n, ctot, h, w) for _ in range(k)]
    xw = rnd(n, x_ctot, h, w)
    xw[:, x_c0:x_c0 + c].flat[::7] = 0.0  # masked exactly at zero too
    acc = parts[0].copy()
    for p in parts[1:]:
        acc = f32(acc + p)
    want = O.relu_backward(O.relu_forward(xw[:, x_c0:x_c0 + c]), acc[:, c0:c0 + c])
    dev = [torch.from_numpy(p).cuda() for p in parts]
    xd = torch.from_numpy(O.relu_forward(xw)).cuda()
    dx = torch.full((n, c, h, w), float("nan"), device="cuda")
    lib = _native.lib()
    lib("bf_relu_bwd_slice_sum_x", xd.data_ptr(), x_c0, x_ctot,
        _native.ptr_array([t.data_ptr() for t in dev]), k, c0, ctot, dx.data_ptr(), n, c, h * w,
        torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert_bitwise(dx.cpu().numpy(), want)
    if k == 1:  # the single-part entry point
        dx.fill_(float("nan"))
        lib("bf_relu_bwd_slice_x", xd.data_ptr(), x_c0, x_ctot, dev[0].data_ptr(), c0, ctot,
            dx.data_ptr(), n, c, h * w, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert_bitwise(dx.cpu().numpy(), want)
