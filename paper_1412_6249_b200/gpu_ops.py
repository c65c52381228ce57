"""Execute hooks of the operator kinds: resolve names -> device buffers, launch.

Each hook has the reference signature ``execute(ctx, op)`` (ops.py:526-533)
and launches one or more sm_100a kernels through the C ABI
(`include/purine_b200.h`) on the CUDA stream the dispatcher assigned to the
operator's lane (``ctx.stream``).  Outputs are written into buffers the
store preallocated; nothing here allocates per launch or synchronises the
host.  A kernel failure surfaces as `KernelError`.
"""

from __future__ import annotations

from . import _native
from .kinds import KernelError, conv_attrs, conv_out_dim, lrn_attrs, pool_attrs, pool_out_dim


def _names(ctx, ids):
    return [ctx.graph.tensors[i].name for i in ids]


def _ins(ctx, op):
    return [ctx.store.get(n) for n in _names(ctx, op.inputs)]


def _outs(ctx, op):
    g = ctx.graph
    return [ctx.store.ensure(g.tensors[i].name, g.tensors[i].shape) for i in op.outputs]


def _ws(ctx):
    w = ctx.workspace
    return w.data_ptr(), w.numel() * 4


def _L():
    return _native.lib()


# ---------------------------------------------------------------------------
# dense layer (ops.py:164-226)


def _fc_fwd(ctx, op):
    x, w, b = _ins(ctx, op)
    (y,) = _outs(ctx, op)
    n, d = x.shape
    m = w.shape[1]
    _L()("bf_fc_fwd", x.ptr, w.ptr, b.ptr, y.ptr, n, d, m, *_ws(ctx), ctx.stream)


def _fc_bwd_parts(ctx, x, w, dy, dx, dw, db):
    n, d = x.shape
    m = w.shape[1]
    lib = _L()
    if dx is not None:
        lib("bf_fc_bwd_data", w.ptr, dy.ptr, dx.ptr, n, d, m, *_ws(ctx), ctx.stream)
    if dw is not None:
        lib("bf_fc_bwd_weight", x.ptr, dy.ptr, dw.ptr, n, d, m, *_ws(ctx), ctx.stream)
    if db is not None:
        lib("bf_fc_bwd_bias", dy.ptr, db.ptr, n, m, ctx.stream)


def _fc_bwd(ctx, op):
    x, w, dy = _ins(ctx, op)
    dx, dw, db = _outs(ctx, op)
    _fc_bwd_parts(ctx, x, w, dy, dx, dw, db)


def _fc_bwd_data(ctx, op):
    w, dy = _ins(ctx, op)
    (dx,) = _outs(ctx, op)
    n, m = dy.shape
    _L()("bf_fc_bwd_data", w.ptr, dy.ptr, dx.ptr, n, w.shape[0], m, *_ws(ctx), ctx.stream)


def _fc_bwd_weight(ctx, op):
    x, dy = _ins(ctx, op)
    (dw,) = _outs(ctx, op)
    n, d = x.shape
    _L()("bf_fc_bwd_weight", x.ptr, dy.ptr, dw.ptr, n, d, dy.shape[1], *_ws(ctx), ctx.stream)


def _fc_bwd_bias(ctx, op):
    (dy,) = _ins(ctx, op)
    (db,) = _outs(ctx, op)
    _L()("bf_fc_bwd_bias", dy.ptr, db.ptr, dy.shape[0], dy.shape[1], ctx.stream)


# ---------------------------------------------------------------------------
# convolution (ops.py:229-352)


def _geom(x, w, attrs):
    stride, pad, floor = conv_attrs(attrs)
    n, c, h, wd = x.shape
    k, _, r, s = w.shape
    p = conv_out_dim(h, r, stride, pad, floor)
    q = conv_out_dim(wd, s, stride, pad, floor)
    return (n, c, h, wd, k, r, s, p, q, stride, pad)


def _conv_fwd_group(ctx, members):
    """Sibling 1x1 convolutions over the same x as one GEMM (dispatcher
    _Plan._group_1x1): each member keeps its own output, bias and fused ReLU
    target (its own tensor or a concat slice)."""
    import ctypes as C

    g = ctx.graph
    x = ctx.store.get(g.tensors[members[0][0].inputs[0]].name)
    n, c, h, wd = x.shape
    k = len(members)
    ws_, bs, ks, ys, rs, r0, rt = [], [], [], [], [], [], []
    for mop, mf in members:
        _x, w, b = _ins(ctx, mop)
        yshape = g.tensors[mop.outputs[0]].shape
        ws_.append(w.ptr)
        bs.append(b.ptr)
        ks.append(w.shape[0])
        ys.append(None if mf.get("no_y") else _outs(ctx, mop)[0].ptr)
        if "relu_slice" in mf:
            name, shape, c0 = mf["relu_slice"]
            rs.append(ctx.store.ensure(name, shape).ptr)
            r0.append(c0)
            rt.append(shape[1])
        elif "relu_out" in mf:
            rs.append(ctx.store.ensure(mf["relu_out"], yshape).ptr)
            r0.append(0)
            rt.append(w.shape[0])
        else:
            rs.append(None)
            r0.append(0)
            rt.append(w.shape[0])
    P = C.c_void_p * k
    I = C.c_int * k
    _L()("bf_conv1x1_fwd_group", x.ptr, n, c, h, wd, k, P(*ws_), P(*bs), I(*ks), P(*ys), P(*rs),
         I(*r0), I(*rt), *_ws(ctx), ctx.stream)


def _conv_fwd(ctx, op):
    fused = getattr(ctx, "fused", None)
    if fused and "group_fwd" in fused:
        _conv_fwd_group(ctx, fused["group_fwd"])
        return
    x, w, b = _ins(ctx, op)
    yshape = ctx.graph.tensors[op.outputs[0]].shape
    # pre-activation elision (dispatcher _Plan._preact_elision): y not stored
    yp = None if fused and fused.get("no_y") else _outs(ctx, op)[0].ptr
    if fused and "relu_slice" in fused:  # ReLU straight into its slice of the concat output
        name, shape, c0 = fused["relu_slice"]
        cat = ctx.store.ensure(name, shape)
        _L()("bf_conv2d_fwd_relu_slice", x.ptr, w.ptr, b.ptr, yp, cat.ptr, c0, shape[1],
             *_geom(x, w, op.attrs), *_ws(ctx), ctx.stream)
        return
    if fused and "relu_out" in fused:  # the following relu_forward runs in this epilogue
        yr = ctx.store.ensure(fused["relu_out"], yshape)
        _L()("bf_conv2d_fwd_relu", x.ptr, w.ptr, b.ptr, yp, yr.ptr, *_geom(x, w, op.attrs),
             *_ws(ctx), ctx.stream)
        return
    (y,) = _outs(ctx, op)
    _L()("bf_conv2d_fwd", x.ptr, w.ptr, b.ptr, y.ptr, *_geom(x, w, op.attrs), *_ws(ctx), ctx.stream)


def _conv_bwd_parts(ctx, attrs, x, w, dy, dx, dw, db):
    g = _geom(x, w, attrs)
    lib = _L()
    # weight and bias first: they feed the parameter exchange; data last
    if dw is not None and db is not None:  # one pass over dy for both
        lib("bf_conv2d_bwd_weight_bias", x.ptr, dy.ptr, dw.ptr, db.ptr, *g, *_ws(ctx), ctx.stream)
        dw = db = None
    if dw is not None:
        lib("bf_conv2d_bwd_weight", x.ptr, dy.ptr, dw.ptr, *g, *_ws(ctx), ctx.stream)
    if db is not None:
        lib("bf_conv2d_bwd_bias", dy.ptr, db.ptr, g[0], g[4], g[7] * g[8], *_ws(ctx), ctx.stream)
    if dx is not None:
        lib("bf_conv2d_bwd_data", w.ptr, dy.ptr, dx.ptr, *g, *_ws(ctx), ctx.stream)


def _conv_bwd(ctx, op):
    x, w, dy = _ins(ctx, op)
    dx, dw, db = _outs(ctx, op)
    _conv_bwd_parts(ctx, op.attrs, x, w, dy, dx, dw, db)


def _relu_fold(ctx, op):
    """(relu_x, output) when the following relu_backward is folded into this
    operator (dispatcher _Plan): write relu_backward's dx instead of our dy."""
    fused = getattr(ctx, "fused", None)
    if not (fused and "relu_x" in fused):
        return None, None
    rx = ctx.store.get(fused["relu_x"])
    return rx, ctx.store.ensure(fused["relu_dx"], rx.shape)


def _conv_bwd_data_group(ctx, op, members):
    """Sibling 1x1 data gradients summed in one GEMM into ``op``'s output
    (dispatcher _Plan._group_1x1_dgrad)."""
    import ctypes as C

    g = ctx.graph
    x = ctx.store.get(g.tensors[op.inputs[0]].name)
    n, c, h, wd = x.shape
    (dx,) = _outs(ctx, op)
    dys, ws_, ks = [], [], []
    for mop in members:
        _x, w, dy = _ins(ctx, mop)
        dys.append(dy.ptr)
        ws_.append(w.ptr)
        ks.append(w.shape[0])
    k = len(members)
    P = C.c_void_p * k
    _L()("bf_conv1x1_dgrad_group", n, c, h, wd, k, P(*dys), P(*ws_), (C.c_int * k)(*ks), dx.ptr,
         *_ws(ctx), ctx.stream)


def _conv_bwd_data(ctx, op):
    fused = getattr(ctx, "fused", None)
    if fused and "group_dgrad" in fused:
        _conv_bwd_data_group(ctx, op, fused["group_dgrad"])
        return
    x, w, dy = _ins(ctx, op)
    rx, rdx = _relu_fold(ctx, op)
    if rx is not None:
        _L()("bf_conv2d_bwd_data_relu", w.ptr, dy.ptr, rdx.ptr, rx.ptr, *_geom(x, w, op.attrs),
             *_ws(ctx), ctx.stream)
        return
    (dx,) = _outs(ctx, op)
    _conv_bwd_parts(ctx, op.attrs, x, w, dy, dx, None, None)


def _conv_bwd_weight(ctx, op):
    x, w, dy = _ins(ctx, op)
    (dw,) = _outs(ctx, op)
    fused = getattr(ctx, "fused", None)
    db = None
    if fused and "db" in fused:  # the sibling conv2d_backward_bias on the same dy
        db = ctx.store.ensure(fused["db"], (w.shape[0],))
    _conv_bwd_parts(ctx, op.attrs, x, w, dy, None, dw, db)


def _conv_bwd_bias(ctx, op):
    (dy,) = _ins(ctx, op)
    (db,) = _outs(ctx, op)
    n, k, p, q = dy.shape
    _L()("bf_conv2d_bwd_bias", dy.ptr, db.ptr, n, k, p * q, *_ws(ctx), ctx.stream)


# ---------------------------------------------------------------------------
# activation / reshape / loss / update / aggregation


def _relu_fwd(ctx, op):
    (x,) = _ins(ctx, op)
    (y,) = _outs(ctx, op)
    _L()("bf_relu_fwd", x.ptr, y.ptr, x.numel, ctx.stream)


def _relu_mask(ctx, op, fused):
    """(pointer, c0, ctot) of the relu_backward's mask: the pre-activation x,
    or -- pre-activation elision -- the ReLU output's channel slice of the
    concat output (relu(a) > 0 <=> a > 0)."""
    c = ctx.graph.tensors[op.inputs[0]].shape[1]
    if "x_slice" in fused:
        name, c0, ctot = fused["x_slice"]
        return ctx.store.get(name).ptr, c0, ctot
    return ctx.store.get(ctx.graph.tensors[op.inputs[0]].name).ptr, 0, c


def _relu_bwd(ctx, op):
    fused = getattr(ctx, "fused", None)
    if fused and "dy_parts" in fused:  # dy = slice of the (elided) sum of concatenated grads
        names, c0, ctot = fused["dy_parts"]
        xp, xc0, xct = _relu_mask(ctx, op, fused)
        (dx,) = _outs(ctx, op)
        parts = _native.ptr_array([ctx.store.get(nm).ptr for nm in names])
        n, c = dx.shape[0], dx.shape[1]
        _L()("bf_relu_bwd_slice_sum_x", xp, xc0, xct, parts, len(names), c0, ctot, dx.ptr, n, c,
             dx.numel // (n * c), ctx.stream)
        return
    if fused and "dy_slice" in fused:  # dy = a channel slice of the concatenated gradient
        name, c0, ctot = fused["dy_slice"]
        xp, xc0, xct = _relu_mask(ctx, op, fused)
        (dx,) = _outs(ctx, op)
        cat = ctx.store.get(name)
        n, c = dx.shape[0], dx.shape[1]
        _L()("bf_relu_bwd_slice_x", xp, xc0, xct, cat.ptr, c0, ctot, dx.ptr, n, c,
             dx.numel // (n * c), ctx.stream)
        return
    x, dy = _ins(ctx, op)
    (dx,) = _outs(ctx, op)
    _L()("bf_relu_bwd", x.ptr, dy.ptr, dx.ptr, x.numel, ctx.stream)


def _flatten_fwd(ctx, op):
    (src,) = _names(ctx, op.inputs)
    (dst,) = _names(ctx, op.outputs)
    if not ctx.store.is_alias_of(dst, src):
        ctx.store.alias(dst, src, ctx.graph.tensors[op.outputs[0]].shape)


def _flatten_bwd(ctx, op):
    _x, dy = _names(ctx, op.inputs)
    (dst,) = _names(ctx, op.outputs)
    if not ctx.store.is_alias_of(dst, dy):
        ctx.store.alias(dst, dy, ctx.graph.tensors[op.outputs[0]].shape)


def _softmax_xent(ctx, op):
    logits, labels = _ins(ctx, op)
    loss, dlogits = _outs(ctx, op)
    n, k = logits.shape
    _L()("bf_softmax_xent", logits.ptr, labels.ptr, loss.ptr, dlogits.ptr, n, k,
         ctx.workspace.data_ptr(), ctx.stream)


def _sgd_update(ctx, op):
    w, g = _ins(ctx, op)
    (out,) = _outs(ctx, op)
    _L()("bf_sgd_update", w.ptr, g.ptr, out.ptr, float(op.attrs["lr"]), w.numel, ctx.stream)


def _sgd_momentum(ctx, op):
    w, g, v = _ins(ctx, op)
    w_new, v_new = _outs(ctx, op)
    _L()("bf_sgd_momentum", w.ptr, g.ptr, v.ptr, w_new.ptr, v_new.ptr, float(op.attrs["lr"]),
         float(op.attrs.get("momentum", 0.0)), w.numel, ctx.stream)


def _aggregate(ctx, op):
    fused = getattr(ctx, "fused", None)
    if fused and "agg_parts" in fused:  # some parts were summed by a grouped data gradient
        parts = [ctx.store.get(n) for n in fused["agg_parts"]]
    else:
        parts = _ins(ctx, op)
    (out,) = _outs(ctx, op)
    mode = op.attrs.get("mode", "mean")
    if mode not in ("sum", "mean"):
        raise KernelError(f"aggregate: unknown mode {mode!r}")
    if len(parts) > 32:
        raise KernelError("aggregate: at most 32 inputs per operator")
    arr = _native.ptr_array([p.ptr for p in parts])
    _L()("bf_aggregate", arr, len(parts), out.ptr, out.numel, int(mode == "mean"), ctx.stream)


def _copy(ctx, op):
    (src,) = _ins(ctx, op)
    (dst,) = _outs(ctx, op)
    sv = ctx.graph.tensors[op.inputs[0]]
    dv = ctx.graph.tensors[op.outputs[0]]
    if ctx.copy_latency_s > 0 and sv.location != dv.location:
        _L()("bf_delay_ns", int(ctx.copy_latency_s * 1e9), ctx.stream)
    sd = src.data.device.index or 0
    dd = dst.data.device.index or 0
    _L()("bf_copy", dst.ptr, dd, src.ptr, sd, src.numel, ctx.stream)


def _gate(ctx, op):
    (src, _token) = _ins(ctx, op)
    (dst,) = _outs(ctx, op)
    d = src.data.device.index or 0
    _L()("bf_copy", dst.ptr, d, src.ptr, d, src.numel, ctx.stream)


def _swap(ctx, op):
    a, b = _names(ctx, op.outputs)
    ctx.store.swap(a, b)


def _no_transport(ctx, op):
    raise KernelError(f"{op.kind} {op.name!r}: no transport attached to this run "
                      "(multi-host transport is out of scope; use the NCCL exchange)")


def _dp_exchange(ctx, op):
    """Lowered parameter-server subgraph for one gradient bucket (exchange.py):
    reduce-scatter(sum) -> fused mean + SGD (or momentum) on the owned shard
    -> all-gather.  Inputs: the bucket's parameters [, velocity shard], then
    its gradients; outputs: the new parameters [, new velocity shard]."""
    from .exchange import check_bucket, shard_of

    ins = _ins(ctx, op)
    outs = _outs(ctx, op)
    a = op.attrs
    mu = float(a.get("momentum", 0.0) or 0.0)
    nb = len(a["offsets"])
    if len(outs) != nb + (mu > 0) or len(ins) != 2 * nb + (mu > 0):
        raise KernelError(f"dp_exchange: {len(ins)} inputs / {len(outs)} outputs do not match "
                          f"{nb} parameters (momentum {mu})")
    w0, g0, o0 = check_bucket(ins[:nb], ins[len(ins) - nb:], outs[:nb], a["offsets"])
    length, world, lr = int(a["flat_len"]), int(a["world"]), float(a["lr"])
    shard, first = shard_of(length, world, int(a["rank"]))
    coll = getattr(ctx.store, "_collective", None)
    if coll is None and world > 1:
        raise KernelError("dp_exchange: no collective attached to this store "
                          "(exchange.setup_nccl or LocalGroup)")
    if coll is not None and coll.world != world:
        raise KernelError(f"dp_exchange: collective spans {coll.world} ranks, op expects {world}")
    if mu > 0:
        v, vn = ins[nb], outs[nb]
        if v.numel != shard or vn.numel != shard:
            raise KernelError(f"dp_exchange: velocity shard holds {v.numel} floats, expected {shard}")
    off = first * 4
    lib = _L()
    if coll is not None:
        coll.reduce_scatter(g0, shard, ctx.stream)
    if mu > 0:
        lib("bf_sgd_mean_momentum", w0 + off, g0 + off, v.ptr, o0 + off, vn.ptr, lr, mu, world,
            shard, ctx.stream)
    else:
        lib("bf_sgd_mean_update", w0 + off, g0 + off, o0 + off, lr, world, shard, ctx.stream)
    if coll is not None:
        coll.all_gather(o0, shard, ctx.stream)


# ---------------------------------------------------------------------------
# pooling / LRN / concat (extension kinds)


def _maxpool_fwd(ctx, op):
    (x,) = _ins(ctx, op)
    k, s, p = pool_attrs(op.attrs)
    n, c, h, w = x.shape
    fused = getattr(ctx, "fused", None) or {}
    g = ctx.graph
    yv = g.tensors[op.outputs[0]]
    y = ctx.store.ensure(yv.name, yv.shape)
    if fused.get("pool_smask"):  # the signed mask (dispatcher _Plan): argmax + sign per window
        sm = ctx.store.ensure(fused["pool_smask"], y.shape)
        _L()("bf_maxpool_fwd_smask", x.ptr, y.ptr, sm.ptr, n, c, h, w, y.shape[2], y.shape[3],
             k, s, p, ctx.stream)
        return
    if fused.get("pool_no_mask"):  # only maxpool_backward reads it, and it recomputes it
        _L()("bf_maxpool_fwd_staged", x.ptr, y.ptr, None, n, c, h, w, y.shape[2], y.shape[3], k,
             s, p, ctx.stream)
        return
    mv = g.tensors[op.outputs[1]]
    mask = ctx.store.ensure(mv.name, mv.shape)
    _L()("bf_maxpool_fwd", x.ptr, y.ptr, mask.ptr, n, c, h, w, y.shape[2], y.shape[3], k, s, p,
         ctx.stream)


def _maxpool_bwd(ctx, op):
    k, s, p = pool_attrs(op.attrs)
    fused = getattr(ctx, "fused", None) or {}
    if fused.get("pool_smask"):  # gather from the signed mask and dy; x is not read
        g = ctx.graph
        xv = g.tensors[op.inputs[0]]
        dy = ctx.store.get(g.tensors[op.inputs[2]].name)
        n, c, h, w = xv.shape
        sm = ctx.store.get(fused["pool_smask"])
        if fused.get("relu_from_x"):  # + the relu_backward of x = relu(a), from the sign
            dx = ctx.store.ensure(fused["relu_dx"], xv.shape)
        else:
            dxv = g.tensors[op.outputs[0]]
            dx = ctx.store.ensure(dxv.name, dxv.shape)
        _L()("bf_maxpool_bwd_smask", sm.ptr, dy.ptr, dx.ptr, int(bool(fused.get("relu_from_x"))),
             n, c, h, w, dy.shape[2], dy.shape[3], k, s, p, ctx.stream)
        return
    if fused.get("pool_recompute"):  # argmax recomputed from x (the mask is elided)
        g = ctx.graph
        x = ctx.store.get(g.tensors[op.inputs[0]].name)
        dy = ctx.store.get(g.tensors[op.inputs[2]].name)
        n, c, h, w = x.shape
        if fused.get("relu_from_x"):  # + the relu_backward of x = relu(a)
            dx = ctx.store.ensure(fused["relu_dx"], x.shape)
        else:
            dxv = g.tensors[op.outputs[0]]
            dx = ctx.store.ensure(dxv.name, dxv.shape)
        _L()("bf_maxpool_bwd_x", x.ptr, dy.ptr, dx.ptr, int(bool(fused.get("relu_from_x"))), n, c,
             h, w, dy.shape[2], dy.shape[3], k, s, p, ctx.stream)
        return
    x, mask, dy = _ins(ctx, op)
    n, c, h, w = x.shape
    rx, rdx = _relu_fold(ctx, op)
    if rx is not None:
        _L()("bf_maxpool_bwd_relu", mask.ptr, dy.ptr, rdx.ptr, rx.ptr, n, c, h, w, dy.shape[2],
             dy.shape[3], k, s, p, ctx.stream)
        return
    (dx,) = _outs(ctx, op)
    _L()("bf_maxpool_bwd", mask.ptr, dy.ptr, dx.ptr, n, c, h, w, dy.shape[2], dy.shape[3], k, s,
         p, ctx.stream)


def _avgpool_fwd(ctx, op):
    (x,) = _ins(ctx, op)
    (y,) = _outs(ctx, op)
    k, s, p = pool_attrs(op.attrs)
    n, c, h, w = x.shape
    _L()("bf_avgpool_fwd", x.ptr, y.ptr, n, c, h, w, y.shape[2], y.shape[3], k, s, p, ctx.stream)


def _avgpool_bwd(ctx, op):
    x, dy = _ins(ctx, op)
    (dx,) = _outs(ctx, op)
    k, s, p = pool_attrs(op.attrs)
    n, c, h, w = x.shape
    _L()("bf_avgpool_bwd", dy.ptr, dx.ptr, n, c, h, w, dy.shape[2], dy.shape[3], k, s, p,
         ctx.stream)


def _lrn_fwd(ctx, op):
    (x,) = _ins(ctx, op)
    g = ctx.graph
    size, alpha, beta, k = lrn_attrs(op.attrs)
    fused = getattr(ctx, "fused", None)
    y = ctx.store.ensure(g.tensors[op.outputs[0]].name, g.tensors[op.outputs[0]].shape)
    if fused and fused.get("lrn_no_scale"):  # scale elided: the backward recomputes it
        _L()("bf_lrn_fwd", x.ptr, y.ptr, None, *x.shape, size, alpha, beta, k, ctx.stream)
        return
    scale = ctx.store.ensure(g.tensors[op.outputs[1]].name, g.tensors[op.outputs[1]].shape)
    _L()("bf_lrn_fwd", x.ptr, y.ptr, scale.ptr, *x.shape, size, alpha, beta, k, ctx.stream)


def _lrn_bwd(ctx, op):
    size, alpha, beta, k = lrn_attrs(op.attrs)
    rx, rdx = _relu_fold(ctx, op)
    fused = getattr(ctx, "fused", None)
    if fused and fused.get("lrn_recompute"):  # x, dy only (scale, y recomputed)
        names = _names(ctx, op.inputs)
        x, dy = ctx.store.get(names[0]), ctx.store.get(names[3])
        dx = rdx if rx is not None else _outs(ctx, op)[0]
        _L()("bf_lrn_bwd_recompute", x.ptr, dy.ptr, dx.ptr, rx.ptr if rx is not None else None,
             *x.shape, size, alpha, beta, k, ctx.stream)
        return
    x, y, scale, dy = _ins(ctx, op)
    if rx is not None:
        _L()("bf_lrn_bwd_relu", x.ptr, y.ptr, scale.ptr, dy.ptr, rdx.ptr, rx.ptr, *x.shape, size,
             alpha, beta, k, ctx.stream)
        return
    (dx,) = _outs(ctx, op)
    _L()("bf_lrn_bwd", x.ptr, y.ptr, scale.ptr, dy.ptr, dx.ptr, *x.shape, size, alpha, beta, k,
         ctx.stream)


def _concat_fwd(ctx, op):
    parts = _ins(ctx, op)
    (y,) = _outs(ctx, op)
    n, _, h, w = y.shape
    _L()("bf_concat_fwd", _native.ptr_array([p.ptr for p in parts]),
         _native.int_array([p.shape[1] for p in parts]), len(parts), y.ptr, n, h, w, ctx.stream)


def _concat_bwd(ctx, op):
    (dy,) = _ins(ctx, op)
    parts = _outs(ctx, op)
    n, _, h, w = dy.shape
    _L()("bf_concat_bwd", dy.ptr, _native.ptr_array([p.ptr for p in parts]),
         _native.int_array([p.shape[1] for p in parts]), len(parts), n, h, w, ctx.stream)


EXECUTORS = {
    "fc_forward": _fc_fwd,
    "fc_backward": _fc_bwd,
    "fc_backward_data": _fc_bwd_data,
    "fc_backward_weight": _fc_bwd_weight,
    "fc_backward_bias": _fc_bwd_bias,
    "conv2d_forward": _conv_fwd,
    "conv2d_backward": _conv_bwd,
    "conv2d_backward_data": _conv_bwd_data,
    "conv2d_backward_weight": _conv_bwd_weight,
    "conv2d_backward_bias": _conv_bwd_bias,
    "relu_forward": _relu_fwd,
    "relu_backward": _relu_bwd,
    "flatten_forward": _flatten_fwd,
    "flatten_backward": _flatten_bwd,
    "softmax_xent": _softmax_xent,
    "sgd_update": _sgd_update,
    "sgd_momentum": _sgd_momentum,
    "aggregate": _aggregate,
    "copy": _copy,
    "gate": _gate,
    "swap": _swap,
    "send": _no_transport,
    "recv": _no_transport,
    "maxpool_forward": _maxpool_fwd,
    "maxpool_backward": _maxpool_bwd,
    "avgpool_forward": _avgpool_fwd,
    "avgpool_backward": _avgpool_bwd,
    "lrn_forward": _lrn_fwd,
    "lrn_backward": _lrn_bwd,
    "concat_forward": _concat_fwd,
    "concat_backward": _concat_bwd,
    "dp_exchange": _dp_exchange,
}

# kinds that launch nothing (host-side handle work only)
HOST_ONLY = frozenset({"swap", "flatten_forward", "flatten_backward"})
# kinds whose outputs alias an input buffer instead of owning storage
ALIASING = {"flatten_forward": 0, "flatten_backward": 1}
