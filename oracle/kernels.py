"""numpy float32 restatement of the reference kernels (TEST INFRASTRUCTURE ONLY).

Every function cites the reference file:line whose algorithm it restates.
Reference kinds keep the reference's arithmetic (BLAS ``@`` for dense
products, an im2col patch tensor contracted with ``np.einsum`` for
convolutions, true division for the mean, no fused multiply-add in SGD) so
that the oracle reproduces the reference's numbers on the same machine.

Extension kinds (no reference implementation — *parity unpinned* by the
reference) follow Caffe's definitions, which is what Purine ran
(arXiv 1412.6249 §4 uses Caffe's layers / cuDNN):
  * max/avg pooling: Caffe "ceil" output size, window clipped to the image,
    max-pool argmax = first maximum in row-major window order, stored as the
    integral flat index ``h*W + w`` inside a float32 tensor;
  * LRN across channels: ``scale = k + alpha/n * sum(x^2 over window)``,
    ``y = x * scale^-beta``;
  * concat along channels;
  * SGD with momentum (Caffe convention ``v' = mu*v + lr*g``, ``w' = w - v'``),
    which reduces bitwise to ``sgd_update`` at ``mu = 0``;
  * floor-mode convolution output size (Caffe), opt-in via ``floor=True``.
"""

from __future__ import annotations

import numpy as np
from numpy.lib.stride_tricks import as_strided

__all__ = [
    "OracleError",
    "f32",
    "conv_out_dim",
    "pool_out_dim",
    "fc_forward",
    "fc_backward",
    "fc_backward_data",
    "fc_backward_weight",
    "fc_backward_bias",
    "conv2d_forward",
    "conv2d_backward",
    "conv2d_backward_data",
    "conv2d_backward_weight",
    "conv2d_backward_bias",
    "relu_forward",
    "relu_backward",
    "flatten_forward",
    "flatten_backward",
    "softmax_xent",
    "sgd_update",
    "sgd_momentum",
    "aggregate",
    "maxpool_forward",
    "maxpool_backward",
    "avgpool_forward",
    "avgpool_backward",
    "lrn_forward",
    "lrn_backward",
    "concat_forward",
    "concat_backward",
    "KERNELS",
]


class OracleError(RuntimeError):
    """Non-conforming data (mirrors the reference's KernelError, ops.py:48)."""


def f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _need(ok: bool, msg: str) -> None:
    if not ok:
        raise OracleError(msg)


def _all_finite(kind: str, *outs) -> None:
    # ops.py:61-64: every kernel output must be finite
    for o in outs:
        if not np.all(np.isfinite(o)):
            raise OracleError(f"{kind}: non-finite value in output")


# ---------------------------------------------------------------------------
# output-size rules


def conv_out_dim(size: int, k: int, stride: int, pad: int, floor: bool = False) -> int:
    """ops.py:229-240 (integral rule); ``floor=True`` is Caffe's floor rule."""
    span = size + 2 * pad - k
    _need(span >= 0, f"conv2d: kernel {k} larger than padded input {size}+2*{pad}")
    if not floor:
        _need(span % stride == 0,
              f"conv2d: non-integral output for size={size} kernel={k} "
              f"stride={stride} pad={pad}")
    return span // stride + 1


def pool_out_dim(size: int, k: int, stride: int, pad: int) -> int:
    """Caffe pooling size: ceil((size + 2p - k)/s) + 1, dropping a last
    window that would start inside the right padding."""
    _need(size + 2 * pad >= k, f"pool: kernel {k} larger than padded input")
    out = -(-(size + 2 * pad - k) // stride) + 1
    if pad > 0 and (out - 1) * stride >= size + pad:
        out -= 1
    return out


# ---------------------------------------------------------------------------
# dense (ops.py:164-226)


def fc_forward(x, w, b):
    """ops.py:164-176: y = x @ w + b."""
    x, w, b = f32(x), f32(w), f32(b)
    _need(x.ndim == 2 and w.ndim == 2 and b.ndim == 1, "fc_forward: ranks")
    _need(x.shape[1] == w.shape[0] == w.shape[0] and w.shape[1] == b.shape[0],
          "fc_forward: shapes do not conform")
    out = np.matmul(x, w) + b
    _all_finite("fc_forward", out)
    return out


def fc_backward_data(w, dy):
    """ops.py:196-205: dx = dy @ w^T."""
    w, dy = f32(w), f32(dy)
    out = np.matmul(dy, w.T)
    _all_finite("fc_backward_data", out)
    return out


def fc_backward_weight(x, dy):
    """ops.py:208-216: dw = x^T @ dy."""
    x, dy = f32(x), f32(dy)
    out = np.matmul(x.T, dy)
    _all_finite("fc_backward_weight", out)
    return out


def fc_backward_bias(dy):
    """ops.py:219-226: column sum of dy."""
    dy = f32(dy)
    out = dy.sum(axis=0)
    _all_finite("fc_backward_bias", out)
    return out


def fc_backward(x, w, dy):
    """ops.py:179-193: (dx, dw, db) in one op."""
    x, w, dy = f32(x), f32(w), f32(dy)
    _need(dy.shape == (x.shape[0], w.shape[1]) and x.shape[1] == w.shape[0],
          "fc_backward: shapes do not conform")
    return fc_backward_data(w, dy), fc_backward_weight(x, dy), fc_backward_bias(dy)


# ---------------------------------------------------------------------------
# convolution (ops.py:229-352): im2col patch tensor + einsum contraction


def _patches(x, r, s, stride, pad, ho, wo):
    """[N, C, R, S, Ho, Wo] patch tensor of the zero-padded input.

    Same patch tensor as ops.py:251-262, built from a strided view instead of
    the reference's per-(i, j) slice loop."""
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    n, c, hp, wp = xp.shape
    sn, sc, sh, sw = xp.strides
    view = as_strided(
        xp,
        shape=(n, c, r, s, ho, wo),
        strides=(sn, sc, sh, sw, sh * stride, sw * stride),
        writeable=False,
    )
    return np.ascontiguousarray(view), xp.shape


def _conv_geometry(x, w, stride, pad, floor):
    _need(x.ndim == 4 and w.ndim == 4, "conv2d: x and w must be 4-d")
    _need(w.shape[1] == x.shape[1], "conv2d: channel mismatch")
    _need(stride >= 1 and pad >= 0, "conv2d: bad stride/pad")
    ho = conv_out_dim(x.shape[2], w.shape[2], stride, pad, floor)
    wo = conv_out_dim(x.shape[3], w.shape[3], stride, pad, floor)
    return ho, wo


def conv2d_forward(x, w, b, stride=1, pad=0, floor=False):
    """ops.py:281-297: y[n,k,h,w] = sum_{c,i,j} patch[n,c,i,j,h,w] * w[k,c,i,j] + b[k]."""
    x, w, b = f32(x), f32(w), f32(b)
    ho, wo = _conv_geometry(x, w, stride, pad, floor)
    _need(b.ndim == 1 and b.shape[0] == w.shape[0], "conv2d: bias shape")
    cols, _ = _patches(x, w.shape[2], w.shape[3], stride, pad, ho, wo)
    y = np.einsum("ncijhw,kcij->nkhw", cols, w, dtype=np.float32)
    y = f32(y + b[None, :, None, None])
    _all_finite("conv2d_forward", y)
    return y


def conv2d_backward(x, w, dy, stride=1, pad=0, floor=False):
    """ops.py:300-329: dx via the transposed contraction + col2im scatter-add
    in (i, j) order, dw via the patch contraction, db = sum over (n, h, w)."""
    x, w, dy = f32(x), f32(w), f32(dy)
    ho, wo = _conv_geometry(x, w, stride, pad, floor)
    k, c, r, s = w.shape
    _need(dy.shape == (x.shape[0], k, ho, wo), "conv2d_backward: dy shape")
    cols, padded_shape = _patches(x, r, s, stride, pad, ho, wo)
    dw = f32(np.einsum("ncijhw,nkhw->kcij", cols, dy, dtype=np.float32))
    db = f32(dy.sum(axis=(0, 2, 3)))
    dcols = np.einsum("nkhw,kcij->ncijhw", dy, w, dtype=np.float32)
    dxp = np.zeros(padded_shape, dtype=np.float32)
    for i in range(r):
        for j in range(s):
            dxp[:, :, i:i + stride * ho:stride, j:j + stride * wo:stride] += dcols[:, :, i, j]
    h, wd = x.shape[2], x.shape[3]
    dx = f32(dxp[:, :, pad:pad + h, pad:pad + wd])
    _all_finite("conv2d_backward", dx, dw, db)
    return dx, dw, db


def conv2d_backward_data(x, w, dy, stride=1, pad=0, floor=False):
    """ops.py:332-336 (reference recomputes the fused backward)."""
    return conv2d_backward(x, w, dy, stride, pad, floor)[0]


def conv2d_backward_weight(x, w, dy, stride=1, pad=0, floor=False):
    """ops.py:339-343."""
    return conv2d_backward(x, w, dy, stride, pad, floor)[1]


def conv2d_backward_bias(dy):
    """ops.py:346-352."""
    dy = f32(dy)
    _need(dy.ndim == 4, "conv2d_backward_bias: dy must be 4-d")
    db = f32(dy.sum(axis=(0, 2, 3)))
    _all_finite("conv2d_backward_bias", db)
    return db


# ---------------------------------------------------------------------------
# activation, loss, update, aggregation (ops.py:359-457)


def relu_forward(x):
    """ops.py:359-364."""
    x = f32(x)
    return np.maximum(x, np.float32(0.0))


def relu_backward(x, dy):
    """ops.py:367-376: dy where x > 0, else 0 (subgradient at 0 is 0)."""
    x, dy = f32(x), f32(dy)
    _need(x.shape == dy.shape, "relu_backward: shape mismatch")
    return np.where(x > np.float32(0.0), dy, np.float32(0.0)).astype(np.float32)


def flatten_forward(x):
    """ops.py:379-382."""
    x = f32(x)
    return x.reshape(x.shape[0], -1)


def flatten_backward(x, dy):
    """ops.py:385-391."""
    x, dy = f32(x), f32(dy)
    return dy.reshape(x.shape)


def softmax_xent(logits, labels):
    """ops.py:394-425: row-max stabilised softmax, mean NLL, (p - onehot)/N."""
    logits, labels = f32(logits), f32(labels)
    _need(logits.ndim == 2, "softmax_xent: logits must be 2-d")
    n, k = logits.shape
    _need(labels.shape == (n,), "softmax_xent: labels shape")
    idx = labels.astype(np.int64)
    _need(bool(np.all(idx == labels) and np.all(idx >= 0) and np.all(idx < k)),
          "softmax_xent: labels must be integral and in range")
    z = logits - logits.max(axis=1, keepdims=True)
    e = np.exp(z)
    denom = e.sum(axis=1, keepdims=True)
    p = e / denom
    rows = np.arange(n)
    nll = -(z[rows, idx] - np.log(denom[:, 0]))
    loss = np.array([nll.mean()], dtype=np.float32)
    grad = p.copy()
    grad[rows, idx] -= np.float32(1.0)
    grad = f32(grad / np.float32(n))
    _all_finite("softmax_xent", loss, grad)
    return loss, grad


def sgd_update(w, g, lr):
    """ops.py:428-437: w - f32(lr) * g, product rounded before the subtract."""
    w, g = f32(w), f32(g)
    _need(w.shape == g.shape, "sgd_update: shape mismatch")
    step = np.multiply(np.float32(lr), g, dtype=np.float32)
    out = np.subtract(w, step, dtype=np.float32)
    _all_finite("sgd_update", out)
    return out


def sgd_momentum(w, g, v, lr, momentum):
    """Extension (SPEC.md:312 leaves momentum "extendable via attrs").

    Caffe convention: v' = mu*v + lr*g, w' = w - v'; each product rounded to
    float32 before the add, so mu = 0 reproduces ``sgd_update`` bitwise."""
    w, g, v = f32(w), f32(g), f32(v)
    _need(w.shape == g.shape == v.shape, "sgd_momentum: shape mismatch")
    keep = np.multiply(np.float32(momentum), v, dtype=np.float32)
    step = np.multiply(np.float32(lr), g, dtype=np.float32)
    v_new = np.add(keep, step, dtype=np.float32)
    w_new = np.subtract(w, v_new, dtype=np.float32)
    _all_finite("sgd_momentum", w_new, v_new)
    return w_new, v_new


def aggregate(parts, mode="mean"):
    """ops.py:440-457: left-to-right sum in rank order; mean divides by f32(k)."""
    _need(len(parts) >= 1, "aggregate: need at least one input")
    _need(mode in ("sum", "mean"), f"aggregate: unknown mode {mode!r}")
    arrs = [f32(p) for p in parts]
    for a in arrs[1:]:
        _need(a.shape == arrs[0].shape, "aggregate: shape mismatch")
    total = arrs[0].copy()
    for a in arrs[1:]:
        np.add(total, a, out=total)
    if mode == "mean":
        np.divide(total, np.float32(len(arrs)), out=total)
    _all_finite("aggregate", total)
    return total


# ---------------------------------------------------------------------------
# pooling (extension; Caffe semantics)


def _pool_window(p, stride, pad, k, size):
    lo = p * stride - pad
    hi = min(lo + k, size)
    return max(lo, 0), hi


def maxpool_forward(x, kernel, stride, pad=0):
    """Returns (y, mask); mask holds the flat index h*W + w of the first
    maximum of each window (row-major scan, strict '>' update)."""
    x = f32(x)
    _need(x.ndim == 4, "maxpool: x must be 4-d")
    n, c, h, w = x.shape
    ph_n = pool_out_dim(h, kernel, stride, pad)
    pw_n = pool_out_dim(w, kernel, stride, pad)
    y = np.empty((n, c, ph_n, pw_n), dtype=np.float32)
    mask = np.empty((n, c, ph_n, pw_n), dtype=np.float32)
    for ph in range(ph_n):
        h0, h1 = _pool_window(ph, stride, pad, kernel, h)
        for pw in range(pw_n):
            w0, w1 = _pool_window(pw, stride, pad, kernel, w)
            best = np.full((n, c), -np.inf, dtype=np.float32)
            arg = np.full((n, c), -1, dtype=np.int64)
            for hh in range(h0, h1):
                for ww in range(w0, w1):
                    v = x[:, :, hh, ww]
                    better = v > best
                    best = np.where(better, v, best)
                    arg = np.where(better, hh * w + ww, arg)
            y[:, :, ph, pw] = best
            mask[:, :, ph, pw] = arg.astype(np.float32)
    _all_finite("maxpool_forward", y)
    return y, mask


def maxpool_backward(x, mask, dy):
    """dx[mask[p]] += dy[p], output positions visited in row-major order."""
    x, mask, dy = f32(x), f32(mask), f32(dy)
    n, c, h, w = x.shape
    _need(mask.shape == dy.shape and dy.shape[:2] == (n, c), "maxpool_backward: shapes")
    dx = np.zeros((n, c, h * w), dtype=np.float32)
    idx = mask.astype(np.int64).reshape(n, c, -1)
    g = dy.reshape(n, c, -1)
    nn, cc = np.meshgrid(np.arange(n), np.arange(c), indexing="ij")
    for p in range(g.shape[2]):
        dx[nn, cc, idx[:, :, p]] += g[:, :, p]
    return dx.reshape(n, c, h, w)


def _avg_window(p, stride, pad, k, size):
    lo = p * stride - pad
    hi = min(lo + k, size + pad)
    count = hi - lo
    return max(lo, 0), min(hi, size), count


def avgpool_forward(x, kernel, stride, pad=0):
    """Caffe AVE pooling: window sum (row-major, float32) / f32(pool_size),
    pool_size counting the padded extent clipped to size + pad."""
    x = f32(x)
    n, c, h, w = x.shape
    ph_n = pool_out_dim(h, kernel, stride, pad)
    pw_n = pool_out_dim(w, kernel, stride, pad)
    y = np.empty((n, c, ph_n, pw_n), dtype=np.float32)
    for ph in range(ph_n):
        h0, h1, ch = _avg_window(ph, stride, pad, kernel, h)
        for pw in range(pw_n):
            w0, w1, cw = _avg_window(pw, stride, pad, kernel, w)
            acc = np.zeros((n, c), dtype=np.float32)
            for hh in range(h0, h1):
                for ww in range(w0, w1):
                    acc = acc + x[:, :, hh, ww]
            y[:, :, ph, pw] = acc / np.float32(ch * cw)
    return y


def avgpool_backward(x, dy, kernel, stride, pad=0):
    """dx[h, w] += dy[p] / f32(pool_size), output positions in row-major order."""
    x, dy = f32(x), f32(dy)
    n, c, h, w = x.shape
    ph_n, pw_n = dy.shape[2], dy.shape[3]
    dx = np.zeros((n, c, h, w), dtype=np.float32)
    for ph in range(ph_n):
        h0, h1, ch = _avg_window(ph, stride, pad, kernel, h)
        for pw in range(pw_n):
            w0, w1, cw = _avg_window(pw, stride, pad, kernel, w)
            share = dy[:, :, ph, pw] / np.float32(ch * cw)
            for hh in range(h0, h1):
                for ww in range(w0, w1):
                    dx[:, :, hh, ww] += share
    return dx


# ---------------------------------------------------------------------------
# local response normalisation across channels (extension; Caffe)


def _lrn_bounds(c, size, channels):
    pre = (size - 1) // 2
    post = size - 1 - pre
    return max(c - pre, 0), min(c + post, channels - 1)


def lrn_forward(x, size=5, alpha=1e-4, beta=0.75, k=1.0):
    """Returns (y, scale): scale = k + alpha/size * sum_{window} x^2 (channel
    order, float32), y = x * scale^-beta."""
    x = f32(x)
    n, c, h, w = x.shape
    sq = np.multiply(x, x, dtype=np.float32)
    a_n = np.float32(alpha) / np.float32(size)
    scale = np.empty_like(x)
    for ci in range(c):
        lo, hi = _lrn_bounds(ci, size, c)
        acc = np.zeros((n, h, w), dtype=np.float32)
        for cj in range(lo, hi + 1):
            acc = acc + sq[:, cj]
        scale[:, ci] = np.float32(k) + a_n * acc
    y = f32(x * np.power(scale, np.float32(-beta), dtype=np.float32))
    _all_finite("lrn_forward", y, scale)
    return y, scale


def lrn_backward(x, y, scale, dy, size=5, alpha=1e-4, beta=0.75, k=1.0):
    """Caffe: dx = dy*scale^-beta - (2*alpha*beta/size) * x *
    sum_{c' whose window holds c} dy[c']*y[c']/scale[c']."""
    x, y, scale, dy = f32(x), f32(y), f32(scale), f32(dy)
    n, c, h, w = x.shape
    ratio = f32(dy * y / scale)
    pre = (size - 1) // 2
    post = size - 1 - pre
    coef = np.float32(2.0) * np.float32(alpha) * np.float32(beta) / np.float32(size)
    dx = np.empty_like(x)
    for ci in range(c):
        lo, hi = max(ci - post, 0), min(ci + pre, c - 1)
        acc = np.zeros((n, h, w), dtype=np.float32)
        for cj in range(lo, hi + 1):
            acc = acc + ratio[:, cj]
        dx[:, ci] = dy[:, ci] * np.power(scale[:, ci], np.float32(-beta), dtype=np.float32) \
            - coef * x[:, ci] * acc
    _all_finite("lrn_backward", dx)
    return f32(dx)


# ---------------------------------------------------------------------------
# concat along channels (extension)


def concat_forward(parts):
    parts = [f32(p) for p in parts]
    return np.concatenate(parts, axis=1)


def concat_backward(dy, channels):
    dy = f32(dy)
    out, lo = [], 0
    for ch in channels:
        out.append(np.ascontiguousarray(dy[:, lo:lo + ch]))
        lo += ch
    return out


# ---------------------------------------------------------------------------
# kind -> callable(ins, attrs) -> outs, for the serial executor


def _conv_a(a):
    return int(a.get("stride", 1)), int(a.get("pad", 0)), bool(a.get("floor", False))


def _pool_a(a):
    return int(a["kernel"]), int(a.get("stride", 1)), int(a.get("pad", 0))


def _lrn_a(a):
    return (int(a.get("size", 5)), float(a.get("alpha", 1e-4)),
            float(a.get("beta", 0.75)), float(a.get("k", 1.0)))


KERNELS = {
    "fc_forward": lambda i, a: [fc_forward(*i)],
    "fc_backward": lambda i, a: list(fc_backward(*i)),
    "fc_backward_data": lambda i, a: [fc_backward_data(*i)],
    "fc_backward_weight": lambda i, a: [fc_backward_weight(*i)],
    "fc_backward_bias": lambda i, a: [fc_backward_bias(*i)],
    "conv2d_forward": lambda i, a: [conv2d_forward(*i, *_conv_a(a))],
    "conv2d_backward": lambda i, a: list(conv2d_backward(*i, *_conv_a(a))),
    "conv2d_backward_data": lambda i, a: [conv2d_backward_data(*i, *_conv_a(a))],
    "conv2d_backward_weight": lambda i, a: [conv2d_backward_weight(*i, *_conv_a(a))],
    "conv2d_backward_bias": lambda i, a: [conv2d_backward_bias(i[0])],
    "relu_forward": lambda i, a: [relu_forward(*i)],
    "relu_backward": lambda i, a: [relu_backward(*i)],
    "flatten_forward": lambda i, a: [flatten_forward(*i)],
    "flatten_backward": lambda i, a: [flatten_backward(*i)],
    "softmax_xent": lambda i, a: list(softmax_xent(*i)),
    "sgd_update": lambda i, a: [sgd_update(i[0], i[1], float(a["lr"]))],
    "sgd_momentum": lambda i, a: list(sgd_momentum(i[0], i[1], i[2], float(a["lr"]),
                                                   float(a.get("momentum", 0.0)))),
    "aggregate": lambda i, a: [aggregate(i, a.get("mode", "mean"))],
    "maxpool_forward": lambda i, a: list(maxpool_forward(i[0], *_pool_a(a))),
    "maxpool_backward": lambda i, a: [maxpool_backward(*i)],
    "avgpool_forward": lambda i, a: [avgpool_forward(i[0], *_pool_a(a))],
    "avgpool_backward": lambda i, a: [avgpool_backward(i[0], i[1], *_pool_a(a))],
    "lrn_forward": lambda i, a: list(lrn_forward(i[0], *_lrn_a(a))),
    "lrn_backward": lambda i, a: [lrn_backward(*i, *_lrn_a(a))],
    "concat_forward": lambda i, a: [concat_forward(i)],
    "concat_backward": lambda i, a: concat_backward(i[0], [int(c) for c in a["channels"]]),
    # pipeline stage entry: passes input 0 through once the token (input 1)
    # exists; the token only orders (ops.py:745-747, 803-804)
    "gate": lambda i, a: [np.array(i[0], dtype=np.float32, copy=True)],
}
