"""Operator-kind registry: the plugin boundary of the hot path.

Drop-in for the reference's registry (`pkg/src/biflow/ops.py:499-809`):
`OpKindSpec(kind, min_in, max_in, n_out, check_shapes, execute,
crosses_location)`, the global `KINDS` table consulted at graph-build time
(graph.py:197-214) and `default_registry()`.

The shape rules below restate the reference's checkers (ops.py:579-742) and
add the kinds the GoogLeNet / NIN configurations need (pooling, LRN,
concat, momentum SGD, floor-mode convolution).  Every ``execute`` hook of a
compute kind launches a hand-written sm_100a kernel through the C-ABI
library (`gpu_ops.py` -> `include/purine_b200.h`); there is no CPU
fallback — if the library is missing the hook raises `KernelError`.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

__all__ = [
    "KINDS",
    "KernelError",
    "MAX_RANK",
    "OpKindSpec",
    "default_registry",
    "conv_out_dim",
    "pool_out_dim",
]

MAX_RANK = 4


class KernelError(RuntimeError):
    """A kernel was applied to nonconforming data or produced non-finite values."""


@dataclass(frozen=True)
class OpKindSpec:
    """Static description of an operator kind (ops.py:499-515)."""

    kind: str
    min_in: int
    max_in: int | None
    n_out: int | None
    check_shapes: Callable[[list, list, dict], None]
    execute: Callable[[object, object], None]
    crosses_location: bool = False


def _req(ok: bool, msg: str) -> None:
    if not ok:
        raise KernelError(msg)


def _arity(kind, ins, outs, n_in, n_out):
    _req(len(ins) == n_in and len(outs) == n_out,
         f"{kind}: expected {n_in} inputs / {n_out} outputs, got {len(ins)} / {len(outs)}")


def _same(kind, got, want, what):
    _req(tuple(got) == tuple(want), f"{kind}: {what} is {tuple(got)}, expected {tuple(want)}")


# ---------------------------------------------------------------------------
# output-size rules


def conv_out_dim(size: int, k: int, stride: int, pad: int, floor: bool = False) -> int:
    """ops.py:229-240; ``floor=True`` selects Caffe's floor rule (GoogLeNet
    conv1 7x7/2 p3 and NIN conv1 11x11/4 at 224 need it)."""
    span = size + 2 * pad - k
    if span < 0 or (not floor and span % stride != 0):
        raise KernelError(f"conv2d: non-integral output dim for size={size} "
                          f"kernel={k} stride={stride} pad={pad}")
    return span // stride + 1


def pool_out_dim(size: int, k: int, stride: int, pad: int) -> int:
    """Caffe ceil-mode pooling size (window may not start in right padding)."""
    if size + 2 * pad < k or stride < 1 or pad < 0:
        raise KernelError(f"pool: kernel {k} does not fit size={size} pad={pad}")
    out = -(-(size + 2 * pad - k) // stride) + 1
    if pad > 0 and (out - 1) * stride >= size + pad:
        out -= 1
    return out


def conv_attrs(attrs: dict) -> tuple[int, int, bool]:
    stride = int(attrs.get("stride", 1))
    pad = int(attrs.get("pad", 0))
    _req(stride >= 1, f"conv2d: stride must be >= 1, got {stride}")
    _req(pad >= 0, f"conv2d: pad must be >= 0, got {pad}")
    return stride, pad, bool(attrs.get("floor", False))


def pool_attrs(attrs: dict) -> tuple[int, int, int]:
    _req("kernel" in attrs, "pool: missing required attr 'kernel'")
    k, s, p = int(attrs["kernel"]), int(attrs.get("stride", 1)), int(attrs.get("pad", 0))
    _req(k >= 1 and s >= 1 and 0 <= p < k, f"pool: bad kernel/stride/pad {k}/{s}/{p}")
    return k, s, p


def lrn_attrs(attrs: dict) -> tuple[int, float, float, float]:
    size = int(attrs.get("size", 5))
    _req(size >= 1, "lrn: size must be >= 1")
    return size, float(attrs.get("alpha", 1e-4)), float(attrs.get("beta", 0.75)), \
        float(attrs.get("k", 1.0))


def _conv_shape(x, w, attrs):
    _req(len(x) == 4 and len(w) == 4, f"conv2d: bad ranks x{x} w{w}")
    _req(w[1] == x[1], f"conv2d: channel mismatch x{x} w{w}")
    s, p, fl = conv_attrs(attrs)
    return (x[0], w[0], conv_out_dim(x[2], w[2], s, p, fl), conv_out_dim(x[3], w[3], s, p, fl))


def _fc_shape(x, w, b):
    _req(len(x) == 2 and len(w) == 2 and len(b) == 1, f"fc: bad ranks x{x} w{w} b{b}")
    _req(x[1] == w[0] and w[1] == b[0], f"fc: shapes do not conform: x{x} w{w} b{b}")
    return (x[0], w[1])


def _pool_shape(x, attrs):
    _req(len(x) == 4, f"pool: x must be 4-d, got {x}")
    k, s, p = pool_attrs(attrs)
    return (x[0], x[1], pool_out_dim(x[2], k, s, p), pool_out_dim(x[3], k, s, p))


# ---------------------------------------------------------------------------
# shape checkers


def _ck_fc_forward(ins, outs, a):
    _arity("fc_forward", ins, outs, 3, 1)
    _same("fc_forward", outs[0], _fc_shape(*ins), "output shape")


def _ck_fc_backward(ins, outs, a):
    _arity("fc_backward", ins, outs, 3, 3)
    x, w, dy = ins
    _same("fc_backward", dy, _fc_shape(x, w, (w[1],)), "dy shape")
    _same("fc_backward", outs[0], x, "dx shape")
    _same("fc_backward", outs[1], w, "dw shape")
    _same("fc_backward", outs[2], (w[1],), "db shape")


def _ck_fc_backward_data(ins, outs, a):
    _arity("fc_backward_data", ins, outs, 2, 1)
    w, dy = ins
    _req(len(w) == 2 and len(dy) == 2 and dy[1] == w[1], "fc_backward_data: shapes do not conform")
    _same("fc_backward_data", outs[0], (dy[0], w[0]), "dx shape")


def _ck_fc_backward_weight(ins, outs, a):
    _arity("fc_backward_weight", ins, outs, 2, 1)
    x, dy = ins
    _req(len(x) == 2 and len(dy) == 2 and x[0] == dy[0], "fc_backward_weight: shapes do not conform")
    _same("fc_backward_weight", outs[0], (x[1], dy[1]), "dw shape")


def _ck_fc_backward_bias(ins, outs, a):
    _arity("fc_backward_bias", ins, outs, 1, 1)
    _req(len(ins[0]) == 2, "fc_backward_bias: dy must be 2-d")
    _same("fc_backward_bias", outs[0], (ins[0][1],), "db shape")


def _ck_conv_forward(ins, outs, a):
    _arity("conv2d_forward", ins, outs, 3, 1)
    x, w, b = ins
    _req(len(b) == 1 and b[0] == w[0], f"conv2d_forward: bad bias shape {b}")
    _same("conv2d_forward", outs[0], _conv_shape(x, w, a), "output shape")


def _ck_conv_backward(ins, outs, a):
    _arity("conv2d_backward", ins, outs, 3, 3)
    x, w, dy = ins
    _same("conv2d_backward", dy, _conv_shape(x, w, a), "dy shape")
    _same("conv2d_backward", outs[0], x, "dx shape")
    _same("conv2d_backward", outs[1], w, "dw shape")
    _same("conv2d_backward", outs[2], (w[0],), "db shape")


def _ck_conv_backward_data(ins, outs, a):
    _arity("conv2d_backward_data", ins, outs, 3, 1)
    x, w, dy = ins
    _same("conv2d_backward_data", dy, _conv_shape(x, w, a), "dy shape")
    _same("conv2d_backward_data", outs[0], x, "dx shape")


def _ck_conv_backward_weight(ins, outs, a):
    _arity("conv2d_backward_weight", ins, outs, 3, 1)
    x, w, dy = ins
    _same("conv2d_backward_weight", dy, _conv_shape(x, w, a), "dy shape")
    _same("conv2d_backward_weight", outs[0], w, "dw shape")


def _ck_conv_backward_bias(ins, outs, a):
    _arity("conv2d_backward_bias", ins, outs, 1, 1)
    _req(len(ins[0]) == 4, "conv2d_backward_bias: dy must be 4-d")
    _same("conv2d_backward_bias", outs[0], (ins[0][1],), "db shape")


def _ck_relu_forward(ins, outs, a):
    _arity("relu_forward", ins, outs, 1, 1)
    _same("relu_forward", outs[0], ins[0], "output shape")


def _ck_relu_backward(ins, outs, a):
    _arity("relu_backward", ins, outs, 2, 1)
    _same("relu_backward", ins[1], ins[0], "dy shape")
    _same("relu_backward", outs[0], ins[0], "dx shape")


def _flat(x):
    n = 1
    for d in x[1:]:
        n *= d
    return (x[0], n)


def _ck_flatten_forward(ins, outs, a):
    _arity("flatten_forward", ins, outs, 1, 1)
    _req(len(ins[0]) >= 2, "flatten_forward: input must have >= 2 dims")
    _same("flatten_forward", outs[0], _flat(ins[0]), "output shape")


def _ck_flatten_backward(ins, outs, a):
    _arity("flatten_backward", ins, outs, 2, 1)
    x, dy = ins
    _same("flatten_backward", dy, _flat(x), "dy shape")
    _same("flatten_backward", outs[0], x, "dx shape")


def _ck_softmax_xent(ins, outs, a):
    _arity("softmax_xent", ins, outs, 2, 2)
    logits, labels = ins
    _req(len(logits) == 2, "softmax_xent: logits must be 2-d")
    _same("softmax_xent", labels, (logits[0],), "labels shape")
    _same("softmax_xent", outs[0], (1,), "loss shape")
    _same("softmax_xent", outs[1], logits, "dlogits shape")


def _ck_sgd_update(ins, outs, a):
    _arity("sgd_update", ins, outs, 2, 1)
    _same("sgd_update", ins[1], ins[0], "grad shape")
    _same("sgd_update", outs[0], ins[0], "output shape")
    _req("lr" in a, "sgd_update: missing required attr 'lr'")


def _ck_sgd_momentum(ins, outs, a):
    _arity("sgd_momentum", ins, outs, 3, 2)
    for i, s in enumerate(ins[1:] + outs):
        _same("sgd_momentum", s, ins[0], f"operand {i + 1} shape")
    _req("lr" in a, "sgd_momentum: missing required attr 'lr'")


def _ck_aggregate(ins, outs, a):
    _req(len(ins) >= 1, "aggregate: need at least one input")
    _req(len(outs) == 1, "aggregate: exactly one output")
    mode = a.get("mode", "mean")
    _req(mode in ("sum", "mean"), f"aggregate: unknown mode {mode!r}")
    for i, s in enumerate(ins):
        _same("aggregate", s, ins[0], f"input {i} shape")
    _same("aggregate", outs[0], ins[0], "output shape")


def _ck_swap(ins, outs, a):
    _req(len(ins) == 0, "swap: takes no inputs")
    _req(len(outs) == 2, "swap: exactly two outputs")
    _same("swap", outs[1], outs[0], "second buffer shape")


def _ck_copy(ins, outs, a):
    _arity("copy", ins, outs, 1, 1)
    _same("copy", outs[0], ins[0], "output shape")


def _ck_maxpool_forward(ins, outs, a):
    _arity("maxpool_forward", ins, outs, 1, 2)
    y = _pool_shape(ins[0], a)
    _same("maxpool_forward", outs[0], y, "output shape")
    _same("maxpool_forward", outs[1], y, "mask shape")


def _ck_maxpool_backward(ins, outs, a):
    _arity("maxpool_backward", ins, outs, 3, 1)
    x, mask, dy = ins
    _same("maxpool_backward", dy, _pool_shape(x, a), "dy shape")
    _same("maxpool_backward", mask, dy, "mask shape")
    _same("maxpool_backward", outs[0], x, "dx shape")


def _ck_avgpool_forward(ins, outs, a):
    _arity("avgpool_forward", ins, outs, 1, 1)
    _same("avgpool_forward", outs[0], _pool_shape(ins[0], a), "output shape")


def _ck_avgpool_backward(ins, outs, a):
    _arity("avgpool_backward", ins, outs, 2, 1)
    x, dy = ins
    _same("avgpool_backward", dy, _pool_shape(x, a), "dy shape")
    _same("avgpool_backward", outs[0], x, "dx shape")


def _ck_lrn_forward(ins, outs, a):
    _arity("lrn_forward", ins, outs, 1, 2)
    _req(len(ins[0]) == 4, "lrn_forward: x must be 4-d")
    lrn_attrs(a)
    _same("lrn_forward", outs[0], ins[0], "output shape")
    _same("lrn_forward", outs[1], ins[0], "scale shape")


def _ck_lrn_backward(ins, outs, a):
    _arity("lrn_backward", ins, outs, 4, 1)
    for i, s in enumerate(ins[1:]):
        _same("lrn_backward", s, ins[0], f"input {i + 1} shape")
    _same("lrn_backward", outs[0], ins[0], "dx shape")


def _ck_concat_forward(ins, outs, a):
    _req(len(ins) >= 1 and len(outs) == 1, "concat_forward: >= 1 inputs, one output")
    first = ins[0]
    _req(len(first) == 4, "concat_forward: inputs must be 4-d")
    for s in ins:
        _req(len(s) == 4 and s[0] == first[0] and s[2:] == first[2:],
             f"concat_forward: input {s} does not stack with {first}")
    total = sum(s[1] for s in ins)
    _same("concat_forward", outs[0], (first[0], total, first[2], first[3]), "output shape")


def _ck_concat_backward(ins, outs, a):
    _req(len(ins) == 1 and len(outs) >= 1, "concat_backward: one input, >= 1 outputs")
    _req("channels" in a, "concat_backward: missing required attr 'channels'")
    ch = [int(c) for c in a["channels"]]
    dy = ins[0]
    _req(len(ch) == len(outs) and sum(ch) == dy[1], "concat_backward: channels do not sum")
    for c, s in zip(ch, outs):
        _same("concat_backward", s, (dy[0], c, dy[2], dy[3]), "piece shape")


def _ck_send(ins, outs, a):
    _req(len(ins) == 1 and len(outs) == 0, "send: one input, no outputs")
    _req("channel" in a, "send: missing required attr 'channel'")


def _ck_recv(ins, outs, a):
    _req(len(ins) == 0 and len(outs) == 1, "recv: no inputs, one output")
    _req("channel" in a, "recv: missing required attr 'channel'")


def _ck_gate(ins, outs, a):
    _req(len(ins) == 2 and len(outs) == 1, "gate: two inputs, one output")
    _same("gate", outs[0], ins[0], "output shape")


def _ck_dp_exchange(ins, outs, a):
    # lowered parameter-server subgraph (exchange.py):
    # [w..., (v_shard), dw...] -> [w_new..., (v_shard_new)]; v only with momentum > 0
    mom = float(a.get("momentum", 0.0) or 0.0) > 0
    n = len(outs) - mom
    _req(n >= 1 and len(ins) == 2 * n + mom,
         "dp_exchange: needs [w*, (v), dw*] -> [w_new*, (v_new)]")
    for i in range(n):
        _same("dp_exchange", ins[n + mom + i], ins[i], f"grad {i} shape")
        _same("dp_exchange", outs[i], ins[i], f"output {i} shape")
    if mom:
        _same("dp_exchange", outs[n], ins[n], "velocity shard shape")
    _req("lr" in a and "world" in a, "dp_exchange: needs attrs lr, world")


# (kind, min_in, max_in, n_out, checker, crosses_location)
_TABLE = [
    ("fc_forward", 3, 3, 1, _ck_fc_forward, False),
    ("fc_backward", 3, 3, 3, _ck_fc_backward, False),
    ("fc_backward_data", 2, 2, 1, _ck_fc_backward_data, False),
    ("fc_backward_weight", 2, 2, 1, _ck_fc_backward_weight, False),
    ("fc_backward_bias", 1, 1, 1, _ck_fc_backward_bias, False),
    ("conv2d_forward", 3, 3, 1, _ck_conv_forward, False),
    ("conv2d_backward", 3, 3, 3, _ck_conv_backward, False),
    ("conv2d_backward_data", 3, 3, 1, _ck_conv_backward_data, False),
    ("conv2d_backward_weight", 3, 3, 1, _ck_conv_backward_weight, False),
    ("conv2d_backward_bias", 1, 1, 1, _ck_conv_backward_bias, False),
    ("relu_forward", 1, 1, 1, _ck_relu_forward, False),
    ("relu_backward", 2, 2, 1, _ck_relu_backward, False),
    ("flatten_forward", 1, 1, 1, _ck_flatten_forward, False),
    ("flatten_backward", 2, 2, 1, _ck_flatten_backward, False),
    ("softmax_xent", 2, 2, 2, _ck_softmax_xent, False),
    ("sgd_update", 2, 2, 1, _ck_sgd_update, False),
    ("sgd_momentum", 3, 3, 2, _ck_sgd_momentum, False),
    ("aggregate", 1, None, 1, _ck_aggregate, False),
    ("swap", 0, 0, 2, _ck_swap, False),
    ("copy", 1, 1, 1, _ck_copy, True),
    ("send", 1, 1, 0, _ck_send, False),
    ("recv", 0, 0, 1, _ck_recv, False),
    ("gate", 2, 2, 1, _ck_gate, False),
    ("maxpool_forward", 1, 1, 2, _ck_maxpool_forward, False),
    ("maxpool_backward", 3, 3, 1, _ck_maxpool_backward, False),
    ("avgpool_forward", 1, 1, 1, _ck_avgpool_forward, False),
    ("avgpool_backward", 2, 2, 1, _ck_avgpool_backward, False),
    ("lrn_forward", 1, 1, 2, _ck_lrn_forward, False),
    ("lrn_backward", 4, 4, 1, _ck_lrn_backward, False),
    ("concat_forward", 1, None, 1, _ck_concat_forward, False),
    ("concat_backward", 1, 1, None, _ck_concat_backward, False),
    ("dp_exchange", 2, None, None, _ck_dp_exchange, False),
]


def _unbound(kind):
    def execute(ctx, op):
        raise KernelError(f"{kind}: no device implementation is registered")
    return execute


def _build() -> dict[str, OpKindSpec]:
    from . import gpu_ops  # execute hooks; importing does not load the CUDA library

    table = {}
    for kind, lo, hi, nout, check, crosses in _TABLE:
        execute = gpu_ops.EXECUTORS.get(kind) or _unbound(kind)
        table[kind] = OpKindSpec(kind, lo, hi, nout, check, execute, crosses)
    return table


KINDS: dict[str, OpKindSpec] = _build()


def default_registry() -> dict[str, OpKindSpec]:
    """A fresh copy of the built-in kind table, safe to extend (ops.py:807-809)."""
    return dict(KINDS)
