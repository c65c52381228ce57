"""Algorithmic work accounting for the roofline.

FLOPs count 2 per multiply-accumulate of the algorithm (never x3 for the
split-TF32 passes); bytes count each tensor read or written once by the
kernel, fp32 = 4 B.
"""

from __future__ import annotations

from math import prod

CONTRACTION_KINDS = frozenset({"conv2d_forward", "conv2d_backward", "conv2d_backward_data",
                               "conv2d_backward_weight", "fc_forward", "fc_backward",
                               "fc_backward_data", "fc_backward_weight"})


def _shape(g, tid):
    return g.tensors[tid].shape


def op_flops(g, op) -> int:
    """Algorithmic FLOPs of one operator (contractions only; others 0)."""
    k = op.kind
    if k.startswith("conv2d") and k != "conv2d_backward_bias":
        x = _shape(g, op.inputs[0])
        w = _shape(g, op.inputs[1])
        if k == "conv2d_forward":
            y = _shape(g, op.outputs[0])
        else:
            y = _shape(g, op.inputs[2])
        macs = y[0] * y[1] * y[2] * y[3] * w[1] * w[2] * w[3]
        passes = 3 if k == "conv2d_backward" else 1
        return 2 * macs * passes
    if k.startswith("fc") and k != "fc_backward_bias":
        if k == "fc_forward":
            x, w = _shape(g, op.inputs[0]), _shape(g, op.inputs[1])
            return 2 * x[0] * w[0] * w[1]
        if k == "fc_backward":
            x, w = _shape(g, op.inputs[0]), _shape(g, op.inputs[1])
            return 3 * 2 * x[0] * w[0] * w[1]
        if k == "fc_backward_data":
            w, dy = _shape(g, op.inputs[0]), _shape(g, op.inputs[1])
            return 2 * dy[0] * w[0] * w[1]
        x, dy = _shape(g, op.inputs[0]), _shape(g, op.inputs[1])
        return 2 * x[0] * x[1] * dy[1]
    return 0


def op_bytes(g, op) -> int:
    """Algorithmic HBM bytes: every input and output tensor once (fp32)."""
    if op.kind in ("swap", "flatten_forward", "flatten_backward"):
        return 0
    return 4 * sum(prod(_shape(g, t)) for t in (*op.inputs, *op.outputs))
