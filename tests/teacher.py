"""Teacher-forced comparison of one executed training graph (test helper).

Every operator of the graph is re-run by a CPU reference on the GPU's OWN
input tensors and its outputs are compared with the GPU's.  Tensors the
fusion plan never materialises (`_Plan.elided`: concat parts, folded ReLU
gradients, the LRN scale) are taken from the reference's own output of the
same pass, so fused chains (conv + ReLU epilogue, data gradient + folded
relu_backward, concat-elided Inception modules) are checked end to end on
identical inputs.  After a full captured step the swap graph has exchanged
every ``w`` / ``w_new`` pair; `pre_swap` maps a name to the buffer that held
it while the training graph ran.
"""

from __future__ import annotations

import numpy as np

CONTRACTIONS = ("conv2d_forward", "conv2d_backward", "conv2d_backward_data",
                "conv2d_backward_weight", "conv2d_backward_bias", "fc_forward", "fc_backward",
                "fc_backward_data", "fc_backward_weight", "fc_backward_bias")
BITWISE = ("relu_forward", "relu_backward", "maxpool_forward", "maxpool_backward",
           "avgpool_forward", "avgpool_backward", "concat_forward", "concat_backward",
           "flatten_forward", "flatten_backward", "sgd_update", "sgd_momentum", "aggregate",
           "dp_exchange")


def pre_swap_map(swap_graph) -> dict[str, str]:
    out = {}
    for op in swap_graph.operators.values():
        a, b = (swap_graph.tensors[t].name for t in op.outputs)
        out[a], out[b] = b, a
    return out


def dp_exchange_ref(ins, attrs):
    """The lowered exchange at world 1 = aggregate(mean of 1) + sgd_update /
    sgd_momentum per parameter (builders.py:581-611)."""
    import oracle

    mu = float(attrs.get("momentum", 0.0) or 0.0)
    nb = len(attrs["offsets"])
    ws, gs = ins[:nb], ins[len(ins) - nb:]
    if mu > 0:
        raise NotImplementedError("momentum shards are checked by test_gpu_exchange")
    return [oracle.sgd_update(w, oracle.aggregate([g], "mean"), float(attrs["lr"]))
            for w, g in zip(ws, gs)]


def teacher_force(graph, read, materialised, reference, on_output, skip=(), mask_of=None):
    """Walk ``graph`` in serial order.  ``read(name)`` -> GPU array,
    ``materialised(name)`` -> whether the GPU wrote it, ``reference(kind,
    inputs, attrs)`` -> list of arrays, ``on_output(op, name, got, want,
    inexact)`` compares one output; ``inexact`` is false for a bit-exact kind
    on GPU inputs, else the kind of the floating-point operator the result
    depends on: the op's own kind, or -- when an input was the reference's
    own value of a tensor the GPU never stored -- the kind that value came
    from, directly or through bit-exact kinds (e.g. a ReLU gradient folded
    into a data-gradient epilogue: bit-exact select, but of a contraction's
    result; a ReLU output whose pre-activation was never stored: the
    forward convolution's).  ``mask_of(tensor_id)`` -> the GPU's stand-in for
    an unstored relu_backward mask (the ReLU output, relu(a) > 0 <=> a > 0:
    what the GPU's kernel reads) or None.  Returns the number of outputs
    compared."""
    from oracle.serial import serial_order

    own: dict[str, np.ndarray] = {}
    inexact_own: dict[str, str] = {}  # own value -> kind of the floating-point op it came from
    n = 0
    for oid in serial_order(graph):
        op = graph.operators[oid]
        if op.kind in skip or op.kind in ("swap", "copy"):
            continue
        ins, inexact = [], (op.kind if op.kind not in BITWISE else False)
        for i, t in enumerate(op.inputs):
            name = graph.tensors[t].name
            stand_in = (mask_of(t) if mask_of is not None and op.kind == "relu_backward"
                        and i == 0 and not materialised(name) else None)
            if stand_in is not None:
                ins.append(stand_in)
            elif materialised(name):
                ins.append(read(name))
            else:
                ins.append(own[name])
                inexact = inexact or inexact_own.get(name, False)
        want = reference(op.kind, ins, dict(op.attrs))
        for t, w in zip(op.outputs, want):
            name = graph.tensors[t].name
            if materialised(name):
                on_output(op, name, read(name), w, inexact)
                n += 1
            else:
                own[name] = w
                if inexact:
                    inexact_own[name] = inexact
    return n


class Tally:
    """Per-kind worst errors: unscaled max |d|, max |d| / max |want|, and the
    count of elements outside |d| <= atol + rtol |want| (unscaled NS bound)."""

    def __init__(self, rtol=1e-4, atol=1e-5):
        self.rtol, self.atol = rtol, atol
        self.rows: dict[str, list] = {}
        self.failures: list[tuple[str, str]] = []  # (kind, message)

    @property
    def fails(self) -> list[str]:
        return [m for _, m in self.failures]

    def fails_except(self, kinds) -> list[str]:
        return [m for k, m in self.failures if k not in kinds]

    def close(self, op, name, got, want):
        got = np.asarray(got, np.float64)
        want = np.asarray(want, np.float64)
        assert got.shape == want.shape, (op.name, name, got.shape, want.shape)
        d = np.abs(got - want)
        scale = max(float(np.abs(want).max()), 1e-30)
        bad = int((d > self.atol + self.rtol * np.abs(want)).sum())
        row = self.rows.setdefault(op.kind, [0, 0.0, 0.0, 0, ""])
        row[0] += 1
        if float(d.max()) > row[1]:
            row[1], row[4] = float(d.max()), f"{op.name}:{name}"
        row[2] = max(row[2], float(d.max()) / scale)
        row[3] += bad
        if bad:
            self.failures.append((op.kind, f"{op.name} -> {name}: {bad}/{d.size} outside rel "
                                           f"{self.rtol} / abs {self.atol}, max |d| "
                                           f"{float(d.max()):.3e} (scale {scale:.3e})"))

    def exact(self, op, name, got, want):
        got = np.ascontiguousarray(got, np.float32)
        want = np.ascontiguousarray(want, np.float32)
        assert got.shape == want.shape, (op.name, name)
        diff = int((got.view(np.uint32) != want.view(np.uint32)).sum())
        row = self.rows.setdefault(op.kind, [0, 0.0, 0.0, 0, ""])
        row[0] += 1
        row[3] += diff
        if diff:
            self.failures.append((op.kind, f"{op.name} -> {name}: {diff} elements differ bitwise"))

    def table(self) -> str:
        out = ["| kind | outputs | max abs err (unscaled) | max err / max abs | NS fails | worst |",
               "|---|---|---|---|---|---|"]
        for k, (n, mx, sc, bad, where) in sorted(self.rows.items()):
            out.append(f"| {k} | {n} | {mx:.3e} | {sc:.3e} | {bad} | {where} |")
        return "\n".join(out)
