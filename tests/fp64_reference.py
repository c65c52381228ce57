"""Float64 ground truth for DAG nets (test infrastructure).

Runs a `DagNet` forward + backward with torch autograd in float64 on the
CPU from the same parameters and batch, so GPU and oracle float32 results
can both be measured against exact-ish arithmetic.  Layer semantics follow
the oracle (Caffe ceil-mode pooling, LRN across channels, floor-mode conv).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F


def _pool_pad_ceil(nd):
    return dict(kernel_size=nd.kernel, stride=nd.stride, padding=nd.pad, ceil_mode=True)


def dag_grads_fp64(net, params: dict, x: np.ndarray, labels: np.ndarray, acts: dict | None = None):
    """Returns (loss, {param name: grad}) in float64.  If ``acts`` is a dict it
    receives ``a{pos}`` -> (activation, activation gradient)."""
    P = {k: torch.tensor(np.asarray(v, np.float64), requires_grad=True)
         for k, v in params.items()}
    vals = {"data": torch.tensor(np.asarray(x, np.float64))}
    for i, nd in enumerate(net.nodes):
        pos = i + 1
        src = [vals[s] for s in nd.inputs]
        if nd.kind == "conv":
            y = F.conv2d(src[0], P[f"w{pos}"], P[f"b{pos}"], stride=nd.stride, padding=nd.pad)
        elif nd.kind == "fc":
            y = src[0].reshape(src[0].shape[0], -1) @ P[f"w{pos}"] + P[f"b{pos}"]
        elif nd.kind == "relu":
            y = torch.relu(src[0])
        elif nd.kind == "maxpool":
            y = F.max_pool2d(src[0], **_pool_pad_ceil(nd))
        elif nd.kind == "avgpool":
            assert nd.pad == 0
            y = F.avg_pool2d(src[0], **_pool_pad_ceil(nd))
        elif nd.kind == "lrn":
            y = F.local_response_norm(src[0], nd.size, alpha=nd.alpha, beta=nd.beta, k=nd.k)
        elif nd.kind == "concat":
            y = torch.cat(src, dim=1)
        else:
            raise ValueError(nd.kind)
        if acts is not None:
            y.retain_grad()
        vals[nd.name] = y
    logits = vals[net.nodes[-1].name]
    logits = logits.reshape(logits.shape[0], -1)
    loss = F.cross_entropy(logits, torch.tensor(np.asarray(labels).astype(np.int64)))
    loss.backward()
    if acts is not None:
        for i, nd in enumerate(net.nodes):
            t = vals[nd.name]
            acts[f"a{i + 1}"] = (t.detach().numpy(), None if t.grad is None else t.grad.numpy())
    return float(loss.detach()), {k: v.grad.numpy() for k, v in P.items()}
