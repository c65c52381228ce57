"""DAG networks for the NS configurations the reference's linear `NetSpec`
cannot express (builders.py:112-160 only chains fc/conv/relu): the
CIFAR-shaped conv-pool net (config 2), Network-in-Network (config 3) and
GoogLeNet / Inception v1 (config 4, the paper's headline).

A `DagNet` plugs into `builders.build_sgd_iteration` / `build_data_parallel`
through the same hooks a `NetSpec` provides (`param_shapes`,
`emit_forward`, `emit_backward`) and follows the reference's naming scheme:
node ``pos`` (1-based) outputs ``a{pos}`` and owns ``w{pos}``/``b{pos}``,
gradients are ``d<tensor>``, replicas append ``_p{k}``.

Backward specifics (the reference has no DAG, so these are our choices,
documented in DESIGN.md):
  * gradient fan-in where a tensor feeds several branches (Inception
    inputs) is an ``aggregate(mode="sum")`` over per-consumer partials
    ``d<T>_c{pos}`` in ascending consumer order;
  * conv / fc backward is always split; weight and bias gradients are
    inserted before the data gradient so a layer's parameter exchange can
    start while its data gradient still runs; the data gradient of the
    network input is never computed (as the reference's split mode).
"""

from __future__ import annotations

from dataclasses import dataclass

from .graph import GraphError
from .kinds import conv_out_dim, pool_out_dim

__all__ = ["Node", "DagNet", "googlenet", "nin", "cifar_convnet", "conv_relu_fc"]


@dataclass(frozen=True)
class Node:
    name: str
    kind: str  # conv | fc | relu | maxpool | avgpool | lrn | concat
    inputs: tuple[str, ...]
    out: int = 0
    kernel: int = 0
    stride: int = 1
    pad: int = 0
    floor: bool = False
    size: int = 5
    alpha: float = 1e-4
    beta: float = 0.75
    k: float = 1.0


@dataclass(frozen=True)
class DagNet:
    input_shape: tuple[int, ...]
    nodes: tuple[Node, ...]
    batch: int = 1
    lr: float = 0.01
    momentum: float = 0.0
    name: str = "dag"

    def __post_init__(self) -> None:
        object.__setattr__(self, "input_shape", tuple(self.input_shape))
        object.__setattr__(self, "nodes", tuple(self.nodes))
        if self.batch < 1:
            raise GraphError(f"batch must be >= 1, got {self.batch}")
        self._resolved()

    # ---- shape resolution --------------------------------------------------

    def _resolved(self):
        cached = self.__dict__.get("_cache")
        if cached is not None:
            return cached
        pos_of: dict[str, int] = {}
        shapes: dict[str, tuple[int, ...]] = {"data": (self.batch, *self.input_shape)}
        tensor_of = {"data": "x"}
        params = []
        for i, nd in enumerate(self.nodes):
            pos = i + 1
            if nd.name in pos_of or nd.name == "data":
                raise GraphError(f"duplicate node name {nd.name!r}")
            for src in nd.inputs:
                if src not in shapes:
                    raise GraphError(f"node {nd.name!r}: unknown input {src!r}")
            ins = [shapes[s] for s in nd.inputs]
            if nd.kind == "conv":
                x = ins[0]
                if len(x) != 4:
                    raise GraphError(f"node {nd.name!r}: conv needs a 4-d input")
                y = (x[0], nd.out, conv_out_dim(x[2], nd.kernel, nd.stride, nd.pad, nd.floor),
                     conv_out_dim(x[3], nd.kernel, nd.stride, nd.pad, nd.floor))
                params += [(f"w{pos}", (nd.out, x[1], nd.kernel, nd.kernel)), (f"b{pos}", (nd.out,))]
            elif nd.kind == "fc":
                x = ins[0]
                d = 1
                for v in x[1:]:
                    d *= v
                y = (x[0], nd.out)
                params += [(f"w{pos}", (d, nd.out)), (f"b{pos}", (nd.out,))]
            elif nd.kind in ("relu", "lrn"):
                y = ins[0]
            elif nd.kind in ("maxpool", "avgpool"):
                x = ins[0]
                y = (x[0], x[1], pool_out_dim(x[2], nd.kernel, nd.stride, nd.pad),
                     pool_out_dim(x[3], nd.kernel, nd.stride, nd.pad))
            elif nd.kind == "concat":
                c = sum(s[1] for s in ins)
                y = (ins[0][0], c, ins[0][2], ins[0][3])
            else:
                raise GraphError(f"node {nd.name!r}: unknown kind {nd.kind!r}")
            pos_of[nd.name] = pos
            shapes[nd.name] = y
            tensor_of[nd.name] = f"a{pos}"
        last = self.nodes[-1].name
        logits = shapes[last]
        flat = 1
        for v in logits[1:]:
            flat *= v
        if flat < 2:
            raise GraphError("loss needs >= 2 logit columns")
        cache = {"pos": pos_of, "shapes": shapes, "tensor": tensor_of, "params": params,
                 "classes": flat}
        object.__setattr__(self, "_cache", cache)
        return cache

    @property
    def classes(self) -> int:
        return self._resolved()["classes"]

    def param_shapes(self):
        return list(self._resolved()["params"])

    def macs_per_image(self) -> dict[str, int]:
        """Forward multiply-accumulates per image (conv + fc)."""
        r = self._resolved()
        conv = fc = 0
        for nd in self.nodes:
            y = r["shapes"][nd.name]
            if nd.kind == "conv":
                cin = r["shapes"][nd.inputs[0]][1]
                conv += y[1] * y[2] * y[3] * cin * nd.kernel * nd.kernel
            elif nd.kind == "fc":
                x = r["shapes"][nd.inputs[0]]
                d = 1
                for v in x[1:]:
                    d *= v
                fc += d * nd.out
        return {"conv": conv, "fc": fc}

    # ---- graph emission ------------------------------------------------------

    def emit_forward(self, g, sfx, loc, thread):
        r = self._resolved()
        g.add_tensor(f"x{sfx}", r["shapes"]["data"], loc)
        for pname, shape in r["params"]:
            g.add_tensor(f"{pname}{sfx}", shape, loc)
        tape = []
        for i, nd in enumerate(self.nodes):
            pos = i + 1
            ins = [r["tensor"][s] + sfx for s in nd.inputs]
            out = f"a{pos}{sfx}"
            shape = r["shapes"][nd.name]
            if nd.kind == "conv":
                g.add_tensor(out, shape, loc)
                attrs = {"stride": nd.stride, "pad": nd.pad}
                if nd.floor:
                    attrs["floor"] = True
                g.add_operator(f"conv{pos}{sfx}", "conv2d_forward",
                               [g.tensor_id(ins[0]), g.tensor_id(f"w{pos}{sfx}"),
                                g.tensor_id(f"b{pos}{sfx}")], [g.tensor_id(out)], loc,
                               thread=thread, attrs=attrs)
            elif nd.kind == "fc":
                src = ins[0]
                if len(g.tensor_named(src).shape) != 2:
                    flat = f"{r['tensor'][nd.inputs[0]]}_flat{sfx}"
                    xs = g.tensor_named(src).shape
                    d = 1
                    for v in xs[1:]:
                        d *= v
                    g.add_tensor(flat, (xs[0], d), loc)
                    g.add_operator(f"flatten{pos}{sfx}", "flatten_forward", [g.tensor_id(src)],
                                   [g.tensor_id(flat)], loc, thread=thread)
                    src = flat
                g.add_tensor(out, shape, loc)
                g.add_operator(f"fc{pos}{sfx}", "fc_forward",
                               [g.tensor_id(src), g.tensor_id(f"w{pos}{sfx}"),
                                g.tensor_id(f"b{pos}{sfx}")], [g.tensor_id(out)], loc,
                               thread=thread)
            elif nd.kind == "relu":
                g.add_tensor(out, shape, loc)
                g.add_operator(f"relu{pos}{sfx}", "relu_forward", [g.tensor_id(ins[0])],
                               [g.tensor_id(out)], loc, thread=thread)
            elif nd.kind == "maxpool":
                g.add_tensor(out, shape, loc)
                g.add_tensor(f"mask{pos}{sfx}", shape, loc)
                g.add_operator(f"maxpool{pos}{sfx}", "maxpool_forward", [g.tensor_id(ins[0])],
                               [g.tensor_id(out), g.tensor_id(f"mask{pos}{sfx}")], loc,
                               thread=thread,
                               attrs={"kernel": nd.kernel, "stride": nd.stride, "pad": nd.pad})
            elif nd.kind == "avgpool":
                g.add_tensor(out, shape, loc)
                g.add_operator(f"avgpool{pos}{sfx}", "avgpool_forward", [g.tensor_id(ins[0])],
                               [g.tensor_id(out)], loc, thread=thread,
                               attrs={"kernel": nd.kernel, "stride": nd.stride, "pad": nd.pad})
            elif nd.kind == "lrn":
                g.add_tensor(out, shape, loc)
                g.add_tensor(f"scale{pos}{sfx}", shape, loc)
                g.add_operator(f"lrn{pos}{sfx}", "lrn_forward", [g.tensor_id(ins[0])],
                               [g.tensor_id(out), g.tensor_id(f"scale{pos}{sfx}")], loc,
                               thread=thread, attrs={"size": nd.size, "alpha": nd.alpha,
                                                     "beta": nd.beta, "k": nd.k})
            elif nd.kind == "concat":
                g.add_tensor(out, shape, loc)
                g.add_operator(f"concat{pos}{sfx}", "concat_forward",
                               [g.tensor_id(t) for t in ins], [g.tensor_id(out)], loc,
                               thread=thread)
            tape.append((pos, nd, ins, out))
        logits = tape[-1][3]
        if len(g.tensor_named(logits).shape) != 2:
            shp = g.tensor_named(logits).shape
            flat = f"{logits[:len(logits) - len(sfx)] if sfx else logits}_flat{sfx}"
            d = 1
            for v in shp[1:]:
                d *= v
            g.add_tensor(flat, (shp[0], d), loc)
            g.add_operator(f"flatten_out{sfx}", "flatten_forward", [g.tensor_id(logits)],
                           [g.tensor_id(flat)], loc, thread=thread)
            tape.append((len(self.nodes) + 1, None, [logits], flat))
            logits = flat
        return tape, logits

    def emit_backward(self, g, tape, sfx, loc, thread, dlogits, split):
        consumers: dict[str, list[int]] = {}
        for pos, nd, ins, _out in tape:
            for t in ins:
                consumers.setdefault(t, []).append(pos)
        x = f"x{sfx}"

        def grad_name(t, pos):
            return f"d{t}" if len(consumers.get(t, [])) == 1 else f"d{t}_c{pos}"

        grads = {}
        for pos, nd, ins, out in reversed(tape):
            dy = f"d{out}"
            cons = consumers.get(out, [])
            if len(cons) > 1:  # gradient fan-in: sum the partials in consumer order
                g.add_tensor(dy, g.tensor_named(out).shape, loc)
                g.add_operator(f"gsum_{out}", "aggregate",
                               [g.tensor_id(f"d{out}_c{c}") for c in sorted(cons)],
                               [g.tensor_id(dy)], loc, thread=thread, attrs={"mode": "sum"})
            if nd is None:  # trailing flatten before the loss
                g.add_tensor(grad_name(ins[0], pos), g.tensor_named(ins[0]).shape, loc)
                g.add_operator(f"bwd_flatten_out{sfx}", "flatten_backward",
                               [g.tensor_id(ins[0]), g.tensor_id(dy)],
                               [g.tensor_id(grad_name(ins[0], pos))], loc, thread=thread)
                continue
            src = ins[0]
            need = src != x
            gin = grad_name(src, pos)
            if nd.kind == "fc" and len(g.tensor_named(src).shape) != 2:
                src = f"{src[:len(src) - len(sfx)] if sfx else src}_flat{sfx}"
            if nd.kind in ("conv", "fc"):
                w, b = f"w{pos}{sfx}", f"b{pos}{sfx}"
                g.add_tensor(f"d{w}", g.tensor_named(w).shape, loc)
                g.add_tensor(f"d{b}", g.tensor_named(b).shape, loc)
                grads[pos] = [(w, f"d{w}", g.tensor_named(w).shape),
                              (b, f"d{b}", g.tensor_named(b).shape)]
                if nd.kind == "conv":
                    attrs = {"stride": nd.stride, "pad": nd.pad}
                    if nd.floor:
                        attrs["floor"] = True
                    g.add_operator(f"bwd_conv{pos}{sfx}_weight", "conv2d_backward_weight",
                                   [g.tensor_id(src), g.tensor_id(w), g.tensor_id(dy)],
                                   [g.tensor_id(f"d{w}")], loc, thread=thread, attrs=attrs)
                    g.add_operator(f"bwd_conv{pos}{sfx}_bias", "conv2d_backward_bias",
                                   [g.tensor_id(dy)], [g.tensor_id(f"d{b}")], loc, thread=thread)
                    if need:
                        g.add_tensor(gin, g.tensor_named(src).shape, loc)
                        g.add_operator(f"bwd_conv{pos}{sfx}_data", "conv2d_backward_data",
                                       [g.tensor_id(src), g.tensor_id(w), g.tensor_id(dy)],
                                       [g.tensor_id(gin)], loc, thread=thread, attrs=attrs)
                else:
                    g.add_operator(f"bwd_fc{pos}{sfx}_weight", "fc_backward_weight",
                                   [g.tensor_id(src), g.tensor_id(dy)], [g.tensor_id(f"d{w}")],
                                   loc, thread=thread)
                    g.add_operator(f"bwd_fc{pos}{sfx}_bias", "fc_backward_bias",
                                   [g.tensor_id(dy)], [g.tensor_id(f"d{b}")], loc, thread=thread)
                    if need:
                        flat_src = src
                        orig = ins[0] if src != ins[0] else None
                        if orig is not None:  # src is a flatten of a 4-d tensor
                            g.add_tensor(f"d{flat_src}", g.tensor_named(flat_src).shape, loc)
                            g.add_operator(f"bwd_fc{pos}{sfx}_data", "fc_backward_data",
                                           [g.tensor_id(w), g.tensor_id(dy)],
                                           [g.tensor_id(f"d{flat_src}")], loc, thread=thread)
                            og = grad_name(orig, pos)
                            g.add_tensor(og, g.tensor_named(orig).shape, loc)
                            g.add_operator(f"bwd_flatten{pos}{sfx}", "flatten_backward",
                                           [g.tensor_id(orig), g.tensor_id(f"d{flat_src}")],
                                           [g.tensor_id(og)], loc, thread=thread)
                        else:
                            g.add_tensor(gin, g.tensor_named(src).shape, loc)
                            g.add_operator(f"bwd_fc{pos}{sfx}_data", "fc_backward_data",
                                           [g.tensor_id(w), g.tensor_id(dy)], [g.tensor_id(gin)],
                                           loc, thread=thread)
                continue
            if not need:
                continue
            if nd.kind == "concat":
                outs = []
                for t in ins:
                    gn = grad_name(t, pos)
                    g.add_tensor(gn, g.tensor_named(t).shape, loc)
                    outs.append(g.tensor_id(gn))
                g.add_operator(f"bwd_concat{pos}{sfx}", "concat_backward", [g.tensor_id(dy)], outs,
                               loc, thread=thread,
                               attrs={"channels": [g.tensor_named(t).shape[1] for t in ins]})
                continue
            g.add_tensor(gin, g.tensor_named(src).shape, loc)
            if nd.kind == "relu":
                g.add_operator(f"bwd_relu{pos}{sfx}", "relu_backward",
                               [g.tensor_id(src), g.tensor_id(dy)], [g.tensor_id(gin)], loc,
                               thread=thread)
            elif nd.kind == "maxpool":
                g.add_operator(f"bwd_maxpool{pos}{sfx}", "maxpool_backward",
                               [g.tensor_id(src), g.tensor_id(f"mask{pos}{sfx}"), g.tensor_id(dy)],
                               [g.tensor_id(gin)], loc, thread=thread,
                               attrs={"kernel": nd.kernel, "stride": nd.stride, "pad": nd.pad})
            elif nd.kind == "avgpool":
                g.add_operator(f"bwd_avgpool{pos}{sfx}", "avgpool_backward",
                               [g.tensor_id(src), g.tensor_id(dy)], [g.tensor_id(gin)], loc,
                               thread=thread,
                               attrs={"kernel": nd.kernel, "stride": nd.stride, "pad": nd.pad})
            elif nd.kind == "lrn":
                g.add_operator(f"bwd_lrn{pos}{sfx}", "lrn_backward",
                               [g.tensor_id(src), g.tensor_id(out), g.tensor_id(f"scale{pos}{sfx}"),
                                g.tensor_id(dy)], [g.tensor_id(gin)], loc, thread=thread,
                               attrs={"size": nd.size, "alpha": nd.alpha, "beta": nd.beta,
                                      "k": nd.k})
        out = []
        for pos in sorted(grads):
            out += grads[pos]
        return out


# ---------------------------------------------------------------------------
# network zoo


class _Builder:
    def __init__(self):
        self.nodes: list[Node] = []

    def add(self, nd: Node) -> str:
        self.nodes.append(nd)
        return nd.name

    def conv(self, name, src, out, k, s=1, p=0, floor=False, relu=True):
        t = self.add(Node(name, "conv", (src,), out, k, s, p, floor))
        return self.add(Node(name + "/relu", "relu", (t,))) if relu else t

    def pool(self, name, src, kind, k, s, p=0):
        return self.add(Node(name, kind, (src,), kernel=k, stride=s, pad=p))

    def lrn(self, name, src):
        return self.add(Node(name, "lrn", (src,), size=5, alpha=1e-4, beta=0.75, k=1.0))


def googlenet(batch: int = 128, lr: float = 0.01, momentum: float = 0.0, image: int = 224,
              classes: int = 1000) -> DagNet:
    """GoogLeNet v1 (Szegedy et al. Table 1; bvlc_googlenet layout): main
    head only, no auxiliary heads, dropout p=0 (identity, omitted)."""
    b = _Builder()
    t = b.conv("conv1/7x7_s2", "data", 64, 7, 2, 3, floor=True)
    t = b.pool("pool1/3x3_s2", t, "maxpool", 3, 2)
    t = b.lrn("pool1/norm1", t)
    t = b.conv("conv2/3x3_reduce", t, 64, 1)
    t = b.conv("conv2/3x3", t, 192, 3, 1, 1)
    t = b.lrn("conv2/norm2", t)
    t = b.pool("pool2/3x3_s2", t, "maxpool", 3, 2)

    def inception(tag, src, c1, c3r, c3, c5r, c5, pp):
        p = f"inception_{tag}/"
        b1 = b.conv(p + "1x1", src, c1, 1)
        b2 = b.conv(p + "3x3", b.conv(p + "3x3_reduce", src, c3r, 1), c3, 3, 1, 1)
        b3 = b.conv(p + "5x5", b.conv(p + "5x5_reduce", src, c5r, 1), c5, 5, 1, 2)
        b4 = b.conv(p + "pool_proj", b.pool(p + "pool", src, "maxpool", 3, 1, 1), pp, 1)
        return b.add(Node(p + "output", "concat", (b1, b2, b3, b4)))

    t = inception("3a", t, 64, 96, 128, 16, 32, 32)
    t = inception("3b", t, 128, 128, 192, 32, 96, 64)
    t = b.pool("pool3/3x3_s2", t, "maxpool", 3, 2)
    t = inception("4a", t, 192, 96, 208, 16, 48, 64)
    t = inception("4b", t, 160, 112, 224, 24, 64, 64)
    t = inception("4c", t, 128, 128, 256, 24, 64, 64)
    t = inception("4d", t, 112, 144, 288, 32, 64, 64)
    t = inception("4e", t, 256, 160, 320, 32, 128, 128)
    t = b.pool("pool4/3x3_s2", t, "maxpool", 3, 2)
    t = inception("5a", t, 256, 160, 320, 32, 128, 128)
    t = inception("5b", t, 384, 192, 384, 48, 128, 128)
    final = image // 32
    t = b.pool("pool5/7x7_s1", t, "avgpool", final, 1)
    b.add(Node("loss3/classifier", "fc", (t,), classes))
    return DagNet((3, image, image), tuple(b.nodes), batch=batch, lr=lr, momentum=momentum,
                  name="googlenet")


def nin(batch: int = 128, lr: float = 0.01, momentum: float = 0.0, image: int = 224,
        classes: int = 1000) -> DagNet:
    """Network-in-Network for ImageNet (Lin et al.; Caffe model-zoo layout)."""
    b = _Builder()
    t = b.conv("conv1", "data", 96, 11, 4, 0, floor=True)
    t = b.conv("cccp1", t, 96, 1)
    t = b.conv("cccp2", t, 96, 1)
    t = b.pool("pool1", t, "maxpool", 3, 2)
    t = b.conv("conv2", t, 256, 5, 1, 2)
    t = b.conv("cccp3", t, 256, 1)
    t = b.conv("cccp4", t, 256, 1)
    t = b.pool("pool2", t, "maxpool", 3, 2)
    t = b.conv("conv3", t, 384, 3, 1, 1)
    t = b.conv("cccp5", t, 384, 1)
    t = b.conv("cccp6", t, 384, 1)
    t = b.pool("pool3", t, "maxpool", 3, 2)
    t = b.conv("conv4-1024", t, 1024, 3, 1, 1)
    t = b.conv("cccp7-1024", t, 1024, 1)
    t = b.conv("cccp8-1024", t, classes, 1)
    size = DagNet((3, image, image), tuple(b.nodes), batch=1)._resolved()["shapes"][t][2]
    b.pool("pool4", t, "avgpool", size, 1)
    return DagNet((3, image, image), tuple(b.nodes), batch=batch, lr=lr, momentum=momentum,
                  name="nin")


def cifar_convnet(batch: int = 16, lr: float = 1e-3, momentum: float = 0.0) -> DagNet:
    """Config 2: conv(32,5,p2)+relu -> maxpool 2/2 -> conv(64,5,p2)+relu ->
    maxpool 2/2 -> fc10 on 3x32x32."""
    b = _Builder()
    t = b.conv("conv1", "data", 32, 5, 1, 2)
    t = b.pool("pool1", t, "maxpool", 2, 2)
    t = b.conv("conv2", t, 64, 5, 1, 2)
    t = b.pool("pool2", t, "maxpool", 2, 2)
    b.add(Node("fc3", "fc", (t,), 10))
    return DagNet((3, 32, 32), tuple(b.nodes), batch=batch, lr=lr, momentum=momentum,
                  name="cifar_convnet")


def conv_relu_fc(batch: int = 16, lr: float = 1e-3):
    """Config 1 as a reference `NetSpec`: conv(32,k5,s1,p2) + relu + fc(10)."""
    from .builders import LayerSpec, NetSpec

    return NetSpec((3, 32, 32), (LayerSpec("conv", 32, 5, 1, 2), LayerSpec("relu"),
                                 LayerSpec("fc", 10)), batch=batch, lr=lr)
