"""Op-DAG builder: static nn.Module → fused op table + planner CompGraph.

Nimble's Graph Rewriter input is a TorchScript graph; here
it is a torch.fx trace plus ShapeProp on the example input (the paper's
"dummy input").  The builder then rewrites the graph the way a
B200 engine wants it before stream assignment:

  1. identities vanish (dropout, flatten of 1x1 maps, contiguous);
  2. BatchNorm folds into the producing conv (also across a concat: NASNet's
     factorized-reduction BN folds slice-wise into both paths); leftover BN
     becomes a per-channel affine op;
  3. residual adds fold into the epilogue of one producer (conv / depthwise /
     pool) — the other operand becomes that kernel's residual input;
  4. activations fold into the single-consumer producer's epilogue; a ReLU
     whose input is shared (NASNet "relu → sep-conv" branches) is instead
     applied on load by each consuming kernel (pre-activation), so it costs
     no kernel and no HBM round trip;
  5. concat is zero-copy: producers write straight into channel slices of
     the concat buffer (NHWC pixel stride = total channels), nested concats
     compose offsets; a copy op remains only when a tensor cannot be placed.

Every surviving node is one kernel task.  Task ids follow fx order; edges are
true data dependencies (writer of every consumed channel slice → reader), so
the planner sees exactly the DAG the engine runs.  ``fuse=False`` keeps one
task per fx op (conv, bn, relu, add, cat, pool …) — the unfused DAG of the
SURVEY probes — for parity and for measuring what fusion buys.
"""

from __future__ import annotations

import operator
from dataclasses import dataclass, field

import torch
import torch.fx as fx
import torch.nn as nn
import torch.nn.functional as F
from torch.fx.passes.shape_prop import ShapeProp

from .graph import CompGraph, MemEvent, TaskNode

ACT_NONE, ACT_RELU, ACT_RELU6, ACT_SILU, ACT_SIGMOID = 0, 1, 2, 3, 4
ALIGN = 256  # bytes; every storage starts 256-B aligned inside the arena


# ----------------------------------------------------------------------------
# IR
# ----------------------------------------------------------------------------

@dataclass(eq=False)
class INode:
    name: str
    kind: str
    inputs: list
    shape: tuple  # (N, C, H, W); 2-D tensors are (N, C, 1, 1)
    attrs: dict = field(default_factory=dict)
    act: int = ACT_NONE
    pre_relu: bool = False
    residual: "INode | None" = None
    alias_of: "INode | None" = None

    def __repr__(self):
        return f"<{self.kind} {self.name} {self.shape}>"


def _shape4(t):
    s = tuple(t)
    if len(s) == 4:
        return s
    if len(s) == 2:
        return (s[0], s[1], 1, 1)
    raise NotImplementedError(f"unsupported tensor rank {len(s)}")


class _Tracer(fx.Tracer):
    def is_leaf_module(self, m, qualname):
        return hasattr(m, "sw_spec") or super().is_leaf_module(m, qualname)


def _pair(v):
    return tuple(v) if isinstance(v, (tuple, list)) else (v, v)


def _conv_node(name, conv: nn.Conv2d, x, shape, stride=None, pad=None, groups_ok=True):
    if conv.dilation not in ((1, 1), 1):
        raise NotImplementedError("dilated conv")
    if conv.padding_mode != "zeros" or isinstance(conv.padding, str):
        raise NotImplementedError("padding mode")
    w = conv.weight.detach().float()
    b = conv.bias.detach().float() if conv.bias is not None else None
    g = conv.groups
    cin = x.shape[1]
    k_out = w.shape[0]
    attrs = {"weight": w, "bias": b, "stride": stride or _pair(conv.stride),
             "pad": pad if pad is not None else _pair(conv.padding), "k": tuple(w.shape[2:]),
             "module": conv}
    if g == 1:
        kind = "conv"
    elif g == cin == k_out:
        kind = "dwconv"
    else:
        raise NotImplementedError(f"grouped conv groups={g}")
    return INode(name, kind, [x], shape, attrs)


def trace_model(model: nn.Module, example: torch.Tensor) -> list[INode]:
    """fx trace + shape propagation → IR nodes in fx (topological) order."""
    model = model.eval()
    gm = fx.GraphModule(model, _Tracer().trace(model))
    with torch.no_grad():
        ShapeProp(gm).propagate(example)
    mods = dict(gm.named_modules())
    env: dict[fx.Node, INode] = {}
    out: list[INode] = []

    def shp(n):
        return _shape4(n.meta["tensor_meta"].shape)

    def arg(a):
        return env[a]

    for n in gm.graph.nodes:
        if n.op == "placeholder":
            node = INode("input", "input", [], shp(n))
        elif n.op == "output":
            res = n.args[0]
            node = INode("output", "output", [arg(res)], env[res].shape,
                         {"raw_shape": tuple(res.meta["tensor_meta"].shape)})
        elif n.op == "call_module":
            m = mods[n.target]
            x = arg(n.args[0]) if n.args else None
            name = n.target
            if hasattr(m, "sw_spec"):
                spec = m.sw_spec(x.shape)
                if spec["kind"] in ("conv", "dwconv"):
                    node = _conv_node(name, spec["module"], x, shp(n), stride=spec["stride"],
                                      pad=spec["pad"])
                    if node.kind != spec["kind"]:
                        raise AssertionError("spec kind mismatch")
                else:
                    node = INode(name, "pool", [x], shp(n),
                                 {"mode": spec["mode"], "k": spec["k"], "stride": spec["stride"],
                                  "pad": spec["pad"], "cip": spec["count_include_pad"]})
            elif isinstance(m, nn.Conv2d):
                node = _conv_node(name, m, x, shp(n))
            elif isinstance(m, nn.Linear):
                node = INode(name, "conv", [x], shp(n),
                             {"weight": m.weight.detach().float()[:, :, None, None],
                              "bias": m.bias.detach().float() if m.bias is not None else None,
                              "stride": (1, 1), "pad": (0, 0), "k": (1, 1), "linear": True,
                              "module": m})
            elif isinstance(m, nn.BatchNorm2d):
                inv = torch.rsqrt(m.running_var.detach().double() + m.eps)
                scale = m.weight.detach().double() * inv if m.affine else inv
                shift = (m.bias.detach().double() if m.affine else 0) - \
                    m.running_mean.detach().double() * scale
                node = INode(name, "bn", [x], shp(n), {"scale": scale, "shift": shift, "module": m})
            elif isinstance(m, (nn.ReLU, nn.ReLU6, nn.SiLU, nn.Sigmoid)):
                code = {nn.ReLU: ACT_RELU, nn.ReLU6: ACT_RELU6, nn.SiLU: ACT_SILU,
                        nn.Sigmoid: ACT_SIGMOID}[type(m)]
                node = INode(name, "act", [x], shp(n), {"act": code})
            elif isinstance(m, nn.MaxPool2d):
                if m.ceil_mode or _pair(m.dilation) != (1, 1):
                    raise NotImplementedError("maxpool ceil/dilation")
                node = INode(name, "pool", [x], shp(n),
                             {"mode": "max", "k": _pair(m.kernel_size),
                              "stride": _pair(m.stride or m.kernel_size), "pad": _pair(m.padding),
                              "cip": True})
            elif isinstance(m, nn.AvgPool2d):
                if m.ceil_mode:
                    raise NotImplementedError("avgpool ceil")
                node = INode(name, "pool", [x], shp(n),
                             {"mode": "avg", "k": _pair(m.kernel_size),
                              "stride": _pair(m.stride or m.kernel_size), "pad": _pair(m.padding),
                              "cip": bool(m.count_include_pad)})
            elif isinstance(m, nn.AdaptiveAvgPool2d):
                if tuple(shp(n)[2:]) != (1, 1):
                    raise NotImplementedError("adaptive pool to non-1x1")
                node = INode(name, "gpool", [x], shp(n))
            elif isinstance(m, (nn.Dropout, nn.Identity, nn.Flatten)):
                node = INode(name, "identity", [x], shp(n))
            else:
                raise NotImplementedError(f"module {type(m).__name__} ({n.target})")
        elif n.op in ("call_function", "call_method"):
            t = n.target
            name = n.name
            if t in (operator.add, operator.iadd, torch.add, "add", "add_"):
                a, b = n.args[0], n.args[1]
                if not isinstance(a, fx.Node) or not isinstance(b, fx.Node):
                    raise NotImplementedError("add with scalar")
                node = INode(name, "add", [arg(a), arg(b)], shp(n))
            elif t in (operator.mul, operator.imul, torch.mul, "mul", "mul_"):
                node = INode(name, "mul", [arg(n.args[0]), arg(n.args[1])], shp(n))
            elif t is torch.cat:
                xs = n.args[0]
                dim = n.args[1] if len(n.args) > 1 else n.kwargs.get("dim", 0)
                if dim != 1:
                    raise NotImplementedError("cat along non-channel dim")
                node = INode(name, "cat", [arg(a) for a in xs], shp(n))
            elif t in (torch.flatten, "flatten", "view", "reshape", "contiguous", F.dropout,
                       "dropout"):
                x = arg(n.args[0])
                if t != "contiguous" and (x.shape[2] != 1 or x.shape[3] != 1):
                    raise NotImplementedError("flatten/view of a spatial map")
                node = INode(name, "identity", [x], shp(n))
            elif t in (F.relu, torch.relu, "relu", "relu_", F.relu6, F.silu, torch.sigmoid,
                       F.sigmoid, "sigmoid"):
                code = ACT_RELU
                if t is F.relu6:
                    code = ACT_RELU6
                elif t is F.silu:
                    code = ACT_SILU
                elif t in (torch.sigmoid, F.sigmoid, "sigmoid"):
                    code = ACT_SIGMOID
                node = INode(name, "act", [arg(n.args[0])], shp(n), {"act": code})
            elif t in (F.max_pool2d, F.avg_pool2d):
                x = arg(n.args[0])
                kw = dict(n.kwargs)
                names = ["kernel_size", "stride", "padding"]
                for i, v in enumerate(n.args[1:4]):
                    kw[names[i]] = v
                k = _pair(kw["kernel_size"])
                s = _pair(kw.get("stride") or k)
                p = _pair(kw.get("padding", 0))
                if kw.get("ceil_mode", False):
                    raise NotImplementedError("ceil_mode")
                if t is F.max_pool2d:
                    node = INode(name, "pool", [x], shp(n), {"mode": "max", "k": k, "stride": s,
                                                              "pad": p, "cip": True})
                else:
                    cip = kw.get("count_include_pad", n.args[5] if len(n.args) > 5 else True)
                    node = INode(name, "pool", [x], shp(n), {"mode": "avg", "k": k, "stride": s,
                                                              "pad": p, "cip": bool(cip)})
            elif t is F.adaptive_avg_pool2d:
                node = INode(name, "gpool", [arg(n.args[0])], shp(n))
            elif getattr(t, "__name__", "") == "stochastic_depth":
                node = INode(name, "identity", [arg(n.args[0])], shp(n))  # eval: identity
            elif t in ("size", getattr):
                env[n] = None
                continue
            else:
                raise NotImplementedError(f"function {t} ({n.name})")
        else:
            raise NotImplementedError(n.op)
        env[n] = node
        out.append(node)
    return out


# ----------------------------------------------------------------------------
# rewrite passes
# ----------------------------------------------------------------------------

def _users(nodes):
    u = {id(n): [] for n in nodes}
    for n in nodes:
        for x in n.inputs:
            u[id(x)].append(n)
        if n.residual is not None:
            u[id(n.residual)].append(n)
    return u


def _replace_uses(nodes, old, new):
    for n in nodes:
        n.inputs = [new if x is old else x for x in n.inputs]
        if n.residual is old:
            n.residual = new


def _drop_identities(nodes):
    keep = []
    for n in nodes:
        if n.kind == "identity":
            _replace_uses(nodes, n, n.inputs[0])
        else:
            keep.append(n)
    return keep


def _fold_bn(nodes):
    users = _users(nodes)
    keep = []
    for n in nodes:
        if n.kind == "bn":
            src = n.inputs[0]
            sc, sh = n.attrs["scale"], n.attrs["shift"]
            if src.kind in ("conv", "dwconv") and len(users[id(src)]) == 1 and src.act == ACT_NONE \
                    and src.residual is None:
                _fold_into(src, sc, sh, 0)
                _replace_uses(nodes, n, src)
                continue
            if src.kind == "cat" and len(users[id(src)]) == 1 and all(
                    x.kind in ("conv", "dwconv") and len(users[id(x)]) == 1 and x.act == ACT_NONE
                    and x.residual is None for x in src.inputs) and \
                    len({id(x) for x in src.inputs}) == len(src.inputs):
                off = 0
                for x in src.inputs:
                    c = x.shape[1]
                    _fold_into(x, sc[off:off + c], sh[off:off + c], 0)
                    off += c
                _replace_uses(nodes, n, src)
                continue
            n.kind = "affine"
        keep.append(n)
    return keep


def _fold_into(conv, scale, shift, _):
    w = conv.attrs["weight"].double()
    b = conv.attrs["bias"].double() if conv.attrs["bias"] is not None else torch.zeros(w.shape[0], dtype=torch.float64)
    conv.attrs["weight"] = (w * scale.view(-1, 1, 1, 1)).float()
    conv.attrs["bias"] = (b * scale + shift).float()


def _reaches(src, dst, memo=None):
    """True when dst depends (transitively) on src."""
    stack = [dst]
    seen = set()
    while stack:
        x = stack.pop()
        if x is src:
            return True
        if id(x) in seen:
            continue
        seen.add(id(x))
        stack.extend(x.inputs)
        if x.residual is not None:
            stack.append(x.residual)
    return False


def _depths(nodes):
    """Longest path (in nodes) from the input: a proxy for when a tensor is ready."""
    d = {}
    for n in nodes:
        ins = list(n.inputs) + ([n.residual] if n.residual is not None else [])
        d[id(n)] = 1 + max((d.get(id(x), 0) for x in ins), default=0)
    return d


def _fold_residual_adds(nodes):
    users = _users(nodes)
    depth = _depths(nodes)
    keep = []
    for n in nodes:
        if n.kind == "add" and len(n.inputs) == 2 and n.inputs[0] is not n.inputs[1]:
            a, b = n.inputs
            done = False
            # fold into the producer that finishes last: its other operand is
            # ready earlier, so the fold adds no serialization
            cands = ((b, a), (a, b)) if depth[id(b)] >= depth[id(a)] else ((a, b), (b, a))
            for p, other in cands:
                if p.kind in ("conv", "dwconv", "pool") and p.residual is None and \
                        p.act == ACT_NONE and len(users[id(p)]) == 1 and \
                        p.shape == other.shape and not _reaches(p, other):
                    p.residual = other
                    _replace_uses(nodes, n, p)
                    users = _users([x for x in nodes])
                    done = True
                    break
            if done:
                continue
        keep.append(n)
    return keep


_ACT_PRODUCERS = ("conv", "dwconv", "pool", "add", "affine", "mul", "gpool")


def _fold_acts(nodes, out_node):
    users = _users(nodes)
    keep = []
    for n in nodes:
        if n.kind == "act":
            src = n.inputs[0]
            if src.kind in _ACT_PRODUCERS and src.act == ACT_NONE and len(users[id(src)]) == 1:
                src.act = n.attrs["act"]
                _replace_uses(nodes, n, src)
                users = _users(nodes)
                continue
            # act over a concat of single-consumer producers → distribute
            if src.kind == "cat" and len(users[id(src)]) == 1 and all(
                    x.kind in _ACT_PRODUCERS and x.act == ACT_NONE and len(users[id(x)]) == 1
                    for x in src.inputs) and len({id(x) for x in src.inputs}) == len(src.inputs):
                for x in src.inputs:
                    x.act = n.attrs["act"]
                _replace_uses(nodes, n, src)
                users = _users(nodes)
                continue
        keep.append(n)
    return keep


_PRE_RELU_CONSUMERS = ("conv", "dwconv", "pool", "gpool")


def _pre_relu(nodes):
    """Shared ReLU inputs: consumers apply ReLU on load; the ReLU task disappears."""
    users = _users(nodes)
    keep = []
    for n in nodes:
        if n.kind == "act" and n.attrs["act"] == ACT_RELU:
            us = users[id(n)]
            movable = [u for u in us if u.kind in _PRE_RELU_CONSUMERS and not u.pre_relu
                       and u.inputs[0] is n and u.residual is not n]
            for u in movable:
                u.inputs = [n.inputs[0]]
                u.pre_relu = True
            if len(movable) == len(us):
                continue  # fully absorbed
        keep.append(n)
    return keep


def _fuse_separable(nodes):
    """depthwise → pointwise 1x1 (single consumer) becomes ONE 'sepconv' task.

    NASNet's sep-convs and MobileNetV2's dw → project both have this shape
    after BN/act folding; the depthwise tile then lives only in shared memory
    and the graph loses a node (csrc/kernels/sepconv.cu).
    """
    users = _users(nodes)
    drop = set()
    for n in nodes:
        if n.kind != "conv" or n.attrs.get("linear"):
            continue
        d = n.inputs[0]
        if d.kind != "dwconv" or len(users[id(d)]) != 1 or d.residual is not None:
            continue
        if tuple(n.attrs["k"]) != (1, 1) or tuple(n.attrs["stride"]) != (1, 1) or \
                tuple(n.attrs["pad"]) != (0, 0):
            continue
        dw_act = d.act
        if n.pre_relu:
            if dw_act not in (ACT_NONE, ACT_RELU):
                continue
            dw_act = ACT_RELU
        n.attrs = {"weight": n.attrs["weight"], "bias": n.attrs["bias"],
                   "dw_weight": d.attrs["weight"], "dw_bias": d.attrs["bias"],
                   "stride": d.attrs["stride"], "pad": d.attrs["pad"], "k": d.attrs["k"],
                   "dw_act": dw_act}
        n.kind = "sepconv"
        n.pre_relu = d.pre_relu
        n.inputs = [d.inputs[0]]
        drop.add(id(d))
    return [n for n in nodes if id(n) not in drop]


def _fuse_sep_pairs(nodes, max_hw: int = 196):
    """sepconv → sepconv (NASNet's BranchSep: the second one stride 1, same k,
    'same' padding, sole consumer of the first) becomes ONE 'sep2' task
    (csrc/kernels/sep2.cu): one graph node instead of two on the cell's
    critical path, the intermediate map kept on chip."""
    users = _users(nodes)
    drop = set()
    for n in nodes:
        if n.kind != "sepconv":
            continue
        d = n.inputs[0]
        if d.kind != "sepconv" or id(d) in drop or len(users[id(d)]) != 1 or d.residual is not None:
            continue
        k = tuple(n.attrs["k"])
        if k[0] != k[1] or tuple(d.attrs["k"]) != k or k[0] not in (3, 5, 7):
            continue
        if tuple(n.attrs["stride"]) != (1, 1) or tuple(n.attrs["pad"]) != (k[0] // 2, k[0] // 2):
            continue
        if n.shape[2] * n.shape[3] > max_hw:
            continue  # one cluster per image: only small maps keep enough CTAs busy
        n.attrs = {"k": k, "stride": d.attrs["stride"], "pad": d.attrs["pad"],
                   "dw1": d.attrs["dw_weight"], "db1": d.attrs["dw_bias"], "dw_act1": d.attrs["dw_act"],
                   "pw1": d.attrs["weight"], "b1": d.attrs["bias"], "act1": d.act,
                   "pre_relu2": n.pre_relu,
                   "dw2": n.attrs["dw_weight"], "db2": n.attrs["dw_bias"], "dw_act2": n.attrs["dw_act"],
                   "pw2": n.attrs["weight"], "b2": n.attrs["bias"], "mid": d.shape[1]}
        n.kind = "sep2"
        n.pre_relu = d.pre_relu
        n.inputs = [d.inputs[0]]
        drop.add(id(d))
    return [n for n in nodes if id(n) not in drop]


def _merge_twin_pools(nodes):
    """add(pool(x), pool'(x)) with two identical pooling ops on the same input
    (NASNet normal cell: i3 = avg3(left) + avg3(left)) becomes ONE pool with an
    output multiplier of 2 — exactly the sum in fp32 (doubling is exact)."""
    users = _users(nodes)
    drop = set()
    for n in nodes:
        if n.kind != "add" or len(n.inputs) != 2:
            continue
        a, b = n.inputs
        if a is b or a.kind != "pool" or b.kind != "pool" or id(a) in drop or id(b) in drop:
            continue
        if a.inputs[0] is not b.inputs[0] or a.attrs != b.attrs or a.act != b.act or a.pre_relu != b.pre_relu:
            continue
        if a.residual is not None or b.residual is not None or len(users[id(a)]) != 1 or \
                len(users[id(b)]) != 1:
            continue
        a.attrs = dict(a.attrs, mul=2)
        _replace_uses(nodes, n, a)
        drop.add(id(b))
        drop.add(id(n))
    return [n for n in nodes if id(n) not in drop]


def optimize(nodes: list[INode], fuse_separable: bool = True, fuse_sep_pairs=False) -> list[INode]:
    out_node = nodes[-1]
    nodes = _drop_identities(nodes)
    nodes = _fold_bn(nodes)
    nodes = _merge_twin_pools(nodes)
    nodes = _fold_residual_adds(nodes)
    nodes = _fold_acts(nodes, out_node)
    nodes = _pre_relu(nodes)
    if fuse_separable:
        nodes = _fuse_separable(nodes)
        if fuse_sep_pairs:
            nodes = _fuse_sep_pairs(nodes, 196 if fuse_sep_pairs is True else int(fuse_sep_pairs))
    return nodes


# ----------------------------------------------------------------------------
# storage placement (zero-copy concat) and lowering
# ----------------------------------------------------------------------------

@dataclass(eq=False)
class Storage:
    sid: int
    n: int
    h: int
    w: int
    c: int
    nchw: bool = False  # network input / spatial output layout
    offset: int = -1    # arena byte offset (filled after pre_run)
    owner: int = -1     # task id whose mem list allocates it
    role: str = "act"   # act | input | output

    @property
    def nbytes(self):
        return self.n * self.h * self.w * self.c * 4

    @property
    def alloc_bytes(self):
        return (self.nbytes + ALIGN - 1) // ALIGN * ALIGN


@dataclass
class View:
    st: Storage
    c_off: int
    c: int

    def strides(self):
        s = self.st
        if s.nchw:
            return (s.c * s.h * s.w, s.w, 1, s.h * s.w)
        return (s.h * s.w * s.c, s.w * s.c, s.c, 1)

    def elem_offset(self):
        s = self.st
        return self.c_off * (s.h * s.w if s.nchw else 1)


@dataclass
class Task:
    tid: int
    kind: str
    name: str
    node: INode | None
    inputs: list            # list[View]
    out: View
    residual: View | None = None
    attrs: dict = field(default_factory=dict)
    deps: set = field(default_factory=set)
    flops: int = 0
    bytes: int = 0


@dataclass
class Program:
    tasks: list
    storages: list
    input_view: View
    output_view: View
    graph: CompGraph | None = None
    fused: bool = True
    out_shape: tuple = ()

    def stats(self):
        kinds = {}
        for t in self.tasks:
            kinds[t.kind] = kinds.get(t.kind, 0) + 1
        return kinds


def _place(nodes):
    """Assign every node output a View; concat inputs become slices."""
    views: dict[int, View] = {}
    storages: list[Storage] = []
    copies = []  # (src_node, dst View) copy tasks needed for unplaceable concat inputs

    def new_storage(shape, nchw=False, role="act"):
        n, c, h, w = shape
        st = Storage(len(storages), n, h, w, c, nchw=nchw, role=role)
        storages.append(st)
        return st

    inp = nodes[0]
    assert inp.kind == "input"
    views[id(inp)] = View(new_storage(inp.shape, nchw=True, role="input"), 0, inp.shape[1])
    # concats last → first so an outer concat places its (inner concat) inputs
    for n in reversed(nodes):
        if n.kind != "cat":
            continue
        if id(n) not in views:
            views[id(n)] = View(new_storage(n.shape), 0, n.shape[1])
        base = views[id(n)]
        off = 0
        seen = set()
        for x in n.inputs:
            c = x.shape[1]
            dst = View(base.st, base.c_off + off, c)
            if id(x) in views or id(x) in seen or x.kind in ("input",) or x.alias_of is not None:
                copies.append((x, dst, n))
            else:
                views[id(x)] = dst
                seen.add(id(x))
            off += c
    for n in nodes:
        if n.kind in ("input", "output", "cat") or id(n) in views:
            continue
        views[id(n)] = View(new_storage(n.shape), 0, n.shape[1])
    _mark_output(nodes, views)
    return views, storages, copies


def _mark_output(nodes, views):
    """The tensor the network returns is written in NCHW directly when it is a
    whole storage (no extra layout-copy task)."""
    src = nodes[-1].inputs[0]
    v = views[id(src)]
    n, c, h, w = src.shape
    if v.st.role == "input" or v.c_off != 0 or v.c != v.st.c:
        return
    v.st.nchw = h * w > 1
    v.st.role = "output"


def lower(nodes: list[INode], fused: bool) -> Program:
    views, storages, copies = _place(nodes) if fused else _place_unfused(nodes)
    tasks: list[Task] = []
    copy_after: dict[int, list] = {}
    for src, dst, cat in copies:
        copy_after.setdefault(id(cat), []).append((src, dst))
    for n in nodes:
        if n.kind in ("input", "output"):
            continue
        if n.kind == "cat":
            if fused:
                for src, dst in copy_after.get(id(n), []):
                    tasks.append(Task(len(tasks), "copy", f"{n.name}.copy", None, [views[id(src)]], dst))
            else:
                tasks.append(Task(len(tasks), "concat", n.name, n, [views[id(x)] for x in n.inputs],
                                  views[id(n)]))
            continue
        t = Task(len(tasks), n.kind, n.name, n, [views[id(x)] for x in n.inputs], views[id(n)],
                 residual=views[id(n.residual)] if n.residual is not None else None)
        tasks.append(t)
    out_node = nodes[-1]
    out_view = views[id(out_node.inputs[0])]
    n, c, h, w = out_node.shape
    need_copy = out_view.st.role != "output"
    if need_copy:
        st = Storage(len(storages), n, h, w, c, nchw=True, role="output")
        storages.append(st)
        dst = View(st, 0, c)
        tasks.append(Task(len(tasks), "copy", "output.copy", None, [out_view], dst))
        out_view = dst
    else:
        out_view.st.role = "output"
    # data dependencies: writer(s) of every consumed channel range → reader
    writers: dict[int, list] = {}
    for t in tasks:
        writers.setdefault(t.out.st.sid, []).append(t)
    for t in tasks:
        reads = list(t.inputs) + ([t.residual] if t.residual is not None else [])
        for v in reads:
            for w in writers.get(v.st.sid, []):
                if w.tid != t.tid and w.out.c_off < v.c_off + v.c and v.c_off < w.out.c_off + w.out.c:
                    t.deps.add(w.tid)
    # storage ownership: the first writer allocates it (reference mem events)
    for t in tasks:
        if t.out.st.owner < 0:
            t.out.st.owner = t.tid
    return Program(tasks, storages, views[id(nodes[0])], out_view, fused=fused,
                   out_shape=tuple(out_node.attrs.get("raw_shape", out_node.shape)))


def _place_unfused(nodes):
    views = {}
    storages = []
    for n in nodes:
        if n.kind == "output":
            continue
        role = "input" if n.kind == "input" else "act"
        nn_, c, h, w = n.shape
        st = Storage(len(storages), nn_, h, w, c, nchw=(n.kind == "input"), role=role)
        storages.append(st)
        views[id(n)] = View(st, 0, c)
    _mark_output(nodes, views)
    return views, storages, []


def to_compgraph(prog: Program, durations=None) -> CompGraph:
    nodes = []
    owned: dict[int, list] = {}
    for st in prog.storages:
        if st.owner >= 0:
            owned.setdefault(st.owner, []).append(st)
    for t in prog.tasks:
        mem = tuple(MemEvent.alloc(st.alloc_bytes) for st in owned.get(t.tid, []))
        d = 1 if durations is None else max(1, int(durations[t.tid]))
        nodes.append(TaskNode(t.tid, d, 1, f"{t.kind}:{t.name}", mem))
    edges = sorted({(d, t.tid) for t in prog.tasks for d in t.deps})
    g = CompGraph.build(nodes, edges)
    prog.graph = g
    return g


def build_program(model: nn.Module, example: torch.Tensor, fuse: bool = True,
                  fuse_separable: bool = True, fuse_sep_pairs: bool = False) -> Program:
    nodes = trace_model(model, example)
    if fuse:
        nodes = optimize(nodes, fuse_separable=fuse_separable, fuse_sep_pairs=fuse_sep_pairs)
    else:
        nodes = _drop_identities(nodes)
        for n in nodes:
            if n.kind == "bn":
                n.kind = "affine"
    prog = lower(nodes, fused=fuse)
    to_compgraph(prog)
    return prog
