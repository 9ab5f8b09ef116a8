"""AoT training step: forward + loss + backward + gradient allreduce + SGD as
ONE captured multi-stream CUDA graph.

Nimble's training claim is the inference story applied to a whole iteration:
the op DAG of forward *and* backward is stream-assigned (the same bit-exact
planner, ``assign_streams`` → ``pre_run``), captured once, and replayed with
one ``cudaGraphLaunch`` per step.  The backward DAG is where multi-stream pays
for chain networks: every weight gradient (wgrad, and the BN dgamma/dbeta
reduction) is off the dgrad critical path, so the planner puts them on side
streams.

    eng = TrainEngine(model, lr=0.05, momentum=0.9, weight_decay=4e-5).prepare(x, y)
    loss = eng.step(x, y)          # host tensors in, host float out

Data-parallel: one process per GPU; ``TrainEngine(..., world=N, rank=r)``
builds an NCCL communicator (unique id broadcast over torch.distributed) and
the graph holds one ``ncclAllReduce(avg)`` of the flat gradient buffer between
the last gradient and the optimizer.

Layout (HBM): one arena, bump-allocated (nothing is freed inside a step, so
no cross-stream reuse hazard — SURVEY D4): activations NHWC fp32; the network
input NCHW; every trainable tensor a slice of ONE flat parameter buffer in
kernel layout (conv [K][R][S][C], depthwise [R][S][C], BN [gamma C | beta C]),
mirrored by the flat gradient and momentum buffers — the allreduce and the
optimizer are single launches over them.

Supported graph vocabulary (MobileNetV2 / EfficientNet-B0 as fx-traced by
trace.py): conv (1x1 any input; k x k only on the network input), depthwise
3x3/5x5, BatchNorm (batch statistics, running-stat update) + ReLU/ReLU6/SiLU
(+ residual add), global average pool, Linear, broadcast mul (squeeze-excite),
standalone activations, add, softmax cross-entropy.  Dropout / stochastic
depth must be disabled (p = 0) — their RNG is not reproduced.
"""

from __future__ import annotations

import ctypes as C
import math
import struct
import time
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn as nn

from . import _native as N
from .assign import StreamAssignment, SyncPlan, assign_streams_full
from .engine import (EP_A, EP_B, EP_OUT, EW_A_SN, EW_ACT, EW_B_SN, EW_C, EW_H, EW_N, EW_NIN, EW_O_SN,
                     EW_OP, EW_W, EW_ADD, EW_COPY, EW_MUL, K_CONV, K_DWCONV, K_ELTWISE, K_GLOBAL_POOL,
                     NUM_SMS, PT_BIAS, PT_IN, PT_OUT, PT_W, SLOT_MULTI, SLOT_MULTI_IO, SLOT_SINGLE,
                     SLOT_SINGLE_IO, SP_ACT, SP_C, SP_H, SP_HAS_RES, SP_IN_SN, SP_K, SP_KPAD, SP_N,
                     SP_OUT_SC, SP_OUT_SN, SP_P, SP_PAD_H, SP_PAD_W, SP_Q, SP_R, SP_S, SP_SPLIT_K,
                     SP_STRIDE_H, SP_STRIDE_W, SP_W, SP_RES_SN, SP_RES_SH, SP_RES_SW, SP_RES_SC, PT_RES,
                     K_CONV_TC, conv_candidates, pick_conv_variant)
from .errors import CudaError
from .graph import CompGraph, TaskNode
from .schedule import pre_run, schedule_arrays
from .trace import ACT_NONE, trace_model, _drop_identities

# csrc/runtime/ops.h training kinds
(K_BN_STATS, K_BN_APPLY, K_BN_BWD_REDUCE, K_BN_BWD_APPLY, K_DW_DGRAD, K_DW_WGRAD, K_GEMM, K_XENT,
 K_SGD, K_ALLREDUCE, K_EW_BWD, K_TRANSPOSE, K_GEMM_REDUCE, K_BN_FWD, K_BN_BWD) = range(9, 24)
(BN_M, BN_C, BN_HW, BN_ACT, BN_HAS_RES, BN_EPS, BN_MOMENTUM, BN_GRID, BN_DO_SN, BN_DO_SP,
 BN_DO_SCALE, BN_LD) = range(12)
(GM_M, GM_N, GM_K, GM_A_I, GM_A_R, GM_B_R, GM_B_J, GM_C_I, GM_SPLIT, GM_HAS_RES, GM_IM2COL,
 GM_X_N, GM_X_H, GM_X_W, GM_X_C, GM_X_P, GM_X_Q, GM_X_R, GM_X_S, GM_X_STRIDE, GM_X_PAD,
 GM_X_SN, GM_X_SH, GM_X_SW, GM_X_SC, GM_PARTIALS_ONLY) = range(26)
TICKET_SPLIT_MAX = 16  # wider splits fold their partials in a separate K_GEMM_REDUCE task
EWB_ACT, EWB_MUL_X, EWB_MUL_S, EWB_BCAST = 0, 1, 2, 3
GEMM_TILE = 64
ALIGN = 256


def fbits(x: float) -> int:
    return struct.unpack("<i", struct.pack("<f", float(x)))[0]


# ----------------------------------------------------------------------------
# buffers and tasks
# ----------------------------------------------------------------------------

@dataclass(eq=False)
class Buf:
    bid: int
    name: str
    nbytes: int
    shape: tuple = ()          # (N, C, H, W) for tensors
    nchw: bool = False
    offset: int = -1           # arena byte offset
    parent: "Buf | None" = None
    sub_offset: int = 0        # byte offset inside parent
    zero: bool = False         # zero-filled once at prepare (workspaces, momentum)

    def strides(self):
        n, c, h, w = self.shape
        if self.nchw:
            return (c * h * w, w, 1, h * w)
        return (h * w * c, w * c, c, 1)


@dataclass(eq=False)
class TTask:
    tid: int
    kind: str
    name: str
    reads: list
    writes: list
    fill: object               # fill(desc, ptr_of) -> None
    deps: set = field(default_factory=set)
    phase: str = "fwd"         # fwd | bwd | comm | opt
    flops: float = 0.0
    bytes: float = 0.0


@dataclass
class ParamRef:
    """One trainable torch tensor and its slice of the flat buffers."""
    name: str
    tensor: torch.Tensor       # the nn.Parameter (torch layout)
    buf: Buf                   # slice of the flat params (kernel layout)
    gbuf: Buf                  # same slice of the flat grads
    to_kernel: object          # torch layout -> kernel-layout flat numpy
    from_kernel: object        # kernel-layout flat numpy -> torch layout tensor


@dataclass
class GradRef:
    """Gradient of a forward value: a dense NHWC buffer, or a pending broadcast
    (global-pool backward) that the consuming BN backward reads in place."""
    buf: Buf
    sn: int
    sp: int
    scale: float = 1.0

    @property
    def dense(self):
        return self.scale == 1.0 and self.sp != 0


class TrainProgram:
    def __init__(self):
        self.bufs: list[Buf] = []
        self.tasks: list[TTask] = []
        self.params: list[ParamRef] = []
        self.running: list[tuple] = []   # (bn module, Buf [mean C | var C])
        self._last_writer: dict[int, list] = {}
        self._readers: dict[int, list] = {}
        self.arena_bytes = 0
        self.graph: CompGraph | None = None

    # -- buffers --
    def buf(self, name, nbytes, shape=(), nchw=False, zero=False) -> Buf:
        b = Buf(len(self.bufs), name, int(nbytes), tuple(shape), nchw, zero=zero)
        self.bufs.append(b)
        return b

    def tensor(self, name, shape, nchw=False) -> Buf:
        n, c, h, w = shape
        return self.buf(name, 4 * n * c * h * w, shape, nchw)

    def sub(self, parent: Buf, name, off_bytes, nbytes, shape=()) -> Buf:
        b = Buf(len(self.bufs), name, int(nbytes), tuple(shape), parent=parent, sub_offset=int(off_bytes))
        self.bufs.append(b)
        return b

    # -- tasks: dependencies from the sequential program order (RAW, WAR, WAW) --
    def task(self, kind, name, reads, writes, fill, phase, flops=0.0, nbytes=0.0) -> TTask:
        t = TTask(len(self.tasks), kind, name, list(reads), list(writes), fill, phase=phase,
                  flops=flops, bytes=nbytes)
        for b in t.reads:
            for k in self._keys(b):
                for w in self._last_writer.get(k, []):
                    t.deps.add(w)
        for b in t.writes:
            for k in self._keys(b):
                for w in self._last_writer.get(k, []):
                    t.deps.add(w)
                for r in self._readers.get(k, []):
                    t.deps.add(r)
        for b in t.reads:
            for k in self._keys(b):
                self._readers.setdefault(k, []).append(t.tid)
        for b in t.writes:
            for k in self._keys(b):
                self._last_writer[k] = [t.tid]
                self._readers[k] = []
        t.deps.discard(t.tid)
        self.tasks.append(t)
        return t

    @staticmethod
    def _keys(b: Buf):
        # a slice conflicts with itself; the flat parents are only touched as a
        # whole by tasks that list every slice, so slices are tracked by id
        return (b.bid,)

    def layout(self):
        off = 0
        for b in self.bufs:
            if b.parent is None:
                b.offset = off
                off += (max(b.nbytes, 4) + ALIGN - 1) // ALIGN * ALIGN
        for b in self.bufs:
            if b.parent is not None:
                b.offset = b.parent.offset + b.sub_offset
        self.arena_bytes = off

    def to_compgraph(self) -> CompGraph:
        nodes = [TaskNode(t.tid, 1, 1, f"{t.kind}:{t.name}", ()) for t in self.tasks]
        edges = sorted({(d, t.tid) for t in self.tasks for d in t.deps})
        self.graph = CompGraph.build(nodes, edges)
        return self.graph


# ----------------------------------------------------------------------------
# op descriptors
# ----------------------------------------------------------------------------

def _spatial_fill(kind, x: Buf, out: Buf, w: Buf | None, bias: Buf | None, k, stride, pad, act=ACT_NONE,
                  res: Buf | None = None):
    n, c, h, wd = x.shape
    _, kk, p, q = out.shape
    R, S = k

    def fill(d, ptr):
        d.kind = kind
        vals = {SP_N: n, SP_H: h, SP_W: wd, SP_C: c, SP_P: p, SP_Q: q, SP_K: kk, SP_R: R, SP_S: S,
                SP_STRIDE_H: stride[0], SP_STRIDE_W: stride[1], SP_PAD_H: pad[0], SP_PAD_W: pad[1],
                SP_ACT: act}
        for j, s in enumerate(x.strides()):
            vals[SP_IN_SN + j] = s
        osn, osh, osw, osc = out.strides()
        vals.update({SP_OUT_SN: osn, SP_OUT_SN + 1: osh, SP_OUT_SN + 2: osw, SP_OUT_SC: osc})
        if kind == K_CONV:
            variant, split = pick_conv_variant(n * p * q, kk, R * S * c, R, S, pad, stride)
            d.variant = variant
            vals[SP_SPLIT_K] = split
            vals[SP_KPAD] = (R * S * c + 31) // 32 * 32
        for key, v in vals.items():
            d.params[key] = int(v)
        d.ptrs[PT_IN] = ptr(x)
        d.ptrs[PT_OUT] = ptr(out)
        d.ptrs[PT_W] = ptr(w) if w is not None else 0
        d.ptrs[PT_BIAS] = ptr(bias) if bias is not None else 0
        if res is not None:
            rsn, rsh, rsw, rsc = res.strides()
            for key, v in {SP_RES_SN: rsn, SP_RES_SH: rsh, SP_RES_SW: rsw, SP_RES_SC: rsc, SP_HAS_RES: 1}.items():
                d.params[key] = int(v)
            d.ptrs[PT_RES] = ptr(res)
    return fill


def _ew_fill(op, ins: list, out: Buf, act=ACT_NONE, gpool=False):
    def fill(d, ptr):
        d.kind = K_GLOBAL_POOL if gpool else K_ELTWISE
        n, c, h, w = (ins[0] if gpool else out).shape
        vals = {EW_N: n, EW_H: h, EW_W: w, EW_C: c, EW_OP: op, EW_ACT: act, EW_NIN: len(ins)}
        for i, b in enumerate(ins):
            s = list(b.strides())
            if not gpool:
                bn, _, bh, bw = b.shape
                if bh == 1 and h > 1:
                    s[1] = 0
                if bw == 1 and w > 1:
                    s[2] = 0
                if bn == 1 and n > 1:
                    s[0] = 0
            base = (EW_A_SN, EW_B_SN)[i]
            for j in range(4):
                d.params[base + j] = int(s[j])
            d.ptrs[(EP_A, EP_B)[i]] = ptr(b)
        for j, s in enumerate(out.strides()):
            d.params[EW_O_SN + j] = int(s)
        for key, v in vals.items():
            d.params[key] = int(v)
        d.ptrs[EP_OUT] = ptr(out)
    return fill


def _gemm_fill(M, Nn, K, A: Buf, a_i, a_r, B: Buf, b_r, b_j, Cb: Buf, c_i, split, ws: Buf | None,
               res: Buf | None = None, bias: Buf | None = None, im2col=None, kind=K_GEMM):
    def fill(d, ptr):
        d.kind = kind
        vals = {GM_M: M, GM_N: Nn, GM_K: K, GM_A_I: a_i, GM_A_R: a_r, GM_B_R: b_r, GM_B_J: b_j,
                GM_C_I: c_i, GM_SPLIT: split, GM_HAS_RES: int(res is not None),
                GM_PARTIALS_ONLY: int(split > TICKET_SPLIT_MAX)}
        if im2col is not None:
            vals[GM_IM2COL] = 1
            (xn, xc, xh, xw), (p, q), (r, s), st, pad, strides = im2col
            vals.update({GM_X_N: xn, GM_X_H: xh, GM_X_W: xw, GM_X_C: xc, GM_X_P: p, GM_X_Q: q,
                         GM_X_R: r, GM_X_S: s, GM_X_STRIDE: st, GM_X_PAD: pad,
                         GM_X_SN: strides[0], GM_X_SH: strides[1], GM_X_SW: strides[2],
                         GM_X_SC: strides[3]})
        for key, v in vals.items():
            d.params[key] = int(v)
        d.ptrs[0] = ptr(A)
        d.ptrs[1] = ptr(B)
        d.ptrs[2] = ptr(Cb)
        d.ptrs[3] = ptr(bias) if bias is not None else 0
        d.ptrs[4] = ptr(res) if res is not None else 0
        d.ptrs[5] = ptr(ws) if ws is not None else 0
    return fill


def gemm_split(M, Nn, K):
    tiles = math.ceil(M / GEMM_TILE) * math.ceil(Nn / GEMM_TILE)
    split = 1
    while split < 16 and tiles * split * 2 <= 2 * NUM_SMS and K // (split * 2) >= 128:
        split *= 2
    return split


def wide_split(M, Nn, K, rows_per_cta=64):
    """Split of a long reduction (weight gradients: K = pixels) so ~2 CTAs per
    SM work on it, each over >= rows_per_cta rows."""
    tiles = math.ceil(M / GEMM_TILE) * math.ceil(Nn / GEMM_TILE)
    return max(1, min(2 * NUM_SMS // tiles, K // rows_per_cta, 256))


def gemm_ws_bytes(M, Nn, split):
    if split <= 1:
        return 0
    tiles = math.ceil(M / GEMM_TILE) * math.ceil(Nn / GEMM_TILE)
    return 4 * split * tiles * GEMM_TILE * GEMM_TILE + 4 * tiles


def chan_tile(c: int) -> int:
    """csrc/kernels/train.cu chan_tile: channels per CTA of the per-channel reductions."""
    return 32


def reduce_grid(m: int, c: int, rows_per_thread: int, cap: int) -> int:
    """Row blocks (grid.x) of a per-channel reduction over m rows: about
    `rows_per_thread` rows per thread, ~2 CTAs per SM overall, and at most
    `cap` partials for the last CTA to fold."""
    tc = chan_tile(c)
    rl = 256 // tc
    gy = math.ceil(c / tc)
    gx = math.ceil(m / (rl * rows_per_thread))
    return max(1, min(gx, cap, max(1, 2 * NUM_SMS // gy)))


def fused_ws_bytes(grid: int, c: int) -> int:
    """Fused BN kinds: fp64 partials [grid][2][c] + (arrive, leave) counters per channel block."""
    return 16 * grid * c + 8 * math.ceil(c / chan_tile(c)) + 16


def reduce_ws_bytes(grid: int, c: int, elem_bytes: int, per_chan: int) -> int:
    """Partials [grid][per_chan][c] + one ticket per channel block."""
    return elem_bytes * grid * per_chan * c + 4 * math.ceil(c / chan_tile(c)) + 16


# ----------------------------------------------------------------------------
# builder
# ----------------------------------------------------------------------------

def _conv_to_kernel(t):   # [K][C][R][S] -> [K][R][S][C]
    return t.detach().float().permute(0, 2, 3, 1).contiguous().numpy().reshape(-1)


def _conv_from_kernel(a, shape):
    k, c, r, s = shape
    return torch.from_numpy(a.reshape(k, r, s, c).copy()).permute(0, 3, 1, 2).contiguous()


def _dw_to_kernel(t):     # [C][1][R][S] -> [R][S][C]
    return t.detach().float()[:, 0].permute(1, 2, 0).contiguous().numpy().reshape(-1)


def _dw_from_kernel(a, shape):
    c, _, r, s = shape
    return torch.from_numpy(a.reshape(r, s, c).copy()).permute(2, 0, 1)[:, None].contiguous()


def _flat_to_kernel(t):
    return t.detach().float().contiguous().numpy().reshape(-1)


class _Builder:
    def __init__(self, model: nn.Module, x_shape, lr, momentum, weight_decay, allreduce: bool,
                 fuse_bn: bool = True):
        self.model = model
        self.x_shape = tuple(x_shape)
        self.prog = TrainProgram()
        self.lr, self.momentum, self.wd = lr, momentum, weight_decay
        self.allreduce = allreduce
        self.fuse_bn = fuse_bn
        self.val: dict[int, Buf] = {}        # INode id -> forward value buffer
        self.grad: dict[int, GradRef] = {}
        self.node_of: dict[int, object] = {}
        self.param_specs = []                 # (name, tensor, nbytes, to_k, from_k)

    # -- params --
    def _param(self, name, tensor, to_k, from_k):
        self.param_specs.append((name, tensor, to_k, from_k))
        return len(self.param_specs) - 1

    def build(self):
        model = self.model
        ex = torch.zeros(self.x_shape)
        nodes = _drop_identities(trace_model(model, ex))
        model.train()
        P = self.prog
        self.nodes = nodes
        users: dict[int, list] = {id(n): [] for n in nodes}
        for n in nodes:
            for x in n.inputs:
                users[id(x)].append(n)
        self.users = users
        self.lin = {id(n): i for i, n in enumerate(nodes)}
        # pattern: bn [+ act] [+ residual add]  → one "bnact" forward op
        fwd_ops = self._group(nodes, users)
        self._ops_by_node = {id(op["node"]): op for op in fwd_ops if "node" in op}
        # flat parameter buffers sized from the param specs
        for op in fwd_ops:
            self._declare_params(op)
        tot = sum(4 * _numel_k(s[1]) for s in self.param_specs)
        tot_al = sum((4 * _numel_k(s[1]) + 15) // 16 * 16 for s in self.param_specs)
        self.flat_p = P.buf("params", tot_al)
        self.flat_g = P.buf("grads", tot_al)
        self.flat_m = P.buf("momentum", tot_al, zero=True)
        self.param_floats = tot_al // 4
        self.param_count = tot // 4
        off = 0
        self.pbuf, self.gbuf = [], []
        for name, tensor, to_k, from_k in self.param_specs:
            nb = 4 * _numel_k(tensor)
            pb = P.sub(self.flat_p, f"p:{name}", off, nb)
            gb = P.sub(self.flat_g, f"g:{name}", off, nb)
            P.params.append(ParamRef(name, tensor, pb, gb, to_k, from_k))
            self.pbuf.append(pb)
            self.gbuf.append(gb)
            off += (nb + 15) // 16 * 16
        # forward
        x = nodes[0]
        self.input = P.tensor("input", x.shape, nchw=True)
        self.val[id(x)] = self.input
        self.labels = P.buf("labels", 4 * x.shape[0])
        self.loss = P.buf("loss", 4)
        self.ones = P.buf("ones", 4 * max(x.shape[0], 1))
        for op in fwd_ops:
            self._forward(op)
        # loss
        out_node = nodes[-1]
        logits = self.val[id(out_node.inputs[0])]
        nb, ncls = logits.shape[0], logits.shape[1]
        dlogits = P.tensor("dlogits", (nb, ncls, 1, 1))

        def fill_xent(d, ptr):
            d.kind = K_XENT
            d.params[0], d.params[1], d.params[2] = nb, ncls, ncls
            d.ptrs[0], d.ptrs[1], d.ptrs[2], d.ptrs[3] = ptr(logits), ptr(self.labels), ptr(self.loss), ptr(dlogits)
        P.task("xent", "loss", [logits, self.labels], [self.loss, dlogits], fill_xent, "loss")
        self.grad[id(out_node.inputs[0])] = GradRef(dlogits, ncls, ncls)
        # backward (reverse forward order)
        for op in reversed(fwd_ops):
            self._backward(op)
        # gradient allreduce (data parallel) and the optimizer
        if self.allreduce:
            def fill_ar(d, ptr):
                d.kind = K_ALLREDUCE
                d.params[0] = self.param_floats
                d.ptrs[0] = ptr(self.flat_g)
            P.task("allreduce", "grads", list(self.gbuf), list(self.gbuf), fill_ar, "comm",
                   nbytes=8.0 * self.param_floats)

        def fill_sgd(d, ptr):
            d.kind = K_SGD
            d.params[0] = self.param_floats
            d.params[1], d.params[2], d.params[3] = fbits(self.lr), fbits(self.momentum), fbits(self.wd)
            d.ptrs[0], d.ptrs[1], d.ptrs[2] = ptr(self.flat_p), ptr(self.flat_g), ptr(self.flat_m)
        P.task("sgd", "params", list(self.gbuf) + list(self.pbuf), list(self.pbuf) + [self.flat_m],
               fill_sgd, "opt", nbytes=20.0 * self.param_floats)
        P.layout()
        P.to_compgraph()
        return P

    # -- grouping --
    def _group(self, nodes, users):
        ops = []
        consumed = set()
        for n in nodes:
            if id(n) in consumed or n.kind in ("input", "output"):
                continue
            if n.kind == "bn":
                grp = {"kind": "bnact", "bn": n, "act": ACT_NONE, "res": None, "out": n}
                cur = n
                us = users[id(cur)]
                if len(us) == 1 and us[0].kind == "act":
                    grp["act"] = us[0].attrs["act"]
                    consumed.add(id(us[0]))
                    cur = us[0]
                    us = users[id(cur)]
                if grp["act"] == ACT_NONE and len(us) == 1 and us[0].kind == "add" and \
                        len(us[0].inputs) == 2 and us[0].inputs[0] is not us[0].inputs[1]:
                    add = us[0]
                    other = add.inputs[1] if add.inputs[0] is cur else add.inputs[0]
                    if self.lin[id(other)] < self.lin[id(add)] and other.shape == add.shape:
                        grp["res"] = other
                        consumed.add(id(add))
                        cur = add
                grp["out"] = cur
                ops.append(grp)
            else:
                ops.append({"kind": n.kind, "node": n, "out": n})
        return ops

    def _declare_params(self, op):
        if op["kind"] == "bnact":
            m = op["bn"].attrs["module"]
            op["pid"] = self._param(f"{op['bn'].name}.gamma_beta", (m.weight, m.bias),
                                    None, None)
        elif op["kind"] in ("conv", "dwconv"):
            n = op["node"]
            m = n.attrs["module"]
            if n.kind == "dwconv":
                op["pid"] = self._param(n.name + ".weight", m.weight, _dw_to_kernel, _dw_from_kernel)
            elif n.attrs.get("linear"):
                op["pid"] = self._param(n.name + ".weight", m.weight, _flat_to_kernel,
                                        lambda a, s: torch.from_numpy(a.reshape(s).copy()))
            else:
                op["pid"] = self._param(n.name + ".weight", m.weight, _conv_to_kernel, _conv_from_kernel)
            op["bid"] = None
            if m.bias is not None:
                op["bid"] = self._param(n.name + ".bias", m.bias, _flat_to_kernel,
                                        lambda a, s: torch.from_numpy(a.reshape(s).copy()))

    # -- forward --
    def _forward(self, op):
        P = self.prog
        k = op["kind"]
        if k == "bnact":
            bn = op["bn"]
            m = bn.attrs["module"]
            y = self.val[id(bn.inputs[0])]
            n, c, h, w = y.shape
            M = n * h * w
            grid = reduce_grid(M, c, 8, 64)
            stats = P.buf(f"{bn.name}.stats", 8 * c)
            running = P.buf(f"{bn.name}.running", 8 * c)
            P.running.append((m, running))
            ws = P.buf(f"{bn.name}.ws", reduce_ws_bytes(grid, c, 8, 2), zero=True)
            out = P.tensor(bn.name + ".out", y.shape)
            gb = self.pbuf[op["pid"]]
            eps, mom = m.eps, (m.momentum if m.momentum is not None else 0.1)
            res = self.val[id(op["res"])] if op["res"] is not None else None
            act = op["act"]
            op.update(y=y, stats=stats, ws=ws, M=M, grid=grid, outb=out, c=c, hw=h * w)

            if self.fuse_bn:
                fws = P.buf(f"{bn.name}.fws", fused_ws_bytes(grid, c), zero=True)

                def fill_fused(d, ptr):
                    d.kind = K_BN_FWD
                    for key, v in {BN_M: M, BN_C: c, BN_HW: h * w, BN_ACT: act, BN_HAS_RES: int(res is not None),
                                   BN_EPS: fbits(eps), BN_MOMENTUM: fbits(mom), BN_GRID: grid, BN_LD: c}.items():
                        d.params[key] = int(v)
                    d.ptrs[0], d.ptrs[1], d.ptrs[2], d.ptrs[3] = ptr(y), ptr(stats), ptr(running), ptr(gb)
                    d.ptrs[4] = ptr(res) if res is not None else 0
                    d.ptrs[5], d.ptrs[7] = ptr(out), ptr(fws)
                P.task("bn_fwd", bn.name, [y, gb] + ([res] if res is not None else []), [stats, running, out, fws],
                       fill_fused, "fwd", nbytes=4.0 * M * c * (3 if res is not None else 2))
                self.val[id(op["out"])] = out
                return

            def fill_stats(d, ptr):
                d.kind = K_BN_STATS
                for key, v in {BN_M: M, BN_C: c, BN_HW: h * w, BN_EPS: fbits(eps),
                               BN_MOMENTUM: fbits(mom), BN_GRID: grid, BN_LD: c}.items():
                    d.params[key] = int(v)
                d.ptrs[0], d.ptrs[1], d.ptrs[2], d.ptrs[7] = ptr(y), ptr(stats), ptr(running), ptr(ws)
            P.task("bn_stats", bn.name, [y], [stats, running, ws], fill_stats, "fwd", nbytes=4.0 * M * c)

            def fill_apply(d, ptr):
                d.kind = K_BN_APPLY
                for key, v in {BN_M: M, BN_C: c, BN_HW: h * w, BN_ACT: act,
                               BN_HAS_RES: int(res is not None), BN_LD: c}.items():
                    d.params[key] = int(v)
                d.ptrs[0], d.ptrs[1], d.ptrs[2] = ptr(y), ptr(stats), ptr(gb)
                d.ptrs[3] = ptr(res) if res is not None else 0
                d.ptrs[4] = ptr(out)
            reads = [y, stats, gb] + ([res] if res is not None else [])
            P.task("bn_apply", bn.name, reads, [out], fill_apply, "fwd",
                   nbytes=4.0 * M * c * (3 if res is not None else 2))
            self.val[id(op["out"])] = out
            return
        n = op["node"]
        ins = [self.val[id(x)] for x in n.inputs]
        if k in ("conv", "dwconv"):
            x = ins[0]
            out = P.tensor(n.name, n.shape)
            wb = self.pbuf[op["pid"]]
            bb = self.pbuf[op["bid"]] if op.get("bid") is not None else None
            kind = K_CONV if k == "conv" else K_DWCONV
            R, S = n.attrs["k"]
            fill = _spatial_fill(kind, x, out, wb, bb, (R, S), n.attrs["stride"], n.attrs["pad"])
            nb, kk, p, q = out.shape
            flops = 2.0 * nb * kk * p * q * R * S * (x.shape[1] if k == "conv" else 1)
            P.task(k, n.name, [x, wb] + ([bb] if bb is not None else []), [out], fill, "fwd", flops=flops)
            self.val[id(n)] = out
        elif k == "gpool":
            out = P.tensor(n.name, n.shape)
            P.task("gpool", n.name, ins, [out], _ew_fill(EW_COPY, ins, out, gpool=True), "fwd")
            self.val[id(n)] = out
        elif k in ("add", "mul"):
            out = P.tensor(n.name, n.shape)
            P.task(k, n.name, ins, [out], _ew_fill(EW_ADD if k == "add" else EW_MUL, ins, out), "fwd")
            self.val[id(n)] = out
        elif k == "act":
            out = P.tensor(n.name, n.shape)
            P.task("act", n.name, ins, [out], _ew_fill(EW_COPY, ins, out, act=n.attrs["act"]), "fwd")
            self.val[id(n)] = out
        elif k == "bn":
            raise AssertionError("bn outside a bnact group")
        else:
            raise NotImplementedError(f"training: forward op {k} ({n.name})")

    # -- gradient bookkeeping --
    def _needs_grad(self, node) -> bool:
        return node.kind != "input"

    def _materialize(self, node_id, shape):
        """Turn a pending broadcast gradient into a dense buffer."""
        P = self.prog
        g = self.grad[node_id]
        n, c, h, w = shape
        out = P.tensor(f"grad.bcast.{node_id}", shape)

        def fill(d, ptr):
            d.kind = K_EW_BWD
            for j, v in enumerate((n, h * w, c, EWB_BCAST, ACT_NONE, 0, fbits(g.scale))):
                d.params[j] = int(v)
            d.ptrs[2], d.ptrs[4] = ptr(g.buf), ptr(out)
        P.task("bcast", f"grad.{node_id}", [g.buf], [out], fill, "bwd")
        self.grad[node_id] = GradRef(out, h * w * c, c)

    def _contribute(self, node, shape, emit):
        """emit(out_buf, res_buf|None) adds a task writing (or accumulating) the
        gradient of `node`; returns nothing."""
        P = self.prog
        key = id(node)
        g = self.grad.get(key)
        if g is not None and not g.dense:
            self._materialize(key, shape)
            g = self.grad[key]
        if g is None:
            n, c, h, w = shape
            out = P.tensor(f"grad.{node.name}", shape)
            emit(out, None)
            self.grad[key] = GradRef(out, h * w * c, c)
        else:
            emit(g.buf, g.buf)

    def _contribute_alias(self, node, shape, gref: GradRef):
        """Identity gradient (residual branch): alias, or accumulate with an add."""
        P = self.prog
        key = id(node)
        g = self.grad.get(key)
        if g is None:
            self.grad[key] = gref
            return
        if not g.dense:
            self._materialize(key, shape)
            g = self.grad[key]
        if not gref.dense:
            raise NotImplementedError("broadcast gradient into an accumulated value")
        P.task("grad_add", f"grad.{node.name}", [g.buf, gref.buf], [g.buf],
               _ew_fill(EW_ADD, [self._view(g.buf, shape), self._view(gref.buf, shape)],
                        self._view(g.buf, shape)), "bwd")

    def _gemm(self, kind, name, reads, out: Buf, M, Nn, K, A, a_i, a_r, B, b_r, b_j, c_i, split,
              res=None, bias=None, im2col=None, flops=0.0):
        """One K_GEMM task, plus a K_GEMM_REDUCE task for splits too wide for
        the in-kernel ticket fold."""
        P = self.prog
        ws = P.buf(f"{name}.{kind}.ws", gemm_ws_bytes(M, Nn, split), zero=True) if split > 1 else None
        wide = split > TICKET_SPLIT_MAX
        extra = [res] if res is not None else []
        args = (M, Nn, K, A, a_i, a_r, B, b_r, b_j, out, c_i, split, ws)
        if not wide:
            P.task(kind, name, reads + extra, [out] + ([ws] if ws is not None else []),
                   _gemm_fill(*args, res=res, bias=bias, im2col=im2col), "bwd", flops=flops)
            return
        P.task(kind, name, reads, [ws], _gemm_fill(*args, res=res, bias=bias, im2col=im2col), "bwd", flops=flops)
        P.task(kind + "_reduce", name, [ws] + ([bias] if bias is not None else []) + extra, [out],
               _gemm_fill(*args, res=res, bias=bias, im2col=im2col, kind=K_GEMM_REDUCE), "bwd")

    def _view(self, b: Buf, shape) -> Buf:
        """Same storage under another logical shape (descriptor fills only)."""
        return self.prog.sub(b, b.name + ".view", 0, b.nbytes, shape)

    def _dense_grad(self, node, shape) -> Buf:
        g = self.grad[id(node)]
        if not g.dense:
            self._materialize(id(node), shape)
            g = self.grad[id(node)]
        return g.buf

    # -- backward --
    def _backward(self, op):
        P = self.prog
        k = op["kind"]
        if k == "bnact":
            bn = op["bn"]
            gout = self.grad.get(id(op["out"]))
            if gout is None:
                return
            y, stats, M, c, hw = op["y"], op["stats"], op["M"], op["c"], op["hw"]
            act = op["act"]
            gb = self.pbuf[op["pid"]]
            gg = self.gbuf[op["pid"]]
            grid = reduce_grid(M, c, 8, 64)
            ws = P.buf(f"{bn.name}.bws", reduce_ws_bytes(grid, c, 8, 2), zero=True)
            if op["res"] is not None:
                self._contribute_alias(op["res"], op["res"].shape, gout)
            bnp = {BN_M: M, BN_C: c, BN_HW: hw, BN_ACT: act, BN_GRID: grid, BN_DO_SN: gout.sn,
                   BN_DO_SP: gout.sp, BN_DO_SCALE: fbits(gout.scale), BN_LD: c}

            src = bn.inputs[0]
            if self.fuse_bn and self._needs_grad(src):
                fws = P.buf(f"{bn.name}.bfws", fused_ws_bytes(grid, c), zero=True)

                def emit_fused(out, res):
                    def fill(d, ptr):
                        d.kind = K_BN_BWD
                        for key, v in bnp.items():
                            d.params[key] = int(v)
                        d.params[BN_HAS_RES] = int(res is not None)
                        d.ptrs[0], d.ptrs[1], d.ptrs[2], d.ptrs[3], d.ptrs[4] = (
                            ptr(gout.buf), ptr(y), ptr(stats), ptr(gb), ptr(gg))
                        d.ptrs[5] = ptr(res) if res is not None else 0
                        d.ptrs[6], d.ptrs[7] = ptr(out), ptr(fws)
                    reads = [gout.buf, y, stats, gb] + ([res] if res is not None else [])
                    P.task("bn_bwd", bn.name, reads, [gg, out, fws], fill, "bwd", nbytes=12.0 * M * c)
                self._contribute(src, y.shape, emit_fused)
                return

            def fill_red(d, ptr):
                d.kind = K_BN_BWD_REDUCE
                for key, v in bnp.items():
                    d.params[key] = int(v)
                d.ptrs[0], d.ptrs[1], d.ptrs[2], d.ptrs[3], d.ptrs[4], d.ptrs[7] = (
                    ptr(gout.buf), ptr(y), ptr(stats), ptr(gb), ptr(gg), ptr(ws))
            P.task("bn_bwd_reduce", bn.name, [gout.buf, y, stats, gb], [gg, ws], fill_red, "bwd",
                   nbytes=8.0 * M * c)
            src = bn.inputs[0]
            if not self._needs_grad(src):
                return

            def emit(out, res):
                def fill_app(d, ptr):
                    d.kind = K_BN_BWD_APPLY
                    for key, v in bnp.items():
                        d.params[key] = int(v)
                    d.params[BN_HAS_RES] = int(res is not None)
                    d.ptrs[0], d.ptrs[1], d.ptrs[2], d.ptrs[3], d.ptrs[4] = (
                        ptr(gout.buf), ptr(y), ptr(stats), ptr(gb), ptr(gg))
                    d.ptrs[5] = ptr(res) if res is not None else 0
                    d.ptrs[6] = ptr(out)
                reads = [gout.buf, y, stats, gb, gg] + ([res] if res is not None else [])
                P.task("bn_bwd_apply", bn.name, reads, [out], fill_app, "bwd", nbytes=12.0 * M * c)
            self._contribute(src, y.shape, emit)
            return
        n = op["node"]
        g = self.grad.get(id(n))
        if g is None:
            return
        if k in ("conv", "dwconv"):
            self._conv_backward(op, n, g)
        elif k == "gpool":
            x = n.inputs[0]
            xb = self.val[id(x)]
            _, c, h, w = xb.shape
            gd = self._dense_grad(n, n.shape)
            gref = GradRef(gd, c, 0, 1.0 / (h * w))
            key = id(x)
            if self.grad.get(key) is None:
                self.grad[key] = gref
            else:
                prev = self.grad[key]
                if not prev.dense:
                    self._materialize(key, xb.shape)
                buf = self.grad[key].buf
                nn_ = xb.shape[0]

                def fill(d, ptr):
                    d.kind = K_EW_BWD
                    for j, v in enumerate((nn_, h * w, c, EWB_BCAST, ACT_NONE, 1, fbits(1.0 / (h * w)))):
                        d.params[j] = int(v)
                    d.ptrs[2], d.ptrs[3], d.ptrs[4] = ptr(gd), ptr(buf), ptr(buf)
                P.task("gpool_bwd", n.name, [gd, buf], [buf], fill, "bwd")
        elif k == "add":
            gd = self._dense_grad(n, n.shape)
            for x in n.inputs:
                if self._needs_grad(x):
                    self._contribute_alias(x, x.shape, GradRef(gd, g.sn, g.sp))
        elif k == "act":
            if op.get("folded"):
                return
            z = n.inputs[0]
            zb = self.val[id(z)]
            gd = self._dense_grad(n, n.shape)
            nn_, c, h, w = n.shape
            act = n.attrs["act"]

            def emit(out, res):
                def fill(d, ptr):
                    d.kind = K_EW_BWD
                    for j, v in enumerate((nn_, h * w, c, EWB_ACT, act, int(res is not None))):
                        d.params[j] = int(v)
                    d.ptrs[0], d.ptrs[1] = ptr(gd), ptr(zb)
                    d.ptrs[3] = ptr(res) if res is not None else 0
                    d.ptrs[4] = ptr(out)
                P.task("act_bwd", n.name, [gd, zb] + ([res] if res is not None else []), [out], fill, "bwd")
            self._contribute(z, zb.shape, emit)
        elif k == "mul":
            self._mul_backward(op, n)
        else:
            raise NotImplementedError(f"training: backward of {k}")

    def _mul_backward(self, op, n):
        P = self.prog
        a, b = n.inputs
        if a.shape == n.shape and b.shape[2:] == (1, 1):
            x, s = a, b
        elif b.shape == n.shape and a.shape[2:] == (1, 1):
            x, s = b, a
        else:
            raise NotImplementedError("training: mul must be a channel-broadcast scale")
        gd = self._dense_grad(n, n.shape)
        xb, sb = self.val[id(x)], self.val[id(s)]
        nn_, c, h, w = n.shape
        if self._needs_grad(x):
            def emit_x(out, res):
                def fill(d, ptr):
                    d.kind = K_EW_BWD
                    for j, v in enumerate((nn_, h * w, c, EWB_MUL_X, ACT_NONE, int(res is not None))):
                        d.params[j] = int(v)
                    d.ptrs[0], d.ptrs[2] = ptr(gd), ptr(sb)
                    d.ptrs[3] = ptr(res) if res is not None else 0
                    d.ptrs[4] = ptr(out)
                P.task("mul_bwd_x", n.name, [gd, sb] + ([res] if res is not None else []), [out], fill, "bwd")
            self._contribute(x, xb.shape, emit_x)
        # scale gradient; fold the producing activation (sigmoid) when s feeds only this mul
        target, act, zs = s, ACT_NONE, None
        sop = self._op_of(s)
        if s.kind == "act" and len(self.users[id(s)]) == 1 and sop is not None:
            target, act, zs = s.inputs[0], s.attrs["act"], self.val[id(s.inputs[0])]
            sop["folded"] = True
        tb = self.val[id(target)]

        def emit_s(out, res):
            if res is not None:
                raise NotImplementedError("accumulated squeeze-excite scale gradient")

            def fill(d, ptr):
                d.kind = K_EW_BWD
                for j, v in enumerate((nn_, h * w, c, EWB_MUL_S, act, 0)):
                    d.params[j] = int(v)
                d.ptrs[0], d.ptrs[1] = ptr(gd), ptr(xb)
                d.ptrs[4] = ptr(out)
                d.ptrs[5] = ptr(zs) if zs is not None else 0
            P.task("mul_bwd_s", n.name, [gd, xb] + ([zs] if zs is not None else []), [out], fill, "bwd")
        self._contribute(target, tb.shape, emit_s)

    def _op_of(self, node):
        return self._ops_by_node.get(id(node)) if hasattr(self, "_ops_by_node") else None

    def _conv_backward(self, op, n, g):
        P = self.prog
        x = n.inputs[0]
        xb = self.val[id(x)]
        gd = self._dense_grad(n, n.shape)
        nb, kk, p, q = n.shape
        _, c, h, w = xb.shape
        R, S = n.attrs["k"]
        st, pad = n.attrs["stride"], n.attrs["pad"]
        wb, gw = self.pbuf[op["pid"]], self.gbuf[op["pid"]]
        M = nb * p * q
        if n.kind == "dwconv":
            grid = reduce_grid(M, c, 4, 32 if R * S <= 9 else 16)
            ws = P.buf(n.name + ".wws", reduce_ws_bytes(grid, c, 4, R * S), zero=True)

            def fill_w(d, ptr):
                _dw_params(d, xb.shape, n.shape, (R, S), st, pad)
                d.kind = K_DW_WGRAD
                d.params[SP_SPLIT_K] = grid
                d.ptrs[0], d.ptrs[1], d.ptrs[2], d.ptrs[5] = ptr(gd), ptr(gw), ptr(xb), ptr(ws)
            P.task("dw_wgrad", n.name, [gd, xb], [gw, ws], fill_w, "bwd", flops=2.0 * M * c * R * S)
            if self._needs_grad(x):
                def emit(out, res):
                    def fill(d, ptr):
                        _dw_params(d, xb.shape, n.shape, (R, S), st, pad)
                        d.kind = K_DW_DGRAD
                        d.params[SP_HAS_RES] = int(res is not None)
                        d.ptrs[0], d.ptrs[1], d.ptrs[2] = ptr(gd), ptr(out), ptr(wb)
                        d.ptrs[4] = ptr(res) if res is not None else 0
                    P.task("dw_dgrad", n.name, [gd, wb] + ([res] if res is not None else []), [out], fill,
                           "bwd", flops=2.0 * nb * h * w * c * R * S)
                self._contribute(x, xb.shape, emit)
            return
        # dense conv / linear: wgrad dW[k, (r,s,c)] = sum_m dY[m,k] X(m; r,s,c)
        Kred = M
        Nn = R * S * c
        split = wide_split(kk, Nn, Kred)
        if (R, S) == (1, 1) and tuple(st) == (1, 1) and tuple(pad) == (0, 0) and not xb.nchw:
            self._gemm("wgrad", n.name, [gd, xb], gw, kk, Nn, Kred, gd, 1, kk, xb, c, 1, Nn, split,
                       flops=2.0 * kk * Nn * Kred)
        else:
            if st[0] != st[1] or pad[0] != pad[1]:
                raise NotImplementedError("training: anisotropic conv stride/pad")
            self._gemm("wgrad", n.name, [gd, xb], gw, kk, Nn, Kred, gd, 1, kk, xb, 0, 0, Nn, split,
                       im2col=(xb.shape, (p, q), (R, S), st[0], pad[0], xb.strides()),
                       flops=2.0 * kk * Nn * Kred)
        if op.get("bid") is not None:
            gbias = self.gbuf[op["bid"]]
            if M > self.ones.nbytes // 4:
                raise NotImplementedError("training: bias gradient over more rows than the batch")
            self._gemm("bgrad", n.name, [gd, self.ones], gbias, 1, kk, M, self.ones, 0, 1, gd, kk, 1, kk,
                       wide_split(1, kk, M, 16) if M > 256 else 1)
        if self._needs_grad(x):
            if (R, S) != (1, 1) or tuple(st) != (1, 1) or tuple(pad) != (0, 0):
                raise NotImplementedError("training: input gradient of a k x k / strided dense conv")

            # dgrad of a 1x1 conv is a 1x1 conv of dY with the transposed weight
            # [C][K]: the autotuned inference conv kernels (conv.cu / conv1x1.cu)
            # run it, accumulating through their residual epilogue.  The
            # transpose reads the weights at step start, off the critical path.
            wt = P.tensor(n.name + ".wT", (c, kk, 1, 1))

            def fill_t(d, ptr):
                d.kind = K_TRANSPOSE
                d.params[0], d.params[1] = kk, c
                d.ptrs[0], d.ptrs[1] = ptr(wb), ptr(wt)
            P.task("transpose", n.name, [wb], [wt], fill_t, "bwd")

            def emit(out, res):
                gview = self._view(gd, (nb, kk, p, q))
                P.task("dgrad", n.name, [gd, wt] + ([res] if res is not None else []), [out],
                       _spatial_fill(K_CONV, gview, self._view(out, xb.shape), wt, None, (1, 1), (1, 1), (0, 0),
                                     res=self._view(res, xb.shape) if res is not None else None), "bwd",
                       flops=2.0 * M * c * kk)
            self._contribute(x, xb.shape, emit)


def _dw_params(d, in_shape, out_shape, k, st, pad):
    n, c, h, w = in_shape
    _, _, p, q = out_shape
    vals = {SP_N: n, SP_H: h, SP_W: w, SP_C: c, SP_P: p, SP_Q: q, SP_K: c, SP_R: k[0], SP_S: k[1],
            SP_STRIDE_H: st[0], SP_STRIDE_W: st[1], SP_PAD_H: pad[0], SP_PAD_W: pad[1]}
    for key, v in vals.items():
        d.params[key] = int(v)


def _numel_k(t) -> int:
    if isinstance(t, tuple):
        return sum(x.numel() for x in t)
    return t.numel()


def build_train_program(model: nn.Module, x_shape, lr=0.05, momentum=0.9, weight_decay=4e-5,
                        allreduce=False, fuse_bn=True) -> "_Builder":
    b = _Builder(model, x_shape, lr, momentum, weight_decay, allreduce, fuse_bn)
    b.build()
    return b


def initial_param_image(b: "_Builder") -> np.ndarray:
    """Flat parameter buffer (kernel layout) from the module's current tensors."""
    out = np.zeros(b.param_floats, dtype=np.float32)
    for ref in b.prog.params:
        off = ref.buf.sub_offset // 4
        if isinstance(ref.tensor, tuple):
            a = np.concatenate([t.detach().float().numpy().reshape(-1) for t in ref.tensor])
        else:
            a = ref.to_kernel(ref.tensor)
        out[off:off + a.size] = a
    return out


def params_from_image(b: "_Builder", flat: np.ndarray) -> dict:
    """Torch-layout tensors (by parameter name) from a flat kernel-layout image."""
    out = {}
    for ref in b.prog.params:
        off = ref.buf.sub_offset // 4
        if isinstance(ref.tensor, tuple):
            g, bt = ref.tensor
            c = g.numel()
            out[ref.name] = (torch.from_numpy(flat[off:off + c].copy()),
                             torch.from_numpy(flat[off + c:off + 2 * c].copy()))
        else:
            a = flat[off:off + ref.tensor.numel()]
            out[ref.name] = ref.from_kernel(a, tuple(ref.tensor.shape))
    return out


def running_image(b: "_Builder") -> list:
    return [(m, np.concatenate([m.running_mean.detach().float().numpy(),
                                m.running_var.detach().float().numpy()]), buf)
            for m, buf in b.prog.running]


def lower_train(b: "_Builder", base: int):
    ops = (N.OpDesc * len(b.prog.tasks))()
    ptr = lambda buf: base + buf.offset  # noqa: E731
    for t in b.prog.tasks:
        t.fill(ops[t.tid], ptr)
    return ops


# ----------------------------------------------------------------------------
# engine
# ----------------------------------------------------------------------------

class TrainEngine:
    """AoT training engine: ``prepare(x, y)`` then ``step(x, y) -> loss``."""

    def __init__(self, model: nn.Module, lr: float = 0.05, momentum: float = 0.9,
                 weight_decay: float = 4e-5, multi_stream: bool = True, device: int = 0,
                 world: int = 1, rank: int = 0, allreduce: bool | None = None, pdl: bool = False,
                 autotune: bool = True, fuse_bn: bool = True):
        self.model = model
        self.lr, self.momentum, self.wd = lr, momentum, weight_decay
        self.multi_stream = multi_stream
        self.device = device
        self.world, self.rank = world, rank
        self.allreduce = (world > 1) if allreduce is None else allreduce
        self.pdl = pdl
        self.autotune = autotune
        self.fuse_bn = fuse_bn
        self.tuning = {}
        self._h = None
        self.prepared = False

    def _autotune(self, reps: int = 5):
        """Kernel selection for the K_CONV tasks (forward convs and 1x1 dgrads),
        as in Engine._autotune: every SIMT / TMA-pointwise tile x split-K
        candidate timed as a graph-captured chain; tcgen05 candidates that need
        weights pre-split at prepare are excluded (these change every step) —
        the pointwise tcgen05 kernel's in-kernel-split variants stay.  Only
        activation / gradient buffers are written while timing."""
        lib = N.lib()
        us = C.c_double()
        for t in self.prog.tasks:
            d = self.ops[t.tid]
            if d.kind != K_CONV:
                continue
            p = d.params
            M = p[SP_N] * p[SP_P] * p[SP_Q]
            # tcgen05 candidates need prepare-time weight copies, except the
            # pointwise kernel's in-kernel-split variants (8100 + BN), which
            # read the step's current fp32 weights
            cands = [c for c in conv_candidates(M, p[SP_K], p[SP_R] * p[SP_S] * p[SP_C], p[SP_R], p[SP_S],
                                                (p[SP_PAD_H], p[SP_PAD_W]))
                     if c[0] != K_CONV_TC or 8100 <= c[1] < 8300]
            trial = N.OpDesc()
            C.memmove(C.byref(trial), C.byref(d), C.sizeof(N.OpDesc))
            best = None
            for kind, variant, split in cands:
                trial.kind, trial.variant = kind, variant
                trial.params[SP_SPLIT_K] = split
                if lib.sw_engine_time_op(self._h, C.byref(trial), reps, C.byref(us)) != 0:
                    continue
                if best is None or us.value < best[0]:
                    best = (us.value, kind, variant, split)
            if best is not None:
                d.kind, d.variant = best[1], best[2]
                d.params[SP_SPLIT_K] = best[3]
                self.tuning[t.tid] = best
        N.check(lib.sw_engine_synchronize(self._h))

    def prepare(self, x: torch.Tensor, y: torch.Tensor) -> "TrainEngine":
        lib = N.lib()
        if not torch.cuda.is_available():
            raise CudaError("TrainEngine.prepare needs a CUDA device (there is no CPU fallback)")
        t0 = time.perf_counter()
        b = build_train_program(self.model, tuple(x.shape), self.lr, self.momentum, self.wd,
                                self.allreduce, self.fuse_bn)
        self.builder, self.prog = b, b.prog
        g = b.prog.graph
        t1 = time.perf_counter()
        f, plan, meg = assign_streams_full(g)
        ts = pre_run(g, f, plan)
        ts_single = pre_run(g, StreamAssignment({t.id: 0 for t in g.nodes}), SyncPlan(()))
        t2 = time.perf_counter()
        self.graph, self.assignment, self.plan, self.meg = g, f, plan, meg
        self.schedule, self.schedule_single = ts, ts_single
        dev = torch.device("cuda", self.device)
        self.arena = torch.zeros(max(b.prog.arena_bytes, 256), dtype=torch.uint8, device=dev)
        base = self.arena.data_ptr()
        self.base = base
        # parameters, running stats, the ones vector
        flat = torch.from_numpy(initial_param_image(b)).to(dev)
        self._dev_view(b.flat_p, torch.float32).copy_(flat)
        for m, img, rb in running_image(b):
            self._dev_view(rb, torch.float32).copy_(torch.from_numpy(img).to(dev))
        self._dev_view(b.ones, torch.float32).fill_(1.0)
        torch.cuda.current_stream(dev).synchronize()  # the engine's stream is not ordered after torch's
        self.ops = lower_train(b, base)
        self.h_in = torch.empty(tuple(x.shape), dtype=torch.float32).pin_memory()
        self.h_lab = torch.empty((x.shape[0],), dtype=torch.int32).pin_memory()
        self.h_loss = torch.empty((1,), dtype=torch.float32).pin_memory()
        h = C.c_void_p()
        N.check(lib.sw_engine_create(self.device, C.byref(h)))
        self._h = h
        N.check(lib.sw_engine_set_io(h, self.h_in.data_ptr(), base + b.input.offset, self.h_in.numel() * 4,
                                     self.h_loss.data_ptr(), base + b.loss.offset, 4))
        N.check(lib.sw_engine_add_input(h, self.h_lab.data_ptr(), base + b.labels.offset,
                                        self.h_lab.numel() * 4))
        # kernel-node host staging (images, labels in; loss out): SW_ENGINE_KERNEL_IO
        N.check(lib.sw_engine_set_flags(h, (1 if self.pdl else 0) | 4))
        if self.allreduce:
            self._init_nccl()
        t_tune = time.perf_counter()
        if self.autotune:
            self._autotune()
        self.tune_seconds = time.perf_counter() - t_tune
        N.check(lib.sw_engine_set_ops(h, len(b.prog.tasks), self.ops))
        t3 = time.perf_counter()
        for slot, sched, io in ((SLOT_MULTI_IO, ts, 1), (SLOT_SINGLE_IO, ts_single, 1),
                                (SLOT_MULTI, ts, 0), (SLOT_SINGLE, ts_single, 0)):
            lens, kinds, args, order = schedule_arrays(sched)
            N.check(lib.sw_engine_capture(h, slot, len(sched.streams), N.ptr64(lens), N.ptr32(kinds),
                                          N.ptr64(args), len(sched.order), N.ptr64(order), io))
        self.plan_seconds = {"build": t1 - t0, "assign+pre_run": t2 - t1,
                             "lower+capture": time.perf_counter() - t3}
        self.eager_order = np.asarray([op.arg for s in ts_single.streams for op in s], dtype=np.int64)
        self.prepared = True
        return self

    def _init_nccl(self):
        import os
        lib = N.lib()
        path = b""
        try:
            import nvidia.nccl as _nc
            cand = os.path.join(list(_nc.__path__)[0], "lib", "libnccl.so.2")
            if os.path.exists(cand):
                path = cand.encode()
        except ImportError:
            pass
        N.check(lib.sw_nccl_load(path))
        uid = C.create_string_buffer(128)
        if self.rank == 0:
            N.check(lib.sw_nccl_unique_id(uid))
        if self.world > 1:
            import torch.distributed as dist
            obj = [bytes(uid.raw)]
            dist.broadcast_object_list(obj, src=0)
            uid = C.create_string_buffer(obj[0], 128)
        N.check(lib.sw_engine_nccl_init(self._h, self.world, self.rank, uid))

    def _dev_view(self, buf: Buf, dtype) -> torch.Tensor:
        nb = buf.nbytes
        return self.arena[buf.offset: buf.offset + nb].view(dtype)

    # -- execution --
    def step(self, x: torch.Tensor, y: torch.Tensor) -> float:
        """One training iteration from host tensors (public API): pinned H2D of
        images + labels, the captured step, D2H of the loss."""
        self.h_in.copy_(x.detach().reshape(self.h_in.shape))
        self.h_lab.copy_(y.detach().to(torch.int32).reshape(-1))
        slot = SLOT_MULTI_IO if self.multi_stream else SLOT_SINGLE_IO
        N.check(N.lib().sw_engine_replay_sync(self._h, slot, None))
        return float(self.h_loss[0])

    def load_batch_device(self, x: torch.Tensor, y: torch.Tensor):
        b = self.builder
        self._dev_view(b.input, torch.float32).copy_(x.detach().reshape(-1).to(self.arena.device))
        self._dev_view(b.labels, torch.int32).copy_(y.detach().to(torch.int32).reshape(-1).to(self.arena.device))
        torch.cuda.current_stream(self.arena.device).synchronize()  # see engine._torch_done

    def replay(self, multi: bool = True, io: bool = False):
        slot = (SLOT_MULTI_IO if multi else SLOT_SINGLE_IO) if io else (SLOT_MULTI if multi else SLOT_SINGLE)
        N.check(N.lib().sw_engine_replay(self._h, slot))

    def run_eager(self):
        lib = N.lib()
        for t in self.eager_order:
            N.check(lib.sw_engine_launch_op(self._h, int(t)))

    def synchronize(self):
        N.check(N.lib().sw_engine_synchronize(self._h))

    def run_framework(self, multi: bool = True):
        """Framework (non-AoT) mode of the training step: the pre_run schedule
        issued op by op by the host on the logical streams (sim.py:69-80)."""
        ts = self.schedule if multi else self.schedule_single
        lens, kinds, args, order = schedule_arrays(ts)
        N.check(N.lib().sw_engine_run_schedule(self._h, len(ts.streams), N.ptr64(lens), N.ptr32(kinds),
                                               N.ptr64(args), len(ts.order), N.ptr64(order)))

    def device_loss(self) -> float:
        return float(self._dev_view(self.builder.loss, torch.float32)[0].item())

    def stream(self):
        sh = C.c_uint64()
        N.check(N.lib().sw_engine_stream(self._h, C.byref(sh)))
        return torch.cuda.ExternalStream(sh.value, device=torch.device("cuda", self.device))

    def parameters(self) -> dict:
        """Current parameters in torch layout (host), by traced parameter name."""
        self.synchronize()
        flat = self._dev_view(self.builder.flat_p, torch.float32)[: self.builder.param_floats].cpu().numpy()
        return params_from_image(self.builder, flat)

    def gradients(self) -> dict:
        self.synchronize()
        flat = self._dev_view(self.builder.flat_g, torch.float32)[: self.builder.param_floats].cpu().numpy()
        return params_from_image(self.builder, flat)

    def running_stats(self) -> list:
        self.synchronize()
        out = []
        for m, rb in self.builder.prog.running:
            v = self._dev_view(rb, torch.float32).cpu()
            c = v.numel() // 2
            out.append((m, v[:c].clone(), v[c:].clone()))
        return out

    def profile_tasks(self, reps: int = 10) -> np.ndarray:
        """Device µs per task, each timed as a graph-captured chain of `reps`
        launches (sw_engine_profile_ops).  Tasks that accumulate in place or
        update state (SGD, running stats) are re-run, so call this on a
        throw-away engine or re-prepare afterwards."""
        out = np.zeros(len(self.eager_order), dtype=np.float64)
        N.check(N.lib().sw_engine_profile_ops(self._h, len(self.eager_order), N.ptr64(self.eager_order), reps,
                                              out.ctypes.data_as(C.POINTER(C.c_double))))
        res = np.zeros_like(out)
        res[self.eager_order] = out
        return res

    def time_replay(self, multi: bool = True, iters: int = 50, io: bool = False):
        slot = (SLOT_MULTI_IO if multi else SLOT_SINGLE_IO) if io else (SLOT_MULTI if multi else SLOT_SINGLE)
        gpu = C.c_double()
        host = C.c_double()
        N.check(N.lib().sw_engine_time_replay(self._h, slot, iters, C.byref(gpu), C.byref(host)))
        return gpu.value, host.value

    def close(self):
        if self._h is not None:
            N.lib().sw_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
