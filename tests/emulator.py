"""Host emulation of the engine's op table — TEST INFRASTRUCTURE ONLY.

Executes exactly the sw_op_desc records `engine.lower_program` produces (same
params, strides, pointers) against one host numpy "device memory", with each
kernel kind restated in torch CPU ops.  It lets the CPU test suite check the
op-DAG builder, fusion passes, zero-copy concat placement and parameter
encoding against the model's own CPU forward, before any GPU time is spent.
It is never used by the product path (engine.py has no CPU fallback).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from paper_2012_02732_b200 import engine as E
from paper_2012_02732_b200.schedule import pre_run
from paper_2012_02732_b200.assign import StreamAssignment, SyncPlan
from paper_2012_02732_b200.trace import build_program


class HostMemory:
    def __init__(self, nbytes):
        self.buf = np.zeros((nbytes + 4095) // 4, dtype=np.float32)
        self.base = self.buf.ctypes.data
        self.top = 0

    def alloc(self, nbytes):
        off = self.top
        self.top += (nbytes + 255) // 256 * 256
        assert self.top <= self.buf.nbytes
        return self.base + off

    def idx(self, ptr):
        assert (ptr - self.base) % 4 == 0
        return (ptr - self.base) // 4

    def gather(self, ptr, shape, strides):
        n, c, h, w = shape
        sn, sh, sw, sc = strides
        i = self.idx(ptr) + (np.arange(n)[:, None, None, None] * sn + np.arange(c)[None, :, None, None] * sc
                             + np.arange(h)[None, None, :, None] * sh + np.arange(w)[None, None, None, :] * sw)
        return torch.from_numpy(self.buf[i].copy())

    def scatter(self, ptr, t, strides):
        n, c, h, w = t.shape
        sn, sh, sw, sc = strides
        i = self.idx(ptr) + (np.arange(n)[:, None, None, None] * sn + np.arange(c)[None, :, None, None] * sc
                             + np.arange(h)[None, None, :, None] * sh + np.arange(w)[None, None, None, :] * sw)
        self.buf[i] = t.numpy()


def _act(x, a):
    if a == 1:
        return F.relu(x)
    if a == 2:
        return F.relu6(x)
    if a == 3:
        return F.silu(x)
    if a == 4:
        return torch.sigmoid(x)
    return x


def _window(x, ph, pw, P, Q, R, S, sh, sw, fill):
    """Zero/fill-padded input covering exactly the P x Q output windows."""
    n, c, h, w = x.shape
    Hp = (P - 1) * sh + R
    Wp = (Q - 1) * sw + S
    out = torch.full((n, c, Hp, Wp), fill, dtype=x.dtype)
    valid = torch.zeros((Hp, Wp), dtype=torch.bool)
    for r in range(Hp):
        ih = r - ph
        if 0 <= ih < h:
            lo = max(0, pw)
            hi = min(Wp, w + pw)
            if lo < hi:
                out[:, :, r, lo:hi] = x[:, :, ih, lo - pw:hi - pw]
                valid[r, lo:hi] = True
    return out, valid


def _sep2(mem, d, p, q):
    """K_SEP2 = two chained sepconvs (csrc/kernels/sep2.cu)."""
    Nb, H, W, Cc, P, Q, K, R = (p[E.SP_N], p[E.SP_H], p[E.SP_W], p[E.SP_C], p[E.SP_P], p[E.SP_Q],
                                p[E.SP_K], p[E.SP_R])
    mid = p[E.S2_MID]
    base = mem.idx(q[E.PT_W])

    def arr(off, n):
        return torch.from_numpy(mem.buf[base + off:base + off + n].copy()).double()
    x = mem.gather(q[E.PT_IN], (Nb, Cc, H, W), (p[E.SP_IN_SN], p[E.SP_IN_SH], p[E.SP_IN_SW], p[E.SP_IN_SC]))
    if p[E.SP_PRE_RELU]:
        x = F.relu(x)
    sh, sw, ph, pw = p[E.SP_STRIDE_H], p[E.SP_STRIDE_W], p[E.SP_PAD_H], p[E.SP_PAD_W]
    w1 = arr(p[E.S2_OFF_DW1], R * R * Cc).view(R, R, Cc).permute(2, 0, 1)[:, None]
    xw, _ = _window(x, ph, pw, P, Q, R, R, sh, sw, 0.0)
    y = F.conv2d(xw.double(), w1, stride=(sh, sw), groups=Cc)
    if p[E.S2_OFF_DB1] >= 0:
        y = y + arr(p[E.S2_OFF_DB1], Cc).view(1, -1, 1, 1)
    y = _act(y.float(), p[E.S2_DW_ACT1]).double()
    pw1 = arr(p[E.S2_OFF_PW1], Cc * mid).view(Cc, mid).t()
    y = F.conv2d(y, pw1[:, :, None, None]) + arr(p[E.S2_OFF_B1], mid).view(1, -1, 1, 1)
    y = _act(y.float(), p[E.S2_ACT1])
    if p[E.S2_PRE_RELU2]:
        y = F.relu(y)
    w2 = arr(p[E.S2_OFF_DW2], R * R * mid).view(R, R, mid).permute(2, 0, 1)[:, None]
    y = F.conv2d(y.double(), w2, padding=R // 2, groups=mid)
    if p[E.S2_OFF_DB2] >= 0:
        y = y + arr(p[E.S2_OFF_DB2], mid).view(1, -1, 1, 1)
    y = _act(y.float(), p[E.S2_DW_ACT2]).double()
    pw2 = arr(p[E.S2_OFF_PW2], mid * K).view(mid, K).t()
    y = (F.conv2d(y, pw2[:, :, None, None]) + arr(p[E.S2_OFF_B2], K).view(1, -1, 1, 1)).float()
    if p[E.SP_HAS_RES]:
        y = y + mem.gather(q[E.PT_RES], (Nb, K, P, Q),
                           (p[E.SP_RES_SN], p[E.SP_RES_SH], p[E.SP_RES_SW], p[E.SP_RES_SC] or 1))
    y = _act(y, p[E.SP_ACT])
    mem.scatter(q[E.PT_OUT], y, (p[E.SP_OUT_SN], p[E.SP_OUT_SH], p[E.SP_OUT_SW], p[E.SP_OUT_SC] or 1))


def run_op(mem: HostMemory, d):
    p = list(d.params)
    q = list(d.ptrs)
    if d.kind == E.K_SEP2:
        _sep2(mem, d, p, q)
        return
    if d.kind in (E.K_CONV, E.K_DWCONV, E.K_POOL, E.K_SEPCONV):
        Nb, H, W, Cc, P, Q, K, R, S = (p[E.SP_N], p[E.SP_H], p[E.SP_W], p[E.SP_C], p[E.SP_P],
                                       p[E.SP_Q], p[E.SP_K], p[E.SP_R], p[E.SP_S])
        sh, sw, ph, pw = p[E.SP_STRIDE_H], p[E.SP_STRIDE_W], p[E.SP_PAD_H], p[E.SP_PAD_W]
        x = mem.gather(q[E.PT_IN], (Nb, Cc, H, W),
                       (p[E.SP_IN_SN], p[E.SP_IN_SH], p[E.SP_IN_SW], p[E.SP_IN_SC]))
        if p[E.SP_PRE_RELU]:
            x = F.relu(x)
        if d.kind == E.K_CONV:
            w = torch.from_numpy(mem.buf[mem.idx(q[E.PT_W]):mem.idx(q[E.PT_W]) + K * R * S * Cc].copy())
            w = w.view(K, R, S, Cc).permute(0, 3, 1, 2)
            xw, _ = _window(x, ph, pw, P, Q, R, S, sh, sw, 0.0)
            y = F.conv2d(xw.double(), w.double(), stride=(sh, sw)).float()
            if q[E.PT_BIAS]:
                b = torch.from_numpy(mem.buf[mem.idx(q[E.PT_BIAS]):mem.idx(q[E.PT_BIAS]) + K].copy())
                y = y + b.view(1, -1, 1, 1)
        elif d.kind == E.K_SEPCONV:
            wdw = torch.from_numpy(mem.buf[mem.idx(q[E.PT_WS]):mem.idx(q[E.PT_WS]) + R * S * Cc].copy())
            wdw = wdw.view(R, S, Cc).permute(2, 0, 1)[:, None]
            xw, _ = _window(x, ph, pw, P, Q, R, S, sh, sw, 0.0)
            dwo = F.conv2d(xw.double(), wdw.double(), stride=(sh, sw), groups=Cc)
            if q[E.PT_DW_BIAS]:
                bdw = torch.from_numpy(mem.buf[mem.idx(q[E.PT_DW_BIAS]):mem.idx(q[E.PT_DW_BIAS]) + Cc].copy())
                dwo = dwo + bdw.double().view(1, -1, 1, 1)
            dwo = _act(dwo.float(), p[E.SP_DW_ACT])
            wpw = torch.from_numpy(mem.buf[mem.idx(q[E.PT_W]):mem.idx(q[E.PT_W]) + K * Cc].copy()).view(Cc, K).t()
            y = F.conv2d(dwo.double(), wpw.double()[:, :, None, None]).float()
            if q[E.PT_BIAS]:
                b = torch.from_numpy(mem.buf[mem.idx(q[E.PT_BIAS]):mem.idx(q[E.PT_BIAS]) + K].copy())
                y = y + b.view(1, -1, 1, 1)
        elif d.kind == E.K_DWCONV:
            w = torch.from_numpy(mem.buf[mem.idx(q[E.PT_W]):mem.idx(q[E.PT_W]) + R * S * Cc].copy())
            w = w.view(R, S, Cc).permute(2, 0, 1)[:, None]
            xw, _ = _window(x, ph, pw, P, Q, R, S, sh, sw, 0.0)
            y = F.conv2d(xw.double(), w.double(), stride=(sh, sw), groups=Cc).float()
            if q[E.PT_BIAS]:
                b = torch.from_numpy(mem.buf[mem.idx(q[E.PT_BIAS]):mem.idx(q[E.PT_BIAS]) + Cc].copy())
                y = y + b.view(1, -1, 1, 1)
            K = Cc
        else:
            K = Cc
            if p[E.SP_POOL_MODE] == 0:
                xw, _ = _window(x, ph, pw, P, Q, R, S, sh, sw, float("-inf"))
                y = F.max_pool2d(xw, (R, S), (sh, sw))
            else:
                xw, valid = _window(x, ph, pw, P, Q, R, S, sh, sw, 0.0)
                s = F.avg_pool2d(xw.double(), (R, S), (sh, sw)) * (R * S)
                if p[E.SP_COUNT_PAD]:
                    cnt = torch.zeros(P, Q)
                    for i in range(P):
                        for j in range(Q):
                            hs = i * sh - ph
                            ws = j * sw - pw
                            he = min(hs + R, H + p[E.SP_PAD_BOTTOM])
                            we = min(ws + S, W + p[E.SP_PAD_RIGHT])
                            cnt[i, j] = (he - hs) * (we - ws)
                else:
                    cnt = F.avg_pool2d(valid.double()[None, None], (R, S), (sh, sw))[0, 0] * (R * S)
                y = (s / cnt.double().clamp(min=1)).float()
            if p[E.SP_POOL_MUL] > 1:
                y = y * float(p[E.SP_POOL_MUL])
        if p[E.SP_HAS_RES]:
            r = mem.gather(q[E.PT_RES], (Nb, K, P, Q),
                           (p[E.SP_RES_SN], p[E.SP_RES_SH], p[E.SP_RES_SW], p[E.SP_RES_SC] or 1))
            y = y + r
        y = _act(y, p[E.SP_ACT])
        osc = p[E.SP_OUT_SC] or 1
        mem.scatter(q[E.PT_OUT], y, (p[E.SP_OUT_SN], p[E.SP_OUT_SH], p[E.SP_OUT_SW], osc))
    elif d.kind in (E.K_ELTWISE, E.K_GLOBAL_POOL):
        Nb, H, W, Cc = p[E.EW_N], p[E.EW_H], p[E.EW_W], p[E.EW_C]
        a = mem.gather(q[E.EP_A], (Nb, Cc, H, W), tuple(p[E.EW_A_SN:E.EW_A_SN + 4]))
        if p[E.EW_PRE_RELU]:
            a = F.relu(a)
        if d.kind == E.K_GLOBAL_POOL:
            y = _act(a.double().mean(dim=(2, 3), keepdim=True).float(), p[E.EW_ACT])
            mem.scatter(q[E.EP_OUT], y, tuple(p[E.EW_O_SN:E.EW_O_SN + 4]))
            return
        nin = p[E.EW_NIN]
        b = mem.gather(q[E.EP_B], (Nb, Cc, H, W), tuple(p[E.EW_B_SN:E.EW_B_SN + 4])) if nin > 1 else 0
        c = mem.gather(q[E.EP_C], (Nb, Cc, H, W), tuple(p[E.EW_C_SN:E.EW_C_SN + 4])) if nin > 2 else 0
        op = p[E.EW_OP]
        if op == E.EW_ADD:
            y = a + b + c
        elif op == E.EW_MUL:
            y = a * b
        elif op == E.EW_AFFINE:
            sc = torch.from_numpy(mem.buf[mem.idx(q[E.EP_SCALE]):mem.idx(q[E.EP_SCALE]) + Cc].copy())
            shf = torch.from_numpy(mem.buf[mem.idx(q[E.EP_SHIFT]):mem.idx(q[E.EP_SHIFT]) + Cc].copy())
            y = a * sc.view(1, -1, 1, 1) + shf.view(1, -1, 1, 1)
        else:
            y = a
        mem.scatter(q[E.EP_OUT], _act(y, p[E.EW_ACT]), tuple(p[E.EW_O_SN:E.EW_O_SN + 4]))
    elif d.kind == E.K_CONCAT:
        Nb, H, W, nin, ctot = p[0], p[1], p[2], p[3], p[4]
        osc = p[5] or 1
        parts = []
        for i in range(nin):
            ci = p[8 + i]
            parts.append(mem.gather(q[i], (Nb, ci, H, W), (H * W * ci, W * ci, ci, 1)))
        y = torch.cat(parts, 1)
        strides = (H * W * ctot, W * ctot, ctot, 1) if osc == 1 else (ctot * H * W, W, 1, H * W)
        mem.scatter(q[7], y, strides)
    else:
        raise NotImplementedError(d.kind)


def emulate(model, x, fuse=True, multi_stream=True, hb_arena=False, fuse_sep_pairs=False):
    """Run the lowered program on the host; returns (output, program, ops).
    hb_arena=True places the activations with the engine's happens-before
    arena (arena.py): storages share memory wherever the capture orders them."""
    prog = build_program(model, x, fuse=fuse, fuse_sep_pairs=fuse_sep_pairs)
    g = prog.graph
    total = sum(st.alloc_bytes for st in prog.storages)
    arrays = E._pack_weights(prog)
    wtotal = sum((a.nbytes + 255) // 256 * 256 for a in arrays.values())
    mem = HostMemory(total + wtotal + 8192)
    if hb_arena:
        from paper_2012_02732_b200 import assign_streams as _as
        from paper_2012_02732_b200.arena import plan_arena
        f0, p0 = _as(g) if multi_stream else (StreamAssignment({t.id: 0 for t in g.nodes}), SyncPlan(()))
        layout = plan_arena(prog, pre_run(g, f0, p0))
        abase = mem.alloc(layout.total)
        base = {st.sid: (mem.alloc(st.alloc_bytes) if st.role == "input" else abase + layout.offsets[st.sid])
                for st in prog.storages}
    else:
        base = {st.sid: mem.alloc(st.alloc_bytes) for st in prog.storages}
    wbase = mem.alloc(wtotal)
    woff = {}
    off = 0
    for key, a in arrays.items():
        woff[key] = off
        i = mem.idx(wbase + off)
        mem.buf[i:i + a.size] = a
        off += (a.nbytes + 255) // 256 * 256
    ops = E.lower_program(prog, lambda st: base[st.sid], wbase, woff)
    inp = prog.input_view.st
    i0 = mem.idx(base[inp.sid])
    mem.buf[i0:i0 + x.numel()] = x.reshape(-1).numpy()
    # execute in the multi-stream capture order (a valid topological order)
    from paper_2012_02732_b200 import assign_streams
    if multi_stream:
        f, plan = assign_streams(g)
    else:
        f, plan = StreamAssignment({t.id: 0 for t in g.nodes}), SyncPlan(())
    ts = pre_run(g, f, plan)
    done = set()
    for s, op in _flat(ts):
        if op.kind == "launch":
            t = prog.tasks[op.arg]
            assert all(dep in done for dep in t.deps), "schedule violates a data dependency"
            run_op(mem, ops[op.arg])
            done.add(op.arg)
    out = prog.output_view
    o = out.st
    shape = (o.n, o.c, o.h, o.w)
    y = mem.gather(base[o.sid] + 4 * out.elem_offset(), shape, out.strides())
    if o.h * o.w == 1:
        y = y.reshape(o.n, o.c)
    return y, prog, ops


def _flat(ts):
    pos = [0] * len(ts.streams)
    for s in ts.order:
        yield s, ts.streams[s][pos[s]]
        pos[s] += 1
