"""Host emulation of the TRAINING op table — TEST INFRASTRUCTURE ONLY.

Runs exactly the sw_op_desc records `train.lower_train` produces (same params
and pointers into one host "arena") in the captured schedule order, with each
kernel kind restated in torch CPU ops (fp64 where the kernel reduces).  The CPU
suite uses it to check the training builder — grouping, gradient routing and
accumulation, parameter layouts, the optimizer — against torch autograd before
any GPU time is spent.  Never used by the product path.
"""

from __future__ import annotations

import struct

import numpy as np
import torch
import torch.nn.functional as F

from paper_2012_02732_b200 import train as T
from paper_2012_02732_b200.assign import StreamAssignment, SyncPlan, assign_streams_full
from paper_2012_02732_b200.schedule import pre_run

from emulator import HostMemory, _act, _flat, run_op


def _f(bits):
    return struct.unpack("<f", struct.pack("<i", int(bits)))[0]


def _act_grad(z, a):
    if a == 1:
        return (z > 0).to(z.dtype)
    if a == 2:
        return ((z > 0) & (z < 6)).to(z.dtype)
    if a == 3:
        s = torch.sigmoid(z)
        return s * (1 + z * (1 - s))
    if a == 4:
        s = torch.sigmoid(z)
        return s * (1 - s)
    return torch.ones_like(z)


def _vec(mem, ptr, n):
    i = mem.idx(ptr)
    return torch.from_numpy(mem.buf[i:i + n].copy())


def _put(mem, ptr, t):
    i = mem.idx(ptr)
    a = t.detach().float().reshape(-1).numpy()
    mem.buf[i:i + a.size] = a


def _mat(mem, ptr, rows, cols, ld):
    i = mem.idx(ptr)
    idx = i + np.arange(rows)[:, None] * ld + np.arange(cols)[None, :]
    return torch.from_numpy(mem.buf[idx].copy())


_PARTIALS = {}


def _clone_desc(d, kind, ptrs):
    from paper_2012_02732_b200 import _native as N
    e = N.OpDesc()
    e.kind = kind
    for i in range(len(d.params)):
        e.params[i] = d.params[i]
    for i, v in enumerate(ptrs):
        e.ptrs[i] = v
    return e


def run_train_op(mem: HostMemory, d, allreduce=None):
    p = list(d.params)
    q = list(d.ptrs)
    k = d.kind
    if k == T.K_BN_FWD:   # = K_BN_STATS then K_BN_APPLY
        run_train_op(mem, _clone_desc(d, T.K_BN_STATS, [q[0], q[1], q[2], 0, 0, 0, 0, q[7]]))
        run_train_op(mem, _clone_desc(d, T.K_BN_APPLY, [q[0], q[1], q[3], q[4], q[5], 0, 0, 0]))
        return
    if k == T.K_BN_BWD:   # = K_BN_BWD_REDUCE then K_BN_BWD_APPLY
        run_train_op(mem, _clone_desc(d, T.K_BN_BWD_REDUCE, [q[0], q[1], q[2], q[3], q[4], 0, 0, q[7]]))
        run_train_op(mem, _clone_desc(d, T.K_BN_BWD_APPLY, q[:7] + [0]))
        return
    if k in (T.K_BN_STATS, T.K_BN_APPLY, T.K_BN_BWD_REDUCE, T.K_BN_BWD_APPLY):
        M, Cc, HW, act, has_res = p[T.BN_M], p[T.BN_C], p[T.BN_HW], p[T.BN_ACT], p[T.BN_HAS_RES]
        ld = p[T.BN_LD] or Cc
        if k == T.K_BN_STATS:
            y = _mat(mem, q[0], M, Cc, ld).double()
            mean = y.mean(0)
            var = y.var(0, unbiased=False)
            eps, mom = _f(p[T.BN_EPS]), _f(p[T.BN_MOMENTUM])
            _put(mem, q[1], torch.cat([mean, 1.0 / torch.sqrt(var + eps)]))
            run = _vec(mem, q[2], 2 * Cc).double()
            unb = var * M / max(M - 1, 1)
            _put(mem, q[2], torch.cat([(1 - mom) * run[:Cc] + mom * mean, (1 - mom) * run[Cc:] + mom * unb]))
            return
        st = _vec(mem, q[1] if k == T.K_BN_APPLY else q[2], 2 * Cc).double()
        mean, istd = st[:Cc], st[Cc:]
        gb = _vec(mem, q[2] if k == T.K_BN_APPLY else q[3], 2 * Cc).double()
        g, b = gb[:Cc], gb[Cc:]
        y = _mat(mem, q[0] if k == T.K_BN_APPLY else q[1], M, Cc, ld).double()
        xh = (y - mean) * istd
        if k == T.K_BN_APPLY:
            o = g * xh + b
            if has_res:
                o = o + _mat(mem, q[3], M, Cc, ld).double()
            _put(mem, q[4], _act(o.float(), act))
            return
        sn, sp, scale = p[T.BN_DO_SN], p[T.BN_DO_SP], _f(p[T.BN_DO_SCALE]) if p[T.BN_DO_SCALE] else 1.0
        m = np.arange(M)
        idx = mem.idx(q[0]) + ((m // HW) * sn + (m % HW) * sp)[:, None] + np.arange(Cc)[None, :]
        dout = torch.from_numpy(mem.buf[idx].copy()).double() * scale
        dz = dout * _act_grad(g * xh + b, act)
        if k == T.K_BN_BWD_REDUCE:
            _put(mem, q[4], torch.cat([(dz * xh).sum(0), dz.sum(0)]))
            return
        dgb = _vec(mem, q[4], 2 * Cc).double()
        dy = g * istd * (dz - dgb[Cc:] / M - xh * dgb[:Cc] / M)
        if has_res:
            dy = dy + _mat(mem, q[5], M, Cc, ld).double()
        _put(mem, q[6], dy)
        return
    if k in (T.K_DW_DGRAD, T.K_DW_WGRAD):
        from paper_2012_02732_b200 import engine as E
        Nb, H, W, Cc, P, Q, R, S = (p[E.SP_N], p[E.SP_H], p[E.SP_W], p[E.SP_C], p[E.SP_P], p[E.SP_Q],
                                    p[E.SP_R], p[E.SP_S])
        st, pad = (p[E.SP_STRIDE_H], p[E.SP_STRIDE_W]), (p[E.SP_PAD_H], p[E.SP_PAD_W])
        dy = _vec(mem, q[0], Nb * P * Q * Cc).view(Nb, P, Q, Cc).permute(0, 3, 1, 2).double()
        if k == T.K_DW_DGRAD:
            w = _vec(mem, q[2], R * S * Cc).view(R, S, Cc).permute(2, 0, 1)[:, None].double()
            dx = torch.nn.grad.conv2d_input((Nb, Cc, H, W), w, dy, stride=st, padding=pad, groups=Cc)
            dx = dx.permute(0, 2, 3, 1)
            if p[E.SP_HAS_RES]:
                dx = dx + _vec(mem, q[4], dx.numel()).view(dx.shape).double()
            _put(mem, q[1], dx)
        else:
            x = _vec(mem, q[2], Nb * H * W * Cc).view(Nb, H, W, Cc).permute(0, 3, 1, 2).double()
            dw = torch.nn.grad.conv2d_weight(x, (Cc, 1, R, S), dy, stride=st, padding=pad, groups=Cc)
            _put(mem, q[1], dw[:, 0].permute(1, 2, 0))
        return
    if k == T.K_GEMM_REDUCE:
        M, Nn = p[T.GM_M], p[T.GM_N]
        Cm = _PARTIALS.pop(q[5])
        if q[3]:
            Cm = Cm + _vec(mem, q[3], Nn).double()[None, :]
        ic = mem.idx(q[2]) + np.arange(M)[:, None] * p[T.GM_C_I] + np.arange(Nn)[None, :]
        if p[T.GM_HAS_RES]:
            ir = mem.idx(q[4]) + np.arange(M)[:, None] * p[T.GM_C_I] + np.arange(Nn)[None, :]
            Cm = Cm + torch.from_numpy(mem.buf[ir].copy()).double()
        mem.buf[ic] = Cm.float().numpy()
        return
    if k == T.K_GEMM:
        M, Nn, K = p[T.GM_M], p[T.GM_N], p[T.GM_K]
        ia = mem.idx(q[0]) + np.arange(M)[:, None] * p[T.GM_A_I] + np.arange(K)[None, :] * p[T.GM_A_R]
        A = torch.from_numpy(mem.buf[ia].copy()).double()
        if p[T.GM_IM2COL]:
            xn, xh, xw, xc = p[T.GM_X_N], p[T.GM_X_H], p[T.GM_X_W], p[T.GM_X_C]
            P_, Q_, R, S = p[T.GM_X_P], p[T.GM_X_Q], p[T.GM_X_R], p[T.GM_X_S]
            stv, pad = p[T.GM_X_STRIDE], p[T.GM_X_PAD]
            x = mem.gather(q[1], (xn, xc, xh, xw),
                           (p[T.GM_X_SN], p[T.GM_X_SH], p[T.GM_X_SW], p[T.GM_X_SC])).double()
            cols = F.unfold(x, (R, S), padding=pad, stride=stv)  # [n, c*R*S, P*Q] (c-major)
            cols = cols.view(xn, xc, R, S, P_ * Q_).permute(0, 4, 2, 3, 1).reshape(xn * P_ * Q_, R * S * xc)
            B = cols
        else:
            ib = mem.idx(q[1]) + np.arange(K)[:, None] * p[T.GM_B_R] + np.arange(Nn)[None, :] * p[T.GM_B_J]
            B = torch.from_numpy(mem.buf[ib].copy()).double()
        Cm = A @ B
        if p[T.GM_PARTIALS_ONLY]:
            _PARTIALS[q[5]] = Cm  # folded by the K_GEMM_REDUCE op
            return
        if q[3]:
            Cm = Cm + _vec(mem, q[3], Nn).double()[None, :]
        ic = mem.idx(q[2]) + np.arange(M)[:, None] * p[T.GM_C_I] + np.arange(Nn)[None, :]
        if p[T.GM_HAS_RES]:
            ir = mem.idx(q[4]) + np.arange(M)[:, None] * p[T.GM_C_I] + np.arange(Nn)[None, :]
            Cm = Cm + torch.from_numpy(mem.buf[ir].copy()).double()
        mem.buf[ic] = Cm.float().numpy()
        return
    if k == T.K_XENT:
        Nb, K, ld = p[0], p[1], p[2]
        z = _mat(mem, q[0], Nb, K, ld).double()
        lab = torch.from_numpy(mem.buf[mem.idx(q[1]):mem.idx(q[1]) + Nb].view(np.int32).astype(np.int64))
        loss = F.cross_entropy(z, lab)
        sm = torch.softmax(z, 1)
        sm[torch.arange(Nb), lab] -= 1
        _put(mem, q[2], loss.reshape(1))
        _put(mem, q[3], sm / Nb)
        return
    if k == T.K_SGD:
        n = p[0]
        lr, mu, wd = _f(p[1]), _f(p[2]), _f(p[3])
        w = _vec(mem, q[0], n)
        g = _vec(mem, q[1], n)
        b = _vec(mem, q[2], n)
        b = mu * b + (g + wd * w)
        _put(mem, q[2], b)
        _put(mem, q[0], w - lr * b)
        return
    if k == T.K_ALLREDUCE:
        if allreduce is not None:
            n = p[0]
            g = _vec(mem, q[0], n)
            _put(mem, q[0], allreduce(g))
        return
    if k == T.K_TRANSPOSE:
        rows, cols = p[0], p[1]
        _put(mem, q[1], _vec(mem, q[0], rows * cols).view(rows, cols).t().contiguous())
        return
    if k == T.K_EW_BWD:
        Nb, HW, Cc, mode, act, has_res = p[0], p[1], p[2], p[3], p[4], p[5]
        if mode == T.EWB_MUL_S:
            dy = _vec(mem, q[0], Nb * HW * Cc).view(Nb, HW, Cc).double()
            x = _vec(mem, q[1], Nb * HW * Cc).view(Nb, HW, Cc).double()
            ds = (dy * x).sum(1)
            if act:
                ds = ds * _act_grad(_vec(mem, q[5], Nb * Cc).view(Nb, Cc).double(), act)
            _put(mem, q[4], ds)
            return
        if mode == T.EWB_ACT:
            dy = _vec(mem, q[0], Nb * HW * Cc).double()
            v = dy * _act_grad(_vec(mem, q[1], Nb * HW * Cc).double(), act)
        elif mode == T.EWB_MUL_X:
            dy = _vec(mem, q[0], Nb * HW * Cc).view(Nb, HW, Cc).double()
            v = (dy * _vec(mem, q[2], Nb * Cc).view(Nb, 1, Cc).double()).reshape(-1)
        else:
            s = _vec(mem, q[2], Nb * Cc).view(Nb, 1, Cc).double() * _f(p[6])
            v = s.expand(Nb, HW, Cc).reshape(-1)
        if has_res:
            v = v + _vec(mem, q[3], Nb * HW * Cc).double()
        _put(mem, q[4], v)
        return
    run_op(mem, d)


class TrainEmulator:
    """A training step on the host with the engine's buffers and op table."""

    def __init__(self, model, x_shape, lr=0.05, momentum=0.9, weight_decay=4e-5, multi_stream=True,
                 allreduce=None):
        self.b = T.build_train_program(model, x_shape, lr, momentum, weight_decay,
                                       allreduce=allreduce is not None)
        self.allreduce_fn = allreduce
        prog = self.b.prog
        self.mem = HostMemory(prog.arena_bytes + 8192)
        self.base = self.mem.alloc(prog.arena_bytes)
        init = T.initial_param_image(self.b)
        i0 = self.mem.idx(self.base + self.b.flat_p.offset)
        self.mem.buf[i0:i0 + init.size] = init
        for m, img, rb in T.running_image(self.b):
            j = self.mem.idx(self.base + rb.offset)
            self.mem.buf[j:j + img.size] = img
        j = self.mem.idx(self.base + self.b.ones.offset)
        self.mem.buf[j:j + self.b.ones.nbytes // 4] = 1.0
        self.ops = T.lower_train(self.b, self.base)
        g = prog.graph
        if multi_stream:
            f, plan, _ = assign_streams_full(g)
        else:
            f, plan = StreamAssignment({t.id: 0 for t in g.nodes}), SyncPlan(())
        self.schedule = pre_run(g, f, plan)
        self.assignment, self.plan = f, plan

    def step(self, x, y):
        b, mem = self.b, self.mem
        i = mem.idx(self.base + b.input.offset)
        mem.buf[i:i + x.numel()] = x.reshape(-1).float().numpy()
        j = mem.idx(self.base + b.labels.offset)
        mem.buf[j:j + y.numel()] = y.to(torch.int32).numpy().view(np.float32)
        done = set()
        tasks = b.prog.tasks
        for s, op in _flat(self.schedule):
            if op.kind == "launch":
                t = tasks[op.arg]
                assert all(dep in done for dep in t.deps), "schedule violates a dependency"
                run_train_op(mem, self.ops[op.arg], self.allreduce_fn)
                done.add(op.arg)
        return float(mem.buf[mem.idx(self.base + b.loss.offset)])

    def _flat_view(self, buf):
        i = self.mem.idx(self.base + buf.offset)
        return self.mem.buf[i:i + self.b.param_floats].copy()

    def parameters(self):
        return T.params_from_image(self.b, self._flat_view(self.b.flat_p))

    def gradients(self):
        return T.params_from_image(self.b, self._flat_view(self.b.flat_g))

    def running_stats(self):
        out = []
        for m, rb in self.b.prog.running:
            i = self.mem.idx(self.base + rb.offset)
            c = rb.nbytes // 8
            v = torch.from_numpy(self.mem.buf[i:i + 2 * c].copy())
            out.append((m, v[:c], v[c:]))
        return out
