"""Happens-before-aware device arena (hard part H3).

The reference arena (`reserve_arena`, schedule.py:118-155) is first-fit over
the *linear* capture trace: a block freed by task X may be handed to a task Y
that runs concurrently with X on another stream — a race on a GPU.
The engine therefore used it only in its "never free" form (every activation
lives for the whole pass), which is race-free but sizes the arena as the sum of
all activations.

This planner reuses memory only where the *captured graph* orders the
accesses.  Happens-before (HB) is the reachability of the capture:

    stream FIFO order (consecutive LAUNCHes of one logical stream)
  ∪ sync edges (RECORD on the source's stream → WAIT before the destination)

— exactly what the CUDA graph enforces (the `enforced_closure` of the
reference's own tests, tests/_brute.py:129-160).  A storage T may overlap a
storage S in memory iff every task that touches S happens-before every task
that writes T.  Placement is first-fit in the walk order of T's first writer
over the storages T conflicts with.  Since the single-stream order is a
linearisation of the multi-stream HB order (pre_run emits every stream FIFO
along the same canonical walk), one layout serves both captured slots and the
eager launch loop.

Zero-copy concat storages have several writers (every producer writes its
channel slice), so "every writer of T" matters, not just the first.
"""

from __future__ import annotations

from dataclasses import dataclass

ALIGN = 256


@dataclass
class HbLayout:
    offsets: dict          # storage id -> byte offset
    total: int             # arena bytes
    reference_total: int   # bytes of the never-free layout (sum of storages)
    conflicts: int         # storage pairs that must not overlap


def happens_before(ts, n_tasks: int) -> list[int]:
    """desc[t]: bitset (python int) of tasks that t happens-before in the
    capture of schedule `ts` (stream FIFO + sync edges), excluding t."""
    succ = [set() for _ in range(n_tasks)]
    rec_task = {}   # event -> task launched last before the RECORD on its stream
    wait_next = []  # (event, stream, index in FIFO)
    for s, fifo in enumerate(ts.streams):
        last = None
        pending_waits = []
        for op in fifo:
            if op.kind == "launch":
                t = op.arg
                if last is not None:
                    succ[last].add(t)
                for ev in pending_waits:
                    wait_next.append((ev, t))
                pending_waits = []
                last = t
            elif op.kind == "record":
                rec_task[op.arg] = last
            else:
                pending_waits.append(op.arg)
    for ev, t in wait_next:
        u = rec_task.get(ev)
        if u is not None:
            succ[u].add(t)
    order = _topo(succ)
    desc = [0] * n_tasks
    for t in reversed(order):
        d = 0
        for v in succ[t]:
            d |= desc[v] | (1 << v)
        desc[t] = d
    return desc


def _topo(succ):
    n = len(succ)
    indeg = [0] * n
    for u in range(n):
        for v in succ[u]:
            indeg[v] += 1
    stack = [u for u in range(n) if indeg[u] == 0]
    out = []
    while stack:
        u = stack.pop()
        out.append(u)
        for v in succ[u]:
            indeg[v] -= 1
            if indeg[v] == 0:
                stack.append(v)
    if len(out) != n:
        raise ValueError("capture order has a cycle")
    return out


def plan_arena(prog, ts, exclude_roles=("input", "output")) -> HbLayout:
    """Offsets for every storage of `prog` (trace.Program) under schedule `ts`."""
    n = len(prog.tasks)
    desc = happens_before(ts, n)
    writers: dict[int, set] = {}
    access: dict[int, set] = {}
    for t in prog.tasks:
        writers.setdefault(t.out.st.sid, set()).add(t.tid)
        access.setdefault(t.out.st.sid, set()).add(t.tid)
        for v in list(t.inputs) + ([t.residual] if t.residual is not None else []):
            access.setdefault(v.st.sid, set()).add(t.tid)
    # after[S] = tasks that come after EVERY access of S (intersection of desc)
    full = (1 << n) - 1
    after = {}
    for sid, acc in access.items():
        a = full
        for t in acc:
            a &= desc[t]
        after[sid] = a
    # placement order: first writer's position in the canonical capture walk
    walk_pos = {}
    walk = []
    seen = set()
    cursor = [0] * len(ts.streams)
    for s in ts.order:
        op = ts.streams[s][cursor[s]]
        cursor[s] += 1
        if op.kind == "launch" and op.arg not in seen:
            seen.add(op.arg)
            walk.append(op.arg)
    for i, t in enumerate(walk):
        walk_pos[t] = i
    sts = [st for st in prog.storages if st.role not in exclude_roles and st.sid in writers]
    sts.sort(key=lambda st: (min(walk_pos[t] for t in writers[st.sid]), st.sid))
    placed = []  # (sid, off, size)
    offsets = {}
    total = 0
    conflicts = 0
    for st in sts:
        wmask = 0
        for t in writers[st.sid]:
            wmask |= 1 << t
        size = (st.nbytes + ALIGN - 1) // ALIGN * ALIGN
        busy = []
        for sid, off, sz in placed:
            if after[sid] & wmask != wmask:  # some writer of st is not after every access of sid
                busy.append((off, sz))
                conflicts += 1
        busy.sort()
        off = 0
        for b_off, b_sz in busy:
            if off + size <= b_off:
                break
            off = max(off, b_off + b_sz)
        offsets[st.sid] = off
        placed.append((st.sid, off, size))
        total = max(total, off + size)
    for st in prog.storages:
        if st.sid not in offsets and st.role not in exclude_roles:
            offsets[st.sid] = total
            total += (st.nbytes + ALIGN - 1) // ALIGN * ALIGN
    ref_total = sum((st.nbytes + ALIGN - 1) // ALIGN * ALIGN for st in prog.storages
                    if st.role not in exclude_roles)
    # storages excluded from reuse (network output) get their own range at the end
    for st in prog.storages:
        if st.role == "output":
            offsets[st.sid] = total
            total += (st.nbytes + ALIGN - 1) // ALIGN * ALIGN
            ref_total += (st.nbytes + ALIGN - 1) // ALIGN * ALIGN
    return HbLayout(offsets, max(total, ALIGN), ref_total, conflicts)


def check_layout(prog, ts, layout: HbLayout) -> None:
    """Independent safety check: any two storages whose byte ranges overlap
    are HB-ordered (all accesses of one before every access of the other)."""
    n = len(prog.tasks)
    desc = happens_before(ts, n)
    access: dict[int, set] = {}
    for t in prog.tasks:
        access.setdefault(t.out.st.sid, set()).add(t.tid)
        for v in list(t.inputs) + ([t.residual] if t.residual is not None else []):
            access.setdefault(v.st.sid, set()).add(t.tid)
    sizes = {st.sid: (st.nbytes + ALIGN - 1) // ALIGN * ALIGN for st in prog.storages}
    items = [(sid, layout.offsets[sid], sizes[sid]) for sid in layout.offsets if sid in access]

    def before(a, b):  # every access of a happens-before every access of b
        return all((desc[x] >> y) & 1 for x in access[a] for y in access[b])

    for i in range(len(items)):
        a, oa, sa = items[i]
        for j in range(i + 1, len(items)):
            b, ob, sb = items[j]
            if oa < ob + sb and ob < oa + sa:
                if not (before(a, b) or before(b, a)):
                    raise AssertionError(f"storages {a} and {b} overlap without a happens-before order")
