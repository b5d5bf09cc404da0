"""Lowering: reference implementation IR -> a plan of B200 kernel launches.

Input is the reference's ``StencilImplementation`` (stencilforge
``ir.py:328-351``: multistages, stages with compute extents, temporaries),
produced unchanged by ``analysis.lower`` (``analysis.py:538-549``).  Output is
a ``Plan``: an ordered list of kernel launches, each an instance of one of the
hand-written templates in ``csrc/templates/``:

``pfused``  PARALLEL stages of one interval fused into one streaming tile
            kernel (``gts_parallel.cuh``): inputs staged through shared
            memory, temporaries kept in registers, each api field crossing HBM
            once.  Hazard rules below decide where a PARALLEL multistage must
            be split.
``pstage``  one PARALLEL stage, one thread per point (the always-correct
            fallback; temporaries in the device arena).
``column``  a run of multistages with zero horizontal extent and no
            cross-column dependencies, containing at least one FORWARD or
            BACKWARD multistage: one thread per (i, j) column sweeping k with
            register k-caches (``gts_column.cuh``); the Thomas sweep of vadv.
``plane``   FORWARD/BACKWARD with horizontal dependencies: per level, per
            stage, one plane launch (the reference's own execution order,
            ``gen.py:343-360``).

Semantics follow the reference engines exactly (``debug.py:301-355``,
``vec.py:129-168``): PARALLEL stages commit over their whole slab before the
next stage starts; sequential multistages sweep level by level.  A fused
launch is only formed where that order is unobservable.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

from ._host import ir

Int3 = tuple[int, int, int]


# ---------------------------------------------------------------------------
# IR queries
# ---------------------------------------------------------------------------


def reads(stmt) -> list:
    """Every FieldAccess read by a statement (ir.py:559-566)."""
    return [e for e in ir.stmt_reads(stmt) if isinstance(e, ir.FieldAccess)]


def writes(stmt) -> set:
    return {w.field for w in ir.stmt_writes(stmt)}


def always_writes(stmt) -> set:
    """Fields assigned on every path through the statement."""
    if isinstance(stmt, ir.Assign):
        return {stmt.target.field}
    if isinstance(stmt, ir.If):
        then_w = set()
        for s in stmt.then_body:
            then_w |= always_writes(s)
        else_w = set()
        for s in stmt.else_body:
            else_w |= always_writes(s)
        return then_w & else_w
    return set()


def horizontal(off) -> bool:
    return off[0] != 0 or off[1] != 0


def zero_extent(stage) -> bool:
    e = stage.compute_extent
    return e.lo[0] == 0 and e.lo[1] == 0 and e.hi[0] == 0 and e.hi[1] == 0


# ---------------------------------------------------------------------------
# Plan
# ---------------------------------------------------------------------------


@dataclass
class StageRef:
    ms: int  # multistage index
    idx: int  # stage index within the multistage
    stage: object  # ir.Stage


@dataclass
class KernelPlan:
    kind: str  # "pfused" | "pstage" | "column" | "plane"
    stages: list  # StageRef, program order
    multistages: list = field(default_factory=list)  # column: ms indices
    interval: Optional[object] = None  # pfused / pstage: ir.Interval
    local_temps: tuple = ()  # pfused: temps living in registers only
    label: str = ""


@dataclass
class Plan:
    impl: object
    kernels: list
    global_temps: tuple  # temps that live in the device arena
    nan_fill_temps: tuple  # arena temps that may be read where unwritten

    def describe(self) -> list:
        return [f"{k.kind}:{k.label}" for k in self.kernels]


def _column_ok(ms) -> bool:
    return all(zero_extent(s) for s in ms.stages)


def _column_safe(mss) -> bool:
    """No read at a horizontal offset of any field written in the run."""
    w = set()
    for ms in mss:
        for st in ms.stages:
            w |= writes(st.body)
    for ms in mss:
        for st in ms.stages:
            for acc in reads(st.body):
                if acc.field in w and horizontal(acc.offset):
                    return False
    return True


def _fuse_parallel(stages: list, temp_names: set, fuse: bool) -> list:
    """Split one PARALLEL multistage into launch groups.

    A stage S joins the current group G (same interval) unless
    (a) S reads a field written in G anywhere but at its own point through
        a temporary with a single writer in G (temporaries are recomputed on
        the tile halo from the extent analysis, analysis.py:451-496), or
    (b) S writes an api field / temporary that G already read somewhere
        other than at the reading thread's own point, or that G wrote, or
        that G read from the arena (another tile could observe the update).
    Non-fusable stages run as single-stage launches.
    """
    groups: list = []
    cur: list = []

    def close():
        nonlocal cur
        if cur:
            groups.append(cur)
        cur = []

    for ref in stages:
        st = ref.stage
        if not fuse:
            close()
            cur = [ref]
            close()
            continue
        if cur and cur[0].stage.interval != st.interval:
            close()
        ok = True
        if cur:
            g_writes: dict = {}
            for r in cur:
                for f in writes(r.stage.body):
                    g_writes.setdefault(f, []).append(r)
            g_reads: list = []
            for r in cur:
                for acc in reads(r.stage.body):
                    g_reads.append((r, acc))
            for acc in reads(st.body):
                if acc.field not in g_writes:
                    continue
                if acc.field in temp_names:
                    if len(g_writes[acc.field]) != 1:
                        ok = False
                    elif acc.field in writes(st.body) and horizontal(acc.offset):
                        ok = False
                else:
                    if horizontal(acc.offset) or not zero_extent(st):
                        ok = False
                    if any(not zero_extent(w.stage) for w in g_writes[acc.field]):
                        ok = False
            for f in writes(st.body):
                if f in g_writes:
                    ok = False  # single writer per field per group
                for r, acc in g_reads:
                    if acc.field != f:
                        continue
                    if f in temp_names:
                        ok = False  # temp read from the arena, then overwritten
                    elif horizontal(acc.offset) or not zero_extent(r.stage):
                        ok = False
        if not ok:
            close()
        cur.append(ref)
    close()
    return groups


def build_plan(impl, options: Optional[dict] = None) -> Plan:
    opts = options or {}
    fuse = bool(opts.get("fuse_parallel", True))
    column = bool(opts.get("column", True))
    temp_names = {t.name for t in impl.temporaries}
    mss = list(impl.multistages)
    kernels: list = []
    i = 0
    while i < len(mss):
        # try a column run starting here
        j = i
        while j < len(mss) and _column_ok(mss[j]) and _column_safe(mss[i:j + 1]):
            j += 1
        run = mss[i:j]
        if run and any(ms.order != ir.PARALLEL for ms in run) and column:
            refs = [StageRef(m, s, st) for m in range(i, j) for s, st in enumerate(mss[m].stages)]
            kernels.append(KernelPlan("column", refs, multistages=list(range(i, j)),
                                      label=f"ms{i}-{j - 1}"))
            i = j
            continue
        ms = mss[i]
        refs = [StageRef(i, s, st) for s, st in enumerate(ms.stages)]
        if ms.order == ir.PARALLEL:
            for g in _fuse_parallel(refs, temp_names, fuse):
                if len(g) == 1 and not fuse:
                    kernels.append(KernelPlan("pstage", g, interval=g[0].stage.interval,
                                              label=f"ms{i}.s{g[0].idx}"))
                else:
                    kernels.append(KernelPlan("pfused", g, interval=g[0].stage.interval,
                                              label=f"ms{i}.s{g[0].idx}-{g[-1].idx}"))
        elif column and _column_ok(ms) and _column_safe([ms]):
            kernels.append(KernelPlan("column", refs, multistages=[i], label=f"ms{i}"))
        else:
            kernels.append(KernelPlan("plane", refs, multistages=[i], label=f"ms{i}"))
        i += 1

    # storage class of every temporary: registers when written and consumed
    # inside one pfused launch only, else the device arena
    writer_kernel: dict = {}
    reader_kernels: dict = {}
    for kidx, k in enumerate(kernels):
        for r in k.stages:
            for f in writes(r.stage.body):
                if f in temp_names:
                    writer_kernel.setdefault(f, set()).add(kidx)
            for acc in reads(r.stage.body):
                if acc.field in temp_names:
                    reader_kernels.setdefault(acc.field, set()).add(kidx)
    global_temps = []
    for t in impl.temporaries:
        wk = writer_kernel.get(t.name, set())
        rk = reader_kernels.get(t.name, set())
        local = (len(wk) == 1 and rk <= wk and kernels[next(iter(wk))].kind == "pfused")
        if local:
            kk = kernels[next(iter(wk))]
            kk.local_temps = tuple(sorted(set(kk.local_temps) | {t.name}))
        else:
            global_temps.append(t.name)
    # arena temporaries that some path may leave unwritten are NaN-filled per
    # call, like the reference engines' NaN-initialised temporaries
    # (debug.py:327-330, vec.py:143-145)
    nan_fill = []
    for t in global_temps:
        for k in kernels:
            for r in k.stages:
                if t in writes(r.stage.body) and t not in always_writes(r.stage.body):
                    nan_fill.append(t)
    return Plan(impl, kernels, tuple(global_temps), tuple(sorted(set(nan_fill))))
