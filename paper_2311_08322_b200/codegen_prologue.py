"""Prologue fusion: a PARALLEL stage group computed inside the column kernel.

A dycore-like program (``kernels/dycore.gts``) runs a horizontal PARALLEL
multistage (flux-limited diffusion: lap -> flx/fly -> uh) whose only product
is a temporary consumed at the reader's own point by the FORWARD sweep of a
following column run (the Thomas solve, ``d := uh``).  Executed as two
launches, uh makes a round trip through HBM (write + read, 16 B per point).

Fused, the column kernel's TMA producer streams the PARALLEL group's inputs
as halo'd boxes (the input's field extent from ``analysis.compute_extents``,
``analysis.py:451-496``) and each consumer thread evaluates the group at its
own (i, j, k) right before the forward recurrence consumes it.  Every stage
is evaluated at every horizontal offset the extent analysis requires of it
(``required_offsets``: lap at the 5-point cross for hdiff), as straight-line
code in program order -- the same values the reference's whole-slab order
produces (``vec.py:160-162``), so the result is bitwise identical.

Legality (``prologue_spec``): the group is one pfused launch of a PARALLEL
multistage over the full vertical interval; everything it writes is a
temporary; the temporaries it exports are read only by the forward sweep of
the next column run, at offset (0, 0, 0); its inputs are api fields the run
does not write, read at vertical offset 0.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from ._host import ir
from .codegen import c_float, emit_cond, emit_expr  # noqa: F401
from .lowering import always_writes, reads, writes

Off = tuple  # (di, dj)


@dataclass
class PrologueSpec:
    kplan: object  # the pfused KernelPlan
    stages: list  # ir.Stage, program order
    exports: list  # temporaries handed to the forward sweep (read there at (0,0,0))
    inputs: list  # api fields read by the group (streamed with halo boxes)
    extent: dict  # input -> (lo_i, hi_i, lo_j, hi_j) covering every read
    required: dict = field(default_factory=dict)  # temp -> sorted offsets it is evaluated at


def _full_interval(iv) -> bool:
    return iv.start.ref == ir.START and iv.start.offset == 0 and iv.end.ref == ir.END and iv.end.offset == 0


def prologue_spec(plan, kpf, kcol, dtypes: dict):
    impl = plan.impl
    if kpf.kind != "pfused" or kcol.kind != "column":
        return None
    if kpf.interval is None or not _full_interval(kpf.interval):
        return None
    api = {f.name for f in impl.api_fields}
    temps = {t.name for t in impl.temporaries}
    stages = [r.stage for r in kpf.stages]
    msf = impl.multistages[kcol.multistages[0]]
    if msf.order != ir.FORWARD:
        return None
    written = set()
    for st in stages:
        written |= writes(st.body)
    if written & api:
        return None
    # every temp of the group has a single writer, always written (no NaN
    # bookkeeping across the fused boundary)
    for st in stages:
        if writes(st.body) - always_writes(st.body):
            return None
    writers = {}
    for si, st in enumerate(stages):
        for f in writes(st.body):
            if f in writers:
                return None
            writers[f] = si
    # who reads the group's temporaries outside the group
    exports = set()
    for mi, ms in enumerate(impl.multistages):
        for st in ms.stages:
            if any(st is s for s in stages):
                continue
            for acc in reads(st.body):
                if acc.field in written:
                    if mi != kcol.multistages[0] or acc.offset != (0, 0, 0):
                        return None
                    exports.add(acc.field)
    if not exports:
        return None
    # run outputs must not feed back into the group
    run_writes = set()
    for mi in kcol.multistages:
        for st in impl.multistages[mi].stages:
            run_writes |= writes(st.body)
    inputs, ext = [], {}
    for st in stages:
        for acc in reads(st.body):
            if acc.offset[2] != 0:
                return None
            if acc.field in api:
                if acc.field in run_writes:
                    return None
                if acc.field not in inputs:
                    inputs.append(acc.field)
            elif acc.field not in written or acc.field not in temps:
                return None  # arena temporaries of earlier launches: not fused
    # offsets each temp is evaluated at: backward propagation from the exports
    req = {f: set() for f in written}
    for f in exports:
        req[f].add((0, 0))
    for si in range(len(stages) - 1, -1, -1):
        st = stages[si]
        outs = writes(st.body)
        offs = set()
        for f in outs:
            offs |= req[f]
        for acc in reads(st.body):
            if acc.field in written:
                for (oi, oj) in offs:
                    req[acc.field].add((oi + acc.offset[0], oj + acc.offset[1]))
    for si, st in enumerate(stages):
        for acc in reads(st.body):
            if acc.field in written and writers[acc.field] >= si:
                return None  # read before (or by) its writer
    for f in inputs:
        lo_i = lo_j = hi_i = hi_j = 0
        for st in stages:
            offs = set()
            for g in writes(st.body):
                offs |= req[g]
            for acc in reads(st.body):
                if acc.field == f:
                    for (oi, oj) in offs:
                        lo_i, hi_i = min(lo_i, oi + acc.offset[0]), max(hi_i, oi + acc.offset[0])
                        lo_j, hi_j = min(lo_j, oj + acc.offset[1]), max(hi_j, oj + acc.offset[1])
        fe = impl.field_extent(f)
        if lo_i < fe.lo[0] or lo_j < fe.lo[1] or hi_i > fe.hi[0] or hi_j > fe.hi[1]:
            return None  # outside the storage the runtime validated
        ext[f] = (lo_i, hi_i, lo_j, hi_j)
    return PrologueSpec(kpf, stages, sorted(exports), inputs, ext,
                        {f: sorted(v) for f, v in req.items()})


def materialized(ps: PrologueSpec) -> dict:
    """Temporaries worth computing ONCE per tile point into shared memory
    instead of per thread at every required offset: those evaluated at >= 3
    offsets (hdiff's ``lap``: the 5-point cross) whose stage reads only the
    group's inputs.  Returns temp -> (lo_i, hi_i, lo_j, hi_j) of the offsets."""
    out = {}
    for st in ps.stages:
        outs = writes(st.body)
        if len(outs) != 1:
            continue
        t = next(iter(outs))
        offs = ps.required.get(t, [])
        if len(offs) < 3:
            continue
        if any(a.field in ps.required for a in reads(st.body)):
            continue
        out[t] = (min(o[0] for o in offs), max(o[0] for o in offs),
                  min(o[1] for o in offs), max(o[1] for o in offs))
    return out


def emit_stage_value(ps: PrologueSpec, name: str, read_input, ctype: dict, out: list, indent: str,
                     target: str) -> None:
    """The stage that writes temp ``name``, evaluated at the point whose
    inputs ``read_input(input, di, dj)`` spells, assigned to C variable
    ``target`` (narrowed to the temp's type)."""
    for st in ps.stages:
        if name in writes(st.body):
            ctx = _PointCtx(ps, read_input, 0, 0)
            ctx.rename = {name: target}
            _emit_stmt(st.body, ctx, ctype, out, indent)
            return
    raise KeyError(name)


def _vn(name: str, oi: int, oj: int) -> str:
    def s(x):
        return f"m{-x}" if x < 0 else str(x)
    return f"pt_{name}_{s(oi)}_{s(oj)}"


class _PointCtx:
    """Reads of one stage evaluated at horizontal offset (oi, oj); ``oj`` may
    be a C expression (the per-lane column of a warp-edge evaluation, which
    reads only the group's inputs)."""

    def __init__(self, ps: PrologueSpec, read_input, oi: int, oj, mat_read=None):
        self.ps, self.read_input, self.oi, self.oj = ps, read_input, oi, oj
        self.pool = None
        self.rename = {}
        self.mat_read = mat_read or {}

    def _col(self, dj):
        if isinstance(self.oj, str):
            return f"({self.oj}{dj:+d})" if dj else self.oj
        return self.oj + dj

    def read(self, name, off):
        di, dj, _ = off
        if name in self.mat_read:
            return f"((double){self.mat_read[name](self.oi + di, self._col(dj))})"
        if name in self.ps.required:
            return _vn(name, self.oi + di, self._col(dj))
        return f"((double){self.read_input(name, self.oi + di, self._col(dj))})"

    def target(self, name):
        return self.rename.get(name) or _vn(name, self.oi, self.oj)


def _emit_stmt(stmt, ctx, ctype: dict, out: list, indent: str) -> None:
    if isinstance(stmt, ir.Assign):
        name = stmt.target.field
        value = emit_expr(stmt.value, ctx)
        out.append(f"{indent}{ctx.target(name)} = (double)({ctype[name]})({value});")
        return
    if isinstance(stmt, ir.If):
        out.append(f"{indent}if ({emit_cond(stmt.cond, ctx)}) {{")
        for s in stmt.then_body:
            _emit_stmt(s, ctx, ctype, out, indent + "  ")
        if stmt.else_body:
            out.append(f"{indent}}} else {{")
            for s in stmt.else_body:
                _emit_stmt(s, ctx, ctype, out, indent + "  ")
        out.append(f"{indent}}}")
        return
    raise TypeError(type(stmt).__name__)


def lane_shuffled(ps: PrologueSpec, st) -> list:
    """Rows ``oi`` at which stage ``st`` is needed at (oi, -1), (oi, 0) AND
    (oi, +1) and reads only the group's inputs (hdiff's ``lap`` on the 5-point
    cross: oi = 0).  With one warp lane per consecutive j column, lane l's
    value at (oi, -1) is lane l-1's at (oi, 0) -- the same instructions on the
    same inputs, so bitwise equal -- and only the two warp-edge lanes need a
    real evaluation: one per-lane evaluation at column ``ex_`` (-1 on lane 0,
    +1 elsewhere) replaces two."""
    if any(a.field in ps.required for a in reads(st.body)):
        return []
    offs = set()
    for g in writes(st.body):
        offs |= set(ps.required[g])
    return sorted(oi for (oi, oj) in offs if oj == 0 and (oi, -1) in offs and (oi, 1) in offs)


def emit_point(ps: PrologueSpec, read_input, ctype: dict, out: list, indent: str,
               mat_read=None, lane: str = None) -> dict:
    """Straight-line evaluation of the group at the thread's own point.
    ``read_input(name, di, dj)`` spells a read of an input at a horizontal
    offset (``dj`` may be a C expression); ``mat_read`` {temp: f(di, dj)}
    spells reads of temporaries already materialized in shared memory (their
    stages are skipped).  ``lane``: the C lane index when the warp's 32 lanes
    are 32 consecutive j columns -- enables the neighbour-lane shuffles of
    ``lane_shuffled``.  Returns {export: C variable holding its value}."""
    mat_read = mat_read or {}
    for f, offs in sorted(ps.required.items()):
        if f in mat_read:
            continue
        for (oi, oj) in offs:
            out.append(f"{indent}double {_vn(f, oi, oj)};")
    edge_decl = False
    for st in ps.stages:
        if writes(st.body) & set(mat_read):
            continue
        offs = set()
        for g in writes(st.body):
            offs |= set(ps.required[g])
        shfl = lane_shuffled(ps, st) if lane is not None else []
        for (oi, oj) in sorted(offs):
            if oi in shfl and oj in (-1, 1):
                continue
            _emit_stmt(st.body, _PointCtx(ps, read_input, oi, oj, mat_read), ctype, out, indent)
        for oi in shfl:
            if not edge_decl:
                out.append(f"{indent}const int ex_ = ({lane}) == 0 ? -1 : 1;  // warp-edge column")
                edge_decl = True
            ctx = _PointCtx(ps, read_input, oi, "ex_", mat_read)
            ctx.rename = {g: f"pe_{g}_{_vn(g, oi, 0)[3:]}" for g in writes(st.body)}
            for g in writes(st.body):
                out.append(f"{indent}double {ctx.rename[g]};")
            _emit_stmt(st.body, ctx, ctype, out, indent)
            for g in writes(st.body):
                own, e = _vn(g, oi, 0), ctx.rename[g]
                # every lane executes both shuffles (full-mask convergence);
                # only the selection depends on the lane
                out.append(f"{indent}const double su_{own} = __shfl_up_sync(0xffffffffu, {own}, 1);")
                out.append(f"{indent}const double sd_{own} = __shfl_down_sync(0xffffffffu, {own}, 1);")
                out.append(f"{indent}{_vn(g, oi, -1)} = ({lane}) == 0 ? {e} : su_{own};")
                out.append(f"{indent}{_vn(g, oi, 1)} = ({lane}) == 31 ? {e} : sd_{own};")
    return {f: _vn(f, 0, 0) for f in ps.exports}


__all__ = ["PrologueSpec", "prologue_spec", "emit_point", "materialized", "emit_stage_value", "c_float"]
