"""Code generation: lowering ``Plan`` -> one CUDA translation unit per stencil.

The TU instantiates the hand-written templates in ``csrc/templates/`` with
stage bodies emitted from the reference IR, and exports the drop-in entry

    int gts_run_<name>_<digest8>(int64 ni, int64 nj, int64 nk,
                                 {T* base, int64 s_i, s_j, s_k, o_i, o_j, o_k}
                                     per api field in declaration order,
                                 double per api scalar in declaration order,
                                 void* stream)

i.e. the reference gen entry ABI (stencilforge ``backends/gen.py:5-14,
269-284``, ``pkg/README.md:142-156``) with device pointers, a trailing CUDA
stream and an ``int`` status (0 = ok, else a cudaError_t or a GTS_ERR_* code).
Scalars are always passed as double, following the debug/vec engines
(``runtime.py:113``) rather than gen's float narrowing of f32 scalars.

Numerics contract: f64 arithmetic in the IR's association
order, f32 operands widened on read and narrowed on every store (register
temporaries included), NaN-propagating min/max (``gen.py:257-266``), IEEE
division (nvcc default ``-prec-div=true``), no FMA contraction
(``--fmad=false``, mirroring gen's ``-ffp-contract=off``, ``gen.py:64-67``),
exact hex literals (``gen.py:111-116``).
"""

from __future__ import annotations

import math
import re
import threading
from typing import Optional

from ._host import ir
from .lowering import Plan, always_writes, reads, writes

GTS_ERR_K_MIN = 1001
GTS_ERR_ALLOC = 1002
GTS_ERR_UNSUPPORTED = 1003

_BUILTIN_CUDA = {
    "abs": "fabs",
    "min": "gts_min",
    "max": "gts_max",
    "sqrt": "sqrt",
    "exp": "exp",
    "log": "log",
    "pow": "pow",
    "floor": "floor",
    "ceil": "ceil",
}
_BINOP = {"and": "&&", "or": "||"}


def c_float(value: float) -> str:
    if math.isnan(value):
        return "GTS_NAN"
    if math.isinf(value):
        return "(-GTS_INF)" if value < 0 else "GTS_INF"
    return float(value).hex()


def entry_name(impl, fp) -> str:
    """Same mangling as the reference gen engine (gen.py:184-185)."""
    return f"gts_run_{impl.name}_{fp.short}"


class DivPool:
    """Shared-reciprocal division (``gts_rcp`` / ``gts_div`` in
    gts_common.cuh): every distinct denominator is refined once per scope and
    reused by later quotients over the same value (vadv divides cp's and
    dp's numerators by the same ``b - a*cp[k-1]``, vadv.gts:10-12).  Results
    stay bitwise the IEEE quotient."""

    def __init__(self, mode: str = "branch"):
        self.map: dict = {}
        self.pending: list = []
        self.depth = 0
        self.n = 0
        # "branch": gts_div (exact, per-quotient slow-path branch)
        # "fast":   gts_div_fast, sets the kernel's bad_ flag (replayed exactly)
        # "exact":  plain IEEE division
        self.mode = mode

    def rcp(self, den: str) -> str:
        if den in self.map:
            return self.map[den]
        var = f"rcp{self.n}"
        self.n += 1
        self.pending.append(f"const GtsRcp {var} = gts_rcp({den});")
        if self.depth == 0:
            self.map[den] = var
        return var

    def flush(self, indent: str, out: list) -> None:
        for ln in self.pending:
            out.append(indent + ln)
        self.pending = []

    def invalidate(self, field: str) -> None:
        keys = [k for k in self.map if f"cur_{field}" in k or f"p.f_{field}," in k]
        for k in keys:
            del self.map[k]


class _Ctx:
    """How a field access at an offset is spelled inside one kernel."""

    pool = None  # optional DivPool

    def __init__(self, dtypes: dict):
        self.dtypes = dtypes  # name -> "f32" | "f64"

    def read(self, name: str, off) -> str:
        raise NotImplementedError


class _MemCtx(_Ctx):
    """Every access goes to device memory at (i, j, k) + offset."""

    def __init__(self, dtypes: dict, kvar: str = "k"):
        super().__init__(dtypes)
        self.kvar = kvar

    def addr(self, name: str, off) -> str:
        di, dj, dk = off
        ii = f"(i{di:+d})" if di else "i"
        jj = f"(j{dj:+d})" if dj else "j"
        kk = f"({self.kvar}{dk:+d})" if dk else self.kvar
        return f"GTS_AT(p.f_{name}, {ii}, {jj}, {kk})"

    def read(self, name: str, off) -> str:
        return f"((double){self.addr(name, off)})"


def emit_expr(e, ctx: _Ctx) -> str:
    if isinstance(e, ir.Literal):
        return c_float(float(e.value))
    if isinstance(e, ir.ScalarRef):
        return f"p.sc_{e.name}"
    if isinstance(e, ir.FieldAccess):
        return ctx.read(e.field, e.offset)
    if isinstance(e, ir.UnaryOp):
        inner = emit_expr(e.operand, ctx)
        return f"(!{inner})" if e.op == "not" else f"(-{inner})"
    if isinstance(e, ir.BinaryOp):
        if e.op == "/" and ctx.pool is not None and ctx.pool.mode != "exact":
            num = emit_expr(e.left, ctx)
            rcp = ctx.pool.rcp(emit_expr(e.right, ctx))
            if ctx.pool.mode == "fast":
                return f"gts_div_fast({num}, {rcp}, bad_)"
            return f"gts_div({num}, {rcp})"
        op = _BINOP.get(e.op, e.op)
        return f"({emit_expr(e.left, ctx)} {op} {emit_expr(e.right, ctx)})"
    if isinstance(e, ir.BuiltinCall):
        args = ", ".join(emit_expr(a, ctx) for a in e.args)
        return f"{_BUILTIN_CUDA[e.name]}({args})"
    raise TypeError(f"cannot generate code for {type(e).__name__}")


# ---------------------------------------------------------------------------
# binary32-exact emission (f32 storage).  The reference evaluates f32 programs
# in binary64 and narrows every store; each narrowing and each
# widening is a 64-bit conversion, which is what bounds an f32 stencil on B200.
# Three rewrites give the same bits with binary32 instructions:
#  * a value that is exactly a binary32 number (an f32 field or temporary, a
#    literal representable in binary32, its negation) is used as a float;
#  * round_to_f32(x op y), op one of + - * / on binary32-exact x, y and
#    evaluated in binary64, equals the binary32 operation x op y: binary64
#    carries 53 >= 2*24 + 2 significand bits and a wider exponent range, so
#    the double rounding is innocuous (Figueroa, "When is double rounding
#    innocuous?", SIGNUM 1995; the asm.js Math.fround argument);
#  * comparisons of two binary32-exact values compare the floats (widening
#    is exact and monotone), and the flux-limiter sign test
#    (x0 - y0) * (x1 - y1) > 0 (or < 0) becomes float comparisons: a nonzero
#    finite difference of binary32 values lies in [2^-149, 2^129], so the
#    binary64 product neither underflows nor overflows and its sign is the
#    product of the signs; NaN / inf * 0 cases make both forms false.
# Contexts opt in with read_f32(); binary64 programs never take these paths.
# ---------------------------------------------------------------------------
_ARITH = ("+", "-", "*", "/")
_CMP = ("<", ">", "<=", ">=", "==", "!=")


def _f32_exact_literal(value) -> bool:
    import struct

    v = float(value)
    if not math.isfinite(v):
        return False
    try:
        return struct.unpack("f", struct.pack("f", v))[0] == v
    except OverflowError:
        return False


def emit_f32(e, ctx) -> Optional[str]:
    """Float spelling of ``e`` when its value is exactly a binary32 number."""
    rd = getattr(ctx, "read_f32", None)
    if rd is None:
        return None
    if isinstance(e, ir.Literal) and not isinstance(e.value, bool) and _f32_exact_literal(e.value):
        return float(e.value).hex() + "f"
    if isinstance(e, ir.FieldAccess):
        return rd(e.field, e.offset)
    if isinstance(e, ir.UnaryOp) and e.op == "-":
        inner = emit_f32(e.operand, ctx)
        return None if inner is None else f"(-{inner})"
    return None


def emit_f32_rounded(e, ctx) -> Optional[str]:
    """Float spelling of round_to_binary32(e evaluated in binary64), when one
    binary32 instruction provably gives it (see above); else None."""
    v = emit_f32(e, ctx)
    if v is not None:
        return v
    if isinstance(e, ir.BinaryOp) and e.op in _ARITH:
        a, b = emit_f32(e.left, ctx), emit_f32(e.right, ctx)
        if a is not None and b is not None:
            return f"({a} {e.op} {b})"
    return None


def _sign_parts(e, ctx):
    """(positive, negative) float conditions of a binary64 value that is one
    +/- of two binary32-exact operands, or binary32-exact itself."""
    v = emit_f32(e, ctx)
    if v is not None:
        return f"({v} > 0.0f)", f"({v} < 0.0f)"
    if isinstance(e, ir.BinaryOp) and e.op in ("-", "+"):
        a, b = emit_f32(e.left, ctx), emit_f32(e.right, ctx)
        if a is not None and b is not None:
            if e.op == "+":
                b = f"(-{b})"
            return f"({a} > {b})", f"({a} < {b})"
    return None


def emit_cond(e, ctx) -> str:
    """A condition, with the binary32 rewrites where they are exact.  (A
    multiply-free sign test for binary64 products -- integer checks on the
    operands' exponents and signs with the multiply on a rare path -- measured
    slower on B200: ptxas predicates the guarded multiply, so it still issues;
    hdiff 17.0 -> 19.9 us, dycore 176 -> 192 us / step.)"""
    if isinstance(e, ir.BinaryOp) and e.op in ("and", "or"):
        op = _BINOP[e.op]
        return f"({emit_cond(e.left, ctx)} {op} {emit_cond(e.right, ctx)})"
    if getattr(ctx, "read_f32", None) is not None and isinstance(e, ir.BinaryOp):
        if e.op in _CMP:
            a, b = emit_f32(e.left, ctx), emit_f32(e.right, ctx)
            if a is not None and b is not None:
                return f"({a} {e.op} {b})"
            if e.op in ("<", ">"):
                prod, zero_right = None, None
                if isinstance(e.right, ir.Literal) and float(e.right.value) == 0.0:
                    prod, zero_right = e.left, True
                elif isinstance(e.left, ir.Literal) and float(e.left.value) == 0.0:
                    prod, zero_right = e.right, False
                if isinstance(prod, ir.BinaryOp) and prod.op == "*":
                    s1, s2 = _sign_parts(prod.left, ctx), _sign_parts(prod.right, ctx)
                    if s1 is not None and s2 is not None:
                        want_pos = (e.op == ">") == zero_right  # P > 0  or  0 < P
                        if want_pos:
                            return f"(({s1[0]} && {s2[0]}) || ({s1[1]} && {s2[1]}))"
                        return f"(({s1[0]} && {s2[1]}) || ({s1[1]} && {s2[0]}))"
    return emit_expr(e, ctx)


# ---------------------------------------------------------------------------
# Statement emission for memory-backed kernels (pstage / plane / column)
# ---------------------------------------------------------------------------


def _store_mem(name: str, value: str, ctx: _MemCtx, ctype: dict) -> str:
    return f"{ctx.addr(name, (0, 0, 0))} = ({ctype[name]})({value});"


def emit_stmt_mem(stmt, ctx: _MemCtx, ctype: dict, indent: str, out: list,
                  on_write=None) -> None:
    if ctx.pool is None:
        ctx.pool = DivPool()
    pool = ctx.pool
    if isinstance(stmt, ir.Assign):
        name = stmt.target.field
        value = emit_expr(stmt.value, ctx)
        pool.flush(indent, out)
        out.append(f"{indent}{{ const double v_ = {value};")
        out.append(f"{indent}  {_store_mem(name, 'v_', ctx, ctype)}")
        if on_write is not None:
            extra = on_write(name, "v_")
            if extra:
                out.append(f"{indent}  {extra}")
        out.append(f"{indent}}}")
        pool.invalidate(name)
        return
    if isinstance(stmt, ir.If):
        cond = emit_cond(stmt.cond, ctx)
        pool.flush(indent, out)
        out.append(f"{indent}if ({cond}) {{")
        pool.depth += 1
        for s in stmt.then_body:
            emit_stmt_mem(s, ctx, ctype, indent + "  ", out, on_write)
        if stmt.else_body:
            out.append(f"{indent}}} else {{")
            for s in stmt.else_body:
                emit_stmt_mem(s, ctx, ctype, indent + "  ", out, on_write)
        pool.depth -= 1
        out.append(f"{indent}}}")
        return
    raise TypeError(f"cannot generate code for {type(stmt).__name__}")


# ---------------------------------------------------------------------------
# Column kernel (k-caches)
# ---------------------------------------------------------------------------


class _ColumnCtx(_MemCtx):
    """Memory accesses, except fields with an active k-cache: reads at the
    current level use ``cur_<f>``; reads ``s`` levels behind in iteration
    order use ``prev<s>_<f>``."""

    def __init__(self, dtypes, direction: int, cached: dict):
        super().__init__(dtypes)
        self.direction = direction  # +1 FORWARD/PARALLEL, -1 BACKWARD
        self.cached = cached  # name -> depth (levels behind kept)

    def read(self, name, off):
        if name in self.cached and not (off[0] or off[1]):
            s = -off[2] * self.direction
            if off[2] == 0:
                return f"cur_{name}"
            if 1 <= s <= self.cached[name]:
                return f"prev{s}_{name}"
        return super().read(name, off)


def _bound(b) -> str:
    return f"{b.offset}" if b.ref == ir.START else f"(nk + {b.offset})"


def _column_kernel(kname: str, plan: Plan, kplan, ctype: dict, dtypes: dict) -> list:
    impl = plan.impl
    out: list = []
    w = out.append
    w(f"__global__ void __launch_bounds__(GTS_COL_THREADS) {kname}(const __grid_constant__ GtsParams p) {{")
    w("  const int j = blockIdx.x * GTS_COL_TJ + (threadIdx.x % GTS_COL_TJ);")
    w("  const int i = blockIdx.y * (GTS_COL_THREADS / GTS_COL_TJ) + (threadIdx.x / GTS_COL_TJ);")
    w("  if (i >= p.ni || j >= p.nj) return;")
    w("  const int nk = p.nk;")
    for m in kplan.multistages:
        ms = impl.multistages[m]
        direction = -1 if ms.order == ir.BACKWARD else 1
        ms_writes = set()
        for st in ms.stages:
            ms_writes |= writes(st.body)
        # k-cache depth per written field read behind the sweep
        cached: dict = {}
        if ms.order != ir.PARALLEL:
            for st in ms.stages:
                for acc in reads(st.body):
                    if acc.field in ms_writes and not (acc.offset[0] or acc.offset[1]) and acc.offset[2]:
                        s = -acc.offset[2] * direction
                        if s > 0:
                            cached[acc.field] = max(cached.get(acc.field, 0), s)
        w(f"  {{ // multistage {m}: {ms.order}")
        for f, depth in sorted(cached.items()):
            for s in range(1, depth + 1):
                w(f"    double prev{s}_{f} = GTS_NAN;")
        ctx = _ColumnCtx(dtypes, direction, cached)
        for interval, stages in _interval_groups(ms):
            w("    {")
            w(f"      const int k0 = {_bound(interval.start)}, k1 = {_bound(interval.end)};")
            w("      if (k0 < k1) {")
            # initialise the k-cache from memory for the levels behind the first
            group_reads_behind: dict = {}
            for st in stages:
                for acc in reads(st.body):
                    if acc.field in cached and not (acc.offset[0] or acc.offset[1]):
                        s = -acc.offset[2] * direction
                        if s > 0:
                            group_reads_behind[acc.field] = max(group_reads_behind.get(acc.field, 0), s)
            kfirst = "k0" if direction > 0 else "(k1 - 1)"
            for f, depth in sorted(group_reads_behind.items()):
                for s in range(1, depth + 1):
                    kk = f"({kfirst} - {s})" if direction > 0 else f"({kfirst} + {s})"
                    w(f"        prev{s}_{f} = ((double)GTS_AT(p.f_{f}, i, j, {kk}));")
            if direction > 0:
                w("        for (int k = k0; k < k1; ++k) {")
            else:
                w("        for (int k = k1 - 1; k >= k0; --k) {")
            # current-level registers for cached fields
            for f in sorted(cached):
                need_load = True
                for st in stages:
                    touched_read = any(acc.field == f and acc.offset == (0, 0, 0) for acc in reads(st.body))
                    if touched_read:
                        break
                    if f in always_writes(st.body) and isinstance(st.body, ir.Assign):
                        need_load = False
                        break
                    if f in writes(st.body):
                        break
                if need_load:
                    w(f"          double cur_{f} = ((double)GTS_AT(p.f_{f}, i, j, k));")
                else:
                    w(f"          double cur_{f};")

            def on_write(name, v):
                if name in cached:
                    return f"cur_{name} = (double)({ctype[name]})({v});"
                return ""

            ctx.pool = DivPool()
            for st in stages:
                emit_stmt_mem(st.body, ctx, ctype, "          ", out, on_write)
            for f, depth in sorted(cached.items()):
                for s in range(depth, 1, -1):
                    w(f"          prev{s}_{f} = prev{s - 1}_{f};")
                w(f"          prev1_{f} = cur_{f};")
            w("        }")
            w("      }")
            w("    }")
        w("  }")
    w("}")
    return out


def _interval_groups(ms) -> list:
    """backends/common.py:38-46."""
    groups: list = []
    for stage in ms.stages:
        if groups and groups[-1][0] == stage.interval:
            groups[-1][1].append(stage)
        else:
            groups.append((stage.interval, [stage]))
    return groups


# ---------------------------------------------------------------------------
# Point kernels (pstage / plane)
# ---------------------------------------------------------------------------


def _point_kernel(kname: str, stage, ctype: dict, dtypes: dict) -> list:
    out: list = []
    w = out.append
    w(f"__global__ void __launch_bounds__(256) {kname}(const __grid_constant__ GtsParams p, "
      "int i0, int i1, int j0, int j1, int kbase) {")
    w("  const int j = j0 + blockIdx.x * 32 + (threadIdx.x & 31);")
    w("  const int i = i0 + blockIdx.y * 8 + (threadIdx.x >> 5);")
    w("  const int k = kbase + blockIdx.z;")
    w("  if (i >= i1 || j >= j1) return;")
    emit_stmt_mem(stage.body, _MemCtx(dtypes), ctype, "  ", out)
    w("}")
    return out


# ---------------------------------------------------------------------------
# Translation unit
# ---------------------------------------------------------------------------


_GEN_LOCK = threading.Lock()


def generate_source(plan: Plan, fp, options: Optional[dict] = None) -> str:
    """One CUDA translation unit for ``plan``.  The template emitters keep
    their geometry in module state while they run (codegen_parallel.configure
    and friends), so concurrent callers are serialised."""
    with _GEN_LOCK:
        return _generate_source(plan, fp, options)


def frame_tile_name(impl, fp) -> str:
    """Exported query of the frame variant's tile (rows << 16 | columns): the
    interior launch of a decomposed step covers exactly the frame launch's
    inner tile rectangle, so no point is computed twice."""
    return "gts_frametile_" + entry_name(impl, fp)[len("gts_run_"):]


def frame_setter_name(impl, fp) -> str:
    """Exported request for a frame launch (decomp.DecomposedStep): the
    calling thread's next launch computes only the tiles that touch the band
    of width (hi, hj) along the domain's sides."""
    return "gts_frame_" + entry_name(impl, fp)[len("gts_run_"):]


def written_api_fields(impl) -> list:
    api = [f.name for f in impl.api_fields]
    w = set()
    for ms in impl.multistages:
        for st in ms.stages:
            w |= writes(st.body)
    return [n for n in api if n in w]


def mirror_setter_name(impl, fp) -> str:
    """Exported setter of the halo-mirror boxes (gen_options ``mirror``)."""
    return "gts_mirror_" + entry_name(impl, fp)[len("gts_run_"):]


def _mirror_field(plan: Plan, opts: dict):
    """gen_options ``mirror``: the api output field whose stores the producing
    kernel also sends into neighbour halos (decomp.PeerFusedStep).  Only a
    field written by exactly one launch can be mirrored: a TMEM column kernel
    or a fused PARALLEL tile kernel (both store it once per point from
    registers; their launches refuse to fall back to templates without the
    mirror stores)."""
    m = opts.get("mirror")
    if not m:
        return None
    if m not in {f.name for f in plan.impl.api_fields}:
        raise ValueError(f"gen_options mirror: '{m}' is not an api field")
    writers = [k for k in plan.kernels if any(m in writes(r.stage.body) for r in k.stages)]
    if len(writers) != 1 or writers[0].kind not in ("column", "pfused"):
        raise ValueError(f"gen_options mirror: '{m}' must be written by exactly one column or fused "
                         f"PARALLEL kernel (plan {' '.join(plan.describe())})")
    return m


def _generate_source(plan: Plan, fp, options: Optional[dict] = None) -> str:
    impl = plan.impl
    from . import codegen_column, codegen_parallel  # template instantiations

    opts = options or {}

    ct = {ir.F32: "float", ir.F64: "double"}
    dtypes = {f.name: f.dtype for f in impl.api_fields}
    dtypes.update({t.name: t.dtype for t in impl.temporaries})
    ctype = {n: ct[d] for n, d in dtypes.items()}
    temps = {t.name: t for t in impl.temporaries}

    out: list = []
    w = out.append
    w("// generated by paper_2311_08322_b200; do not edit")
    w(f"// stencil: {impl.name}  fingerprint: {fp.digest}")
    w(f"// plan: {' '.join(plan.describe())}")
    w('#include "gts_common.cuh"')
    w('#include "gts_sm100.cuh"')
    w("")
    # temporaries with device storage: the plan's arena temporaries, plus the
    # register-only temporaries of fused launches (used only by their
    # per-stage fallback when the fields are not TMA-compatible)
    local_of = {}
    for kidx, k in enumerate(plan.kernels):
        if k.kind == "pfused":
            for t in k.local_temps:
                local_of[t] = kidx
    arena_temps = list(plan.global_temps) + sorted(local_of)
    mirror = _mirror_field(plan, opts)
    w("struct GtsParams {")
    w("  int ni, nj, nk;")
    for f in impl.api_fields:
        w(f"  GtsField<{ctype[f.name]}> f_{f.name};")
        w(f"  int tsh_{f.name}_i, tsh_{f.name}_j, tsh_{f.name}_k;")
    for t in arena_temps:
        w(f"  GtsField<{ctype[t]}> f_{t};")
    for s in impl.api_scalars:
        w(f"  double sc_{s.name};")
    if mirror:
        w(f"  GtsMirror<{ctype[mirror]}> mir;")
    w("};")
    w("")
    if mirror:
        # host-side mirror boxes, set by gts_mirror_<name>_<digest8> for the
        # calling thread's NEXT launch and consumed by it (copied into that
        # launch's parameters, so a CUDA graph captures the boxes set for the
        # captured launch; no box outlives the launch it was set for)
        w(f"static thread_local GtsMirror<{ctype[mirror]}> g_mirror;")
        w('extern "C" __attribute__((visibility("default")))')
        w(f"int {mirror_setter_name(impl, fp)}(int n, const int64_t* desc) {{")
        w(f"  if (n < 0 || n > 8) return {GTS_ERR_UNSUPPORTED};")
        w("  g_mirror.n = n;")
        w("  for (int d = 0; d < n; ++d) {")
        w("    const int64_t* q = desc + 8 * d;")
        w("    g_mirror.i0[d] = (int)q[0]; g_mirror.i1[d] = (int)q[1]; g_mirror.j0[d] = (int)q[2]; g_mirror.j1[d] = (int)q[3];")
        w(f"    g_mirror.base[d] = ({ctype[mirror]}*)(intptr_t)q[4];")
        w("    g_mirror.si[d] = q[5]; g_mirror.sj[d] = q[6]; g_mirror.sk[d] = q[7];")
        w("  }")
        w("  return 0;")
        w("}")
        w("")

    # frame launches (decomp.DecomposedStep): a single fused PARALLEL kernel
    # whose re-execution on a point is idempotent (no api field both read and
    # written), so frame tiles may recompute points the interior launch wrote
    api_reads = {a.field for ms in impl.multistages for st in ms.stages for a in reads(st.body)}
    api_written = set(written_api_fields(impl))
    frame_ok = (len(plan.kernels) == 1 and plan.kernels[0].kind == "pfused"
                and not (api_reads & api_written) and opts.get("pf_frame_variant", True))
    if frame_ok:
        # per side: bands of width ilo / ihi / jlo / jhi along the low-i,
        # high-i, low-j, high-j sides (0: no band, e.g. no neighbour there)
        w("static thread_local int g_frame_ilo = -1, g_frame_ihi = -1, g_frame_jlo = -1, g_frame_jhi = -1;")
        w('extern "C" __attribute__((visibility("default")))')
        w(f"int {frame_setter_name(impl, fp)}(int ilo, int ihi, int jlo, int jhi) {{")
        w("  if (ilo < 0 || ihi < 0 || jlo < 0 || jhi < 0) return %d;" % GTS_ERR_UNSUPPORTED)
        w("  g_frame_ilo = ilo; g_frame_ihi = ihi; g_frame_jlo = jlo; g_frame_jhi = jhi;  // the calling thread's NEXT launch only")
        w("  return 0;")
        w("}")
        w("")

    launches: list = []  # host-side launch code lines
    prelude: list = []  # host-side lines before the arena is sized
    fused_ok: dict = {}  # kernel index -> C flag name

    def pstage_launch(kname, st):
        e = st.compute_extent
        return [
            "  {",
            f"    const int k0 = {_bound(st.interval.start)}, k1 = {_bound(st.interval.end)};",
            f"    const int i0 = {e.lo[0]}, i1 = (int)ni + {e.hi[0]};",
            f"    const int j0 = {e.lo[1]}, j1 = (int)nj + {e.hi[1]};",
            "    if (k0 < k1 && i0 < i1 && j0 < j1) {",
            "      for (int kb = k0; kb < k1; kb += 65535) {",
            "        dim3 grid((unsigned)((j1 - j0 + 31) / 32), (unsigned)((i1 - i0 + 7) / 8),"
            " (unsigned)((k1 - kb) < 65535 ? (k1 - kb) : 65535));",
            f"        {kname}<<<grid, 256, 0, st>>>(p, i0, i1, j0, j1, kb);",
            "      }",
            "    }",
            "  }",
        ]

    from . import codegen_prologue

    skip = set()
    for kidx, k in enumerate(plan.kernels):
        if kidx in skip:
            continue
        kname = f"gts_k{kidx}_{k.kind}"
        # a pfused group whose only product is consumed at the reader's own
        # point by the next column run's forward sweep: fused into the TMEM
        # column kernel as its prologue (codegen_prologue), with the two-launch
        # form kept as the run-time fallback
        fused_col = None
        nxt = plan.kernels[kidx + 1] if kidx + 1 < len(plan.kernels) else None
        if (k.kind == "pfused" and nxt is not None and nxt.kind == "column"
                and opts.get("tmem", True) and opts.get("fuse_prologue", True)):
            pro = codegen_prologue.prologue_spec(plan, k, nxt, dtypes)
            if pro is not None:
                sp_f = codegen_column.spec(plan, nxt, dtypes, pro)
                if sp_f is not None:
                    fused_col = sp_f
        if k.kind == "pfused":
            saved_launches = launches
            if fused_col is not None:
                launches = []
            res = resL = resT = resF = None
            if opts.get("tma", True):
                res = codegen_parallel.emit(kname, plan, k, ctype, dtypes, opts)
                # binary64 groups: extra geometries for large and for tiny domains,
                # chosen at launch (codegen_parallel.LARGE / TINY)
                if (res is not None and codegen_parallel.last_esize() == 8 and "pf_nw" not in opts
                        and "pf_ri" not in opts and opts.get("pf_dual", True)):
                    resL = codegen_parallel.emit(kname + "L", plan, k, ctype, dtypes,
                                                 {**opts, **codegen_parallel.LARGE})
                    resT = codegen_parallel.emit(kname + "T", plan, k, ctype, dtypes,
                                                 {**opts, **codegen_parallel.TINY})
                # the frame launch of a decomposed step (decomp.DecomposedStep)
                if res is not None and frame_ok:
                    resF = codegen_parallel.emit(kname + "F", plan, k, ctype, dtypes,
                                                 {**opts, **codegen_parallel.FRAME_GEOMETRY})
            fb = []
            for r in k.stages:
                nm = f"{kname}_s{r.idx}"
                out.extend(_point_kernel(nm, r.stage, ctype, dtypes))
                fb += pstage_launch(nm, r.stage)
            if mirror and any(mirror in writes(r.stage.body) for r in k.stages):
                # the mirrored field's stores exist only in the tile template
                if res is None:
                    raise ValueError(f"gen_options mirror: '{mirror}' needs the fused PARALLEL tile template")
                fb = [f"  return {GTS_ERR_UNSUPPORTED};  // mirrored field: no fallback without the mirror stores"]
            if res is None:
                launches += fb
                for t in k.local_temps:
                    local_of[t] = -1  # always needs its arena slot
            elif resL is None:
                code, pre, launch = res
                out.extend(code)
                flag = f"fz_ok_{kidx}"
                fused_ok[kidx] = flag
                prelude += pre
                launches += [f"  if ({flag}) {{"] + launch + ["  } else {"] + fb + ["  }"]
            else:
                code, pre, launch = res
                codeL, preL, launchL = resL
                out.extend(code + codeL)
                flag, flagL = f"fz_ok_{kidx}", f"fz_okL_{kidx}"
                prelude += pre + [ln.replace(flag, flagL) for ln in preL]
                pts = f"(long long)ni * nj * nk"
                prelude.append(f"  const bool fzs_{kidx} = {pts} < {codegen_parallel.LARGE_POINTS}LL;"
                               "  // not large: the default geometry")
                head = []
                if resT is not None:
                    codeT, preT, launchT = resT
                    out.extend(codeT)
                    flagT = f"fz_okT_{kidx}"
                    prelude += [ln.replace(flag, flagT) for ln in preT]
                    prelude.append(f"  const bool fzt_{kidx} = {pts} < {codegen_parallel.TINY_POINTS}LL;")
                    fused_ok[kidx] = f"({flag} || {flagL} || {flagT})"
                    head = [f"  if ({flagT} && fzt_{kidx}) {{"] + launchT + ["  } else"]
                else:
                    fused_ok[kidx] = f"({flag} || {flagL})"
                launches += (head + [f"  if ({flag} && (fzs_{kidx} || !{flagL})) {{"] + launch
                             + [f"  }} else if ({flagL}) {{"] + launchL + ["  } else {"] + fb + ["  }"])
            if resF is not None:
                # frame requested (gts_frame_<name>_<digest8>) and the frame
                # variant's tensor maps are valid: the frame tiles only;
                # otherwise the full launch below (idempotent: frame_ok)
                codeF, preF, launchF = resF
                out.extend(codeF)
                out.append('extern "C" __attribute__((visibility("default")))')
                out.append(f"int {frame_tile_name(impl, fp)}(void) {{ return ({codegen_parallel.TI} << 16) | "
                           f"{codegen_parallel.TJ}; }}  // frame tile rows, columns")
                flagF = f"fz_okF_{kidx}"
                prelude += [ln.replace(f"fz_ok_{kidx}", flagF) for ln in preF]
                pos = len(launches) - 1
                while not launches[pos].startswith("  if ("):
                    pos -= 1
                while pos > 0 and launches[pos - 1] == "  } else":
                    pos -= 1
                    while not launches[pos].startswith("  if ("):
                        pos -= 1
                launches[pos:pos] = [f"  if (fr_ilo >= 0 && {flagF}) {{"] + launchF + ["  } else"]
            if fused_col is not None:
                pf_lines = launches
                launches = saved_launches
                cname = f"gts_k{kidx + 1}_column"
                out.extend(_column_kernel(cname, plan, nxt, ctype, dtypes))
                generic = [
                    "  {",
                    "    dim3 grid((unsigned)((nj + GTS_COL_TJ - 1) / GTS_COL_TJ),"
                    " (unsigned)((ni + (GTS_COL_THREADS / GTS_COL_TJ) - 1) / (GTS_COL_THREADS / GTS_COL_TJ)), 1);",
                    f"    {cname}<<<grid, GTS_COL_THREADS, 0, st>>>(p);",
                    "  }",
                ]
                code, launch = codegen_column.emit(cname, plan, nxt, fused_col, ctype, dtypes, opts,
                                                   fallback=pf_lines + generic)
                out.extend(code)
                launches += launch
                skip.add(kidx + 1)
            w("")
            continue
        if k.kind == "pstage":
            st = k.stages[0].stage
            out.extend(_point_kernel(kname, st, ctype, dtypes))
            e = st.compute_extent
            launches += [
                "  {",
                f"    const int k0 = {_bound(st.interval.start)}, k1 = {_bound(st.interval.end)};",
                f"    const int i0 = {e.lo[0]}, i1 = (int)ni + {e.hi[0]};",
                f"    const int j0 = {e.lo[1]}, j1 = (int)nj + {e.hi[1]};",
                "    if (k0 < k1 && i0 < i1 && j0 < j1) {",
                "      for (int kb = k0; kb < k1; kb += 65535) {",
                "        dim3 grid((unsigned)((j1 - j0 + 31) / 32), (unsigned)((i1 - i0 + 7) / 8),"
                " (unsigned)((k1 - kb) < 65535 ? (k1 - kb) : 65535));",
                f"        {kname}<<<grid, 256, 0, st>>>(p, i0, i1, j0, j1, kb);",
                "      }",
                "    }",
                "  }",
            ]
        elif k.kind == "plane":
            ms = impl.multistages[k.multistages[0]]
            stage_names = {}
            for r in k.stages:
                nm = f"{kname}_s{r.idx}"
                stage_names[id(r.stage)] = nm
                out.extend(_point_kernel(nm, r.stage, ctype, dtypes))
            launches.append("  {")
            for interval, stages in _interval_groups(ms):
                launches.append(f"    {{ const int k0 = {_bound(interval.start)}, k1 = {_bound(interval.end)};")
                if ms.order == ir.BACKWARD:
                    launches.append("      for (int k = k1 - 1; k >= k0; --k) {")
                else:
                    launches.append("      for (int k = k0; k < k1; ++k) {")
                for st in stages:
                    e = st.compute_extent
                    launches += [
                        f"        {{ const int i0 = {e.lo[0]}, i1 = (int)ni + {e.hi[0]};",
                        f"          const int j0 = {e.lo[1]}, j1 = (int)nj + {e.hi[1]};",
                        "          if (i0 < i1 && j0 < j1) {",
                        "            dim3 grid((unsigned)((j1 - j0 + 31) / 32), (unsigned)((i1 - i0 + 7) / 8), 1);",
                        f"            {stage_names[id(st)]}<<<grid, 256, 0, st>>>(p, i0, i1, j0, j1, k);",
                        "          }",
                        "        }",
                    ]
                launches.append("      }")
                launches.append("    }")
            launches.append("  }")
        elif k.kind == "column":
            out.extend(_column_kernel(kname, plan, k, ctype, dtypes))
            sp = codegen_column.spec(plan, k, dtypes) if opts.get("tmem", True) else None
            if sp is None and mirror and any(mirror in writes(r.stage.body) for r in k.stages):
                raise ValueError(f"gen_options mirror: '{mirror}' needs the TMEM column template")
            if sp is not None:
                code, launch = codegen_column.emit(kname, plan, k, sp, ctype, dtypes, opts)
                out.extend(code)
                launches += launch
                continue
            launches += [
                "  {",
                "    dim3 grid((unsigned)((nj + GTS_COL_TJ - 1) / GTS_COL_TJ),"
                " (unsigned)((ni + (GTS_COL_THREADS / GTS_COL_TJ) - 1) / (GTS_COL_THREADS / GTS_COL_TJ)), 1);",
                f"    {kname}<<<grid, GTS_COL_THREADS, 0, st>>>(p);",
                "  }",
            ]
        else:
            raise ValueError(k.kind)
        w("")

    # ---- host entry ----
    params = ["int64_t ni", "int64_t nj", "int64_t nk"]
    for f in impl.api_fields:
        params.append(f"{ctype[f.name]}* f_{f.name}")
        params += [f"int64_t s_{f.name}_{a}" for a in "ijk"]
        params += [f"int64_t o_{f.name}_{a}" for a in "ijk"]
    for s in impl.api_scalars:
        params.append(f"double sc_{s.name}")
    params.append("void* stream")
    name = entry_name(impl, fp)
    w('extern "C" __attribute__((visibility("default")))')
    w(f"int {name}(" + ", ".join(params) + ") {")
    w("  if (ni <= 0 || nj <= 0 || nk <= 0) return 0;")
    w(f"  if (nk < {impl.k_min}) return {GTS_ERR_K_MIN};")
    w("  if (ni > 0x3fffffff || nj > 0x3fffffff || nk > 0x3fffffff) return %d;" % GTS_ERR_UNSUPPORTED)
    w("  cudaStream_t st = (cudaStream_t)stream;")
    w("  GtsParams p;")
    w("  p.ni = (int)ni; p.nj = (int)nj; p.nk = (int)nk;")
    for f in impl.api_fields:
        n = f.name
        w(f"  p.f_{n} = gts_field(f_{n}, s_{n}_i, s_{n}_j, s_{n}_k, o_{n}_i, o_{n}_j, o_{n}_k);")
    for s in impl.api_scalars:
        w(f"  p.sc_{s.name} = sc_{s.name};")
    if frame_ok:
        w("  const int fr_ilo = g_frame_ilo, fr_ihi = g_frame_ihi, fr_jlo = g_frame_jlo, fr_jhi = g_frame_jhi;  // consumed by this launch")
        w("  g_frame_ilo = g_frame_ihi = g_frame_jlo = g_frame_jhi = -1;")
    if mirror:
        # the boxes apply to this launch only (set again before every launch)
        w("  p.mir = g_mirror;")
        w("  g_mirror.n = 0;")
    out.extend(prelude)
    if arena_temps:
        w("  // device arena for temporaries: shape = domain + extent (common.py:58-69),")
        w("  // k outermost, j contiguous, rows padded to 128 B; persistent across calls")
        w("  size_t arena_bytes = 0;")
        for t in arena_temps:
            e = temps[t].extent
            kk = local_of.get(t)
            need = f"!{fused_ok[kk]}" if kk is not None and kk in fused_ok else "true"
            w(f"  const bool need_{t} = {need};")
            w(f"  const int64_t td_{t}_i = ni + {e.hi[0] - e.lo[0]}, td_{t}_j = nj + {e.hi[1] - e.lo[1]};")
            w(f"  const int64_t tp_{t} = gts_pad_row(td_{t}_j, sizeof({ctype[t]}));")
            w(f"  const size_t toff_{t} = arena_bytes;")
            w(f"  if (need_{t}) arena_bytes += gts_round_up((size_t)(td_{t}_i * tp_{t} * nk) * sizeof({ctype[t]}), 256);")
        w("  GtsArenaLease lease(arena_bytes, st);  // held until every launch below is enqueued")
        w("  char* arena = lease.ptr;")
        w(f"  if (arena_bytes && !arena) return {GTS_ERR_ALLOC};")
        for t in arena_temps:
            e = temps[t].extent
            w(f"  if (need_{t}) p.f_{t} = gts_field(({ctype[t]}*)(arena + toff_{t}), tp_{t}, 1, td_{t}_i * tp_{t},"
              f" {-e.lo[0]}, {-e.lo[1]}, 0);")
        nanf = set(plan.nan_fill_temps)
        for k in plan.kernels:
            for t in k.local_temps:
                for r in k.stages:
                    if t in writes(r.stage.body) and t not in always_writes(r.stage.body):
                        nanf.add(t)
        for t in sorted(nanf):
            w(f"  if (need_{t}) gts_fill_nan(arena + toff_{t}, (size_t)(td_{t}_i * tp_{t} * nk), sizeof({ctype[t]}), st);")
    out.extend(launches)
    w("  return (int)cudaGetLastError();")
    w("}")
    w("")
    # count every triple-chevron launch (gts_b200_module_launch_count; the
    # gts_launch_pdl / gts_fill_nan helpers count their own)
    return _LAUNCH_RE.sub(r"\1++g_gts_launches; \2", "\n".join(out))


_LAUNCH_RE = re.compile(r"^([ \t]*)(\w+<<<)", re.M)
