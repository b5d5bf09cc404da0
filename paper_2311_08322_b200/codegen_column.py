"""Column template with Tensor-Memory column storage (the vadv-class kernel).

Instantiates the FORWARD-elimination / BACKWARD-substitution pattern of
implicit vertical solvers (stencilforge ``kernels/vadv.gts:4-16``) as one
persistent, warp-specialised sm_100a kernel:

* one CTA per SM, 4 consumer warps = 128 (i, j) columns per tile
  (32 contiguous j x 4 i), 1 producer warp;
* the producer streams every pure input of the FORWARD sweep with TMA
  (``cp.async.bulk.tensor.3d``, box 32 x 4 x KB levels per field) into a
  multi-stage shared-memory ring guarded by full/empty mbarriers, running
  ahead across tiles so HBM stays busy during the backward sweeps;
* consumers sweep k with register k-caches; temporaries produced by the
  forward sweep and consumed by the backward sweep (vadv's cp, dp) are kept
  in TMEM -- each thread owns one TMEM lane (512 x 32-bit columns), so the
  whole column history never touches HBM or L2 (the reference gen engine
  streams them through a malloc'd arena, ``gen.py:301-323``);
* the backward sweep reads them back with ``tcgen05.ld`` and writes the
  outputs with coalesced stores.

Eligibility (checked by ``spec()``; otherwise the generic column kernel of
``codegen.py`` runs): exactly [FORWARD, BACKWARD] multistages; the forward
sweep writes only temporaries and reads api fields only at offset (0,0,0);
the backward sweep reads forward temporaries only at (0,0,0); temporaries of
the backward sweep are not read by other launches.  At run time the TMEM
kernel needs nk * words-per-level <= 512 and TMA-compatible inputs (16-B
aligned origin and byte strides); the entry falls back otherwise.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

from ._host import ir
from .codegen import GTS_ERR_UNSUPPORTED, DivPool, _bound, _interval_groups, _MemCtx, c_float, emit_cond, emit_expr  # noqa: F401
from . import codegen_prologue
from .lowering import always_writes, reads, writes

KB = 8  # levels per TMA box (W=1 variant)
TI, TJ = 4, 32  # tile rows per consumer-warp group x 32 contiguous columns
RING_BUDGET = 196 * 1024
MAX_STAGES = 8
SMEM_MAX = 232448  # max dynamic shared memory per CTA on sm_100a


@dataclass
class ThomasSpec:
    ms_f: int
    ms_b: int
    streamed: list  # fields streamed through the TMA ring (forward reads): api fields / arena temps
    cross: list  # temps written in forward, read in backward -> TMEM
    words: dict  # temp -> 32-bit words per level
    offsets: dict  # temp -> word offset within a level
    w_level: int  # words per level
    stage_bytes: int
    offs_in_stage: dict  # streamed field -> byte offset within a ring stage
    nstages: int
    ms_e: Optional[int] = None  # fused PARALLEL epilogue multistage (zero extent)
    ewin: tuple = ()  # backward-written fields the epilogue reads, via a register window
    elo: int = 0  # window covers levels [m + elo, m + ehi] of epilogue level m
    ehi: int = 0
    pro: Optional[object] = None  # codegen_prologue.PrologueSpec fused in front of the forward sweep
    halo: dict = field(default_factory=dict)  # prologue input -> HaloBox
    coop: bool = True  # materialize multi-offset prologue temps cooperatively in smem
    deep_ring: bool = True  # also instantiate the deeper-ring W=2 geometry
    pro_warps: int = 0  # gen_options pro_warps: prologue warps (0 = consumers evaluate it)


@dataclass
class HaloBox:
    """TMA box of a prologue input: tile + its horizontal halo, KB levels."""

    lo_i: int
    rows_extra: int  # hi_i - lo_i
    cshift: int  # map base column lo_j - cshift is 16-B aligned
    bstart: int  # box start column relative to the tile's first column (= lo_j - cshift)
    cols: int  # box width (16-B multiple)
    esize: int


def _halo_box(ext, esize: int, rows: int) -> HaloBox:
    lo_i, hi_i, lo_j, hi_j = ext
    align = 16 // esize
    cshift = lo_j % align
    bstart = lo_j - cshift
    cols = (TJ - 1 + hi_j) - bstart + 1
    cols = -(-cols // align) * align
    return HaloBox(lo_i, hi_i - lo_i, cshift, bstart, cols, esize)


def _epilogue_ok(impl, mse, wf: set, wb: set, run_reads: set):
    """A trailing PARALLEL multistage fused into the backward sweep: it may
    read fields written by the backward sweep at vertical offsets (a register
    window, level m computed once level m + lo is known), pure inputs at any
    vertical offset (global loads) and its own temporaries at (0,0,0); it
    writes api fields nobody else in the run reads, or its own temps."""
    if mse.order != ir.PARALLEL:
        return None
    we = set()
    for st in mse.stages:
        we |= writes(st.body)
    if we & (wf | wb):
        return None
    win, lo, hi = set(), 0, 0
    for st in mse.stages:
        for acc in reads(st.body):
            di, dj, dk = acc.offset
            if di or dj:
                return None
            if acc.field in wf:
                return None  # forward temporaries are gone by then (TMEM reused)
            if acc.field in wb:
                if acc.field in {f.name for f in impl.api_fields}:
                    return None  # api outputs of the sweep: no register copy kept
                win.add(acc.field)
                lo, hi = min(lo, dk), max(hi, dk)
            elif acc.field in we and dk != 0:
                return None
    if we & run_reads:
        return None
    return tuple(sorted(win)), lo, hi


def spec(plan, kplan, dtypes: dict, pro=None) -> Optional[ThomasSpec]:
    """``pro``: a PrologueSpec (codegen_prologue) to fuse in front of the
    forward sweep; its exports are computed in-kernel instead of streamed."""
    impl = plan.impl
    if kplan.kind != "column" or len(kplan.multistages) not in (2, 3):
        return None
    mf, mb = kplan.multistages[:2]
    msf, msb = impl.multistages[mf], impl.multistages[mb]
    if msf.order != ir.FORWARD or msb.order != ir.BACKWARD:
        return None
    api = {f.name for f in impl.api_fields}
    wf, wb = set(), set()
    for st in msf.stages:
        wf |= writes(st.body)
    for st in msb.stages:
        wb |= writes(st.body)
    if wf & api:
        return None
    # readers outside this run: every temporary the run writes must stay
    # kernel-local (the template keeps them in TMEM / registers only)
    outside = set()
    for mi, ms in enumerate(impl.multistages):
        if mi in kplan.multistages:
            continue
        for st in ms.stages:
            outside |= {a.field for a in reads(st.body)}
    if (wf | wb) & outside & set(plan.global_temps):
        return None
    run_reads = set()
    for ms in (msf, msb):
        for st in ms.stages:
            run_reads |= {a.field for a in reads(st.body)}
    ms_e, ewin, elo, ehi = None, (), 0, 0
    if len(kplan.multistages) == 3:
        ms_e = kplan.multistages[2]
        got = _epilogue_ok(impl, impl.multistages[ms_e], wf, wb, run_reads)
        if got is None:
            return None
        ewin, elo, ehi = got
    streamed = []
    for st in msf.stages:
        for acc in reads(st.body):
            # api inputs, and arena temporaries produced by an earlier launch
            # (unless a fused prologue computes them in-kernel)
            if pro is not None and acc.field in pro.exports:
                if acc.offset != (0, 0, 0):
                    return None
                continue
            if acc.field in api or (acc.field in plan.global_temps and acc.field not in wf | wb):
                if acc.offset != (0, 0, 0) or acc.field in wb:
                    return None
                if acc.field not in streamed:
                    streamed.append(acc.field)
    cross = []
    for st in msb.stages:
        for acc in reads(st.body):
            if acc.field in wf:
                if acc.offset != (0, 0, 0):
                    return None
                if acc.field not in cross:
                    cross.append(acc.field)
    if not streamed and pro is None:
        return None
    halo = {}
    if pro is not None:
        for f in pro.inputs:
            if f in streamed:
                return None  # read both with and without halo: not supported
            halo[f] = pro.extent[f]
    cross.sort()
    words = {t: (2 if dtypes[t] == ir.F64 else 1) for t in cross}
    offsets, w = {}, 0
    for t in cross:
        offsets[t] = w
        w += words[t]
    esize = {f: (8 if dtypes[f] == ir.F64 else 4) for f in streamed}
    offs, sb = {}, 0
    for f in streamed:
        offs[f] = sb
        sb += KB * TI * TJ * esize[f]
    nstages = max(2, min(MAX_STAGES, RING_BUDGET // sb))
    if nstages * sb > RING_BUDGET:
        return None
    for f in halo:  # capacity check with the W=1 geometry (the largest boxes per level)
        hb = _halo_box(halo[f], 8 if dtypes[f] == ir.F64 else 4, TI)
        sb += KB * (TI + hb.rows_extra) * hb.cols * hb.esize
    if 2 * sb > RING_BUDGET:
        return None
    return ThomasSpec(mf, mb, streamed, cross, words, offsets, max(w, 1), sb, offs, nstages,
                      ms_e, ewin, elo, ehi, pro, halo)


class _Ctx(_MemCtx):
    """Field access spelling inside the TMEM column kernel."""

    def __init__(self, dtypes, sp: ThomasSpec, phase: str, cached: dict, ctype: dict):
        super().__init__(dtypes)
        self.sp, self.phase, self.cached, self.ctype = sp, phase, cached, ctype
        self.ring = True  # forward reads of streamed fields come from the TMA ring
        self.div_mode = "fast"

    def addr(self, name, off):
        di, dj, dk = off
        ii = f"(ic{di:+d})" if di else "ic"
        jj = f"(jc{dj:+d})" if dj else "jc"
        kk = f"(k{dk:+d})" if dk else "k"
        return f"GTS_AT(p.f_{name}, {ii}, {jj}, {kk})"

    pro_vals: dict = {}
    kstride = None  # level stride of a ring stage (default rows * TJ)

    def read(self, name, off):
        if self.phase == "f" and name in self.pro_vals and off == (0, 0, 0):
            return self.pro_vals[name]
        if self.phase == "f" and self.ring and name in self.sp.streamed:
            # ur_<f>: this thread's element of level 0 of the stage (hoisted
            # per stage), so each level is an immediate-offset shared load
            return f"((double)ur_{name}[kk * {self.kstride or self.rows * TJ}])"
        direction = 1 if self.phase == "f" else -1
        if name in self.cached and not (off[0] or off[1]):
            if off[2] == 0:
                return f"cur_{name}"
            s = -off[2] * direction
            if 1 <= s <= self.cached[name]:
                return f"prev{s}_{name}"
        return super().read(name, off)


_NOSTORE = False
_MIRROR = None  # gen_options mirror: api field whose stores also go to neighbour halos
# gen_options mirror_inline: mirror stores at production (per level, targets
# resolved per column at tile start) instead of the tile-end pass.  Bitwise
# (tools/peer_fused_check.py --inline, 2 / 4 processes) but slower
# (tools/mirror_cost.py, dycore 512^2x80: 185.7 / 193.9 us/step with 0 / 8
# neighbours against 171-175 / 189 for the pass: the live target registers
# cost the recurrence), so opt-in.
_MIRROR_INLINE = False


def _emit_stmt(stmt, ctx: _Ctx, ctype, api: set, indent: str, out: list) -> None:
    pool = ctx.pool
    if isinstance(stmt, ir.Assign):
        name = stmt.target.field
        value = emit_expr(stmt.value, ctx)
        pool.flush(indent, out)
        out.append(f"{indent}{{ const double v_ = {value};")
        if name in api:
            guard = "valid && v_ == 1234.5678" if _NOSTORE else "valid"  # tmem_debug nostore (timing)
            out.append(f"{indent}  {{ {ctype[name]}* xp_ = colp_{name} + (long long)k * p.f_{name}.sk;"
                       f" if ({guard}) *xp_ = ({ctype[name]})(v_); }}")
            if _MIRROR_INLINE and name == _MIRROR:
                # mirror stores at production: this column's resolved targets
                # (warp-uniform skip for warps without a boundary column)
                t_ = ctype[name]
                out.append(f"{indent}  if (wmir_) {{")
                for m in range(3):
                    out.append(f"{indent}    if (nmi_ > {m}) mq{m}_[(long long)k * mk{m}_] = ({t_})(v_);")
                out.append(f"{indent}  }}")
        if name in ctx.cached or name not in api:
            out.append(f"{indent}  cur_{name} = (double)({ctype[name]})(v_);")
        out.append(f"{indent}}}")
        pool.invalidate(name)
        return
    if isinstance(stmt, ir.If):
        cond = emit_cond(stmt.cond, ctx)
        pool.flush(indent, out)
        out.append(f"{indent}if ({cond}) {{")
        pool.depth += 1
        for s in stmt.then_body:
            _emit_stmt(s, ctx, ctype, api, indent + "  ", out)
        if stmt.else_body:
            out.append(f"{indent}}} else {{")
            for s in stmt.else_body:
                _emit_stmt(s, ctx, ctype, api, indent + "  ", out)
        pool.depth -= 1
        out.append(f"{indent}}}")
        return
    raise TypeError(type(stmt).__name__)


def _caches(ms, direction: int) -> dict:
    w = set()
    for st in ms.stages:
        w |= writes(st.body)
    cached = {}
    for st in ms.stages:
        for acc in reads(st.body):
            if acc.field in w and not (acc.offset[0] or acc.offset[1]) and acc.offset[2]:
                s = -acc.offset[2] * direction
                if s > 0:
                    cached[acc.field] = max(cached.get(acc.field, 0), s)
    return cached


def _need_load(stages, f) -> bool:
    for st in stages:
        if any(acc.field == f and acc.offset == (0, 0, 0) for acc in reads(st.body)):
            return True
        if f in always_writes(st.body) and isinstance(st.body, ir.Assign):
            return False
        if f in writes(st.body):
            return True
    return True



@dataclass
class Variant:
    """One launch configuration of the TMEM column template.

    W consumer warps per SM sub-partition (4*W consumer warps, one producer);
    tile = 4*W rows x 32 columns; the per-column history of the cross
    temporaries lives in TMEM for the first ``tl`` levels (each thread owns
    512/W columns of its TMEM lane) and in shared memory for the next ``sl``
    levels, so the kernel serves any nk <= tl + sl."""

    w: int
    kb: int
    nst: int
    stage_bytes: int
    offs: dict
    tl: int
    sl: int
    smem_bytes: int
    hist_off: int
    hbox: dict = field(default_factory=dict)  # prologue input -> HaloBox for this geometry
    tx: int = 0  # bytes the TMA boxes of one ring stage deliver (mbarrier expect-tx)
    mat: dict = field(default_factory=dict)  # materialized prologue temp -> (smem offset in a set, rows, cols, esize, region)
    mat_off: int = 0  # smem offset of the two materialization buffer sets
    mat_half: int = 0  # bytes of one set
    cps: int = 1  # CTAs per SM (TMEM and shared memory split between them)


def variants(sp: ThomasSpec, dtypes: dict, geoms_override=None) -> list:
    esize = {f: (8 if dtypes[f] == ir.F64 else 4) for f in sp.streamed}
    hist_bytes = 4 * sp.w_level  # bytes per level per column
    out = []
    # deeper-ring W=2 geometry first: its smaller history tier serves nk <= 80
    # (the benchmark depth), and the extra stages keep HBM busy while the
    # backward sweeps run; the regular W=2 and the W=1 geometry cover deeper
    # columns
    seen = set()
    geoms = ((2, 4, 160 * 1024), (2, 4, 128 * 1024), (1, 8, RING_BUDGET))
    if not sp.deep_ring:
        # without a prologue, two CTAs per SM (W=1, 4-level stages, 64 KiB
        # rings, TMEM and shared memory halved) first: the two pipelines run
        # out of phase.  tools/abtest.py (medians of 5 / 3): vadv 256^2 35.58 ->
        # 35.24 us, 512^2 131.1 -> 129.3, f32 256^2 35.56 -> 35.03; 2- or 8-level
        # stages and an 80 KiB ring were slower; the dycore kernel (prologue)
        # measured 175.5 -> 177.9 us/step, so it keeps one CTA per SM
        geoms = ((1, 4, 64 * 1024, 2),) + geoms[1:]
    if geoms_override:  # gen_options tmem_geom: [[w, kb, ring KiB(, CTAs per SM)], ...] (experiments)
        geoms = tuple((int(g[0]), int(g[1]), int(g[2]) * 1024) + tuple(int(x) for x in g[3:4])
                      for g in geoms_override)
    for geom in geoms:
        w, kb, budget = geom[:3]
        cps = geom[3] if len(geom) > 3 else 1
        rows = 4 * w
        offs, sb = {}, 0
        for f in sp.streamed:
            offs[f] = sb
            sb += kb * rows * TJ * esize[f]
        tx = sb
        hboxes = {}
        for f, ext in sp.halo.items():
            hb = _halo_box(ext, 8 if dtypes[f] == ir.F64 else 4, rows)
            hboxes[f] = hb
            sb = -(-sb // 128) * 128
            offs[f] = sb
            nb = kb * (rows + hb.rows_extra) * hb.cols * hb.esize
            sb += nb
            tx += nb
        sb = -(-sb // 128) * 128
        nst = max(2, min(MAX_STAGES, budget // sb))
        ring = nst * sb
        nct = 32 * rows
        # cooperative prologue: temporaries materialized per ring stage in two
        # alternating shared-memory sets (codegen_prologue.materialized)
        mat, half = {}, 0
        if sp.pro is not None and sp.coop:
            for t, (li, hi, lj, hj) in codegen_prologue.materialized(sp.pro).items():
                e = 8 if dtypes[t] == ir.F64 else 4
                rr, cc = rows + hi - li, TJ + hj - lj
                mat[t] = (half, rr, cc, e, (li, hi, lj, hj))
                half += -(-(kb * rr * cc * e) // 128) * 128
        bars = (3 if sp.pro_warps else 2) * 8 * nst + 16
        free = (SMEM_MAX if cps == 1 else SMEM_MAX // cps - 1024) - ring - 2 * half - bars - 64
        sl = max(0, free // (nct * hist_bytes))
        hist_off = ring + 2 * half
        smem = ring + 2 * half + sl * nct * hist_bytes + bars + 16
        tl = (512 // cps // w) // sp.w_level
        if nst * sb > budget or (w, nst, cps) in seen or free < 0:
            continue
        seen.add((w, nst, cps))
        out.append(Variant(w, kb, nst, sb, offs, tl, sl, smem, hist_off, hboxes, tx, mat, ring, half, cps))
    return out


def _base_nst(sp, v, dtypes) -> int:
    """Ring depth of the regular geometry of width v.w (kernel naming)."""
    budget = 128 * 1024 if v.w == 2 else RING_BUDGET
    return max(2, min(MAX_STAGES, budget // v.stage_bytes))


def emit(kname: str, plan, kplan, sp: ThomasSpec, ctype: dict, dtypes: dict, opts=None,
         fallback=None):
    """``fallback``: host lines run when no variant can launch (default: the
    generic column kernel; with a fused prologue, the prologue's own launch
    followed by the generic column kernel)."""
    code, launch_variants = [], []
    only_w = (opts or {}).get("tmem_w")  # gen_options: restrict to one geometry (experiments)
    # cooperative materialization measured slower (235 vs 179 us/step: the per-stage
    # consumer barrier serialises the 8 warps), so it is opt-in
    sp.coop = bool((opts or {}).get("pro_coop", False)) and bool((opts or {}).get("pro_batch", True))
    # measured: the deeper ring helps the fused dycore kernel (181 -> 177 us/step)
    # and costs vadv ~0.9 us at 256^2, so it defaults on with a prologue only
    sp.deep_ring = bool((opts or {}).get("deep_ring", sp.pro is not None))
    # gen_options pro_warps: the fused prologue runs on its own warps, one
    # ring stage ahead of the consumers (see _emit_variant)
    sp.pro_warps = int((opts or {}).get("pro_warps", 0)) if sp.pro is not None and not sp.coop else 0
    for v in variants(sp, dtypes, (opts or {}).get("tmem_geom")):
        if only_w and v.w != int(only_w):
            continue
        c, cond, call = _emit_variant(kname, plan, sp, v, ctype, dtypes, opts)
        code += c
        launch_variants.append((cond, call, v))
    launch = ["  {"]
    for f in list(sp.streamed) + list(sp.halo):
        launch.append(f"    CUtensorMap tm_{f}[{max(1, len(launch_variants))}];")
    launch.append("    bool launched = false;")
    for vi, (cond, call, v) in enumerate(launch_variants):
        launch.append(f"    if (!launched && nk <= {v.tl + v.sl}) {{")
        launch.append("      bool ok = true;")
        for f in sp.streamed:
            e = 8 if dtypes[f] == ir.F64 else 4
            launch.append(
                f"      ok = ok && gts_make_tmap_3d(&tm_{f}[{vi}], (const void*)p.f_{f}.p, {e}, nj, ni, nk,"
                f" p.f_{f}.si, p.f_{f}.sj, p.f_{f}.sk, {TJ}, {4 * v.w}, {v.kb});")
        for f, hb in v.hbox.items():
            lo_i, hi_i, lo_j, hi_j = sp.halo[f]
            launch.append(
                f"      ok = ok && gts_make_tmap_3d(&tm_{f}[{vi}], (const void*)&GTS_AT(p.f_{f}, {lo_i}, {hb.bstart}, 0),"
                f" {hb.esize}, nj + {hi_j - hb.bstart}, ni + {hi_i - lo_i}, nk,"
                f" p.f_{f}.si, p.f_{f}.sj, p.f_{f}.sk, {hb.cols}, {4 * v.w + hb.rows_extra}, {v.kb});")
        launch.append("      if (ok) {")
        launch += ["        " + ln for ln in call(vi)]
        launch.append("        launched = true;")
        launch.append("      }")
        launch.append("    }")
    if (opts or {}).get("mirror"):
        fallback = [f"  return {GTS_ERR_UNSUPPORTED};  // a mirrored field needs this template"]
    if fallback is None:
        fallback = [
            "  {",
            "    dim3 grid((unsigned)((nj + GTS_COL_TJ - 1) / GTS_COL_TJ),"
            " (unsigned)((ni + (GTS_COL_THREADS / GTS_COL_TJ) - 1) / (GTS_COL_THREADS / GTS_COL_TJ)), 1);",
            f"    {kname}<<<grid, GTS_COL_THREADS, 0, st>>>(p);",
            "  }",
        ]
    launch += ["    if (!launched) {"] + ["    " + ln for ln in fallback] + ["    }", "  }"]
    return code, launch


def _emit_variant(kname, plan, sp: ThomasSpec, v: Variant, ctype, dtypes, opts):
    """Persistent warp-specialised kernel: per tile, a FORWARD sweep fed by
    the TMA ring writes the column history (TMEM tier, then shared-memory
    tier), then a BACKWARD sweep reads it back.  Each ring stage / history
    batch is emitted as straight-line code specialised for the interval
    group and history tier it falls in, so the compiler can overlap the
    independent work of neighbouring levels with the serial recurrence; a
    generic per-level-checked body covers partial stages and group
    boundaries."""
    dbg = (opts or {}).get("tmem_debug", "")
    global _NOSTORE, _MIRROR, _MIRROR_INLINE
    _NOSTORE = dbg == "nostore"
    _MIRROR = (opts or {}).get("mirror") or None
    _MIRROR_INLINE = bool(_MIRROR) and bool((opts or {}).get("mirror_inline", False))
    impl = plan.impl
    api = {f.name for f in impl.api_fields}
    msf, msb = impl.multistages[sp.ms_f], impl.multistages[sp.ms_b]
    rows = 4 * v.w
    ncw = 4 * v.w
    nct = 32 * ncw
    # prologue warps (gen_options pro_warps): warps ncw+1 .. ncw+PW evaluate
    # the fused prologue for a ring stage as soon as its boxes land and
    # write the exports over the stage's (then consumed) halo boxes; the
    # consumers' forward sweep reads them from there (one more mbarrier per
    # stage).  Needs the exports (binary64 slots) to fit the halo boxes.
    PW = sp.pro_warps if (sp.pro is not None and v.hbox and not v.mat) else 0
    slot_off, slot_bytes = {}, v.kb * rows * TJ * 8
    if PW:
        h0 = min(v.offs[f] for f in v.hbox)
        room = sum(v.kb * (rows + hb_.rows_extra) * hb_.cols * hb_.esize for hb_ in v.hbox.values())
        if rows % PW or len(sp.pro.exports) * slot_bytes > room:
            PW = 0
        else:
            for n_, f in enumerate(sp.pro.exports):
                slot_off[f] = h0 + n_ * slot_bytes
    threads = nct + 32 + 32 * PW
    kn = f"{kname}_tmem_w{v.w}" + (f"s{v.nst}" if v.nst != _base_nst(sp, v, dtypes) else "") + (f"c{v.cps}" if v.cps > 1 else "")
    wl = sp.w_level
    hb = 4 * wl
    hoff, o = {}, 0
    for t in sp.cross:
        hoff[t] = o
        o += 4 * sp.words[t] * nct
    KB = v.kb
    assert v.tl % KB == 0
    out: list = []
    w = out.append
    tm_fields = list(sp.streamed) + list(sp.halo)
    # two-height tile plan (gts_col_split): the last rounds' tiles are h2 < rows
    # i-rows high so every SM carries a similar load; streamed-only kernels.
    # Measured (tools/ksweep.py, B200): 444x256x80 69.2 -> 67.7 us and
    # 148x256x80 32.6 -> 31.1 us, but 256^2x80 38.2 -> 38.6 us (its second
    # round is bandwidth-bound either way) and +1% where no split applies
    # (the runtime level stride), so it is opt-in
    split = not v.hbox and not v.mat and bool((opts or {}).get("col_split", False))
    # gen_options col_l2pf: in two-round grids, L2 prefetch of a CTA's second
    # tile's next col_l2pf stages once the ring holds its first ones;
    # col_l2pf0: the first tile's first stages before griddepcontrol.wait.
    # Measured (tools/abtest.py, medians of 5): vadv 256^2 36.66 -> 35.56 us with
    # 8 stages (2/4/10/12 stages: 36.10/35.80/36.01/36.46; the next tile's stages
    # issued one ring depth before the current tile's end instead: 39.5 us, removed);
    # dycore (prologue kernels) +1 us, so off there.  With the two-CTA geometry
    # (4-level stages) re-swept, medians of 7: 4/5/6/7/8 stages 35.02/34.94/34.91/
    # 34.98/35.23 us
    l2pf = 0 if split else int((opts or {}).get("col_l2pf", 6 if sp.pro is None else 0))
    # measured: vadv 256^2 38.22 -> 36.64 us with 4 stages (one-CTA geometry); dycore
    # neutral; re-swept with the two-CTA geometry (medians of 7): 4/5/6/8 stages
    # 34.89/34.77/34.79/34.97 us
    l2pf0 = int((opts or {}).get("col_l2pf0", 5 if sp.pro is None else 0))
    tm_params = ", ".join(f"const __grid_constant__ CUtensorMap tm_{f}" for f in tm_fields)
    if split:
        tm_params += ", " + ", ".join(f"const __grid_constant__ CUtensorMap tm2_{f}" for f in tm_fields)
    w(f"// TMEM column kernel, W={v.w}: {nct} columns/CTA, streamed {sp.streamed} (ring {v.nst} x"
      f" {v.stage_bytes} B), history {sp.cross}: TMEM levels [0,{v.tl}), smem levels"
      f" [{v.tl},{v.tl + v.sl})")
    w(f"__global__ void __launch_bounds__({threads}, {v.cps}) {kn}(const __grid_constant__ GtsParams p, "
      f"{tm_params}, int tiles_j, int ntiles" + (", int n1, int isplit, int h2" if split else "") + ") {")
    w("  extern __shared__ __align__(1024) unsigned char smem[];")
    w(f"  constexpr int NST = {v.nst};")
    w(f"  constexpr unsigned STB = {v.stage_bytes}u;")
    w(f"  constexpr int TL = {v.tl};")
    w(f"  unsigned char* hist = smem + {v.hist_off};")
    nbar = 3 if sp.pro_warps else 2  # variants() sized the barrier block
    w(f"  uint64_t* full = (uint64_t*)(smem + {v.smem_bytes - (nbar * 8 * v.nst + 16) - 16});")
    w("  uint64_t* empty = full + NST;")
    if nbar == 3:
        w("  uint64_t* pfull = empty + NST;  // prologue exports of a stage written")
        w("  uint32_t* tslot = (uint32_t*)(pfull + NST);")
    else:
        w("  uint32_t* tslot = (uint32_t*)(empty + NST);")
    w("  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;")
    w(f"  if (warp == 0) gts_tmem_alloc<{512 // v.cps}>(tslot);")
    w("  if (threadIdx.x == 0) {")
    w(f"    for (int s = 0; s < NST; ++s) {{ gts_mbar_init(&full[s], 1); gts_mbar_init(&empty[s], {ncw}); }}")
    if PW:
        w(f"    for (int s = 0; s < NST; ++s) gts_mbar_init(&pfull[s], {PW});")
    w("    gts_fence_mbar_init();")
    w("  }")
    w("  gts_tmem_fence_before_sync();")
    w("  __syncthreads();")
    w("  gts_tmem_fence_after_sync();")
    w("  gts_griddep_launch_dependents();")
    if l2pf0 and not split:
        # the first tile's first levels into L2 while the previous grid drains
        # (an L2 prefetch is coherent with its writes, see gts_tma_prefetch_l2_3d)
        w(f"  if (warp == {ncw} && lane == 0 && (int)blockIdx.x < ntiles) {{")
        w(f"    const int jf_ = ((int)blockIdx.x % tiles_j) * {TJ}, if_ = ((int)blockIdx.x / tiles_j) * {rows};")
        w(f"    for (int q_ = 0; q_ < {l2pf0} && q_ * {KB} < p.nk; ++q_) {{")
        for f in tm_fields:
            w(f"      gts_tma_prefetch_l2_3d(&tm_{f}, jf_, if_, q_ * {KB});")
        w("    }")
        w("  }")
    w("  gts_griddep_wait();  // PDL: previous grid complete before any global access")
    w("  const uint32_t tbase = *tslot;")
    w("  const int nk = p.nk;")
    w(f"  const int nkb = (nk + {KB - 1}) / {KB};")
    w(f"  if (warp == {ncw}) {{")
    w("    if (lane == 0) {")
    for f in tm_fields:
        w(f"      gts_prefetch_tensormap(&tm_{f});")
    w("      int it = 0;")
    w("      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {")
    if split:
        assert v.tx % rows == 0
        w("        const bool c2_ = t >= n1;")
        w("        const int u_ = c2_ ? t - n1 : t;")
        w(f"        const int j0 = (u_ % tiles_j) * {TJ}, i0 = c2_ ? isplit + (u_ / tiles_j) * h2 : (u_ / tiles_j) * {rows};")
        w(f"        const uint32_t txb_ = c2_ ? (uint32_t)h2 * {v.tx // rows}u : {v.tx}u;")
    else:
        w(f"        const int j0 = (t % tiles_j) * {TJ}, i0 = (t / tiles_j) * {rows};")
    w("        for (int kb = 0; kb < nkb; ++kb, ++it) {")
    w("          const int s = it % NST;")
    w("          const uint32_t ph = (uint32_t)(it / NST) & 1u;")
    sleep_ns = int((opts or {}).get("col_sleep_ns", 200))  # producer back-off on a full ring
    w(f"          if (it >= NST) gts_mbar_wait_sleep<{sleep_ns}>(&empty[s], ph ^ 1u);")
    if split:
        w("          gts_mbar_arrive_expect_tx(&full[s], txb_);")
        w("          if (c2_) {")
        for f in tm_fields:
            w(f"            gts_tma_load_3d(smem + s * STB + {v.offs[f]}, &tm2_{f}, &full[s], j0, i0, kb * {KB});")
        w("          } else {")
        for f in tm_fields:
            w(f"            gts_tma_load_3d(smem + s * STB + {v.offs[f]}, &tm_{f}, &full[s], j0, i0, kb * {KB});")
        w("          }")
    else:
        w(f"          gts_mbar_arrive_expect_tx(&full[s], {v.tx}u);")
        for f in tm_fields:
            w(f"          gts_tma_load_3d(smem + s * STB + {v.offs[f]}, &tm_{f}, &full[s], j0, i0, kb * {KB});")
        if l2pf:
            # default: once the ring holds this (non-first) tile's first NST
            # stages -- the previous tile's forward sweep is ending -- warm L2
            # with the next col_l2pf stages, streamed while its backward runs.
            # Only in two-round grids (every CTA in phase, so all backward
            # sweeps leave HBM idle at once); with more rounds the CTAs drift
            # apart and HBM stays busy (measured: 512^2 131.4 -> 133.5 us)
            w(f"          if (kb == NST - 1 && t != (int)blockIdx.x && ntiles <= 2 * (int)gridDim.x) {{")
            w(f"            for (int q_ = NST; q_ < NST + {l2pf} && q_ < nkb; ++q_) {{")
            for f in tm_fields:
                w(f"              gts_tma_prefetch_l2_3d(&tm_{f}, j0, i0, q_ * {KB});")
            w("            }")
            w("          }")
    w("        }")
    w("      }")
    w("    }")
    if PW:
        _emit_prologue_warps(w, out, sp, v, ctype, ncw, PW, rows, slot_off)
    w("  } else {")
    w(f"    const uint32_t tl = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * {512 // v.cps // v.w});")
    w("    const int ct = threadIdx.x;")
    w("    int it = 0;")
    gf = _interval_groups(msf)
    gb = _interval_groups(msb)
    for gi, (iv, _) in enumerate(gf):
        w(f"    const int f{gi}k0 = {_bound(iv.start)}, f{gi}k1 = {_bound(iv.end)};")
    for gi, (iv, _) in enumerate(gb):
        w(f"    const int b{gi}k0 = {_bound(iv.start)}, b{gi}k1 = {_bound(iv.end)};")
    w("    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {")
    if split:
        w("      const bool c2_ = t >= n1;")
        w("      const int u_ = c2_ ? t - n1 : t;")
        w(f"      const int h_ = c2_ ? h2 : {rows};")
        w(f"      const int hs_ = h_ * {TJ};  // level stride of a ring stage's boxes")
        w(f"      const int j = (u_ % tiles_j) * {TJ} + lane, i = (c2_ ? isplit + (u_ / tiles_j) * h2 : (u_ / tiles_j) * {rows}) + warp;")
        w("      if (warp >= h_ || i >= p.ni) {  // no row of this tile: keep the ring's phases only")
        w("        for (int kb = 0; kb < nkb; ++kb, ++it) {")
        w("          gts_mbar_wait(&full[it % NST], (uint32_t)(it / NST) & 1u);")
        w("          __syncwarp();")
        w("          if (lane == 0) gts_mbar_arrive(&empty[it % NST]);")
        w("        }")
        w("        continue;")
        w("      }")
    else:
        w(f"      const int j = (t % tiles_j) * {TJ} + lane, i = (t / tiles_j) * {rows} + warp;")
    w("      const bool valid = (i < p.ni) && (j < p.nj);")
    w("      const int ic = i < p.ni ? i : p.ni - 1, jc = j < p.nj ? j : p.nj - 1;")
    w("      (void)ic; (void)jc;")
    mse = impl.multistages[sp.ms_e] if sp.ms_e is not None else None
    epi_stages = list(mse.stages) if mse is not None else []
    for f in impl.api_fields:
        if any(f.name in writes(st.body) for st in list(msb.stages) + epi_stages):
            w(f"      {ctype[f.name]}* const colp_{f.name} = &GTS_AT(p.f_{f.name}, ic, jc, 0);")
    if _MIRROR_INLINE:
        # gen_options mirror_inline: this column's (at most 3) mirror targets,
        # resolved once per tile; stores follow the column's own (_emit_stmt)
        t_ = ctype[_MIRROR]
        w(f"      {t_}* mq0_ = nullptr; {t_}* mq1_ = nullptr; {t_}* mq2_ = nullptr;")
        w("      long long mk0_ = 0, mk1_ = 0, mk2_ = 0;")
        w("      int nmi_ = 0;")
        w("      if (valid) {")
        w("        for (int d = 0; d < p.mir.n; ++d) {")
        w("          if (i < p.mir.i0[d] || i >= p.mir.i1[d] || j < p.mir.j0[d] || j >= p.mir.j1[d]) continue;")
        w(f"          {t_}* const q_ = p.mir.base[d] + (long long)i * p.mir.si[d] + (long long)j * p.mir.sj[d];")
        w("          if (nmi_ == 0) { mq0_ = q_; mk0_ = p.mir.sk[d]; }")
        w("          else if (nmi_ == 1) { mq1_ = q_; mk1_ = p.mir.sk[d]; }")
        w("          else { mq2_ = q_; mk2_ = p.mir.sk[d]; }")
        w("          ++nmi_;")
        w("        }")
        w("      }")
        w("      const bool wmir_ = __any_sync(0xffffffffu, nmi_ > 0);")
    cf = _caches(msf, 1)
    wf = set()
    for st in msf.stages:
        wf |= writes(st.body)
    tracked_f = sorted(wf)
    cached_f = {f: d for f, d in cf.items()} | {f: 0 for f in tracked_f if f not in cf}

    def store_hist(indent, tier):
        if tier == "tmem":
            for t in sp.cross:
                col = f"(uint32_t)(k * {wl} + {sp.offsets[t]})"
                if sp.words[t] == 2:
                    w(f"{indent}gts_tmem_store_f64(tl + {col}, cur_{t});")
                else:
                    w(f"{indent}gts_tmem_store_f32(tl + {col}, (float)cur_{t});")
        else:
            w(f"{indent}{{ unsigned char* hl = hist + (size_t)(k - TL) * {hb * nct};")
            for t in sp.cross:
                w(f"{indent}  (({ctype[t]}*)(hl + {hoff[t]}))[ct] = ({ctype[t]})cur_{t};")
            w(f"{indent}}}")

    def prologue_rd(ring: bool):
        # dj may be a C expression (a warp-edge lane's per-lane column)
        if ring:
            def rd(name, di, dj):
                hb = v.hbox[name]
                off = di * hb.cols + dj if isinstance(dj, int) else f"{di * hb.cols} + {dj}"
                return f"uh_{name}[kk * {(rows + hb.rows_extra) * hb.cols} + {off}]"
        else:
            def rd(name, di, dj):
                ii = f"(ic{di:+d})" if di else "ic"
                jj = (f"(jc{dj:+d})" if dj else "jc") if isinstance(dj, int) else f"(jc + {dj})"
                return f"GTS_AT(p.f_{name}, {ii}, {jj}, k)"
        return rd

    # neighbour-lane shuffles in the prologue (codegen_prologue.lane_shuffled):
    # consumer lanes are 32 consecutive j columns of one i row.  Bitwise, but
    # measured slower (tools/abtest.py, dycore 512^2x80, medians of 3: 190.5 vs
    # 172.8 us/step: the edge evaluation's per-lane column defeats the
    # compiler's sharing of the cross's loads and the body grows from 3816 to
    # 4656 instructions), so it is opt-in
    pro_lane = "lane" if (opts or {}).get("pro_shfl", False) else None

    pro_batch = sp.pro is not None and (opts or {}).get("pro_batch", True) and not PW

    def mat_reads():
        """Phase-B spellings of the materialized temps (this stage's set)."""
        reads_ = {}
        for t, (off, rr, cc, e, (li, hi, lj, hj)) in v.mat.items():
            def rd(di, dj, off=off, rr=rr, cc=cc, li=li, lj=lj, t=t):
                return (f"((const {ctype[t]}*)(smem + {v.mat_off} + (it & 1) * {v.mat_half} + {off}))"
                        f"[(kk * {rr} + (warp + {di - li})) * {cc} + (lane + {dj - lj})]")
            reads_[t] = rd
        return reads_

    def coop_phase(indent):
        """Phase A: every consumer thread computes a share of each
        materialized temp over the tile + its halo for the KB levels of
        this stage; one named barrier (consumers only) publishes them.  Two
        alternating sets make a second barrier unnecessary: a set is reused
        two stages later, after every consumer passed the next barrier."""
        for t, (off, rr, cc, e, (li, hi, lj, hj)) in v.mat.items():
            n = KB * rr * cc
            w(f"{indent}{{ {ctype[t]}* const mb_ = ({ctype[t]}*)(smem + {v.mat_off} + (it & 1) * {v.mat_half} + {off});")
            w(f"{indent}  for (int q_ = ct; q_ < {n}; q_ += {nct}) {{")
            w(f"{indent}    const int kk = q_ / {rr * cc}, rem_ = q_ - kk * {rr * cc};")
            w(f"{indent}    const int r_ = rem_ / {cc} + ({li}), c_ = rem_ % {cc} + ({lj});")

            def rd(name, di, dj):
                hb = v.hbox[name]
                return (f"((const {ctype[name]}*)(sb + {v.offs[name]}))"
                        f"[(kk * {rows + hb.rows_extra} + (r_ + {di - hb.lo_i})) * {hb.cols}"
                        f" + (c_ + {dj - hb.bstart})]")
            w(f"{indent}    double mv_;")
            codegen_prologue.emit_stage_value(sp.pro, t, rd, ctype, out, indent + "    ", "mv_")
            w(f"{indent}    mb_[q_] = ({ctype[t]})mv_;")
            w(f"{indent}  }}")
            w(f"{indent}}}")
        w(f'{indent}asm volatile("bar.sync 1, {nct};" ::: "memory");')

    def prologue_batch(indent):
        """The fused prologue for all KB levels of a full ring stage up front
        (independent of the recurrence: the scheduler can overlap it)."""
        if v.mat:
            coop_phase(indent)
        for f in sp.pro.exports:
            w(f"{indent}double pv_{f}[{KB}];")
        w(f"{indent}#pragma unroll")
        w(f"{indent}for (int kk = 0; kk < {KB}; ++kk) {{")
        vals = codegen_prologue.emit_point(sp.pro, prologue_rd(True), ctype, out, indent + "  ",
                                           mat_read=mat_reads(), lane=pro_lane)
        for f, var in vals.items():
            w(f"{indent}  pv_{f}[kk] = {var};")
        w(f"{indent}}}")

    def forward_level(ctx, indent, group=None, tier=None, batched=False):
        """group: index of the statically known interval group (None =
        dispatch per level); tier: "tmem" / "smem" (None = per-level);
        batched: the prologue values were computed by prologue_batch."""
        for f in tracked_f:
            w(f"{indent}double cur_{f} = GTS_NAN;")
        if PW and ctx.ring:
            # written by the prologue warps over this stage's halo boxes
            ctx.pro_vals = {f: f"pvs_{f}[kk * {rows * TJ}]" for f in sp.pro.exports}
        elif batched:
            ctx.pro_vals = {f: f"pv_{f}[kk]" for f in sp.pro.exports}
        elif sp.pro is not None:
            # the fused PARALLEL prologue at this thread's (i, j, k)
            w(f"{indent}// fused prologue ({', '.join(sp.pro.exports)})")
            # the exact-division replay reads global memory at clamped columns:
            # a lane past the domain's edge would hand its neighbour the wrong
            # value, so only ring reads (box columns = lane columns) shuffle
            ctx.pro_vals = codegen_prologue.emit_point(sp.pro, prologue_rd(ctx.ring), ctype, out, indent,
                                                       lane=pro_lane if ctx.ring else None)
        groups = [gf[group]] if group is not None else gf
        for gi, (iv, stages) in enumerate(groups):
            if group is None:
                kw = "if" if gi == 0 else "else if"
                w(f"{indent}{kw} (k >= f{gi}k0 && k < f{gi}k1) {{")
            else:
                w(f"{indent}{{")
            ctx.pool = DivPool(ctx.div_mode)
            for st in stages:
                _emit_stmt(st.body, ctx, ctype, api, indent + "  ", out)
            w(f"{indent}}}")
        if tier is None:
            w(f"{indent}if (k < TL) {{")
            store_hist(indent + "  ", "tmem")
            w(f"{indent}}} else {{")
            store_hist(indent + "  ", "smem")
            w(f"{indent}}}")
        else:
            store_hist(indent, tier)
        for f, depth in sorted(cf.items()):
            for s_ in range(depth, 1, -1):
                w(f"{indent}prev{s_}_{f} = prev{s_ - 1}_{f};")
            w(f"{indent}prev1_{f} = cur_{f};")

    for f, depth in sorted(cf.items()):
        for s_ in range(1, depth + 1):
            w(f"      double prev{s_}_{f} = GTS_NAN;")
    w("      bool bad_ = false;")
    w("      for (int kb = 0; kb < nkb; ++kb, ++it) {")
    w("        const int s = it % NST;")
    w("        const uint32_t ph = (uint32_t)(it / NST) & 1u;")
    w("        gts_mbar_wait(&full[s], ph);")
    if PW:
        w("        gts_mbar_wait(&pfull[s], ph);")
    w("        const unsigned char* sb = smem + s * STB;")
    for f, so in slot_off.items():
        w(f"        const double* const pvs_{f} = (const double*)(sb + {so}) + warp * {TJ} + lane;")
    for f in sp.streamed:
        w(f"        const {ctype[f]}* const ur_{f} = (const {ctype[f]}*)(sb + {v.offs[f]}) + warp * {TJ} + lane;")
    for f, hbx in v.hbox.items():
        w(f"        const {ctype[f]}* const uh_{f} = (const {ctype[f]}*)(sb + {v.offs[f]})"
          f" + (warp - ({hbx.lo_i})) * {hbx.cols} + (lane - ({hbx.bstart}));")
    w(f"        const int kbase = kb * {KB};")
    w(f"        const bool fullst = kbase + {KB} <= nk;")
    ctx_f = _Ctx(dtypes, sp, "f", cached_f, ctype)
    ctx_f.rows, ctx_f.kb, ctx_f.offs = rows, KB, v.offs
    ctx_f.kstride = "hs_" if split else str(rows * TJ)
    first = True
    if dbg == "streamonly":  # timing experiment: ring traffic only, no arithmetic
        w("        if (true) {")
        first = False
    for tier, tcond in (("tmem", "kbase < TL"), ("smem", "kbase >= TL")):
        for gi in range(len(gf)):
            kw = "if" if first else "} else if"
            first = False
            w(f"        {kw} (fullst && {tcond} && kbase >= f{gi}k0 && kbase + {KB} <= f{gi}k1) {{")
            if pro_batch:
                prologue_batch("          ")
            w("          #pragma unroll")
            w(f"          for (int kk = 0; kk < {KB}; ++kk) {{")
            w("            const int k = kbase + kk;")
            forward_level(ctx_f, "            ", gi, tier, batched=pro_batch)
            w("          }")
    w("        } else if (" + ("false" if dbg == "streamonly" else "true") + ") {")
    if pro_batch and v.mat:
        # one consumer barrier per stage on every path keeps the two
        # materialization sets' reuse distance safe (see coop_phase)
        w(f'          asm volatile("bar.sync 1, {nct};" ::: "memory");')
    w("          #pragma unroll")
    w(f"          for (int kk = 0; kk < {KB}; ++kk) {{")
    w("            const int k = kbase + kk;")
    w("            if (k < nk) {")
    forward_level(ctx_f, "              ")
    w("            }")
    w("          }")
    w("        }")
    w("        __syncwarp();")
    w("        if (lane == 0) gts_mbar_arrive(&empty[s]);")
    w("      }")
    # columns outside the domain (TMA zero-fill of a partial tile) never force
    # the exact replay: their values are never stored
    w("      if (__any_sync(0xffffffffu, bad_ && valid)) {")
    for f, depth in sorted(cf.items()):
        for s_ in range(1, depth + 1):
            w(f"        prev{s_}_{f} = GTS_NAN;")
    w("        for (int k = 0; k < nk; ++k) {")
    ctx_r = _Ctx(dtypes, sp, "f", cached_f, ctype)
    ctx_r.ring, ctx_r.div_mode = False, "exact"
    forward_level(ctx_r, "          ")
    w("        }")
    w("      }")
    w("      gts_tmem_wait_st();")
    w("      __syncwarp();")
    # ---------------- backward
    cb = _caches(msb, -1)
    wb = set()
    for st in msb.stages:
        wb |= writes(st.body)
    for f, depth in sorted(cb.items()):
        for s_ in range(1, depth + 1):
            w(f"      double prev{s_}_{f} = GTS_NAN;")
    cached_b = {t: 0 for t in sp.cross}
    cached_b.update({f: 0 for f in wb if f not in api})
    cached_b.update(cb)
    ctx_b = _Ctx(dtypes, sp, "b", cached_b, ctype)
    need_load = {f: any(_need_load(stg, f) for _, stg in gb) for f in wb if f in api and f in cb}

    # fused PARALLEL epilogue: level m = k - elo runs once the backward sweep
    # has produced level k (the lowest level the epilogue reads); the fields
    # it reads from the sweep sit in a register window ew_<f>_<d> = f(k + d)
    ge = _interval_groups(mse) if mse is not None else []
    D = sp.ehi - sp.elo
    we_all = set()
    for st in epi_stages:
        we_all |= writes(st.body)
    for gi, (iv, _) in enumerate(ge):
        w(f"      const int e{gi}k0 = {_bound(iv.start)}, e{gi}k1 = {_bound(iv.end)};")
    for f in sp.ewin:
        for d in range(D + 1):
            w(f"      double ew_{f}_{d} = GTS_NAN;")
    ctx_e = _EpiCtx(dtypes, sp, ctype, we_all - api)

    def epilogue_level(indent, shift_in):
        """Shift the window (``shift_in``: the new level-k values) and run the
        epilogue at level m = k - elo when it lies in [0, nk)."""
        for f in sp.ewin:
            for d in range(D, 0, -1):
                w(f"{indent}ew_{f}_{d} = ew_{f}_{d - 1};")
            w(f"{indent}ew_{f}_0 = {shift_in(f)};")
        w(f"{indent}{{ const int m_ = k - ({sp.elo});")
        w(f"{indent}  if (m_ >= 0 && m_ < nk) {{ const int k = m_;")
        for t in sorted(we_all - api):
            w(f"{indent}    double cur_{t} = GTS_NAN;")
        for gi, (iv, stages) in enumerate(ge):
            kw = "if" if gi == 0 else "else if"
            w(f"{indent}    {kw} (k >= e{gi}k0 && k < e{gi}k1) {{")
            ctx_e.pool = DivPool("branch")
            for st in stages:
                _emit_stmt(st.body, ctx_e, ctype, api, indent + "      ", out)
            w(f"{indent}    }}")
        w(f"{indent}  }}")
        w(f"{indent}}}")

    def backward_level(indent, hist_value, group=None):
        for t in sp.cross:
            w(f"{indent}const double cur_{t} = {hist_value(t)};")
        for f in sorted(wb):
            if f in api:
                if f in cb:
                    if need_load[f]:
                        w(f"{indent}double cur_{f} = ((double)GTS_AT(p.f_{f}, ic, jc, k));")
                    else:
                        w(f"{indent}double cur_{f};")
            else:
                w(f"{indent}double cur_{f} = GTS_NAN;")
        groups = [gb[group]] if group is not None else gb
        for gi, (iv, stages) in enumerate(groups):
            if group is None:
                kw = "if" if gi == 0 else "else if"
                w(f"{indent}{kw} (k >= b{gi}k0 && k < b{gi}k1) {{")
            else:
                w(f"{indent}{{")
            ctx_b.pool = DivPool("branch")
            for st in stages:
                _emit_stmt(st.body, ctx_b, ctype, api, indent + "  ", out)
            w(f"{indent}}}")
        for f, depth in sorted(cb.items()):
            for s_ in range(depth, 1, -1):
                w(f"{indent}prev{s_}_{f} = prev{s_ - 1}_{f};")
            w(f"{indent}prev1_{f} = cur_{f};")
        if mse is not None:
            epilogue_level(indent, lambda f: f"cur_{f}")

    if dbg in ("fwdonly", "streamonly"):
        w("      if (nk > 100000) {")
    # shared-memory tier: levels [TL, nk), visited first, in chunks of 4
    def from_smem(t):
        return f"(double)((const {ctype[t]}*)(hist + (size_t)(k - TL) * {hb * nct} + {hoff[t]}))[ct]"

    w("      if (nk > TL) {")
    w("        for (int c4 = (nk - 1 - TL) / 4; c4 >= 0; --c4) {")
    w("          const int klo = TL + 4 * c4, khi = klo + 3;")
    first = True
    for gi in range(len(gb)):
        kw = "if" if first else "} else if"
        first = False
        w(f"          {kw} (khi < nk && klo >= b{gi}k0 && khi < b{gi}k1) {{")
        w("            #pragma unroll")
        w("            for (int r = 3; r >= 0; --r) {")
        w("              const int k = klo + r;")
        backward_level("              ", from_smem, gi)
        w("            }")
    w("          } else {")
    w("            #pragma unroll")
    w("            for (int r = 3; r >= 0; --r) {")
    w("              const int k = klo + r;")
    w("              if (k < nk) {")
    backward_level("                ", from_smem)
    w("              }")
    w("            }")
    w("          }")
    w("        }")
    w("      }")
    # TMEM tier: batches of B levels (32 words per tcgen05.ld), double-buffered
    if 32 % wl:
        raise NotImplementedError("history words per level must divide 32")
    B = 32 // wl

    def from_regs(t):
        base = f"r * {wl} + {sp.offsets[t]}"
        if sp.words[t] == 2:
            return f"__hiloint2double((int)hb_[{base} + 1], (int)hb_[{base}])"
        return f"(double)__uint_as_float(hb_[{base}])"

    w("      {")
    w("        const int ktop = (nk < TL ? nk : TL) - 1;")
    w("        if (ktop >= 0) {")
    w("          uint32_t hb_[32], nb_[32];")
    w(f"          int bi = ktop / {B};")
    w("          gts_tmem_ld32(tl + (uint32_t)(bi * 32), nb_);")
    w("          gts_tmem_wait_ld32(nb_);")
    w("          for (; bi >= 0; --bi) {")
    w("            #pragma unroll")
    w("            for (int q = 0; q < 32; ++q) hb_[q] = nb_[q];")
    w("            if (bi > 0) gts_tmem_ld32(tl + (uint32_t)((bi - 1) * 32), nb_);")
    w(f"            const int klo = bi * {B}, khi = klo + {B - 1};")
    first = True
    for gi in range(len(gb)):
        kw = "if" if first else "} else if"
        first = False
        w(f"            {kw} (khi <= ktop && klo >= b{gi}k0 && khi < b{gi}k1) {{")
        w("              #pragma unroll")
        w(f"              for (int r = {B - 1}; r >= 0; --r) {{")
        w("                const int k = klo + r;")
        backward_level("                ", from_regs, gi)
        w("              }")
    w("            } else {")
    w("              #pragma unroll")
    w(f"              for (int r = {B - 1}; r >= 0; --r) {{")
    w("                const int k = klo + r;")
    w("                if (k <= ktop) {")
    backward_level("                  ", from_regs)
    w("                }")
    w("              }")
    w("            }")
    w("            gts_tmem_wait_ld32(nb_);")
    w("          }")
    w("        }")
    w("      }")
    if mse is not None and sp.elo < 0:
        # epilogue levels whose lowest read lies below level 0
        w(f"      for (int k = -1; k >= {sp.elo}; --k) {{")
        epilogue_level("        ", lambda f: "GTS_NAN")
        w("      }")
    if dbg in ("fwdonly", "streamonly"):
        w("      }")
    if _MIRROR and not _MIRROR_INLINE:
        # gen_options mirror: the tile's columns that lie in a neighbour's halo
        # (up to 3: i-face, j-face, corner) send their finished column of the
        # mirrored field there (peer stores), re-read from the tile's own
        # stores; kept out of the level loops so they keep their registers
        t_ = ctype[_MIRROR]
        w("      {")
        w(f"        {t_}* mp0_ = nullptr; {t_}* mp1_ = nullptr; {t_}* mp2_ = nullptr;")
        w("        long long mk0_ = 0, mk1_ = 0, mk2_ = 0;")
        w("        int nm_ = 0;")
        w("        if (valid) {")
        w("          for (int d = 0; d < p.mir.n; ++d) {")
        w("            if (i < p.mir.i0[d] || i >= p.mir.i1[d] || j < p.mir.j0[d] || j >= p.mir.j1[d]) continue;")
        w(f"            {t_}* const q_ = p.mir.base[d] + (long long)i * p.mir.si[d] + (long long)j * p.mir.sj[d];")
        w("            if (nm_ == 0) { mp0_ = q_; mk0_ = p.mir.sk[d]; }")
        w("            else if (nm_ == 1) { mp1_ = q_; mk1_ = p.mir.sk[d]; }")
        w("            else { mp2_ = q_; mk2_ = p.mir.sk[d]; }")
        w("            ++nm_;")
        w("          }")
        w("        }")
        # lane-parallel over levels: the warp takes its boundary columns up to 8
        # at a time, every lane loads levels lane, lane+32, lane+64 of each
        # (one round of independent loads), then stores them to the targets
        w(f"        const {t_}* const src_ = colp_{_MIRROR};")
        w(f"        const long long sk_ = p.f_{_MIRROR}.sk;")
        w("        __syncwarp();  // the column owners' stores before other lanes re-read them")
        w("        unsigned bm_ = __ballot_sync(0xffffffffu, nm_ > 0);")
        w("        while (bm_) {")
        w("          int cl_[8];")
        w("          #pragma unroll")
        w("          for (int c = 0; c < 8; ++c) { cl_[c] = bm_ ? __ffs(bm_) - 1 : -1; bm_ &= bm_ ? bm_ - 1 : 0u; }")
        w("          for (int k0 = 0; k0 < nk; k0 += 96) {")
        w(f"            {t_} v_[8][3];")
        w("            #pragma unroll")
        w("            for (int c = 0; c < 8; ++c) {")
        w("              if (cl_[c] < 0) break;")
        w(f"              const {t_}* const s_ = ({t_}*)__shfl_sync(0xffffffffu, (unsigned long long)src_, cl_[c]);")
        w("              #pragma unroll")
        w("              for (int m = 0; m < 3; ++m) {")
        w("                const int k = k0 + lane + 32 * m;")
        w("                if (k < nk) v_[c][m] = s_[(long long)k * sk_];")
        w("              }")
        w("            }")
        w("            #pragma unroll")
        w("            for (int c = 0; c < 8; ++c) {")
        w("              if (cl_[c] < 0) break;")
        w(f"              {t_}* const q0_ = ({t_}*)__shfl_sync(0xffffffffu, (unsigned long long)mp0_, cl_[c]);")
        w(f"              {t_}* const q1_ = ({t_}*)__shfl_sync(0xffffffffu, (unsigned long long)mp1_, cl_[c]);")
        w(f"              {t_}* const q2_ = ({t_}*)__shfl_sync(0xffffffffu, (unsigned long long)mp2_, cl_[c]);")
        w("              const long long m0_ = __shfl_sync(0xffffffffu, mk0_, cl_[c]);")
        w("              const long long m1_ = __shfl_sync(0xffffffffu, mk1_, cl_[c]);")
        w("              const long long m2_ = __shfl_sync(0xffffffffu, mk2_, cl_[c]);")
        w("              #pragma unroll")
        w("              for (int m = 0; m < 3; ++m) {")
        w("                const long long k = k0 + lane + 32 * m;")
        w("                if (k >= nk) break;")
        w("                q0_[k * m0_] = v_[c][m];")
        w("                if (q1_) q1_[k * m1_] = v_[c][m];")
        w("                if (q2_) q2_[k * m2_] = v_[c][m];")
        w("              }")
        w("            }")
        w("          }")
        w("        }")
        w("      }")
    w("      __syncwarp();")
    w("    }")
    w("  }")
    w("  gts_tmem_fence_before_sync();")
    w("  __syncthreads();")
    w(f"  if (warp == 0) {{ gts_tmem_fence_after_sync(); gts_tmem_dealloc<{512 // v.cps}>(tbase); }}")
    w("}")

    def call(vi):
        tm_args = ", ".join(f"tm_{f}[{vi}]" for f in tm_fields)
        if not split:
            return [
                f"const int tiles_j = (int)((nj + {TJ - 1}) / {TJ});",
                f"const int ntiles = tiles_j * (int)((ni + {rows - 1}) / {rows});",
                f"int grid = {v.cps} * gts_sm_count(); if (grid > ntiles) grid = ntiles;",
                f"static bool attr_{kn} = false;",
                f"if (!attr_{kn}) {{ cudaFuncSetAttribute({kn}, cudaFuncAttributeMaxDynamicSharedMemorySize, {v.smem_bytes}); attr_{kn} = true; }}",
                f"gts_launch_pdl({kn}, dim3(grid), dim3({threads}), {v.smem_bytes}, st, p, {tm_args}, tiles_j, ntiles);",
            ]
        lines = [
            f"const int tiles_j = (int)((nj + {TJ - 1}) / {TJ});",
            f"GtsColSplit cs_ = gts_col_split((int)ni, (int)nj, {rows}, gts_sm_count());",
        ]
        for f in tm_fields:
            e = 8 if dtypes[f] == ir.F64 else 4
            lines.append(f"CUtensorMap tm2_{f} = tm_{f}[{vi}];")
            lines.append(
                f"if (cs_.h2 > 0 && !gts_make_tmap_3d(&tm2_{f}, (const void*)p.f_{f}.p, {e}, nj, ni, nk,"
                f" p.f_{f}.si, p.f_{f}.sj, p.f_{f}.sk, {TJ}, (unsigned)cs_.h2, {v.kb}))"
                f" cs_ = {{tiles_j * (int)((ni + {rows - 1}) / {rows}), 0, 0, tiles_j * (int)((ni + {rows - 1}) / {rows})}};")
        tm2_args = ", ".join(f"tm2_{f}" for f in tm_fields)
        lines += [
            "int grid = gts_sm_count(); if (grid > cs_.ntiles) grid = cs_.ntiles;",
            f"static bool attr_{kn} = false;",
            f"if (!attr_{kn}) {{ cudaFuncSetAttribute({kn}, cudaFuncAttributeMaxDynamicSharedMemorySize, {v.smem_bytes}); attr_{kn} = true; }}",
            f"gts_launch_pdl({kn}, dim3(grid), dim3({threads}), {v.smem_bytes}, st, p, {tm_args}, {tm2_args},"
            " tiles_j, cs_.ntiles, cs_.n1, cs_.isplit, cs_.h2 > 0 ? cs_.h2 : 1);",
        ]
        return lines

    return out, None, call


def _emit_prologue_warps(w, out, sp, v, ctype, ncw, PW, rows, slot_off):
    """Prologue warps: per ring stage, wait for its boxes, evaluate the fused
    prologue at the tile's rows x 32 columns x KB levels (rows / PW rows per
    warp, one column per lane), then -- after every prologue warp has read
    the halo boxes (named barrier 3) -- store the exports over them as
    binary64 slots [kk][row][lane] and arrive on pfull[s].  The consumers
    release the stage (empty[s]) only after reading the slots, so the next
    TMA fill cannot race them; the proxy fence orders these generic stores
    before that async-proxy overwrite."""
    rpw = rows // PW
    kb = v.kb
    w(f"  }} else if (warp > {ncw}) {{")
    w(f"    const int pw_ = warp - {ncw + 1};")
    w("    int it = 0;")
    w("    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {")
    w("      for (int kb = 0; kb < nkb; ++kb, ++it) {")
    w("        const int s = it % NST;")
    w("        gts_mbar_wait(&full[s], (uint32_t)(it / NST) & 1u);")
    w("        unsigned char* const sbw = smem + s * STB;")
    for f in sp.pro.exports:
        w(f"        double ov_{f}[{kb}][{rpw}];")
    for rr in range(rpw):
        w("        {")
        w(f"          const int prow = pw_ * {rpw} + {rr};")
        for f, hbx in v.hbox.items():
            w(f"          const {ctype[f]}* const uh_{f} = (const {ctype[f]}*)(sbw + {v.offs[f]})"
              f" + (prow - ({hbx.lo_i})) * {hbx.cols} + (lane - ({hbx.bstart}));")
        w("          #pragma unroll")
        w(f"          for (int kk = 0; kk < {kb}; ++kk) {{")

        def rd(name, di, dj):
            hbx = v.hbox[name]
            off = di * hbx.cols + dj if isinstance(dj, int) else f"{di * hbx.cols} + {dj}"
            return f"uh_{name}[kk * {(rows + hbx.rows_extra) * hbx.cols} + {off}]"
        vals = codegen_prologue.emit_point(sp.pro, rd, ctype, out, "            ")
        for f, var in vals.items():
            w(f"            ov_{f}[kk][{rr}] = {var};")
        w("          }")
        w("        }")
    w(f'        asm volatile("bar.sync 3, {32 * PW};" ::: "memory");  // halo boxes read by every prologue warp')
    for f, so in slot_off.items():
        w(f"        {{ double* const o_ = (double*)(sbw + {so}) + lane;")
        for rr in range(rpw):
            for kk in range(kb):
                w(f"          o_[({kk} * {rows} + pw_ * {rpw} + {rr}) * {TJ}] = ov_{f}[{kk}][{rr}];")
        w("        }")
    w("        gts_fence_proxy_async();")
    w("        __syncwarp();")
    w("        if (lane == 0) gts_mbar_arrive(&pfull[s]);")
    w("      }")
    w("    }")


class _EpiCtx(_MemCtx):
    """Reads inside the fused epilogue: backward-sweep outputs from the
    register window, its own temporaries from cur_*, pure inputs from
    global memory at (ic, jc, k + dk)."""

    def __init__(self, dtypes, sp: ThomasSpec, ctype: dict, local: set):
        super().__init__(dtypes)
        self.sp, self.ctype, self.local = sp, ctype, set(local)
        self.cached = {t: 0 for t in local}  # _emit_stmt keeps cur_<t> for these

    def addr(self, name, off):
        di, dj, dk = off
        kk = f"(k{dk:+d})" if dk else "k"
        return f"GTS_AT(p.f_{name}, ic, jc, {kk})"

    def read(self, name, off):
        if name in self.sp.ewin:
            return f"ew_{name}_{off[2] - self.sp.elo}"
        if name in self.local:
            return f"cur_{name}"
        return super().read(name, off)


class _PrefCtx(_Ctx):
    """_Ctx with a per-sweep name prefix for the k-cache chains."""

    def __init__(self, dtypes, sp, phase, cached, ctype, prefix):
        super().__init__(dtypes, sp, phase, cached, ctype)
        self.prefix = prefix

    def read(self, name, off):
        r = super().read(name, off)
        if r.startswith("prev"):
            return self.prefix + r[4:]
        return r
