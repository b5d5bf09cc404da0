"""Fused PARALLEL template: one streaming tile kernel for a group of stages.

Instantiates hdiff-class PARALLEL multistages (stencilforge
``kernels/hdiff.gts:3-15``: Laplacian -> limited fluxes -> update) as one
persistent sm_100a kernel in which every api field crosses HBM once:

* tile = one k-plane x (NW*RI rows) x (32*VJ columns); 4 warps per CTA,
  several CTAs per SM, a static round-robin over tiles;
* each input field's tile plus its halo (the field extent from
  ``analysis.compute_extents``, ``analysis.py:451-496``) is brought into
  shared memory by ONE TMA box load (``cp.async.bulk.tensor.3d``) into a
  double buffer, the next tile's box in flight while this one computes;
* each warp streams its RI-row strip along i; lane l owns VJ consecutive
  j columns.  Every stage is computed at its leading row (row + its i-extent
  ``hi``) over its column span (VJ columns + its j-extent), so temporaries
  live in small rolling register windows -- recomputed on the horizontal
  halo exactly as the extent analysis prescribes, never stored;
* outputs are written straight from registers.

Semantics: within a fused group every temporary has a single writer and
every read of a group-written api field is at the reader's own point
(lowering._fuse_parallel), so executing all stages per point in program
order equals the reference's whole-slab-per-stage order (``vec.py:160-162``).
Reads the streaming scheme does not cover (vertical offsets, arena
temporaries) go to global memory directly.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from ._host import ir
from .codegen import DivPool, _bound, c_float, emit_cond, emit_expr, emit_f32_rounded  # noqa: F401
from .lowering import always_writes, reads, writes

NW = 4  # warps per CTA
RI = 8  # rows per warp strip
VJ = 4  # columns per lane
TJ = 32 * VJ  # columns per tile
TI = NW * RI  # rows per tile
SMEM_BUDGET = 110 * 1024  # per CTA
NBUF = 1  # tile buffers per CTA: latency is hidden across the CTAs of an SM


@dataclass
class Win:
    name: str
    kind: str  # "temp" (register window fed by a stage) | "stream" (TMA tile) | "own" (api written, own point)
    rlo: int = 0  # rows relative to the step row
    rhi: int = 0
    clo: int = 0  # columns relative to the lane's first column
    chi: int = 0
    producer: int = -1
    # stream geometry
    box_cols: int = 0
    box_rows: int = 0
    cshift: int = 0  # the map base column (lo_j - cshift) is 16-B aligned
    bstart: int = 0  # box start column relative to the tile's first column
    smem_off: int = 0
    esize: int = 8


@dataclass
class Geo:
    stages: list
    ext: list  # per stage (li, hi, lj, hj)
    wins: dict = field(default_factory=dict)
    min_step: int = 0
    buf_bytes: int = 0  # one buffer (all streamed fields)
    rot: int = 0  # emission-time step counter (window rotation)
    buffered: set = field(default_factory=set)  # api outputs stored per row at step end


def _phys(geo, wv, d: int) -> int:
    """Rotating register windows: logical row d of a window lives in physical
    row (d + step) mod depth, so sliding the window costs no register moves
    in the fully unrolled step sequence."""
    depth = wv.rhi - wv.rlo + 1
    return (d + geo.rot) % depth


def _cn(col: int) -> str:
    return f"m{-col}" if col < 0 else str(col)


def _stage_ext(st):
    e = st.compute_extent
    return (e.lo[0], e.hi[0], e.lo[1], e.hi[1])


def analyse(plan, kplan, dtypes: dict) -> Geo:
    impl = plan.impl
    api = {f.name for f in impl.api_fields}
    stages = [r.stage for r in kplan.stages]
    ext = [_stage_ext(st) for st in stages]
    geo = Geo(stages, ext)
    local = set(kplan.local_temps)
    written = set()
    for si, st in enumerate(stages):
        li, hi, lj, hj = ext[si]
        for acc in reads(st.body):
            di, dj, dk = acc.offset
            name = acc.field
            if dk != 0:
                continue  # vertical reads of pure inputs: direct loads
            if name in local:
                kind = "temp"
            elif name in written and name in api:
                kind = "own"
            elif name in api and all(name not in writes(s2.body) for s2 in stages):
                kind = "stream"
            else:
                continue  # arena temporaries / other: direct loads
            rows = (hi + di, hi + di)
            cols = (lj + dj, VJ - 1 + hj + dj)
            wv = geo.wins.get(name)
            if wv is None:
                wv = geo.wins[name] = Win(name, kind, rows[0], rows[1], cols[0], cols[1])
            else:
                wv.rlo, wv.rhi = min(wv.rlo, rows[0]), max(wv.rhi, rows[1])
                wv.clo, wv.chi = min(wv.clo, cols[0]), max(wv.chi, cols[1])
        for f in writes(st.body):
            written.add(f)
            if f in geo.wins and geo.wins[f].kind == "temp" and geo.wins[f].producer < 0:
                geo.wins[f].producer = si
    for si, st in enumerate(stages):
        for f in writes(st.body):
            if f in local:
                wv = geo.wins.get(f)
                if wv is None:
                    geo.wins[f] = Win(f, "temp", 0, 0, 0, 0, producer=si)
                else:
                    wv.producer = si
    for name, wv in geo.wins.items():
        if wv.kind == "temp":
            li, hi, lj, hj = ext[wv.producer]
            # the window keeps rows [rlo, hi] of the producer's output
            wv.rhi = hi
            wv.rlo = min(wv.rlo, hi)
            wv.clo = min(wv.clo, lj)
            wv.chi = max(wv.chi, VJ - 1 + hj)
    geo.min_step = min(li - hi for (li, hi, lj, hj) in ext)
    writers: dict = {}
    for si, st in enumerate(stages):
        for f in writes(st.body):
            writers.setdefault(f, []).append(si)
    for f, ws in writers.items():
        if f in api and len(ws) == 1 and ext[ws[0]] == (0, 0, 0, 0) and f in always_writes(stages[ws[0]].body):
            geo.buffered.add(f)
    off = 0
    for name, wv in sorted(geo.wins.items()):
        if wv.kind != "stream":
            continue
        if PREFETCH:
            # one extra row slot: each step loads the row the NEXT step needs,
            # so shared-memory load latency overlaps a whole step of arithmetic
            wv.rhi += PREFETCH
        e = 8 if dtypes[name] == ir.F64 else 4
        wv.esize = e
        align = 16 // e
        lo_j = plan.impl.field_extent(name).lo[1]
        wv.cshift = lo_j % align  # map base column lo_j - cshift is 16-B aligned
        mb = lo_j - wv.cshift
        # TMA boxes must start on a 16-B boundary of the inner dimension:
        # round the box start down onto the map's 16-B grid
        wv.bstart = mb + ((wv.clo - mb) // align) * align
        ncols = (TJ - VJ + wv.chi) - wv.bstart + 1
        ncols = -(-ncols // align) * align
        wv.box_cols = ncols
        wv.box_rows = TI + (wv.rhi - wv.rlo) - geo.min_step
        wv.smem_off = off
        off += wv.box_cols * wv.box_rows * e
        off = -(-off // 128) * 128
    geo.buf_bytes = off
    return geo


def eligible(plan, kplan, dtypes: dict):
    geo = analyse(plan, kplan, dtypes)
    for st in geo.stages:
        for acc in reads(st.body):
            if acc.offset[2] != 0 or acc.field not in geo.wins:
                return None  # vertical offsets / arena reads: per-stage kernels
    if not any(w.kind == "stream" for w in geo.wins.values()):
        return None
    for w in geo.wins.values():
        if w.kind == "stream" and (w.box_cols > 256 or w.box_rows > 256):
            return None
    if NBUF * geo.buf_bytes + 64 > SMEM_BUDGET:
        return None
    return geo


class _Ctx:
    """Read spelling inside one (row-offset, column) point of a stage."""

    pool = None

    def __init__(self, geo: Geo, ctype: dict, stage_hi: int, col: int):
        self.geo, self.ctype, self.hi, self.col = geo, ctype, stage_hi, col

    f32x = True  # binary32-exact rewrites for f32 storage (codegen.emit_f32)

    def read_f32(self, name, off):
        """Float spelling of an f32 field / temporary (None: not binary32)."""
        if not self.f32x or self.ctype.get(name) != "float":
            return None
        di, dj, dk = off
        wv = self.geo.wins.get(name)
        if wv is not None and dk == 0:
            row = _phys(self.geo, wv, self.hi + di - wv.rlo)
            return f"wf_{name}[{row}][{self.col + dj - wv.clo}]"
        return f"GTS_AT(p.f_{name}, (r + {self.hi + di}), (jl + {self.col + dj}), (kk + {dk}))"

    def read(self, name, off):
        di, dj, dk = off
        wv = self.geo.wins.get(name)
        if wv is not None and dk == 0:
            row = _phys(self.geo, wv, self.hi + di - wv.rlo)
            c = self.col + dj - wv.clo
            return f"w_{name}[{row}][{c}]"
        # direct global load at the point (row r + hi + di, column j + col + dj)
        return (f"((double)GTS_AT(p.f_{name}, (r + {self.hi + di}), "
                f"(jl + {self.col + dj}), (kk + {dk})))")


def _emit_point(stmt, ctx: _Ctx, ctype, api: set, out: list, indent: str, local: set,
                geo: Geo) -> None:
    """Stage body at one (row, column) point; writes go to the window slot of
    a temp / own-point api field, api stores are guarded by validity."""
    pool = ctx.pool
    if isinstance(stmt, ir.Assign):
        name = stmt.target.field
        f32 = ctx.f32x and ctype[name] == "float"
        fv = emit_f32_rounded(stmt.value, ctx) if f32 else None
        if fv is not None:
            # one binary32 instruction gives the narrowed value exactly
            pool.flush(indent, out)
            out.append(f"{indent}{{ const float vf_ = {fv};")
            sv = "vf_"
        else:
            value = emit_expr(stmt.value, ctx)
            pool.flush(indent, out)
            out.append(f"{indent}{{ const double v_ = {value};")
            if f32:
                out.append(f"{indent}  const float vf_ = (float)v_;")
                sv = "vf_"
            else:
                sv = f"({ctype[name]})(v_)"
        wv = geo.wins.get(name)
        if wv is not None and wv.kind in ("temp", "own"):
            row = _phys(geo, wv, ctx.hi - wv.rlo)
            c = ctx.col - wv.clo
            if f32:
                out.append(f"{indent}  wf_{name}[{row}][{c}] = vf_;")
                out.append(f"{indent}  w_{name}[{row}][{c}] = (double)vf_;")
            else:
                out.append(f"{indent}  w_{name}[{row}][{c}] = (double)({ctype[name]})(v_);")
        if name in api and name in geo.buffered:
            out.append(f"{indent}  o_{name}[{ctx.col}] = {sv};")
        elif name in api:
            out.append(f"{indent}  if (ok_{_cn(ctx.col)}) GTS_AT(p.f_{name}, r, (jl + {ctx.col}), kk) = {sv};")
        elif name in ctx.arena:
            # arena copy for later launches: every point of the stage's extent
            li, hi, lj, hj = ctx.stage_ext
            out.append(f"{indent}  if ((r + {hi}) < ni + {hi} && (jl + {ctx.col}) >= {lj} && (jl + {ctx.col}) < nj + {hj})"
                       f" GTS_AT(p.f_{name}, (r + {hi}), (jl + {ctx.col}), kk) = {sv};")
        out.append(f"{indent}}}")
        pool.invalidate(name)
        return
    if isinstance(stmt, ir.If):
        cond = emit_cond(stmt.cond, ctx)
        pool.flush(indent, out)
        out.append(f"{indent}if ({cond}) {{")
        pool.depth += 1
        for s in stmt.then_body:
            _emit_point(s, ctx, ctype, api, out, indent + "  ", local, geo)
        if stmt.else_body:
            out.append(f"{indent}}} else {{")
            for s in stmt.else_body:
                _emit_point(s, ctx, ctype, api, out, indent + "  ", local, geo)
        pool.depth -= 1
        out.append(f"{indent}}}")
        return
    raise TypeError(type(stmt).__name__)


PREFETCH = 0  # gen_options pf_prefetch: stream rows loaded this many steps early
SWZ = False  # gen_options pf_swz: lane-alternating paired row loads (bank spreading)
PDL = "off"  # gen_options pf_pdl: programmatic dependent launch off | early | late
FRAME = False  # frame variant: the launch enumerates only the tiles outside an inner tile rectangle
FASTDIV = True  # tile index division by multiply-high (gts_div_c) instead of the XU-pipe division
MIRROR = None  # gen_options mirror: the buffered api output also stored into neighbour halo boxes
L2PF0 = 0  # gen_options pf_l2pf0: with PDL, this many of the CTA's first tiles prefetched into L2 before the wait
TMAST = False  # gen_options pf_tmastore: outputs staged per warp strip and written by one TMA bulk store
DEFAULTS = {"pf_nw": 4, "pf_ri": 8, "pf_vj": 4, "pf_nbuf": 1, "pf_prefetch": 0, "pf_swz": 0, "pf_pdl": "off",
            "pf_frame": 0, "pf_fastdiv": 1, "pf_l2pf0": 0, "pf_tmastore": 0}
# Measured defaults per element size (profiles/sweep_hdiff_r1.md, hdiff
# 256x256x80 on one B200, CUDA-graph timed):
#  f64: 16x128 tiles, double-buffered TMA boxes: 16.9 us vs 18.1 us for
#       32x128 single-buffered (HBM-bound; shorter tiles shrink the tail);
#  f32: 16x128 tiles with 2 warps x 8 rows, double-buffered: FP64-pipe bound
#       (f64 arithmetic on f32 storage), so fewer halo recomputations win.
#  pf_prefetch (rows loaded one step early) + pf_swz (bank-spread row loads):
#       interleaved A/B (tools/abtest.py, medians of 5): f64 256^2 17.00 -> 16.59 us,
#       512x1024 112.3 -> 113.0 us (noise); f32 prefetch alone 15.68 -> 15.12 us
#       (f32 with pf_swz: 17.6 us, so not for f32).
#  f64 then 2 warps per CTA (8x128 tiles): 16.52 -> 16.07 us at 256^2, 112.6 -> 112.1
#       at 512x1024 (tools/abtest.py); 1 or 3 warps, 6- or 8-row strips, 1 or 3
#       buffers all measured slower.
#  f64 pf_pdl "late" (dependent launch triggered at each CTA's last tile): 16.14 ->
#       15.97 us at 256^2, 6.13 -> 5.98 us at 128^2x64; f32 15.15 -> 15.22 (off).
#  pf_fastdiv (tile index by multiply-high instead of the XU-pipe integer
#       division; tools/abtest.py, medians of 7): f64 256^2 15.95 -> 15.79 us; f32
#       15.12 -> 16.28 us (the f32 body schedules worse around it), so off for f32.
#  pf_l2pf0 (round 2; with PDL, the CTA's first tile prefetched into L2 before
#       griddepcontrol.wait, so its first TMA load overlaps the previous grid's
#       tail; tools/abtest.py, medians of 5): f64 256^2 15.70 -> 14.93 us (2 tiles:
#       16.52), 512x1024 112.6 -> 112.1; f32 with late PDL 15.09 -> 13.72 us
#       (late PDL alone 15.12, 2 tiles 14.62).
#  pf_tmastore (round 2; each warp stages its strip's output rows in shared
#       memory and writes them with one TMA bulk tensor store per tile): f64 256^2
#       14.97 -> 14.36 us, 512x1024 112.9 -> 108.5 us; f32 13.72 -> 15.26 us (off).
GEOMETRY = {8: {"pf_nw": 2, "pf_ri": 4, "pf_vj": 4, "pf_nbuf": 2, "pf_prefetch": 1, "pf_swz": 1,
                "pf_pdl": "late", "pf_fastdiv": 1, "pf_l2pf0": 1, "pf_tmastore": 1},
            4: {"pf_nw": 2, "pf_ri": 8, "pf_vj": 4, "pf_nbuf": 2, "pf_prefetch": 1, "pf_swz": 0,
                "pf_pdl": "late", "pf_fastdiv": 0, "pf_l2pf0": 1}}


# Large binary64 domains use 4 warps per CTA: in eager launches 512x1024x80 runs
# 129.4 us with the 2-warp default and 116.4 us with 4 warps (graph replay:
# 112.5 vs 115.1); at 256^2 the 2-warp geometry wins (graph 16.07 vs 16.52,
# eager equal).  Domains of >= LARGE_POINTS points launch the LARGE variant.
LARGE = {"pf_nw": 4}
LARGE_POINTS = 16 * 1024 * 1024
# Tiny binary64 domains (< TINY_POINTS) use 2-row strips: 128^2x64 5.97 -> 5.58 us,
# but 192^2x80 12.54 -> 14.10 us (tools/abtest.py).
TINY = {"pf_ri": 2, "pf_tmastore": 0}  # bulk stores: 128^2x64 4.98 -> 5.07 us, so row stores there
TINY_POINTS = 2 * 1024 * 1024
# The frame launch of a decomposed step (decomp.DecomposedStep): after the
# halo exchange, only the tiles that touch the halo-dependent band run, in
# thin tiles (4 rows x 32 columns: 2 warps x 2 rows, 1 column per lane) so
# the band's j-sides cost 2 x 32 columns instead of 2 x 128.
FRAME_GEOMETRY = {"pf_ri": 2, "pf_vj": 1, "pf_frame": 1, "pf_swz": 0}
_LAST_ESIZE = 0


def last_esize() -> int:
    """Element size the last emit() configured for (8: binary64 group)."""
    return _LAST_ESIZE


def configure(opts, esize: int = 0) -> None:
    """Tile geometry (gen_options pf_nw / pf_ri / pf_vj / pf_nbuf; part of the
    fingerprint like the reference gen engine's tile options, gen.py:235-238).
    Unset options take the measured default of the group's smallest streamed
    element size ``esize`` (0: the generic DEFAULTS)."""
    global NW, RI, VJ, TJ, TI, NBUF, PREFETCH, SWZ, PDL, FRAME, FASTDIV, L2PF0, TMAST
    o = dict(DEFAULTS)
    o.update(GEOMETRY.get(esize, {}))
    o.update({k: v for k, v in (opts or {}).items() if k in DEFAULTS})
    NW, RI, VJ, NBUF = int(o["pf_nw"]), int(o["pf_ri"]), int(o["pf_vj"]), int(o["pf_nbuf"])
    PREFETCH = int(o["pf_prefetch"])
    SWZ = bool(int(o["pf_swz"]))
    PDL = str(o["pf_pdl"])
    FRAME = bool(int(o["pf_frame"]))
    FASTDIV = bool(int(o["pf_fastdiv"]))
    L2PF0 = int(o["pf_l2pf0"])
    TMAST = bool(int(o["pf_tmastore"]))
    TJ, TI = 32 * VJ, NW * RI


def _min_esize(plan, kplan, dtypes: dict) -> int:
    api = {f.name for f in plan.impl.api_fields}
    sizes = [8 if dtypes[a.field] == ir.F64 else 4
             for r in kplan.stages for a in reads(r.stage.body) if a.field in api]
    return min(sizes) if sizes else 0


def emit(kname: str, plan, kplan, ctype: dict, dtypes: dict, opts=None):
    global _LAST_ESIZE, MIRROR
    _LAST_ESIZE = _min_esize(plan, kplan, dtypes)
    configure(opts, _LAST_ESIZE)
    geo = eligible(plan, kplan, dtypes)
    if geo is None:
        return None
    MIRROR = (opts or {}).get("mirror") or None
    if MIRROR and not any(MIRROR in writes(st.body) for st in geo.stages):
        MIRROR = None  # another launch of the plan writes it
    if MIRROR and MIRROR not in geo.buffered:
        return None  # a mirrored output must be stored from registers once per point
    impl = plan.impl
    api = {f.name for f in impl.api_fields}
    local = set(kplan.local_temps)
    streams = [w for _, w in sorted(geo.wins.items()) if w.kind == "stream"]
    regw = [w for _, w in sorted(geo.wins.items()) if w.kind != "stream"]
    nst = len(streams)
    out: list = []
    w = out.append
    tm = ", ".join(f"const __grid_constant__ CUtensorMap tm_{s.name}" for s in streams)
    smem = NBUF * geo.buf_bytes
    bar_off = smem
    bar_bytes = -(-8 * NBUF // 16) * 16  # the NBUF full barriers
    # gen_options pf_tmastore: each warp stages its strip's rows of the buffered
    # api outputs in shared memory and stores them with ONE TMA bulk tensor
    # store per tile (cp.async.bulk.tensor ... bulk_group) instead of per-row STG
    tmast = TMAST and not FRAME and len(geo.buffered) > 0
    stg_off, stg_bytes = {}, {}
    if tmast:
        o = -(-(bar_off + bar_bytes) // 128) * 128
        for f in sorted(geo.buffered):
            e = 8 if dtypes[f] == ir.F64 else 4
            stg_off[f], stg_bytes[f] = o, RI * TJ * e  # per warp
            o += NW * RI * TJ * e
        smem = o - bar_bytes  # smem_bytes below adds the barrier slot back
    w(f"// fused PARALLEL tile kernel: {TI}x{TJ} tile per k-plane, {NW} warps x {RI} rows, "
      f"{VJ} columns/lane; streamed {[s.name for s in streams]}, register windows "
      f"{[(x.name, x.rlo, x.rhi, x.clo, x.chi) for x in regw]}")
    minb = int((opts or {}).get("pf_minb", 0))  # min resident CTAs/SM (register cap), 0 = compiler's choice
    lb = f"{32 * NW}, {minb}" if minb else f"{32 * NW}"
    frame_args = ", int fi0, int fi1, int fj0, int fj1" if FRAME else ", GtsFastDiv dvp, GtsFastDiv dvj"
    tmo = ("".join(f", const __grid_constant__ CUtensorMap tmo_{f}" for f in sorted(geo.buffered)) + ", int tmo_on"
           if tmast else "")
    w(f"__global__ void __launch_bounds__({lb}) {kname}(const __grid_constant__ GtsParams p, {tm}{tmo}, "
      f"int k0, int nkr, int tiles_i, int tiles_j, int ntiles{frame_args}) {{")
    w("  extern __shared__ __align__(1024) unsigned char smem[];")
    w(f"  uint64_t* full = (uint64_t*)(smem + {bar_off});")
    w("  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;")
    w(f"  if (threadIdx.x == 0) {{ for (int b = 0; b < {NBUF}; ++b) gts_mbar_init(&full[b], 1); gts_fence_mbar_init(); }}")
    w("  __syncthreads();")
    pdl = PDL  # off | early | late (configure(): per element size, gen_options pf_pdl)
    if pdl == "early":
        w("  gts_griddep_launch_dependents();")
    w(f"  const int ni = p.ni, nj = p.nj;")

    def tile_coords(tvar, sfx, indent):
        """k-plane and tile origin of tile index ``tvar`` (frame variant: the
        plane's tiles outside the inner rectangle [fi0, fi1) x [fj0, fj1))."""
        if FRAME:
            w(f"{indent}const int per{sfx} = tiles_i * tiles_j - (fi1 - fi0) * (fj1 - fj0);")
            w(f"{indent}const int kk{sfx} = k0 + {tvar} / per{sfx};")
            w(f"{indent}int ti{sfx}, tj{sfx};")
            w(f"{indent}gts_frame_tile({tvar} % per{sfx}, tiles_j, fi0, fi1, fj0, fj1, ti{sfx}, tj{sfx});")
            w(f"{indent}const int i0{sfx} = ti{sfx} * {TI}, j0{sfx} = tj{sfx} * {TJ};")
        elif not FASTDIV:
            w(f"{indent}const int kk{sfx} = k0 + {tvar} / (tiles_i * tiles_j);")
            w(f"{indent}const int rem{sfx} = {tvar} % (tiles_i * tiles_j);")
            w(f"{indent}const int i0{sfx} = (rem{sfx} / tiles_j) * {TI}, j0{sfx} = (rem{sfx} % tiles_j) * {TJ};")
        else:
            # tile index -> (plane, row, column) by multiply-high division (no XU)
            w(f"{indent}const int q{sfx} = gts_div_c({tvar}, dvp);")
            w(f"{indent}const int kk{sfx} = k0 + q{sfx};")
            w(f"{indent}const int rem{sfx} = {tvar} - q{sfx} * (tiles_i * tiles_j);")
            w(f"{indent}const int r{sfx}_ = gts_div_c(rem{sfx}, dvj);")
            w(f"{indent}const int i0{sfx} = r{sfx}_ * {TI}, j0{sfx} = (rem{sfx} - r{sfx}_ * tiles_j) * {TJ};")

    def issue(tvar, buf):
        w(f"    {{ const int tt = {tvar};")
        tile_coords("tt", "_", "      ")
        w(f"      gts_mbar_arrive_expect_tx(&full[{buf}], {sum(x.box_cols * x.box_rows * x.esize for x in streams)}u);")
        for s in streams:
            w(f"      gts_tma_load_3d(smem + {buf} * {geo.buf_bytes} + {s.smem_off}, &tm_{s.name}, &full[{buf}], "
              f"j0_ + ({s.bstart}) + jsh_{s.name}, i0_ + ({geo.min_step + s.rlo}) + ish_{s.name}, kk_ + ksh_{s.name});")
        w("    }")

    # the tensor maps start at the field's extent corner; shifts passed as constants
    for s in streams:
        w(f"  const int jsh_{s.name} = p.tsh_{s.name}_j, ish_{s.name} = p.tsh_{s.name}_i, ksh_{s.name} = p.tsh_{s.name}_k;")
    if pdl != "off":
        if L2PF0:
            # this CTA's first tiles into L2 while the previous grid drains (an
            # L2 prefetch is coherent with its writes: gts_tma_prefetch_l2_3d)
            w("  if (threadIdx.x == 0) {")
            w(f"    for (int m_ = 0; m_ < {L2PF0}; ++m_) {{")
            w("      const int tp = (int)blockIdx.x + m_ * (int)gridDim.x;")
            w("      if (tp >= ntiles) break;")
            tile_coords("tp", "p_", "      ")
            for s in streams:
                w(f"      gts_tma_prefetch_l2_3d(&tm_{s.name}, j0p_ + ({s.bstart}) + jsh_{s.name}, "
                  f"i0p_ + ({geo.min_step + s.rlo}) + ish_{s.name}, kkp_ + ksh_{s.name});")
            w("    }")
            w("  }")
        w("  gts_griddep_wait();  // PDL: previous grid complete before any global access")
    w("  int it = 0;")
    w("  if (threadIdx.x == 0) {")
    for m in range(NBUF - 1):
        w(f"    if ((int)blockIdx.x + {m} * (int)gridDim.x < ntiles) {{")
        issue(f"(int)blockIdx.x + {m} * (int)gridDim.x", m)
        w("    }")
    w("  }")
    w("  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {")
    if pdl == "late":
        w("    if (t + (int)gridDim.x >= ntiles) gts_griddep_launch_dependents();  // last tile of this CTA")
    w(f"    const int buf = it % {NBUF};")
    w(f"    const uint32_t ph = (uint32_t)(it / {NBUF}) & 1u;")
    w(f"    // issue tile t + {NBUF - 1} grid strides ahead into the buffer freed by the last tile")
    w(f"    if (threadIdx.x == 0 && t + {NBUF - 1} * (int)gridDim.x < ntiles) {{")
    w("      gts_fence_proxy_async();")
    for b in range(NBUF):
        w(f"      if ((it + {NBUF - 1}) % {NBUF} == {b}) {{")
        issue(f"t + {NBUF - 1} * (int)gridDim.x", b)
        w("      }")
    w("    }")
    w("    gts_mbar_wait(&full[buf], ph);")
    w("    const unsigned char* sb = smem + buf * " + str(geo.buf_bytes) + ";")
    tile_coords("t", "", "    ")

    w(f"    const int jl = j0 + lane * {VJ};")
    w(f"    const int ra = i0 + warp * {RI};")
    if MIRROR in geo.buffered:
        # the mirror boxes (gen_options mirror) this tile intersects, uniform per
        # CTA: up to 3 (a face in i, a face in j, their corner) are kept in
        # registers -- target plane pointer, row range, this lane's column mask
        # -- so a boundary row costs a few predicated stores; more (a tile
        # spanning the whole domain) take the general loop
        t_ = ctype[MIRROR]
        w("    int nmir_ = 0;")
        w(f"    {t_}* mbp_[3] = {{nullptr, nullptr, nullptr}};")
        w("    long long msi_[3] = {0, 0, 0}, msj_[3] = {0, 0, 0};")
        w("    int mi0_[3] = {0, 0, 0}, mi1_[3] = {0, 0, 0};")
        w("    unsigned mcm_[3] = {0u, 0u, 0u};")
        w("    for (int d = 0; d < p.mir.n; ++d) {")
        w(f"      if (!(i0 < p.mir.i1[d] && i0 + {TI} > p.mir.i0[d] && j0 < p.mir.j1[d] && j0 + {TJ} > p.mir.j0[d])) continue;")
        w("      unsigned cm = 0u;")
        w(f"      for (int q = 0; q < {VJ}; ++q) {{ const int c = jl + q; if (c < nj && c >= p.mir.j0[d] && c < p.mir.j1[d]) cm |= 1u << q; }}")
        for m in range(3):  # static slots (a runtime index would put the arrays in local memory)
            w(f"      {'if' if m == 0 else 'else if'} (nmir_ == {m}) {{ mbp_[{m}] = p.mir.base[d] + (long long)kk * p.mir.sk[d]; "
              f"msi_[{m}] = p.mir.si[d]; msj_[{m}] = p.mir.sj[d]; mi0_[{m}] = p.mir.i0[d]; mi1_[{m}] = p.mir.i1[d]; "
              f"mcm_[{m}] = cm; }}")
        w("      ++nmir_;")
        w("    }")
    # per-column store validity
    for c in range(VJ):
        w(f"    const bool okc_{c} = (jl + {c}) < nj;")
    # register windows
    f32x = bool((opts or {}).get("f32x", True))
    # timing experiments: "streamonly" = TMA tiles + barriers only; "nostore" = no output stores
    pf_debug = (opts or {}).get("pf_debug", "")
    for x in regw:
        w(f"    double w_{x.name}[{x.rhi - x.rlo + 1}][{x.chi - x.clo + 1}];")
        if f32x and ctype[x.name] == "float":
            w(f"    float wf_{x.name}[{x.rhi - x.rlo + 1}][{x.chi - x.clo + 1}];")
    # stream windows are read from smem directly: define accessor macros
    for s in streams:
        row_base = geo.min_step + s.rlo  # smem row 0 <-> absolute row i0 + row_base
        w(f"    const {ctype[s.name]}* const sp_{s.name} = (const {ctype[s.name]}*)(sb + {s.smem_off});")
        w(f"    double w_{s.name}[{s.rhi - s.rlo + 1}][{s.chi - s.clo + 1}];")
        if f32x and ctype[s.name] == "float":
            w(f"    float wf_{s.name}[{s.rhi - s.rlo + 1}][{s.chi - s.clo + 1}];")
    steps_lo = geo.min_step
    nsteps = RI - steps_lo  # steps r = ra + min_step .. ra + RI - 1

    # Shared-memory bank spreading: lane l reads VJ consecutive elements, so
    # with a lane stride S = VJ * esize bytes > the vector width V, lanes l
    # and l + 128/S hit the same banks in one instruction (f64: 2-way, half
    # the LDS bandwidth).  Chunks are loaded in pairs whose offsets differ by
    # V..S-V (mod S): lane groups alternate which one they load first, so one
    # instruction covers all 32 banks; selects put the values back in place.
    # Measured alone (tools/ksweep.py): f64 256^2 17.11 -> 16.77 us, 512x1024
    # 113.1 -> 116.1 us, f32 slower; with pf_prefetch it is the f64 default
    # (GEOMETRY above).
    lane_stride = {s.name: VJ * s.esize for s in streams}
    swz = {}
    for s in streams:
        S = lane_stride[s.name]
        g = 128 // S if S and 128 % S == 0 else 0
        if SWZ and g >= 1 and (g & (g - 1)) == 0 and 1 < g <= 16:
            swz[s.name] = g
    for g in sorted(set(swz.values())):
        w(f"    const int swz{g}_ = (lane / {g}) & 1;")

    def load_stream_row(s, rowidx, rel_row):
        # absolute row = r + rel_row; smem row = (r + rel_row) - (i0 + min_step + rlo);
        # 8/16-B vector loads where the layout allows (rows are 16-B multiples)
        off = s.clo - s.bstart
        ncol = s.chi - s.clo + 1
        rowexpr = f"(size_t)((r + {rel_row}) - (i0 + {geo.min_step + s.rlo})) * {s.box_cols}"
        vmax = 16 // s.esize
        chunks = []
        c = 0
        while c < ncol:
            v = vmax
            while v > 1 and not ((off + c) % v == 0 and VJ % v == 0 and c + v <= ncol):
                v //= 2
            chunks.append((c, v))
            c += v
        prow = _phys(geo, s, rowidx)
        fl = f32x and s.esize == 4
        comps = "xyzw"
        S = lane_stride[s.name]

        def assign(c, v, q):
            for k in range(v):
                w(f"        w_{s.name}[{prow}][{c + k}] = (double){q}.{comps[k]};")
                if fl:
                    w(f"        wf_{s.name}[{prow}][{c + k}] = {q}.{comps[k]};")

        # pair chunks for bank spreading
        pairs, used = [], set()
        if s.name in swz:
            for a, (ca, va) in enumerate(chunks):
                if a in used or va == 1 or va * s.esize >= S:
                    continue
                V = va * s.esize
                for b in range(a + 1, len(chunks)):
                    cb, vb = chunks[b]
                    if b in used or vb != va:
                        continue
                    d = ((cb - ca) * s.esize) % S
                    if V <= d <= S - V:
                        pairs.append((a, b))
                        used |= {a, b}
                        break
        partner = {a: b for a, b in pairs}
        for a, (c, v) in enumerate(chunks):
            idx = f"{rowexpr} + lane * {VJ} + {off + c}"
            if v == 1 and a not in used:
                w(f"      w_{s.name}[{prow}][{c}] = (double)sp_{s.name}[{idx}];")
                if fl:
                    w(f"      wf_{s.name}[{prow}][{c}] = sp_{s.name}[{idx}];")
                continue
            vt = {(8, 2): "double2", (4, 2): "float2", (4, 4): "float4"}[(s.esize, v)]
            if a in partner:
                b = partner[a]
                cb = chunks[b][0]
                sw = f"swz{swz[s.name]}_"
                dlt = cb - c
                w(f"      {{ const {vt} qa_ = *reinterpret_cast<const {vt}*>(sp_{s.name} + {idx} + {sw} * {dlt});")
                w(f"        const {vt} qb_ = *reinterpret_cast<const {vt}*>(sp_{s.name} + {idx} + (1 - {sw}) * {dlt});")
                w(f"        const {vt} q0_ = {sw} ? qb_ : qa_;")
                w(f"        const {vt} q1_ = {sw} ? qa_ : qb_;")
                assign(c, v, "q0_")
                assign(cb, v, "q1_")
                w("      }")
                continue
            if a in used:
                continue  # loaded with its partner
            w(f"      {{ const {vt} q_ = *reinterpret_cast<const {vt}*>(sp_{s.name} + {idx});")
            assign(c, v, "q_")
            w("      }")

    def emit_mirror(f):
        # gen_options mirror: the row's values inside a neighbour's halo
        # box also go there (peer stores; boundary tiles only)
        w("        if (nmir_ > 0) {")
        w("          if (nmir_ <= 3) {")
        w("            #pragma unroll")
        w("            for (int m = 0; m < 3; ++m) {")
        w("              if (m < nmir_ && r >= mi0_[m] && r < mi1_[m] && mcm_[m]) {")
        w(f"                {ctype[f]}* const mb_ = mbp_[m] + (long long)r * msi_[m];")
        for q in range(VJ):
            w(f"                if (mcm_[m] & {1 << q}u) mb_[(long long)(jl + {q}) * msj_[m]] = o_{f}[{q}];")
        w("              }")
        w("            }")
        w("          } else {")
        w("            for (int d = 0; d < p.mir.n; ++d) {")
        w("              if (r < p.mir.i0[d] || r >= p.mir.i1[d]) continue;")
        w(f"              {ctype[f]}* const mb_ = p.mir.base[d] + (long long)r * p.mir.si[d] + (long long)kk * p.mir.sk[d];")
        for q in range(VJ):
            w(f"              if (jl + {q} < nj && jl + {q} >= p.mir.j0[d] && jl + {q} < p.mir.j1[d]) "
              f"mb_[(long long)(jl + {q}) * p.mir.sj[d]] = o_{f}[{q}];")
        w("            }")
        w("          }")
        w("        }")

    if tmast:
        # the warp's staging tile is free once its previous bulk store has read it
        w('    if (tmo_on && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");')
        w("    __syncwarp();")
        for f in sorted(geo.buffered):
            w(f"    {ctype[f]}* const stg_{f} = ({ctype[f]}*)(smem + {stg_off[f]} + warp * {stg_bytes[f]});")
    # fully unrolled steps (prologue + main)
    for step in range(nsteps):
        rel = steps_lo + step  # r = ra + rel
        w(f"    {{ // step r = ra + {rel}")
        w(f"      const int r = ra + {rel};")
        geo.rot = step  # windows slide by rotation, no moves
        for f in sorted(geo.buffered):
            w(f"      {ctype[f]} o_{f}[{VJ}];")
        # load stream rows: at the first step the whole window, later the top row
        for s in streams:
            if step == 0:
                for d in range(s.rhi - s.rlo + 1):
                    load_stream_row(s, d, s.rlo + d)
            else:
                load_stream_row(s, s.rhi - s.rlo, s.rhi)
        # stages in program order; stage s computes row r + hi_s if that row is needed
        for si, st in enumerate(geo.stages):
            li, hi, lj, hj = geo.ext[si]
            # needed rows for stage s: [ra + li, ra + RI - 1 + hi]; row computed = r + hi
            if rel + hi < li or pf_debug == "streamonly":
                continue  # prologue: this stage has nothing to produce yet
            w(f"      {{ // stage {si} at row r + {hi}")
            for col in range(lj, VJ + hj):
                ctx = _Ctx(geo, ctype, hi, col)
                ctx.f32x = f32x
                ctx.pool = DivPool("branch")
                ctx.arena = set(plan.global_temps)
                ctx.stage_ext = geo.ext[si]
                w(f"        {{ const bool ok_{_cn(col)} = {'okc_' + str(col) if 0 <= col < VJ else 'false'} && (r + {hi}) < ni && {hi} == 0;")
                for f in sorted(writes(st.body) - always_writes(st.body)):
                    wv = geo.wins.get(f)
                    if wv is not None and wv.kind in ("temp", "own"):
                        # a conditionally written temporary reads as NaN where
                        # unwritten, like the reference's NaN-initialised ones
                        w(f"          w_{f}[{_phys(geo, wv, hi - wv.rlo)}][{col - wv.clo}] = GTS_NAN;")
                        if f32x and ctype[f] == "float":
                            w(f"          wf_{f}[{_phys(geo, wv, hi - wv.rlo)}][{col - wv.clo}] = __int_as_float(0x7fffffff);")
                _emit_point(st.body, ctx, ctype, api, out, "          ", local, geo)
                w("        }")
            w("      }")
        if rel >= 0 and pf_debug != "streamonly" and tmast:
            # staged rows: the strip leaves as one TMA bulk store after the steps
            w("      if (tmo_on) {")
            for f in sorted(geo.buffered):
                e = 8 if dtypes[f] == ir.F64 else 4
                if e == 8:
                    for q in range(0, VJ, 2):
                        w(f"      *reinterpret_cast<double2*>(stg_{f} + {rel * TJ} + lane * {VJ} + {q}) = "
                          f"make_double2(o_{f}[{q}], o_{f}[{q + 1}]);")
                else:
                    for q in range(0, VJ, 4):
                        w(f"      *reinterpret_cast<float4*>(stg_{f} + {rel * TJ} + lane * {VJ} + {q}) = "
                          f"make_float4(o_{f}[{q}], o_{f}[{q + 1}], o_{f}[{q + 2}], o_{f}[{q + 3}]);")
            if MIRROR in geo.buffered:
                w("      if (r < ni) {")
                emit_mirror(MIRROR)
                w("      }")
            w("      } else {")  # no store map for this layout: the row stores below
        if rel >= 0 and pf_debug != "streamonly":
            # buffered api outputs: one row of VJ values per lane, vector store
            for f in sorted(geo.buffered):
                e = 8 if dtypes[f] == ir.F64 else 4
                w(f"      if (r < ni{' && nkr < 0' if pf_debug == 'nostore' else ''}) {{")
                w(f"        {ctype[f]}* const op = &GTS_AT(p.f_{f}, r, jl, kk);")
                vec = 16 // e  # elements per 16-B vector store
                if VJ % vec == 0:
                    w(f"        if (jl + {VJ} <= nj && p.f_{f}.sj == 1 && (((uintptr_t)op) & 15) == 0) {{")
                    if e == 8:
                        for q in range(0, VJ, 2):
                            w(f"          *reinterpret_cast<double2*>(op + {q}) = make_double2(o_{f}[{q}], o_{f}[{q + 1}]);")
                    else:
                        for q in range(0, VJ, 4):
                            w(f"          *reinterpret_cast<float4*>(op + {q}) = make_float4(o_{f}[{q}], o_{f}[{q + 1}], o_{f}[{q + 2}], o_{f}[{q + 3}]);")
                    w("        } else {")
                else:  # fewer columns per lane than one vector (the frame variant): scalar stores
                    w("        {")
                for q in range(VJ):
                    w(f"          if (jl + {q} < nj) op[(long long){q} * p.f_{f}.sj] = o_{f}[{q}];")
                w("        }")
                if f == MIRROR:
                    emit_mirror(f)
                w("      }")
            if tmast:
                w("      }")
        w("    }")
    if tmast:
        w("    if (tmo_on) {")
        w('    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the staged rows, to the TMA engine')
        w("    __syncwarp();")
        w("    if (lane == 0) {")
        for f in sorted(geo.buffered):
            w(f'      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {{%1, %2, %3}}], [%4];"'
              f' :: "l"(reinterpret_cast<uint64_t>(&tmo_{f})), "r"(j0), "r"(ra), "r"(kk),'
              f' "r"(gts_smem_u32(stg_{f})) : "memory");')
        w('      asm volatile("cp.async.bulk.commit_group;" ::: "memory");')
        w("    }")
        w("    }")
    w("    __syncthreads();  // both buffers' readers done before the next prefetch reuses this one")
    w("  }")
    if tmast:
        w('  if (tmo_on && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");')
    w("}")

    smem_bytes = smem + bar_bytes
    flag = f"fz_ok_{kname.split('_')[1][1:]}"
    pre = [f"  // TMA maps of {kname}: each covers the field's required region (its extent)"]
    for s in streams:
        pre.append(f"  CUtensorMap tm_{kname}_{s.name};")
    pre.append(f"  bool {flag} = true;")
    for s in streams:
        e = s.esize
        fe = plan.impl.field_extent(s.name)
        pre += [
            f"  p.tsh_{s.name}_i = -({fe.lo[0]}); p.tsh_{s.name}_j = -({fe.lo[1]} - {s.cshift}); p.tsh_{s.name}_k = 0;",
            f"  {flag} = {flag} && gts_make_tmap_3d(&tm_{kname}_{s.name}, (const void*)&GTS_AT(p.f_{s.name}, {fe.lo[0]}, {fe.lo[1]} - {s.cshift}, 0), {e},"
            f" nj + {fe.hi[1] - fe.lo[1]} + {s.cshift}, ni + {fe.hi[0] - fe.lo[0]}, nk, p.f_{s.name}.si, p.f_{s.name}.sj, p.f_{s.name}.sk,"
            f" {s.box_cols}, {s.box_rows}, 1);",
        ]
    tm_args = ", ".join(f"tm_{kname}_{s.name}" for s in streams)
    if tmast:
        # store maps: the output's compute domain at its origin, box = one warp's strip
        for f in sorted(geo.buffered):
            e = 8 if dtypes[f] == ir.F64 else 4
            pre += [
                f"  CUtensorMap tmo_{kname}_{f};",
                f"  memset(&tmo_{kname}_{f}, 0, sizeof(CUtensorMap));",
                f"  const bool tmok_{kname}_{f} = gts_make_tmap_3d(&tmo_{kname}_{f}, (const void*)&GTS_AT(p.f_{f}, 0, 0, 0),"
                f" {e}, nj, ni, nk, p.f_{f}.si, p.f_{f}.sj, p.f_{f}.sk, {TJ}, {RI}, 1);",
            ]
        # a layout without a valid store map (16-B alignment) keeps the row stores
        tm_args += "".join(f", tmo_{kname}_{f}" for f in sorted(geo.buffered))
        tm_args += ", (int)(" + " && ".join(f"tmok_{kname}_{f}" for f in sorted(geo.buffered)) + ")"
    if FRAME:
        # inner tile rectangle: tiles whose points all lie at least the band
        # width of their side inside the domain (they need no halo cell of a
        # field of that extent); a side without a band reaches the domain edge
        # (its last partial tile included: decomp.frame_interior clips it)
        tiles = [
            "      const int tiles_i = (int)((ni + %d) / %d), tiles_j = (int)((nj + %d) / %d);" % (TI - 1, TI, TJ - 1, TJ),
            "      int fi0 = (fr_ilo + %d) / %d, fi1 = fr_ihi ? ((int)ni - fr_ihi) / %d : tiles_i;" % (TI - 1, TI, TI),
            "      int fj0 = (fr_jlo + %d) / %d, fj1 = fr_jhi ? ((int)nj - fr_jhi) / %d : tiles_j;" % (TJ - 1, TJ, TJ),
            "      if (fi1 < fi0) fi1 = fi0;",
            "      if (fj1 < fj0) fj1 = fj0;",
            "      const int nkr = k1 - k0;",
            "      if (nkr > 0 && tiles_i * tiles_j > (fi1 - fi0) * (fj1 - fj0)) {",
            "        const int ntiles = (tiles_i * tiles_j - (fi1 - fi0) * (fj1 - fj0)) * nkr;",
        ]
        targs = f"{tm_args}, k0, nkr, tiles_i, tiles_j, ntiles, fi0, fi1, fj0, fj1"
    else:
        tiles = [
            f"      const int tiles_i = (int)((ni + {TI - 1}) / {TI}), tiles_j = (int)((nj + {TJ - 1}) / {TJ});",
            "      const int nkr = k1 - k0;",
            "      if (nkr > 0) {",
            "        const int ntiles = tiles_i * tiles_j * nkr;",
        ]
        targs = f"{tm_args}, k0, nkr, tiles_i, tiles_j, ntiles, gts_fastdiv(tiles_i * tiles_j), gts_fastdiv(tiles_j)"
    launch = [
        "    {",
        f"      const int k0 = {_bound(kplan.interval.start)}, k1 = {_bound(kplan.interval.end)};",
        *tiles,
        "        static bool attr = false;",
        "        static int per_sm = 1;",
        f"        if (!attr) {{ cudaFuncSetAttribute({kname}, cudaFuncAttributeMaxDynamicSharedMemorySize, {smem_bytes});",
        f"          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, {kname}, {32 * NW}, {smem_bytes}); if (per_sm < 1) per_sm = 1; attr = true; }}",
        "        int grid = per_sm * gts_sm_count(); if (grid > ntiles) grid = ntiles;",
        (f"        gts_launch_pdl({kname}, dim3(grid), dim3({32 * NW}), {smem_bytes}, st, p, {targs});"
         if pdl != "off" else
         f"        {kname}<<<grid, {32 * NW}, {smem_bytes}, st>>>(p, {targs});"),
        "      }",
        "    }",
    ]
    return out, pre, launch

