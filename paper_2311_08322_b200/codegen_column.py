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

from dataclasses import dataclass
from typing import Optional

from ._host import ir
from .codegen import _bound, _interval_groups, _MemCtx, c_float, emit_expr  # noqa: F401
from .lowering import always_writes, reads, writes

KB = 8  # levels per TMA box
TI, TJ = 4, 32  # tile: 4 rows (one per consumer warp) x 32 contiguous columns
RING_BUDGET = 196 * 1024
MAX_STAGES = 8


@dataclass
class ThomasSpec:
    ms_f: int
    ms_b: int
    streamed: list  # api fields streamed through the TMA ring (forward reads)
    cross: list  # temps written in forward, read in backward -> TMEM
    words: dict  # temp -> 32-bit words per level
    offsets: dict  # temp -> word offset within a level
    w_level: int  # words per level
    stage_bytes: int
    offs_in_stage: dict  # streamed field -> byte offset within a ring stage
    nstages: int


def spec(plan, kplan, dtypes: dict) -> Optional[ThomasSpec]:
    impl = plan.impl
    if kplan.kind != "column" or len(kplan.multistages) != 2:
        return None
    mf, mb = kplan.multistages
    msf, msb = impl.multistages[mf], impl.multistages[mb]
    if msf.order != ir.FORWARD or msb.order != ir.BACKWARD:
        return None
    api = {f.name for f in impl.api_fields}
    temps = {t.name for t in impl.temporaries}
    wf, wb = set(), set()
    for st in msf.stages:
        wf |= writes(st.body)
    for st in msb.stages:
        wb |= writes(st.body)
    if wf & api:
        return None
    if any(f in plan.global_temps and f in wb for f in wb):
        return None  # backward temporaries must stay kernel-local
    streamed = []
    for st in msf.stages:
        for acc in reads(st.body):
            if acc.field in api:
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
    # temporaries of the forward sweep read by later launches would need the
    # arena: not supported by this template
    for t in wf:
        if t in plan.global_temps and t not in cross:
            return None
    if not streamed:
        return None
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
    return ThomasSpec(mf, mb, streamed, cross, words, offsets, max(w, 1), sb, offs, nstages)


class _Ctx(_MemCtx):
    """Field access spelling inside the TMEM column kernel."""

    def __init__(self, dtypes, sp: ThomasSpec, phase: str, cached: dict, ctype: dict):
        super().__init__(dtypes)
        self.sp, self.phase, self.cached, self.ctype = sp, phase, cached, ctype

    def addr(self, name, off):
        di, dj, dk = off
        ii = f"(ic{di:+d})" if di else "ic"
        jj = f"(jc{dj:+d})" if dj else "jc"
        kk = f"(k{dk:+d})" if dk else "k"
        return f"GTS_AT(p.f_{name}, {ii}, {jj}, {kk})"

    def read(self, name, off):
        if self.phase == "f" and name in self.sp.streamed:
            return f"((double)((const {self.ctype[name]}*)(sb + {self.sp.offs_in_stage[name]}))[(kk * {TI} + warp) * {TJ} + lane])"
        direction = 1 if self.phase == "f" else -1
        if name in self.cached and not (off[0] or off[1]):
            if off[2] == 0:
                return f"cur_{name}"
            s = -off[2] * direction
            if 1 <= s <= self.cached[name]:
                return f"prev{s}_{name}"
        return super().read(name, off)


def _emit_stmt(stmt, ctx: _Ctx, ctype, api: set, indent: str, out: list) -> None:
    if isinstance(stmt, ir.Assign):
        name = stmt.target.field
        out.append(f"{indent}{{ const double v_ = {emit_expr(stmt.value, ctx)};")
        if name in api:
            out.append(f"{indent}  if (valid) GTS_AT(p.f_{name}, i, j, k) = ({ctype[name]})(v_);")
        if name in ctx.cached or name not in api:
            out.append(f"{indent}  cur_{name} = (double)({ctype[name]})(v_);")
        out.append(f"{indent}}}")
        return
    if isinstance(stmt, ir.If):
        out.append(f"{indent}if ({emit_expr(stmt.cond, ctx)}) {{")
        for s in stmt.then_body:
            _emit_stmt(s, ctx, ctype, api, indent + "  ", out)
        if stmt.else_body:
            out.append(f"{indent}}} else {{")
            for s in stmt.else_body:
                _emit_stmt(s, ctx, ctype, api, indent + "  ", out)
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


def emit(kname: str, plan, kplan, sp: ThomasSpec, ctype: dict, dtypes: dict):
    impl = plan.impl
    api = {f.name for f in impl.api_fields}
    msf, msb = impl.multistages[sp.ms_f], impl.multistages[sp.ms_b]
    out: list = []
    w = out.append
    tm_params = ", ".join(f"const __grid_constant__ CUtensorMap tm_{f}" for f in sp.streamed)
    w(f"// TMEM column kernel: streamed {sp.streamed}, TMEM {sp.cross} ({sp.w_level} words/level),"
      f" ring {sp.nstages} x {sp.stage_bytes} B")
    w(f"__global__ void __launch_bounds__(160, 1) {kname}_tmem(const __grid_constant__ GtsParams p, "
      f"{tm_params}, int tiles_j, int ntiles) {{")
    w("  extern __shared__ __align__(1024) unsigned char smem[];")
    w(f"  constexpr int NST = {sp.nstages};")
    w(f"  constexpr unsigned STB = {sp.stage_bytes}u;")
    w("  uint64_t* full = (uint64_t*)(smem + NST * STB);")
    w("  uint64_t* empty = full + NST;")
    w("  uint32_t* tslot = (uint32_t*)(empty + NST);")
    w("  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;")
    w("  if (warp == 0) gts_tmem_alloc<512>(tslot);")
    w("  if (threadIdx.x == 0) {")
    w("    for (int s = 0; s < NST; ++s) { gts_mbar_init(&full[s], 1); gts_mbar_init(&empty[s], 4); }")
    w("    gts_fence_mbar_init();")
    w("  }")
    w("  gts_tmem_fence_before_sync();")
    w("  __syncthreads();")
    w("  gts_tmem_fence_after_sync();")
    w("  const uint32_t tbase = *tslot;")
    w("  const int nk = p.nk;")
    w(f"  const int nkb = (nk + {KB - 1}) / {KB};")
    w("  if (warp == 4) {")
    w("    if (lane == 0) {")
    for f in sp.streamed:
        w(f"      gts_prefetch_tensormap(&tm_{f});")
    w("      int it = 0;")
    w("      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {")
    w(f"        const int j0 = (t % tiles_j) * {TJ}, i0 = (t / tiles_j) * {TI};")
    w("        for (int kb = 0; kb < nkb; ++kb, ++it) {")
    w("          const int s = it % NST;")
    w("          const uint32_t ph = (uint32_t)(it / NST) & 1u;")
    w("          if (it >= NST) gts_mbar_wait(&empty[s], ph ^ 1u);")
    w("          gts_mbar_arrive_expect_tx(&full[s], STB);")
    for f in sp.streamed:
        w(f"          gts_tma_load_3d(smem + s * STB + {sp.offs_in_stage[f]}, &tm_{f}, &full[s], j0, i0, kb * {KB});")
    w("        }")
    w("      }")
    w("    }")
    w("  } else {")
    w("    const uint32_t tl = tbase + ((uint32_t)(warp * 32) << 16);")
    w("    int it = 0;")
    # interval bounds
    gf = _interval_groups(msf)
    gb = _interval_groups(msb)
    for gi, (iv, _) in enumerate(gf):
        w(f"    const int f{gi}k0 = {_bound(iv.start)}, f{gi}k1 = {_bound(iv.end)};")
    for gi, (iv, _) in enumerate(gb):
        w(f"    const int b{gi}k0 = {_bound(iv.start)}, b{gi}k1 = {_bound(iv.end)};")
    w("    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {")
    w(f"      const int j = (t % tiles_j) * {TJ} + lane, i = (t / tiles_j) * {TI} + warp;")
    w("      const bool valid = (i < p.ni) && (j < p.nj);")
    w("      const int ic = i < p.ni ? i : p.ni - 1, jc = j < p.nj ? j : p.nj - 1;")
    w("      (void)ic; (void)jc;")
    # ---------------- forward
    cf = _caches(msf, 1)
    wf = set()
    for st in msf.stages:
        wf |= writes(st.body)
    tracked_f = sorted(wf)  # every forward-written temp lives in a register per level
    for f, depth in sorted(cf.items()):
        for s in range(1, depth + 1):
            w(f"      double prev{s}_{f} = GTS_NAN;")
    w("      for (int kb = 0; kb < nkb; ++kb, ++it) {")
    w("        const int s = it % NST;")
    w("        const uint32_t ph = (uint32_t)(it / NST) & 1u;")
    w("        gts_mbar_wait(&full[s], ph);")
    w("        const unsigned char* sb = smem + s * STB;")
    w(f"        #pragma unroll 2")
    w(f"        for (int kk = 0; kk < {KB}; ++kk) {{")
    w(f"          const int k = kb * {KB} + kk;")
    w("          if (k < nk) {")
    for f in tracked_f:
        w(f"            double cur_{f} = GTS_NAN;")
    ctx_f = _Ctx(dtypes, sp, "f", {f: d for f, d in cf.items()} | {f: 0 for f in tracked_f if f not in cf}, ctype)
    for gi, (iv, stages) in enumerate(gf):
        kw = "if" if gi == 0 else "else if"
        w(f"            {kw} (k >= f{gi}k0 && k < f{gi}k1) {{")
        for st in stages:
            _emit_stmt(st.body, ctx_f, ctype, api, "              ", out)
        w("            }")
    # TMEM stores of the cross temporaries (converged, warp-uniform)
    for t in sp.cross:
        col = f"(uint32_t)(k * {sp.w_level} + {sp.offsets[t]})"
        if sp.words[t] == 2:
            w(f"            gts_tmem_store_f64(tl + {col}, cur_{t});")
        else:
            w(f"            gts_tmem_store_f32(tl + {col}, (float)cur_{t});")
    for f, depth in sorted(cf.items()):
        for s_ in range(depth, 1, -1):
            w(f"            prev{s_}_{f} = prev{s_ - 1}_{f};")
        w(f"            prev1_{f} = cur_{f};")
    w("          }")
    w("        }")
    w("        gts_fence_proxy_async();")
    w("        __syncwarp();")
    w("        if (lane == 0) gts_mbar_arrive(&empty[s]);")
    w("      }")
    w("      gts_tmem_wait_st();")
    # ---------------- backward
    cb = _caches(msb, -1)
    wb = set()
    for st in msb.stages:
        wb |= writes(st.body)
    for f, depth in sorted(cb.items()):
        for s in range(1, depth + 1):
            w(f"      double prev{s}_{f} = GTS_NAN;")
    w("      for (int k = nk - 1; k >= 0; --k) {")
    for t in sp.cross:
        col = f"(uint32_t)(k * {sp.w_level} + {sp.offsets[t]})"
        if sp.words[t] == 2:
            w(f"        uint32_t lo_{t}, hi_{t};")
            w(f"        gts_tmem_ld2(tl + {col}, lo_{t}, hi_{t});")
        else:
            w(f"        uint32_t lo_{t};")
            w(f"        gts_tmem_ld1(tl + {col}, lo_{t});")
    w("        gts_tmem_wait_ld();")
    for t in sp.cross:
        if sp.words[t] == 2:
            w(f"        const double cur_{t} = __hiloint2double((int)hi_{t}, (int)lo_{t});")
        else:
            w(f"        const double cur_{t} = (double)__uint_as_float(lo_{t});")
    for f in sorted(wb):
        if f in api:
            if f in cb:
                # current value of a cached api output: memory unless written first
                first_groups = gb
                need = any(_need_load(stg, f) for _, stg in first_groups)
                if need:
                    w(f"        double cur_{f} = ((double)GTS_AT(p.f_{f}, ic, jc, k));")
                else:
                    w(f"        double cur_{f};")
        else:
            w(f"        double cur_{f} = GTS_NAN;")
    cached_b = {t: 0 for t in sp.cross}
    cached_b.update({f: 0 for f in wb if f not in api})
    cached_b.update(cb)
    ctx_b = _Ctx(dtypes, sp, "b", cached_b, ctype)
    for gi, (iv, stages) in enumerate(gb):
        kw = "if" if gi == 0 else "else if"
        w(f"        {kw} (k >= b{gi}k0 && k < b{gi}k1) {{")
        for st in stages:
            _emit_stmt(st.body, ctx_b, ctype, api, "          ", out)
        w("        }")
    for f, depth in sorted(cb.items()):
        for s_ in range(depth, 1, -1):
            w(f"        prev{s_}_{f} = prev{s_ - 1}_{f};")
        w(f"        prev1_{f} = cur_{f};")
    w("      }")
    w("    }")
    w("  }")
    w("  gts_tmem_fence_before_sync();")
    w("  __syncthreads();")
    w("  if (warp == 0) { gts_tmem_fence_after_sync(); gts_tmem_dealloc<512>(tbase); }")
    w("}")

    # ---------------- host launch (falls back to the generic column kernel)
    smem_bytes = sp.nstages * sp.stage_bytes + 2 * 8 * sp.nstages + 16
    launch = ["  {", "    bool tmem_ok = (nk * %d <= 512);" % sp.w_level]
    for f in sp.streamed:
        e = 8 if dtypes[f] == ir.F64 else 4
        launch.append(f"    CUtensorMap tm_{f};")
        launch.append(
            f"    tmem_ok = tmem_ok && gts_make_tmap_3d(&tm_{f}, (const void*)p.f_{f}.p, {e}, nj, ni, nk,"
            f" p.f_{f}.si, p.f_{f}.sj, p.f_{f}.sk, {TJ}, {TI}, {KB});")
    tm_args = ", ".join(f"tm_{f}" for f in sp.streamed)
    launch += [
        "    if (tmem_ok) {",
        f"      const int tiles_j = (int)((nj + {TJ - 1}) / {TJ});",
        f"      const int ntiles = tiles_j * (int)((ni + {TI - 1}) / {TI});",
        "      int grid = gts_sm_count(); if (grid > ntiles) grid = ntiles;",
        "      static bool attr_set = false;",
        "      if (!attr_set) {",
        f"        cudaFuncSetAttribute({kname}_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, {smem_bytes});",
        "        attr_set = true;",
        "      }",
        f"      {kname}_tmem<<<grid, 160, {smem_bytes}, st>>>(p, {tm_args}, tiles_j, ntiles);",
        "    } else {",
        "      dim3 grid((unsigned)((nj + GTS_COL_TJ - 1) / GTS_COL_TJ),"
        " (unsigned)((ni + (GTS_COL_THREADS / GTS_COL_TJ) - 1) / (GTS_COL_THREADS / GTS_COL_TJ)), 1);",
        f"      {kname}<<<grid, GTS_COL_THREADS, 0, st>>>(p);",
        "    }",
        "  }",
    ]
    return out, launch
