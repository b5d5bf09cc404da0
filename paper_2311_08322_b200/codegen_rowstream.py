"""Fused PARALLEL template, row-streaming form (default for hdiff-class groups).

Same per-point semantics and register-window machinery as the tile form in
``codegen_parallel`` (stages computed at their leading row over their column
span, temporaries in rotating register windows), but the work is organised
for continuous HBM streaming on 148 SMs:

* the whole launch is a flattened sequence of output rows
  (k-plane, 32*VJ-column block, i); warp g of G owns the contiguous range
  [g*U/G, (g+1)*U/G), so every warp gets the same number of rows (+-1) --
  no tile quantisation on small domains;
* each warp streams its input rows itself: lane 0 issues one TMA row box
  (``cp.async.bulk.tensor.3d``, 1 row x (32*VJ + halo) columns) per row into a
  private ring of NSLOT shared-memory slots with one mbarrier each, NSLOT
  rows ahead of the computation; a row is read into registers exactly once,
  so its slot is refilled immediately;
* a range crossing a k-plane or column-block boundary simply restarts the
  window (a 2-row prologue for hdiff's extents).
"""

from __future__ import annotations

from math import lcm

from ._host import ir
from .codegen import DivPool, _bound
from .codegen_parallel import _Ctx, _emit_point, _phys, _cn, analyse
from .lowering import always_writes, reads, writes
from . import codegen_parallel as cp

SLOT_BUDGET = 12 * 1024  # shared memory per warp for row slots
MAX_SLOTS = 16


def eligible(plan, kplan, dtypes):
    cp.configure({"pf_nw": 4, "pf_ri": 8, "pf_vj": 4, "pf_nbuf": 1})
    geo = analyse(plan, kplan, dtypes)
    for st in geo.stages:
        for acc in reads(st.body):
            if acc.offset[2] != 0 or acc.field not in geo.wins:
                return None
    if not any(w.kind == "stream" for w in geo.wins.values()):
        return None
    for w in geo.wins.values():
        if w.kind == "stream" and w.box_cols > 256:
            return None
    return geo


def emit(kname: str, plan, kplan, ctype: dict, dtypes: dict, opts=None):
    geo = eligible(plan, kplan, dtypes)
    if geo is None:
        return None
    o = opts or {}
    NW = int(o.get("rs_nw", 4))
    VJ = cp.VJ
    TJ = 32 * VJ
    impl = plan.impl
    api = {f.name for f in impl.api_fields}
    local = set(kplan.local_temps)
    streams = [w for _, w in sorted(geo.wins.items()) if w.kind == "stream"]
    regw = [w for _, w in sorted(geo.wins.items()) if w.kind != "stream"]
    row_bytes = {s.name: -(-(s.box_cols * s.esize) // 128) * 128 for s in streams}
    per_row = sum(row_bytes.values())
    nslot = int(o.get("rs_slots", max(4, min(MAX_SLOTS, SLOT_BUDGET // per_row))))
    warp_bytes = nslot * per_row
    bars_off = NW * warp_bytes
    nbar = NW * len(streams) * nslot
    smem_bytes = bars_off + 8 * nbar + 16
    P = 1
    for x in list(geo.wins.values()):
        P = lcm(P, x.rhi - x.rlo + 1)
    ms = geo.min_step  # <= 0
    out: list = []
    w = out.append
    tm = ", ".join(f"const __grid_constant__ CUtensorMap tm_{s.name}" for s in streams)
    w(f"// fused PARALLEL row-stream kernel: {NW} warps/CTA, {VJ} columns/lane ({TJ}-column blocks),"
      f" {nslot} TMA row slots/warp/stream, window unroll {P}; streamed {[s.name for s in streams]}")
    minb = int(o.get("rs_minb", 4))
    w(f"__global__ void __launch_bounds__({32 * NW}, {minb}) {kname}(const __grid_constant__ GtsParams p, {tm}, "
      "int k0, int tiles_j, long long U) {")
    w("  extern __shared__ __align__(1024) unsigned char smem[];")
    w("  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;")
    w(f"  uint64_t* bars = (uint64_t*)(smem + {bars_off}) + warp * {len(streams) * nslot};")
    w(f"  unsigned char* wsm = smem + warp * {warp_bytes};")
    w("  if (lane == 0) {")
    w(f"    for (int q = 0; q < {len(streams) * nslot}; ++q) gts_mbar_init(&bars[q], 1);")
    w("    gts_fence_mbar_init();")
    w("  }")
    w("  __syncwarp();")
    w("  const int ni = p.ni, nj = p.nj;")
    w(f"  const long long G = (long long)gridDim.x * {NW};")
    w(f"  const long long g = (long long)blockIdx.x * {NW} + warp;")
    w("  const long long u0 = (g * U) / G, u1 = ((g + 1) * U) / G;")
    w("  if (u0 >= u1) return;")
    w("  const long long plane = (long long)tiles_j * ni;")
    soff = 0
    for si, s in enumerate(streams):
        w(f"  const {ctype[s.name]}* const rs_{s.name} = (const {ctype[s.name]}*)(wsm + {soff});")
        w(f"  uint64_t* const bar_{s.name} = bars + {si * nslot};")
        w(f"  const int jsh_{s.name} = p.tsh_{s.name}_j, ish_{s.name} = p.tsh_{s.name}_i, ksh_{s.name} = p.tsh_{s.name}_k;")
        # producer cursor: segment start unit, request index within it, requests issued
        w(f"  long long pu_{s.name} = u0; int pq_{s.name} = 0, pn_{s.name} = 0, cn_{s.name} = 0;")
        # cached segment of the producer cursor (divisions only per segment)
        w(f"  int pkb_{s.name} = 0, pjb_{s.name} = 0, pia_{s.name} = 0, pib_{s.name} = 0;")
        w(f"  {{ const int kb_ = (int)(u0 / plane); const long long rm_ = u0 - (long long)kb_ * plane;")
        w(f"    pkb_{s.name} = kb_; pjb_{s.name} = (int)(rm_ / ni); pia_{s.name} = (int)(rm_ % ni);")
        w(f"    pib_{s.name} = (int)(((long long)ni < (long long)pia_{s.name} + (u1 - u0)) ? ni : (long long)pia_{s.name} + (u1 - u0)); }}")
        soff += nslot * row_bytes[s.name]

    def produce(indent):
        """Refill every ring up to NSLOT rows ahead of consumption."""
        for s in streams:
            n = s.name
            cnt_extra = (s.rhi - s.rlo) - ms  # requests per segment = (ib - ia) + cnt_extra
            w(f"{indent}while (pn_{n} - cn_{n} < {nslot} && pu_{n} < u1) {{")
            w(f"{indent}  const int kb_ = pkb_{n}, jb_ = pjb_{n}, ia_ = pia_{n}, ib_ = pib_{n};")
            w(f"{indent}  if (lane == 0) {{")
            w(f"{indent}    const int sl_ = pn_{n} % {nslot};")
            w(f"{indent}    gts_fence_proxy_async();")
            w(f"{indent}    gts_mbar_arrive_expect_tx(&bar_{n}[sl_], {s.box_cols * s.esize}u);")
            w(f"{indent}    gts_tma_load_3d((void*)(rs_{n} + (size_t)sl_ * {row_bytes[n] // s.esize}), &tm_{n}, &bar_{n}[sl_],"
              f" jb_ * {TJ} + ({s.bstart}) + jsh_{n}, ia_ + ({ms + s.rlo}) + pq_{n} + ish_{n}, k0 + kb_ + ksh_{n});")
            w(f"{indent}  }}")
            w(f"{indent}  ++pn_{n};")
            w(f"{indent}  if (++pq_{n} == (ib_ - ia_) + {cnt_extra}) {{")
            w(f"{indent}    pq_{n} = 0; pu_{n} += ib_ - ia_;")
            w(f"{indent}    if (pu_{n} < u1) {{ const int kb2 = (int)(pu_{n} / plane); const long long rm2 = pu_{n} - (long long)kb2 * plane;")
            w(f"{indent}      pkb_{n} = kb2; pjb_{n} = (int)(rm2 / ni); pia_{n} = (int)(rm2 % ni);")
            w(f"{indent}      pib_{n} = (int)(((long long)ni < (long long)pia_{n} + (u1 - pu_{n})) ? ni : (long long)pia_{n} + (u1 - pu_{n})); }}")
            w(f"{indent}  }}")
            w(f"{indent}}}")

    def consume_row(s, logical_row, indent):
        """Wait for the next row of stream s and read this lane's columns into
        the window's logical row (vector loads where aligned)."""
        n = s.name
        prow = _phys(geo, s, logical_row)
        w(f"{indent}{{ const int sl_ = cn_{n} % {nslot};")
        w(f"{indent}  gts_mbar_wait(&bar_{n}[sl_], (uint32_t)(cn_{n} / {nslot}) & 1u);")
        w(f"{indent}  const {ctype[n]}* const rp_ = rs_{n} + (size_t)sl_ * {row_bytes[n] // s.esize} + lane * {VJ};")
        off = s.clo - s.bstart
        ncol = s.chi - s.clo + 1
        vmax = 16 // s.esize
        c = 0
        while c < ncol:
            v = vmax
            while v > 1 and not ((off + c) % v == 0 and VJ % v == 0 and c + v <= ncol):
                v //= 2
            if v == 1:
                w(f"{indent}  w_{n}[{prow}][{c}] = (double)rp_[{off + c}];")
            else:
                vt = {(8, 2): "double2", (4, 2): "float2", (4, 4): "float4"}[(s.esize, v)]
                w(f"{indent}  {{ const {vt} q_ = *reinterpret_cast<const {vt}*>(rp_ + {off + c});")
                for q in range(v):
                    w(f"{indent}    w_{n}[{prow}][{c + q}] = (double)q_.{'xyzw'[q]};")
                w(f"{indent}  }}")
            c += v
        w(f"{indent}  ++cn_{n};")
        w(f"{indent}}}")

    def step(rel_static, rot, guard, indent):
        """One row step: r = row of the zero-extent stages. ``rel_static``:
        offset from the segment start when known (prologue), else None."""
        geo.rot = rot
        w(f"{indent}{{")
        ind = indent + "  "
        for s in streams:
            consume_row(s, s.rhi - s.rlo, ind)
        w(f"{ind}__syncwarp();")
        produce(ind)
        for f in sorted(geo.buffered):
            w(f"{ind}{ctype[f]} o_{f}[{VJ}];")
        for si, st in enumerate(geo.stages):
            li, hi, lj, hj = geo.ext[si]
            if rel_static is not None and rel_static + hi < li:
                continue
            w(f"{ind}{{ // stage {si} at row r + {hi}")
            for col in range(lj, VJ + hj):
                ctx = _Ctx(geo, ctype, hi, col)
                ctx.pool = DivPool("branch")
                ctx.arena = set(plan.global_temps)
                ctx.stage_ext = geo.ext[si]
                okc = f"okc_{col}" if 0 <= col < VJ else "false"
                w(f"{ind}  {{ const bool ok_{_cn(col)} = {okc} && {hi} == 0;")
                for f in sorted(writes(st.body) - always_writes(st.body)):
                    wv = geo.wins.get(f)
                    if wv is not None and wv.kind in ("temp", "own"):
                        w(f"{ind}    w_{f}[{_phys(geo, wv, hi - wv.rlo)}][{col - wv.clo}] = GTS_NAN;")
                _emit_point(st.body, ctx, ctype, api, out, ind + "    ", local, geo)
                w(f"{ind}  }}")
            w(f"{ind}}}")
        if rel_static is None or rel_static >= 0:
            for f in sorted(geo.buffered):
                w(f"{ind}{{ {ctype[f]}* const op = &GTS_AT(p.f_{f}, r, jl, kk);")
                w(f"{ind}  if (jl + {VJ} <= nj && p.f_{f}.sj == 1 && (((uintptr_t)op) & 15) == 0) {{")
                if dtypes[f] == ir.F64:
                    for q in range(0, VJ, 2):
                        w(f"{ind}    *reinterpret_cast<double2*>(op + {q}) = make_double2(o_{f}[{q}], o_{f}[{q + 1}]);")
                else:
                    for q in range(0, VJ, 4):
                        w(f"{ind}    *reinterpret_cast<float4*>(op + {q}) = make_float4(o_{f}[{q}], o_{f}[{q + 1}], o_{f}[{q + 2}], o_{f}[{q + 3}]);")
                w(f"{ind}  }} else {{")
                for q in range(VJ):
                    w(f"{ind}    if (jl + {q} < nj) op[(long long){q} * p.f_{f}.sj] = o_{f}[{q}];")
                w(f"{ind}  }}")
                w(f"{ind}}}")
        w(f"{indent}}}")

    produce("  ")
    w("  for (long long cu = u0; cu < u1; ) {")
    w("    const int kb = (int)(cu / plane); const long long rm = cu - (long long)kb * plane;")
    w("    const int jb = (int)(rm / ni), ia = (int)(rm % ni);")
    w("    const int ib = (int)(((long long)ni < (long long)ia + (u1 - cu)) ? ni : (long long)ia + (u1 - cu));")
    w("    const int kk = k0 + kb;")
    w(f"    const int jl = jb * {TJ} + lane * {VJ};")
    for c in range(VJ):
        w(f"    const bool okc_{c} = (jl + {c}) < nj;")
    for x in regw + streams:
        w(f"    double w_{x.name}[{x.rhi - x.rlo + 1}][{x.chi - x.clo + 1}];")
    # window fill: logical rows 0 .. depth-2 of every stream at rot 0
    geo.rot = 0
    for s in streams:
        for d in range(s.rhi - s.rlo):
            consume_row(s, d, "    ")
    # prologue steps (rows whose outputs are not stored)
    for q, rel in enumerate(range(ms, 0)):
        w(f"    {{ const int r = ia + ({rel});")
        step(rel, q, None, "      ")
        w("    }")
    base_rot = -ms
    w("    int r = ia;")
    w(f"    for (; r + {P} <= ib; r += {P}) {{")
    for q in range(P):
        w(f"      {{ const int r_ = r + {q}; {{ const int r = r_;")
        step(None, base_rot + q, None, "        ")
        w("      } }")
    w("    }")
    for q in range(P - 1):
        w(f"    if (r + {q} < ib) {{ const int r_ = r + {q}; {{ const int r = r_;")
        step(None, base_rot + q, None, "      ")
        w("    } }")
    w("    cu += ib - ia;")
    w("  }")
    w("}")

    flag = f"fz_ok_{kname.split('_')[1][1:]}"
    pre = [f"  // TMA row maps of {kname}: each covers the field's required region (its extent)"]
    for s in streams:
        pre.append(f"  CUtensorMap tm_{kname}_{s.name};")
    pre.append(f"  bool {flag} = true;")
    for s in streams:
        fe = plan.impl.field_extent(s.name)
        pre += [
            f"  p.tsh_{s.name}_i = -({fe.lo[0]}); p.tsh_{s.name}_j = -({fe.lo[1]} - {s.cshift}); p.tsh_{s.name}_k = 0;",
            f"  {flag} = {flag} && gts_make_tmap_3d(&tm_{kname}_{s.name}, (const void*)&GTS_AT(p.f_{s.name}, {fe.lo[0]}, {fe.lo[1]} - {s.cshift}, 0), {s.esize},"
            f" nj + {fe.hi[1] - fe.lo[1]} + {s.cshift}, ni + {fe.hi[0] - fe.lo[0]}, nk, p.f_{s.name}.si, p.f_{s.name}.sj, p.f_{s.name}.sk,"
            f" {s.box_cols}, 1, 1);",
        ]
    tm_args = ", ".join(f"tm_{kname}_{s.name}" for s in streams)
    launch = [
        "    {",
        f"      const int k0 = {_bound(kplan.interval.start)}, k1 = {_bound(kplan.interval.end)};",
        f"      const int tiles_j = (int)((nj + {TJ - 1}) / {TJ});",
        "      const long long U = (long long)(k1 - k0) * tiles_j * ni;",
        "      if (U > 0) {",
        "        static bool attr = false;",
        "        static int per_sm = 1;",
        f"        if (!attr) {{ cudaFuncSetAttribute({kname}, cudaFuncAttributeMaxDynamicSharedMemorySize, {smem_bytes});",
        f"          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, {kname}, {32 * NW}, {smem_bytes}); if (per_sm < 1) per_sm = 1; attr = true; }}",
        "        long long grid = (long long)per_sm * gts_sm_count();",
        f"        const long long need = (U + 1) / 2;  // >= 2 rows per warp",
        f"        if (grid * {NW} > need) grid = (need + {NW - 1}) / {NW};",
        "        if (grid < 1) grid = 1;",
        f"        {kname}<<<(unsigned)grid, {32 * NW}, {smem_bytes}, st>>>(p, {tm_args}, k0, tiles_j, U);",
        "      }",
        "    }",
    ]
    return out, pre, launch
