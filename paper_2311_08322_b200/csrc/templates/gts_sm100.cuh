// gts_sm100.cuh -- sm_100a building blocks used by the stencil templates:
// mbarriers, TMA tensor loads (cp.async.bulk.tensor), Tensor Memory
// (tcgen05.alloc / st / ld) and host-side tensor-map encoding through the
// driver entry point (no libcuda link needed).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <vector>

// ---------------------------------------------------------------------------
// mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t gts_smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void gts_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(gts_smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void gts_fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void gts_mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(gts_smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void gts_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(gts_smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void gts_mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = gts_smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// Wait with back-off: for a producer warp that shares an SM sub-partition
// with a consumer warp, so its polling does not steal issue slots.
__device__ __forceinline__ bool gts_mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(gts_smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
template <int kSleepNs = 200>
__device__ __forceinline__ void gts_mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  while (!gts_mbar_try(bar, parity)) {
    if (kSleepNs > 0) __nanosleep(kSleepNs);
  }
}

// Generic-proxy reads of a smem buffer must be ordered before the async
// proxy (TMA) overwrites it.
__device__ __forceinline__ void gts_fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------
// TMA
// ---------------------------------------------------------------------------
__device__ __forceinline__ void gts_tma_load_3d(void* smem_dst, const CUtensorMap* map,
                                                uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(gts_smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(gts_smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// Warm L2 with one box (no shared-memory destination, no barrier).  L2 is the
// point of coherence of device memory, so this is safe even before
// griddepcontrol.wait: a later write by the previous grid lands in the line.
__device__ __forceinline__ void gts_tma_prefetch_l2_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

__device__ __forceinline__ void gts_prefetch_tensormap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ---------------------------------------------------------------------------
// Tensor Memory (TMEM): 128 lanes x 512 columns x 32 bit per SM.  Warp w of
// the CTA owns lanes 32*(w%4) .. 32*(w%4)+31; with 32x32b shapes thread t of
// the warp reads / writes its own lane.
// ---------------------------------------------------------------------------
template <int kCols>
__device__ __forceinline__ void gts_tmem_alloc(uint32_t* smem_addr_slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   gts_smem_u32(smem_addr_slot)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <int kCols>
__device__ __forceinline__ void gts_tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
               : "memory");
}

__device__ __forceinline__ void gts_tmem_fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void gts_tmem_fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void gts_tmem_st2(uint32_t taddr, uint32_t r0, uint32_t r1) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(r0),
               "r"(r1));
}
__device__ __forceinline__ void gts_tmem_st1(uint32_t taddr, uint32_t r0) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(r0));
}
__device__ __forceinline__ void gts_tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void gts_tmem_ld2(uint32_t taddr, uint32_t& r0, uint32_t& r1) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(taddr));
}
__device__ __forceinline__ void gts_tmem_ld1(uint32_t taddr, uint32_t& r0) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
               : "=r"(r0)
               : "r"(taddr));
}
__device__ __forceinline__ void gts_tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// wait::ld tied to the destination registers, so no use of them can be
// scheduled before the wait completes.
__device__ __forceinline__ void gts_tmem_wait_ld_r2(uint32_t& r0, uint32_t& r1) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r0), "+r"(r1)::"memory");
}
__device__ __forceinline__ void gts_tmem_wait_ld_r4(uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                                    uint32_t& r3) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r0), "+r"(r1), "+r"(r2), "+r"(r3)::"memory");
}
__device__ __forceinline__ void gts_tmem_ld4(uint32_t taddr, uint32_t& r0, uint32_t& r1,
                                             uint32_t& r2, uint32_t& r3) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(taddr));
}


// 32 consecutive TMEM columns of this thread's lane in one instruction
// (e.g. 8 levels x 4 words of a Thomas history), and a wait tied to them.
__device__ __forceinline__ void gts_tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(taddr));
}
__device__ __forceinline__ void gts_tmem_wait_ld32(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])::"memory");
}

__device__ __forceinline__ void gts_tmem_store_f64(uint32_t taddr, double v) {
  gts_tmem_st2(taddr, (uint32_t)__double2loint(v), (uint32_t)__double2hiint(v));
}
__device__ __forceinline__ void gts_tmem_store_f32(uint32_t taddr, float v) {
  gts_tmem_st1(taddr, __float_as_uint(v));
}

// ---------------------------------------------------------------------------
// Division by a launch-constant divisor without the XU pipe: n / d as a
// multiply-high and a shift (Granlund-Montgomery round-up method, exact for
// 0 <= n < 2^31, 1 <= d < 2^31).  A 32-bit integer division otherwise
// expands to I2F + MUFU.RCP + F2I on the XU pipe -- the pipe that also
// carries every binary32 <-> binary64 conversion, which bounds the f32-storage
// tile kernel (ncu: XU 66 % active).
// ---------------------------------------------------------------------------
struct GtsFastDiv {
  uint32_t d, m, s;
};
static inline GtsFastDiv gts_fastdiv(int d) {
  GtsFastDiv f;
  f.d = (uint32_t)(d > 0 ? d : 1);
  uint32_t l = 0;
  while ((1u << l) < f.d) ++l;  // ceil(log2 d)
  const uint32_t p = 31 + l;
  f.m = (uint32_t)(((1ull << p) + f.d - 1) / f.d);
  f.s = p - 32;
  return f;
}
__device__ __forceinline__ int gts_div_c(int n, const GtsFastDiv& f) {
  return f.d == 1 ? n : (int)(__umulhi((uint32_t)n, f.m) >> f.s);
}

// ---------------------------------------------------------------------------
// Frame tiles: the tiles of a tiles_i x tiles_j plane outside the inner
// rectangle [fi0, fi1) x [fj0, fj1), enumerated row by row (the frame launch
// of a decomposed step: top rows, then the left / right tiles of the middle
// rows, then the bottom rows).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void gts_frame_tile(int u, int tiles_j, int fi0, int fi1, int fj0, int fj1,
                                               int& ti, int& tj) {
  const int top = fi0 * tiles_j;
  if (u < top) {
    ti = u / tiles_j;
    tj = u - ti * tiles_j;
    return;
  }
  u -= top;
  const int side = tiles_j - (fj1 - fj0);
  const int mid = (fi1 - fi0) * side;
  if (u < mid) {
    const int r = u / side;
    const int c = u - r * side;
    ti = fi0 + r;
    tj = c < fj0 ? c : c + (fj1 - fj0);
    return;
  }
  u -= mid;
  ti = fi1 + u / tiles_j;
  tj = u - (u / tiles_j) * tiles_j;
}

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL): a persistent stencil kernel lets the
// next launch in the stream start as soon as every CTA of this one is
// resident, and waits for the previous grid's completion (and memory flush)
// before its first global access -- the next kernel's launch latency and
// setup (mbarrier init, TMEM alloc, tensor-map prefetch) overlap this one's
// tail.  Kernels that call gts_griddep_wait() before touching global memory
// are launched through gts_launch_pdl(); all others keep full serialisation.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void gts_griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void gts_griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
static cudaError_t gts_launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                  cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++g_gts_launches;
  return cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
}

// ---------------------------------------------------------------------------
// Host: tensor maps
// ---------------------------------------------------------------------------
typedef CUresult (*gts_encode_tiled_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                        const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                        const cuuint32_t*, CUtensorMapInterleave,
                                        CUtensorMapSwizzle, CUtensorMapL2promotion,
                                        CUtensorMapFloatOOBfill);

static gts_encode_tiled_fn gts_get_encode_tiled() {
  static gts_encode_tiled_fn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (gts_encode_tiled_fn)p;
  }
  return fn;
}

// 3-D tiled map over a field with j contiguous: dims {nj, ni, nk}, element
// strides {1, s_i, s_k}; ``origin`` points at element (0, 0, 0) of the box
// coordinate system.  Returns false when the field is not TMA-compatible
// (16-B aligned base and byte strides) -- the caller then uses the
// non-TMA kernel.
static bool gts_make_tmap_3d(CUtensorMap* map, const void* origin, int itemsize, long long nj,
                             long long ni, long long nk, long long s_i, long long s_j,
                             long long s_k, unsigned bj, unsigned bi, unsigned bk) {
  gts_encode_tiled_fn enc = gts_get_encode_tiled();
  if (!enc) return false;
  if (s_j != 1) return false;
  if (((uintptr_t)origin) % 16) return false;
  if ((s_i * itemsize) % 16 || (s_k * itemsize) % 16) return false;
  if (s_i <= 0 || s_k <= 0) return false;
  // repeat calls on the same fields reuse the encoded map (a small per-thread
  // cache keyed by every encoding input): the host cost of a repeated launch
  struct Key {
    const void* o;
    long long v[8];
    unsigned b[3];
  };
  struct Entry {
    Key k;
    CUtensorMap m;
    bool used;
  };
  static thread_local Entry cache[16];
  static thread_local unsigned next_slot = 0;
  Key key;
  memset(&key, 0, sizeof(key));
  key.o = origin;
  key.v[0] = itemsize, key.v[1] = nj, key.v[2] = ni, key.v[3] = nk;
  key.v[4] = s_i, key.v[5] = s_j, key.v[6] = s_k;
  key.b[0] = bj, key.b[1] = bi, key.b[2] = bk;
  for (int e = 0; e < 16; ++e)
    if (cache[e].used && memcmp(&cache[e].k, &key, sizeof(key)) == 0) {
      *map = cache[e].m;
      return true;
    }
  cuuint64_t dims[3] = {(cuuint64_t)nj, (cuuint64_t)ni, (cuuint64_t)nk};
  cuuint64_t strides[2] = {(cuuint64_t)(s_i * itemsize), (cuuint64_t)(s_k * itemsize)};
  cuuint32_t box[3] = {bj, bi, bk};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, itemsize == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   3, const_cast<void*>(origin), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  Entry& slot = cache[next_slot++ % 16];
  slot.k = key;
  slot.m = *map;
  slot.used = true;
  return true;
}

static int gts_sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// ---------------------------------------------------------------------------
// Two-height tile plan of the persistent column kernels.  Tiles are `rows`
// i-rows x 32 j-columns; CTA b of a grid of G takes tiles b, b+G, ...  When
// the tile count is not a multiple of G, the last round leaves SMs idle while
// the others run a whole extra tile (256^2 x 80 vadv: 256 tiles on 148 SMs).
// The plan covers i in [0, isplit) with rows-high tiles (the first n1 tiles)
// and i in [isplit, ni) with h2-high tiles, chosen to minimise the most
// loaded SM.  Cost of an h-row tile ~ max(h, 0.72 rows): measured on B200, a
// lone 8-row tile runs in ~13 us (its serial recurrence) against ~18 us per
// bandwidth-bound round of 8-row tiles (tools/ksweep.py).
// ---------------------------------------------------------------------------
struct GtsColSplit {
  int n1, isplit, h2, ntiles;
};

static long gts_col_split_cost(int ni, int tj, int rows, int isplit, int h2, int G) {
  static thread_local std::vector<long> load;
  load.assign((size_t)G, 0);
  const long lat = (72L * rows + 99) / 100;
  long t = 0, worst = 0;
  auto add = [&](int h, int count) {
    const long c = (h > lat ? h : lat);
    for (int q = 0; q < count; ++q, ++t) {
      long& l = load[(size_t)(t % G)];
      l += c;
      if (l > worst) worst = l;
    }
  };
  for (int i0 = 0; i0 < isplit; i0 += rows) add(i0 + rows <= ni ? rows : ni - i0, tj);
  if (h2 > 0)
    for (int i0 = isplit; i0 < ni; i0 += h2) add(i0 + h2 <= ni ? h2 : ni - i0, tj);
  return worst;
}

static GtsColSplit gts_col_split(int ni, int nj, int rows, int G) {
  static thread_local int cni = -1, cnj = -1, crows = -1, cG = -1;
  static thread_local GtsColSplit cached;
  if (ni == cni && nj == cnj && rows == crows && G == cG) return cached;
  const int tj = (nj + 31) / 32;
  const int full = (ni + rows - 1) / rows;
  GtsColSplit best = {full * tj, full * rows, 0, full * tj};
  if ((long)full * tj > G && ((long)full * tj) % G != 0) {
    long bc = gts_col_split_cost(ni, tj, rows, full * rows, 0, G);
    // the h2 tiles only ever need to cover the last ~2 rounds
    // (largest isplit first: at equal cost, keep more full-height tiles)
    const int span = 2 * ((G + tj - 1) / tj) * rows + rows;
    const int is_lo = full * rows - span > 0 ? ((full * rows - span) / rows) * rows : 0;
    for (int is = ((ni - 1) / rows) * rows; is >= is_lo; is -= rows)
      for (int h2 = rows - 1; h2 >= 1; --h2) {
        const long c = gts_col_split_cost(ni, tj, rows, is, h2, G);
        if (c * 50 < bc * 49) {  // > 2% better than the best so far
          bc = c;
          best = {(is / rows) * tj, is, h2, (is / rows) * tj + ((ni - is + h2 - 1) / h2) * tj};
        }
      }
  }
  cni = ni, cnj = nj, crows = rows, cG = G, cached = best;
  return best;
}
