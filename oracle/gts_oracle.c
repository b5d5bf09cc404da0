/*
 * gts_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference's two benchmark stencils, used
 * as the parity checker by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py.  Nothing in paper_2311_08322_b200/ links,
 * loads or calls this file; the product path fails loudly without its CUDA
 * libraries instead of falling back here.
 *
 * What it restates (reference = stencilforge 0.1.0 under /root/reference):
 *   - hdiff: pkg/src/stencilforge/kernels/hdiff.gts:3-15, lowered as in
 *     pkg/tests/golden/hdiff_implementation.txt:11-24 (four stages, extents
 *     lap [-1..1,-1..1], flx [-1..0,0..0], fly [0..0,-1..0], out [0..0,0..0];
 *     association order exactly as that dump prints it).
 *   - vadv: pkg/src/stencilforge/kernels/vadv.gts:4-16 (Thomas forward
 *     elimination seeded on interval [0,1), backward substitution seeded on
 *     [K-1,K)); dp's denominator is recomputed, not reused, exactly like
 *     the source statement (vadv.gts:12).
 *   - numerics follow the gen emitter (backends/gen.py:134-177, 229-369):
 *     f64 arithmetic, f32 operands widened on read and narrowed on every
 *     store (temporaries included: analysis.py:424-443 makes hdiff's
 *     lap/flx/fly f32 when inp/out are f32), compiled with
 *     -ffp-contract=off so no FMA contraction (gen.py:64-67).
 *   - entry ABI = the gen entry ABI (gen.py:5-14, 269-284): domain, then per
 *     api field {base, stride_i, stride_j, stride_k, origin_i, origin_j,
 *     origin_k} in element units, then scalars (always double here, like the
 *     debug/vec engines: runtime.py:113), plus a thread count.
 *
 * Build: see oracle/Makefile (gcc -O3 -fopenmp -ffp-contract=off).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t gi;

#define AT(p, s, o, I, J, K) \
  (p)[(size_t)(((I) + (o)[0]) * (s)[0] + ((J) + (o)[1]) * (s)[1] + ((K) + (o)[2]) * (s)[2])]

static void set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
}

/* ------------------------------------------------------------------ hdiff */
/* One k-plane of hdiff; T = storage type of the api fields and of the
 * temporaries (TT), arithmetic in double.  Temporaries are (ni+2)x(nj+2),
 * (ni+1)xnj, nix(nj+1) planes indexed with the stage-extent origin shift
 * (common.py:58-69). */
#define HDIFF_PLANE(T, TT)                                                          \
  {                                                                                 \
    const gi LI = nj + 2, FI = nj, YI = nj + 1;                                     \
    TT* lap = tmp;                                                                  \
    TT* flx = tmp + (size_t)(ni + 2) * (nj + 2);                                    \
    TT* fly = flx + (size_t)(ni + 1) * nj;                                          \
    /* stage 1: lap over [-1, ni+1) x [-1, nj+1) */                                  \
    for (gi i = -1; i < ni + 1; ++i)                                                \
      for (gi j = -1; j < nj + 1; ++j) {                                            \
        double c = (double)AT(inp, si, oi, i, j, k);                                \
        double v = (4.0 * c) - ((((double)AT(inp, si, oi, i - 1, j, k) +            \
                                  (double)AT(inp, si, oi, i + 1, j, k)) +           \
                                 (double)AT(inp, si, oi, i, j - 1, k)) +            \
                                (double)AT(inp, si, oi, i, j + 1, k));              \
        lap[(i + 1) * LI + (j + 1)] = (TT)v;                                        \
      }                                                                             \
    /* stage 2: flx over [-1, ni) x [0, nj) */                                       \
    for (gi i = -1; i < ni; ++i)                                                    \
      for (gi j = 0; j < nj; ++j) {                                                 \
        double l1 = (double)lap[(i + 2) * LI + (j + 1)];                            \
        double l0 = (double)lap[(i + 1) * LI + (j + 1)];                            \
        double d = (double)AT(inp, si, oi, i + 1, j, k) - (double)AT(inp, si, oi, i, j, k); \
        if (((l1 - l0) * d) > 0.0)                                                  \
          flx[(i + 1) * FI + j] = (TT)0.0;                                          \
        else                                                                        \
          flx[(i + 1) * FI + j] = (TT)(l1 - l0);                                    \
      }                                                                             \
    /* stage 3: fly over [0, ni) x [-1, nj) */                                       \
    for (gi i = 0; i < ni; ++i)                                                     \
      for (gi j = -1; j < nj; ++j) {                                                \
        double l1 = (double)lap[(i + 1) * LI + (j + 2)];                            \
        double l0 = (double)lap[(i + 1) * LI + (j + 1)];                            \
        double d = (double)AT(inp, si, oi, i, j + 1, k) - (double)AT(inp, si, oi, i, j, k); \
        if (((l1 - l0) * d) > 0.0)                                                  \
          fly[i * YI + (j + 1)] = (TT)0.0;                                          \
        else                                                                        \
          fly[i * YI + (j + 1)] = (TT)(l1 - l0);                                    \
      }                                                                             \
    /* stage 4: out over [0, ni) x [0, nj) */                                        \
    for (gi i = 0; i < ni; ++i)                                                     \
      for (gi j = 0; j < nj; ++j) {                                                 \
        double fx0 = (double)flx[(i + 1) * FI + j], fxm = (double)flx[i * FI + j];  \
        double fy0 = (double)fly[i * YI + (j + 1)], fym = (double)fly[i * YI + j];  \
        double v = (double)AT(inp, si, oi, i, j, k) -                               \
                   (coeff * (((fx0 - fxm) + fy0) - fym));                           \
        AT(out, so, oo, i, j, k) = (T)v;                                            \
      }                                                                             \
  }

#define HDIFF_ENTRY(NAME, T)                                                        \
  int NAME(gi ni, gi nj, gi nk, const T* inp, gi si0, gi si1, gi si2, gi oi0,       \
           gi oi1, gi oi2, T* out, gi so0, gi so1, gi so2, gi oo0, gi oo1, gi oo2,  \
           double coeff, int nthreads) {                                            \
    if (ni <= 0 || nj <= 0 || nk <= 0) return 0;                                    \
    const gi si[3] = {si0, si1, si2}, oi[3] = {oi0, oi1, oi2};                      \
    const gi so[3] = {so0, so1, so2}, oo[3] = {oo0, oo1, oo2};                      \
    set_threads(nthreads);                                                          \
    const size_t plane = (size_t)(ni + 2) * (nj + 2) + (size_t)(ni + 1) * nj +      \
                         (size_t)ni * (nj + 1);                                     \
    int nt = 1;                                                                     \
    _Pragma("omp parallel") {                                                       \
      _Pragma("omp single") nt = omp_nt();                                          \
    }                                                                               \
    T* arena = (T*)malloc(sizeof(T) * plane * (size_t)nt);                          \
    if (!arena) return 2;                                                           \
    _Pragma("omp parallel") {                                                       \
      T* tmp = arena + plane * (size_t)omp_tid();                                   \
      _Pragma("omp for schedule(static)") for (gi k = 0; k < nk; ++k)               \
          HDIFF_PLANE(T, T)                                                         \
    }                                                                               \
    free(arena);                                                                    \
    return 0;                                                                       \
  }

static int omp_nt(void) {
#ifdef _OPENMP
  return omp_get_num_threads();
#else
  return 1;
#endif
}
static int omp_tid(void) {
#ifdef _OPENMP
  return omp_get_thread_num();
#else
  return 0;
#endif
}

HDIFF_ENTRY(oracle_hdiff_f64, double)
HDIFF_ENTRY(oracle_hdiff_f32, float)

/* ------------------------------------------------------------------- vadv */
/* Per column (i, j): FORWARD over k then BACKWARD over k.  The reference
 * runs level by level over whole planes (gen.py:343-360); columns are
 * independent (all extents are zero), so iterating column-major computes
 * identical values.  cp/dp are per-column scratch of nk elements of the
 * temporary dtype (f32 when all of a,b,c,d are f32: analysis.py:424-443). */
#define VADV_ENTRY(NAME, T)                                                         \
  int NAME(gi ni, gi nj, gi nk, const T* a, gi sa0, gi sa1, gi sa2, gi oa0,         \
           gi oa1, gi oa2, const T* b, gi sb0, gi sb1, gi sb2, gi ob0, gi ob1,      \
           gi ob2, const T* c, gi sc0, gi sc1, gi sc2, gi oc0, gi oc1, gi oc2,      \
           const T* d, gi sd0, gi sd1, gi sd2, gi od0, gi od1, gi od2, T* x,        \
           gi sx0, gi sx1, gi sx2, gi ox0, gi ox1, gi ox2, int nthreads) {          \
    if (ni <= 0 || nj <= 0 || nk <= 0) return 0;                                    \
    const gi sa[3] = {sa0, sa1, sa2}, oa[3] = {oa0, oa1, oa2};                      \
    const gi sb[3] = {sb0, sb1, sb2}, ob[3] = {ob0, ob1, ob2};                      \
    const gi sc[3] = {sc0, sc1, sc2}, oc[3] = {oc0, oc1, oc2};                      \
    const gi sd[3] = {sd0, sd1, sd2}, od[3] = {od0, od1, od2};                      \
    const gi sx[3] = {sx0, sx1, sx2}, ox[3] = {ox0, ox1, ox2};                      \
    set_threads(nthreads);                                                          \
    int fail = 0;                                                                   \
    _Pragma("omp parallel") {                                                       \
      T* cp = (T*)malloc(sizeof(T) * (size_t)nk);                                   \
      T* dp = (T*)malloc(sizeof(T) * (size_t)nk);                                   \
      if (!cp || !dp) {                                                             \
        _Pragma("omp atomic write") fail = 1;                                       \
      } else {                                                                      \
        _Pragma("omp for schedule(static) collapse(2)") for (gi i = 0; i < ni; ++i) \
            for (gi j = 0; j < nj; ++j) {                                           \
          /* FORWARD, interval [0, 1): vadv.gts:6-8 */                              \
          {                                                                         \
            double bb = (double)AT(b, sb, ob, i, j, 0);                             \
            cp[0] = (T)((double)AT(c, sc, oc, i, j, 0) / bb);                       \
            dp[0] = (T)((double)AT(d, sd, od, i, j, 0) / bb);                       \
          }                                                                         \
          /* FORWARD, interval [1, K): vadv.gts:9-12 */                             \
          for (gi k = 1; k < nk; ++k) {                                             \
            double aa = (double)AT(a, sa, oa, i, j, k);                             \
            double bb = (double)AT(b, sb, ob, i, j, k);                             \
            double cpm = (double)cp[k - 1];                                         \
            cp[k] = (T)((double)AT(c, sc, oc, i, j, k) / (bb - (aa * cpm)));        \
            dp[k] = (T)(((double)AT(d, sd, od, i, j, k) - (aa * (double)dp[k - 1])) / \
                        (bb - (aa * cpm)));                                         \
          }                                                                         \
          /* BACKWARD, interval [K-1, K): vadv.gts:14-15 */                         \
          AT(x, sx, ox, i, j, nk - 1) = (T)(double)dp[nk - 1];                      \
          /* BACKWARD, interval [0, K-1): vadv.gts:16 */                            \
          for (gi k = nk - 2; k >= 0; --k)                                          \
            AT(x, sx, ox, i, j, k) =                                                \
                (T)((double)dp[k] - ((double)cp[k] * (double)AT(x, sx, ox, i, j, k + 1))); \
        }                                                                           \
      }                                                                             \
      free(cp);                                                                     \
      free(dp);                                                                     \
    }                                                                               \
    return fail ? 2 : 0;                                                            \
  }

VADV_ENTRY(oracle_vadv_f64, double)
VADV_ENTRY(oracle_vadv_f32, float)

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
