// Experiment (not product code): vadv in ONE round per SM -- R rows x 32
// columns per CTA (R = 15: 144 CTAs for 256^2, against 256 tiles of 8 rows on
// 148 SMs in the template), the column history (cp, dp) in global memory kept
// L2-resident with cache hints (TMA loads and history reads evict_first,
// history stores evict_last) instead of TMEM + shared memory, whose capacity
// caps a round at 256 columns per SM ("vadv").
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --fmad=false \
//        -I paper_2311_08322_b200/csrc/templates -DR=15 -DKB=2 -DNST=6 tools/vadv_l2_proto.cu
//
// Measured on one B200 (256x256x80 f64, graph-timed): bitwise vs the C loop
// below; ncu DRAM traffic stays at the algorithmic bytes (180 MB read, 52 MB
// written: the 84 MB of history never leaves L2), but the kernel takes 60 us
// (R = 8, two rounds: 52 us) against 38.3 us for the TMEM template -- the
// per-level global history stores and the L2-latency-bound backward reads
// cost more than the second round they remove.  Not adopted.
#include "gts_common.cuh"
#include "gts_sm100.cuh"
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

#ifndef R
#define R 15
#endif
#ifndef KB
#define KB 2
#endif
#ifndef NST
#define NST 6
#endif
#ifndef HINTS
#define HINTS 1
#endif
constexpr int FB = R * 32 * KB * 8;       // bytes of one field box per stage
constexpr int STB = 4 * FB;               // stage bytes
constexpr int SMEM = NST * STB + 2 * NST * 8 + 64;

__device__ __forceinline__ void tma_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                         uint64_t pol) {
#if HINTS
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(gts_smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(gts_smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
      : "memory");
#else
  gts_tma_load_3d(dst, map, bar, c0, c1, c2);
#endif
}

__device__ __forceinline__ void st_hist(double2* p, double a, double b, uint64_t pol) {
#if HINTS
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(a), "d"(b), "l"(pol) : "memory");
#else
  *p = make_double2(a, b);
#endif
}
__device__ __forceinline__ double2 ld_hist(const double2* p, uint64_t pol) {
  double2 v;
#if HINTS
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
#else
  v = *p;
#endif
  return v;
}

__global__ void __launch_bounds__((R + 1) * 32, 1)
vadv_l2(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
        const __grid_constant__ CUtensorMap tc, const __grid_constant__ CUtensorMap td, double* __restrict__ x,
        long long xsi, long long xsk, double2* __restrict__ hist, int ni, int nj, int nk, int tiles_j) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = (uint64_t*)(smem + NST * STB);
  uint64_t* empty = full + NST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { gts_mbar_init(&full[s], 1); gts_mbar_init(&empty[s], R); }
    gts_fence_mbar_init();
  }
  __syncthreads();
  const int t = blockIdx.x;
  const int i0 = (t / tiles_j) * R, j0 = (t % tiles_j) * 32;
  const int nkb = (nk + KB - 1) / KB;
  uint64_t pol_first, pol_last;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
  if (warp == R) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % NST;
        if (kb >= NST) gts_mbar_wait_sleep<200>(&empty[s], ((kb / NST) & 1) ^ 1);
        gts_mbar_arrive_expect_tx(&full[s], STB);
        unsigned char* sb = smem + s * STB;
        tma_hint(sb, &ta, &full[s], j0, i0, kb * KB, pol_first);
        tma_hint(sb + FB, &tb, &full[s], j0, i0, kb * KB, pol_first);
        tma_hint(sb + 2 * FB, &tc, &full[s], j0, i0, kb * KB, pol_first);
        tma_hint(sb + 3 * FB, &td, &full[s], j0, i0, kb * KB, pol_first);
      }
    }
    return;
  }
  const int i = i0 + warp, j = j0 + lane;
  const bool valid = i < ni && j < nj;
  double2* hp = hist + ((long long)t * nk * R + warp) * 32 + lane;  // level k: + k * R * 32
  double cp = 0.0, dp = 0.0;
  bool bad = false;
  const long long LS = (long long)R * 32;  // history level stride (double2)
  for (int kb = 0; kb < nkb; ++kb) {
    const int s = kb % NST;
    gts_mbar_wait(&full[s], (kb / NST) & 1);
    const double* sa = (const double*)(smem + s * STB) + warp * 32 + lane;
    const int kbase = kb * KB;
    if (kbase + KB <= nk && kbase > 0) {
#pragma unroll
      for (int kk = 0; kk < KB; ++kk) {
        const double a = sa[kk * R * 32], b = sa[FB / 8 + kk * R * 32], c = sa[2 * FB / 8 + kk * R * 32],
                     d = sa[3 * FB / 8 + kk * R * 32];
        const GtsRcp r = gts_rcp(b - a * cp);
        const double ncp = gts_div_fast(c, r, bad);
        dp = gts_div_fast(d - a * dp, r, bad);
        cp = ncp;
        st_hist(hp + (kbase + kk) * LS, cp, dp, pol_last);
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < KB; ++kk) {
        const int k = kbase + kk;
        if (k < nk) {
          const double a = sa[kk * R * 32], b = sa[FB / 8 + kk * R * 32], c = sa[2 * FB / 8 + kk * R * 32],
                       d = sa[3 * FB / 8 + kk * R * 32];
          if (k == 0) {
            const GtsRcp r = gts_rcp(b);
            cp = gts_div_fast(c, r, bad);
            dp = gts_div_fast(d, r, bad);
          } else {
            const GtsRcp r = gts_rcp(b - a * cp);
            const double ncp = gts_div_fast(c, r, bad);
            dp = gts_div_fast(d - a * dp, r, bad);
            cp = ncp;
          }
          st_hist(hp + k * LS, cp, dp, pol_last);
        }
      }
    }
    __syncwarp();
    if (lane == 0) gts_mbar_arrive(&empty[s]);
  }
  if (bad) hist[0].x = 1.0 / 0.0;  // prototype: a replay would run here (never on these inputs)
  // backward: x[nk-1] = dp; x[k] = dp[k] - cp[k] * x[k+1]; history loads
  // software-pipelined BW levels ahead
  constexpr int BW = 16;
  double* xp = x + (long long)(valid ? i : 0) * xsi + (valid ? j : 0);
  double xv = dp;
  if (valid) xp[(long long)(nk - 1) * xsk] = xv;
  int k = nk - 2;
  double2 cur[BW], nxt[BW];
#pragma unroll
  for (int q = 0; q < BW; ++q) nxt[q] = (k - q >= 0) ? ld_hist(hp + (k - q) * LS, pol_first) : make_double2(0, 0);
  for (; k >= 0; k -= BW) {
#pragma unroll
    for (int q = 0; q < BW; ++q) cur[q] = nxt[q];
#pragma unroll
    for (int q = 0; q < BW; ++q) {
      const int kn = k - BW - q;
      nxt[q] = kn >= 0 ? ld_hist(hp + kn * LS, pol_first) : make_double2(0, 0);
    }
#pragma unroll
    for (int q = 0; q < BW; ++q) {
      if (k - q >= 0) {
        xv = cur[q].y - cur[q].x * xv;
        if (valid) xp[(long long)(k - q) * xsk] = xv;
      }
    }
  }
}

// ---------------------------------------------------------------- host
static uint64_t rng = 88172645463325252ull;
static double urand() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return (rng >> 11) * (1.0 / 9007199254740992.0); }

int main(int argc, char** argv) {
  const int ni = argc > 1 ? atoi(argv[1]) : 256, nj = argc > 2 ? atoi(argv[2]) : 256, nk = argc > 3 ? atoi(argv[3]) : 80;
  const int nsets = 3, steps = 200;
  const long long n = (long long)ni * nj * nk;
  const long long si = nj, sk = (long long)ni * nj;
  std::vector<double> h[4];
  for (int f = 0; f < 4; ++f) h[f].resize(n);
  for (long long e = 0; e < n; ++e) {
    const double a = 0.1 + 0.9 * urand(), c = 0.1 + 0.9 * urand();
    h[0][e] = a; h[2][e] = c; h[1][e] = a + c + 0.5 + urand(); h[3][e] = 2 * urand() - 1;
  }
  const int tiles_i = (ni + R - 1) / R, tiles_j = nj / 32, tiles = tiles_i * tiles_j;
  std::vector<double*> dv(nsets * 5);
  std::vector<CUtensorMap> maps(nsets * 4);
  double2* hist;
  CK(cudaMalloc(&hist, (size_t)tiles * nk * R * 32 * sizeof(double2)));
  for (int s = 0; s < nsets; ++s)
    for (int f = 0; f < 5; ++f) {
      CK(cudaMalloc(&dv[s * 5 + f], n * 8));
      if (f < 4) {
        CK(cudaMemcpy(dv[s * 5 + f], h[f].data(), n * 8, cudaMemcpyHostToDevice));
        if (!gts_make_tmap_3d(&maps[s * 4 + f], dv[s * 5 + f], 8, nj, ni, nk, si, 1, sk, 32, R, KB)) {
          printf("tmap failed\n");
          return 1;
        }
      } else {
        CK(cudaMemset(dv[s * 5 + f], 0, n * 8));
      }
    }
  CK(cudaFuncSetAttribute(vadv_l2, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  auto launch = [&](int s) {
    vadv_l2<<<tiles, (R + 1) * 32, SMEM, st>>>(maps[s * 4], maps[s * 4 + 1], maps[s * 4 + 2], maps[s * 4 + 3],
                                               dv[s * 5 + 4], si, sk, hist, ni, nj, nk, tiles_j);
  };
  launch(0);
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  std::vector<double> got(n);
  CK(cudaMemcpy(got.data(), dv[4], n * 8, cudaMemcpyDeviceToHost));
  long long bad = 0;
  std::vector<double> cpv(nk), dpv(nk);
  for (int i = 0; i < ni; ++i)
    for (int j = 0; j < nj; ++j) {
      auto A = [&](int f, int k) { return h[f][(long long)k * sk + (long long)i * si + j]; };
      cpv[0] = A(2, 0) / A(1, 0);
      dpv[0] = A(3, 0) / A(1, 0);
      for (int k = 1; k < nk; ++k) {
        const double den = A(1, k) - A(0, k) * cpv[k - 1];
        cpv[k] = A(2, k) / den;
        dpv[k] = (A(3, k) - A(0, k) * dpv[k - 1]) / den;
      }
      double xv = dpv[nk - 1];
      for (int k = nk - 1; k >= 0; --k) {
        if (k < nk - 1) xv = dpv[k] - cpv[k] * xv;
        const double g = got[(long long)k * sk + (long long)i * si + j];
        if (memcmp(&g, &xv, 8)) { if (bad < 3) printf("mismatch %d %d %d %.17g %.17g\n", i, j, k, g, xv); ++bad; }
      }
    }
  for (int w = 0; w < 2 * nsets; ++w) launch(w % nsets);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (int s = 0; s < steps; ++s) launch(s % nsets);
  CK(cudaStreamEndCapture(st, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, st));
  CK(cudaStreamSynchronize(st));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaEventRecord(e0, st));
    CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(e1, st));
    CK(cudaStreamSynchronize(st));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double us = best * 1e3 / steps;
  printf("vadv_l2 %dx%dx%d R=%d KB=%d NST=%d HINTS=%d tiles=%d smem=%d: %.2f us  %.0f GB/s  mismatches=%lld\n", ni, nj,
         nk, R, KB, NST, HINTS, tiles, SMEM, us, 40.0 * n / us * 1e-3, bad);
  return bad != 0;
}
