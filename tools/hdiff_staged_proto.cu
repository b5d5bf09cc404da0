// Experiment (not product code): a stage-by-stage hdiff tile kernel that
// evaluates every temporary ONCE per point in shared memory -- the binary32
// input tile widened to binary64 once, lap over the tile + 1 halo ring, then
// flx / fly / out per column strip with the j-1 flux from the neighbour lane --
// instead of the template's register windows, which re-evaluate lap on the
// warp's halo rows and columns ("hdiff f32").  Checked
// bitwise against a C restatement of the reference numerics (NaN payloads
// aside) and timed like bench.py (CUDA graph of 200 launches over rotating
// sets larger than L2).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --fmad=false -lineinfo \
//        -I paper_2311_08322_b200/csrc/templates [-DTI=8|16|32] tools/hdiff_staged_proto.cu -o /tmp/hs
//
// Measured on one B200 (256x256x80): f32 23.2 us (TI=16; 26.2 at TI=8, 25.4 at
// TI=32) against 15.1 us for the register-window template, f64 22.2 us
// against 15.8.  ncu: 13.9 M warp instructions against 8.5 M (85 per point:
// the re-reads of the staged temporaries, selects and the lane-0 neighbour
// evaluation outweigh the recomputation they remove), 6.6 conversions per
// point against 7.75, 0.84 M shared-memory bank conflicts.  Not adopted.
#include "gts_common.cuh"
#include "gts_sm100.cuh"
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cmath>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

#ifndef TI
#define TI 16
#endif
constexpr int TJ = 128, NT = 256;
constexpr int BR = TI + 4, BC = TJ + 8;  // raw/wide box: rows -2..TI+1, cols -4..TJ+3
constexpr int LR = TI + 2, LC = TJ + 4;  // lap: rows -1..TI, cols -2..TJ+1
constexpr int RH = TI / 2;               // rows per thread in stage O

template <typename T> struct Sm {
  static constexpr int raw = BR * BC * sizeof(T);
  static constexpr int wide = sizeof(T) == 4 ? BR * BC * 8 : 0;
  static constexpr int lap = LR * LC * sizeof(T);
  static constexpr int off_wide = 2 * raw;
  static constexpr int off_lap = off_wide + wide;
  static constexpr int off_bar = (off_lap + lap + 15) / 16 * 16;
  static constexpr int total = off_bar + 16;
};

template <typename T>
__global__ void __launch_bounds__(NT) hdiff_staged(const __grid_constant__ CUtensorMap tm, T* __restrict__ out,
                                                   long long osi, long long osk, int ni, int nj, int tiles_i,
                                                   int tiles_j, int ntiles, double coeff) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = (uint64_t*)(smem + Sm<T>::off_bar);
  T* lap = (T*)(smem + Sm<T>::off_lap);
  const int t = threadIdx.x, lane = t & 31;
  if (t == 0) { gts_mbar_init(&full[0], 1); gts_mbar_init(&full[1], 1); gts_fence_mbar_init(); }
  __syncthreads();
  const int per = tiles_i * tiles_j;
  auto issue = [&](int tt, int b) {
    const int kk = tt / per, rem = tt - kk * per;
    const int ti = rem / tiles_j, tj = rem - ti * tiles_j;
    gts_mbar_arrive_expect_tx(&full[b], Sm<T>::raw);
    gts_tma_load_3d(smem + b * Sm<T>::raw, &tm, &full[b], tj * TJ, ti * TI, kk);
  };
  if (t == 0 && (int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int buf = it & 1;
    __syncthreads();  // previous tile's readers of wide / lap / raw[buf^1] are done
    if (t == 0 && tile + (int)gridDim.x < ntiles) { gts_fence_proxy_async(); issue(tile + gridDim.x, buf ^ 1); }
    gts_mbar_wait(&full[buf], (it >> 1) & 1);
    const int kk = tile / per, rem = tile - kk * per;
    const int ti = rem / tiles_j, tj = rem - ti * tiles_j;
    const int i0 = ti * TI, j0 = tj * TJ;
    const double* W;
    if constexpr (sizeof(T) == 4) {
      const float4* src = (const float4*)(smem + buf * Sm<T>::raw);
      double2* dst = (double2*)(smem + Sm<T>::off_wide);
      for (int q = t; q < BR * BC / 4; q += NT) {
        const float4 v = src[q];
        dst[2 * q] = make_double2((double)v.x, (double)v.y);
        dst[2 * q + 1] = make_double2((double)v.z, (double)v.w);
      }
      W = (const double*)(smem + Sm<T>::off_wide);
      __syncthreads();
    } else {
      W = (const double*)(smem + buf * Sm<T>::raw);
    }
#define WA(r, c) W[((r) + 2) * BC + (c) + 4]
#define LA(r, c) lap[((r) + 1) * LC + (c) + 2]
    // stage L: lap at rows -1..TI, cols -1..TJ
    {
      const int c = t & 127, h = t >> 7;
      const int r0 = h ? RH + 0 : -1, r1 = h ? TI : RH - 1;  // inclusive: -1..RH-1 and RH..TI
      double wm = WA(r0 - 1, c), w0 = WA(r0, c);
#pragma unroll
      for (int r = r0; r <= r1; ++r) {
        const double wp = WA(r + 1, c);
        const double v = 4.0 * w0 - (((wm + wp) + WA(r, c - 1)) + WA(r, c + 1));
        LA(r, c) = (T)v;
        wm = w0; w0 = wp;
      }
      if (t < 2 * (TI + 2)) {
        const int ce = t < TI + 2 ? -1 : TJ, r = (t < TI + 2 ? t : t - (TI + 2)) - 1;
        const double v = 4.0 * WA(r, ce) - (((WA(r - 1, ce) + WA(r + 1, ce)) + WA(r, ce - 1)) + WA(r, ce + 1));
        LA(r, ce) = (T)v;
      }
    }
    __syncthreads();
    // stage O: out at rows h*RH .. h*RH+RH-1, col c
    {
      const int c = t & 127, h = t >> 7;
      const int r0 = h * RH;
      const int j = j0 + c;
      auto flx_at = [&](int r) -> double {
        const T d = LA(r + 1, c) - LA(r, c);
        const bool z = (double)d * (WA(r + 1, c) - WA(r, c)) > 0.0;
        return z ? 0.0 : (double)d;
      };
      auto fly_at = [&](int r, int cc) -> double {
        const T d = LA(r, cc + 1) - LA(r, cc);
        const bool z = (double)d * (WA(r, cc + 1) - WA(r, cc)) > 0.0;
        return z ? 0.0 : (double)d;
      };
      double fxm = flx_at(r0 - 1);
      T* op = out + (long long)kk * osk + (long long)(i0 + r0) * osi + j;
#pragma unroll
      for (int r = r0; r < r0 + RH; ++r) {
        const double fx = flx_at(r);
        const double fy = fly_at(r, c);
        double fyl = __shfl_up_sync(0xffffffffu, fy, 1);
        if (lane == 0) fyl = fly_at(r, c - 1);
        const double v = WA(r, c) - coeff * (((fx - fxm) + fy) - fyl);
        if (i0 + r < ni && j < nj) *op = (T)v;
        op += osi;
        fxm = fx;
      }
    }
#undef WA
#undef LA
  }
}

// ---------------------------------------------------------------- host
template <typename T>
static void cpu_hdiff(const T* in, T* out, long long si, long long sk, long long osi, long long osk, int ni, int nj,
                      int nk, double coeff) {
  // in points at domain (0,0,0); halo 2 valid
  auto I = [&](int i, int j, int k) { return (double)in[(long long)k * sk + (long long)i * si + j]; };
  std::vector<T> lap((ni + 2) * (nj + 2)), flx((ni + 1) * nj), fly(ni * (nj + 1));
  for (int k = 0; k < nk; ++k) {
    for (int i = -1; i <= ni; ++i)
      for (int j = -1; j <= nj; ++j)
        lap[(i + 1) * (nj + 2) + j + 1] =
            (T)(4.0 * I(i, j, k) - (((I(i - 1, j, k) + I(i + 1, j, k)) + I(i, j - 1, k)) + I(i, j + 1, k)));
    auto L = [&](int i, int j) { return (double)lap[(i + 1) * (nj + 2) + j + 1]; };
    for (int i = -1; i < ni; ++i)
      for (int j = 0; j < nj; ++j) {
        double v;
        if ((L(i + 1, j) - L(i, j)) * (I(i + 1, j, k) - I(i, j, k)) > 0.0) v = 0.0; else v = L(i + 1, j) - L(i, j);
        flx[(i + 1) * nj + j] = (T)v;
      }
    for (int i = 0; i < ni; ++i)
      for (int j = -1; j < nj; ++j) {
        double v;
        if ((L(i, j + 1) - L(i, j)) * (I(i, j + 1, k) - I(i, j, k)) > 0.0) v = 0.0; else v = L(i, j + 1) - L(i, j);
        fly[i * (nj + 1) + j + 1] = (T)v;
      }
    for (int i = 0; i < ni; ++i)
      for (int j = 0; j < nj; ++j) {
        const double fx = flx[(i + 1) * nj + j], fxm = flx[i * nj + j];
        const double fy = fly[i * (nj + 1) + j + 1], fym = fly[i * (nj + 1) + j];
        out[(long long)k * osk + (long long)i * osi + j] = (T)(I(i, j, k) - coeff * (((fx - fxm) + fy) - fym));
      }
  }
}

static uint64_t rng = 88172645463325252ull;
static double urand() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return (rng >> 11) * (1.0 / 9007199254740992.0); }

template <typename T>
static int run(int ni, int nj, int nk, int nsets, int steps, int balance) {
  const int hi = 2, hj = 4;
  long long pitch = nj + 2 * hj;
  pitch = (pitch * sizeof(T) + 15) / 16 * 16 / sizeof(T);
  const long long si = pitch, sk = pitch * (ni + 2 * hi);
  const long long in_elems = sk * nk;
  const long long opitch = (nj * sizeof(T) + 15) / 16 * 16 / sizeof(T);
  const long long osi = opitch, osk = opitch * ni, out_elems = osk * nk;
  std::vector<T*> din(nsets), dout(nsets);
  std::vector<CUtensorMap> maps(nsets);
  std::vector<T> h0(in_elems);
  for (int s = 0; s < nsets; ++s) {
    std::vector<T> h(in_elems);
    for (auto& x : h) x = (T)(urand() * 2.0 - 1.0);
    if (s == 0) {  // a few special values
      h[sk * 3 + si * 7 + 9] = (T)INFINITY; h[sk * 4 + si * 50 + 60] = (T)NAN; h[sk * 5 + si * 20 + 33] = (T)-0.0;
      h[sk * 6 + si * 30 + 40] = (T)1e30; h[sk * 6 + si * 31 + 40] = (T)-1e30;
      for (int q = 0; q < 40; ++q) h[sk * 7 + si * (10 + q) + 100] = h[sk * 7 + si * 10 + 100];  // flat column
      h0 = h;
    }
    CK(cudaMalloc(&din[s], in_elems * sizeof(T)));
    CK(cudaMalloc(&dout[s], out_elems * sizeof(T)));
    CK(cudaMemcpy(din[s], h.data(), in_elems * sizeof(T), cudaMemcpyHostToDevice));
    CK(cudaMemset(dout[s], 0, out_elems * sizeof(T)));
    // map origin at domain (-2, -4): element hi-2=0 row, hj-4=0 col
    const T* origin = din[s];
    if (!gts_make_tmap_3d(&maps[s], origin, sizeof(T), nj + 8, ni + 4, nk, si, 1, sk, BC, BR, 1)) {
      printf("tmap failed\n"); return 1;
    }
  }
  const int tiles_i = (ni + TI - 1) / TI, tiles_j = (nj + TJ - 1) / TJ, ntiles = tiles_i * tiles_j * nk;
  const int smem = Sm<T>::total;
  CK(cudaFuncSetAttribute(hdiff_staged<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hdiff_staged<T>, NT, smem));
  int grid = per_sm * gts_sm_count();
  if (balance) { const int per_cta = (ntiles + grid - 1) / grid; grid = (ntiles + per_cta - 1) / per_cta; }
  if (grid > ntiles) grid = ntiles;
  const double coeff = 0.025;
  cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  auto launch = [&](int s) {
    hdiff_staged<T><<<grid, NT, smem, st>>>(maps[s], dout[s], osi, osk, ni, nj, tiles_i, tiles_j, ntiles, coeff);
  };
  launch(0);
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  // parity
  std::vector<T> got(out_elems), ref(out_elems, (T)0);
  CK(cudaMemcpy(got.data(), dout[0], out_elems * sizeof(T), cudaMemcpyDeviceToHost));
  cpu_hdiff<T>(h0.data() + hi * si + hj, ref.data(), si, sk, osi, osk, ni, nj, nk, coeff);
  long long bad = 0;
  for (int k = 0; k < nk; ++k)
    for (int i = 0; i < ni; ++i)
      for (int j = 0; j < nj; ++j) {
        const long long o = k * osk + i * osi + j;
        if (memcmp(&got[o], &ref[o], sizeof(T)) && !(got[o] != got[o] && ref[o] != ref[o])) { if (bad < 5) printf("mismatch %d %d %d: %g vs %g\n", i, j, k, (double)got[o], (double)ref[o]); ++bad; }
      }
  // timing: graph of `steps` launches over rotating sets
  for (int w = 0; w < 2 * nsets; ++w) launch(w % nsets);
  cudaGraph_t g; cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (int s = 0; s < steps; ++s) launch(s % nsets);
  CK(cudaStreamEndCapture(st, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, st));
  CK(cudaStreamSynchronize(st));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaEventRecord(e0, st));
    CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(e1, st));
    CK(cudaStreamSynchronize(st));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double us = best * 1e3 / steps;
  const double bytes = (double)sizeof(T) * ((double)(ni + 4) * (nj + 4) * nk + (double)ni * nj * nk);
  printf("%s %dx%dx%d TI=%d grid=%d per_sm=%d smem=%d: %.2f us  %.0f GB/s  mismatches=%lld\n",
         sizeof(T) == 4 ? "f32" : "f64", ni, nj, nk, TI, grid, per_sm, smem, us, bytes / us * 1e-3, bad);
  return bad != 0;
}

int main(int argc, char** argv) {
  int ni = argc > 1 ? atoi(argv[1]) : 256, nj = argc > 2 ? atoi(argv[2]) : 256, nk = argc > 3 ? atoi(argv[3]) : 80;
  int rc = 0;
  if (getenv("PROF")) { rc |= run<float>(ni, nj, nk, 2, 4, 0); rc |= run<double>(ni, nj, nk, 2, 4, 0); return rc; }
  for (int bal = 0; bal < 2; ++bal) {
    rc |= run<float>(ni, nj, nk, 8, 200, bal);
    rc |= run<double>(ni, nj, nk, 6, 200, bal);
  }
  rc |= run<float>(37, 300, 9, 3, 20, 0);
  rc |= run<double>(37, 300, 9, 3, 20, 0);
  return rc;
}
