// Micro-benchmarks of the instruction latencies / throughputs that bound the
// column (Thomas) and f32 tile kernels on B200.  Build + run on the box:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a --fmad=false -o /tmp/ub tools/ubench.cu && /tmp/ub
// Latency: one thread, a dependent chain of N ops timed with clock64.
// Throughput: 148 x 1024 threads, 8 independent chains each, timed with events.
#include <cstdio>
#include <cuda_runtime.h>

#define N 4096

__global__ void lat_dadd(double* out, double x, long long* cyc) {
  double a = x;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) a = a + x;
  long long t1 = clock64();
  out[0] = a; cyc[0] = t1 - t0;
}
__global__ void lat_dfma(double* out, double x, long long* cyc) {
  double a = x;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) a = fma(a, x, x);
  long long t1 = clock64();
  out[0] = a; cyc[0] = t1 - t0;
}
__global__ void lat_rcp(double* out, double x, long long* cyc) {
  double a = x;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a)); a = r; }
  long long t1 = clock64();
  out[0] = a; cyc[0] = t1 - t0;
}
__global__ void lat_div(double* out, double x, long long* cyc) {
  double a = x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) a = x / a;
  long long t1 = clock64();
  out[0] = a; cyc[0] = t1 - t0;
}
__global__ void lat_cvt(double* out, double x, long long* cyc) {
  double a = x;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) a = (double)(float)a;
  long long t1 = clock64();
  out[0] = a; cyc[0] = t1 - t0;
}

template <int OP>
__global__ void thr(double* out, double x) {
  double a[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) a[q] = x + q + threadIdx.x;
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (OP == 0) a[q] = a[q] + x;
      if (OP == 1) a[q] = (double)(float)a[q] + 1.0;  // 2 cvt + 1 dadd
      if (OP == 2) a[q] = (double)((float)a[q] + 1.0f);  // 2 cvt + 1 fadd
      if (OP == 3) a[q] = fma(a[q], x, x);
      if (OP == 4) {  // narrow + widen, nothing else (asm: no folding)
        float f; double d;
        asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(a[q]));
        asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(f));
        a[q] = d;
      }
      if (OP == 5) {  // widen only (+ an FADD to make a new float)
        float f = __double2float_rn(x) + (float)q;
        double d;
        asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(f));
        a[q] = a[q] + d;
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += a[q];
  if (s == 12345.0) out[0] = s;
}

template <class K>
float run_thr(K k, double* o) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<148 * 4, 256>>>(o, 1.0000001);
  cudaEventRecord(e0);
  k<<<148 * 4, 256>>>(o, 1.0000001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* o; long long* c; long long h;
  cudaMalloc(&o, 64); cudaMalloc(&c, 64);
  const char* names[] = {"DADD", "DFMA", "MUFU.RCP64H", "div.rn.f64 (full)", "f64->f32->f64"};
  void (*ks[])(double*, double, long long*) = {lat_dadd, lat_dfma, lat_rcp, lat_div, lat_cvt};
  for (int i = 0; i < 5; ++i) {
    ks[i]<<<1, 1>>>(o, 1.0000001, c); ks[i]<<<1, 1>>>(o, 1.0000001, c);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("latency %-20s %.1f cycles\n", names[i], (double)h / N);
  }
  const double ops = 148.0 * 4 * 256 * 256 * 8;
  float t;
  t = run_thr(thr<0>, o); printf("throughput DADD            %.1f Gop/s (%.1f /clk/SM @1.965GHz)\n", ops / t / 1e6, ops / t / 1e6 / 148 / 1.965);
  t = run_thr(thr<3>, o); printf("throughput DFMA            %.1f Gop/s (%.1f /clk/SM)\n", ops / t / 1e6, ops / t / 1e6 / 148 / 1.965);
  t = run_thr(thr<1>, o); printf("throughput 2cvt+DADD       %.1f Gop/s (%.1f groups/clk/SM)\n", ops / t / 1e6, ops / t / 1e6 / 148 / 1.965);
  t = run_thr(thr<2>, o); printf("throughput 2cvt+FADD       %.1f Gop/s (%.1f groups/clk/SM)\n", ops / t / 1e6, ops / t / 1e6 / 148 / 1.965);
  t = run_thr(thr<4>, o); printf("throughput cvt.f32.f64+cvt.f64.f32 %.1f Gop/s (%.1f pairs/clk/SM)\n", ops / t / 1e6, ops / t / 1e6 / 148 / 1.965);
  t = run_thr(thr<5>, o); printf("throughput cvt.f64.f32+DADD %.1f Gop/s (%.1f pairs/clk/SM)\n", ops / t / 1e6, ops / t / 1e6 / 148 / 1.965);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
