// Test-only: gts_div (shared-reciprocal division) must equal the IEEE
// quotient __ddiv_rn bit for bit.  Inputs: random bit patterns (all
// exponents, NaN/Inf/denormals included), random "typical" values, and a
// table of special values crossed with each other.
#include "gts_common.cuh"

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33; return x;
}

__constant__ double kSpecial[20];

__global__ void div_check(long long n, unsigned long long seed, unsigned long long* bad,
                          double* example) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; t < n; t += (long long)gridDim.x * blockDim.x) {
    unsigned long long h1 = mix(seed ^ (2 * t + 1)), h2 = mix(seed + 0x9e3779b97f4a7c15ULL * (t + 7));
    double a, b, c;
    int mode = (int)(h1 % 4);
    if (mode == 0) {  // raw bit patterns
      a = __longlong_as_double((long long)h1);
      b = __longlong_as_double((long long)h2);
    } else if (mode == 1) {  // typical magnitudes
      a = (double)(long long)(h1 >> 11) * 0x1.0p-53 * 2.0 - 1.0;
      b = (double)(long long)(h2 >> 11) * 0x1.0p-53 + 0.25;
    } else if (mode == 2) {  // wide exponent range, normal numbers
      a = ldexp(1.0 + (double)(h1 >> 12) * 0x1.0p-52, (int)(h1 % 2046) - 1022);
      b = ldexp(1.0 + (double)(h2 >> 12) * 0x1.0p-52, (int)(h2 % 2046) - 1022);
      if (h1 & 1) a = -a;
      if (h2 & 2) b = -b;
    } else {  // specials crossed with randoms
      a = kSpecial[h1 % 20];
      b = (h2 & 1) ? kSpecial[(h2 >> 1) % 20] : __longlong_as_double((long long)h2);
    }
    GtsRcp r = gts_rcp(b);
    double q1 = gts_div(a, r);
    // second quotient over the same reciprocal (the vadv pattern)
    c = a * 0.75 - 1.0;
    double q2 = gts_div(c, r);
    double w1 = __ddiv_rn(a, b), w2 = __ddiv_rn(c, b);
    if (__double_as_longlong(q1) != __double_as_longlong(w1) ||
        __double_as_longlong(q2) != __double_as_longlong(w2)) {
      unsigned long long old = atomicAdd(bad, 1ULL);
      if (old == 0) { example[0] = a; example[1] = b; example[2] = q1; example[3] = w1; }
    }
  }
}

extern "C" int run_div_check(long long n, unsigned long long seed, unsigned long long* mismatches,
                             double* example) {
  const double inf = __builtin_inf(), nan = __builtin_nan("");
  double sp[20] = {0.0, -0.0, 1.0, -1.0, inf, -inf, nan,
                   4.9406564584124654e-324, -4.9406564584124654e-324, 2.2250738585072014e-308,
                   2.2250738585072009e-308, 1.7976931348623157e308, -1.7976931348623157e308,
                   1e-300, 1e300, 3.0, 0.1, 1e-310, 6.5e-37, 1.5e-39};
  cudaMemcpyToSymbol(kSpecial, sp, sizeof(sp));
  unsigned long long* d_bad; double* d_ex;
  cudaMalloc(&d_bad, 8); cudaMalloc(&d_ex, 32);
  cudaMemset(d_bad, 0, 8);
  div_check<<<148 * 8, 256>>>(n, seed, d_bad, d_ex);
  cudaMemcpy(mismatches, d_bad, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(example, d_ex, 32, cudaMemcpyDeviceToHost);
  cudaFree(d_bad); cudaFree(d_ex);
  return (int)cudaGetLastError();
}
