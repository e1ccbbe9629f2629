// Throughput of the verify inner step acc = fma((double)a, (double)b, acc):
// F2F.F64.F32 conversions vs an integer-pipe widening of normal floats.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ double widen(float f) {
  const uint32_t u = __float_as_uint(f);
  // normal floats only: exponent re-biased by 896, mantissa shifted by 29
  const uint32_t hi = (u & 0x80000000u) | ((((u >> 23) & 0xffu) + 896u) << 20) | ((u & 0x7fffffu) >> 3);
  const uint32_t lo = u << 29;
  return __hiloint2double((int)hi, (int)lo);
}
template <int MODE>
__global__ void k(double *out, int iters, float s) {
  float x[8], y[8];
  double acc[8];
  for (int j = 0; j < 8; ++j) { x[j] = 1.0f + threadIdx.x * 1e-3f + j; y[j] = 0.5f + j; acc[j] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x[j] = fmaf(x[j], s, 1e-3f);
      y[j] = fmaf(y[j], s, 2e-3f);
      if (MODE == 0) acc[j] = fma((double)x[j], (double)y[j], acc[j]);
      if (MODE == 1) acc[j] = fma(widen(x[j]), widen(y[j]), acc[j]);
      if (MODE == 2) acc[j] = fma(acc[j], 0.999, (double)(x[j] * y[j]));   // one cvt
      if (MODE == 3) { float p = x[j] * y[j]; acc[j] += __hiloint2double(__float_as_int(p), __float_as_int(x[j])); }  // no cvt
    }
  }
  double t = 0;
  for (int j = 0; j < 8; ++j) t += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int MODE>
void run(const char *name, double *d) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2048;
  k<MODE><<<148 * 8, 256>>>(d, iters, 0.9999f);
  cudaEventRecord(e0);
  k<MODE><<<148 * 8, 256>>>(d, iters, 0.9999f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double steps = 148.0 * 8 * 256 * iters * 8;
  printf("%-28s %.3f ms  %.1f G steps/s  %.2f SM-cycles per 32 steps\n", name, ms, steps / ms / 1e6,
         ms * 1e-3 * 1.965e9 * 148 / (steps / 32));
}
int main() {
  double *d; cudaMalloc(&d, 1 << 26);
  run<0>("fma(cvt a, cvt b)", d);
  run<1>("fma(widen a, widen b)", d);
  run<2>("fma + one cvt", d);
  run<3>("dadd, no cvt", d);
}
