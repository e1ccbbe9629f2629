// FP64 dependent-chain latency and throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lat(double *out, long long *cyc, int iters, double a) {
  double acc = threadIdx.x * 1e-3, m = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) acc = __dadd_rn(acc, __dmul_rn(m, acc));
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_tp(double *out, int iters, double a) {
  double acc[8];
  for (int j = 0; j < 8; ++j) acc[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn(a, acc[j]));
  double s = 0;
  for (int j = 0; j < 8; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double *d; long long *c; cudaMalloc(&d, 1 << 26); cudaMalloc(&c, 8);
  k_lat<<<1, 32>>>(d, c, 4096, 0.999); cudaDeviceSynchronize();
  k_lat<<<1, 32>>>(d, c, 4096, 0.999); long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  printf("dependent dmul+dadd: %.1f cycles per step\n", cy / 4096.0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  k_tp<<<148 * 8, 256>>>(d, iters, 0.999);
  cudaEventRecord(e0);
  k_tp<<<148 * 8, 256>>>(d, iters, 0.999);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 148.0 * 8 * 256 * iters * 8 * 2;
  printf("fp64 mul+add throughput: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
}
