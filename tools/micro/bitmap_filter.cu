// Microbenchmark: L2-resident bitmap duplicate filter for masked keys.
// pass 1: atomicOr into a per-unit "seen" bitmap, second arrivals set "dup";
// pass 2: every element reads "dup" -> candidate count.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <random>
__device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z ^= z >> 33; z *= 0xff51afd7ed558ccdULL; z ^= z >> 33; z *= 0xc4ceb9fe1a85ec53ULL; z ^= z >> 33; return z;
}
struct Units { uint64_t kept[32]; uint64_t salt[32]; };
template <int RPT>
__global__ void __launch_bounds__(256) k_pass1(const uint64_t *__restrict__ codes, int n, Units U, int nu,
                                              int lgbits, uint32_t *seen, uint32_t *dup) {
  const size_t words = size_t(1) << (lgbits - 5);
  int base = (blockIdx.x * 256 * RPT) + threadIdx.x;
  uint64_t c[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) c[i] = (base + i * 256 < n) ? codes[base + i * 256] : 0;
  for (int u = 0; u < nu; ++u) {
    const uint64_t kept = U.kept[u], salt = U.salt[u];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      if (base + i * 256 >= n) continue;
      uint64_t h = fmix64(salt ^ (c[i] & kept));
      uint32_t idx = (uint32_t)(h >> (64 - lgbits));
      uint32_t bit = 1u << (idx & 31);
      uint32_t old = atomicOr(seen + u * words + (idx >> 5), bit);
      if (old & bit) atomicOr(dup + u * words + (idx >> 5), bit);
    }
  }
}
template <int RPT>
__global__ void __launch_bounds__(256) k_pass2(const uint64_t *__restrict__ codes, int n, Units U, int nu,
                                              int lgbits, const uint32_t *dup, unsigned long long *cnt) {
  const size_t words = size_t(1) << (lgbits - 5);
  int base = (blockIdx.x * 256 * RPT) + threadIdx.x;
  uint64_t c[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) c[i] = (base + i * 256 < n) ? codes[base + i * 256] : 0;
  uint32_t my = 0;
  for (int u = 0; u < nu; ++u) {
    const uint64_t kept = U.kept[u], salt = U.salt[u];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      if (base + i * 256 >= n) continue;
      uint64_t h = fmix64(salt ^ (c[i] & kept));
      uint32_t idx = (uint32_t)(h >> (64 - lgbits));
      uint32_t bit = 1u << (idx & 31);
      if (__ldcg(dup + u * words + (idx >> 5)) & bit) ++my;
    }
  }
  for (int o = 16; o; o >>= 1) my += __shfl_xor_sync(~0u, my, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(cnt, (unsigned long long)my);
}
int main() {
  const int n = 1600000;
  std::vector<uint64_t> h(n);
  std::mt19937_64 g(1);
  for (int i = 0; i < n; ++i) h[i] = g() & ((1ull << 48) - 1);
  for (int i = 0; i < n / 100; ++i) h[g() % n] = h[g() % n];   // some duplicates
  uint64_t *d; cudaMalloc(&d, n * 8); cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  Units U;
  for (int u = 0; u < 32; ++u) { uint64_t m = (1ull<<48)-1; for (int b=0;b<3;++b){int blk=(u*7+b*5)%12; m &= ~(0xFull << (4*blk));} U.kept[u]=m; U.salt[u]=0x2545f4914f6cdd1dULL*(u+1); }
  uint32_t *seen, *dup; unsigned long long *cnt;
  cudaMalloc(&seen, size_t(256) << 20); cudaMalloc(&dup, size_t(256) << 20); cudaMalloc(&cnt, 8);
  cudaEvent_t e0, e1, e2; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
  for (int lg : {23, 24, 25, 26}) for (int nu : {4, 8, 16}) {
    size_t bytes = (size_t(1) << (lg - 3)) * nu;
    if (bytes > (size_t(256) << 20)) continue;
    float t1s = 0, t2s = 0; unsigned long long c = 0;
    for (int rep = 0; rep < 6; ++rep) {
      cudaMemsetAsync(seen, 0, bytes); cudaMemsetAsync(dup, 0, bytes); cudaMemsetAsync(cnt, 0, 8);
      cudaEventRecord(e0);
      k_pass1<4><<<(n + 1023) / 1024, 256>>>(d, n, U, nu, lg, seen, dup);
      cudaEventRecord(e1);
      k_pass2<4><<<(n + 1023) / 1024, 256>>>(d, n, U, nu, lg, dup, cnt);
      cudaEventRecord(e2); cudaEventSynchronize(e2);
      float a, b; cudaEventElapsedTime(&a, e0, e1); cudaEventElapsedTime(&b, e1, e2);
      if (rep >= 2) { t1s += a; t2s += b; }
      cudaMemcpy(&c, cnt, 8, cudaMemcpyDeviceToHost);
    }
    printf("lgbits %d units %2d bitmap %6.1f MB: pass1 %.3f ms pass2 %.3f ms  per-unit %.4f ms  cand frac %.4f\n",
           lg, nu, 2.0 * bytes / 1e6, t1s / 4, t2s / 4, (t1s + t2s) / 4 / nu, double(c) / (double(n) * nu));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
