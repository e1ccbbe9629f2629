// plan.cuh -- sampled cost probe behind eg_msm_plan.
//
// The MSM output is the set {(i, j): popcount(c_i ^ c_j) <= d}, independent of
// the block count k (hamming_join.py:300-375): any partition
// of the code into k' > d blocks, with the canonical-mask rule taken over
// those k' blocks, emits every such pair exactly once.  The block count only
// trades the number of units C(k', d) (each a pass over all n rows) against
// the pairs visited inside equal-key groups (coarser keys -> bigger groups).
// Which side wins depends on the code distribution (skewed LSH bits make
// groups far larger than the uniform estimate), so eg_msm_plan measures it:
// every probe CTA hashes a strided sample of rows under one mask and counts
// sum_g C(g, 2) and the largest group with a shared-memory hash table.
#pragma once

#include "common.cuh"

namespace eg {

constexpr int PLAN_SAMPLE = 6144;          // rows per cost probe (max)
constexpr int PLAN_REF_SAMPLE = 2048;      // rows per oversize probe (max)
constexpr int PLAN_TABLE = 8192;           // load factor <= 0.75; 96 KB: two probe CTAs per SM
#ifndef EG_PLAN_NT
#define EG_PLAN_NT 1024   // 6 sampled rows per thread: the probe is latency-bound
#endif
constexpr int PLAN_NT = EG_PLAN_NT;
constexpr uint64_t PLAN_SALT = 0x6a09e667f3bcc909ULL;

// One CTA per probe.  kept[p][4]: bits of the code kept by probe p;
// sample[p]: rows it hashes (strided over [0, n)).
// out_pairs[p] = sum over sampled groups of C(g, 2); out_max[p] = max g.
template <int W>
__global__ void __launch_bounds__(PLAN_NT) k_msm_plan(const uint64_t *__restrict__ codes,
                                                      int64_t n,
                                                      const int *__restrict__ sample,
                                                      const unsigned long long *__restrict__ kept,
                                                      unsigned long long *out_pairs,
                                                      uint32_t *out_max) {
  extern __shared__ unsigned long long ptab[];      // [PLAN_TABLE] keys
  uint32_t *pcnt = reinterpret_cast<uint32_t *>(ptab + PLAN_TABLE);
  __shared__ unsigned long long red[PLAN_NT / 32];
  __shared__ uint32_t redm[PLAN_NT / 32];
  const int p = blockIdx.x;
  const int S = sample[p];
  uint64_t kp[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) kp[w] = kept[p * 4 + w];
  for (int i = threadIdx.x; i < PLAN_TABLE; i += PLAN_NT) {
    ptab[i] = ~0ull;
    pcnt[i] = 0;
  }
  __syncthreads();
  unsigned long long my_pairs = 0;
  for (int i = threadIdx.x; i < S; i += PLAN_NT) {
    const int64_t row = (int64_t)i * n / S;         // strided, deterministic
    uint64_t c[W];
#pragma unroll
    for (int w = 0; w < W; ++w) c[w] = __ldg(codes + row * W + w);
    uint64_t h = hash_key<W>(c, kp, PLAN_SALT);
    if (h == ~0ull) h = ~1ull;
    uint32_t slot = (uint32_t)h & (PLAN_TABLE - 1);
    while (true) {
      const unsigned long long old = atomicCAS(&ptab[slot], ~0ull, h);
      if (old == ~0ull || old == h) break;
      slot = (slot + 1) & (PLAN_TABLE - 1);
    }
    my_pairs += atomicAdd(&pcnt[slot], 1u);          // rank within the group
  }
  __syncthreads();
  uint32_t my_max = 0;
  for (int i = threadIdx.x; i < PLAN_TABLE; i += PLAN_NT) my_max = max(my_max, pcnt[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    my_pairs += __shfl_xor_sync(0xffffffffu, my_pairs, o);
    my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    red[wid] = my_pairs;
    redm[wid] = my_max;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    uint32_t m = 0;
    for (int w = 0; w < PLAN_NT / 32; ++w) {
      t += red[w];
      m = max(m, redm[w]);
    }
    out_pairs[p] = t;
    out_max[p] = m;
  }
}

// ------------------------------------------------------- output estimate
// Pairs with popcount(c_a ^ c_b) <= d among a strided sample of S rows of
// each probed replicate (the MSM output restricted to the sample), for the
// output-capacity estimate of eg_msm_estimate_pairs.  Grid: (tile pairs,
// replicates); 256-row tiles staged in shared memory.
constexpr int EST_SAMPLE = 8192, EST_T = 256, EST_MAXREPS = 4;
__global__ void __launch_bounds__(EST_T) k_est_pairs(const uint64_t *__restrict__ codes, int64_t n,
                                                     int W, int S, int d,
                                                     unsigned long long *__restrict__ out) {
  __shared__ uint64_t tb[EST_T * 4];
  __shared__ unsigned long long red[EST_T / 32];
  const int nt = (S + EST_T - 1) / EST_T;
  // tile pair (ta <= tb) of the upper triangle, row-major
  int ta = 0, rem = blockIdx.x;
  while (rem >= nt - ta) { rem -= nt - ta; ++ta; }
  const int tbi = ta + rem;
  const uint64_t *cr = codes + (int64_t)blockIdx.y * n * W;
  auto row_of = [&](int s) { return (int64_t)((double)s * (double)n / (double)S); };
  for (int i = threadIdx.x; i < EST_T * W; i += EST_T) {
    const int s = tbi * EST_T + i / W;
    tb[i] = s < S ? cr[row_of(s) * W + i % W] : 0ull;
  }
  uint64_t a[4] = {0, 0, 0, 0};
  const int sa = ta * EST_T + threadIdx.x;
  if (sa < S)
    for (int w = 0; w < W; ++w) a[w] = cr[row_of(sa) * W + w];
  __syncthreads();
  unsigned long long c = 0;
  if (sa < S) {
    const int j0 = ta == tbi ? threadIdx.x + 1 : 0;
    for (int j = j0; j < EST_T && tbi * EST_T + j < S; ++j) {
      int pc = 0;
      for (int w = 0; w < W; ++w) pc += __popcll(a[w] ^ tb[j * W + w]);
      c += pc <= d;
    }
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int i = 0; i < EST_T / 32; ++i) t += red[i];
    if (t) atomicAdd(out, t);
  }
}

}  // namespace eg
