// verify.cuh -- exact verification of candidate pairs against epsilon.
//
// Reference: filter_exact (pipeline.py:183-223): x -> fp64, norms =
// sqrt(einsum(x.x)), dist = 1 - dot/(n_i n_j), clip [0, 2], keep dist <= eps
// (fp64 compare), lexsort (i, j).  Euclidean (north-star extension):
// ||x_i - x_j|| in fp64.
//
// One warp per pair: lanes stride the dimension with 16-byte loads, fp64
// accumulation of exact fp32 products, fixed butterfly reduction -- so a
// pair's distance is the same whichever unit, launch or GPU verifies it.
// Candidates arrive sorted by (i, j), so consecutive warps reuse x_i from L1/L2.
#pragma once

#include "common.cuh"

namespace eg {

template <typename TX>
__device__ __forceinline__ void accum_pair(const TX *__restrict__ xi, const TX *__restrict__ xj,
                                           int dim, int lane, int metric, double &acc) {
  if (sizeof(TX) == 4 && (dim & 3) == 0) {
    const float4 *a4 = reinterpret_cast<const float4 *>(xi);
    const float4 *b4 = reinterpret_cast<const float4 *>(xj);
    for (int q = lane; q < dim / 4; q += 32) {
      float4 a = __ldg(a4 + q), b = __ldg(b4 + q);
      if (metric == EG_METRIC_COSINE) {
        acc = fma((double)a.x, (double)b.x, acc);
        acc = fma((double)a.y, (double)b.y, acc);
        acc = fma((double)a.z, (double)b.z, acc);
        acc = fma((double)a.w, (double)b.w, acc);
      } else {
        double t;
        t = (double)a.x - (double)b.x; acc = fma(t, t, acc);
        t = (double)a.y - (double)b.y; acc = fma(t, t, acc);
        t = (double)a.z - (double)b.z; acc = fma(t, t, acc);
        t = (double)a.w - (double)b.w; acc = fma(t, t, acc);
      }
    }
  } else {
    for (int q = lane; q < dim; q += 32) {
      double a = (double)xi[q], b = (double)xj[q];
      if (metric == EG_METRIC_COSINE) acc = fma(a, b, acc);
      else { double t = a - b; acc = fma(t, t, acc); }
    }
  }
}

template <typename TX>
__global__ void __launch_bounds__(256) k_verify(const TX *__restrict__ x, int64_t n, int dim,
                                                const double *__restrict__ norms,
                                                const uint64_t *__restrict__ keys, int64_t m,
                                                int metric, double eps,
                                                uint8_t *__restrict__ flags,
                                                double *__restrict__ dist,
                                                unsigned long long *__restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * 8;
  for (int64_t p = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); p < m; p += warps) {
    const uint64_t key = keys[p];
    const int64_t i = (int64_t)(key >> 32), j = (int64_t)(key & 0xffffffffu);
    if (!(i < n && j < n)) {
      if (lane == 0) { atomicMin(bad, (unsigned long long)p); flags[p] = 0; dist[p] = 0.0; }
      continue;
    }
    double acc = 0.0;
    accum_pair<TX>(x + i * dim, x + j * dim, dim, lane, metric, acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      double dd;
      if (metric == EG_METRIC_COSINE) {
        dd = 1.0 - acc / (norms[i] * norms[j]);
        dd = dd < 0.0 ? 0.0 : (dd > 2.0 ? 2.0 : dd);
      } else {
        dd = sqrt(acc);
      }
      dist[p] = dd;
      flags[p] = dd <= eps;
    }
  }
}

}  // namespace eg
