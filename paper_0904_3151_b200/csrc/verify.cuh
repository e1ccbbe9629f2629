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

// Fast path (fp32 rows, dim % 4 == 0, dim <= 512): each warp takes a
// contiguous run of the (i, j)-sorted candidates, so consecutive pairs share
// x_i, which stays in registers (each lane holds its <= 4 float4 slices);
// only x_j is loaded per pair, all of a lane's slices at once.  Same
// per-lane summation order as accum_pair, so distances are identical.
constexpr int VER_VU = 4;
template <int VU>
__device__ __forceinline__ void ver_load_row(const float *__restrict__ xr, int d4, int lane,
                                             float4 (&v)[VU]) {
  const float4 *x4 = reinterpret_cast<const float4 *>(xr);
#pragma unroll
  for (int u = 0; u < VU; ++u) {
    const int q = lane + 32 * u;
    v[u] = q < d4 ? __ldg(x4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// VU = ceil(dim / 128) float4 slices per lane on the fast path (0: general path)
template <typename TX, int VU>
__global__ void __launch_bounds__(256) k_verify(const TX *__restrict__ x, int64_t n, int dim,
                                                const double *__restrict__ norms,
                                                const uint64_t *__restrict__ keys, int64_t m,
                                                int metric, double eps,
                                                uint8_t *__restrict__ flags,
                                                double *__restrict__ dist,
                                                unsigned long long *__restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * 8;
  const int64_t wid = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if constexpr (VU > 0) {
    const int d4 = dim / 4;
    const int64_t per = (m + warps - 1) / warps;
    const int64_t p0 = wid * per, p1 = min(m, p0 + per);
    int64_t cur = -1;
    float4 a[VU];
    for (int64_t p = p0; p < p1; ++p) {
      const uint64_t key = keys[p];
      const int64_t i = (int64_t)(key >> 32), j = (int64_t)(key & 0xffffffffu);
      if (!(i < n && j < n)) {
        if (lane == 0) { atomicMin(bad, (unsigned long long)p); flags[p] = 0; dist[p] = 0.0; }
        continue;
      }
      float4 b[VU];
      ver_load_row(reinterpret_cast<const float *>(x) + j * dim, d4, lane, b);
      if (i != cur) {
        ver_load_row(reinterpret_cast<const float *>(x) + i * dim, d4, lane, a);
        cur = i;
      }
      double acc = 0.0;
#pragma unroll
      for (int u = 0; u < VU; ++u) {
        if (lane + 32 * u >= d4) break;
        if (metric == EG_METRIC_COSINE) {
          acc = fma((double)a[u].x, (double)b[u].x, acc);
          acc = fma((double)a[u].y, (double)b[u].y, acc);
          acc = fma((double)a[u].z, (double)b[u].z, acc);
          acc = fma((double)a[u].w, (double)b[u].w, acc);
        } else {
          double t;
          t = (double)a[u].x - (double)b[u].x; acc = fma(t, t, acc);
          t = (double)a[u].y - (double)b[u].y; acc = fma(t, t, acc);
          t = (double)a[u].z - (double)b[u].z; acc = fma(t, t, acc);
          t = (double)a[u].w - (double)b[u].w; acc = fma(t, t, acc);
        }
      }
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
  } else {
    for (int64_t p = wid; p < m; p += warps) {
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
}

// Narrow rows (fp32, dim % 4 == 0, dim <= 128): LP lanes per pair, 32 / LP
// pairs per warp step.  Each LP-lane group walks its own contiguous run of
// the (i, j)-sorted candidates, keeps x_i in registers across a run of equal
// i, adds lane-local products in ascending slice order and reduces over the
// group with a fixed butterfly (xor LP/2, ..., 1) -- one summation order for
// every pair of a given shape, so distances stay per-pair deterministic.
template <int LP, int VU8>
__global__ void __launch_bounds__(256) k_verify8(const float *__restrict__ x, int64_t n, int dim,
                                                 const double *__restrict__ norms,
                                                 const uint64_t *__restrict__ keys, int64_t m,
                                                 int metric, double eps,
                                                 uint8_t *__restrict__ flags,
                                                 double *__restrict__ dist,
                                                 unsigned long long *__restrict__ bad) {
  const int lane = threadIdx.x & 31, gl = lane & (LP - 1);
  const int64_t groups = (int64_t)gridDim.x * (256 / LP);
  const int64_t gid = ((int64_t)blockIdx.x * 256 + threadIdx.x) / LP;
  const int d4 = dim / 4;
  const int64_t per = (m + groups - 1) / groups;
  const int64_t p0 = gid * per, p1 = min(m, p0 + per);
  const int64_t steps = per;                 // uniform trip count across the warp
  int64_t cur = -1;
  float4 a[VU8];
  for (int64_t t = 0; t < steps; ++t) {
    const int64_t p = p0 + t;
    const bool live = p < p1;
    const uint64_t key = live ? keys[p] : 0ull;
    const int64_t i = (int64_t)(key >> 32), j = (int64_t)(key & 0xffffffffu);
    const bool ok = live && i < n && j < n;
    if (live && !ok && gl == 0) { atomicMin(bad, (unsigned long long)p); flags[p] = 0; dist[p] = 0.0; }
    float4 b[VU8];
    const float4 *xj = reinterpret_cast<const float4 *>(x + (ok ? j : 0) * dim);
#pragma unroll
    for (int u = 0; u < VU8; ++u) {
      const int q = gl + LP * u;
      b[u] = (ok && q < d4) ? __ldg(xj + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (ok && i != cur) {
      const float4 *xi = reinterpret_cast<const float4 *>(x + i * dim);
#pragma unroll
      for (int u = 0; u < VU8; ++u) {
        const int q = gl + LP * u;
        a[u] = q < d4 ? __ldg(xi + q) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      cur = i;
    }
    double acc = 0.0;
    if (ok) {
#pragma unroll
      for (int u = 0; u < VU8; ++u) {
        if (gl + LP * u >= d4) break;
        if (metric == EG_METRIC_COSINE) {
          acc = fma((double)a[u].x, (double)b[u].x, acc);
          acc = fma((double)a[u].y, (double)b[u].y, acc);
          acc = fma((double)a[u].z, (double)b[u].z, acc);
          acc = fma((double)a[u].w, (double)b[u].w, acc);
        } else {
          double tt;
          tt = (double)a[u].x - (double)b[u].x; acc = fma(tt, tt, acc);
          tt = (double)a[u].y - (double)b[u].y; acc = fma(tt, tt, acc);
          tt = (double)a[u].z - (double)b[u].z; acc = fma(tt, tt, acc);
          tt = (double)a[u].w - (double)b[u].w; acc = fma(tt, tt, acc);
        }
      }
    }
#pragma unroll
    for (int o = LP / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (ok && gl == 0) {
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
