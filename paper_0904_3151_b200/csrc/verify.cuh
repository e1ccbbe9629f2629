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

// ------------------------------------------------- cluster-ordered verify
// Large clustered outputs (configs 4 and 5): the candidates of one row i
// (a "run" of the (i, j)-sorted keys) mostly pair i with the members of its
// cluster, and the runs of a cluster's rows share those j rows -- but
// consecutive i's belong to unrelated clusters (row ids are a random
// permutation), so the sorted-order sweep above streams every cluster's
// rows through L2 over and over (config 4: 109 GB of DRAM per build).
// Here the runs are visited in the order of their first j (equal for the
// rows of one cluster) in CH-pair chunks dealt grid-stride, so the groups
// resident at any moment work on the same few clusters and the j rows are
// served from L2.  Per-pair arithmetic is k_verify8's (same lanes, same
// slices, same butterfly): identical distances, written at the pairs'
// sorted positions.
constexpr int VR_CH = 256;        // pairs per work chunk

// run bounds per row: start[i] = first position of i's run, end[i] = one
// past its last (start preset to ~0 = no run)
__global__ void k_run_bounds(const uint64_t *__restrict__ keys, int64_t m, int64_t n,
                             uint32_t *__restrict__ start, uint32_t *__restrict__ end,
                             unsigned long long *__restrict__ bad) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(keys[p] >> 32);
    if ((int64_t)i >= n || (int64_t)(keys[p] & 0xffffffffu) >= n) {
      atomicMin(bad, (unsigned long long)p);
      continue;
    }
    if (p == 0 || (uint32_t)(keys[p - 1] >> 32) != i) start[i] = (uint32_t)p;
    if (p == m - 1 || (uint32_t)(keys[p + 1] >> 32) != i) end[i] = (uint32_t)(p + 1);
  }
}

// rows with a run -> (first j << 32 | i) run keys, appended in any order
__global__ void k_run_keys(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ start,
                           int64_t n, uint64_t *__restrict__ rkeys,
                           unsigned long long *__restrict__ count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t s = start[i];
    const bool has = s != 0xffffffffu;
    const unsigned long long slot = warp_append(has, count);
    if (has) rkeys[slot] = ((keys[s] & 0xffffffffull) << 32) | (uint64_t)i;
  }
}

// chunks of each sorted run (inclusive prefix, for the work-item search)
__global__ void k_run_chunks(const uint64_t *__restrict__ rkeys, int64_t R,
                             const uint32_t *__restrict__ start, const uint32_t *__restrict__ end,
                             uint32_t *__restrict__ nch) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)rkeys[r];
    nch[r] = (end[i] - start[i] + VR_CH - 1) / VR_CH;
  }
}

template <int LP, int VU8>
__global__ void __launch_bounds__(256) k_verify8_runs(
    const float *__restrict__ x, int64_t n, int dim, const double *__restrict__ norms,
    const uint64_t *__restrict__ keys, const uint64_t *__restrict__ rkeys,
    const uint32_t *__restrict__ cstart /* exclusive chunk prefix, R + 1 */, int64_t R,
    const uint32_t *__restrict__ start, const uint32_t *__restrict__ end, int metric, double eps,
    uint8_t *__restrict__ flags, double *__restrict__ dist) {
  const int lane = threadIdx.x & 31, gl = lane & (LP - 1);
  const int64_t groups = (int64_t)gridDim.x * (256 / LP);
  const int64_t gid = ((int64_t)blockIdx.x * 256 + threadIdx.x) / LP;
  const int d4 = dim / 4;
  const int64_t T = cstart[R];
  for (int64_t t = gid; t < T; t += groups) {
    // run r with cstart[r] <= t < cstart[r + 1]
    int64_t lo = 0, hi = R;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)cstart[mid] <= t) lo = mid; else hi = mid;
    }
    const uint32_t i = (uint32_t)rkeys[lo];
    const int64_t p0 = (int64_t)start[i] + (t - cstart[lo]) * VR_CH;
    const int64_t p1 = min((int64_t)end[i], p0 + VR_CH);
    float4 a[VU8];
    const float4 *xi = reinterpret_cast<const float4 *>(x + (int64_t)i * dim);
#pragma unroll
    for (int u = 0; u < VU8; ++u) {
      const int q = gl + LP * u;
      a[u] = q < d4 ? __ldg(xi + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const double ni = norms[i];
    for (int64_t p = p0; p < p1; ++p) {   // uniform within the LP-lane group
      const int64_t j = (int64_t)(keys[p] & 0xffffffffu);
      float4 b[VU8];
      const float4 *xj = reinterpret_cast<const float4 *>(x + j * dim);
#pragma unroll
      for (int u = 0; u < VU8; ++u) {
        const int q = gl + LP * u;
        b[u] = q < d4 ? __ldg(xj + q) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      double acc = 0.0;
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
      // the LP lanes of a group share p: the butterfly stays within the group
      const unsigned gmask = (LP == 32 ? 0xffffffffu : ((1u << LP) - 1u)) << (lane & ~(LP - 1));
#pragma unroll
      for (int o = LP / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(gmask, acc, o);
      if (gl == 0) {
        double dd;
        if (metric == EG_METRIC_COSINE) {
          dd = 1.0 - acc / (ni * norms[j]);
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

}  // namespace eg
