// project.cuh -- row statistics and the LSH projection with sign packing.
//
// Reference: lsh.py:96-113 (_sign_bits: bit = sequential fp64 sum of
// x[i,q]*r[t,q] > 0, multiply and add separately rounded), lsh.py:128-147
// (_project_words), bitpool.py:125-141 (little-endian packing).
//
// B200 design: the contraction n x D . D x (l*r) is evaluated once in fp32 on
// the SIMT pipes with register tiling (X tile staged transposed in shared
// memory, directions resident per K-slab); the epilogue decides every sign
// whose |s| exceeds a certified error band tau * ||x_i|| * ||r_t|| (warp
// ballot -> 32 packed bits per store) and appends the few in-band entries to
// a fix-up list that a second kernel recomputes exactly with __dmul_rn /
// __dadd_rn in ascending q (bit-identical to the reference).
#pragma once

#include "common.cuh"

namespace eg {

// ----------------------------------------------------------- row stats
constexpr int ROWST_WARPS = 4;
template <typename TX>
__global__ void __launch_bounds__(ROWST_WARPS * 32) k_row_stats(const TX *__restrict__ x, int64_t n,
                                                   int dim,
                                                   double *__restrict__ norms,
                                                   unsigned long long *__restrict__ bad) {
  // One warp per 32 rows: 32x32 tiles staged through shared memory with
  // coalesced loads; each lane then adds its own row's squares (fma, fp64)
  // into eight partial sums by (q mod 32 >= 16, q mod 4), each in ascending
  // q, combined pairwise -- the order the tensor-core projection's two
  // converter threads per row use, so both paths give bit-identical norms.
  __shared__ TX tile[ROWST_WARPS][32][33];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * ROWST_WARPS + wib) * 32;
  if (r0 >= n) return;
  const int64_t row = r0 + lane;
  // partial sums by (q mod 32 >= 16, q mod 4), each in ascending q
  double s8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  bool finite = true;
  for (int q0 = 0; q0 < dim; q0 += 32) {
    const int q = q0 + lane;
#pragma unroll 8
    for (int e = 0; e < 32; ++e)
      tile[wib][e][lane] = (r0 + e < n && q < dim) ? x[(r0 + e) * dim + q] : (TX)0;
    __syncwarp();
    // OOB columns are zero: fma(0, 0, s) == s, so every row sums 32 columns
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double v = (double)tile[wib][lane][j];
      finite &= isfinite(v);
      s8[(j >> 4) * 4 + (j & 3)] = fma(v, v, s8[(j >> 4) * 4 + (j & 3)]);
    }
    __syncwarp();
  }
  const double s = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
  if (row < n) {
    norms[row] = sqrt(s);
    if (!finite) atomicMin(&bad[0], (unsigned long long)row);
    if (s == 0.0) atomicMin(&bad[1], (unsigned long long)row);
  }
}

// --------------------------------------------------------- projection
constexpr int PJ_NT = 256;        // 8 warps
constexpr int PJ_BM = 64;         // rows per CTA (8 per warp)
constexpr int PJ_BK = 32;         // K slab
constexpr int PJ_TM = 8;          // rows per warp

struct FixupList {
  unsigned long long *count;      // device counter
  unsigned long long *items;      // (row << 32) | col
  unsigned long long cap;
};

// Transposed fp32 copy of the directions: rt[q * cols_pad + c] = (float)r[c*dim + q].
__global__ void k_prep_directions(const double *__restrict__ r, int cols, int dim, int cols_pad,
                                  float *__restrict__ rt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)dim * cols_pad;
  if (i >= total) return;
  int q = (int)(i / cols_pad), c = (int)(i % cols_pad);
  rt[i] = c < cols ? (float)r[(int64_t)c * dim + q] : 0.0f;
}

__device__ __forceinline__ void or_bits(uint64_t *codes, int64_t n, int L, int W, int64_t row,
                                        int c0, uint32_t bits, int nvalid) {
  int off = 0;
  while (off < nvalid) {
    int c = c0 + off;
    int h = c / L, t = c - h * L;
    int seg = min(nvalid - off, min(L - t, 64 - (t & 63)));
    uint64_t piece = (uint64_t)((bits >> off) & (seg >= 32 ? 0xffffffffu : ((1u << seg) - 1u)));
    if (piece) atomicOr((unsigned long long *)&codes[((int64_t)h * n + row) * W + (t >> 6)],
                        (unsigned long long)(piece << (t & 63)));
    off += seg;
  }
}

// TN column groups of 32 per warp per column pass (32*TN columns per pass).
template <typename TX, int TN>
__global__ void __launch_bounds__(PJ_NT) k_project(const TX *__restrict__ x, int64_t n, int dim,
                                                   const float *__restrict__ rt, int cols,
                                                   int cols_pad, const double *__restrict__ xnorm,
                                                   const double *__restrict__ rnorm, double tau,
                                                   int L, int W, uint64_t *__restrict__ codes,
                                                   FixupList fix) {
  __shared__ __align__(16) float xs[PJ_BK][PJ_BM];
  __shared__ __align__(16) float rs[PJ_BK][32 * TN];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t row0 = (int64_t)blockIdx.x * PJ_BM;
  // loader mapping for X: thread -> (row lr, 8 consecutive k)
  const int lr = threadIdx.x & 63, lk = (threadIdx.x >> 6) * 8;

  for (int c0 = 0; c0 < cols; c0 += 32 * TN) {
    float acc[PJ_TM][TN];
#pragma unroll
    for (int j = 0; j < PJ_TM; ++j)
#pragma unroll
      for (int m = 0; m < TN; ++m) acc[j][m] = 0.f;

    for (int k0 = 0; k0 < dim; k0 += PJ_BK) {
      __syncthreads();
      {  // X slab, transposed into xs[k][row]
        int64_t grow = row0 + lr;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          int q = k0 + lk + e;
          float v = 0.f;
          if (grow < n && q < dim) v = (float)x[grow * dim + q];
          xs[lk + e][lr] = v;
        }
      }
      // directions slab rs[k][c] from rt (k-major, contiguous in c)
      for (int i = threadIdx.x; i < PJ_BK * 32 * TN; i += PJ_NT) {
        int kk = i / (32 * TN), cc = i - kk * (32 * TN);
        int q = k0 + kk, c = c0 + cc;
        rs[kk][cc] = (q < dim && c < cols_pad) ? rt[(int64_t)q * cols_pad + c] : 0.f;
      }
      __syncthreads();
      const int kmax = min(PJ_BK, dim - k0);
      for (int kk = 0; kk < kmax; ++kk) {
        float4 a0 = *reinterpret_cast<const float4 *>(&xs[kk][wid * PJ_TM]);
        float4 a1 = *reinterpret_cast<const float4 *>(&xs[kk][wid * PJ_TM + 4]);
        float a[PJ_TM] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        float b[TN];
#pragma unroll
        for (int m = 0; m < TN; ++m) b[m] = rs[kk][lane + 32 * m];
#pragma unroll
        for (int j = 0; j < PJ_TM; ++j)
#pragma unroll
          for (int m = 0; m < TN; ++m) acc[j][m] = fmaf(a[j], b[m], acc[j][m]);
      }
    }
    // epilogue: certified sign decisions, packed by ballot
#pragma unroll
    for (int j = 0; j < PJ_TM; ++j) {
      const int64_t row = row0 + wid * PJ_TM + j;
      const bool row_ok = row < n;
      const double xn = row_ok ? xnorm[row] : 0.0;
#pragma unroll
      for (int m = 0; m < TN; ++m) {
        const int cbase = c0 + 32 * m;
        const int c = cbase + lane;
        const bool ok = row_ok && c < cols;
        bool pos = false, unc = false;
        if (ok) {
          double band = tau * xn * rnorm[c] + 1e-30;
          double s = (double)acc[j][m];
          pos = s > band;
          unc = !(s > band) && !(s < -band);
        }
        uint32_t bits = __ballot_sync(0xffffffffu, pos);
        if (lane == 0 && row_ok && cbase < cols)
          or_bits(codes, n, L, W, row, cbase, bits, min(32, cols - cbase));
        unsigned long long slot = warp_append(unc, fix.count);
        if (unc && slot < fix.cap)
          fix.items[slot] = ((unsigned long long)row << 32) | (unsigned)c;
      }
    }
  }
}

__device__ __forceinline__ void set_code_bit(uint64_t *codes, int64_t n, int L, int W,
                                             int64_t row, int c, bool one) {
  const int h = c / L, t = c - h * L;
  unsigned long long *w =
      (unsigned long long *)&codes[((int64_t)h * n + row) * W + (t >> 6)];
  if (one) atomicOr(w, 1ull << (t & 63));
  else atomicAnd(w, ~(1ull << (t & 63)));
}

// The reference's sign: sequential fp64 sum, separately rounded mul/add
// (lsh.py:107-112).  __dmul_rn/__dadd_rn are never contracted into DFMA.
template <typename TX>
__device__ __forceinline__ bool exact_sign(const TX *__restrict__ xr, const double *__restrict__ rr,
                                           int dim) {
  double acc = 0.0;
  for (int q = 0; q < dim; ++q) acc = __dadd_rn(acc, __dmul_rn((double)xr[q], rr[q]));
  return acc > 0.0;
}

// Exact recompute of listed (in-band) entries.
template <typename TX>
__global__ void k_fixup(const TX *__restrict__ x, int64_t n, int dim, const double *__restrict__ r,
                        int L, int W, uint64_t *__restrict__ codes,
                        const unsigned long long *__restrict__ items,
                        const unsigned long long *__restrict__ count, unsigned long long cap,
                        int cols) {
  const unsigned long long total = min(*count, cap);
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long it = items[i];
    const int64_t row = (int64_t)(it >> 32);
    const int c = (int)(it & 0xffffffffu);
    if (exact_sign<TX>(x + row * dim, r + (int64_t)c * dim, dim))
      set_code_bit(codes, n, L, W, row, c, true);
  }
}

// Band list overflowed (adversarial data): recompute every sign exactly.
// Exits immediately in the normal case.
template <typename TX>
__global__ void k_fixup_overflow(const TX *__restrict__ x, int64_t n, int dim,
                                 const double *__restrict__ r, int L, int W,
                                 uint64_t *__restrict__ codes,
                                 const unsigned long long *__restrict__ count,
                                 unsigned long long cap, int cols) {
  if (*count <= cap) return;
  const unsigned long long total = (unsigned long long)n * cols;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const int64_t row = (int64_t)(i / cols);
    const int c = (int)(i % cols);
    set_code_bit(codes, n, L, W, row, c, exact_sign<TX>(x + row * dim, r + (int64_t)c * dim, dim));
  }
}

}  // namespace eg
