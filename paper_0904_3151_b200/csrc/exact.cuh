// exact.cuh -- exhaustive all-pairs enumeration on the GPU (SURVEY.md 8(f)
// row 1): the ground truth of exact.brute_force_cosine / brute_force_hamming
// (reference exact.py:57-121) at sizes the reference's n <= 50k guard
// (exact.py:27) keeps the CPU away from.
//
// Cosine: the rows are scaled to unit length and rounded to fp16 once
// (k_unit_f16, zero-padded to a multiple of 64 columns); a tcgen05 kernel
// (kind::f16, fp32 accumulator in TMEM) forms every 128 x 256 tile of
// U U^T in the upper triangle and keeps the pairs whose approximate cosine
// is >= 1 - eps - delta.  delta bounds the fp16 rounding of both unit rows
// (2 * 2^-11 relative + the 2^-25 subnormal floor) and the fp32
// accumulation, with a 4x margin, so the screen never drops a true edge; the
// exact fp64 distance of each candidate is then computed by eg_verify
// (the reference's filter formula, pipeline.py:205-214), which also decides
// membership.
//
// Hamming: XOR + popcount over all pairs (SIMT; a 256-row block of codes in
// shared memory, each thread streams its j rows).
#pragma once

#include <cuda_fp16.h>

#include "project_h16.cuh"

namespace eg {

constexpr int BF_BK = 64;                   // K elements per chunk (128 B fp16 rows)
constexpr int BF_BM = 128, BF_BN = 256;     // i tile (UMMA M), j tile (UMMA N)
constexpr int BF_THREADS = 192;             // producer, MMA, 4 epilogue warps
constexpr size_t BF_ACHUNK = (size_t)BF_BM * 128, BF_BSTAGE = (size_t)BF_BN * 128;
constexpr int BF_MAXSTAGES = 8;

__host__ __device__ inline int bf_dpad(int dim) { return (dim + BF_BK - 1) / BF_BK * BF_BK; }

// u[i, q] = fp16(x[i, q] / |x_i|), zero for q >= dim (row stride dp).
template <typename TX>
__global__ void k_unit_f16(const TX *__restrict__ x, int64_t n, int dim, int dp,
                           const double *__restrict__ norms, __half *__restrict__ u) {
  const int64_t total = n * (int64_t)dp;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / dp;
    const int q = (int)(e - i * dp);
    const double v = q < dim ? (double)x[i * dim + q] / norms[i] : 0.0;
    u[e] = __double2half((float)v);
  }
}

struct BfBars {
  uint64_t afull, aempty, bfull[BF_MAXSTAGES], bempty[BF_MAXSTAGES], accfull[2], accempty[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ void bf_tma_load(void *dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// Candidate pairs (i < j, approximate cosine >= thr) of the fp16 unit rows,
// as keys (i << 32) | j in no particular order.  Every CTA owns i tiles
// I = g * gridDim.x + blockIdx.x (g = 0, 1, ...): the A tile stays resident
// in shared memory while the j tiles J >= I / 2 stream through a TMA ring;
// CTAs of one group walk the same j tiles a few tiles apart, so the stream
// is served from L2.
__global__ void __launch_bounds__(BF_THREADS, 1) k_bf_cosine_tc(
    const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
    int64_t n, int dp, int nb, float thr, unsigned long long *__restrict__ keys,
    unsigned long long cap, unsigned long long *__restrict__ count) {
  extern __shared__ __align__(1024) unsigned char bf_smem_raw[];
  unsigned char *smem = bf_smem_raw + ((1024u - (smem_u32(bf_smem_raw) & 1023u)) & 1023u);
  const int nkc = dp / BF_BK;
  unsigned char *abuf = smem;
  unsigned char *bring = smem + nkc * BF_ACHUNK;
  BfBars &B = *reinterpret_cast<BfBars *>(bring + nb * BF_BSTAGE);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ti = (n + BF_BM - 1) / BF_BM, tj = (n + BF_BN - 1) / BF_BN;

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&B.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&B.afull, 1);
    mbar_init(&B.aempty, 1);
    for (int s = 0; s < nb; ++s) {
      mbar_init(&B.bfull[s], 1);
      mbar_init(&B.bempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&B.accfull[b], 1);
      mbar_init(&B.accempty[b], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&amap) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&bmap) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t s = 0, ph = 0, ga = 0;
      for (int64_t I = blockIdx.x; I < ti; I += gridDim.x, ++ga) {
        mbar_wait(&B.aempty, (ga & 1) ^ 1);
        mbar_expect_tx(&B.afull, (uint32_t)(nkc * BF_ACHUNK));
        for (int kc = 0; kc < nkc; ++kc)
          bf_tma_load(abuf + kc * BF_ACHUNK, &amap, kc * BF_BK, (int)(I * BF_BM), &B.afull);
        for (int64_t J = I * BF_BM / BF_BN; J < tj; ++J) {
          for (int kc = 0; kc < nkc; ++kc) {
            mbar_wait(&B.bempty[s], ph ^ 1);
            mbar_expect_tx(&B.bfull[s], (uint32_t)BF_BSTAGE);
            bf_tma_load(bring + s * BF_BSTAGE, &bmap, kc * BF_BK, (int)(J * BF_BN), &B.bfull[s]);
            if (++s == (uint32_t)nb) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------------- MMA
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_f16(BF_BN);
      uint32_t s = 0, ph = 0, ga = 0, t = 0;
      for (int64_t I = blockIdx.x; I < ti; I += gridDim.x, ++ga) {
        mbar_wait(&B.afull, ga & 1);
        tc_fence_after();
        const uint32_t a0 = smem_u32(abuf);
        for (int64_t J = I * BF_BM / BF_BN; J < tj; ++J, ++t) {
          const uint32_t b = t & 1;
          mbar_wait(&B.accempty[b], ((t >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t dcol = tmem + b * BF_BN;
          for (int kc = 0; kc < nkc; ++kc) {
            mbar_wait(&B.bfull[s], ph);
            tc_fence_after();
            const uint32_t bs = smem_u32(bring + s * BF_BSTAGE);
#pragma unroll
            for (int j = 0; j < BF_BK / 16; ++j)
              umma_f16(dcol, umma_desc_sw128(a0 + kc * (uint32_t)BF_ACHUNK + j * 32),
                          umma_desc_sw128(bs + j * 32), idesc, (kc | j) ? 1u : 0u);
            umma_commit(&B.bempty[s]);
            if (++s == (uint32_t)nb) {
              s = 0;
              ph ^= 1;
            }
          }
          umma_commit(&B.accfull[b]);
        }
        umma_commit(&B.aempty);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;                       // TMEM lane quarter
    uint32_t t = 0;
    for (int64_t I = blockIdx.x; I < ti; I += gridDim.x) {
      const int64_t i = I * BF_BM + q * 32 + lane;
      for (int64_t J = I * BF_BM / BF_BN; J < tj; ++J, ++t) {
        const uint32_t b = t & 1;
        mbar_wait(&B.accfull[b], (t >> 1) & 1);
        tc_fence_after();
        uint32_t hit[BF_BN / 32];
        uint32_t nhit = 0;
#pragma unroll
        for (int g = 0; g < BF_BN / 32; ++g) {
          uint32_t v[32];
          tmem_ld32(tmem + b * BF_BN + ((uint32_t)(q * 32) << 16) + (uint32_t)(g * 32), v);
          uint32_t m = 0;
#pragma unroll
          for (int k = 0; k < 32; ++k) m |= (__uint_as_float(v[k]) >= thr ? 1u : 0u) << k;
          // valid j: i < j < n
          const int64_t j0 = J * BF_BN + g * 32;
          const int64_t lo = i + 1 - j0, hi = n - j0;     // keep k in [lo, hi)
          if (lo > 0) m &= lo >= 32 ? 0u : ~((1u << lo) - 1u);
          if (hi < 32) m &= hi <= 0 ? 0u : ((1u << hi) - 1u);
          if (i >= n) m = 0;
          hit[g] = m;
          nhit += __popc(m);
        }
        tc_fence_before();
        mbar_arrive(&B.accempty[b]);
        if (nhit) {
          unsigned long long pos = atomicAdd(count, (unsigned long long)nhit);
#pragma unroll
          for (int g = 0; g < BF_BN / 32; ++g) {
            uint32_t m = hit[g];
            while (m) {
              const int k = __ffs(m) - 1;
              m &= m - 1;
              if (pos < cap)
                keys[pos] = ((unsigned long long)i << 32) |
                            (unsigned long long)(J * BF_BN + g * 32 + k);
              ++pos;
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Hamming: all pairs (i < j) with popcount(c_i ^ c_j) <= d.  Each CTA takes
// a block of BFH_ROWS i rows into shared memory; its threads stream the j
// rows >= the block start and test each against the whole block.
constexpr int BFH_ROWS = 256, BFH_NT = 256, BFH_MAXW = 4;
__global__ void __launch_bounds__(BFH_NT) k_bf_hamming(
    const uint64_t *__restrict__ codes, int64_t n, int W, int d,
    unsigned long long *__restrict__ keys, unsigned long long cap,
    unsigned long long *__restrict__ count) {
  __shared__ uint64_t blk[BFH_MAXW][BFH_ROWS];
  const int64_t nblk = (n + BFH_ROWS - 1) / BFH_ROWS;
  for (int64_t bi = blockIdx.y; bi < nblk; bi += gridDim.y) {
    const int64_t i0 = bi * BFH_ROWS;
    const int rows = (int)min((int64_t)BFH_ROWS, n - i0);
    __syncthreads();
    for (int e = threadIdx.x; e < rows * W; e += BFH_NT) {
      const int r = e / W, w = e - r * W;
      blk[w][r] = codes[(i0 + r) * W + w];
    }
    __syncthreads();
    for (int64_t j = i0 + 1 + (int64_t)blockIdx.x * BFH_NT + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * BFH_NT) {
      uint64_t cj[BFH_MAXW];
#pragma unroll
      for (int w = 0; w < BFH_MAXW; ++w) cj[w] = w < W ? codes[j * W + w] : 0ull;
      const int rmax = (int)min((int64_t)rows, j - i0);    // i < j
      for (int r = 0; r < rmax; ++r) {
        int pc = 0;
#pragma unroll
        for (int w = 0; w < BFH_MAXW; ++w)
          if (w < W) pc += __popcll(cj[w] ^ blk[w][r]);
        if (pc <= d) {
          const unsigned long long pos = atomicAdd(count, 1ull);
          if (pos < cap) keys[pos] = ((unsigned long long)(i0 + r) << 32) | (unsigned long long)j;
        }
      }
    }
  }
}

}  // namespace eg
