// common.cuh -- shared device helpers for the eps-graph kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/epsgraph_b200.h"

namespace eg {

// ---------------------------------------------------------------- errors
void set_error(const char *fmt, ...);

#define EG_CUDA_TRY(expr)                                                     \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      ::eg::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,              \
                      cudaGetErrorString(_e));                                \
      return EG_ERR_CUDA;                                                     \
    }                                                                         \
  } while (0)

#define EG_LAUNCH_CHECK() EG_CUDA_TRY(cudaGetLastError())

// ------------------------------------------------------- instrumentation
// Every kernel launch is counted (eg_launch_count); when profiling is on,
// a pair of CUDA events brackets each launch (or launch group) on its
// stream and eg_profile_read() folds them into per-class milliseconds.
enum ProfClass {
  PC_ROW_STATS, PC_PROJECT, PC_FIXUP, PC_MSM_HIST, PC_MSM_SCAN, PC_MSM_SCATTER, PC_MSM_GROUP,
  PC_MSM_SPILL, PC_MSM_BATCH, PC_SORT_UPSWEEP, PC_SCAN, PC_SORT_DOWNSWEEP, PC_VERIFY,
  PC_COMPACT, PC_MISC, PC_MSM_STAGE, PC_SORT_STAGE, PC_VERIFY_STAGE, PC_COUNT
};
void prof_begin(int cls, cudaStream_t st, int launches);
void prof_end(int cls, cudaStream_t st);
struct ProfScope {
  int cls;
  cudaStream_t st;
  ProfScope(int c, cudaStream_t s, int launches = 1) : cls(c), st(s) { prof_begin(c, s, launches); }
  ~ProfScope() { prof_end(cls, st); }
};
#define EG_CAT2(a, b) a##b
#define EG_CAT(a, b) EG_CAT2(a, b)
#define EG_PROF(cls, st) ::eg::ProfScope EG_CAT(_eg_prof_, __LINE__)((cls), (st))
#define EG_PROF_GROUP(cls, st) ::eg::ProfScope EG_CAT(_eg_prof_, __LINE__)((cls), (st), 0)

// --------------------------------------------------------------- options
// Path overrides for tests and tuning, set through eg_set_option (never
// from the environment).  The defaults are the product's choices.
struct Options {
  int project_path = 0;          // 0 auto, 1 SIMT, 2 kind::tf32, 3 unfused norms, 4 non-TMA tc
  int fixup_force_seq = 0;       // 1: every band entry by the sequential fallback
  long long fixup_cap = 0;       // > 0: cap the fix-up entry list (overflow path)
  int msm_blocks = 0;            // > 0: force the block count (or a design's plan code); < 0: keep the reference's
  int msm_designs = 1;           // 0: the plan considers complete designs only
  int msm_streams = 2;           // 1: batches run on the caller's stream only
  int plan_debug = 0;            // 1: eg_msm_plan prints its candidates to stderr
  int msm_batches = 0;           // > 0: at least this many launch batches
  int verify_wide = 0;           // 1: warp-per-pair verify even for dim <= 128
  int sort_path = -1;            // -1 auto, 0 onesweep, 1 classic LSD passes
};
Options &options();

// ------------------------------------------------------------- workspace
// Bump allocator over the caller's workspace (256-byte aligned slices).
struct Arena {
  char *base;
  size_t size, used;
  __host__ Arena(void *b, size_t s) : base((char *)b), size(s), used(0) {}
  template <typename T>
  __host__ T *take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
    if (used + bytes > size) return nullptr;
    T *p = reinterpret_cast<T *>(base + used);
    used += bytes;
    return p;
  }
};
__host__ inline size_t ws_bytes(size_t count, size_t elem) {
  return (count * elem + 255) & ~size_t(255);
}

// ----------------------------------------------------------------- hashing
// 64-bit finaliser (murmur3 fmix64): equal keys -> equal hashes; distinct
// keys spread uniformly, so hash digits give balanced buckets even when the
// LSH bits themselves are heavily skewed (all-positive data, config 3).
__device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z ^= z >> 33;
  z *= 0xff51afd7ed558ccdULL;
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ULL;
  z ^= z >> 33;
  return z;
}

// Hash of a masked key: per word half of murmur3's fmix64 (xor-shift,
// one multiply, xor-shift): the pre-shift folds the high bits down, the
// multiply carries every bit upward into the top bits (the MSD bucket
// digit), the post-shift folds them into the low 32 bits (the in-bucket
// group key h2).  Equal keys give equal hashes and h2 collisions between
// distinct keys are removed by the exact compare, so only speed depends on
// the mixing.  EG_HASH_FMIX=1 restores the full finaliser.
#ifndef EG_HASH_FMIX
#define EG_HASH_FMIX 0
#endif
template <int W>
__device__ __forceinline__ uint64_t hash_key(const uint64_t (&c)[W], const uint64_t *kept,
                                             uint64_t salt) {
  uint64_t h = salt;
#if EG_HASH_FMIX
#pragma unroll
  for (int w = 0; w < W; ++w) h = fmix64(h ^ (c[w] & kept[w]) ^ (0x9e3779b97f4a7c15ULL * (w + 1)));
#else
#pragma unroll
  for (int w = 0; w < W; ++w) {
    h ^= (c[w] & kept[w]) ^ (0x9e3779b97f4a7c15ULL * (w + 1));
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdULL;
    h ^= h >> 33;
  }
#endif
  return h;
}

// ------------------------------------------------------------ block scan
// Exclusive scan of one value per thread over the CTA; returns the total.
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t &total,
                                                         uint32_t *smem_warp /*[NT/32]*/) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = lane < NT / 32 ? smem_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NT / 32) smem_warp[lane] = s;
  }
  __syncthreads();
  total = smem_warp[NT / 32 - 1];
  uint32_t warp_base = wid ? smem_warp[wid - 1] : 0;
  __syncthreads();
  return warp_base + x - v;
}

template <int NT>
__device__ __forceinline__ unsigned long long block_exclusive_scan64(
    unsigned long long v, unsigned long long &total, unsigned long long *smem_warp) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    unsigned long long s = lane < NT / 32 ? smem_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NT / 32) smem_warp[lane] = s;
  }
  __syncthreads();
  total = smem_warp[NT / 32 - 1];
  unsigned long long warp_base = wid ? smem_warp[wid - 1] : 0;
  __syncthreads();
  return warp_base + x - v;
}

// Warp-aggregated append: every converged lane with `pred` gets a unique
// slot (safe inside divergent loops: only the currently active lanes vote).
__device__ __forceinline__ unsigned long long warp_append(bool pred,
                                                          unsigned long long *counter) {
  const unsigned active = __activemask();
  const unsigned mask = __ballot_sync(active, pred);
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (mask) {
    const int leader = __ffs(mask) - 1;
    if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(mask));
    base = __shfl_sync(active, base, leader);
  }
  return base + __popc(mask & ((1u << lane) - 1u));
}

// Warp-aggregated append onto a shared-memory counter.  `active` is the
// lane set captured ONCE by the caller (the same mask must be used for the
// ballot and the broadcast: a second __activemask() may see a different set
// after divergence, and lanes outside the shuffle would read garbage);
// `mask` = __ballot_sync(active, pred).
__device__ __forceinline__ uint32_t smem_append(unsigned active, unsigned mask,
                                                uint32_t *counter) {
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(counter, (uint32_t)__popc(mask));
  base = __shfl_sync(active, base, leader);
  return base + __popc(mask & ((1u << lane) - 1u));
}

__host__ __device__ inline int ilog2_ceil(uint64_t v) {
  int l = 0;
  while ((1ull << l) < v) ++l;
  return l;
}

}  // namespace eg
