// project_tc.cuh -- LSH projection on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulator in TMEM), 3xTF32 split precision,
// with the certified sign band + exact fp64 fix-up of project.cuh.
//
// Reference: lsh.py:96-113 (_sign_bits), lsh.py:128-147 (_project_words),
// bitpool.py:125-141 (packing).  D = X . R^T with X n x dim fp32 rows and
// R (replicates*length) x dim fp64 directions.
//
// Split: x = xh + xl with xh = x with the low 13 mantissa bits cleared
// (exactly representable in TF32) and xl = x - xh (exact in fp32); the
// directions likewise r ~ rh + rl.  D ~= xh.rh + xh.rl + xl.rh, accumulated
// in fp32 in TMEM.  The epilogue decides every sign with |D| > tau * |x| |r|
// (tau bounds the split + accumulation error, see tc_tau()); the rest are
// listed for the exact fp64 recompute (k_fixup), so the packed codes equal
// the reference's sequential-fp64 signs bit for bit.
//
// Per CTA (128 threads, persistent over 128-row tiles): for each 32-wide K
// chunk the threads load the X chunk (one row per thread), split it and
// store xh/xl into a 128B-swizzled K-major tile; the pre-swizzled rh/rl
// chunk images are copied in; thread 0 issues 12 MMAs (M=128, N=cols,
// K=8 x 4 steps x 3 terms) and commits them to the stage's mbarrier.  Two
// stages overlap the next chunk's loads with the current MMAs.  After the
// last chunk of a tile, tcgen05.ld brings row t of the accumulator to
// thread t, which packs its signs into the row's code words.
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "project.cuh"

namespace eg {

constexpr int TC_M = 128;       // rows per tile (UMMA M)
constexpr int TC_BK = 32;       // fp32 elements per K chunk = one 128B swizzle row
constexpr int TC_NT = 128;      // threads per CTA
constexpr int TC_MAXN = 256;    // UMMA N limit (cols per pass)

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity));
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B: 8-row groups of
// 128-byte rows at SBO = 1024 B; LBO unused (1); version 1 (sm100).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)1 << 16;                 // LBO (16 B units)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO
  d |= (uint64_t)1 << 46;                 // version
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

// Instruction descriptor: D f32, A/B tf32, K-major both, N, M=128.
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(TC_M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
      smem_u32(bar)));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
        "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Byte offset of (row, 16-byte chunk c) in a 128B-swizzled K-major tile.
__host__ __device__ __forceinline__ uint32_t sw128_off(uint32_t row, uint32_t c) {
  return row * 128u + ((c ^ (row & 7u)) << 4);
}

__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xffffe000u);
}

// Pre-swizzled direction images: img[(kc * 2 + part) * npad * 32 + swizzled]
// with part 0 = rh (tf32-exact), 1 = rl = tf32-rounded residual.
__global__ void k_tc_prep_directions(const double *__restrict__ r, int cols, int dim, int npad,
                                     float *__restrict__ img) {
  const int nkc = (dim + TC_BK - 1) / TC_BK;
  const int64_t total = (int64_t)nkc * npad * TC_BK;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int kc = (int)(i / ((int64_t)npad * TC_BK));
    const int rem = (int)(i % ((int64_t)npad * TC_BK));
    const int n = rem / TC_BK, kk = rem % TC_BK;
    const int q = kc * TC_BK + kk;
    double v = (n < cols && q < dim) ? r[(int64_t)n * dim + q] : 0.0;
    float hi = tf32_hi((float)v);
    float lo = (float)(v - (double)hi);
    const uint32_t off = sw128_off((uint32_t)n, (uint32_t)(kk >> 2)) / 4 + (kk & 3);
    float *base = img + (int64_t)kc * 2 * npad * TC_BK;
    base[off] = hi;
    base[(int64_t)npad * TC_BK + off] = lo;
  }
}

struct TcSmem {
  // two stages; each: xh [128][32], xl [128][32], rh [npad][32], rl [npad][32]
  // (sizes depend on npad, carved from the dynamic buffer)
  uint64_t bar[2];
  uint64_t done;
  uint32_t tmem_base;
};

__host__ __device__ inline size_t tc_stage_bytes(int npad) {
  return (size_t)(2 * TC_M + 2 * npad) * TC_BK * 4;
}

// 1024-byte aligned dynamic smem: [stage0][stage1][TcSmem]
__global__ void __launch_bounds__(TC_NT, 1) k_project_tc(
    const float *__restrict__ x, int64_t n, int dim, const float *__restrict__ img, int cols,
    int npad, const double *__restrict__ xnorm, const double *__restrict__ rnorm, double tau,
    int L, int W, uint64_t *__restrict__ codes, FixupList fix, float *__restrict__ dbg) {
  extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
  // align the stage buffers to 1024 B in the shared window (SW128 atoms)
  unsigned char *smem = tc_smem_raw + ((1024u - (smem_u32(tc_smem_raw) & 1023u)) & 1023u);
  const size_t sb = tc_stage_bytes(npad);
  TcSmem &S = *reinterpret_cast<TcSmem *>(smem + 2 * sb);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nkc = (dim + TC_BK - 1) / TC_BK;
  const uint32_t ncols_alloc = npad <= 32 ? 32 : npad <= 64 ? 64 : npad <= 128 ? 128 : 256;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&S.tmem_base)),
                 "r"(ncols_alloc));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    mbar_init(&S.done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  const uint32_t idesc = umma_idesc_tf32(npad);
  uint32_t phase[2] = {0, 0}, done_phase = 0;
  uint32_t issued[2] = {0, 0};   // outstanding commit on stage s

  const int64_t ntiles = (n + TC_M - 1) / TC_M;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * TC_M;
    const int64_t grow = row0 + tid;
    const bool row_ok = grow < n;
    const float *xr = x + (row_ok ? grow : 0) * dim;
    for (int kc = 0; kc < nkc; ++kc) {
      const int s = kc & 1;
      unsigned char *st = smem + s * sb;
      // this thread's row chunk (issue loads before waiting on the stage)
      float4 v[8];
      const int q0 = kc * TC_BK;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int q = q0 + c * 4;
        v[c] = (row_ok && q < dim) ? __ldg(reinterpret_cast<const float4 *>(xr + q))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (issued[s]) {   // MMAs that read this stage two chunks ago
        mbar_wait(&S.bar[s], phase[s]);
        phase[s] ^= 1;
        issued[s] = 0;
      }
      float *xh = reinterpret_cast<float *>(st);
      float *xl = xh + TC_M * TC_BK;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float4 h = make_float4(tf32_hi(v[c].x), tf32_hi(v[c].y), tf32_hi(v[c].z), tf32_hi(v[c].w));
        float4 l = make_float4(v[c].x - h.x, v[c].y - h.y, v[c].z - h.z, v[c].w - h.w);
        const uint32_t off = sw128_off((uint32_t)tid, (uint32_t)c) / 4;
        *reinterpret_cast<float4 *>(xh + off) = h;
        *reinterpret_cast<float4 *>(xl + off) = l;
      }
      {  // direction images (L2-resident, pre-swizzled): straight 16B copies
        const float4 *src = reinterpret_cast<const float4 *>(img + (int64_t)kc * 2 * npad * TC_BK);
        float4 *dst = reinterpret_cast<float4 *>(xl + TC_M * TC_BK);
        const int nv = 2 * npad * TC_BK / 4;
        for (int i = tid; i < nv; i += TC_NT) dst[i] = __ldg(src + i);
      }
      fence_async_smem();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const uint32_t a_h = smem_u32(xh), a_l = smem_u32(xl);
        const uint32_t b_h = a_l + TC_M * TC_BK * 4, b_l = b_h + npad * TC_BK * 4;
#pragma unroll
        for (int j = 0; j < TC_BK / 8; ++j) {   // K = 8 per MMA (32 bytes)
          const uint32_t o = j * 32;
          umma_tf32(tmem, umma_desc_sw128(a_h + o), umma_desc_sw128(b_h + o), idesc,
                    (kc | j) ? 1u : 0u);
          umma_tf32(tmem, umma_desc_sw128(a_h + o), umma_desc_sw128(b_l + o), idesc, 1u);
          umma_tf32(tmem, umma_desc_sw128(a_l + o), umma_desc_sw128(b_h + o), idesc, 1u);
        }
        umma_commit(&S.bar[s]);
        if (kc == nkc - 1) umma_commit(&S.done);
      }
      issued[s] = 1;
    }
    // epilogue: row tid of the accumulator -> this thread
    mbar_wait(&S.done, done_phase);
    done_phase ^= 1;
    tc_fence_after();
    const double xn = row_ok ? xnorm[grow] : 0.0;
    uint64_t word = 0;
    int cur_word = -1;   // flattened (h * W + w) of `word`
    for (int c0 = 0; c0 < npad; c0 += 16) {
      uint32_t acc[16];
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, acc);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int c = c0 + j;
        bool unc = false;
        if (row_ok && c < cols) {
          const double sv = (double)__uint_as_float(acc[j]);
          if (dbg) dbg[grow * cols + c] = __uint_as_float(acc[j]);
          const double band = tau * xn * __ldg(rnorm + c) + 1e-30;
          const int h = c / L, t = c - h * L;
          const int wi = h * W + (t >> 6);
          if (wi != cur_word) {
            if (cur_word >= 0 && word)
              atomicOr((unsigned long long *)&codes[((int64_t)(cur_word / W) * n + grow) * W +
                                                    (cur_word % W)],
                       (unsigned long long)word);
            cur_word = wi;
            word = 0;
          }
          if (sv > band) word |= 1ull << (t & 63);
          unc = !(sv > band) && !(sv < -band);
        }
        const unsigned long long slot = warp_append(unc, fix.count);
        if (unc && slot < fix.cap) fix.items[slot] = ((unsigned long long)grow << 32) | (unsigned)c;
      }
    }
    if (cur_word >= 0 && word)
      atomicOr((unsigned long long *)&codes[((int64_t)(cur_word / W) * n + grow) * W +
                                            (cur_word % W)],
               (unsigned long long)word);
    tc_fence_before();
    __syncthreads();   // TMEM reads done before the next tile's MMAs overwrite it
  }
  // drain outstanding stage commits before freeing TMEM
  for (int s = 0; s < 2; ++s)
    if (issued[s]) mbar_wait(&S.bar[s], phase[s]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(ncols_alloc));
}


// ====================================================================
// Warp-specialised, TMA-fed version (the production path).
//   warp 0      : producer -- TMA 2D load of the X chunk (128 rows x 128 B,
//                 SWIZZLE_128B, OOB rows zero-filled) + one bulk copy of the
//                 pre-swizzled rh/rl chunk image, both completing on full[s]
//   warp 1      : TMEM allocation; lane 0 issues the 12 MMAs per chunk into
//                 one of two TMEM accumulators, commits empty[s] / accfull[b]
//   warps 4-7   : converters -- split the landed X chunk into xh (in place)
//                 and xl, fence.proxy.async, arrive conv[s]
//   warps 8-11  : epilogue -- tcgen05.ld their lane quarter of the finished
//                 accumulator, certified signs -> packed code words, fix-up
//                 list; arrive accempty[b]
// Stages are ring-buffered with mbarrier phase parity; the accumulator is
// double-buffered so the epilogue of tile t overlaps the MMAs of tile t+1.
constexpr int TC2_THREADS = 512;

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes,
                                          uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct Tc2Bars {
  uint64_t full[4], conv[4], empty[4], accfull[2], accempty[2], normfull[2], normempty[2];
  uint32_t tmem_base;
  double xss[2][2][TC_M];    // fused half-row sums of squares [buffer][half][row]
  // epilogue column tables: word index (h * W + t / 64), bit (t % 64),
  // tau * ||r_c|| (fp32, rounded up)
  alignas(16) float colband[TC_MAXN];
};

__host__ __device__ inline size_t tc2_stage_bytes(int npad) {
  return (size_t)(2 * TC_M + 2 * npad) * TC_BK * 4;   // x/xh, xl, rh, rl
}

__global__ void __launch_bounds__(TC2_THREADS, 1) k_project_tc2(
    const __grid_constant__ CUtensorMap xmap, int64_t n, int dim, const float *__restrict__ img,
    int cols, int npad, int nstages, const double *__restrict__ xnorm,
    const double *__restrict__ rnorm, double tau, int L, int W, uint64_t *__restrict__ codes,
    uint64_t *__restrict__ unc_bits, float *__restrict__ dbg,
    double *__restrict__ norms_out, unsigned long long *__restrict__ bad) {
  // norms_out != nullptr: the converters also produce the fp64 row norms
  // (sequential fma over ascending q, as k_row_stats) and the bad-row flags,
  // and hand the norms to the epilogue through shared memory (xnorm is not
  // read); the rows then cross HBM once for norms and projection together.
  const bool fuse = norms_out != nullptr;
  extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
  unsigned char *smem = tc_smem_raw + ((1024u - (smem_u32(tc_smem_raw) & 1023u)) & 1023u);
  const size_t sb = tc2_stage_bytes(npad);
  Tc2Bars &B = *reinterpret_cast<Tc2Bars *>(smem + nstages * sb);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nkc = (dim + TC_BK - 1) / TC_BK;
  const int64_t ntiles = (n + TC_M - 1) / TC_M;
  const uint32_t xbytes = TC_M * TC_BK * 4, rbytes = 2u * npad * TC_BK * 4;

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&B.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int c = tid; c < TC_MAXN; c += TC2_THREADS)
    B.colband[c] = c < cols ? (float)(tau * rnorm[c] * (1.0 + 1e-6)) : 0.f;
  if (tid == 0) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(&B.full[s], 1);
      mbar_init(&B.conv[s], 256);
      mbar_init(&B.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&B.accfull[b], 1);
      mbar_init(&B.accempty[b], 128);
      mbar_init(&B.normfull[b], 256);
      mbar_init(&B.normempty[b], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&xmap) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int s = it % nstages;
          const uint32_t use = it / nstages;
          mbar_wait(&B.empty[s], (use & 1) ^ 1);
          unsigned char *st = smem + s * sb;
          mbar_expect_tx(&B.full[s], xbytes + rbytes);
          tma_load_2d(st, &xmap, kc * TC_BK, (int)(tile * TC_M), &B.full[s]);
          bulk_load(st + 2 * xbytes, img + (int64_t)kc * 2 * npad * TC_BK, rbytes, &B.full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------------- MMA
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_tf32(npad);
      uint32_t it = 0, t = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++t) {
        const uint32_t b = t & 1, buse = t >> 1;
        mbar_wait(&B.accempty[b], (buse & 1) ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem + b * 256;
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int s = it % nstages;
          const uint32_t use = it / nstages;
          mbar_wait(&B.conv[s], use & 1);
          tc_fence_after();
          const uint32_t a_h = smem_u32(smem + s * sb), a_l = a_h + xbytes;
          const uint32_t b_h = a_l + xbytes, b_l = b_h + npad * TC_BK * 4;
#pragma unroll
          for (int j = 0; j < TC_BK / 8; ++j) {
            const uint32_t o = j * 32;
            umma_tf32(dcol, umma_desc_sw128(a_h + o), umma_desc_sw128(b_h + o), idesc,
                      (kc | j) ? 1u : 0u);
            umma_tf32(dcol, umma_desc_sw128(a_h + o), umma_desc_sw128(b_l + o), idesc, 1u);
            umma_tf32(dcol, umma_desc_sw128(a_l + o), umma_desc_sw128(b_h + o), idesc, 1u);
          }
          umma_commit(&B.empty[s]);
          if (kc == nkc - 1) umma_commit(&B.accfull[b]);
        }
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ---------------------------------------------------------- converters
    // two threads per row: warps 4-7 take 16-byte chunks 0-3 of the row's
    // 128-byte K chunk, warps 8-11 chunks 4-7
    const uint32_t row = (uint32_t)((warp & 3) * 32 + lane), half = (uint32_t)(warp - 4) >> 2;
    uint32_t it = 0, t = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++t) {
      // four interleaved partial sums per half (q mod 4; k_row_stats uses
      // the same order), so each fp64 fma chain is an eighth of the row
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      for (int kc = 0; kc < nkc; ++kc, ++it) {
        const int s = it % nstages;
        const uint32_t use = it / nstages;
        mbar_wait(&B.full[s], use & 1);
        float *xh = reinterpret_cast<float *>(smem + s * sb);
        float *xl = xh + TC_M * TC_BK;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const uint32_t off = sw128_off(row, half * 4 + (uint32_t)cc) / 4;
          const float4 v = *reinterpret_cast<const float4 *>(xh + off);
          if (fuse) {   // OOB columns are TMA zero-fill: fma(0, 0, s) == s
            s0 = fma((double)v.x, (double)v.x, s0);
            s1 = fma((double)v.y, (double)v.y, s1);
            s2 = fma((double)v.z, (double)v.z, s2);
            s3 = fma((double)v.w, (double)v.w, s3);
          }
          const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
          *reinterpret_cast<float4 *>(xh + off) = h;
          *reinterpret_cast<float4 *>(xl + off) =
              make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        }
        fence_async_smem();
        mbar_arrive(&B.conv[s]);
      }
      if (fuse) {
        const uint32_t b = t & 1, buse = t >> 1;
        mbar_wait(&B.normempty[b], (buse & 1) ^ 1);
        B.xss[b][half][row] = (s0 + s1) + (s2 + s3);
        mbar_arrive(&B.normfull[b]);
      }
    }
  } else if (warp >= 12) {
    // ------------------------------------------------------------ epilogue
    const int q = warp - 12;                      // == warp % 4: TMEM lane quarter
    uint32_t t = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++t) {
      const uint32_t b = t & 1, buse = t >> 1;
      mbar_wait(&B.accfull[b], buse & 1);
      tc_fence_after();
      const int64_t grow = tile * TC_M + q * 32 + lane;
      const bool row_ok = grow < n;
      float xn;
      if (fuse) {
        // the row's norm: the two halves' sums, then the flags (as k_row_stats)
        mbar_wait(&B.normfull[b], buse & 1);
        const double ss = B.xss[b][0][q * 32 + lane] + B.xss[b][1][q * 32 + lane];
        mbar_arrive(&B.normempty[b]);
        const double nrm = sqrt(ss);
        if (row_ok) {
          norms_out[grow] = nrm;
          if (!isfinite(ss)) atomicMin(&bad[0], (unsigned long long)grow);
          if (ss == 0.0) atomicMin(&bad[1], (unsigned long long)grow);
        }
        xn = row_ok ? (float)(nrm * (1.0 + 1e-6)) : 0.f;
      } else {
        xn = row_ok ? (float)(__ldg(xnorm + grow) * (1.0 + 1e-6)) : 0.f;
      }
      // Each row's words are produced entirely by this thread, in column
      // order.  Per 32-column group the certified signs and the band flags
      // become two 32-bit masks (one predicated OR per column); the masks
      // are then cut at replicate / word boundaries into the row's code
      // words (a word is stored, not OR-ed, when it completes).
      const int ncols = cols;
      uint64_t word = 0, uword = 0;
      int h = 0, t = 0;                 // (replicate, bit) of column c0
      for (int c0 = 0; c0 < ncols; c0 += 32) {
        uint32_t acc[32];
        tmem_ld32(tmem + b * 256 + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, acc);
        float bnd[32];
#pragma unroll
        for (int v = 0; v < 8; ++v)
          *reinterpret_cast<float4 *>(&bnd[4 * v]) =
              *reinterpret_cast<const float4 *>(&B.colband[c0 + 4 * v]);
        uint32_t pos = 0, unc = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float sv = __uint_as_float(acc[j]);
          const float band = bnd[j] * xn + 1e-30f;
          if (sv > band) pos |= 1u << j;
          else if (!(sv < -band)) unc |= 1u << j;
        }
        if (dbg && row_ok) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < cols) dbg[grow * cols + c0 + j] = __uint_as_float(acc[j]);
        }
        int j = 0;
        const int jend = min(32, ncols - c0);
        while (j < jend) {
          // segment: columns up to the end of the current word / replicate
          const int wend = min(L, ((t >> 6) + 1) << 6);
          const int len = min(jend - j, wend - t);
          const uint64_t m = len >= 32 ? 0xffffffffull : ((1ull << len) - 1ull);
          word |= ((uint64_t)(pos >> j) & m) << (t & 63);
          uword |= ((uint64_t)(unc >> j) & m) << (t & 63);
          t += len;
          j += len;
          if (t == wend) {
            if (row_ok) {
              const int64_t idx = ((int64_t)h * n + grow) * W + ((t - 1) >> 6);
              codes[idx] = word;
              unc_bits[idx] = uword;
            }
            word = 0;
            uword = 0;
            if (t == L) {
              t = 0;
              ++h;
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&B.accempty[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Band entries flagged in the bitmap (layout of the codes) -> entry list
// (row << 32 | column).  Each CTA pass takes 8 words per thread, scans the
// popcounts and reserves its output with ONE global atomic (a single shared
// counter under per-warp atomics serialises at L2).  Entries past `cap` are
// counted but not stored; k_fixup_bits then redoes the whole bitmap.
constexpr int COLLECT_NT = 256, COLLECT_WPT = 8;
__global__ void __launch_bounds__(COLLECT_NT) k_collect_bits(
    const uint64_t *__restrict__ unc_bits, int64_t n, int W, int L, int reps,
    unsigned long long *__restrict__ items, unsigned long long *__restrict__ count,
    unsigned long long cap) {
  __shared__ uint32_t sw[COLLECT_NT / 32];
  __shared__ unsigned long long sbase;
  const int64_t total = (int64_t)reps * n * W;
  constexpr int64_t PER = (int64_t)COLLECT_NT * COLLECT_WPT;
  for (int64_t b0 = (int64_t)blockIdx.x * PER; b0 < total; b0 += (int64_t)gridDim.x * PER) {
    uint64_t u[COLLECT_WPT];
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < COLLECT_WPT; ++j) {
      const int64_t i = b0 + (int64_t)j * COLLECT_NT + threadIdx.x;
      u[j] = i < total ? unc_bits[i] : 0ull;
      cnt += __popcll(u[j]);
    }
    uint32_t tot;
    uint32_t off = block_exclusive_scan<COLLECT_NT>(cnt, tot, sw);
    if (threadIdx.x == 0) sbase = tot ? atomicAdd(count, (unsigned long long)tot) : 0ull;
    __syncthreads();
    const unsigned long long base = sbase + off;
    uint32_t k = 0;
#pragma unroll
    for (int j = 0; j < COLLECT_WPT; ++j) {
      uint64_t x = u[j];
      if (!x) continue;
      const int64_t i = b0 + (int64_t)j * COLLECT_NT + threadIdx.x;
      const int64_t hw = i / W;
      const int h = (int)(hw / n), w = (int)(i - hw * W);
      const int64_t row = hw - (int64_t)h * n;
      while (x) {
        const int bit = __ffsll((long long)x) - 1;
        x &= x - 1;
        if (base + k < cap)
          items[base + k] = ((unsigned long long)row << 32) | (unsigned)(h * L + w * 64 + bit);
        ++k;
      }
    }
    __syncthreads();   // sbase / sw reused by the next pass
  }
}

// Band entries, one warp per entry (the production fix-up).  The lanes form
// the entry's separately rounded products x_q * r_q (__dmul_rn, as the
// reference), add them in a fixed tree and also add S = sum |x_q r_q|.  The
// reference's sequential sum differs from the exact dot product by at most
// (D + 1) u S (u = 2^-53: D product roundings and D additions, each bounded
// by u S), and so does the tree sum; when |tree| exceeds twice that bound
// (inflated by 1 %) the exact value, and with it the sequential sum, has the
// tree's sign.  Otherwise (|dot| within ~1e-13 relative of zero, exact
// zeros included) lane 0 redoes the reference's sequential sum in ascending
// q from the products staged in shared memory (lsh.py:107-112).
constexpr int FIXW_NT = 256;
__global__ void __launch_bounds__(FIXW_NT) k_fixup_warp(
    const float *__restrict__ x, int dim, const double *__restrict__ r, int64_t n, int L, int W,
    uint64_t *__restrict__ codes, const unsigned long long *__restrict__ items,
    const unsigned long long *__restrict__ count, unsigned long long cap, int force_seq) {
  extern __shared__ double fw_prod[];                 // [warps][dim] (fallback only)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double *prod = fw_prod + (size_t)wib * dim;
  const unsigned long long total = min(*count, cap);
  const unsigned long long nw = (unsigned long long)gridDim.x * (FIXW_NT / 32);
  // force_seq (tests): every entry takes the sequential path
  const double bound = force_seq ? INFINITY : 2.02 * (double)(dim + 1) * 0x1p-53;
  for (unsigned long long e = (unsigned long long)blockIdx.x * (FIXW_NT / 32) + wib; e < total;
       e += nw) {
    const unsigned long long it = items[e];
    const int64_t row = (int64_t)(it >> 32);
    const int c = (int)(it & 0xffffffffu);
    const float *xr = x + row * dim;
    const double *rr = r + (int64_t)c * dim;
    double sum = 0.0, sabs = 0.0;
    constexpr int U = 4;
    for (int q0 = lane; q0 < dim; q0 += 32 * U) {
      float xv[U];
      double rv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + 32 * u;
        xv[u] = q < dim ? __ldg(xr + q) : 0.f;
        rv[u] = q < dim ? __ldg(rr + q) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double p = __dmul_rn((double)xv[u], rv[u]);
        sum += p;
        sabs += fabs(p);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sum += __shfl_xor_sync(0xffffffffu, sum, o);
      sabs += __shfl_xor_sync(0xffffffffu, sabs, o);
    }
    bool pos;
    if (fabs(sum) > bound * sabs) {
      pos = sum > 0.0;
    } else {
      for (int q = lane; q < dim; q += 32) prod[q] = __dmul_rn((double)__ldg(xr + q), __ldg(rr + q));
      __syncwarp();
      double acc = 0.0;
      if (lane == 0)
        for (int q = 0; q < dim; ++q) acc = __dadd_rn(acc, prod[q]);
      pos = __shfl_sync(0xffffffffu, acc, 0) > 0.0;
      __syncwarp();
    }
    if (lane == 0 && pos) {
      const int h = c / L, t = c - h * L;
      atomicOr((unsigned long long *)&codes[((int64_t)h * n + row) * W + (t >> 6)],
               1ull << (t & 63));
    }
  }
}

// Exact recompute of the band entries flagged in the bitmap (same layout as
// the codes) -- the overflow path of k_collect_bits/k_fixup_warp (exits at
// once unless the list overflowed).  One warp per 32 rows: lanes compute the
// separately rounded products of one entry in parallel (coalesced row
// reads), lane 0 adds them in ascending q (lsh.py:107-112).
__global__ void __launch_bounds__(256) k_fixup_bits(const float *__restrict__ x, int64_t n,
                                                    int dim, const double *__restrict__ r, int L,
                                                    int W, int reps,
                                                    uint64_t *__restrict__ codes,
                                                    const uint64_t *__restrict__ unc_bits,
                                                    const unsigned long long *__restrict__ count,
                                                    unsigned long long cap) {
  if (*count <= cap) return;
  extern __shared__ double prod_all[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double *prod = prod_all + (int64_t)wib * dim;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t base = ((int64_t)blockIdx.x * (blockDim.x >> 5) + wib) * 32; base < n;
       base += nwarps * 32) {
    const int64_t row = base + lane;
    for (int h = 0; h < reps; ++h) {
      for (int w = 0; w < W; ++w) {
        uint64_t u = row < n ? unc_bits[((int64_t)h * n + row) * W + w] : 0ull;
        unsigned pend = __ballot_sync(0xffffffffu, u != 0);
        while (pend) {
          const int src = __ffs(pend) - 1;
          uint64_t uu = __shfl_sync(0xffffffffu, u, src);
          const int64_t rr = base + src;
          while (uu) {
            const int bit = __ffsll((long long)uu) - 1;
            uu &= uu - 1;
            const int t = w * 64 + bit;
            const int c = h * L + t;
            const float *xr = x + rr * dim;
            const double *rc = r + (int64_t)c * dim;
            for (int qq = lane; qq < dim; qq += 32) prod[qq] = __dmul_rn((double)xr[qq], rc[qq]);
            __syncwarp();
            if (lane == 0) {
              double acc = 0.0;
              int qq = 0;
              for (; qq + 8 <= dim; qq += 8) {     // loads issued ahead of the add chain
                double p8[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) p8[e] = prod[qq + e];
#pragma unroll
                for (int e = 0; e < 8; ++e) acc = __dadd_rn(acc, p8[e]);
              }
              for (; qq < dim; ++qq) acc = __dadd_rn(acc, prod[qq]);
              if (acc > 0.0) codes[((int64_t)h * n + rr) * W + w] |= 1ull << bit;
            }
            __syncwarp();
          }
          pend &= pend - 1;
        }
      }
    }
  }
}

// Error band of the 3xTF32 product relative to ||x|| ||r|| (see header):
// dropped xl.rl and the TF32 truncation of both residuals (<= 3 * 2^-20 per
// product) plus one fp32 rounding of the TMEM accumulator per MMA
// (3 * ceil(dim/8) MMAs, each <= 2^-22 of the running |sum| allowing
// round-toward-zero with a guard bit), doubled; plus the reference's own
// fp64 error.  Validated by tests/test_gpu_parity.py::
// test_tc_projection_error_band, which measures the worst observed error.
__host__ inline double tc_tau(int dim) {
  const double mmas = 3.0 * (double)((dim + 7) / 8);
  return 2.0 * (mmas * ldexp(1.0, -22) + 3.0 * ldexp(1.0, -20)) + (double)dim * ldexp(1.0, -52);
}

}  // namespace eg
