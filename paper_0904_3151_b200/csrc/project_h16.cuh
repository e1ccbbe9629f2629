// project_h16.cuh -- LSH projection on tcgen05 tensor cores in kind::f16
// (2-term fp16 splits, fp32 accumulator in TMEM): the production path for
// fp32 rows.  Same pipeline as k_project_tc2 (project_tc.cuh) -- TMA-fed,
// warp-specialised, double-buffered TMEM accumulator, certified sign band +
// exact fp64 fix-up -- at twice the tensor-pipe rate of kind::tf32 and about
// half the shared-memory traffic per K element.
//
// Reference: lsh.py:96-113 (_sign_bits), lsh.py:128-147 (_project_words),
// bitpool.py:125-141 (packing).
//
// Split.  x = xh + xl + ex with xh = fp16_rn(x), xl = fp16_rn(x - xh) (the
// difference is exact in fp32), so |ex| <= 2^-22 |x| + 2^-25 (the absolute
// term: fp16 subnormal spacing 2^-24).  Each direction column c is scaled by
// a power of two s_c (max |s_c r_c| in [2^13, 2^14): exact, and it cannot
// change the sign of column c) and split the same way.  The MMAs compute
// xh.rh + xh.rl + xl.rh; with the dropped xl.rl term
//   |D - s_c x.r_c| <= 3 * 2^-22 |x||s r| + 2^-24 sqrt(D) (|s r| + |x|)
// plus one fp32 accumulator rounding (<= 2^-22 of the running sum) per MMA.
// The band below doubles all of it.  Rows holding |x_q| >= 2^15 (fp16
// overflow) or a non-finite entry have every entry sent to the fix-up.
//
// Two rings (K chunk = 64 elements; fp16 operands are 128-byte rows in the
// SWIZZLE_128B K-major layout):
//   X ring, nx slots   : [X fp32 2 boxes of 128 x 128 B, SW128, TMA] -- released by the
//                        converters as soon as they have read it, so the
//                        row stream keeps nx chunks in flight;
//   operand ring, no   : [rh npad x 128 B][rl npad x 128 B] in shared memory
//                        plus the A operand xh | xl in TMEM (64 columns per
//                        slot: the converters tcgen05.st their rows' fp16
//                        pairs straight into the MMA's A tile, so A never
//                        touches shared memory) -- released by the MMA commit.
// TMEM: two accumulators of `acc` columns (npad rounded to 32), then the A
// slots.  Warp roles: 0 = X producer (TMA), 2 = direction producer (bulk
// copy), 1 = TMEM allocation + MMA issue (A from TMEM, B from shared
// memory), 4-11 = converters, 12-15 = epilogue.
#pragma once

#include <cuda_fp16.h>

#include "project_tc.cuh"

namespace eg {

constexpr int H16_THREADS = 512;

// Instruction descriptor: D f32, A/B f16, K-major both, N, M=128.
__host__ __device__ constexpr uint32_t umma_idesc_f16(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t da, uint64_t db,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

constexpr int H16_MAXSLOTS = 8;
constexpr int H16_BK = 64;                         // K elements per chunk
constexpr size_t H16_XSLOT = (size_t)2 * TC_M * 128;  // two 32-column fp32 boxes
__host__ __device__ inline size_t h16_oslot_bytes(int npad) { return (size_t)(2 * npad) * 128; }
__host__ __device__ inline int h16_acc_cols(int npad) { return (npad + 31) / 32 * 32; }
// the TMEM plan fits: two accumulators + 64 A columns per operand slot
__host__ inline bool h16_fits(int npad, int no) { return 2 * h16_acc_cols(npad) + 64 * no <= 512; }

// D[tmem] (+)= A[tmem] . B[smem]
__device__ __forceinline__ void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}

// ring position (slot, phase) advanced per chunk without divisions
struct RingPos {
  uint32_t s = 0, ph = 0;
  __device__ __forceinline__ void next(uint32_t n) {
    if (++s == n) {
      s = 0;
      ph ^= 1u;
    }
  }
};

// Per column: s_c (power of two), then the pre-swizzled fp16 images
// img[(kc * 2 + part) * npad * 32 + swizzled] (part 0 = rh, 1 = rl) of
// s_c r_c.  One CTA per (padded) column.
__global__ void __launch_bounds__(128) k_h16_prep_directions(const double *__restrict__ r,
                                                             int cols, int dim, int npad,
                                                             __half *__restrict__ img,
                                                             double *__restrict__ colscale) {
  __shared__ double red[4];
  const int c = blockIdx.x;
  const bool live = c < cols;
  double m = 0.0;
  if (live)
    for (int q = threadIdx.x; q < dim; q += blockDim.x) m = fmax(m, fabs(r[(int64_t)c * dim + q]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  m = fmax(fmax(red[0], red[1]), fmax(red[2], red[3]));
  // s = 2^(13 - floor(log2 m)): max |s r| in [2^13, 2^14)
  const double s = (m > 0.0 && isfinite(m)) ? ldexp(1.0, 13 - ilogb(m)) : 1.0;
  if (threadIdx.x == 0 && live) colscale[c] = s;
  const int nkc = (dim + H16_BK - 1) / H16_BK;
  for (int i = threadIdx.x; i < nkc * H16_BK; i += blockDim.x) {
    const int kc = i / H16_BK, kk = i - kc * H16_BK, q = kc * H16_BK + kk;
    const double v = (live && q < dim) ? r[(int64_t)c * dim + q] * s : 0.0;
    const __half hi = __double2half(v);
    const __half lo = __double2half(v - (double)__half2float(hi));
    const uint32_t off = sw128_off((uint32_t)c, (uint32_t)(kk >> 3)) / 2 + (kk & 7);
    __half *base = img + (int64_t)kc * 2 * npad * H16_BK;
    base[off] = hi;
    base[(int64_t)npad * H16_BK + off] = lo;
  }
}

struct H16Bars {
  uint64_t xfull[H16_MAXSLOTS], xempty[H16_MAXSLOTS];
  uint64_t rfull[H16_MAXSLOTS], conv[H16_MAXSLOTS], ofree[H16_MAXSLOTS];
  uint64_t accfull[2], accempty[2], normfull[2], normempty[2];
  uint32_t tmem_base;
  double xss[2][2][TC_M];      // fused half-row sums of squares [buffer][half][row]
  uint32_t ovf[2][2][TC_M];    // row needs the exact path (fp16 overflow / non-finite)
  alignas(16) float colA[TC_MAXN];   // band = colA * |x| + colB
  alignas(16) float colB[TC_MAXN];
  float colinv[TC_MAXN];             // 1 / s_c (debug dump only)
};

// Band coefficients of the fp16 split relative to |x| |s r| (see header).
__host__ inline double h16_tau(int dim) {
  const double mmas = 3.0 * (double)((dim + 15) / 16);
  return 2.0 * (mmas + 3.0) * ldexp(1.0, -22) + (double)dim * ldexp(1.0, -52);
}

__global__ void __launch_bounds__(H16_THREADS, 1) k_project_h16(
    const __grid_constant__ CUtensorMap xmap, int64_t n, int dim, const __half *__restrict__ img,
    const double *__restrict__ colscale, int cols, int npad, int nx, int no,
    const double *__restrict__ xnorm, const double *__restrict__ rnorm, double tau, int L, int W,
    uint64_t *__restrict__ codes, uint64_t *__restrict__ unc_bits, float *__restrict__ dbg,
    double *__restrict__ norms_out, unsigned long long *__restrict__ bad) {
  const bool fuse = norms_out != nullptr;
  extern __shared__ __align__(1024) unsigned char h16_smem_raw[];
  unsigned char *smem = h16_smem_raw + ((1024u - (smem_u32(h16_smem_raw) & 1023u)) & 1023u);
  const size_t ob = h16_oslot_bytes(npad);
  unsigned char *oring = smem + nx * H16_XSLOT;
  H16Bars &B = *reinterpret_cast<H16Bars *>(oring + no * ob);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nkc = (dim + H16_BK - 1) / H16_BK;
  const int64_t ntiles = (n + TC_M - 1) / TC_M;
  const uint32_t xbytes = (uint32_t)H16_XSLOT;
  const uint32_t rbytes = 2u * npad * H16_BK * 2;

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&B.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  {
    const double fl = sqrt((double)dim) * ldexp(1.0, -23);   // 2 * sqrt(D) * 2^-24
    for (int c = tid; c < TC_MAXN; c += H16_THREADS) {
      const double rs = c < cols ? rnorm[c] * colscale[c] : 0.0;
      B.colA[c] = c < cols ? (float)((tau * rs + fl) * (1.0 + 1e-6)) : 0.f;
      B.colB[c] = c < cols ? (float)(fl * rs * (1.0 + 1e-6)) : 0.f;
      B.colinv[c] = c < cols ? (float)(1.0 / colscale[c]) : 0.f;
    }
  }
  if (tid == 0) {
    for (int s = 0; s < nx; ++s) {
      mbar_init(&B.xfull[s], 1);
      mbar_init(&B.xempty[s], 256);
    }
    for (int s = 0; s < no; ++s) {
      mbar_init(&B.rfull[s], 1);
      mbar_init(&B.conv[s], 256);
      mbar_init(&B.ofree[s], 1);
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

  const uint32_t acc = (uint32_t)h16_acc_cols(npad);
  const uint32_t acol = tmem + 2 * acc;          // A slot s at acol + 64 s
  if (warp == 0) {
    // ---------------------------------------------------------- X producer
    if (lane == 0) {
      RingPos p;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int kc = 0; kc < nkc; ++kc, p.next(nx)) {
          mbar_wait(&B.xempty[p.s], p.ph ^ 1);
          mbar_expect_tx(&B.xfull[p.s], xbytes);
          unsigned char *dst = smem + p.s * H16_XSLOT;
          tma_load_2d(dst, &xmap, kc * H16_BK, (int)(tile * TC_M), &B.xfull[p.s]);
          tma_load_2d(dst + H16_XSLOT / 2, &xmap, kc * H16_BK + 32, (int)(tile * TC_M),
                      &B.xfull[p.s]);
        }
      }
    }
  } else if (warp == 2) {
    // -------------------------------------------------- direction producer
    if (lane == 0) {
      RingPos p;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int kc = 0; kc < nkc; ++kc, p.next(no)) {
          mbar_wait(&B.ofree[p.s], p.ph ^ 1);
          mbar_expect_tx(&B.rfull[p.s], rbytes);
          bulk_load(oring + p.s * ob, img + (int64_t)kc * 2 * npad * H16_BK, rbytes,
                    &B.rfull[p.s]);
        }
      }
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------------- MMA
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_f16(npad);
      RingPos p;
      uint32_t t = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++t) {
        const uint32_t b = t & 1, buse = t >> 1;
        mbar_wait(&B.accempty[b], (buse & 1) ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem + b * acc;
        for (int kc = 0; kc < nkc; ++kc, p.next(no)) {
          mbar_wait(&B.conv[p.s], p.ph);
          mbar_wait(&B.rfull[p.s], p.ph);
          tc_fence_after();
          const uint32_t a_h = acol + 64 * p.s, a_l = a_h + 32;
          const uint32_t b_h = smem_u32(oring + p.s * ob), b_l = b_h + npad * 128;
#pragma unroll
          for (int j = 0; j < H16_BK / 16; ++j) {
            const uint32_t o = j * 32;   // K=16 fp16 = 32 B along the 128 B row
            umma_f16_ts(dcol, a_h + 8 * j, umma_desc_sw128(b_h + o), idesc, (kc | j) ? 1u : 0u);
            umma_f16_ts(dcol, a_h + 8 * j, umma_desc_sw128(b_l + o), idesc, 1u);
            umma_f16_ts(dcol, a_l + 8 * j, umma_desc_sw128(b_h + o), idesc, 1u);
          }
          umma_commit(&B.ofree[p.s]);
          if (kc == nkc - 1) umma_commit(&B.accfull[b]);
        }
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ---------------------------------------------------------- converters
    // two threads per row: in each 32-column box, warps 4-7 take elements
    // 0-15 (K step 2 * box), warps 8-11 elements 16-31 (K step 2 * box + 1)
    const uint32_t row = (uint32_t)((warp & 3) * 32 + lane), half = (uint32_t)(warp - 4) >> 2;
    const uint32_t lanebase = (uint32_t)((warp & 3) * 32) << 16;
    RingPos px, po;
    uint32_t t = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++t) {
      // four interleaved partial sums per half (q mod 4) over the elements
      // with (q mod 32 >= 16) == half, ascending -- k_row_stats' order
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      bool ovf = false;
      for (int kc = 0; kc < nkc; ++kc, px.next(nx), po.next(no)) {
        mbar_wait(&B.xfull[px.s], px.ph);
        uint32_t hw[2][8], lw[2][8];
#pragma unroll
        for (int box = 0; box < 2; ++box) {
          const float *xs = reinterpret_cast<const float *>(smem + px.s * H16_XSLOT +
                                                            box * (H16_XSLOT / 2));
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const float4 v = *reinterpret_cast<const float4 *>(
                xs + sw128_off(row, half * 4 + (uint32_t)cc) / 4);
            if (fuse) {   // OOB columns are TMA zero-fill: fma(0, 0, s) == s
              s0 = fma((double)v.x, (double)v.x, s0);
              s1 = fma((double)v.y, (double)v.y, s1);
              s2 = fma((double)v.z, (double)v.z, s2);
              s3 = fma((double)v.w, (double)v.w, s3);
            }
            ovf |= !(fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))) <
                     32768.f) ||
                   v.x != v.x || v.y != v.y || v.z != v.z || v.w != v.w;
            const __half2 h01 = __floats2half2_rn(v.x, v.y), h23 = __floats2half2_rn(v.z, v.w);
            const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
            const __half2 l01 = __floats2half2_rn(v.x - f01.x, v.y - f01.y);
            const __half2 l23 = __floats2half2_rn(v.z - f23.x, v.w - f23.y);
            hw[box][2 * cc] = *reinterpret_cast<const uint32_t *>(&h01);
            hw[box][2 * cc + 1] = *reinterpret_cast<const uint32_t *>(&h23);
            lw[box][2 * cc] = *reinterpret_cast<const uint32_t *>(&l01);
            lw[box][2 * cc + 1] = *reinterpret_cast<const uint32_t *>(&l23);
          }
        }
        mbar_arrive(&B.xempty[px.s]);        // X slot read: the next TMA may land
        mbar_wait(&B.ofree[po.s], po.ph ^ 1);
        tc_fence_after();
        // K step k = 2 * box + half: 8 TMEM columns of fp16 pairs each
        const uint32_t a = acol + 64 * po.s + 8 * half + lanebase;
        tmem_st8(a, hw[0]);
        tmem_st8(a + 16, hw[1]);
        tmem_st8(a + 32, lw[0]);
        tmem_st8(a + 48, lw[1]);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&B.conv[po.s]);
      }
      const uint32_t b = t & 1, buse = t >> 1;
      mbar_wait(&B.normempty[b], (buse & 1) ^ 1);
      B.xss[b][half][row] = (s0 + s1) + (s2 + s3);
      B.ovf[b][half][row] = ovf ? 1u : 0u;
      mbar_arrive(&B.normfull[b]);
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
      mbar_wait(&B.normfull[b], buse & 1);
      const double ss = B.xss[b][0][q * 32 + lane] + B.xss[b][1][q * 32 + lane];
      const bool ovf = (B.ovf[b][0][q * 32 + lane] | B.ovf[b][1][q * 32 + lane]) != 0u;
      mbar_arrive(&B.normempty[b]);
      float xn;
      if (fuse) {
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
      // certified signs and band flags per 32-column group, cut at
      // replicate / word boundaries into the row's code words
      uint64_t word = 0, uword = 0;
      int h = 0, tb = 0;                // (replicate, bit) of column c0
      for (int c0 = 0; c0 < cols; c0 += 32) {
        uint32_t accv[32];
        tmem_ld32(tmem + b * acc + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, accv);
        float ca[32], cb[32];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          *reinterpret_cast<float4 *>(&ca[4 * v]) =
              *reinterpret_cast<const float4 *>(&B.colA[c0 + 4 * v]);
          *reinterpret_cast<float4 *>(&cb[4 * v]) =
              *reinterpret_cast<const float4 *>(&B.colB[c0 + 4 * v]);
        }
        uint32_t pos = 0, unc = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float sv = __uint_as_float(accv[j]);
          const float band = fmaf(ca[j], xn, cb[j]) + 1e-30f;
          if (sv > band) pos |= 1u << j;
          else if (!(sv < -band)) unc |= 1u << j;
        }
        if (ovf) {
          pos = 0u;
          unc = 0xffffffffu;
        }
        if (dbg && row_ok) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < cols)
              dbg[grow * cols + c0 + j] = __uint_as_float(accv[j]) * B.colinv[c0 + j];
        }
        int j = 0;
        const int jend = min(32, cols - c0);
        while (j < jend) {
          const int wend = min(L, ((tb >> 6) + 1) << 6);
          const int len = min(jend - j, wend - tb);
          const uint64_t m = len >= 32 ? 0xffffffffull : ((1ull << len) - 1ull);
          word |= ((uint64_t)(pos >> j) & m) << (tb & 63);
          uword |= ((uint64_t)(unc >> j) & m) << (tb & 63);
          tb += len;
          j += len;
          if (tb == wend) {
            if (row_ok) {
              const int64_t idx = ((int64_t)h * n + grow) * W + ((tb - 1) >> 6);
              codes[idx] = word;
              unc_bits[idx] = uword;
            }
            word = 0;
            uword = 0;
            if (tb == L) {
              tb = 0;
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

}  // namespace eg
