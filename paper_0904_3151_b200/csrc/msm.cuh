// msm.cuh -- the multiple sorting method on B200: per-(replicate, mask) unit
// masked sort, group detection and in-group pair enumeration.
//
// Reference (hamming_join.py): masked_key_table (bitpool.py:224-253) ->
// LSD counting passes (_counting_pass :52-82) -> _group_bounds (:85-101) ->
// _emit_group_pairs (:104-149), one mask at a time (:339), then the
// cross-replicate first-witness fold (pipeline.py:286-314).
//
// B200 design (per batch of up to MSM_MAXU units sharing one launch):
//  1. k_msm_hist    : masked key -> 64-bit hash; the top lgB bits are an MSD
//                     radix digit ("coarse bucket").  Shared-memory digit
//                     histograms, one global atomic per (CTA, digit).
//  2. k_msm_scan    : bucket offsets (exclusive scan), cursors reset.
//  3. k_msm_scatter : stable-enough MSD scatter of (h2 << 32 | row) into the
//                     buckets (only grouping matters, as in the reference,
//                     whose bucket order is first-seen, not lexicographic).
//  4. k_msm_group   : one CTA per bucket, entirely in shared memory: counting
//                     sort on the next hash digits, run detection (equal
//                     keys are exactly the runs), code gather for multi-row
//                     runs only, then a member-parallel pair loop (lane =
//                     grouped row, circulant partner order) with popcount
//                     <= d, the O(1) canonical-mask rule (or a covering
//                     design's first-member rule), staged emission.
//  5. k_msm_spill   : buckets larger than the shared-memory capacity (giant
//                     groups) are enumerated by 128x128 tile pairs.
// Equal masked keys always share a bucket and a run, so every reference
// group is visited; hash collisions are filtered by an exact key compare.
#pragma once

#include "common.cuh"

namespace eg {

#ifndef EG_MSM_MAXU
#define EG_MSM_MAXU 64   // 105 cfg3 units -> 2 batches: fewer per-batch tails (6.50 -> 6.29 ms)
#endif
constexpr int MSM_MAXU = EG_MSM_MAXU;   // units per launch batch
constexpr int MSM_IPT = 8;              // items per thread, hist/scatter
constexpr int MSM_NT = 1024;            // threads, hist/scatter
constexpr int MSM_TILE = MSM_IPT * MSM_NT;
constexpr int MSM_SC_NT = 512;          // threads, scatter (16 items each)
#ifndef EG_MSM_TARGET
#define EG_MSM_TARGET 3072
#endif
constexpr int MSM_TARGET = EG_MSM_TARGET;   // target mean bucket size (tuned on cfg3)
constexpr int MSM_SPILL_T = 128;        // spill tile edge
constexpr int MSM_MAX_LGB = 14;         // at most 16384 buckets per unit
constexpr int MSM_STAGE_MAX_B = 4096;   // scatter stages runs in smem up to this B
#ifndef EG_PAIR_SPLIT
#define EG_PAIR_SPLIT 262144u   // 65536: cfg3 stage 2.67 ms; 262144 and above: 2.58 ms
#endif
constexpr uint32_t MSM_PAIR_SPLIT = EG_PAIR_SPLIT;  // small-tier buckets with more pairs -> medium

constexpr int MSM_MAXT = 4;             // tail blocks of the O(1) canonical test
constexpr int MSM_MAXDESIGN = 64;       // members of a covering design (units per replicate)
#ifndef EG_TAIL_REGS
#define EG_TAIL_REGS 0   // 1: tail masks in registers (measured slower: register pressure)
#endif
#ifndef EG_SMALL_GDIV
#define EG_SMALL_GDIV 2  // small tier: at most CAP/4 groups per bucket (smem for 5 CTAs/SM)
#endif

struct UnitBatch {
  int count;
  int rep[MSM_MAXU];
  unsigned long long maskbits[MSM_MAXU];
  unsigned long long kept[MSM_MAXU][4];
  unsigned long long salt[MSM_MAXU];
  // Canonical-mask test without computing the mask (see canonical_tail_ok):
  // the unit's masked blocks above its lowest kept block, as bit ranges
  // [tail_lo, tail_hi); ntail > MSM_MAXT selects the general computation.
  uint8_t ntail[MSM_MAXU];
  uint16_t tail_lo[MSM_MAXU][MSM_MAXT];
  uint16_t tail_hi[MSM_MAXU][MSM_MAXT];
  // Covering-design units (ndesign > 0): the units of a replicate are the
  // ndesign members of an ordered family of masked block sets (each of >= d
  // blocks, every d-subset of blocks inside at least one member); a pair is
  // owned by the FIRST member whose kept bits it agrees on.  dq = the unit's
  // position in the family, dkept = the kept bits of every member.
  int ndesign;
  uint8_t dq[MSM_MAXU];
  unsigned long long dkept[MSM_MAXDESIGN][4];
};

struct MsmArgs {
  const uint64_t *codes;         // [reps][n][W]
  int64_t n;
  int L, W, k, d, lgB, reps;
  int B;                         // buckets per unit (any count <= 2^MSM_MAX_LGB)
  uint32_t *counts;              // [MAXU][B]
  uint32_t *starts;              // [MAXU][B+1]
  uint32_t *cursor;              // [MAXU][B]
  uint64_t *elems;               // [MAXU][n]
  uint32_t *gcnt;                // [MAXU][n] (spill group counts)
  const uint8_t *bit2blk;        // [EG_MAX_LENGTH]
  unsigned long long *out_keys;
  unsigned long long out_cap;
  unsigned long long *ctr;       // [0] emitted, [1] max group, [2] unused,
                                 // [3..3+reps) raw, [3+reps..) new
  unsigned long long *spill_ctr; // [0] entries on this scratch set's spill list,
                                 // [1] how many of them k_msm_scan listed (oversized buckets)
  int small_cap;                 // SmallCfg<W>::CAP: larger buckets are listed by k_msm_scan
  uint32_t *spill;               // [MAXU * (B+1)][3]: unit slot, start, size
  int64_t spill_cap;
  int gcnt_min;                  // spilled buckets above this size count groups
  int hist_smem;                  // dynamic shared memory of k_msm_hist (bytes)
  int scatter_staged;             // 1: k_msm_scatter reorders runs in smem
  uint16_t *out_rep;             // non-null: emit raw pairs tagged with their
                                 // replicate; the cross-replicate rule runs
                                 // later in k_xrep_filter (off the group
                                 // kernels' critical path)
};

template <int W>
__device__ __forceinline__ void load_code(const uint64_t *__restrict__ codes, int64_t row,
                                          uint64_t (&c)[W]) {
  if (W == 1) {
    c[0] = __ldg(codes + row);
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) c[w] = __ldg(codes + row * W + w);
  }
}

// MSD bucket of a key hash: multiply-high of the top 32 bits (any bucket
// count, not only powers of two; the low 32 bits stay the secondary key h2).
__device__ __forceinline__ uint32_t bucket_of(uint64_t h, int B) {
  return (uint32_t)(((h >> 32) * (uint64_t)(uint32_t)B) >> 32);
}

// ------------------------------------------------------------------ 1
// Bucket histogram for every unit of the batch: each CTA reads its code tile
// once (registers) and hashes it under each unit's mask, so the codes cross
// L2 once per batch instead of once per unit.  Shared-memory histograms
// (units_per_pass x B counters), one global atomic per non-empty (CTA, unit,
// bucket).
template <int W>
__global__ void __launch_bounds__(MSM_NT) k_msm_hist(const __grid_constant__ MsmArgs a,
                                                     const __grid_constant__ UnitBatch ub) {
  extern __shared__ uint32_t hist[];
  const int B = a.B;
  const int upp = max(1, min(ub.count, (int)(a.hist_smem / (B * 4))));
  const int64_t base = (int64_t)blockIdx.x * MSM_TILE;
  // all units of one batch share a replicate except at replicate boundaries
  for (int u0 = 0; u0 < ub.count; u0 += upp) {
    const int nu = min(upp, ub.count - u0);
    for (int i = threadIdx.x; i < nu * B; i += MSM_NT) hist[i] = 0;
    __syncthreads();
    int cur_rep = -1;
    uint64_t c[MSM_IPT][W];
    for (int uu = 0; uu < nu; ++uu) {
      const int u = u0 + uu;
      if (ub.rep[u] != cur_rep) {
        cur_rep = ub.rep[u];
        const uint64_t *codes = a.codes + (int64_t)cur_rep * a.n * W;
#pragma unroll
        for (int i = 0; i < MSM_IPT; ++i) {
          const int64_t row = base + (int64_t)i * MSM_NT + threadIdx.x;
          if (row < a.n) load_code<W>(codes, row, c[i]);
        }
      }
      const unsigned long long *kept = ub.kept[u];
      const uint64_t salt = ub.salt[u];
      uint32_t *hu = hist + uu * B;
#pragma unroll
      for (int i = 0; i < MSM_IPT; ++i) {
        const int64_t row = base + (int64_t)i * MSM_NT + threadIdx.x;
        if (row < a.n) {
          const uint64_t h = hash_key<W>(c[i], (const uint64_t *)kept, salt);
          atomicAdd(&hu[bucket_of(h, B)], 1u);
        }
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nu * B; i += MSM_NT) {
      const uint32_t v = hist[i];
      if (v) atomicAdd(&a.counts[(int64_t)(u0 + i / B) * B + (i % B)], v);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ 2
__global__ void __launch_bounds__(1024) k_msm_scan(const __grid_constant__ MsmArgs a) {
  __shared__ uint32_t sw[32];
  const int u = blockIdx.x;
  const int B = a.B;
  uint32_t *cnt = a.counts + (int64_t)u * B;
  uint32_t *st = a.starts + (int64_t)u * (B + 1);
  uint32_t *cur = a.cursor + (int64_t)u * B;
  const int per = (B + 1023) / 1024;
  uint32_t local = 0;
  for (int i = 0; i < per; ++i) {
    int b = threadIdx.x * per + i;
    if (b < B) local += cnt[b];
  }
  uint32_t tot;
  uint32_t run = block_exclusive_scan<1024>(local, tot, sw);
  for (int i = 0; i < per; ++i) {
    int b = threadIdx.x * per + i;
    if (b < B) {
      uint32_t c = cnt[b];
      st[b] = run;
      cur[b] = run;
      cnt[b] = 0;
      // buckets above the small tier's capacity are known here, before any
      // grouping: listed now, the medium tier takes them while the small
      // tier runs instead of after it (spill_ctr was zeroed before this kernel)
      if (c > (uint32_t)a.small_cap) {
        const unsigned long long slot = atomicAdd(&a.spill_ctr[0], 1ull);
        if ((int64_t)slot < a.spill_cap) {
          a.spill[slot * 3 + 0] = (uint32_t)u;
          a.spill[slot * 3 + 1] = run;
          a.spill[slot * 3 + 2] = c;
        }
      }
      run += c;
    }
  }
  if (threadIdx.x == 0) st[B] = tot;
}

// ------------------------------------------------------------------ 3
// MSD scatter of (h2 << 32 | row) into the unit's buckets.  Elements are
// first reordered by bucket in shared memory, so each (CTA, bucket) run is
// written by consecutive threads (coalesced) after one global atomic per
// non-empty bucket reserves its range.
template <int W>
__global__ void __launch_bounds__(MSM_SC_NT, 2) k_msm_scatter(const __grid_constant__ MsmArgs a,
                                                              const __grid_constant__ UnitBatch ub) {
  extern __shared__ __align__(16) unsigned char smsc[];
  const int u = blockIdx.y;
  const int B = a.B;
  const bool staged = a.scatter_staged;
  uint64_t *stage = reinterpret_cast<uint64_t *>(smsc);                    // [MSM_TILE]
  uint16_t *sbk = reinterpret_cast<uint16_t *>(stage + MSM_TILE);        // [MSM_TILE]
  uint32_t *hist = staged ? reinterpret_cast<uint32_t *>(sbk + MSM_TILE)
                          : reinterpret_cast<uint32_t *>(smsc);          // [B]
  uint32_t *tstart = hist + B;                                            // [B] (staged)
  uint32_t *gbase = staged ? tstart + B : hist + B;                       // [B]
  __shared__ uint32_t sw[MSM_SC_NT / 32];
  for (int i = threadIdx.x; i < B; i += MSM_SC_NT) hist[i] = 0;
  // the scan kernel before this one listed the oversized buckets; nothing
  // else is appended until the group kernel (which waits for this kernel)
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) a.spill_ctr[1] = a.spill_ctr[0];
  __syncthreads();
  const uint64_t *codes = a.codes + (int64_t)ub.rep[u] * a.n * W;
  const unsigned long long *kept = ub.kept[u];
  const uint64_t salt = ub.salt[u];
  const int64_t base = (int64_t)blockIdx.x * MSM_TILE;
  constexpr int IPT = MSM_TILE / MSM_SC_NT;
  // (bucket << 13) | rank: B <= 2^14, rank < MSM_TILE = 2^13
  static_assert(MSM_TILE <= (1 << 13) && MSM_MAX_LGB <= 19, "br packing");
  uint32_t br[IPT], h2[IPT];
  {
    // all code loads first (the smem atomics below would otherwise
    // serialise one load latency per item)
    uint64_t c[IPT][W];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int64_t row = base + (int64_t)i * MSM_SC_NT + threadIdx.x;
      if (row < a.n) load_code<W>(codes, row, c[i]);
    }
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int64_t row = base + (int64_t)i * MSM_SC_NT + threadIdx.x;
      if (row < a.n) {
        const uint64_t h = hash_key<W>(c[i], (const uint64_t *)kept, salt);
        const uint32_t b = bucket_of(h, B);
        h2[i] = (uint32_t)h;
        br[i] = (b << 13) | atomicAdd(&hist[b], 1u);
      }
    }
  }
  __syncthreads();
  uint32_t *cur = a.cursor + (int64_t)u * B;
  if (staged) {  // tile-local bucket starts (blocked scan) and global reservations
    const int per = (B + MSM_SC_NT - 1) / MSM_SC_NT;
    uint32_t loc = 0;
    for (int q = 0; q < per; ++q) {
      const int b = threadIdx.x * per + q;
      if (b < B) loc += hist[b];
    }
    uint32_t tot;
    uint32_t run = block_exclusive_scan<MSM_SC_NT>(loc, tot, sw);
    for (int q = 0; q < per; ++q) {
      const int b = threadIdx.x * per + q;
      if (b < B) {
        const uint32_t c = hist[b];
        tstart[b] = run;
        gbase[b] = c ? atomicAdd(&cur[b], c) : 0u;
        run += c;
      }
    }
  } else {
    for (int b = threadIdx.x; b < B; b += MSM_SC_NT) {
      const uint32_t c = hist[b];
      gbase[b] = c ? atomicAdd(&cur[b], c) : 0u;
    }
  }
  __syncthreads();
  uint64_t *el = a.elems + (int64_t)u * a.n;
  if (!staged) {
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int64_t row = base + (int64_t)i * MSM_SC_NT + threadIdx.x;
      if (row < a.n)
        el[gbase[br[i] >> 13] + (br[i] & 0x1fffu)] = ((uint64_t)h2[i] << 32) | (uint64_t)row;
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int64_t row = base + (int64_t)i * MSM_SC_NT + threadIdx.x;
    if (row < a.n) {
      const uint32_t pos = tstart[br[i] >> 13] + (br[i] & 0x1fffu);
      stage[pos] = ((uint64_t)h2[i] << 32) | (uint64_t)row;
      sbk[pos] = (uint16_t)(br[i] >> 13);
    }
  }
  __syncthreads();
  const int valid = (int)min((int64_t)MSM_TILE, a.n - base);
  for (int j = threadIdx.x; j < valid; j += MSM_SC_NT) {
    const uint32_t b = sbk[j];
    el[gbase[b] + (j - tstart[b])] = stage[j];
  }
}

// ------------------------------------------------------- pair predicate
// Canonical mask of a differing-bit pattern x (popcount(x) <= d): the blocks
// where the pair differs, filled up with the smallest untouched blocks --
// the lexicographically first d-subset containing them, i.e. the first mask
// (itertools.combinations order, hamming_join.py:333) under which the
// reference's _emit_group_pairs (hamming_join.py:130-141) emits the pair.
template <int W>
__device__ __forceinline__ uint64_t canonical_mask(const uint64_t (&x)[W], const uint8_t *b2b,
                                                   int k, int d) {
  uint64_t delta = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    uint64_t y = x[w];
    while (y) {
      int t = __ffsll((long long)y) - 1;
      delta |= 1ull << b2b[w * 64 + t];
      y &= y - 1;
    }
  }
  int need = d - __popcll(delta);
  uint64_t comp = ~delta & (k == 64 ? ~0ull : ((1ull << k) - 1));
  for (int i = 0; i < need; ++i) {
    uint64_t low = comp & (~comp + 1);
    delta |= low;
    comp ^= low;
  }
  return delta;
}

// Canonical-mask test for a pair whose differing bits x all lie in the
// unit's masked blocks M (x & kept == 0, so the differing-block set D is a
// subset of M).  canonical(D) = D + the lowest d-|D| blocks outside D equals
// M  iff  every block of M\D lies below the lowest kept block P  iff  every
// block of M above P differs, i.e. x has a bit in each tail range.  The tail
// ranges become W-word masks once per bucket (registers), so the test is
// |tail| AND-and-compare steps instead of a bit walk plus a fill loop.
template <int W>
struct TailTest {
  int nt;                          // tail blocks; > MSM_MAXT: general path
  int dq;                          // >= 0: covering-design unit at this position
  const unsigned long long *dk;    // [MSM_MAXDESIGN][4] kept bits of the design members
  uint64_t maskbits;
  const uint64_t *m;               // [MSM_MAXT][W] masks in shared memory
  // every thread calls load (same u); the masks are written by the first
  // MSM_MAXT * W threads -- the caller synchronises before the first ok()
  __device__ __forceinline__ void load(const UnitBatch &ub, int u, uint64_t *sm) {
    nt = ub.ntail[u];
    dq = ub.ndesign > 0 ? (int)ub.dq[u] : -1;
    dk = &ub.dkept[0][0];
    maskbits = ub.maskbits[u];
    m = sm;
    const int i = threadIdx.x;
    if (i < MSM_MAXT * W) {
      const int t = i / W, w = i - t * W;
      const int lo = t < nt ? ub.tail_lo[u][t] : 0, hi = t < nt ? ub.tail_hi[u][t] : 0;
      const int wl = max(lo - 64 * w, 0), wh = min(hi - 64 * w, 64);
      sm[i] = wl < wh ? (wh - wl == 64 ? ~0ull : ((1ull << (wh - wl)) - 1ull)) << wl : 0ull;
    }
  }
#if EG_TAIL_REGS
  uint64_t r[MSM_MAXT * W];        // register copy of the tail masks
  // after the barrier that follows load(): uniform registers for the pair loop
  __device__ __forceinline__ void fetch() {
#pragma unroll
    for (int i = 0; i < MSM_MAXT * W; ++i) r[i] = m[i];
  }
#else
  __device__ __forceinline__ void fetch() {}
#endif
  __device__ __forceinline__ bool ok(const uint64_t (&x)[W], int pc, const uint8_t *b2b, int k,
                                     int d) const {
    if (dq >= 0) {
      // design units: an earlier member that keeps none of the differing bits
      // groups the pair too, and owns it (uniform loop, uniform loads)
      for (int q = 0; q < dq; ++q) {
        uint64_t any = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) any |= x[w] & dk[q * 4 + w];
        if (!any) return false;
      }
      return true;
    }
    if (nt > MSM_MAXT) return canonical_mask<W>(x, b2b, k, d) == maskbits;
    if (nt > pc) return false;       // every tail block needs a differing bit
#if EG_TAIL_REGS
#pragma unroll
    for (int t = 0; t < MSM_MAXT; ++t) {
      if (t < nt) {
        uint64_t any = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) any |= x[w] & r[t * W + w];
        if (!any) return false;
      }
    }
#else
    for (int t = 0; t < nt; ++t) {
      uint64_t any = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) any |= x[w] & m[t * W + w];
      if (!any) return false;
    }
#endif
    return true;
  }
};

// Full predicate for one in-group pair.  Returns 0 = rejected, 1 = raw only
// (an earlier replicate owns it), 2 = emit.
template <int W>
__device__ __forceinline__ int pair_verdict(const uint64_t (&ca)[W], const uint64_t (&cb)[W],
                                            uint32_t ra, uint32_t rb, const MsmArgs &a,
                                            const TailTest<W> &tt,
                                            const unsigned long long *kept, int rep,
                                            const uint8_t *b2b) {
  uint64_t x[W];
  int pc = 0;
  uint64_t keydiff = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    x[w] = ca[w] ^ cb[w];
    pc += __popcll(x[w]);
    keydiff |= x[w] & kept[w];
  }
  if (keydiff || pc > a.d) return 0;
  if (!tt.ok(x, pc, b2b, a.k, a.d)) return 0;
  if (a.out_rep) return 2;
  for (int g = 0; g < rep; ++g) {
    const uint64_t *cg = a.codes + (int64_t)g * a.n * W;
    int pg = 0;
#pragma unroll
    for (int w = 0; w < W; ++w)
      pg += __popcll(__ldg(cg + (int64_t)ra * W + w) ^ __ldg(cg + (int64_t)rb * W + w));
    if (pg <= a.d) return 1;
  }
  return 2;
}

// ------------------------------------------------------------------ 4
// Bucket processing, entirely in shared memory.  An open-addressing table
// keyed by the 32-bit secondary hash groups the bucket's rows exactly by
// (h2), which is the masked key up to 2^-32 collisions (filtered later by an
// exact key compare).  Only rows of multi-row groups are materialised
// (rows + gathered codes, grouped contiguously); singletons -- the vast
// majority -- cost one table insert.  A member-parallel pair loop then
// visits every in-group pair once (the reference's group visits,
// hamming_join.py:116-122) and applies pair_verdict.
#ifndef EG_SMALL_MDIV
#define EG_SMALL_MDIV 1
#endif
#ifndef EG_GROUP_FILTER
#define EG_GROUP_FILTER 1
#endif
#ifndef EG_PAIR_UNROLL
#define EG_PAIR_UNROLL 2
#endif
#ifndef EG_RANK_ATOMIC32
#define EG_RANK_ATOMIC32 1
#endif
// Member capacity of a bucket tier: CAP / MDIV grouped rows, half as many
// groups.
template <int CAP, int MDIV>
struct MemberCap {
  static constexpr uint32_t M = CAP / MDIV,
                            G = CAP / MDIV / 2 / (MDIV == EG_SMALL_MDIV && CAP < 4096 ? EG_SMALL_GDIV : 1);
};

template <int W, int CAP, int NT, int MDIV = 1>
struct HGroupSmem {
  static constexpr uint32_t MCAP = MemberCap<CAP, MDIV>::M, GCAP = MemberCap<CAP, MDIV>::G;
  // The grouped rows and their codes overlay the hash table once every
  // thread has read its member position out of it (see process_bucket).
  static constexpr bool OVERLAY = (4 + 8 * W) * MCAP <= 16 * CAP;
  static constexpr size_t TAB_BYTES = 16 * (size_t)CAP;
  static constexpr size_t MEM_BYTES = (size_t)(4 + 8 * W) * MCAP;
  alignas(16) unsigned char big[OVERLAY ? TAB_BYTES : TAB_BYTES + MEM_BYTES];
  uint32_t mslot[GCAP];      // slots holding >= 2 rows (one entry per group)
  uint32_t runs[GCAP];       // (start << 16) | len, one per group
  uint16_t mgid[MCAP];       // group of every grouped row (index into runs)
  uint8_t b2b[EG_MAX_LENGTH];
  unsigned long long sw[NT / 32];
  uint32_t nruns, maxrun, raw, neu, ncand, nout, chunk;
  unsigned long long obase;
  uint64_t tmask[MSM_MAXT * W];    // tail masks of the bucket's unit (TailTest)
  // Emitted pairs are staged here during the pair loop (the table is dead
  // by then; with OVERLAY only the part past the member arrays is free) and
  // written out with one global reservation per bucket.
  static constexpr size_t OUT_OFF = OVERLAY ? MEM_BYTES : 0;
  static constexpr uint32_t OUTCAP = (uint32_t)((TAB_BYTES - OUT_OFF) / 8);
  __device__ unsigned long long *outbuf() {
    return reinterpret_cast<unsigned long long *>(big + OUT_OFF);
  }
  // (h2 << 32 | rows) per slot; later (member offset << 32 | rows)
  __device__ unsigned long long *tab() { return reinterpret_cast<unsigned long long *>(big); }
  __device__ uint64_t *codes() {
    return reinterpret_cast<uint64_t *>(big + (OVERLAY ? 0 : TAB_BYTES));
  }
  __device__ uint32_t *members() {
    return reinterpret_cast<uint32_t *>(big + (OVERLAY ? 0 : TAB_BYTES) + 8 * W * MCAP);
  }
};

constexpr unsigned long long HG_EMPTY = ~0ull;

// Optional per-bucket counters (compile with -DEG_MSM_STATS=1): buckets
// reaching the group stage, rows, filter candidates, groups, grouped rows,
// in-group pair visits, buckets re-queued for too many groups / too many
// grouped rows.  Read with eg_debug_msm_stats.
#ifndef EG_MSM_STATS
#define EG_MSM_STATS 0
#endif
__device__ unsigned long long g_msm_stats[8];

__device__ __forceinline__ uint32_t pow2_at_least(uint32_t v) {
  return v <= 1 ? 1u : 1u << (32 - __clz(v - 1));
}

// Returns false (without emitting anything) if the bucket's multi-row groups
// hold more rows than the member capacity (CAP/2) or more groups than CAP/4;
// the caller then re-queues it for the next tier.
// pair_limit: return false (re-queue) when the bucket's groups hold more
// pairs.  (Splitting one bucket's flattened pairs over several CTAs would
// need a canonical member order: group and member positions come from
// shared-memory atomics and differ from CTA to CTA.)
template <int W, int CAP, int NT, int MDIV>
__device__ __forceinline__ bool process_bucket(HGroupSmem<W, CAP, NT, MDIV> &S,
                                               const MsmArgs &a, const UnitBatch &ub, int u,
                                               const uint64_t *el, uint32_t s,
                                               uint32_t pair_limit = 0xffffffffu) {
  constexpr int PT = CAP / NT;
  constexpr uint32_t MCAP = HGroupSmem<W, CAP, NT, MDIV>::MCAP;
  constexpr uint32_t GCAP = HGroupSmem<W, CAP, NT, MDIV>::GCAP;
  constexpr uint32_t OUTCAP = HGroupSmem<W, CAP, NT, MDIV>::OUTCAP;
  const int rep = ub.rep[u];
  // 1. load the bucket (coalesced; from global or from the smem stage)
  uint64_t e[PT];
#pragma unroll
  for (int j = 0; j < PT; ++j) {
    const uint32_t i = threadIdx.x + j * NT;
    e[j] = i < s ? el[i] : 0ull;
  }
#if EG_GROUP_FILTER
  // 2. atomic-free singleton filter: every row writes its local index into
  //    a slot chosen by the high bits of h2 (plain stores, last writer
  //    wins); a row that reads back someone else's index, or finds its slot
  //    marked contested, may share its key and becomes a candidate.  Only
  //    candidates (true group members + ~s/FS false ones) enter the exact
  //    hash table below, so the expensive shared-memory atomics touch a
  //    small fraction of the bucket.
  constexpr uint32_t FS = 2 * CAP * 4;            // u16 slots overlaying tab
  constexpr int FSB = 31 - __builtin_clz(FS);
  uint16_t *F = reinterpret_cast<uint16_t *>(S.tab());
  for (uint32_t i = threadIdx.x * 8; i < FS; i += NT * 8)
    *reinterpret_cast<uint4 *>(&F[i]) = make_uint4(~0u, ~0u, ~0u, ~0u);
  if (threadIdx.x == 0) {
    S.nruns = 0; S.maxrun = 1; S.raw = 0; S.neu = 0; S.ncand = 0; S.nout = 0; S.chunk = 0;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < PT; ++j) {
    const uint32_t i = threadIdx.x + j * NT;
    if (i < s) F[(uint32_t)(e[j] >> 32) >> (32 - FSB)] = (uint16_t)i;
  }
  __syncthreads();
  uint32_t cand = 0;
#pragma unroll
  for (int j = 0; j < PT; ++j) {
    const uint32_t i = threadIdx.x + j * NT;
    if (i < s && F[(uint32_t)(e[j] >> 32) >> (32 - FSB)] != (uint16_t)i) cand |= 1u << j;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < PT; ++j)
    if (cand >> j & 1) F[(uint32_t)(e[j] >> 32) >> (32 - FSB)] = 0xfffe;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < PT; ++j) {
    const uint32_t i = threadIdx.x + j * NT;
    if (i < s && !(cand >> j & 1) && F[(uint32_t)(e[j] >> 32) >> (32 - FSB)] == 0xfffe)
      cand |= 1u << j;
  }
  // compact the candidates to the front of the CTA (dense registers): the
  //    sparse phases below then run ceil(ncand/NT) iterations, not PT
  uint32_t ncand;
  {
    uint32_t coff = block_exclusive_scan<NT>((uint32_t)__popc(cand), ncand,
                                             reinterpret_cast<uint32_t *>(S.sw));
    if (ncand == 0) {
      __syncthreads();
      return true;
    }
    uint64_t *clist = reinterpret_cast<uint64_t *>(S.big);   // F is dead now
#pragma unroll
    for (int j = 0; j < PT; ++j)
      if (cand >> j & 1) clist[coff++] = e[j];
    __syncthreads();
    cand = 0;
#pragma unroll
    for (int j = 0; j < PT; ++j) {
      const uint32_t i = threadIdx.x + j * NT;
      if (i < ncand) {
        e[j] = clist[i];
        cand |= 1u << j;
      }
    }
    __syncthreads();
  }
#else
  // no prefilter: every row enters the exact table (cheaper when most rows
  // sit in multi-row groups)
  uint32_t cand = 0;
#pragma unroll
  for (int j = 0; j < PT; ++j)
    if (threadIdx.x + j * NT < s) cand |= 1u << j;
  const uint32_t ncand = s;
  if (threadIdx.x == 0) {
    S.nruns = 0; S.maxrun = 1; S.raw = 0; S.neu = 0; S.ncand = 0; S.nout = 0; S.chunk = 0;
  }
  if (ncand == 0) {
    __syncthreads();
    return true;
  }
#endif
  const uint32_t T = pow2_at_least(2 * ncand);
  for (uint32_t i = threadIdx.x * 2; i < T; i += NT * 2)
    *reinterpret_cast<ulonglong2 *>(&S.tab()[i]) = make_ulonglong2(HG_EMPTY, HG_EMPTY);
  __syncthreads();
  // 3. insert candidates: one CAS claims an empty slot; a repeated h2 bumps
  //    the slot's count and the second row registers it as a group
  uint32_t slr[PT];   // (slot << 16) | rank within the group
#pragma unroll
  for (int j = 0; j < PT; ++j) {
    if (cand >> j & 1) {
      uint32_t h2 = (uint32_t)(e[j] >> 32);
      if (h2 == 0xffffffffu) h2 = 0xfffffffeu;
      const unsigned long long mine = ((unsigned long long)h2 << 32) | 1ull;
      uint32_t slot = h2 & (T - 1), rank = 0;
      while (true) {
        const unsigned long long old = atomicCAS(&S.tab()[slot], HG_EMPTY, mine);
        if (old == HG_EMPTY) break;
        if ((uint32_t)(old >> 32) == h2) {
          // 32-bit add on the count word (a 64-bit shared atomic add is a
          // CAS loop, which a large group's members serialise on)
#if EG_RANK_ATOMIC32
          rank = atomicAdd(reinterpret_cast<uint32_t *>(&S.tab()[slot]), 1u);
#else
          rank = (uint32_t)atomicAdd(&S.tab()[slot], 1ull);
#endif
          break;
        }
        slot = (slot + 1) & (T - 1);
      }
      slr[j] = (slot << 16) | rank;
      if (rank == 1) {
        const uint32_t r = atomicAdd(&S.nruns, 1u);
        if (r < GCAP) S.mslot[r] = slot;
      }
    }
  }
  __syncthreads();
  const uint32_t R = S.nruns;
  if (R == 0) {
    __syncthreads();
    return true;
  }
  if (R > GCAP) {
#if EG_MSM_STATS
    if (threadIdx.x == 0) atomicAdd(&g_msm_stats[6], 1ull);   // re-queued: too many groups
#endif
    __syncthreads();
    return false;
  }
  // 3. start the code gathers for rows of multi-row groups (latency overlaps
  //    the offset scan below)
  const uint64_t *codes = a.codes + (int64_t)rep * a.n * W;
  uint64_t cg[PT][W];
  uint32_t grouped = 0;   // bit j: element j sits in a multi-row group
#pragma unroll
  for (int j = 0; j < PT; ++j) {
    if ((cand >> j & 1) && (uint32_t)S.tab()[slr[j] >> 16] >= 2) {
      grouped |= 1u << j;
      const uint32_t row = (uint32_t)e[j];
#pragma unroll
      for (int w = 0; w < W; ++w) cg[j][w] = __ldg(codes + (int64_t)row * W + w);
    }
  }
  // 4. one scan over the groups gives member offsets and the pair prefix
  constexpr int RP = (GCAP + NT - 1) / NT;
  uint32_t c_my[RP];
  unsigned long long loc = 0;
#pragma unroll
  for (int q = 0; q < RP; ++q) {
    const uint32_t r = threadIdx.x * RP + q;
    c_my[q] = r < R ? (uint32_t)S.tab()[S.mslot[r]] : 0u;
    loc += ((unsigned long long)c_my[q] << 32) | (c_my[q] * (c_my[q] - 1) / 2);
  }
  unsigned long long tot;
  unsigned long long run = block_exclusive_scan64<NT>(loc, tot, S.sw);
  if ((uint32_t)(tot >> 32) > MCAP) {     // uniform: too many grouped rows
#if EG_MSM_STATS
    if (threadIdx.x == 0) atomicAdd(&g_msm_stats[7], 1ull);   // re-queued: too many grouped rows
#endif
    __syncthreads();
    return false;
  }
#pragma unroll
  for (int q = 0; q < RP; ++q) {
    const uint32_t r = threadIdx.x * RP + q;
    if (r < R) {
      const uint32_t off = (uint32_t)(run >> 32);
      S.tab()[S.mslot[r]] = ((unsigned long long)r << 48) | ((unsigned long long)off << 32) | c_my[q];
      S.runs[r] = (off << 16) | c_my[q];
      atomicMax(&S.maxrun, c_my[q]);
      run += ((unsigned long long)c_my[q] << 32) | (c_my[q] * (c_my[q] - 1) / 2);
    }
  }
#if EG_MSM_STATS
  if (threadIdx.x == 0) {
    atomicAdd(&g_msm_stats[0], 1ull);
    atomicAdd(&g_msm_stats[1], (unsigned long long)s);
    atomicAdd(&g_msm_stats[2], (unsigned long long)ncand);
    atomicAdd(&g_msm_stats[3], (unsigned long long)R);
    atomicAdd(&g_msm_stats[4], tot >> 32);
    atomicAdd(&g_msm_stats[5], tot & 0xffffffffull);
  }
#endif
  __syncthreads();
  // member positions out of the table first; then the (possibly overlaid)
  // member arrays are written
  // (group index << 16) | member position
#pragma unroll
  for (int j = 0; j < PT; ++j)
    if (grouped >> j & 1) {
      const uint32_t og = (uint32_t)(S.tab()[slr[j] >> 16] >> 32);
      slr[j] = (og & 0xffff0000u) | ((og & 0xffffu) + (slr[j] & 0xffffu));
    }
  // Overlay layout sized by the bucket's own member count M (uniform): M
  // codes, M rows, and everything behind them stages emitted pairs -- a
  // dense pool (config 5: ~1700 pairs per bucket) then rarely overflows
  // into per-pair reservations on the global output counter.
  constexpr bool OVL = HGroupSmem<W, CAP, NT, MDIV>::OVERLAY;
  const uint32_t Mrows = (uint32_t)(tot >> 32);
  uint64_t *mcodes = S.codes();
  uint32_t *mrows = OVL ? reinterpret_cast<uint32_t *>(S.big + (size_t)8 * W * Mrows) : S.members();
  const uint32_t out_off = ((uint32_t)(8 * W + 4) * Mrows + 7u) & ~7u;
  unsigned long long *const obuf =
      OVL ? reinterpret_cast<unsigned long long *>(S.big + out_off) : S.outbuf();
  const uint32_t ocap =
      OVL ? (uint32_t)((HGroupSmem<W, CAP, NT, MDIV>::TAB_BYTES - out_off) / 8) : OUTCAP;
  if (OVL) __syncthreads();
#pragma unroll
  for (int j = 0; j < PT; ++j) {
    if (grouped >> j & 1) {
      const uint32_t pos = slr[j] & 0xffffu;
      mrows[pos] = (uint32_t)e[j];
      S.mgid[pos] = (uint16_t)(slr[j] >> 16);
#pragma unroll
      for (int w = 0; w < W; ++w) mcodes[pos * W + w] = cg[j][w];
    }
  }
  __syncthreads();
  // 5. every in-group pair once.  Warps take chunks of 32 consecutive
  //    grouped rows (members of a group are contiguous); lane = one member
  //    with its code in registers.  Member i of a group of L visits
  //    (i + t) mod L for t = 1 .. L/2 (for even L the last step only from
  //    the lower half): every unordered pair exactly once, the same trip
  //    count for every member of a group (no divergence inside large
  //    groups, no per-pair bookkeeping), partners at consecutive addresses.
  const uint32_t P = (uint32_t)tot;
  if (P > pair_limit) {    // uniform: hand the bucket to the sliced medium tier
    __syncthreads();
    return false;
  }
  const uint32_t M = (uint32_t)(tot >> 32);
  const unsigned long long *kept = ub.kept[u];
  TailTest<W> tt;
  tt.load(ub, u, S.tmask);
  __syncthreads();
  tt.fetch();
  uint32_t my_raw = 0, my_new = 0;
  const uint32_t lane = threadIdx.x & 31;
  // loop invariants pinned in registers (ptxas otherwise re-reads them from
  // the constant bank and recomputes the shared window base every visit)
  uint64_t kp[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    kp[w] = kept[w];
    asm volatile("" : "+l"(kp[w]));
  }
  // Identical codes (popcount 0) are grouped by every unit and owned by the
  // one whose rule accepts the empty set of differing blocks -- the first
  // design member / the mask {0..d-1}.  Every other unit drops them in the
  // fast test below instead of walking the ownership rule for each: on
  // config 3 two thirds of the pairs that pass the Hamming test are such
  // duplicates, seen 14 times each.  (pc - lo) > dlim, unsigned: lo = 1
  // makes pc = 0 wrap around.
  const uint32_t lo0 = (tt.dq >= 0 ? tt.dq == 0 : tt.nt == 0) ? 0u : 1u;
  uint32_t dmax = (uint32_t)a.d - lo0, plo = lo0;
  uint32_t mc_s = (uint32_t)__cvta_generic_to_shared(mcodes);
  asm volatile("" : "+r"(dmax), "+r"(mc_s), "+r"(plo));
  constexpr uint32_t CB = 8 * W;   // bytes per code
  while (true) {
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(&S.chunk, 1u);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c * 32 >= M) break;
    const uint32_t pos = c * 32 + lane;
    uint32_t trips = 0, ra = 0, p = 0, p_first = 0, p_end = 0;
    uint64_t ca[W];
#pragma unroll
    for (int w = 0; w < W; ++w) ca[w] = 0;
    if (pos < M) {
      const uint32_t rr = S.runs[S.mgid[pos]];
      const uint32_t start = rr >> 16, len = rr & 0xffffu, idx = pos - start;
      ra = mrows[pos];
#pragma unroll
      for (int w = 0; w < W; ++w) ca[w] = mcodes[pos * W + w];
      // trips of this member: t*2 < len, plus t*2 == len from the lower half
      trips = (len >> 1) - ((len & 1u) == 0 && idx * 2 >= len ? 1u : 0u);
      p_first = mc_s + start * CB;
      p_end = p_first + len * CB;
      p = mc_s + pos * CB;
    }
    // one visit: partner code at shared address q; returns false when the
    // pair is rejected by the key / Hamming test (the common case)
    // (the exact key compare -- distinct keys sharing h2, 2^-32 per pair --
    // waits for the rare path: a colliding pair almost never passes the
    // popcount test)
    auto reject = [&](uint32_t q, uint64_t (&x)[W], uint32_t &pc) -> bool {
      pc = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        uint64_t cbw;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(cbw) : "r"(q + 8 * w));
        x[w] = ca[w] ^ cbw;
        pc += __popcll(x[w]);
      }
      return pc - plo > dmax;
    };
    // rare: within d on equal keys -- ownership, then the replicate rule
    auto accept = [&](uint32_t q, const uint64_t (&x)[W], uint32_t pc) {
      uint64_t keydiff = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) keydiff |= x[w] & kp[w];
      if (keydiff != 0 || !tt.ok(x, (int)pc, S.b2b, a.k, a.d)) return;
      const uint32_t rb = mrows[(q - mc_s) / CB];
      int v = 2;
      if (!a.out_rep) {
        for (int g = 0; g < rep && v == 2; ++g) {
          const uint64_t *cg2 = a.codes + (int64_t)g * a.n * W;
          int pg = 0;
#pragma unroll
          for (int w = 0; w < W; ++w)
            pg += __popcll(__ldg(cg2 + (int64_t)ra * W + w) ^ __ldg(cg2 + (int64_t)rb * W + w));
          if (pg <= a.d) v = 1;
        }
      }
      my_raw += 1;
      if (v == 2) {
        ++my_new;
        const unsigned long long key = ((unsigned long long)min(ra, rb) << 32) | max(ra, rb);
        const uint32_t so = atomicAdd(&S.nout, 1u);
        if (so < ocap) {
          obuf[so] = key;
        } else {
          const unsigned long long slot = atomicAdd(&a.ctr[0], 1ull);
          if (slot < a.out_cap) {
            a.out_keys[slot] = key;
            if (a.out_rep) a.out_rep[slot] = (uint16_t)rep;
          }
        }
      }
    };
    // EG_PAIR_UNROLL partners per step: independent load / xor / popcount
    // chains (the loop is latency-bound, not issue-bound)
    constexpr int PU = EG_PAIR_UNROLL;
    for (; trips >= (uint32_t)PU; trips -= PU) {
      uint32_t q[PU];
      uint64_t x[PU][W];
      uint32_t pc[PU];
      bool any = false;
      bool rj[PU];
#pragma unroll
      for (int i = 0; i < PU; ++i) {
        p += CB;
        if (p == p_end) p = p_first;
        q[i] = p;
      }
#pragma unroll
      for (int i = 0; i < PU; ++i) {
        rj[i] = reject(q[i], x[i], pc[i]);
        any |= !rj[i];
      }
      if (!any) continue;
#pragma unroll
      for (int i = 0; i < PU; ++i)
        if (!rj[i]) accept(q[i], x[i], pc[i]);
    }
    for (; trips; --trips) {
      p += CB;
      if (p == p_end) p = p_first;
      uint64_t x1[W];
      uint32_t pc1;
      if (!reject(p, x1, pc1)) accept(p, x1, pc1);
    }
  }
  if (my_raw) atomicAdd(&S.raw, my_raw);
  if (my_new) atomicAdd(&S.neu, my_new);
  __syncthreads();
  const uint32_t nst = min(S.nout, ocap);
  if (threadIdx.x == 0) {
    if (S.raw) atomicAdd(&a.ctr[3 + rep], (unsigned long long)S.raw);
    if (S.neu) atomicAdd(&a.ctr[3 + a.reps + rep], (unsigned long long)S.neu);
    atomicMax(&a.ctr[1], (unsigned long long)S.maxrun);
    if (nst) S.obase = atomicAdd(&a.ctr[0], (unsigned long long)nst);
  }
  __syncthreads();
  if (nst) {
    const unsigned long long base = S.obase;
    for (uint32_t i = threadIdx.x; i < nst; i += NT) {
      if (base + i < a.out_cap) {
        a.out_keys[base + i] = obuf[i];
        if (a.out_rep) a.out_rep[base + i] = (uint16_t)rep;
      }
    }
    __syncthreads();
  }
  return true;
}

// Rows of a spill-list entry: a contiguous bucket of elems[u].
__device__ __forceinline__ const uint64_t *spill_elems(const MsmArgs &a, int u, uint32_t s0) {
  return a.elems + (int64_t)u * a.n + s0;
}
__device__ __forceinline__ uint32_t *spill_gcnt(const MsmArgs &a, int u, uint32_t s0) {
  return a.gcnt + (int64_t)u * a.n + s0;
}

// Spill-list routing.  Tag bit 31: re-queued by the small tier (member room
// exhausted) -> medium tier.  Tag bit 30: re-queued by the medium tier ->
// tile kernel.  Untagged: routed by size.
constexpr uint32_t SPILL_FROM_SMALL = 0x80000000u, SPILL_FROM_MEDIUM = 0x40000000u;
__device__ __forceinline__ bool spill_for_tiles(uint32_t tag, uint32_t s, uint32_t med_cap) {
  return (tag & SPILL_FROM_MEDIUM) || (!(tag & SPILL_FROM_SMALL) && s > med_cap);
}

template <int W>
#ifndef EG_SMALL_CAP
#define EG_SMALL_CAP 2048
#endif
#ifndef EG_SMALL_NT
#define EG_SMALL_NT 256
#endif
#ifndef EG_SMALL_MINCTAS
#define EG_SMALL_MINCTAS 5   // cfg3 group kernel 2.75 -> 2.60 ms (4 -> 5 CTAs/SM)
#endif
struct SmallCfg {               // one CTA per bucket, several CTAs per SM
  static constexpr int CAP = W <= 2 ? EG_SMALL_CAP : EG_SMALL_CAP / 2;
  static constexpr int NT = EG_SMALL_NT;
  static constexpr int MIN_CTAS = EG_SMALL_MINCTAS;
  static constexpr int MDIV = EG_SMALL_MDIV;
};
#ifndef EG_MEDIUM_CAP
#define EG_MEDIUM_CAP 4096
#endif
template <int W>
struct MediumCfg {
  static constexpr int CAP = W <= 2 ? EG_MEDIUM_CAP : EG_MEDIUM_CAP / 2;
  static constexpr int NT = 512;
};

// Small buckets (s <= SmallCfg::CAP): grid (B, units).  Larger buckets are queued
// on the spill list for k_msm_medium / k_msm_spill.
template <int W>
__global__ void __launch_bounds__(SmallCfg<W>::NT, SmallCfg<W>::MIN_CTAS) k_msm_group(const __grid_constant__ MsmArgs a,
                                                       const __grid_constant__ UnitBatch ub) {
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr int CAP = SmallCfg<W>::CAP, NT = SmallCfg<W>::NT;
  using Smem = HGroupSmem<W, CAP, NT, SmallCfg<W>::MDIV>;
  Smem &S = *reinterpret_cast<Smem *>(smraw);
  const int u = blockIdx.y;
  const int b = blockIdx.x;
  const int B = a.B;
  const uint32_t *st = a.starts + (int64_t)u * (B + 1);
  const uint32_t s0 = st[b];
  const uint32_t s = st[b + 1] - s0;
  const uint64_t *src = a.elems + (int64_t)u * a.n + s0;
  if (s < 2) return;
  if (s > CAP) {   // listed by k_msm_scan for the medium / tile tiers
    if (s > (uint32_t)MediumCfg<W>::CAP && (int64_t)s * 4 > a.n) {
      uint32_t *g = spill_gcnt(a, u, s0);   // group counts for the warning
      for (uint32_t i = threadIdx.x; i < s; i += NT) g[i] = 0;
    }
    return;
  }
  for (int i = threadIdx.x; i < a.L; i += NT) S.b2b[i] = a.bit2blk[i];
  const bool ok = process_bucket(S, a, ub, u, src, s, MSM_PAIR_SPLIT);
  if (!ok) {
    // grouped rows exceed the member capacity, or the groups hold more than
    // MSM_PAIR_SPLIT pairs: hand the bucket to the medium tier (any size up
    // to its own capacity; 512 threads per bucket, off the small tier's
    // critical path)
    if (threadIdx.x == 0) {
      const unsigned long long slot = atomicAdd(&a.spill_ctr[0], 1ull);
      if ((int64_t)slot < a.spill_cap) {
        a.spill[slot * 3 + 0] = (uint32_t)u | SPILL_FROM_SMALL;
        a.spill[slot * 3 + 1] = s0;
        a.spill[slot * 3 + 2] = s;
      }
    }
  }
}

// Medium buckets (SmallCfg::CAP < s <= MediumCfg::CAP) from the spill list,
// persistent CTAs.
template <int W>
#ifndef EG_MEDIUM_MINCTAS
#define EG_MEDIUM_MINCTAS 2   // two 512-thread CTAs per SM where shared memory allows (W <= 2)
#endif
__global__ void __launch_bounds__(MediumCfg<W>::NT, EG_MEDIUM_MINCTAS) k_msm_medium(
    const __grid_constant__ MsmArgs a, const __grid_constant__ UnitBatch ub, const int phase) {
  extern __shared__ __align__(16) unsigned char smraw[];
  using Smem = HGroupSmem<W, MediumCfg<W>::CAP, MediumCfg<W>::NT, 1>;
  Smem &S = *reinterpret_cast<Smem *>(smraw);
  // phase 0 (beside the small tier): the oversized buckets k_msm_scan listed;
  // phase 1 (after it): the buckets the small tier re-queued
  const unsigned long long listed = min(a.spill_ctr[1], (unsigned long long)a.spill_cap);
  const unsigned long long first = phase == 0 ? 0ull : listed;
  const unsigned long long nspill =
      phase == 0 ? listed : min(a.spill_ctr[0], (unsigned long long)a.spill_cap);
  for (int i = threadIdx.x; i < a.L; i += MediumCfg<W>::NT) S.b2b[i] = a.bit2blk[i];
  for (unsigned long long sb = first + blockIdx.x; sb < nspill; sb += gridDim.x) {
    const uint32_t s = a.spill[sb * 3 + 2];
    const uint32_t tag = a.spill[sb * 3];
    const bool requeued = tag & SPILL_FROM_SMALL;     // small tier ran out of member room
    if ((tag & SPILL_FROM_MEDIUM) || (!requeued && s <= (uint32_t)SmallCfg<W>::CAP) ||
        s > (uint32_t)MediumCfg<W>::CAP)
      continue;
    const int u = (int)(tag & 0x3fffffffu);
    const uint32_t s0 = a.spill[sb * 3 + 1];
    if (!process_bucket(S, a, ub, u, spill_elems(a, u, s0), s)) {
      // still too many grouped rows: the tile kernel takes it
      if ((int64_t)s * 4 > a.n) {
        uint32_t *g = spill_gcnt(a, u, s0);
        for (uint32_t i = threadIdx.x; i < s; i += MediumCfg<W>::NT) g[i] = 0;
      }
      if (threadIdx.x == 0) {
        const unsigned long long slot = atomicAdd(&a.spill_ctr[0], 1ull);
        if ((int64_t)slot < a.spill_cap) {
          a.spill[slot * 3 + 0] = (uint32_t)u | SPILL_FROM_MEDIUM;
          a.spill[slot * 3 + 1] = s0;
          a.spill[slot * 3 + 2] = s;
        }
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------ 5
// Oversized buckets: all pairs by 128 x 128 tile pairs, grid-strided.  A
// bucket of size s costs O(s^2) hash compares -- the same order as the
// reference's in-group visits for the giant group that caused the spill.
template <int W>
__global__ void __launch_bounds__(MSM_SPILL_T) k_msm_spill(const __grid_constant__ MsmArgs a,
                                                                const __grid_constant__ UnitBatch ub) {
  __shared__ uint64_t ea[MSM_SPILL_T], eb[MSM_SPILL_T];
  __shared__ uint64_t cb_s[MSM_SPILL_T * W];
  __shared__ uint64_t tmask_s[MSM_MAXT * W];
  __shared__ uint8_t b2b[EG_MAX_LENGTH];
  __shared__ uint32_t sraw, sneu;
  __shared__ uint32_t sw_spill[MSM_SPILL_T / 32];
  __shared__ unsigned long long sbase;
  for (int i = threadIdx.x; i < a.L; i += MSM_SPILL_T) b2b[i] = a.bit2blk[i];
  const unsigned long long nspill = min(a.spill_ctr[0], (unsigned long long)a.spill_cap);
  for (unsigned long long sb = 0; sb < nspill; ++sb) {
    const uint32_t tag = a.spill[sb * 3 + 0];
    const int u = (int)(tag & 0x3fffffffu);
    const uint32_t s0 = a.spill[sb * 3 + 1], s = a.spill[sb * 3 + 2];
    if (!spill_for_tiles(tag, s, MediumCfg<W>::CAP)) continue;
    const uint32_t nt = (s + MSM_SPILL_T - 1) / MSM_SPILL_T;
    const unsigned long long ntp = (unsigned long long)nt * (nt + 1) / 2;
    const int rep = ub.rep[u];
    const unsigned long long *kept = ub.kept[u];
    TailTest<W> tt;
    __syncthreads();                  // previous entry done with tmask_s
    tt.load(ub, u, tmask_s);
    const uint64_t *el = spill_elems(a, u, s0);
    const uint64_t *codes = a.codes + (int64_t)rep * a.n * W;
    const bool count_groups = (int64_t)s * 4 > a.n;
    uint32_t *gc = spill_gcnt(a, u, s0);
    for (unsigned long long tp = blockIdx.x; tp < ntp; tp += gridDim.x) {
      // decode tile pair (ta <= tb), row-major over the upper triangle
      uint32_t ta = 0;
      {
        double dd = (double)(2 * nt + 1);
        double disc = dd * dd - 8.0 * (double)tp;
        ta = (uint32_t)floor((dd - sqrt(disc > 0 ? disc : 0)) * 0.5);
        auto T = [nt](unsigned long long x) { return x * nt - x * (x - 1) / 2; };
        while (ta > 0 && T(ta) > tp) --ta;
        while (ta + 1 < nt && T(ta + 1) <= tp) ++ta;
      }
      const uint32_t tb = ta + (uint32_t)(tp - ((unsigned long long)ta * nt -
                                                  (unsigned long long)ta * (ta - 1) / 2));
      __syncthreads();
      if (threadIdx.x == 0) { sraw = 0; sneu = 0; }
      const uint32_t ia0 = ta * MSM_SPILL_T, ib0 = tb * MSM_SPILL_T;
      {
        uint32_t i = threadIdx.x;
        ea[i] = ia0 + i < s ? el[ia0 + i] : ~0ull;
        eb[i] = ib0 + i < s ? el[ib0 + i] : ~0ull;
        if (ib0 + i < s) {
          const uint32_t row = (uint32_t)eb[i];
#pragma unroll
          for (int w = 0; w < W; ++w) cb_s[i * W + w] = __ldg(codes + (int64_t)row * W + w);
        }
      }
      __syncthreads();
      tt.fetch();
      const uint32_t i = threadIdx.x;
      uint32_t my_raw = 0, my_new = 0, my_eq = 0;
      uint32_t emask[MSM_SPILL_T / 32] = {};   // emitted partners j of this row
      uint32_t ra = 0;
      if (ia0 + i < s) {
        const uint64_t e = ea[i];
        const uint32_t h2 = (uint32_t)(e >> 32);
        ra = (uint32_t)e;
        uint64_t ca[W];
#pragma unroll
        for (int w = 0; w < W; ++w) ca[w] = __ldg(codes + (int64_t)ra * W + w);
        const uint32_t jlo = (ta == tb) ? i + 1 : 0;
        for (uint32_t j = jlo; j < MSM_SPILL_T; ++j) {
          const uint64_t f = eb[j];
          if (ib0 + j < s && (uint32_t)(f >> 32) == h2) {
            uint64_t cb[W];
            uint64_t kd = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) { cb[w] = cb_s[j * W + w]; kd |= (ca[w] ^ cb[w]) & kept[w]; }
            if (!kd) {
              ++my_eq;
              if (count_groups) atomicAdd(&gc[ib0 + j], 1u);
              const uint32_t rb = (uint32_t)f;
              int v = pair_verdict<W>(ca, cb, ra, rb, a, tt, kept, rep, b2b);
              my_raw += v > 0;
              my_new += v == 2;
              if (v == 2) emask[j >> 5] |= 1u << (j & 31);
            }
          }
        }
        if (count_groups && my_eq) atomicAdd(&gc[ia0 + i], my_eq);
      }
      // one global reservation per tile pair (a per-warp-step atomic on the
      // shared output counter serialised giant-group buckets), then every
      // thread writes its emitted pairs at its offset
      uint32_t tot;
      const uint32_t off = block_exclusive_scan<MSM_SPILL_T>(my_new, tot, sw_spill);
      if (threadIdx.x == 0) sbase = tot ? atomicAdd(&a.ctr[0], (unsigned long long)tot) : 0ull;
      __syncthreads();
      if (my_new) {
        unsigned long long slot = sbase + off;
#pragma unroll
        for (int q = 0; q < MSM_SPILL_T / 32; ++q) {
          uint32_t mbits = emask[q];
          while (mbits) {
            const int b = __ffs(mbits) - 1;
            mbits &= mbits - 1;
            const uint32_t rb = (uint32_t)eb[q * 32 + b];
            if (slot < a.out_cap) {
              a.out_keys[slot] = ((unsigned long long)min(ra, rb) << 32) | max(ra, rb);
              if (a.out_rep) a.out_rep[slot] = (uint16_t)rep;
            }
            ++slot;
          }
        }
      }
      if (my_raw) atomicAdd(&sraw, my_raw);
      if (my_new) atomicAdd(&sneu, my_new);
      __syncthreads();
      if (threadIdx.x == 0) {
        if (sraw) atomicAdd(&a.ctr[3 + rep], (unsigned long long)sraw);
        if (sneu) atomicAdd(&a.ctr[3 + a.reps + rep], (unsigned long long)sneu);
      }
    }
  }
}

// Largest group inside spilled buckets that could trip the reference's
// oversized warning (hamming_join.py:341-344): max(gcnt) + 1.
__global__ void k_msm_spill_maxgroup(const __grid_constant__ MsmArgs a) {
  const unsigned long long nspill = min(a.spill_ctr[0], (unsigned long long)a.spill_cap);
  for (unsigned long long sb = blockIdx.x; sb < nspill; sb += gridDim.x) {
    const uint32_t tag = a.spill[sb * 3 + 0];
    const int u = (int)(tag & 0x3fffffffu);
    const uint32_t s0 = a.spill[sb * 3 + 1], s = a.spill[sb * 3 + 2];
    if ((int64_t)s * 4 <= a.n || !spill_for_tiles(tag, s, (uint32_t)a.gcnt_min)) continue;
    const uint32_t *gc = spill_gcnt(a, u, s0);
    uint32_t mx = 0;
    for (uint32_t i = threadIdx.x; i < s; i += blockDim.x) mx = max(mx, gc[i]);
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&a.ctr[1], (unsigned long long)mx + 1);
  }
}

// ------------------------------------------- cross-replicate first witness
// Deferred form of the fold in pipeline.py:286-314: a raw pair of replicate
// h survives iff its Hamming distance exceeds d in every replicate g < h.
// Counts survivors per replicate (per_replicate_new).
constexpr int XREP_SMEM_REPS = 1024;   // replicates counted in shared memory
// keep == nullptr: a dropped pair's key is overwritten with ~0 instead (it
// then sorts behind every real key; the caller sorts the whole array and
// keeps the first sum(new_counts) keys -- no compaction pass).
__global__ void k_xrep_filter(uint64_t *__restrict__ keys, const uint16_t *__restrict__ reps,
                              int64_t m, const uint64_t *__restrict__ codes, int64_t n, int W,
                              int d, int nreps, uint8_t *__restrict__ keep,
                              unsigned long long *__restrict__ new_counts) {
  __shared__ unsigned int cnt[XREP_SMEM_REPS];
  for (int i = threadIdx.x; i < nreps && i < XREP_SMEM_REPS; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[p];
    const int64_t i = (int64_t)(key >> 32), j = (int64_t)(key & 0xffffffffu);
    const int h = reps[p];
    bool ok = true;
    for (int g = 0; g < h && ok; ++g) {
      const uint64_t *cg = codes + (int64_t)g * n * W;
      int pc = 0;
      for (int w = 0; w < W; ++w) pc += __popcll(__ldg(cg + i * W + w) ^ __ldg(cg + j * W + w));
      ok = pc > d;
    }
    if (keep) keep[p] = ok;
    else if (!ok) keys[p] = ~0ull;
    if (ok) {
      if (h < XREP_SMEM_REPS) atomicAdd(&cnt[h], 1u);
      else atomicAdd(&new_counts[h], 1ull);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nreps && i < XREP_SMEM_REPS; i += blockDim.x)
    if (cnt[i]) atomicAdd(&new_counts[i], (unsigned long long)cnt[i]);
}

// ------------------------------------------------------ full-code filter
// Pairs enumerated on a code prefix (strings longer than the kernels' 256
// bits, see engine.msm_candidates) are a superset of the answer; keep[p] =
// popcount of the FULL codes of the pair's replicate <= d, and raw[h]
// counts the survivors per replicate.
__global__ void k_hamming_filter(const uint64_t *__restrict__ keys, const uint16_t *__restrict__ reps,
                                 int64_t m, const uint64_t *__restrict__ codes, int64_t n, int W,
                                 int d, int nreps, uint8_t *__restrict__ keep,
                                 unsigned long long *__restrict__ raw) {
  __shared__ unsigned int cnt[XREP_SMEM_REPS];
  for (int i = threadIdx.x; i < nreps && i < XREP_SMEM_REPS; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[p];
    const int64_t i = (int64_t)(key >> 32), j = (int64_t)(key & 0xffffffffu);
    const int h = reps ? reps[p] : 0;
    const uint64_t *c = codes + (int64_t)h * n * W;
    int pc = 0;
    for (int w = 0; w < W && pc <= d; ++w) pc += __popcll(__ldg(c + i * W + w) ^ __ldg(c + j * W + w));
    const bool ok = pc <= d;
    keep[p] = ok;
    if (ok) {
      if (h < XREP_SMEM_REPS) atomicAdd(&cnt[h], 1u);
      else atomicAdd(&raw[h], 1ull);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nreps && i < XREP_SMEM_REPS; i += blockDim.x)
    if (cnt[i]) atomicAdd(&raw[i], (unsigned long long)cnt[i]);
}

// ------------------------------------------------------ first witness
__global__ void k_first_witness(const uint64_t *__restrict__ keys, int64_t m,
                                const uint64_t *const *__restrict__ pools, int npools, int W,
                                int d, uint8_t *__restrict__ keep) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[p];
    const int64_t i = (int64_t)(key >> 32), j = (int64_t)(key & 0xffffffffu);
    uint8_t ok = 1;
    for (int g = 0; g < npools && ok; ++g) {
      int pc = 0;
      for (int w = 0; w < W; ++w) pc += __popcll(pools[g][i * W + w] ^ pools[g][j * W + w]);
      if (pc <= d) ok = 0;
    }
    keep[p] = ok;
  }
}

// ------------------------------------------------------- grouped sort API
// grouped_radix_sort (hamming_join.py:275-297) reproduced pass for pass:
// the masked key is split into chunk_bits-wide chunks, MSB first
// (masked_key_table, bitpool.py:224-253), and the chunks are applied last to
// first, each as a stable counting pass whose buckets are laid out in
// FIRST-SEEN order (_counting_pass, hamming_join.py:52-82).  On the device a
// pass is: chunk value of every position + atomicMin of the position into a
// per-value table (= the bucket's first occurrence), then a stable LSD radix
// sort of the permutation by that first occurrence.
__global__ void k_iota(uint32_t *__restrict__ p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (uint32_t)i;
}

__device__ __forceinline__ uint32_t chunk_value(const uint64_t *__restrict__ codes, int64_t row,
                                                int W, const int32_t *__restrict__ cols, int c0,
                                                int cb, int ncols) {
  uint32_t v = 0;
  for (int q = 0; q < cb; ++q) {
    const int ci = c0 + q;
    uint32_t bit = 0;
    if (ci < ncols) {
      const int t = cols[ci];
      bit = (uint32_t)(codes[row * W + (t >> 6)] >> (t & 63)) & 1u;
    }
    v = (v << 1) | bit;        // zero padding at the low end of the last chunk
  }
  return v;
}

__global__ void k_chunk_first(const uint64_t *__restrict__ codes, const uint32_t *__restrict__ perm,
                              int64_t n, int W, const int32_t *__restrict__ cols, int c0, int cb,
                              int ncols, uint32_t *__restrict__ first, uint32_t *__restrict__ vbuf) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = chunk_value(codes, perm[p], W, cols, c0, cb, ncols);
    vbuf[p] = v;
    atomicMin(&first[v], (uint32_t)p);
  }
}

__global__ void k_chunk_rank(const uint32_t *__restrict__ vbuf, const uint32_t *__restrict__ first,
                             const uint32_t *__restrict__ perm, int64_t n,
                             uint64_t *__restrict__ key, uint32_t *__restrict__ val) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    key[p] = first[vbuf[p]];
    val[p] = perm[p];
  }
}

template <int WMAX>
__global__ void k_group_flags(const uint64_t *__restrict__ codes, const uint32_t *__restrict__ perm,
                              int64_t n, int W, const __grid_constant__ UnitBatch ub, uint8_t *__restrict__ flags,
                              uint64_t *__restrict__ idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool start = i == 0;
    if (!start) {
      const int64_t ra = perm[i - 1], rb = perm[i];
      for (int w = 0; w < W; ++w)
        start |= ((codes[ra * W + w] ^ codes[rb * W + w]) & ub.kept[0][w]) != 0;
    }
    flags[i] = start;
    idx[i] = (uint64_t)i;
  }
}

}  // namespace eg
