// scan_sort.cuh -- device-wide exclusive scan, stable LSD radix sort and
// stable compaction (hand-written, sm_100a).
//
// These replace the host-side np.lexsort calls of the reference
// (hamming_join.py:369-375, pipeline.py:222) and provide the prefix sums the
// count -> allocate -> write kernels need.
#pragma once

#include "common.cuh"

namespace eg {

// ------------------------------------------------------------------ scan
// Reduce-then-scan over uint32 (totals must fit in uint32).
constexpr int SCAN_NT = 256;
constexpr int SCAN_IPT = 16;
constexpr int SCAN_TILE = SCAN_NT * SCAN_IPT;

__global__ void __launch_bounds__(SCAN_NT) k_scan_reduce(const uint32_t *__restrict__ in,
                                                         int64_t L, uint32_t *__restrict__ sums) {
  __shared__ uint32_t sw[SCAN_NT / 32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    int64_t idx = base + (int64_t)i * SCAN_NT + threadIdx.x;
    if (idx < L) s += in[idx];
  }
  uint32_t tot;
  block_exclusive_scan<SCAN_NT>(s, tot, sw);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SCAN_NT) k_scan_tiles(const uint32_t *__restrict__ in,
                                                        int64_t L, uint32_t *__restrict__ out,
                                                        const uint32_t *__restrict__ tile_base) {
  __shared__ uint32_t sw[SCAN_NT / 32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  // blocked arrangement: thread t owns [t*IPT, t*IPT+IPT) of the tile
  uint32_t v[SCAN_IPT];
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    int64_t idx = base + (int64_t)threadIdx.x * SCAN_IPT + i;
    v[i] = idx < L ? in[idx] : 0;
    s += v[i];
  }
  uint32_t tot;
  uint32_t ex = block_exclusive_scan<SCAN_NT>(s, tot, sw);
  uint32_t run = ex + (tile_base ? tile_base[blockIdx.x] : 0);
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    int64_t idx = base + (int64_t)threadIdx.x * SCAN_IPT + i;
    if (idx < L) out[idx] = run;
    run += v[i];
  }
}

__host__ inline size_t scan_workspace(int64_t L) {
  size_t total = 0;
  while (L > SCAN_TILE) {
    int64_t nb = (L + SCAN_TILE - 1) / SCAN_TILE;
    total += ws_bytes(nb, 4) * 2;
    L = nb;
  }
  return total + 256;
}

// out[i] = sum_{j<i} in[j]; in/out may alias.  Recursive over tile sums.
__host__ inline int scan_exclusive_u32(const uint32_t *in, uint32_t *out, int64_t L, Arena &ar,
                                       cudaStream_t st) {
  if (L <= 0) return EG_OK;
  int64_t nb = (L + SCAN_TILE - 1) / SCAN_TILE;
  if (nb == 1) {
    EG_PROF(PC_SCAN, st);
    k_scan_tiles<<<1, SCAN_NT, 0, st>>>(in, L, out, nullptr);
    EG_LAUNCH_CHECK();
    return EG_OK;
  }
  uint32_t *sums = ar.take<uint32_t>(nb);
  uint32_t *sums_x = ar.take<uint32_t>(nb);
  if (!sums || !sums_x) return EG_ERR_WORKSPACE;
  {
    EG_PROF(PC_SCAN, st);
    k_scan_reduce<<<(unsigned)nb, SCAN_NT, 0, st>>>(in, L, sums);
  }
  EG_LAUNCH_CHECK();
  int rc = scan_exclusive_u32(sums, sums_x, nb, ar, st);
  if (rc) return rc;
  {
    EG_PROF(PC_SCAN, st);
    k_scan_tiles<<<(unsigned)nb, SCAN_NT, 0, st>>>(in, L, out, sums_x);
  }
  EG_LAUNCH_CHECK();
  return EG_OK;
}

// ------------------------------------------------------------ radix sort
// Stable LSD radix sort, 8-bit digits.  Per pass: upsweep (tile digit
// histograms, digit-major), exclusive scan, downsweep (warp-level
// match_any ranking, tile-local reorder in shared memory, coalesced-run
// scatter).  Keys uint64, optional uint32 values.
constexpr int RS_NT = 256;
constexpr int RS_IPT = 8;
constexpr int RS_TILE = RS_NT * RS_IPT;
constexpr int RS_WARPS = RS_NT / 32;

__global__ void __launch_bounds__(RS_NT) k_radix_upsweep(const uint64_t *__restrict__ keys,
                                                         int64_t m, int shift, int64_t ntiles,
                                                         uint32_t *__restrict__ counts) {
  __shared__ uint32_t hist[256];
  hist[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll
  for (int i = 0; i < RS_IPT; ++i) {
    int64_t idx = base + (int64_t)i * RS_NT + threadIdx.x;
    if (idx < m) atomicAdd(&hist[(keys[idx] >> shift) & 0xff], 1u);
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = hist[threadIdx.x];
}

template <bool VALS>
__global__ void __launch_bounds__(RS_NT) k_radix_downsweep(
    const uint64_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
    uint64_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out, int64_t m, int shift,
    int64_t ntiles, const uint32_t *__restrict__ offsets) {
  __shared__ uint64_t skeys[RS_TILE];
  __shared__ uint32_t svals[VALS ? RS_TILE : 1];
  __shared__ uint32_t wcnt[RS_WARPS][256];
  __shared__ uint32_t tstart[256];
  __shared__ uint32_t gbase[256];
  __shared__ uint32_t sw[RS_NT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_NT) (&wcnt[0][0])[i] = 0;
  gbase[threadIdx.x] = offsets[(int64_t)threadIdx.x * ntiles + blockIdx.x];
  __syncthreads();

  const int64_t base = (int64_t)blockIdx.x * RS_TILE + (int64_t)wid * 32 * RS_IPT;
  uint64_t k[RS_IPT];
  uint32_t v[RS_IPT];
  uint32_t rank[RS_IPT];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < RS_IPT; ++i) {
    int64_t idx = base + i * 32 + lane;
    bool ok = idx < m;
    k[i] = ok ? keys_in[idx] : 0;
    if (VALS) v[i] = ok ? vals_in[idx] : 0;
    uint32_t dg = ok ? (uint32_t)((k[i] >> shift) & 0xff) : 0x100u;
    unsigned peers = __match_any_sync(0xffffffffu, dg);
    uint32_t before = 0;
    if (ok) before = wcnt[wid][dg];
    rank[i] = before + __popc(peers & lt);
    __syncwarp();
    if (ok && (peers & lt) == 0) wcnt[wid][dg] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per-digit prefix over warps, then tile-local digit starts
  {
    const int dgt = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
      uint32_t c = wcnt[w][dgt];
      wcnt[w][dgt] = run;
      run += c;
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_scan<RS_NT>(run, tot, sw);
    tstart[dgt] = ex;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < RS_IPT; ++i) {
    int64_t idx = base + i * 32 + lane;
    if (idx < m) {
      uint32_t dg = (uint32_t)((k[i] >> shift) & 0xff);
      uint32_t pos = tstart[dg] + wcnt[wid][dg] + rank[i];
      skeys[pos] = k[i];
      if (VALS) svals[pos] = v[i];
    }
  }
  __syncthreads();
  int64_t tile0 = (int64_t)blockIdx.x * RS_TILE;
  int valid = (int)min((int64_t)RS_TILE, m - tile0);
  for (int j = threadIdx.x; j < valid; j += RS_NT) {
    uint64_t key = skeys[j];
    uint32_t dg = (uint32_t)((key >> shift) & 0xff);
    uint32_t dst = gbase[dg] + (j - tstart[dg]);
    keys_out[dst] = key;
    if (VALS) vals_out[dst] = svals[j];
  }
}

// ------------------------------------------------- onesweep radix sort
// One kernel per 8-bit digit pass (after one histogram pass over all
// digits): each CTA takes the next tile from an atomic ticket, ranks its
// keys as k_radix_downsweep does, publishes its per-digit counts and finds
// its global per-digit offsets by decoupled look-back over the tiles before
// it, then scatters the tile-locally sorted run.  Status words are 64-bit:
// flag (bits 62-63: 1 = tile aggregate, 2 = inclusive prefix) | count.
constexpr int OS_MAXPASS = 8;
#ifndef EG_OS_IPT
#define EG_OS_IPT 16
#endif
// keys per thread of a onesweep tile (key-value sorts use RS_IPT: the value
// stage must fit the 48 KB of static shared memory)
constexpr int OS_IPT = EG_OS_IPT;
constexpr unsigned long long OS_AGG = 1ull << 62, OS_INC = 2ull << 62,
                             OS_VAL = (1ull << 62) - 1;

__global__ void __launch_bounds__(RS_NT) k_radix_hist_all(const uint64_t *__restrict__ keys,
                                                          int64_t m, const int *__restrict__ sh,
                                                          int npass,
                                                          unsigned long long *__restrict__ hist) {
  __shared__ uint32_t h[OS_MAXPASS][256];
  for (int i = threadIdx.x; i < OS_MAXPASS * 256; i += RS_NT) (&h[0][0])[i] = 0;
  __syncthreads();
  int shl[OS_MAXPASS];
#pragma unroll
  for (int p = 0; p < OS_MAXPASS; ++p) shl[p] = p < npass ? sh[p] : 0;
  for (int64_t i = (int64_t)blockIdx.x * RS_NT + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * RS_NT) {
    const uint64_t k = keys[i];
#pragma unroll
    for (int p = 0; p < OS_MAXPASS; ++p)
      if (p < npass) atomicAdd(&h[p][(k >> shl[p]) & 0xff], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * 256; i += RS_NT)
    if ((&h[0][0])[i]) atomicAdd(&hist[i], (unsigned long long)(&h[0][0])[i]);
}

// hist[p][d] -> exclusive digit bases (in place), one CTA of 256 threads
__global__ void __launch_bounds__(256) k_radix_digit_bases(unsigned long long *__restrict__ hist,
                                                           int npass) {
  __shared__ unsigned long long sw[8];
  for (int p = 0; p < npass; ++p) {
    const unsigned long long v = hist[p * 256 + threadIdx.x];
    unsigned long long tot;
    const unsigned long long ex = block_exclusive_scan64<256>(v, tot, sw);
    hist[p * 256 + threadIdx.x] = ex;
    __syncthreads();
  }
}

#ifndef EG_OS_LB
#define EG_OS_LB 4     // 16 -> 4 and 3 CTAs/SM: 1.8x at 2e8-1.4e9 keys
#endif
#ifndef EG_OS_MINB
#define EG_OS_MINB 3
#endif
constexpr int OS_LB = EG_OS_LB;   // look-back window (predecessor tiles per round)
template <bool VALS, int IPT>
__global__ void __launch_bounds__(RS_NT, EG_OS_MINB) k_radix_onesweep(
    const uint64_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
    uint64_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out, int64_t m, int shift,
    const unsigned long long *__restrict__ digit_base, unsigned long long *status,
    unsigned int *ticket) {
  __shared__ uint64_t skeys[(RS_NT * IPT)];
  __shared__ uint32_t svals[VALS ? (RS_NT * IPT) : 1];
  __shared__ uint32_t wcnt[RS_WARPS][257];     // column 256: out-of-range items
  __shared__ uint32_t tstart[256];
  __shared__ unsigned long long gbase[256];
  __shared__ uint32_t sw[RS_NT / 32];
  __shared__ unsigned int stile;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) stile = atomicAdd(ticket, 1u);
  for (int i = threadIdx.x; i < RS_WARPS * 257; i += RS_NT) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t tile = stile;
  const int64_t base = tile * (RS_NT * IPT) + (int64_t)wid * 32 * IPT;
  uint64_t k[IPT];
  uint32_t v[IPT];
  uint32_t rank[IPT];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {           // all loads in flight before ranking
    const int64_t idx = base + i * 32 + lane;
    k[i] = idx < m ? keys_in[idx] : 0;
    if (VALS) v[i] = idx < m ? vals_in[idx] : 0;
  }
  // 1. the tile's digit counts first (order-free shared-memory atomics),
  //    published at once as this tile's aggregate: successors looking back
  //    find it long before this tile has ranked its keys
  volatile unsigned long long *st = status;
  {
    uint32_t *tcnt = tstart;   // reused: the tile-local starts come later
    tcnt[threadIdx.x] = 0;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; ++i)
      if (base + i * 32 + lane < m) atomicAdd(&tcnt[(uint32_t)((k[i] >> shift) & 0xff)], 1u);
    __syncthreads();
    const uint32_t c = tcnt[threadIdx.x];
    if (tile == 0) st[threadIdx.x] = OS_INC | c;
    else st[tile * 256 + threadIdx.x] = OS_AGG | c;
  }
  // 2. stable ranks: per warp and digit, a leader adds its peer count to the
  //    warp's counter and broadcasts the old value -- the atomics of
  //    successive items pipeline (same-address atomics of a warp execute in
  //    program order), with no shared-memory round trip per item
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const bool ok = base + i * 32 + lane < m;
    const uint32_t dg = ok ? (uint32_t)((k[i] >> shift) & 0xff) : 0x100u;
    // lanes with the same digit: 9 ballots (8 digit bits + validity) --
    // fully pipelined, where match.any's long latency stalled every item
    unsigned peers = __ballot_sync(0xffffffffu, ok);
    if (!ok) peers = ~peers;
#pragma unroll
    for (int bit = 0; bit < 8; ++bit) {
      const unsigned bb = __ballot_sync(0xffffffffu, (dg >> bit) & 1u);
      peers &= ((dg >> bit) & 1u) ? bb : ~bb;
    }
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (lane == leader) old = atomicAdd(&wcnt[wid][dg], (uint32_t)__popc(peers));
    rank[i] = __shfl_sync(0xffffffffu, old, leader) + __popc(peers & lt);
  }
  __syncthreads();
  {
    const int dgt = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
      const uint32_t c = wcnt[w][dgt];
      wcnt[w][dgt] = run;
      run += c;
    }
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan<RS_NT>(run, tot, sw);   // syncs: tcnt reads done
    tstart[dgt] = ex;
    if (tile == 0) {
      gbase[dgt] = digit_base[dgt];
    } else {
      // look back in windows of OS_LB predecessors: the window's loads are
      // independent (in flight together), then consumed newest first
      unsigned long long pre = 0;
      bool done = false;
      for (int64_t t = tile - 1; t >= 0 && !done; t -= OS_LB) {
        unsigned long long w[OS_LB];
#pragma unroll
        for (int q = 0; q < OS_LB; ++q) w[q] = t - q >= 0 ? st[(t - q) * 256 + dgt] : 0ull;
#pragma unroll
        for (int q = 0; q < OS_LB; ++q) {
          if (done || t - q < 0) continue;
          unsigned long long x = w[q];
          while ((x >> 62) == 0) x = st[(t - q) * 256 + dgt];
          pre += x & OS_VAL;
          if ((x >> 62) == 2) done = true;
        }
      }
      __threadfence();
      st[tile * 256 + dgt] = OS_INC | (pre + run);
      gbase[dgt] = digit_base[dgt] + pre;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int64_t idx = base + i * 32 + lane;
    if (idx < m) {
      const uint32_t dg = (uint32_t)((k[i] >> shift) & 0xff);
      const uint32_t pos = tstart[dg] + wcnt[wid][dg] + rank[i];
      skeys[pos] = k[i];
      if (VALS) svals[pos] = v[i];
    }
  }
  __syncthreads();
  const int64_t tile0 = tile * (RS_NT * IPT);
  const int valid = (int)min((int64_t)(RS_NT * IPT), m - tile0);
  for (int j = threadIdx.x; j < valid; j += RS_NT) {
    const uint64_t key = skeys[j];
    const uint32_t dg = (uint32_t)((key >> shift) & 0xff);
    const unsigned long long dst = gbase[dg] + (unsigned long long)(j - (int)tstart[dg]);
    keys_out[dst] = key;
    if (VALS) vals_out[dst] = svals[j];
  }
}

__host__ inline size_t radix_workspace(int64_t m, bool vals) {
  int64_t ntiles = (m + RS_TILE - 1) / RS_TILE;
  size_t b = ws_bytes(m, 8) + (vals ? ws_bytes(m, 4) : 0);
  b += ws_bytes(ntiles * 256, 4);
  b += scan_workspace(ntiles * 256);
  // onesweep: status words per (pass, tile, digit), tickets, histograms, shifts
  b += ws_bytes((size_t)OS_MAXPASS * ntiles * 256, 8) + ws_bytes(OS_MAXPASS * 256 + 64, 8);
  return b + 2048;
}

// Onesweep LSD sort (see above); same contract as radix_sort.
__host__ inline int radix_sort_onesweep(uint64_t *keys, uint32_t *vals, int64_t m,
                                        const int *shifts, int npass, Arena &ar,
                                        cudaStream_t st) {
  if (m <= 1 || npass == 0) return EG_OK;
  if (npass > OS_MAXPASS || m >= (1ll << 32)) return EG_ERR_UNSUPPORTED;
  const int64_t tilek = (int64_t)RS_NT * (vals ? RS_IPT : OS_IPT);
  const int64_t ntiles = (m + tilek - 1) / tilek;
  uint64_t *kalt = ar.take<uint64_t>(m);
  uint32_t *valt = vals ? ar.take<uint32_t>(m) : nullptr;
  unsigned long long *status = ar.take<unsigned long long>((size_t)npass * ntiles * 256);
  // [hist npass*256][tickets 16 (u32 pairs)][shifts 8 (int)]
  unsigned long long *meta = ar.take<unsigned long long>(OS_MAXPASS * 256 + 64);
  if (!kalt || (vals && !valt) || !status || !meta) return EG_ERR_WORKSPACE;
  unsigned long long *hist = meta;
  unsigned int *tickets = reinterpret_cast<unsigned int *>(meta + OS_MAXPASS * 256);
  int *dshift = reinterpret_cast<int *>(meta + OS_MAXPASS * 256 + 32);
  EG_CUDA_TRY(cudaMemsetAsync(status, 0, (size_t)npass * ntiles * 256 * 8, st));
  EG_CUDA_TRY(cudaMemsetAsync(meta, 0, (OS_MAXPASS * 256 + 32) * 8, st));
  EG_CUDA_TRY(cudaMemcpyAsync(dshift, shifts, npass * sizeof(int), cudaMemcpyHostToDevice, st));
  {
    EG_PROF(PC_SORT_UPSWEEP, st);
    const unsigned g = (unsigned)std::min<int64_t>((m + RS_NT * 16 - 1) / (RS_NT * 16),
                                                   (int64_t)1184);
    k_radix_hist_all<<<g, RS_NT, 0, st>>>(keys, m, dshift, npass, hist);
    k_radix_digit_bases<<<1, 256, 0, st>>>(hist, npass);
  }
  EG_LAUNCH_CHECK();
  uint64_t *ksrc = keys, *kdst = kalt;
  uint32_t *vsrc = vals, *vdst = valt;
  for (int p = 0; p < npass; ++p) {
    EG_PROF(PC_SORT_DOWNSWEEP, st);
    unsigned long long *stp = status + (size_t)p * ntiles * 256;
    if (vals)
      k_radix_onesweep<true, RS_IPT><<<(unsigned)ntiles, RS_NT, 0, st>>>(
          ksrc, vsrc, kdst, vdst, m, shifts[p], hist + p * 256, stp, tickets + p);
    else
      k_radix_onesweep<false, OS_IPT><<<(unsigned)ntiles, RS_NT, 0, st>>>(
          ksrc, nullptr, kdst, nullptr, m, shifts[p], hist + p * 256, stp, tickets + p);
    EG_LAUNCH_CHECK();
    uint64_t *t = ksrc; ksrc = kdst; kdst = t;
    uint32_t *tv = vsrc; vsrc = vdst; vdst = tv;
  }
  if (ksrc != keys) {
    EG_CUDA_TRY(cudaMemcpyAsync(keys, ksrc, m * 8, cudaMemcpyDeviceToDevice, st));
    if (vals) EG_CUDA_TRY(cudaMemcpyAsync(vals, vsrc, m * 4, cudaMemcpyDeviceToDevice, st));
  }
  return EG_OK;
}

// Sort keys (and vals) by the 8-bit digits at the given shifts, least
// significant first.  Result ends in keys/vals.
__host__ inline int radix_sort_classic(uint64_t *keys, uint32_t *vals, int64_t m,
                                       const int *shifts, int npass, Arena &ar, cudaStream_t st) {
  if (m <= 1 || npass == 0) return EG_OK;
  if (m >= (1ll << 32)) return EG_ERR_UNSUPPORTED;
  int64_t ntiles = (m + RS_TILE - 1) / RS_TILE;
  uint64_t *kalt = ar.take<uint64_t>(m);
  uint32_t *valt = vals ? ar.take<uint32_t>(m) : nullptr;
  uint32_t *counts = ar.take<uint32_t>(ntiles * 256);
  if (!kalt || (vals && !valt) || !counts) return EG_ERR_WORKSPACE;
  size_t mark = ar.used;
  uint64_t *ksrc = keys, *kdst = kalt;
  uint32_t *vsrc = vals, *vdst = valt;
  for (int p = 0; p < npass; ++p) {
    ar.used = mark;
    {
      EG_PROF(PC_SORT_UPSWEEP, st);
      k_radix_upsweep<<<(unsigned)ntiles, RS_NT, 0, st>>>(ksrc, m, shifts[p], ntiles, counts);
    }
    EG_LAUNCH_CHECK();
    int rc = scan_exclusive_u32(counts, counts, ntiles * 256, ar, st);
    if (rc) return rc;
    EG_PROF(PC_SORT_DOWNSWEEP, st);
    if (vals)
      k_radix_downsweep<true><<<(unsigned)ntiles, RS_NT, 0, st>>>(ksrc, vsrc, kdst, vdst, m,
                                                                 shifts[p], ntiles, counts);
    else
      k_radix_downsweep<false><<<(unsigned)ntiles, RS_NT, 0, st>>>(ksrc, nullptr, kdst, nullptr,
                                                                  m, shifts[p], ntiles, counts);
    EG_LAUNCH_CHECK();
    uint64_t *t = ksrc; ksrc = kdst; kdst = t;
    uint32_t *tv = vsrc; vsrc = vdst; vdst = tv;
  }
  if (ksrc != keys) {
    EG_CUDA_TRY(cudaMemcpyAsync(keys, ksrc, m * 8, cudaMemcpyDeviceToDevice, st));
    if (vals) EG_CUDA_TRY(cudaMemcpyAsync(vals, vsrc, m * 4, cudaMemcpyDeviceToDevice, st));
  }
  return EG_OK;
}

// Production sort: onesweep at every size (tile counts published before the
// ranking, ballot-based stable ranks: 2.5M keys 0.31 -> 0.26 ms, 1.4e9 keys
// 88 -> 77 ms against the three-kernel upsweep / scan / downsweep passes,
// which stay for the sort_path option and for m >= 2^32 tiles).
__host__ inline int radix_sort(uint64_t *keys, uint32_t *vals, int64_t m, const int *shifts,
                               int npass, Arena &ar, cudaStream_t st) {
  const int forced = options().sort_path;
  const bool classic = forced >= 0 ? forced == 1 : false;
  if (classic || npass > OS_MAXPASS) return radix_sort_classic(keys, vals, m, shifts, npass, ar, st);
  return radix_sort_onesweep(keys, vals, m, shifts, npass, ar, st);
}

// Digit shifts for pair keys (i << 32 | j) with i, j < n: only the low
// ceil(log2 n) bits of each half are non-zero.
__host__ inline int pair_key_shifts(int64_t n, int *shifts) {
  int b = ilog2_ceil((uint64_t)(n > 1 ? n : 2));
  int np = 0;
  for (int s = 0; s < b; s += 8) shifts[np++] = s;
  for (int s = 0; s < b; s += 8) shifts[np++] = 32 + s;
  return np;
}

// ------------------------------------------------------------ compaction
constexpr int CP_NT = 256;
constexpr int CP_IPT = 16;
constexpr int CP_TILE = CP_NT * CP_IPT;

__global__ void __launch_bounds__(CP_NT) k_flag_count(const uint8_t *__restrict__ flags, int64_t m,
                                                      uint32_t *__restrict__ tile_counts) {
  __shared__ uint32_t sw[CP_NT / 32];
  int64_t base = (int64_t)blockIdx.x * CP_TILE;
  uint32_t c = 0;
#pragma unroll
  for (int i = 0; i < CP_IPT; ++i) {
    int64_t idx = base + (int64_t)i * CP_NT + threadIdx.x;
    if (idx < m) c += flags[idx] ? 1 : 0;
  }
  uint32_t tot;
  block_exclusive_scan<CP_NT>(c, tot, sw);
  if (threadIdx.x == 0) tile_counts[blockIdx.x] = tot;
}

// Stable scatter: blocked arrangement inside each tile keeps input order.
// Stable scatter of the flagged elements, coalesced: iteration i of a tile
// covers elements [i * CP_NT, (i + 1) * CP_NT), a block scan per iteration
// places them in ascending index order; fully kept tiles (the common case
// of a verify that keeps almost every candidate) are copied straight and
// empty tiles exit.
template <typename V>
__global__ void __launch_bounds__(CP_NT) k_flag_scatter(const uint64_t *__restrict__ keys,
                                                        const V *__restrict__ vals,
                                                        const uint8_t *__restrict__ flags,
                                                        int64_t m,
                                                        const uint32_t *__restrict__ tile_off,
                                                        uint64_t *__restrict__ out_keys,
                                                        V *__restrict__ out_vals) {
  __shared__ uint32_t sw[CP_NT / 32];
  const int64_t base = (int64_t)blockIdx.x * CP_TILE;
  const uint32_t t0 = tile_off[blockIdx.x], tn = tile_off[blockIdx.x + 1] - t0;
  if (tn == 0) return;
  const int64_t valid = min((int64_t)CP_TILE, m - base);
  if ((int64_t)tn == valid) {
#pragma unroll 4
    for (int i = 0; i < CP_IPT; ++i) {
      const int64_t k = (int64_t)i * CP_NT + threadIdx.x;
      if (k < valid) {
        out_keys[t0 + k] = keys[base + k];
        if (vals) out_vals[t0 + k] = vals[base + k];
      }
    }
    return;
  }
  uint32_t run = t0;
  for (int i = 0; i < CP_IPT; ++i) {
    const int64_t idx = base + (int64_t)i * CP_NT + threadIdx.x;
    const uint32_t f = (idx < m && flags[idx]) ? 1u : 0u;
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan<CP_NT>(f, tot, sw);
    if (f) {
      out_keys[run + ex] = keys[idx];
      if (vals) out_vals[run + ex] = vals[idx];
    }
    run += tot;
    __syncthreads();                     // sw is reused by the next scan
  }
}

__host__ inline size_t compact_workspace(int64_t m) {
  int64_t nt = (m + CP_TILE - 1) / CP_TILE;
  return ws_bytes(nt + 1, 4) + scan_workspace(nt + 1) + 512;
}

// Returns the kept count via *h_count (synchronises `st`).
template <typename V>
__host__ inline int compact(const uint64_t *keys, const V *vals, const uint8_t *flags, int64_t m,
                            uint64_t *out_keys, V *out_vals, int64_t *h_count, Arena &ar,
                            cudaStream_t st) {
  if (m <= 0) {
    *h_count = 0;
    return EG_OK;
  }
  int64_t nt = (m + CP_TILE - 1) / CP_TILE;
  uint32_t *tc = ar.take<uint32_t>(nt + 1);
  if (!tc) return EG_ERR_WORKSPACE;
  EG_CUDA_TRY(cudaMemsetAsync(tc + nt, 0, 4, st));
  {
    EG_PROF(PC_COMPACT, st);
    k_flag_count<<<(unsigned)nt, CP_NT, 0, st>>>(flags, m, tc);
  }
  EG_LAUNCH_CHECK();
  int rc = scan_exclusive_u32(tc, tc, nt + 1, ar, st);
  if (rc) return rc;
  {
    EG_PROF(PC_COMPACT, st);
    k_flag_scatter<V><<<(unsigned)nt, CP_NT, 0, st>>>(keys, vals, flags, m, tc, out_keys,
                                                      out_vals);
  }
  EG_LAUNCH_CHECK();
  uint32_t total = 0;
  EG_CUDA_TRY(cudaMemcpyAsync(&total, tc + nt, 4, cudaMemcpyDeviceToHost, st));
  EG_CUDA_TRY(cudaStreamSynchronize(st));
  *h_count = total;
  return EG_OK;
}

// ------------------------------------------------------------ merge runs
// Two sorted key runs (+ 64-bit payloads) -> one, by merge path: every
// thread binary-searches its output diagonal, then merges MP_IT outputs
// sequentially (ties: a before b, so the merge is stable).  The multi-GPU
// build merges the ranks' sorted edge runs with log2(ranks) rounds of this
// instead of re-sorting them.
constexpr int MP_IT = 8, MP_NT = 256;
__global__ void __launch_bounds__(MP_NT) k_merge_path(const uint64_t *__restrict__ a,
                                                      const uint64_t *__restrict__ av, int64_t na,
                                                      const uint64_t *__restrict__ b,
                                                      const uint64_t *__restrict__ bv, int64_t nb,
                                                      uint64_t *__restrict__ out,
                                                      uint64_t *__restrict__ outv) {
  const int64_t total = na + nb;
  for (int64_t d0 = ((int64_t)blockIdx.x * MP_NT + threadIdx.x) * MP_IT; d0 < total;
       d0 += (int64_t)gridDim.x * MP_NT * MP_IT) {
    // i = number of a-elements among the first d0 outputs
    int64_t lo = d0 > nb ? d0 - nb : 0, hi = d0 < na ? d0 : na;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (a[mid] <= b[d0 - mid - 1]) lo = mid + 1; else hi = mid;
    }
    int64_t i = lo, j = d0 - lo;
    const int64_t end = d0 + MP_IT < total ? d0 + MP_IT : total;
    for (int64_t o = d0; o < end; ++o) {
      const bool take_a = j >= nb || (i < na && a[i] <= b[j]);
      if (take_a) {
        out[o] = a[i];
        if (outv) outv[o] = av[i];
        ++i;
      } else {
        out[o] = b[j];
        if (outv) outv[o] = bv[j];
        ++j;
      }
    }
  }
}

}  // namespace eg
