// format.cuh -- edge-list text output on the GPU.
//
// Reference: io.write_edges (io.py:145-158) writes one "i j dist" line per
// edge with f"{i} {j} {dist:.9f}\n" from a Python loop -- at 2e8-1.4e9 edges
// (configs 4 and 5) that loop, not the build, is the wall time.  Here every
// edge is formatted by one thread: line lengths -> exclusive scan -> each
// thread writes its line at its offset.  %.9f is reproduced exactly: the
// double x = mant * 2^e is scaled to x * 10^9 in 128-bit integer arithmetic
// and rounded half-to-even on the exact value (Python's correctly rounded
// float formatting), so the bytes equal the reference's.
#pragma once

#include "common.cuh"

namespace eg {

constexpr int FMT_MAX_LINE = 64;

__device__ __forceinline__ int dec_len(unsigned long long v) {
  int n = 1;
  while (v >= 10ull) {
    v /= 10ull;
    ++n;
  }
  return n;
}

// round_half_even(|x| * 10^9) for finite x with |x| * 10^9 < 2^63; returns
// false when out of range.
__device__ __forceinline__ bool scaled_1e9(double x, unsigned long long &N, bool &neg) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  neg = (bits >> 63) != 0;
  const int bexp = (int)((bits >> 52) & 0x7ff);
  unsigned long long mant = bits & ((1ull << 52) - 1);
  if (bexp == 0x7ff) return false;
  int e;
  if (bexp == 0) {
    e = -1074;                       // subnormal
  } else {
    mant |= 1ull << 52;
    e = bexp - 1075;
  }
  // P = mant * 10^9 as a 128-bit integer (hi, lo)
  const unsigned long long k = 1000000000ull;
  unsigned long long lo = mant * k, hi = __umul64hi(mant, k);
  if (e >= 0) {
    if (e >= 63 || hi != 0 || (lo >> (63 - e)) != 0) return false;
    N = lo << e;
    return true;
  }
  const int s = -e;
  if (s >= 128) {
    N = 0;                            // P < 2^83 < half an ulp of the result
    return true;
  }
  // q = P >> s, r = P mod 2^s, compare r with 2^(s-1)
  unsigned long long qlo, qhi;
  if (s >= 64) {
    qlo = hi >> (s - 64);
    qhi = 0;
  } else {
    qlo = (lo >> s) | (s ? (hi << (64 - s)) : 0ull);
    qhi = hi >> s;
  }
  if (qhi != 0 || (qlo >> 63) != 0) return false;
  // remainder bits and the half point
  int cmp;                            // r vs half: -1, 0, +1
  if (s >= 64) {
    const int t = s - 64;             // r = (hi mod 2^t, lo); half = 2^(s-1)
    const unsigned long long rhi = t ? (hi & ((1ull << t) - 1)) : 0ull;
    if (t == 0) {
      const unsigned long long half = 1ull << 63;
      cmp = lo > half ? 1 : (lo == half ? 0 : -1);
    } else {
      const unsigned long long hhalf = 1ull << (t - 1);
      cmp = rhi > hhalf ? 1 : (rhi < hhalf ? -1 : (lo > 0 ? 1 : 0));
    }
  } else {
    const unsigned long long r = lo & ((1ull << s) - 1);
    const unsigned long long half = 1ull << (s - 1);
    cmp = r > half ? 1 : (r == half ? 0 : -1);
  }
  if (cmp > 0 || (cmp == 0 && (qlo & 1ull))) ++qlo;
  N = qlo;
  return true;
}

__device__ __forceinline__ int edge_line_len(unsigned long long key, double dist, bool &ok) {
  unsigned long long N;
  bool neg;
  ok = scaled_1e9(dist, N, neg);
  if (!ok) return 0;
  const unsigned long long ip = N / 1000000000ull;
  return dec_len(key >> 32) + 1 + dec_len(key & 0xffffffffull) + 1 + (neg ? 1 : 0) +
         dec_len(ip) + 1 + 9 + 1;
}

__device__ __forceinline__ char *put_dec(char *p, unsigned long long v) {
  char tmp[20];
  int n = 0;
  do {
    tmp[n++] = (char)('0' + v % 10ull);
    v /= 10ull;
  } while (v);
  while (n) *p++ = tmp[--n];
  return p;
}

__global__ void k_edge_len(const uint64_t *__restrict__ keys, const double *__restrict__ dist,
                           int64_t m, uint32_t *__restrict__ len,
                           unsigned long long *__restrict__ bad) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    bool ok;
    const int l = edge_line_len(keys[p], dist[p], ok);
    if (!ok) atomicMin(bad, (unsigned long long)p);
    len[p] = (uint32_t)l;
  }
}

__global__ void k_edge_write(const uint64_t *__restrict__ keys, const double *__restrict__ dist,
                             int64_t m, const uint32_t *__restrict__ off,
                             char *__restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = keys[p];
    unsigned long long N;
    bool neg;
    if (!scaled_1e9(dist[p], N, neg)) continue;
    char line[FMT_MAX_LINE];
    char *q = put_dec(line, key >> 32);
    *q++ = ' ';
    q = put_dec(q, key & 0xffffffffull);
    *q++ = ' ';
    if (neg) *q++ = '-';
    q = put_dec(q, N / 1000000000ull);
    *q++ = '.';
    unsigned long long f = N % 1000000000ull;
    for (int d = 8; d >= 0; --d) {
      q[d] = (char)('0' + f % 10ull);
      f /= 10ull;
    }
    q += 9;
    *q++ = '\n';
    char *dst = out + off[p];
    for (char *s = line; s < q; ++s) *dst++ = *s;
  }
}

}  // namespace eg
