// xsum.cuh -- exact, order-independent global sums on the GPU (DESIGN.md CAC-2).
//
// Definition (CAC-2): for rounded fp64 summands p_r,
//   xsum(p) = RNE( sum_r Q(p_r) ),  Q(p) = p truncated toward zero to a multiple of 2^-200,
// with |p_r| < 2^100 (else a sticky range error).  The sum is carried exactly as a
// signed big integer in base 2^32 ("digits"), 10 int64 limbs per accumulator, so
// partial sums from any thread, block or GPU combine with plain integer adds
// (warp shuffles, shared memory, global atomics, NCCL int64 all-reduce) and the
// result is bitwise independent of the reduction tree and the GPU count.
//
// Why exact sums: Alg. 2 runs Lanczos without
// reorthogonalization, which amplifies any rounding difference (SURVEY.md
// Appendix A), so the dot products on the feedback path must not depend on the
// summation order.
#pragma once
#include <cstdint>

namespace scg {

constexpr int kLimbs = 10;       // 10 x 32-bit digits (int64 carry-save): LSB 2^-200
constexpr int kLsbExp = -200;

struct XAcc {
  long long d[kLimbs];
};

__device__ __forceinline__ void xacc_zero(XAcc &a) {
#pragma unroll
  for (int i = 0; i < kLimbs; ++i) a.d[i] = 0;
}

// Add the double p exactly (after Q).  err is set for |p| >= 2^100 or non-finite p.
__device__ __forceinline__ void xacc_add(XAcc &a, double p, int &err) {
  unsigned long long b = (unsigned long long)__double_as_longlong(p);
  if ((b << 1) == 0ull) return;  // +-0
  int e = (int)((b >> 52) & 0x7ffull);
  if (e >= 1123) { err = 1; return; }  // |p| >= 2^100, inf, nan
  unsigned long long m = b & 0x000fffffffffffffull;
  if (e) m |= 0x0010000000000000ull; else e = 1;
  // p = m 2^(e-1075); position of the mantissa LSB relative to 2^-200
  int s = e - 1075 - kLsbExp;
  if (s < 0) {
    int sh = -s;
    m = sh >= 64 ? 0ull : (m >> sh);  // Q: truncation toward zero
    s = 0;
    if (!m) return;
  }
  const int q = s >> 5, r = s & 31;  // q <= 7 because e <= 1122
  const unsigned int d0 = (unsigned int)(m << r);
  const unsigned int d1 = r ? (unsigned int)(m >> (32 - r)) : (unsigned int)(m >> 32);
  const unsigned int d2 = r ? (unsigned int)(m >> (64 - r)) : 0u;
  long long s0 = (long long)d0, s1 = (long long)d1, s2 = (long long)d2;
  if (b >> 63) { s0 = -s0; s1 = -s1; s2 = -s2; }
  switch (q) {  // static register indices (no local-memory array)
    case 0: a.d[0] += s0; a.d[1] += s1; a.d[2] += s2; break;
    case 1: a.d[1] += s0; a.d[2] += s1; a.d[3] += s2; break;
    case 2: a.d[2] += s0; a.d[3] += s1; a.d[4] += s2; break;
    case 3: a.d[3] += s0; a.d[4] += s1; a.d[5] += s2; break;
    case 4: a.d[4] += s0; a.d[5] += s1; a.d[6] += s2; break;
    case 5: a.d[5] += s0; a.d[6] += s1; a.d[7] += s2; break;
    case 6: a.d[6] += s0; a.d[7] += s1; a.d[8] += s2; break;
    default: a.d[7] += s0; a.d[8] += s1; a.d[9] += s2; break;
  }
}

// ---------------------------------------------------------------------------
// Register-light per-thread accumulator: a 4-digit window [qa, qa+3] of the full
// 10-digit number, anchored at the digit class of the thread's first summand.
// A summand whose 3 digits fall in the window is added in registers; any other
// summand is added exactly, digit by digit, to the block's shared-memory
// accumulator (rare slow path).  Exactness does not depend on the anchor.
struct XWin {
  long long w0, w1, w2, w3, w4;
  int qa;  // window digits [qa, qa+4]; -1: no summand yet
};

__device__ __forceinline__ void xwin_init(XWin &a) {
  a.w0 = a.w1 = a.w2 = a.w3 = a.w4 = 0;
  a.qa = -1;
}

// Split p (after Q) into its digit class q and three signed 32-bit digits.
// Returns false for +-0 or a summand truncated to 0; sets err on range error.
__device__ __forceinline__ bool xs_split(double p, int &q, long long &s0, long long &s1, long long &s2, int &err) {
  unsigned long long b = (unsigned long long)__double_as_longlong(p);
  if ((b << 1) == 0ull) return false;
  int e = (int)((b >> 52) & 0x7ffull);
  if (e >= 1123) { err = 1; return false; }
  unsigned long long m = b & 0x000fffffffffffffull;
  if (e) m |= 0x0010000000000000ull; else e = 1;
  int s = e - 1075 - kLsbExp;
  if (s < 0) {
    const int sh = -s;
    m = sh >= 64 ? 0ull : (m >> sh);
    s = 0;
    if (!m) return false;
  }
  q = s >> 5;
  const int r = s & 31;
  const unsigned lo = (unsigned)m, hi = (unsigned)(m >> 32);
  s0 = (long long)(lo << r);
  s1 = (long long)__funnelshift_l(lo, hi, r);
  s2 = (long long)__funnelshift_l(hi, 0u, r);
  if (b >> 63) { s0 = -s0; s1 = -s1; s2 = -s2; }
  return true;
}

// The window covers the digit classes qa, qa+1, qa+2, centred on the class of
// the thread's first summand (magnitudes straddling a class boundary stay fast).
// Normal summands (the fast path): the signed 54-bit mantissa M (two's complement) shifted by r
// is split as d0 + d1 2^32 + d2 2^64 with d0, d1 unsigned and d2 signed -- no per-digit negation.
__device__ __forceinline__ void xwin_add(XWin &a, double p, int &err, long long *blk) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(p);
  const int e = (int)((b >> 52) & 0x7ffull);
  if ((unsigned)(e - (1075 + kLsbExp)) < (unsigned)(1123 - (1075 + kLsbExp))) {  // no Q truncation, in range
    const unsigned long long m = (b & 0x000fffffffffffffull) | 0x0010000000000000ull;
    const long long ms = (long long)b < 0 ? -(long long)m : (long long)m;
    const int s = e - (1075 + kLsbExp);
    const int q = s >> 5, r = s & 31;
    const unsigned lo = (unsigned)ms, hi = (unsigned)((unsigned long long)ms >> 32);
    const long long d0 = (long long)(lo << r);
    const long long d1 = (long long)__funnelshift_l(lo, hi, r);
    const long long d2 = (long long)(int)__funnelshift_l(hi, (unsigned)((int)hi >> 31), r);
    if (a.qa < 0) a.qa = q < 1 ? 0 : (q > 6 ? 5 : q - 1);
    const int d = q - a.qa;
    if (d == 0) { a.w0 += d0; a.w1 += d1; a.w2 += d2; }
    else if (d == 1) { a.w1 += d0; a.w2 += d1; a.w3 += d2; }
    else if (d == 2) { a.w2 += d0; a.w3 += d1; a.w4 += d2; }
    else {
      atomicAdd(reinterpret_cast<unsigned long long *>(&blk[q]), (unsigned long long)d0);
      atomicAdd(reinterpret_cast<unsigned long long *>(&blk[q + 1]), (unsigned long long)d1);
      atomicAdd(reinterpret_cast<unsigned long long *>(&blk[q + 2]), (unsigned long long)d2);
    }
    return;
  }
  int q;
  long long s0, s1, s2;
  if (!xs_split(p, q, s0, s1, s2, err)) return;
  if (a.qa < 0) a.qa = q < 1 ? 0 : (q > 6 ? 5 : q - 1);
  const int d = q - a.qa;
  if (d == 0) { a.w0 += s0; a.w1 += s1; a.w2 += s2; }
  else if (d == 1) { a.w1 += s0; a.w2 += s1; a.w3 += s2; }
  else if (d == 2) { a.w2 += s0; a.w3 += s1; a.w4 += s2; }
  else {
    atomicAdd(reinterpret_cast<unsigned long long *>(&blk[q]), (unsigned long long)s0);
    atomicAdd(reinterpret_cast<unsigned long long *>(&blk[q + 1]), (unsigned long long)s1);
    atomicAdd(reinterpret_cast<unsigned long long *>(&blk[q + 2]), (unsigned long long)s2);
  }
}

// xwin_add for summands known to be >= 0 (squares): the same exact result without the
// sign handling (a product x*x is never negative; -0 contributes nothing either way).
__device__ __forceinline__ void xwin_add_nn(XWin &a, double p, int &err, long long *blk) {
  unsigned long long b = (unsigned long long)__double_as_longlong(p) & 0x7fffffffffffffffull;
  if (b == 0ull) return;
  int e = (int)(b >> 52);
  if (e >= 1123) { err = 1; return; }
  unsigned long long m = b & 0x000fffffffffffffull;
  if (e) m |= 0x0010000000000000ull; else e = 1;
  int s = e - 1075 - kLsbExp;
  if (s < 0) {
    const int sh = -s;
    m = sh >= 64 ? 0ull : (m >> sh);
    s = 0;
    if (!m) return;
  }
  const int q = s >> 5, r = s & 31;
  const unsigned lo = (unsigned)m, hi = (unsigned)(m >> 32);
  const long long s0 = (long long)(lo << r);
  const long long s1 = (long long)__funnelshift_l(lo, hi, r);
  const long long s2 = (long long)__funnelshift_l(hi, 0u, r);
  if (a.qa < 0) a.qa = q < 1 ? 0 : (q > 6 ? 5 : q - 1);
  const int d = q - a.qa;
  if (d == 0) { a.w0 += s0; a.w1 += s1; a.w2 += s2; }
  else if (d == 1) { a.w1 += s0; a.w2 += s1; a.w3 += s2; }
  else if (d == 2) { a.w2 += s0; a.w3 += s1; a.w4 += s2; }
  else {
    atomicAdd(reinterpret_cast<unsigned long long *>(&blk[q]), (unsigned long long)s0);
    atomicAdd(reinterpret_cast<unsigned long long *>(&blk[q + 1]), (unsigned long long)s1);
    atomicAdd(reinterpret_cast<unsigned long long *>(&blk[q + 2]), (unsigned long long)s2);
  }
}

// Flush a thread's window into the block accumulator (all 32 lanes of the warp call this).
// The lanes' windows are placed at their absolute digit positions inside the warp's common span
// [qlo, qhi + 4] (a register re-indexing, no arithmetic), then each digit of the span is summed with
// one shuffle tree and lane 0 adds it to the block accumulator: one reduction round whatever the
// mix of anchors (lanes whose first summands differ in magnitude).
__device__ __forceinline__ void xwin_flush(const XWin &a, long long *blk) {
  const bool has = a.qa >= 0;
  int qlo = has ? a.qa : 1 << 20, qhi = has ? a.qa : -1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    qlo = min(qlo, __shfl_xor_sync(0xffffffffu, qlo, o));
    qhi = max(qhi, __shfl_xor_sync(0xffffffffu, qhi, o));
  }
  if (qhi < 0) return;  // no lane has a summand
  const bool mine = (threadIdx.x & 31) == 0;
  const long long w[5] = {a.w0, a.w1, a.w2, a.w3, a.w4};
  const int sh = has ? a.qa - qlo : 0;  // this lane's offset inside the span
#pragma unroll 2
  for (int p = 0; p <= qhi - qlo + 4; ++p) {  // digit qlo + p (warp-uniform bound, <= kLimbs)
    const int j = p - sh;  // this lane's window word at that digit
    long long v = 0;
#pragma unroll
    for (int u = 0; u < 5; ++u) v = (has && j == u) ? w[u] : v;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (mine && v) atomicAdd(reinterpret_cast<unsigned long long *>(&blk[qlo + p]), (unsigned long long)v);
  }
}

// Round the exact value held in limbs to the nearest double (ties to even).
// Register-only: every array index below is a compile-time constant (fully unrolled loops,
// selects instead of dynamic indexing), so nothing goes through local memory -- this runs
// on one thread at the end of every reduction, on the critical path.
__device__ __noinline__ double xacc_round(const long long *limbs) {
  long long d[kLimbs];
#pragma unroll
  for (int i = 0; i < kLimbs; ++i) d[i] = limbs[i];
  // carry-normalize digits 0..8 into [0, 2^32)
#pragma unroll
  for (int i = 0; i < kLimbs - 1; ++i) {
    const long long c = d[i] >> 32;  // arithmetic shift = floor division
    d[i] -= c * 4294967296ll;
    d[i + 1] += c;
  }
  const bool neg = d[kLimbs - 1] < 0;
  if (neg) {  // negate every limb and renormalize: value becomes non-negative
#pragma unroll
    for (int i = 0; i < kLimbs; ++i) d[i] = -d[i];
#pragma unroll
    for (int i = 0; i < kLimbs - 1; ++i) {
      const long long c = d[i] >> 32;
      d[i] -= c * 4294967296ll;
      d[i + 1] += c;
    }
  }
  constexpr int ND = kLimbs + 1;
  unsigned int mag[ND];
#pragma unroll
  for (int i = 0; i < kLimbs - 1; ++i) mag[i] = (unsigned int)d[i];
  mag[kLimbs - 1] = (unsigned int)((unsigned long long)d[kLimbs - 1] & 0xffffffffull);
  mag[kLimbs] = (unsigned int)((unsigned long long)d[kLimbs - 1] >> 32);
  int top = -1;
  unsigned int mtop = 0u;
#pragma unroll
  for (int i = 0; i < ND; ++i)
    if (mag[i]) { top = i; mtop = mag[i]; }
  if (top < 0) return 0.0;
  const int B = top * 32 + (31 - __clz(mtop));  // highest set bit
  // word j of the magnitude (0 outside [0, ND)), by select
  auto word = [&](int j) -> unsigned int {
    unsigned int w = 0u;
#pragma unroll
    for (int i = 0; i < ND; ++i) w = (i == j) ? mag[i] : w;
    return w;
  };
  // bits [lo, lo + cnt) (cnt <= 64, lo >= 0)
  auto bits = [&](int lo, int cnt) -> unsigned long long {
    const int di = lo >> 5, off = lo & 31;
    const unsigned __int128 w = ((unsigned __int128)word(di + 2) << 64) | ((unsigned __int128)word(di + 1) << 32) |
                                (unsigned __int128)word(di);
    const unsigned long long out = (unsigned long long)(w >> off);
    return cnt >= 64 ? out : (out & ((1ull << cnt) - 1ull));
  };
  double res;
  if (B <= 52) {
    const unsigned long long M = bits(0, B + 1);
    res = (double)M * 0x1p-200;  // exact: M < 2^53, result normal
  } else {
    const int shift = B - 52;  // bits dropped
    unsigned long long keep = bits(shift, 53);
    const unsigned long long rbit = bits(shift - 1, 1);
    // sticky: any of the bits [0, shift - 1)
    const int hi = shift - 1, full = hi >> 5, rem = hi & 31;
    unsigned int any = 0u;
#pragma unroll
    for (int i = 0; i < ND; ++i) {
      any |= (i < full) ? mag[i] : 0u;
      any |= (i == full && rem) ? (mag[i] & ((1u << rem) - 1u)) : 0u;
    }
    const bool sticky = any != 0u;
    if (rbit && (sticky || (keep & 1ull))) keep += 1ull;
    // value = keep * 2^(shift - 200); build the power of two from its exponent bits
    const int ex = shift + kLsbExp;  // in [-147, 160]
    const double p2 = __longlong_as_double((long long)(ex + 1023) << 52);
    res = (double)keep * p2;
  }
  return neg ? -res : res;
}

}  // namespace scg
