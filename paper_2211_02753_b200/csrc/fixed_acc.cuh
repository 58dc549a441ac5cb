// Order-independent float64 summation for atomic group-by accumulators.
//
// atomicAdd(double) sums in whatever order the warps arrive, so a float SUM
// computed with it differs from run to run in the last bits.  Here every
// value is converted to a fixed-point integer (resolution 2^-128) and added
// into a per-cell 256-bit accumulator with 64-bit integer atomics; integer
// addition is associative, so the cell's final value -- and its conversion
// back to the nearest double -- is bitwise identical whatever the order.
//
// Cell layout (kFixedWords u64 words): pos[4] and neg[4] hold the sums of
// the positive and negative values' magnitudes (no sign extension: a value
// touches only the two words its 53-bit mantissa straddles, plus carries),
// word 8 is a double side accumulator for the values outside the fixed-point
// range (|x| >= 2^88, inf, NaN), where ordinary float addition applies.
// Values below 2^-128 in magnitude are truncated (absolute error <= n 2^-128
// per cell).  The result is the correctly rounded exact sum of the (fixed-
// point) values plus the side accumulator -- at least as accurate as the
// reference's sequential np.add.at (tq/kernels.py:147-153).
#pragma once

#include <cstdint>

namespace tdp {

constexpr int kFixedWords = 9;
constexpr int kFixedScale = 128;  // value = integer * 2^-128
constexpr int kFixedMaxExp = 88;  // |x| < 2^88 goes to the integer words

__device__ __forceinline__ void fixed_add_words(unsigned long long* w, int word,
                                                unsigned long long lo, unsigned long long hi) {
  // add (hi:lo) << (64 * word) to the 4-word unsigned accumulator w
  unsigned long long carry = 0;
  for (int i = word; i < 4; ++i) {
    const unsigned long long t = i == word ? lo : (i == word + 1 ? hi : 0ull);
    const unsigned long long t2 = t + carry;
    const unsigned long long wrap = t2 < t ? 1ull : 0ull;
    carry = wrap;
    if (t2 != 0ull) {
      const unsigned long long old = atomicAdd(w + i, t2);
      carry += (old + t2 < old) ? 1ull : 0ull;
    }
    if (carry == 0ull && i > word) break;
  }
}

__device__ __forceinline__ void fixed_add(unsigned long long* cell, double x) {
  const long long bits = __double_as_longlong(x);
  const int e = (int)((bits >> 52) & 0x7ff);
  if (e == 0) return;  // +-0 and subnormals (< 2^-1022): below the resolution
  if (e == 0x7ff || e - 1075 + 53 > kFixedMaxExp) {
    atomicAdd(reinterpret_cast<double*>(cell + 8), x);  // inf / NaN / huge
    return;
  }
  const unsigned long long m = ((unsigned long long)bits & ((1ull << 52) - 1)) | (1ull << 52);
  const int sh = e - 1075 + kFixedScale;  // bit position of the mantissa's lsb
  if (sh <= -53) return;                  // |x| < 2^-128: truncated
  unsigned long long* w = bits < 0 ? cell + 4 : cell;
  if (sh < 0) {
    fixed_add_words(w, 0, m >> (-sh), 0ull);
  } else {
    const int word = sh >> 6, r = sh & 63;
    fixed_add_words(w, word, m << r, r ? (m >> (64 - r)) : 0ull);
  }
}

// The cell's sum as the nearest double (round-to-nearest-even of the exact
// fixed-point total), plus the side accumulator.
__device__ __forceinline__ double fixed_value(const unsigned long long* cell) {
  unsigned long long d[4];
  unsigned long long borrow = 0;
  for (int i = 0; i < 4; ++i) {  // d = pos - neg (256-bit two's complement)
    const unsigned long long a = cell[i], b = cell[4 + i];
    const unsigned long long t = a - b;
    const unsigned long long b1 = a < b ? 1ull : 0ull;
    d[i] = t - borrow;
    borrow = b1 | (t < borrow ? 1ull : 0ull);
  }
  const bool neg = (d[3] >> 63) != 0;
  if (neg) {  // magnitude
    unsigned long long c = 1;
    for (int i = 0; i < 4; ++i) {
      d[i] = ~d[i] + c;
      c = (c && d[i] == 0ull) ? 1ull : 0ull;
    }
  }
  int top = 3;
  while (top >= 0 && d[top] == 0ull) --top;
  const double side = __longlong_as_double((long long)cell[8]);
  if (top < 0) return 0.0 + side;
  const int s = __clzll((long long)d[top]);
  unsigned long long hi = d[top] << s;
  unsigned long long rest = 0;
  if (top > 0) {
    if (s) hi |= d[top - 1] >> (64 - s);
    rest = s ? (d[top - 1] << s) : d[top - 1];
    for (int i = top - 2; i >= 0; --i) rest |= d[i];
  }
  if (rest) hi |= 1ull;  // sticky bit: far below the 53-bit rounding position
  const int msb = 64 * top + 63 - s;  // bit index of the leading one
  double v = __ull2double_rn(hi);
  v = ldexp(v, msb - 63 - kFixedScale);
  return (neg ? -v : v) + side;
}

}  // namespace tdp
