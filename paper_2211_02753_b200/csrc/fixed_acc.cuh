// Order-independent float64 summation for atomic group-by accumulators.
//
// atomicAdd(double) sums in whatever order the warps arrive, so a float SUM
// computed with it differs from run to run in the last bits.  Here every
// value is converted to a fixed-point integer (resolution 2^-128) and added
// into a per-cell 256-bit two's-complement accumulator with 64-bit integer
// atomics; integer addition is associative, so the cell's final value -- and
// its conversion back to the nearest double -- is bitwise identical whatever
// the order of the additions.
//
// Cell layout (kFixedWords u64 words): w[0..3] the 256-bit accumulator
// (little-endian words), w[4] a double side accumulator for the values
// outside the fixed-point range (|x| >= 2^88, inf, NaN), where ordinary
// float addition applies.  |x| < 2^88 keeps 2^40 additions of headroom.
// Bits below 2^-128 are truncated (a value keeps its full 53-bit mantissa
// down to |x| ~ 2^-75).  The result is the correctly rounded exact sum of the
// fixed-point values plus the side accumulator -- at least as accurate as the
// reference's sequential np.add.at (tq/kernels.py:147-153).
#pragma once

#include <cstdint>

namespace tdp {

constexpr int kFixedWords = 5;
constexpr int kFixedScale = 128;  // value = integer * 2^-128
constexpr int kFixedMaxExp = 88;  // |x| < 2^88 goes to the integer words

// w += v (4-word two's complement), one atomic per nonzero word + carries;
// words below `first` of v are zero.
__device__ __forceinline__ void fixed_add_words(unsigned long long* w, const unsigned long long v[4],
                                                int first) {
  unsigned long long carry = 0;
  for (int i = first; i < 4; ++i) {
    const unsigned long long t = v[i] + carry;
    carry = t < v[i] ? 1ull : 0ull;  // v[i] = ~0 and a carry in: wraps to 0
    if (t != 0ull) {
      const unsigned long long old = atomicAdd(w + i, t);
      carry += (old + t < old) ? 1ull : 0ull;
    }
  }
}

__device__ __forceinline__ void fixed_add(unsigned long long* cell, double x) {
  const long long bits = __double_as_longlong(x);
  const int e = (int)((bits >> 52) & 0x7ff);
  if (e == 0) return;  // +-0 and subnormals (< 2^-1022): below the resolution
  if (e == 0x7ff || e - 1075 + 53 > kFixedMaxExp) {
    atomicAdd(reinterpret_cast<double*>(cell + 4), x);  // inf / NaN / huge
    return;
  }
  const unsigned long long m = ((unsigned long long)bits & ((1ull << 52) - 1)) | (1ull << 52);
  const int sh = e - 1075 + kFixedScale;  // bit position of the mantissa's lsb
  if (sh <= -53) return;                  // |x| < 2^-128: truncated
  unsigned long long v[4] = {0ull, 0ull, 0ull, 0ull};
  int first = 0;
  if (sh < 0) {
    v[0] = m >> (-sh);
  } else {
    const int word = sh >> 6, r = sh & 63;
    v[word] = m << r;
    if (r && word < 3) v[word + 1] = m >> (64 - r);
    first = word;
  }
  if (bits < 0) {  // two's complement of the magnitude: ~v + 1 over all words
    unsigned long long c = 1;
    for (int i = 0; i < 4; ++i) {
      v[i] = ~v[i] + c;
      c = (c && v[i] == 0ull) ? 1ull : 0ull;
    }
    // the words below the magnitude's lowest set word stay zero
  }
  fixed_add_words(cell, v, first);
}

// The cell's sum as the nearest double (round-to-nearest-even of the exact
// fixed-point total), plus the side accumulator.
__device__ __forceinline__ double fixed_value(const unsigned long long* cell) {
  unsigned long long d[4] = {cell[0], cell[1], cell[2], cell[3]};
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
  const double side = __longlong_as_double((long long)cell[4]);
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
