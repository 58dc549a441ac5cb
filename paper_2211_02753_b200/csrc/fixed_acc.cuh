// Order-independent float64 summation for atomic group-by accumulators.
//
// atomicAdd(double) sums in whatever order the warps arrive, so a float SUM
// computed with it differs from run to run in the last bits.  Here every
// value is converted to a fixed-point integer (resolution 2^-128) and added
// into a per-cell accumulator with integer atomics; integer addition is
// associative, so the cell's final value -- and its conversion back to the
// nearest double -- is bitwise identical whatever the order of the additions.
//
// Cell layout (kFixedWords u64 words): w[0..7] eight signed limb
// accumulators, limb j weighing 2^(32 j) of the 256-bit fixed-point value; an
// add splits the value's shifted 53-bit mantissa into (at most three) 32-bit
// pieces and adds each, negated for a negative value, to its limb with a
// non-returning 64-bit atomic (RED) -- no carry propagation at add time (a
// limb absorbs 2^31 additions), so no returning atomics: the carries are
// resolved once when the cell is read.  w[8] is a double side accumulator for
// the values outside the fixed-point range (|x| >= 2^88, inf, NaN), where
// ordinary float addition applies.  Bits below 2^-128 are truncated (a value
// keeps its full 53-bit mantissa down to |x| ~ 2^-75).  The result is the
// correctly rounded exact sum of the fixed-point values plus the side
// accumulator -- at least as accurate as the reference's sequential np.add.at
// (tq/kernels.py:147-153).
#pragma once

#include <cstdint>

namespace tdp {

constexpr int kFixedWords = 9;
constexpr int kFixedLimbs = 8;
constexpr int kFixedScale = 128;  // value = integer * 2^-128
constexpr int kFixedMaxExp = 88;  // |x| < 2^88 goes to the limbs

// A signed 64-bit add into a 64-bit word kept as two 32-bit halves (shared
// memory: 32-bit atomics are native there, 64-bit ones a CAS loop): the low
// half's returned old value gives this add's carry / borrow into the high
// half, so the word's total is exact under any interleaving.
__device__ __forceinline__ void split_add64(unsigned long long* word, unsigned long long x) {
  unsigned* h = reinterpret_cast<unsigned*>(word);  // [0] low, [1] high (little-endian)
  const unsigned lo = (unsigned)x;
  unsigned hi = (unsigned)(x >> 32);
  if (lo) {
    const unsigned old = atomicAdd(h, lo);
    hi += old > 0xffffffffu - lo ? 1u : 0u;  // carry out of the low half
  }
  if (hi) atomicAdd(h + 1, hi);
}

__device__ __forceinline__ void split_sub32(unsigned long long* word, unsigned x) {
  unsigned* h = reinterpret_cast<unsigned*>(word);
  const unsigned old = atomicSub(h, x);
  if (old < x) atomicSub(h + 1, 1u);  // borrow
}

template <bool kSplit>
__device__ __forceinline__ void fixed_add_impl(unsigned long long* cell, double x);

__device__ __forceinline__ void fixed_add(unsigned long long* cell, double x) {
  fixed_add_impl<false>(cell, x);
}

// fixed_add for a cell in shared memory (32-bit atomics, same words)
__device__ __forceinline__ void fixed_add_shared(unsigned long long* cell, double x) {
  fixed_add_impl<true>(cell, x);
}

template <bool kSplit>
__device__ __forceinline__ void fixed_add_impl(unsigned long long* cell, double x) {
  const long long bits = __double_as_longlong(x);
  const int e = (int)((bits >> 52) & 0x7ff);
  if (e == 0) return;  // +-0 and subnormals (< 2^-1022): below the resolution
  if (e == 0x7ff || e - 1075 + 53 > kFixedMaxExp) {
    atomicAdd(reinterpret_cast<double*>(cell + kFixedLimbs), x);  // inf / NaN / huge
    return;
  }
  unsigned long long m = ((unsigned long long)bits & ((1ull << 52) - 1)) | (1ull << 52);
  int sh = e - 1075 + kFixedScale;  // bit position of the mantissa's lsb
  if (sh <= -53) return;            // |x| < 2^-128: truncated
  if (sh < 0) {
    m >>= -sh;
    sh = 0;
  }
  const int j0 = sh >> 5, r = sh & 31;
  const unsigned __int128 t = (unsigned __int128)m << r;  // <= 84 bits
  const bool neg = bits < 0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const unsigned long long piece = (unsigned long long)(t >> (32 * i)) & 0xffffffffull;
    if (piece != 0ull && j0 + i < kFixedLimbs) {
      if (kSplit) {
        if (neg)
          split_sub32(cell + j0 + i, (unsigned)piece);
        else
          split_add64(cell + j0 + i, piece);
      } else {
        atomicAdd(cell + j0 + i, neg ? (unsigned long long)(-(long long)piece) : piece);
      }
    }
  }
}

// The cell's sum as the nearest double (round-to-nearest-even of the exact
// fixed-point total), plus the side accumulator.
__device__ __forceinline__ double fixed_value(const unsigned long long* cell) {
  // resolve the limbs' carries: a 256-bit two's-complement total in d[4]
  unsigned long long d[4] = {0ull, 0ull, 0ull, 0ull};
  __int128 carry = 0;
#pragma unroll
  for (int j = 0; j < kFixedLimbs; ++j) {
    const __int128 t = (__int128)(long long)cell[j] + carry;
    d[j >> 1] |= ((unsigned long long)t & 0xffffffffull) << (32 * (j & 1));
    carry = t >> 32;  // arithmetic: floor division
  }
  const bool neg = carry < 0;  // totals stay within +-2^255
  if (neg) {  // magnitude
    unsigned long long c = 1;
    for (int i = 0; i < 4; ++i) {
      d[i] = ~d[i] + c;
      c = (c && d[i] == 0ull) ? 1ull : 0ull;
    }
  }
  int top = 3;
  while (top >= 0 && d[top] == 0ull) --top;
  const double side = __longlong_as_double((long long)cell[kFixedLimbs]);
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
