// Shared pieces of the streaming skinny-product kernels (linear.cu, llp.cu):
// the bulk-copy producer of the shared-memory ring, vector loads of one
// lane's feature slice, the per-warp row-dot transposition and the float64
// reduction of per-warp weight-gradient partials.
#pragma once

#include "tdp_common.cuh"

namespace tdp {
namespace {

constexpr int kRingWarps = 8;
constexpr int kRingThreads = (kRingWarps + 1) * 32;

// Producer: per stage, the tile's X rows (in 8 KB bulk copies, so several
// requests are in flight) and, when G != nullptr, its G rows behind them.
// Returns through *g_in_smem whether G tiles are staged (their byte count must
// be a multiple of 16 for every tile).
template <class T>
__device__ __forceinline__ void ring_produce(const T* __restrict__ X, const T* __restrict__ G, int K,
                                             i64 n, int d, int rows, int stages,
                                             size_t stage_bytes, unsigned char* ring, u64* full,
                                             u64* empty) {
  const unsigned long long pol = l2_evict_first_policy();
  const i64 ntiles = (n + rows - 1) / rows;
  constexpr unsigned kChunk = 8 * 1024;
  int s = 0;
  unsigned eph = 0;
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(smem_addr(&empty[s]), eph ^ 1u);
    const i64 r0 = t * rows;
    const i64 nr = (n - r0) < rows ? (n - r0) : rows;
    const unsigned xbytes = (unsigned)(nr * d * (i64)sizeof(T));
    const unsigned gbytes = G ? (unsigned)(nr * K * (i64)sizeof(T)) : 0u;
    const unsigned bar = smem_addr(&full[s]);
    mbar_expect_tx(bar, xbytes + gbytes);
    unsigned char* dst = ring + (size_t)s * stage_bytes;
    const unsigned char* src = reinterpret_cast<const unsigned char*>(X + r0 * d);
    for (unsigned off = 0; off < xbytes; off += kChunk) {
      const unsigned b = xbytes - off < kChunk ? xbytes - off : kChunk;
      bulk_load(smem_addr(dst + off), src + off, b, bar, pol);
    }
    if (G)
      bulk_load(smem_addr(dst + (size_t)rows * d * sizeof(T)), G + r0 * K, gbytes, bar, pol);
    if (++s == stages) {
      s = 0;
      eph ^= 1u;
    }
  }
}

// ---------------------------------------------------------------------------
// vector ring path (d = 32*V): lane l owns features [l*V, l*V+V) of every row;
// stages hold kVecRows = 256 rows so the consumer loops have compile-time trip
// counts.  Full stages (all but the tail) run without bounds checks.
// ---------------------------------------------------------------------------
template <class T, int V>
struct VecLoad;
template <>
struct VecLoad<float, 1> {
  __device__ static void ld(const float* p, float* o) { o[0] = p[0]; }
};
template <>
struct VecLoad<float, 2> {
  __device__ static void ld(const float* p, float* o) {
    const float2 v = *reinterpret_cast<const float2*>(p);
    o[0] = v.x;
    o[1] = v.y;
  }
};
template <>
struct VecLoad<float, 4> {
  __device__ static void ld(const float* p, float* o) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    o[0] = v.x;
    o[1] = v.y;
    o[2] = v.z;
    o[3] = v.w;
  }
};
template <>
struct VecLoad<float, 8> {
  __device__ static void ld(const float* p, float* o) {
    VecLoad<float, 4>::ld(p, o);
    VecLoad<float, 4>::ld(p + 4, o + 4);
  }
};
template <int V>
struct VecLoad<double, V> {
  __device__ static void ld(const double* p, double* o) {
#pragma unroll
    for (int i = 0; i < V; i += 2) {
      if (i + 1 < V) {
        const double2 v = *reinterpret_cast<const double2*>(p + i);
        o[i] = v.x;
        o[i + 1] = v.y;
      } else {
        o[i] = p[i];
      }
    }
  }
};

constexpr int kVecRows = kRingWarps * 32;  // rows per stage in the vector kernels

// vector ring path: d = 32*V with a 256-row stage of at most 64 KB
template <class T>
int vec_width(const T* X, i64 n, int d) {
  if ((((uintptr_t)X) & 15) != 0 || n < (i64)kVecRows * 4 || d % 32 != 0) return 0;
  const int V = d / 32;
  if ((V != 1 && V != 2 && V != 4 && V != 8) || (size_t)d * sizeof(T) > 256) return 0;
  return V;
}

// Row dots of one 32-row group g of a stage: lane r ends with
// out[j] = sum_f X[r0 + 32g + r, f] W[f, j] (no bias) for its row r, via a
// butterfly transposition of the 32 x KC per-lane partial dots.  The first
// butterfly stage is applied as rows r and r+16 are computed, so at most
// 16 x KC partials are live; K is split into chunks of KC columns
// (re-reading the group's features from shared memory per chunk) to stay
// within the register budget of a 9-warp CTA (168 registers).
template <class T>
struct DotChunk {
  static constexpr int kc = sizeof(T) == 4 ? 8 : 2;
};

template <class T, int V, bool FULL>
__device__ __forceinline__ void load_row_slice(const T* __restrict__ sx, int g, int r, i64 r0,
                                               i64 n, int lane, T (&x)[V]) {
  constexpr int d = 32 * V;
  if (FULL || r0 + g * 32 + r < n) {
    VecLoad<T, V>::ld(sx + (size_t)(g * 32 + r) * d + lane * V, x);
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) x[v] = T(0);
  }
}

template <class T, int K, int V, bool FULL>
__device__ __forceinline__ void vec_row_dots(const T* __restrict__ sx, int g, i64 r0, i64 n,
                                             const T (&w)[V][K], int lane, T (&out)[K]) {
  constexpr int KC = K < DotChunk<T>::kc ? K : DotChunk<T>::kc;
  const bool upper16 = (lane & 16) != 0;
#pragma unroll
  for (int j0 = 0; j0 < K; j0 += KC) {
    T p[16][KC];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      T xa[V], xb[V];
      load_row_slice<T, V, FULL>(sx, g, r, r0, n, lane, xa);
      load_row_slice<T, V, FULL>(sx, g, r + 16, r0, n, lane, xb);
#pragma unroll
      for (int jj = 0; jj < KC; ++jj) {
        if (j0 + jj < K) {
          T a = xa[0] * w[0][j0 + jj];
          T b = xb[0] * w[0][j0 + jj];
#pragma unroll
          for (int v = 1; v < V; ++v) {
            a += xa[v] * w[v][j0 + jj];
            b += xb[v] * w[v][j0 + jj];
          }
          const T send = upper16 ? a : b;
          const T keep = upper16 ? b : a;
          p[r][jj] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
      }
    }
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
      const bool upper = (lane & o) != 0;
#pragma unroll
      for (int r = 0; r < o; ++r) {
#pragma unroll
        for (int jj = 0; jj < KC; ++jj) {
          if (j0 + jj < K) {
            const T send = upper ? p[r][jj] : p[r + o][jj];
            const T keep = upper ? p[r + o][jj] : p[r][jj];
            p[r][jj] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
      }
    }
#pragma unroll
    for (int jj = 0; jj < KC; ++jj)
      if (j0 + jj < K) out[j0 + jj] = p[0][jj];
  }
}

template <class T>
__global__ void wgrad_reduce_kernel(const double* __restrict__ part, int rows, int width,
                                    T* __restrict__ dW, T* __restrict__ db, int dk) {
  const int lane = threadIdx.x & 31;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < width;
       t += (gridDim.x * blockDim.x) >> 5) {
    double v = 0.0;
    for (int r = lane; r < rows; r += 32) v += part[(i64)r * width + t];
    v = warp_sum(v);
    if (lane == 0) {
      if (t < dk) dW[t] = (T)v;
      else if (db) db[t - dk] = (T)v;
    }
  }
}

}  // namespace
}  // namespace tdp
