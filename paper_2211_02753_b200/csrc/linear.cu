// Skinny dense layers of the models embedded in trainable queries:
//   Y[n, k] = X[n, d] . W[d, k]            (tdp_linear_fwd)
//   dW[d, k] = X^T . G,  db[k] = sum_i G   (tdp_linear_wgrad)
// for k <= 8 output classes and d <= 256 features.
//
// Reference: matmul and its VJP, tq/tensor.py:437-454, reached through
// Linear.__call__ (tq/models.py:26-27) inside a classifier TVF.  In the LLP
// query (SURVEY config 4) these two products read the [1e8, 64] feature matrix
// and dominate the step; a general GEMM library treats m = 1e8, n = 2 as a
// tall-skinny problem and runs it far below HBM bandwidth.
//
// Both kernels stream X in row tiles: a CTA loads TILE consecutive rows (one
// contiguous span of TILE*d elements) with fully coalesced 16-byte loads into
// shared memory laid out with an odd row stride (d+1) so that per-row and
// per-column reads are bank-conflict free, then computes from shared memory.
// The arithmetic intensity is ~k/2 flop/byte -- far below the tensor-core
// ridge -- so CUDA-core FMAs at HBM speed are the roofline.
#include "stream_ring.cuh"

namespace tdp {
namespace {

constexpr int kMaxK = 8;
constexpr int kMaxD = 256;
constexpr int kMaxTile = 128;  // rows per tile (fewer for wide float64 rows)
constexpr int kThreadsL = 256;

template <class T>
__device__ __forceinline__ void load_tile(const T* __restrict__ X, i64 row0, i64 n, int d,
                                          int tile, T* __restrict__ s) {
  // tile*d contiguous elements starting at row0*d; rows past n read as 0
  const i64 base = row0 * d;
  const i64 total = (i64)tile * d;
  const i64 limit = n * (i64)d - base;
  if (sizeof(T) == 4 && (d % 4) == 0 && ((((uintptr_t)(X + base)) & 15) == 0)) {
    const float4* src = reinterpret_cast<const float4*>(X + base);
    for (i64 v = threadIdx.x; v < total / 4; v += blockDim.x) {
      const i64 e = v * 4;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < limit) q = __ldg(src + v);
      const int r = (int)(e / d), c = (int)(e % d);
      T* dst = s + r * (d + 1) + c;
      dst[0] = (T)q.x;
      dst[1] = (T)q.y;
      dst[2] = (T)q.z;
      dst[3] = (T)q.w;
    }
  } else {
    for (i64 e = threadIdx.x; e < total; e += blockDim.x) {
      const int r = (int)(e / d), c = (int)(e % d);
      s[r * (d + 1) + c] = e < limit ? __ldg(X + base + e) : T(0);
    }
  }
}

// Y = X W (+ b).  Warp w owns 32 rows of the tile; lane l owns features
// l, l+32, ... (its W entries live in registers).  Every lane forms partial dot
// products for all 32 rows, then a butterfly "transpose reduction" (5 levels
// of shuffles, halving the live partials each level) leaves the full sums of
// row (base + l) in lane l: ~2 shuffles per row instead of a 5-level
// reduction per row.  Shared-memory reads are conflict-free (a warp reads
// consecutive features of one row).
template <class T, int K>
__global__ void __launch_bounds__(kThreadsL)
    linear_fwd_kernel(const T* __restrict__ X, i64 n, int d, int tile, const T* __restrict__ W,
                      const T* __restrict__ bias, T* __restrict__ Y) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sx = reinterpret_cast<T*>(smem_raw);
  constexpr int kF = kMaxD / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nf = (d + 31) / 32;
  T w[kF][K];
#pragma unroll
  for (int f = 0; f < kF; ++f) {
    const int c = f * 32 + lane;
#pragma unroll
    for (int j = 0; j < K; ++j) w[f][j] = (f < nf && c < d) ? W[c * K + j] : T(0);
  }
  T bj[K];
#pragma unroll
  for (int j = 0; j < K; ++j) bj[j] = bias ? bias[j] : T(0);
  const i64 ntiles = (n + tile - 1) / tile;
  const int groups = tile / 32;
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    __syncthreads();
    load_tile<T>(X, t * tile, n, d, tile, sx);
    __syncthreads();
    for (int g = warp; g < groups; g += kThreadsL / 32) {
      if constexpr (K > 2) {
        // wide outputs: a plain per-row warp reduction keeps registers low
        for (int r = 0; r < 32; ++r) {
          const T* xr = sx + (g * 32 + r) * (d + 1);
          T q[K];
#pragma unroll
          for (int j = 0; j < K; ++j) q[j] = T(0);
#pragma unroll
          for (int f = 0; f < kF; ++f) {
            const int c = f * 32 + lane;
            if (f < nf && c < d) {
              const T x = xr[c];
#pragma unroll
              for (int j = 0; j < K; ++j) q[j] += x * w[f][j];
            }
          }
#pragma unroll
          for (int j = 0; j < K; ++j) q[j] = warp_sum(q[j]);
          const i64 row = t * tile + g * 32 + r;
          if (lane == 0 && row < n) {
#pragma unroll
            for (int j = 0; j < K; ++j) Y[row * K + j] = q[j] + bj[j];
          }
        }
        continue;
      }
      T p[32][K];
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const T* xr = sx + (g * 32 + r) * (d + 1);
#pragma unroll
        for (int j = 0; j < K; ++j) p[r][j] = T(0);
#pragma unroll
        for (int f = 0; f < kF; ++f) {
          if (f < nf) {
            const int c = f * 32 + lane;
            const T x = c < d ? xr[c] : T(0);
#pragma unroll
            for (int j = 0; j < K; ++j) p[r][j] += x * w[f][j];
          }
        }
      }
      // transpose reduction: after the level with offset o, lane l holds the
      // partial sums of the rows whose index bits above o match lane l's.
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int r = 0; r < o; ++r) {
#pragma unroll
          for (int j = 0; j < K; ++j) {
            const T send = upper ? p[r][j] : p[r + o][j];
            const T keep = upper ? p[r + o][j] : p[r][j];
            p[r][j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
      }
      const i64 row = t * tile + g * 32 + lane;
      if (row < n) {
#pragma unroll
        for (int j = 0; j < K; ++j) Y[row * K + j] = p[0][j] + bj[j];
      }
    }
  }
}

// dW = X^T G, db = sum G.  Thread t owns feature c = t mod (d+1) (c == d is
// the bias, x = 1) for every class and a row group t / (d+1); it sums its rows
// of each tile in T with K independent FMA chains and folds the tile sum into
// float64.  Row groups are combined in shared memory at the end; one partial
// row per CTA, reduced in a fixed order by wgrad_reduce_kernel.
template <class T, int K>
__global__ void __launch_bounds__(kThreadsL)
    linear_wgrad_kernel(const T* __restrict__ X, const T* __restrict__ G, i64 n, int d, int tile,
                        double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sx = reinterpret_cast<T*>(smem_raw);
  T* sg = sx + tile * (d + 1);
  const int nfeat = d + 1;
  const int ngroups = kThreadsL / nfeat > 0 ? kThreadsL / nfeat : 1;
  double acc[2][K];  // a thread owns <= 2 features when d + 1 > 256 threads
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int j = 0; j < K; ++j) acc[a][j] = 0.0;
  const i64 ntiles = (n + tile - 1) / tile;
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    __syncthreads();
    load_tile<T>(X, t * tile, n, d, tile, sx);
    for (int e = threadIdx.x; e < tile * K; e += blockDim.x) {
      const i64 row = t * tile + e / K;
      sg[e] = row < n ? G[t * tile * K + e] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int q = threadIdx.x + a * kThreadsL;
      const int c = q % nfeat, rg = q / nfeat;
      if (rg >= ngroups || (a == 1 && nfeat <= kThreadsL)) continue;
      double s[K];
#pragma unroll
      for (int j = 0; j < K; ++j) s[j] = 0.0;
      for (int r = rg; r < tile; r += ngroups) {
        const double x = c < d ? (double)sx[r * (d + 1) + c] : 1.0;
#pragma unroll
        for (int j = 0; j < K; ++j) s[j] += x * (double)sg[r * K + j];
      }
#pragma unroll
      for (int j = 0; j < K; ++j) acc[a][j] += (double)s[j];
    }
  }
  // combine row groups: reuse the tile buffer as [ngroups][nfeat*K] doubles
  __syncthreads();
  double* red = reinterpret_cast<double*>(smem_raw);
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int q = threadIdx.x + a * kThreadsL;
    const int c = q % nfeat, rg = q / nfeat;
    if (rg >= ngroups || (a == 1 && nfeat <= kThreadsL)) continue;
#pragma unroll
    for (int j = 0; j < K; ++j) red[(size_t)rg * nfeat * K + c * K + j] = acc[a][j];
  }
  __syncthreads();
  const int W = d * K + K;
  for (int e = threadIdx.x; e < nfeat * K; e += blockDim.x) {
    double v = 0.0;
    for (int rg = 0; rg < ngroups; ++rg) v += red[(size_t)rg * nfeat * K + e];
    // layout of the partial row: dW (d*K, row-major [c][j]) then db (K)
    part[(i64)blockIdx.x * W + e] = v;
  }
}

// ---------------------------------------------------------------------------
// bulk-copy ring variants: one producer warp streams contiguous row tiles of X
// (rows*d*sizeof(T) bytes each) into a shared-memory ring with
// cp.async.bulk (TMA engine); 8 consumer warps compute from shared memory.
// Unpadded tiles are conflict-free for both kernels (a warp reads consecutive
// features of one row).  Used when d*sizeof(T) is a multiple of 16 bytes.
// ---------------------------------------------------------------------------

struct RingShape {
  int rows;   // rows per stage (multiple of 32)
  int stages;
  size_t stage_bytes;
};

template <class T>
RingShape ring_shape(int d) {
  RingShape r;
  const size_t row_bytes = (size_t)d * sizeof(T);
  int rows = (int)((48 * 1024) / row_bytes);
  rows = (rows / 32) * 32;
  if (rows > 256) rows = 256;
  if (rows < 32) rows = 32;
  r.rows = rows;
  r.stage_bytes = (size_t)rows * row_bytes;
  int st = (int)((192 * 1024) / r.stage_bytes);
  r.stages = st < 2 ? 2 : (st > 4 ? 4 : st);
  return r;
}


template <class T, int K, int NF>
__global__ void __launch_bounds__(kRingThreads)
    linear_fwd_ring_kernel(const T* __restrict__ X, i64 n, int d, int rows, int stages,
                           const T* __restrict__ W, const T* __restrict__ bias, T* __restrict__ Y) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) u64 full[4];
  __shared__ __align__(8) u64 empty[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t stage_bytes = (size_t)rows * d * sizeof(T);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(smem_addr(&full[s]), 1);
      mbar_init(smem_addr(&empty[s]), kRingWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kRingWarps) {
    if (lane == 0) ring_produce<T>(X, nullptr, 0, n, d, rows, stages, stage_bytes, ring, full, empty);
    return;
  }
  constexpr int kF = NF;
  const int nf = (d + 31) / 32;
  T w[kF][K];
#pragma unroll
  for (int f = 0; f < kF; ++f) {
    const int c = f * 32 + lane;
#pragma unroll
    for (int j = 0; j < K; ++j) w[f][j] = (f < nf && c < d) ? W[c * K + j] : T(0);
  }
  T bj[K];
#pragma unroll
  for (int j = 0; j < K; ++j) bj[j] = bias ? bias[j] : T(0);
  const i64 ntiles = (n + rows - 1) / rows;
  int s = 0;
  unsigned fph = 0;
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(smem_addr(&full[s]), fph);
    const T* sx = reinterpret_cast<const T*>(ring + (size_t)s * stage_bytes);
    const i64 r0 = t * rows;
    for (int g = warp; g < rows / 32; g += kRingWarps) {
      if (r0 + g * 32 >= n) break;
      if constexpr (K > 2) {
        for (int r = 0; r < 32; ++r) {
          const i64 row = r0 + g * 32 + r;
          if (row >= n) break;
          const T* xr = sx + (size_t)(g * 32 + r) * d;
          T q[K];
#pragma unroll
          for (int j = 0; j < K; ++j) q[j] = T(0);
#pragma unroll
          for (int f = 0; f < kF; ++f) {
            const int c = f * 32 + lane;
            if (f < nf && c < d) {
              const T x = xr[c];
#pragma unroll
              for (int j = 0; j < K; ++j) q[j] += x * w[f][j];
            }
          }
#pragma unroll
          for (int j = 0; j < K; ++j) q[j] = warp_sum(q[j]);
          if (lane == 0) {
#pragma unroll
            for (int j = 0; j < K; ++j) Y[row * K + j] = q[j] + bj[j];
          }
        }
      } else {
        T p[32][K];
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const bool valid = r0 + g * 32 + r < n;
          const T* xr = sx + (size_t)(g * 32 + r) * d;
#pragma unroll
          for (int j = 0; j < K; ++j) p[r][j] = T(0);
#pragma unroll
          for (int f = 0; f < kF; ++f) {
            const int c = f * 32 + lane;
            if (f < nf) {
              const T x = (valid && c < d) ? xr[c] : T(0);
#pragma unroll
              for (int j = 0; j < K; ++j) p[r][j] += x * w[f][j];
            }
          }
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
          const bool upper = (lane & o) != 0;
#pragma unroll
          for (int r = 0; r < o; ++r) {
#pragma unroll
            for (int j = 0; j < K; ++j) {
              const T send = upper ? p[r][j] : p[r + o][j];
              const T keep = upper ? p[r + o][j] : p[r][j];
              p[r][j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
        }
        const i64 row = r0 + g * 32 + lane;
        if (row < n) {
#pragma unroll
          for (int j = 0; j < K; ++j) Y[row * K + j] = p[0][j] + bj[j];
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_addr(&empty[s]));
    if (++s == stages) {
      s = 0;
      fph ^= 1u;
    }
  }
}

template <class T, int K, int NF>
__global__ void __launch_bounds__(kRingThreads)
    linear_wgrad_ring_kernel(const T* __restrict__ X, const T* __restrict__ G, i64 n, int d,
                             int rows, int stages, int stage_g, double* __restrict__ part) {
  // Warp w takes rows w, w+8, ... of each staged tile; lane l owns features
  // l, l+32, ...: per row one conflict-free shared-memory read of the X row,
  // a broadcast read of the G row, independent float64 FMAs per (feature,
  // class).  Lane 0 also sums G for the bias.  One partial row per warp.
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) u64 full[4];
  __shared__ __align__(8) u64 empty[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t xbytes = (size_t)rows * d * sizeof(T);
  const size_t stage_bytes = xbytes + (size_t)rows * K * sizeof(T);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(smem_addr(&full[s]), 1);
      mbar_init(smem_addr(&empty[s]), kRingWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kRingWarps) {
    if (lane == 0)
      ring_produce<T>(X, stage_g ? G : nullptr, K, n, d, rows, stages, stage_bytes, ring, full,
                      empty);
    return;
  }
  constexpr int kF = NF;
  const int nf = (d + 31) / 32;
  double acc[kF][K];
  double bacc[K];
#pragma unroll
  for (int f = 0; f < kF; ++f)
#pragma unroll
    for (int j = 0; j < K; ++j) acc[f][j] = 0.0;
#pragma unroll
  for (int j = 0; j < K; ++j) bacc[j] = 0.0;
  const i64 ntiles = (n + rows - 1) / rows;
  int s = 0;
  unsigned fph = 0;
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(smem_addr(&full[s]), fph);
    const T* sx = reinterpret_cast<const T*>(ring + (size_t)s * stage_bytes);
    const T* sg = reinterpret_cast<const T*>(ring + (size_t)s * stage_bytes + xbytes);
    const i64 r0 = t * rows;
    const int nr = (int)((n - r0) < rows ? (n - r0) : rows);
    for (int r = warp; r < nr; r += kRingWarps) {
      double g[K];
#pragma unroll
      for (int j = 0; j < K; ++j)
        g[j] = stage_g ? (double)sg[r * K + j] : (double)__ldg(G + (r0 + r) * K + j);
      const T* xr = sx + (size_t)r * d;
#pragma unroll
      for (int f = 0; f < kF; ++f) {
        const int c = f * 32 + lane;
        if (f < nf && c < d) {
          const double x = (double)xr[c];
#pragma unroll
          for (int j = 0; j < K; ++j) acc[f][j] += x * g[j];
        }
      }
#pragma unroll
      for (int j = 0; j < K; ++j) bacc[j] += g[j];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_addr(&empty[s]));
    if (++s == stages) {
      s = 0;
      fph ^= 1u;
    }
  }
  const int W = d * K + K;
  double* out = part + ((i64)blockIdx.x * kRingWarps + warp) * W;
#pragma unroll
  for (int f = 0; f < kF; ++f) {
    const int c = f * 32 + lane;
    if (f < nf && c < d) {
#pragma unroll
      for (int j = 0; j < K; ++j) out[c * K + j] = acc[f][j];
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < K; ++j) out[d * K + j] = bacc[j];
  }
}

// ---------------------------------------------------------------------------
// vectorised ring kernels for d = 32 * V (the common model widths): lane l
// owns the V consecutive features [l*V, l*V + V) and reads them with one
// vector shared-memory load per row; every stage holds 256 rows (32 per
// consumer warp) so all consumer warps work on every stage; full stages run
// without bounds checks.
// ---------------------------------------------------------------------------

template <class T, int K, int V>
__global__ void __launch_bounds__(kRingThreads)
    linear_fwd_vec_kernel(const T* __restrict__ X, i64 n, int stages, const T* __restrict__ W,
                          const T* __restrict__ bias, T* __restrict__ Y) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) u64 full[4];
  __shared__ __align__(8) u64 empty[4];
  constexpr int d = 32 * V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t stage_bytes = (size_t)kVecRows * d * sizeof(T);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(smem_addr(&full[s]), 1);
      mbar_init(smem_addr(&empty[s]), kRingWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kRingWarps) {
    if (lane == 0)
      ring_produce<T>(X, nullptr, 0, n, d, kVecRows, stages, stage_bytes, ring, full, empty);
    return;
  }
  T w[V][K];
#pragma unroll
  for (int v = 0; v < V; ++v)
#pragma unroll
    for (int j = 0; j < K; ++j) w[v][j] = W[(lane * V + v) * K + j];
  T bj[K];
#pragma unroll
  for (int j = 0; j < K; ++j) bj[j] = bias ? bias[j] : T(0);
  const i64 ntiles = (n + kVecRows - 1) / kVecRows;
  int s = 0;
  unsigned fph = 0;
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(smem_addr(&full[s]), fph);
    const T* sx = reinterpret_cast<const T*>(ring + (size_t)s * stage_bytes);
    const i64 r0 = t * kVecRows;
    T z[K];
    const i64 row = r0 + warp * 32 + lane;
    if (r0 + kVecRows <= n) {
      vec_row_dots<T, K, V, true>(sx, warp, r0, n, w, lane, z);
#pragma unroll
      for (int j = 0; j < K; ++j) Y[row * K + j] = z[j] + bj[j];
    } else if (r0 + warp * 32 < n) {
      vec_row_dots<T, K, V, false>(sx, warp, r0, n, w, lane, z);
      if (row < n) {
#pragma unroll
        for (int j = 0; j < K; ++j) Y[row * K + j] = z[j] + bj[j];
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_addr(&empty[s]));
    if (++s == stages) {
      s = 0;
      fph ^= 1u;
    }
  }
}

// dW / db: warp w takes rows w, w+8, ... of each stage; lane l owns features
// [l*V, l*V+V); per stage the products are summed in T (at most 32 rows per
// warp) and folded into float64 accumulators.  G's tile is staged behind X's.
template <class T, int K, int V>
__global__ void __launch_bounds__(kRingThreads)
    linear_wgrad_vec_kernel(const T* __restrict__ X, const T* __restrict__ G, i64 n, int stages,
                            int stage_g, double* __restrict__ part) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) u64 full[4];
  __shared__ __align__(8) u64 empty[4];
  constexpr int d = 32 * V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t xbytes = (size_t)kVecRows * d * sizeof(T);
  const size_t stage_bytes = xbytes + (size_t)kVecRows * K * sizeof(T);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(smem_addr(&full[s]), 1);
      mbar_init(smem_addr(&empty[s]), kRingWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kRingWarps) {
    if (lane == 0)
      ring_produce<T>(X, stage_g ? G : nullptr, K, n, d, kVecRows, stages, stage_bytes, ring,
                      full, empty);
    return;
  }
  double acc[V][K];
  double bacc[K];
#pragma unroll
  for (int v = 0; v < V; ++v)
#pragma unroll
    for (int j = 0; j < K; ++j) acc[v][j] = 0.0;
#pragma unroll
  for (int j = 0; j < K; ++j) bacc[j] = 0.0;
  const i64 ntiles = (n + kVecRows - 1) / kVecRows;
  int s = 0;
  unsigned fph = 0;
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(smem_addr(&full[s]), fph);
    const T* sx = reinterpret_cast<const T*>(ring + (size_t)s * stage_bytes);
    const T* sg = reinterpret_cast<const T*>(ring + (size_t)s * stage_bytes + xbytes);
    const i64 r0 = t * kVecRows;
    const int nr = (int)((n - r0) < kVecRows ? (n - r0) : kVecRows);
    T ps[V][K], pb[K];
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int j = 0; j < K; ++j) ps[v][j] = T(0);
#pragma unroll
    for (int j = 0; j < K; ++j) pb[j] = T(0);
    auto row = [&](int r) {
      T x[V], g[K];
      VecLoad<T, V>::ld(sx + (size_t)r * d + lane * V, x);
#pragma unroll
      for (int j = 0; j < K; ++j) g[j] = stage_g ? sg[r * K + j] : __ldg(G + (r0 + r) * K + j);
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int j = 0; j < K; ++j) ps[v][j] += x[v] * g[j];
#pragma unroll
      for (int j = 0; j < K; ++j) pb[j] += g[j];
    };
    if (nr == kVecRows) {
      // full stage: 32 rows per warp, unrolled so all shared loads issue early
#pragma unroll
      for (int i = 0; i < kVecRows / kRingWarps; ++i) row(warp + i * kRingWarps);
    } else {
      for (int r = warp; r < nr; r += kRingWarps) row(r);
    }
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int j = 0; j < K; ++j) acc[v][j] += (double)ps[v][j];
#pragma unroll
    for (int j = 0; j < K; ++j) bacc[j] += (double)pb[j];
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_addr(&empty[s]));
    if (++s == stages) {
      s = 0;
      fph ^= 1u;
    }
  }
  const int W = d * K + K;
  double* out = part + ((i64)blockIdx.x * kRingWarps + warp) * W;
#pragma unroll
  for (int v = 0; v < V; ++v)
#pragma unroll
    for (int j = 0; j < K; ++j) out[(lane * V + v) * K + j] = acc[v][j];
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < K; ++j) out[d * K + j] = bacc[j];
  }
}


// rows per tile: a multiple of 32 fitting 96 KB of shared memory, <= kMaxTile
template <class T>
int tile_rows(int d) {
  int t = (int)((96 * 1024) / ((size_t)(d + 1) * sizeof(T)));
  if (t > kMaxTile) t = kMaxTile;
  t = (t / 32) * 32;
  return t < 32 ? 32 : t;
}

template <class T>
size_t fwd_smem(int d, int k) {
  (void)k;
  return (size_t)tile_rows<T>(d) * (d + 1) * sizeof(T);
}

template <class T>
size_t wgrad_smem(int d, int k) {
  const int t = tile_rows<T>(d);
  const size_t tiles = (size_t)t * (d + 1) * sizeof(T) + (size_t)t * k * sizeof(T);
  const size_t red = (size_t)(kThreadsL + d + 1) * k * sizeof(double);  // row-group combine
  return tiles > red ? tiles : red;
}

template <class T>
int wgrad_grid(i64 n, int d) { return stream_grid((n + tile_rows<T>(d) - 1) / tile_rows<T>(d), 1, 2); }

// feature groups of 32 lanes, rounded up to a power of two (kernel template)
inline int nf_bucket(int d) {
  const int nf = (d + 31) / 32;
  return nf <= 1 ? 1 : nf <= 2 ? 2 : nf <= 4 ? 4 : 8;
}

template <class T>
bool ring_ok(const T* X, i64 n, int d) {
  return ((size_t)d * sizeof(T)) % 16 == 0 && (((uintptr_t)X) & 15) == 0 &&
         n >= (i64)ring_shape<T>(d).rows * 4;
}

template <class T>
int ring_wgrad_grid(i64 n, int d) {
  return stream_grid((n + ring_shape<T>(d).rows - 1) / ring_shape<T>(d).rows, 1, 1);
}

template <class T>
int vec_stages(int d, int k) {
  const size_t stage = (size_t)kVecRows * (d + k) * sizeof(T);
  const int st = (int)((200 * 1024) / stage);
  return st < 2 ? 2 : (st > 4 ? 4 : st);
}

template <class T>
int launch_fwd(const T* X, i64 n, int d, int k, const T* W, const T* b, T* Y, cudaStream_t st) {
  if (const int V = vec_width<T>(X, n, d)) {
    const int stages = vec_stages<T>(d, 0);
    const size_t smem = (size_t)stages * kVecRows * d * sizeof(T);
    const int grid = stream_grid((n + kVecRows - 1) / kVecRows, 1, 1);
    bool launched = false;
#define TDP_CASE(KK, VV)                                                                      \
  if constexpr (sizeof(T) == 4 || VV == 1) if (k == KK && V == VV) {                                                                \
    TDP_CUDA_TRY(cudaFuncSetAttribute(linear_fwd_vec_kernel<T, KK, VV>,                       \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    linear_fwd_vec_kernel<T, KK, VV><<<grid, kRingThreads, smem, st>>>(X, n, stages, W, b, Y); \
    launched = true;                                                                          \
  }
#define TDP_CASES(KK) TDP_CASE(KK, 1) TDP_CASE(KK, 2)
    TDP_CASES(1) TDP_CASES(2) TDP_CASES(3) TDP_CASES(4) TDP_CASES(5) TDP_CASES(6) TDP_CASES(7) TDP_CASES(8)
#undef TDP_CASES
#undef TDP_CASE
    if (launched) {
      TDP_LAUNCH_CHECK("linear_fwd_vec_kernel");
      return TDP_OK;
    }
  }
  if (ring_ok<T>(X, n, d)) {
    const RingShape rs = ring_shape<T>(d);
    const size_t smem = rs.stages * rs.stage_bytes;
    const int grid = stream_grid((n + rs.rows - 1) / rs.rows, 1, 1);
    const int nf = nf_bucket(d);
    bool launched = false;
#define TDP_CASE(KK, NN)                                                                     \
  if (k == KK && nf == NN) {                                                                 \
    TDP_CUDA_TRY(cudaFuncSetAttribute(linear_fwd_ring_kernel<T, KK, NN>,                     \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    linear_fwd_ring_kernel<T, KK, NN><<<grid, kRingThreads, smem, st>>>(X, n, d, rs.rows,    \
                                                                        rs.stages, W, b, Y); \
    launched = true;                                                                         \
  }
#define TDP_CASES(KK) TDP_CASE(KK, 1) TDP_CASE(KK, 2) TDP_CASE(KK, 4) TDP_CASE(KK, 8)
    TDP_CASES(1) TDP_CASES(2) TDP_CASES(3) TDP_CASES(4) TDP_CASES(5) TDP_CASES(6) TDP_CASES(7) TDP_CASES(8)
#undef TDP_CASES
#undef TDP_CASE
    if (!launched) return set_error(TDP_EINVAL, "linear: k=%d > %d", k, kMaxK);
    TDP_LAUNCH_CHECK("linear_fwd_ring_kernel");
    return TDP_OK;
  }
  const size_t smem = fwd_smem<T>(d, k);
  const int tile = tile_rows<T>(d);
  const int grid = stream_grid((n + tile - 1) / tile, 1, 4);
  switch (k) {
#define TDP_CASE(KK)                                                                        \
  case KK:                                                                                  \
    if (smem > 48 * 1024)                                                                   \
      TDP_CUDA_TRY(cudaFuncSetAttribute(linear_fwd_kernel<T, KK>,                           \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    linear_fwd_kernel<T, KK><<<grid, kThreadsL, smem, st>>>(X, n, d, tile, W, b, Y);        \
    break;
    TDP_CASE(1) TDP_CASE(2) TDP_CASE(3) TDP_CASE(4) TDP_CASE(5) TDP_CASE(6) TDP_CASE(7) TDP_CASE(8)
#undef TDP_CASE
    default:
      return set_error(TDP_EINVAL, "linear: k=%d > %d", k, kMaxK);
  }
  TDP_LAUNCH_CHECK("linear_fwd_kernel");
  return TDP_OK;
}

template <class T>
int launch_wgrad(const T* X, const T* G, i64 n, int d, int k, T* dW, T* db, double* ws,
                 size_t ws_bytes, cudaStream_t st) {
  if (const int V = vec_width<T>(X, n, d)) {
    const int stages = vec_stages<T>(d, k);
    const size_t smem = (size_t)stages * kVecRows * (d + k) * sizeof(T);
    const int grid = stream_grid((n + kVecRows - 1) / kVecRows, 1, 1);
    const int width = d * k + k;
    const int prow = grid * kRingWarps;
    const int stage_g = (((size_t)kVecRows * k * sizeof(T)) % 16 == 0) &&
                        (((size_t)(n % kVecRows) * k * sizeof(T)) % 16 == 0) &&
                        ((((uintptr_t)G) & 15) == 0);
    TDP_REQUIRE(ws_bytes >= (size_t)prow * width * sizeof(double), "linear_wgrad workspace too small");
    bool launched = false;
#define TDP_CASE(KK, VV)                                                                      \
  if constexpr (sizeof(T) == 4 || VV == 1) if (k == KK && V == VV) {                                                                \
    TDP_CUDA_TRY(cudaFuncSetAttribute(linear_wgrad_vec_kernel<T, KK, VV>,                     \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    linear_wgrad_vec_kernel<T, KK, VV><<<grid, kRingThreads, smem, st>>>(X, G, n, stages,     \
                                                                         stage_g, ws);        \
    launched = true;                                                                          \
  }
#define TDP_CASES(KK) TDP_CASE(KK, 1) TDP_CASE(KK, 2)
    TDP_CASES(1) TDP_CASES(2) TDP_CASES(3) TDP_CASES(4) TDP_CASES(5) TDP_CASES(6) TDP_CASES(7) TDP_CASES(8)
#undef TDP_CASES
#undef TDP_CASE
    if (launched) {
      TDP_LAUNCH_CHECK("linear_wgrad_vec_kernel");
      wgrad_reduce_kernel<T><<<(unsigned)ceil_div((i64)width * 32, 256), 256, 0, st>>>(
          ws, prow, width, dW, db, d * k);
      TDP_LAUNCH_CHECK("wgrad_reduce_kernel");
      return TDP_OK;
    }
  }
  if (ring_ok<T>(X, n, d)) {
    const RingShape rs = ring_shape<T>(d);
    const size_t stage = rs.stage_bytes + (size_t)rs.rows * k * sizeof(T);
    const size_t smem = rs.stages * stage;
    const int grid = ring_wgrad_grid<T>(n, d);
    const int width = d * k + k;
    const int prow = grid * kRingWarps;
    const int stage_g = (((size_t)rs.rows * k * sizeof(T)) % 16 == 0) &&
                        (((size_t)(n % rs.rows) * k * sizeof(T)) % 16 == 0) &&
                        ((((uintptr_t)G) & 15) == 0);
    TDP_REQUIRE(ws_bytes >= (size_t)prow * width * sizeof(double), "linear_wgrad workspace too small");
    const int nf = nf_bucket(d);
    bool launched = false;
#define TDP_CASE(KK, NN)                                                                     \
  if (k == KK && nf == NN) {                                                                 \
    TDP_CUDA_TRY(cudaFuncSetAttribute(linear_wgrad_ring_kernel<T, KK, NN>,                   \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    linear_wgrad_ring_kernel<T, KK, NN><<<grid, kRingThreads, smem, st>>>(X, G, n, d, rs.rows, \
                                                                          rs.stages, stage_g, ws); \
    launched = true;                                                                         \
  }
#define TDP_CASES(KK) TDP_CASE(KK, 1) TDP_CASE(KK, 2) TDP_CASE(KK, 4) TDP_CASE(KK, 8)
    TDP_CASES(1) TDP_CASES(2) TDP_CASES(3) TDP_CASES(4) TDP_CASES(5) TDP_CASES(6) TDP_CASES(7) TDP_CASES(8)
#undef TDP_CASES
#undef TDP_CASE
    if (!launched) return set_error(TDP_EINVAL, "linear: k=%d > %d", k, kMaxK);
    TDP_LAUNCH_CHECK("linear_wgrad_ring_kernel");
    wgrad_reduce_kernel<T><<<(unsigned)ceil_div((i64)width * 32, 256), 256, 0, st>>>(
        ws, prow, width, dW, db, d * k);
    TDP_LAUNCH_CHECK("wgrad_reduce_kernel");
    return TDP_OK;
  }
  const int grid = wgrad_grid<T>(n, d);
  const int width = d * k + k;
  const size_t smem = wgrad_smem<T>(d, k);
  const int tile = tile_rows<T>(d);
  TDP_REQUIRE(ws_bytes >= (size_t)grid * width * sizeof(double), "linear_wgrad workspace too small");
  switch (k) {
#define TDP_CASE(KK)                                                                        \
  case KK:                                                                                  \
    if (smem > 48 * 1024)                                                                   \
      TDP_CUDA_TRY(cudaFuncSetAttribute(linear_wgrad_kernel<T, KK>,                         \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    linear_wgrad_kernel<T, KK><<<grid, kThreadsL, smem, st>>>(X, G, n, d, tile, ws);        \
    break;
    TDP_CASE(1) TDP_CASE(2) TDP_CASE(3) TDP_CASE(4) TDP_CASE(5) TDP_CASE(6) TDP_CASE(7) TDP_CASE(8)
#undef TDP_CASE
    default:
      return set_error(TDP_EINVAL, "linear: k=%d > %d", k, kMaxK);
  }
  TDP_LAUNCH_CHECK("linear_wgrad_kernel");
  wgrad_reduce_kernel<T><<<(unsigned)ceil_div((i64)width * 32, 256), 256, 0, st>>>(ws, grid, width,
                                                                                 dW, db, d * k);
  TDP_LAUNCH_CHECK("wgrad_reduce_kernel");
  return TDP_OK;
}

}  // namespace
}  // namespace tdp

using namespace tdp;

extern "C" {

int tdp_linear_fwd(const void* X, int32_t dtype, int64_t n, int32_t d, int32_t k, const void* W,
                   const void* bias, void* Y, void* stream) {
  TDP_REQUIRE(n >= 0 && d >= 1 && d <= kMaxD && k >= 1 && k <= kMaxK,
              "linear: shape n=%lld d=%d k=%d outside 1<=d<=%d, 1<=k<=%d", (long long)n, d, k,
              kMaxD, kMaxK);
  if (n == 0) return TDP_OK;
  cudaStream_t st = as_stream(stream);
  if (dtype == TDP_F32)
    return launch_fwd<float>((const float*)X, n, d, k, (const float*)W, (const float*)bias,
                             (float*)Y, st);
  if (dtype == TDP_F64)
    return launch_fwd<double>((const double*)X, n, d, k, (const double*)W, (const double*)bias,
                              (double*)Y, st);
  return set_error(TDP_EINVAL, "linear: float32/float64 only");
}

size_t tdp_linear_wgrad_workspace(int64_t n, int32_t d, int32_t k) {
  int g = wgrad_grid<double>(n, d);
  const int cands[4] = {wgrad_grid<float>(n, d), ring_wgrad_grid<float>(n, d) * kRingWarps,
                        ring_wgrad_grid<double>(n, d) * kRingWarps,
                        stream_grid((n + kVecRows - 1) / kVecRows, 1, 1) * kRingWarps};
  for (int c : cands) g = c > g ? c : g;
  return (size_t)g * (size_t)(d * k + k) * sizeof(double) + 256;
}

int tdp_linear_wgrad(const void* X, const void* G, int32_t dtype, int64_t n, int32_t d, int32_t k,
                     void* dW, void* db, void* ws, size_t ws_bytes, void* stream) {
  TDP_REQUIRE(n >= 0 && d >= 1 && d <= kMaxD && k >= 1 && k <= kMaxK, "linear_wgrad: bad shape");
  cudaStream_t st = as_stream(stream);
  if (dtype == TDP_F32)
    return launch_wgrad<float>((const float*)X, (const float*)G, n, d, k, (float*)dW, (float*)db,
                               (double*)ws, ws_bytes, st);
  if (dtype == TDP_F64)
    return launch_wgrad<double>((const double*)X, (const double*)G, n, d, k, (double*)dW,
                                (double*)db, (double*)ws, ws_bytes, st);
  return set_error(TDP_EINVAL, "linear_wgrad: float32/float64 only");
}

}  // extern "C"
