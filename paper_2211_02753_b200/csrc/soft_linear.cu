// One-pass soft group-by COUNT whose single dense key is the PE column of a
// linear classifier head:  P = softmax(X W + b)  (pe_encode(Linear(X))).
//
// Reference (tq = /root/reference/pkg/src/tensorquery): the LLP query of
// SURVEY config 4 runs Linear.__call__ (tq/models.py:26-27: matmul + add,
// tq/tensor.py:437-447, :330-338), pe_encode's softmax (tq/encodings.py:143-151,
// tq/tensor.py:515-527) and soft_groupby's joint + reduce_sum
// (tq/kernels.py:190-229) as separate tape ops, each materialising an [n, k]
// (or [n, prod k]) intermediate.  Here
//
//   forward   grid[cell(i, c)] += P[i, c]           one pass over X
//   backward  dZ = P * (G[cell(i, .)] - <P, G[cell(i, .)]>)
//             dW = X^T dZ,  db = sum_i dZ           one pass over X (P recomputed)
//
// so the step reads X twice and nothing else of size n except the one-hot
// codes.  The per-row arithmetic (row dots, softmax, fixed-point count cells,
// softmax VJP) is the one of the unfused kernels (linear.cu, soft.cu), so the
// values agree with the composed path up to float32 rounding of dW's partials.
//
// Layout: X row-major [n, d] streamed through the bulk-copy ring of
// stream_ring.cuh (d = 32 V); the count grid (fixed point, 2 x u32 per cell)
// or the float copy of the upstream gradient grid lives in shared memory.
#include <cstring>

#include "stream_ring.cuh"

namespace tdp {
namespace {

constexpr int kMaxOneHot = 7;
constexpr int kMaxK = 8;
constexpr int kMaxCells = 8192;
constexpr double kFixScale = 1073741824.0;  // 2^30, as soft_fwd_count_smem_kernel

struct OneHotKeys {
  int n;
  int staged;  // codes of full stages ride in the ring behind the X rows
  const i64* codes[kMaxOneHot];
  i64 stride[kMaxOneHot];
  i64 dense_stride;
};

__device__ __forceinline__ i64 onehot_cell(const OneHotKeys& oh, i64 row) {
  i64 base = 0;
#pragma unroll
  for (int j = 0; j < kMaxOneHot; ++j)
    if (j < oh.n) base += __ldg(oh.codes[j] + row) * oh.stride[j];
  return base;
}

// Cell base of stage row `local` (global row `row`): from the stage's staged
// code rows when present (full stages), else from global memory.
__device__ __forceinline__ i64 onehot_cell_stage(const OneHotKeys& oh, const i64* __restrict__ sc,
                                                 bool full, int local, i64 row) {
  if (!(full && oh.staged)) return onehot_cell(oh, row);
  i64 base = 0;
#pragma unroll
  for (int j = 0; j < kMaxOneHot; ++j)
    if (j < oh.n) base += sc[j * kVecRows + local] * oh.stride[j];
  return base;
}

// Bytes of one ring stage: the X rows, then (staged) one 2 KB code row per key.
template <class T>
__host__ __device__ __forceinline__ size_t codes_offset(int d) {
  return (size_t)kVecRows * d * sizeof(T);
}
template <class T>
__host__ __device__ __forceinline__ size_t stage_size(int d, int staged_keys) {
  return codes_offset<T>(d) + (size_t)staged_keys * kVecRows * sizeof(i64);
}

// Producer of the soft-linear ring: X rows in 8 KB bulk copies (several in
// flight) and, for full stages, the tile's one-hot codes, so no consumer
// waits on a dependent global load of the group keys.
template <class T>
__device__ __forceinline__ void ring_produce_codes(const T* __restrict__ X, const OneHotKeys& oh,
                                                   i64 n, int d, int stages, size_t stage_bytes,
                                                   unsigned char* ring, u64* full, u64* empty) {
  const unsigned long long pol = l2_evict_first_policy();
  const i64 ntiles = (n + kVecRows - 1) / kVecRows;
  constexpr unsigned kChunk = 8 * 1024;
  int s = 0;
  unsigned eph = 0;
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(smem_addr(&empty[s]), eph ^ 1u);
    const i64 r0 = t * kVecRows;
    const i64 nr = (n - r0) < kVecRows ? (n - r0) : kVecRows;
    const unsigned xbytes = (unsigned)(nr * d * (i64)sizeof(T));
    const bool codes = oh.staged && nr == kVecRows;
    const unsigned cbytes = codes ? (unsigned)(oh.n * kVecRows * sizeof(i64)) : 0u;
    const unsigned bar = smem_addr(&full[s]);
    mbar_expect_tx(bar, xbytes + cbytes);
    unsigned char* dst = ring + (size_t)s * stage_bytes;
    const unsigned char* src = reinterpret_cast<const unsigned char*>(X + r0 * d);
    for (unsigned off = 0; off < xbytes; off += kChunk) {
      const unsigned b = xbytes - off < kChunk ? xbytes - off : kChunk;
      bulk_load(smem_addr(dst + off), src + off, b, bar, pol);
    }
    if (codes)
#pragma unroll
      for (int j = 0; j < kMaxOneHot; ++j)
        if (j < oh.n)
          bulk_load(smem_addr(dst + codes_offset<T>(d) + (size_t)j * kVecRows * sizeof(i64)),
                  oh.codes[j] + r0, kVecRows * sizeof(i64), bar, pol);
    if (++s == stages) {
      s = 0;
      eph ^= 1u;
    }
  }
}

// softmax of one row held in registers; same operation order as
// softmax_rows_kernel (soft.cu)
template <class T, int K>
__device__ __forceinline__ void softmax_row(const T (&z)[K], T (&p)[K]) {
  T m = z[0];
#pragma unroll
  for (int c = 1; c < K; ++c) m = nan_max(m, z[c]);
  T s = 0;
  T e[K];
#pragma unroll
  for (int c = 0; c < K; ++c) {
    e[c] = t_exp<T>(z[c] - m);
    s += e[c];
  }
#pragma unroll
  for (int c = 0; c < K; ++c) p[c] = e[c] / s;
}

// 64-bit fixed-point cell update in two u32 words (see soft.cu)
__device__ __forceinline__ void fix_add(unsigned* lo, unsigned* hi, double* grid, i64 cell,
                                        double prod) {
  if (prod >= 0.0 && prod <= 3.0) {
    const unsigned q = __double2uint_rn(prod * kFixScale);
    const unsigned old = atomicAdd(lo + cell, q);
    if (old > 0xffffffffu - q) atomicAdd(hi + cell, 1u);
  } else {
    atomicAdd(grid + cell, prod);
  }
}

template <class T, int K, int V>
__device__ __forceinline__ void load_head(const T* __restrict__ W, const T* __restrict__ bias,
                                          int lane, T (&w)[V][K], T (&bj)[K]) {
#pragma unroll
  for (int v = 0; v < V; ++v)
#pragma unroll
    for (int j = 0; j < K; ++j) w[v][j] = W[(lane * V + v) * K + j];
#pragma unroll
  for (int j = 0; j < K; ++j) bj[j] = bias ? bias[j] : T(0);
}

// Feature ownership of a lane: contiguous (features lane*V .. lane*V+V-1,
// d == 32 V, one vector load per row) or strided (features lane + 32 v, any
// d <= 32 V that is a multiple of 4, masked): the strided layout serves
// feature counts that are not a multiple of 32 with the same warp algorithms.
template <bool kStrided, int V>
__device__ __forceinline__ int feat(int lane, int v) {
  return kStrided ? lane + 32 * v : lane * V + v;
}

template <class T, int K, int V, bool kStrided>
__device__ __forceinline__ void load_head_l(const T* __restrict__ W, const T* __restrict__ bias,
                                            int lane, int d, T (&w)[V][K], T (&bj)[K]) {
  if constexpr (!kStrided) {
    load_head<T, K, V>(W, bias, lane, w, bj);
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int f = feat<kStrided, V>(lane, v);
#pragma unroll
      for (int j = 0; j < K; ++j) w[v][j] = f < d ? W[f * K + j] : T(0);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) bj[j] = bias ? bias[j] : T(0);
  }
}

template <class T, int V, bool kStrided>
__device__ __forceinline__ void load_row_l(const T* __restrict__ sxrow, int lane, int d,
                                           T (&x)[V]) {
  if constexpr (!kStrided) {
    VecLoad<T, V>::ld(sxrow + lane * V, x);
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int f = lane + 32 * v;
      x[v] = f < d ? sxrow[f] : T(0);
    }
  }
}

// Row dots of one 32-row group (see vec_row_dots, stream_ring.cuh): the
// contiguous layout is exactly vec_row_dots; the strided one the same
// butterfly transposition over the strided feature slices.
template <class T, int K, int V, bool FULL, bool kStrided>
__device__ __forceinline__ void row_dots(const T* __restrict__ sx, int g, i64 r0, i64 n, int d,
                                         const T (&w)[V][K], int lane, T (&out)[K]) {
  if constexpr (!kStrided) {
    vec_row_dots<T, K, V, FULL>(sx, g, r0, n, w, lane, out);
  } else {
    constexpr int KC = K < DotChunk<T>::kc ? K : DotChunk<T>::kc;
    const bool upper16 = (lane & 16) != 0;
#pragma unroll
    for (int j0 = 0; j0 < K; j0 += KC) {
      T p[16][KC];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        T xa[V], xb[V];
        if (FULL || r0 + g * 32 + r < n) load_row_l<T, V, true>(sx + (size_t)(g * 32 + r) * d, lane, d, xa);
        else
#pragma unroll
          for (int v = 0; v < V; ++v) xa[v] = T(0);
        if (FULL || r0 + g * 32 + r + 16 < n)
          load_row_l<T, V, true>(sx + (size_t)(g * 32 + r + 16) * d, lane, d, xb);
        else
#pragma unroll
          for (int v = 0; v < V; ++v) xb[v] = T(0);
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
}

// first maximum, NaN counting as the maximum (np.argmax, tdp_pe_argmax)
template <class T, int K>
__device__ __forceinline__ int argmax_row(const T (&p)[K]) {
  int best = 0;
  T bv = p[0];
  bool bnan = bv != bv;
#pragma unroll
  for (int c = 1; c < K; ++c) {
    const bool vn = p[c] != p[c];
    if (!bnan && (vn || p[c] > bv)) {
      best = c;
      bv = p[c];
      bnan = vn;
    }
  }
  return best;
}

// kArgmax: the exact swap of the same query (pe_decode of the head's PE column,
// tq/encodings.py:154-165, then an exact COUNT by the decoded keys): each row
// adds 1 to the cell of argmax(P) instead of P to every cell; grid is then a
// uint64 count grid.
template <class T, int K, int V, bool kArgmax, bool kStrided>
__global__ void __launch_bounds__(kRingThreads)
    soft_linear_count_fwd_kernel(const T* __restrict__ X, i64 n, int d_rt, int stages,
                                 const T* __restrict__ W, const T* __restrict__ bias,
                                 OneHotKeys oh, int cells, double* __restrict__ grid) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) u64 full[4];
  __shared__ __align__(8) u64 empty[4];
  const int d = kStrided ? d_rt : 32 * V;  // a compile-time constant unless strided
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t stage_bytes = stage_size<T>(d, oh.staged ? oh.n : 0);
  unsigned* lo = reinterpret_cast<unsigned*>(ring + (size_t)stages * stage_bytes);
  unsigned* hi = lo + cells;
  for (int c = threadIdx.x; c < 2 * cells; c += blockDim.x) lo[c] = 0u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(smem_addr(&full[s]), 1);
      mbar_init(smem_addr(&empty[s]), kRingWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kRingWarps) {
    if (lane == 0) ring_produce_codes<T>(X, oh, n, d, stages, stage_bytes, ring, full, empty);
  } else {
    T w[V][K], bj[K];
    load_head_l<T, K, V, kStrided>(W, bias, lane, d, w, bj);
    const i64 ntiles = (n + kVecRows - 1) / kVecRows;
    int s = 0;
    unsigned fph = 0;
    for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
      mbar_wait(smem_addr(&full[s]), fph);
      const T* sx = reinterpret_cast<const T*>(ring + (size_t)s * stage_bytes);
      const i64* sc = reinterpret_cast<const i64*>(ring + (size_t)s * stage_bytes + codes_offset<T>(d));
      const i64 r0 = t * kVecRows;
      const i64 row = r0 + warp * 32 + lane;
      const bool full_stage = r0 + kVecRows <= n;
      T z[K];
      bool valid = false;
      i64 base = 0;
      if (full_stage) {
        base = onehot_cell_stage(oh, sc, true, warp * 32 + lane, row);
        row_dots<T, K, V, true, kStrided>(sx, warp, r0, n, d, w, lane, z);
        valid = true;
      } else if (r0 + warp * 32 < n) {
        row_dots<T, K, V, false, kStrided>(sx, warp, r0, n, d, w, lane, z);
        valid = row < n;
        if (valid) base = onehot_cell(oh, row);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_addr(&empty[s]));
      if (valid) {
#pragma unroll
        for (int j = 0; j < K; ++j) z[j] += bj[j];
        T p[K];
        softmax_row<T, K>(z, p);
        if (kArgmax) {
          atomicAdd(lo + base + argmax_row<T, K>(p) * oh.dense_stride, 1u);
        } else {
#pragma unroll
          for (int j = 0; j < K; ++j)
            fix_add(lo, hi, grid, base + j * oh.dense_stride, (double)p[j]);
        }
      }
      if (++s == stages) {
        s = 0;
        fph ^= 1u;
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < cells; c += blockDim.x) {
    const unsigned l = lo[c], h = hi[c];
    if (kArgmax) {
      if (l) atomicAdd(reinterpret_cast<unsigned long long*>(grid) + c, (unsigned long long)l);
    } else if (l | h) {
      atomicAdd(grid + c, ((double)h * 4294967296.0 + (double)l) / kFixScale);
    }
  }
}

// Backward: per 32-row group, lane r recomputes P for row r, forms dZ from
// the shared copy of the upstream grid gradient and publishes it in shared
// memory; then every lane accumulates x[r, its features] * dZ[r, :] over the
// group's 32 rows (features re-read from the stage, released afterwards).
template <class T, int K, int V, bool kStrided>
__global__ void __launch_bounds__(kRingThreads)
    soft_linear_count_bwd_kernel(const T* __restrict__ X, i64 n, int d_rt, int stages,
                                 const T* __restrict__ W, const T* __restrict__ bias,
                                 OneHotKeys oh, int cells, const double* __restrict__ G,
                                 double* __restrict__ part) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) u64 full[4];
  __shared__ __align__(8) u64 empty[4];
  const int d = kStrided ? d_rt : 32 * V;  // a compile-time constant unless strided
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t stage_bytes = stage_size<T>(d, oh.staged ? oh.n : 0);
  T* sG = reinterpret_cast<T*>(ring + (size_t)stages * stage_bytes);
  T* sdz = sG + ((cells + 3) & ~3);  // [kRingWarps][32][K]
  for (int c = threadIdx.x; c < cells; c += blockDim.x) sG[c] = (T)G[c];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(smem_addr(&full[s]), 1);
      mbar_init(smem_addr(&empty[s]), kRingWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kRingWarps) {
    if (lane == 0) ring_produce_codes<T>(X, oh, n, d, stages, stage_bytes, ring, full, empty);
    return;
  }
  T w[V][K], bj[K];
  load_head_l<T, K, V, kStrided>(W, bias, lane, d, w, bj);
  T* mydz = sdz + warp * 32 * K;
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
    const i64* sc = reinterpret_cast<const i64*>(ring + (size_t)s * stage_bytes + codes_offset<T>(d));
    const i64 r0 = t * kVecRows;
    const i64 row = r0 + warp * 32 + lane;
    const bool active = r0 + warp * 32 < n;  // warp-uniform
    T z[K];
    bool valid = false;
    const bool full_stage = r0 + kVecRows <= n;
    i64 base = 0;
    if (full_stage) base = onehot_cell_stage(oh, sc, true, warp * 32 + lane, row);
    if (full_stage) {
      row_dots<T, K, V, true, kStrided>(sx, warp, r0, n, d, w, lane, z);
      valid = true;
    } else if (active) {
      row_dots<T, K, V, false, kStrided>(sx, warp, r0, n, d, w, lane, z);
      valid = row < n;
    }
    if (active) {
      T dz[K];
#pragma unroll
      for (int j = 0; j < K; ++j) dz[j] = T(0);
      if (valid) {
#pragma unroll
        for (int j = 0; j < K; ++j) z[j] += bj[j];
        T p[K], g[K];
        softmax_row<T, K>(z, p);
        if (!full_stage) base = onehot_cell(oh, row);
        T inner = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) {
          g[j] = sG[base + j * oh.dense_stride];
          inner += g[j] * p[j];
        }
#pragma unroll
        for (int j = 0; j < K; ++j) dz[j] = p[j] * (g[j] - inner);
      }
#pragma unroll
      for (int j = 0; j < K; ++j) {
        mydz[lane * K + j] = dz[j];
        bacc[j] += (double)dz[j];
      }
      __syncwarp();
      // dW partial: x[r, this lane's features] * dZ[r, :] over the group
      T ps[V][K];
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int j = 0; j < K; ++j) ps[v][j] = T(0);
      const int nrow = full_stage ? 32 : (int)((n - (r0 + warp * 32)) < 32 ? (n - (r0 + warp * 32)) : 32);
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        if (full_stage || r < nrow) {
          T x[V];
          if constexpr (kStrided)
            load_row_l<T, V, true>(sx + (size_t)(warp * 32 + r) * d, lane, d, x);
          else
            VecLoad<T, V>::ld(sx + (size_t)(warp * 32 + r) * (32 * V) + lane * V, x);
#pragma unroll
          for (int j = 0; j < K; ++j) {
            const T dr = mydz[r * K + j];
#pragma unroll
            for (int v = 0; v < V; ++v) ps[v][j] += x[v] * dr;
          }
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int j = 0; j < K; ++j) acc[v][j] += (double)ps[v][j];
    }
    __syncwarp();  // stage and mydz are reused after this point
    if (lane == 0) mbar_arrive(smem_addr(&empty[s]));
    if (++s == stages) {
      s = 0;
      fph ^= 1u;
    }
  }
  const int Wd = d * K + K;
  double* out = part + ((i64)blockIdx.x * kRingWarps + warp) * Wd;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int f = feat<kStrided, V>(lane, v);
    if (!kStrided || f < d)
#pragma unroll
      for (int j = 0; j < K; ++j) out[f * K + j] = acc[v][j];
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double b = warp_sum(bacc[j]);
    if (lane == 0) out[d * K + j] = b;
  }
}

// ---- host side ---------------------------------------------------------------

struct Plan {
  int V;          // features per lane (contiguous) or the strided VMAX
  bool strided;
  int stages;
  size_t smem;
  int grid;
};

// Strided instantiations: VMAX 4 (d <= 128; two 256-row stages must also fit
// shared memory, which bounds d to ~104 fp32 / ~52 fp64), within the
// register budget of the backward (168 registers at 288 threads): fp32
// k <= 4, fp64 k == 1.
template <class T>
constexpr bool strided_ok(int k, int vmax) {
  return vmax == 4 && (sizeof(T) == 4 ? k <= 4 : k == 1);
}

// Contiguous layout for d = 32 or 64 (fp32) / 32 (fp64); strided for any
// other d that is a multiple of 4 (bulk-copy granularity) up to 32 * VMAX.
template <class T>
bool plan_layout(const void* X, i64 n, int d, int k, int* V, bool* strided) {
  const int vw = vec_width<T>(reinterpret_cast<const T*>(X), n, d);
  if (vw >= 1 && vw <= 2 && (sizeof(T) == 4 || vw == 1)) {
    *V = vw;
    *strided = false;
    return true;
  }
  if ((((uintptr_t)X) & 15) != 0 || n < (i64)kVecRows * 4 || d < 1 || d % 4 != 0) return false;
  const int need = (d + 31) / 32;
  const int vmax = 4;
  if (need > vmax || !strided_ok<T>(k, vmax)) return false;
  *V = vmax;
  *strided = true;
  return true;
}

template <class T>
bool make_plan(const void* X, i64 n, int d, int k, i64 cells, bool bwd, int staged_keys, Plan* p) {
  int V = 0;
  bool strided = false;
  if (!plan_layout<T>(X, n, d, k, &V, &strided)) return false;
  if (k < 1 || k > kMaxK || cells < 1 || cells > kMaxCells) return false;
  const size_t stage = stage_size<T>(d, staged_keys);
  const size_t extra = bwd ? (size_t)((cells + 3) & ~3) * sizeof(T) +
                                 (size_t)kRingWarps * 32 * k * sizeof(T)
                           : (size_t)cells * 2 * sizeof(unsigned);
  const size_t budget = 220 * 1024;
  if (extra + 2 * stage > budget) return false;
  int st = (int)((budget - extra) / stage);
  st = st > 4 ? 4 : st;
  p->V = V;
  p->strided = strided;
  p->stages = st;
  p->smem = (size_t)st * stage + extra;
  p->grid = stream_grid((n + kVecRows - 1) / kVecRows, 1, 1);
  return true;
}

int make_keys(const tdp_soft_key* keys, int nkeys, int dense_key, int k, i64* cells,
              OneHotKeys* oh) {
  TDP_REQUIRE(keys != nullptr && nkeys >= 1 && nkeys <= kMaxOneHot + 1, "soft_linear: 1..%d keys",
              kMaxOneHot + 1);
  TDP_REQUIRE(dense_key >= 0 && dense_key < nkeys, "soft_linear: dense key index out of range");
  TDP_REQUIRE(keys[dense_key].kind == TDP_SOFT_DENSE && keys[dense_key].k == k,
              "soft_linear: key %d must be the dense [n, %d] PE of the linear head", dense_key, k);
  std::memset(oh, 0, sizeof(*oh));
  i64 stride = 1;
  for (int j = nkeys - 1; j >= 0; --j) {
    TDP_REQUIRE(keys[j].k >= 1, "soft_linear: key %d has no classes", j);
    if (j == dense_key) {
      oh->dense_stride = stride;
    } else {
      TDP_REQUIRE(keys[j].kind == TDP_SOFT_ONEHOT && keys[j].data != nullptr,
                  "soft_linear: key %d must be a one-hot code column", j);
      oh->codes[oh->n] = reinterpret_cast<const i64*>(keys[j].data);
      oh->stride[oh->n] = stride;
      ++oh->n;
    }
    stride *= keys[j].k;
    TDP_REQUIRE(stride <= kMaxCells, "soft_linear: grid exceeds %d cells", kMaxCells);
  }
  *cells = stride;
  // stage the codes in the ring when every code array is 16-byte aligned
  // (bulk-copy requirement; full stages start at multiples of 256 rows)
  oh->staged = oh->n > 0 ? 1 : 0;
  for (int j = 0; j < oh->n; ++j)
    if (((uintptr_t)oh->codes[j] & 15) != 0) oh->staged = 0;
  return TDP_OK;
}

template <class T, bool kArgmax = false>
int launch_fwd(const void* X, i64 n, int d, int k, const void* W, const void* b,
               const OneHotKeys& oh_in, i64 cells, double* grid, cudaStream_t st) {
  Plan p;
  OneHotKeys oh = oh_in;
  if (oh.staged && !make_plan<T>(X, n, d, k, cells, false, oh.n, &p)) oh.staged = 0;
  if (!oh.staged && !make_plan<T>(X, n, d, k, cells, false, 0, &p))
    return set_error(TDP_ENOTSUP, "soft_linear: unsupported shape (n=%lld d=%d k=%d cells=%lld)",
                     (long long)n, d, k, (long long)cells);
  bool launched = false;
#define TDP_CASE(KK, VV, SS)                                                                   \
  if constexpr (SS ? strided_ok<T>(KK, VV) : (sizeof(T) == 4 || VV == 1))                      \
  if (k == KK && p.V == VV && p.strided == SS) {                                               \
    TDP_CUDA_TRY(cudaFuncSetAttribute(soft_linear_count_fwd_kernel<T, KK, VV, kArgmax, SS>,    \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem)); \
    soft_linear_count_fwd_kernel<T, KK, VV, kArgmax, SS><<<p.grid, kRingThreads, p.smem, st>>>( \
        (const T*)X, n, d, p.stages, (const T*)W, (const T*)b, oh, (int)cells, grid);          \
    launched = true;                                                                           \
  }
#define TDP_CASES(KK) TDP_CASE(KK, 1, false) TDP_CASE(KK, 2, false) TDP_CASE(KK, 4, true)
  TDP_CASES(1) TDP_CASES(2) TDP_CASES(3) TDP_CASES(4) TDP_CASES(5) TDP_CASES(6) TDP_CASES(7) TDP_CASES(8)
#undef TDP_CASES
#undef TDP_CASE
  if (!launched) return set_error(TDP_ENOTSUP, "soft_linear: no kernel for k=%d V=%d", k, p.V);
  TDP_LAUNCH_CHECK("soft_linear_count_fwd_kernel");
  return TDP_OK;
}

template <class T>
int launch_bwd(const void* X, i64 n, int d, int k, const void* W, const void* b,
               const OneHotKeys& oh_in, i64 cells, const double* G, void* dW, void* db, void* ws,
               size_t ws_bytes, cudaStream_t st) {
  Plan p;
  OneHotKeys oh = oh_in;
  if (oh.staged && !make_plan<T>(X, n, d, k, cells, true, oh.n, &p)) oh.staged = 0;
  if (!oh.staged && !make_plan<T>(X, n, d, k, cells, true, 0, &p))
    return set_error(TDP_ENOTSUP, "soft_linear: unsupported shape (n=%lld d=%d k=%d cells=%lld)",
                     (long long)n, d, k, (long long)cells);
  const int width = d * k + k;
  const int prow = p.grid * kRingWarps;
  TDP_REQUIRE(ws_bytes >= (size_t)prow * width * sizeof(double), "soft_linear: workspace too small");
  double* part = reinterpret_cast<double*>(ws);
  bool launched = false;
#define TDP_CASE(KK, VV, SS)                                                                   \
  if constexpr (SS ? strided_ok<T>(KK, VV) : (sizeof(T) == 4 || VV == 1))                      \
  if (k == KK && p.V == VV && p.strided == SS) {                                               \
    TDP_CUDA_TRY(cudaFuncSetAttribute(soft_linear_count_bwd_kernel<T, KK, VV, SS>,             \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem)); \
    soft_linear_count_bwd_kernel<T, KK, VV, SS><<<p.grid, kRingThreads, p.smem, st>>>(         \
        (const T*)X, n, d, p.stages, (const T*)W, (const T*)b, oh, (int)cells, G, part);       \
    launched = true;                                                                           \
  }
#define TDP_CASES(KK) TDP_CASE(KK, 1, false) TDP_CASE(KK, 2, false) TDP_CASE(KK, 4, true)
  TDP_CASES(1) TDP_CASES(2) TDP_CASES(3) TDP_CASES(4) TDP_CASES(5) TDP_CASES(6) TDP_CASES(7) TDP_CASES(8)
#undef TDP_CASES
#undef TDP_CASE
  if (!launched) return set_error(TDP_ENOTSUP, "soft_linear: no kernel for k=%d V=%d", k, p.V);
  TDP_LAUNCH_CHECK("soft_linear_count_bwd_kernel");
  wgrad_reduce_kernel<T><<<(unsigned)ceil_div((i64)width * 32, 256), 256, 0, st>>>(
      part, prow, width, (T*)dW, (T*)db, d * k);
  TDP_LAUNCH_CHECK("wgrad_reduce_kernel");
  return TDP_OK;
}

}  // namespace
}  // namespace tdp

using namespace tdp;

extern "C" {

int tdp_soft_linear_supported(int32_t dtype, int64_t n, int32_t d, int32_t k, int64_t cells,
                              const void* X) {
  Plan p;
  if (dtype == TDP_F32)
    return make_plan<float>(X, n, d, k, cells, false, 0, &p) &&
           make_plan<float>(X, n, d, k, cells, true, 0, &p);
  if (dtype == TDP_F64)
    return make_plan<double>(X, n, d, k, cells, false, 0, &p) &&
           make_plan<double>(X, n, d, k, cells, true, 0, &p);
  return 0;
}

int tdp_soft_linear_count_fwd(const void* X, int32_t dtype, int64_t n, int32_t d, int32_t k,
                              const void* W, const void* bias, const tdp_soft_key* keys,
                              int32_t nkeys, int32_t dense_key, double* out_grid, void* stream) {
  i64 cells = 0;
  OneHotKeys oh;
  if (int rc = make_keys(keys, nkeys, dense_key, k, &cells, &oh)) return rc;
  cudaStream_t st = as_stream(stream);
  TDP_CUDA_TRY(cudaMemsetAsync(out_grid, 0, (size_t)cells * sizeof(double), st));
  if (n == 0) return TDP_OK;
  if (dtype == TDP_F32) return launch_fwd<float>(X, n, d, k, W, bias, oh, cells, out_grid, st);
  if (dtype == TDP_F64) return launch_fwd<double>(X, n, d, k, W, bias, oh, cells, out_grid, st);
  return set_error(TDP_EINVAL, "soft_linear: float32/float64 only");
}

int tdp_linear_argmax_count(const void* X, int32_t dtype, int64_t n, int32_t d, int32_t k,
                            const void* W, const void* bias, const tdp_soft_key* keys,
                            int32_t nkeys, int32_t dense_key, int64_t* out_counts, void* stream) {
  i64 cells = 0;
  OneHotKeys oh;
  if (int rc = make_keys(keys, nkeys, dense_key, k, &cells, &oh)) return rc;
  cudaStream_t st = as_stream(stream);
  TDP_CUDA_TRY(cudaMemsetAsync(out_counts, 0, (size_t)cells * sizeof(int64_t), st));
  if (n == 0) return TDP_OK;
  double* grid = reinterpret_cast<double*>(out_counts);
  if (dtype == TDP_F32) return launch_fwd<float, true>(X, n, d, k, W, bias, oh, cells, grid, st);
  if (dtype == TDP_F64) return launch_fwd<double, true>(X, n, d, k, W, bias, oh, cells, grid, st);
  return set_error(TDP_EINVAL, "linear_argmax_count: float32/float64 only");
}

size_t tdp_soft_linear_count_bwd_workspace(int64_t n, int32_t d, int32_t k) {
  const int grid = stream_grid((n + kVecRows - 1) / kVecRows, 1, 1);
  return (size_t)grid * kRingWarps * (size_t)(d * k + k) * sizeof(double) + 256;
}

int tdp_soft_linear_count_bwd(const void* X, int32_t dtype, int64_t n, int32_t d, int32_t k,
                              const void* W, const void* bias, const tdp_soft_key* keys,
                              int32_t nkeys, int32_t dense_key, const double* grad_grid, void* dW,
                              void* db, void* ws, size_t ws_bytes, void* stream) {
  i64 cells = 0;
  OneHotKeys oh;
  if (int rc = make_keys(keys, nkeys, dense_key, k, &cells, &oh)) return rc;
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    const size_t es = dtype == TDP_F64 ? 8 : 4;
    TDP_CUDA_TRY(cudaMemsetAsync(dW, 0, (size_t)d * k * es, st));
    if (db) TDP_CUDA_TRY(cudaMemsetAsync(db, 0, (size_t)k * es, st));
    return TDP_OK;
  }
  if (dtype == TDP_F32)
    return launch_bwd<float>(X, n, d, k, W, bias, oh, cells, grad_grid, dW, db, ws, ws_bytes, st);
  if (dtype == TDP_F64)
    return launch_bwd<double>(X, n, d, k, W, bias, oh, cells, grad_grid, dW, db, ws, ws_bytes, st);
  return set_error(TDP_EINVAL, "soft_linear: float32/float64 only");
}

}  // extern "C"
