// One pass over X per LLP training step.
//
// The LLP query (SURVEY config 4) is a soft COUNT grouped by a one-hot bag key
// and the PE column of a linear head with k = 2 classes:
//   grid[b, c] = sum_{i in bag b} P_ic,   P_i = softmax(x_i W + bias)
// (tq/kernels.py:190-229 over tq/models.py:26-27, tq/encodings.py:143-151).
// Its backward (tq/tensor.py:474, :364-365, softmax VJP :515-527) is, for
// upstream grid gradient G,
//   dZ_i = P_i0 P_i1 (G[b_i, 0] - G[b_i, 1]) [1, -1]
// because the softmax VJP P (g - <P, g>) collapses for two classes.  So
//   dW[:, 0] = sum_b g_b S_b,  dW[:, 1] = -dW[:, 0],  db = sum_b g_b Q_b [1, -1]
// with g_b = G[b, 0] - G[b, 1] and the per-bag statistics
//   S_b = sum_{i in b} P_i0 P_i1 x_i  (d values),  Q_b = sum_{i in b} P_i0 P_i1,
// formed in the forward pass at the same W.  The backward is then a tiny
// kernel over bags x features, and X is read once per step instead of twice.
//
// Rows are visited in bag order through a bag index of the one-hot key column
// (a stable permutation plus bag offsets, built once per code column, like an
// index on it): a warp owns a contiguous range of the bag-ordered rows, keeps
// S / Q / the two counts of the current bag in float64 registers and flushes
// them when the bag changes -- a few flushes per warp, into order-independent
// fixed-point cells (fixed_acc.cuh), so the statistics are bitwise
// repeatable.  Each warp step loads 32 whole rows (one coalesced 256-byte
// load per row for d = 64), forms the row dots with the butterfly
// transposition of the ring kernels (lane j ends with row j's logits), and
// the softmax per lane in the operation order of softmax_rows_kernel.
#include <cstring>

#include "fixed_acc.cuh"
#include "tdp_common.cuh"

namespace tdp {
namespace {

constexpr int kOpWarps = 4;
constexpr int kOpThreads = kOpWarps * 32;
constexpr int kOpCtasPerSm = 3;

// cell words of one bag: count c0, count c1, Q, then S[d]
__host__ __device__ __forceinline__ i64 op_cell(int bag, int d, int j) {
  return ((i64)bag * (3 + d) + j) * kFixedWords;
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem_dst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Gather 32 bag-ordered rows (row j = pj of lane j) into a warp's buffer with
// 16-byte async copies (measured faster here than one 256-byte bulk copy per
// row: 5.2 vs 6.2 ms at 1e8 x 64); the next group's rows are in flight while
// this one is computed.
template <int V>
__device__ __forceinline__ void op_issue(float* dst, const float* __restrict__ X, int pj, int cnt,
                                         int lane) {
  constexpr int d = 32 * V;
  constexpr int per_row = d / 4;  // 16-byte chunks per row
  constexpr int total = 32 * per_row;
#pragma unroll
  for (int c = lane; c < total; c += 32) {
    const int j = c / per_row, off = (c % per_row) * 4;
    const int row = __shfl_sync(0xffffffffu, pj, j);
    if (j < cnt) cp_async16(dst + j * d + off, X + (i64)row * d + off);
  }
  cp_async_commit();
}

template <int V>
__global__ void __launch_bounds__(kOpThreads, kOpCtasPerSm)
    llp_onepass_kernel(const float* __restrict__ X, i64 n, const int* __restrict__ perm,
                       const i64* __restrict__ offs, int B, const float* __restrict__ W,
                       const float* __restrict__ bias, i64 rows_per_warp,
                       unsigned long long* __restrict__ cells) {
  constexpr int d = 32 * V;
  extern __shared__ __align__(16) float op_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* buf = op_smem + (size_t)warp * 2 * 32 * d;  // [2][32][d]
  const i64 gw = (i64)blockIdx.x * kOpWarps + warp;
  const i64 r0 = gw * rows_per_warp;
  if (r0 >= n) return;
  const i64 r1 = r0 + rows_per_warp < n ? r0 + rows_per_warp : n;
  float w[V][2];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    w[v][0] = W[(lane * V + v) * 2];
    w[v][1] = W[(lane * V + v) * 2 + 1];
  }
  const float b0 = bias ? bias[0] : 0.f, b1 = bias ? bias[1] : 0.f;
  // the bag of row r0: offs is ascending, offs[0] = 0, offs[B] = n
  int lo = 0, hi = B;  // the last bag with offs[bag] <= r0
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(offs + mid) <= r0) lo = mid; else hi = mid;
  }
  int bag = lo;
  i64 next = __ldg(offs + bag + 1);
  double s[V], a0 = 0.0, a1 = 0.0, aq = 0.0;
#pragma unroll
  for (int v = 0; v < V; ++v) s[v] = 0.0;
#define TDP_FLUSH()                                                                      \
  do {                                                                                   \
    _Pragma("unroll") for (int v = 0; v < V; ++v) {                                      \
      fixed_add(cells + op_cell(bag, d, 3 + lane * V + v), s[v]);                        \
      s[v] = 0.0;                                                                        \
    }                                                                                    \
    if (lane == 0) {                                                                     \
      fixed_add(cells + op_cell(bag, d, 0), a0);                                         \
      fixed_add(cells + op_cell(bag, d, 1), a1);                                         \
      fixed_add(cells + op_cell(bag, d, 2), aq);                                         \
    }                                                                                    \
    a0 = a1 = aq = 0.0;                                                                  \
  } while (0)
  auto group_cnt = [&](i64 g) { return (int)(r1 - g < 32 ? r1 - g : 32); };
  int pj = r0 + lane < r1 ? __ldg(perm + r0 + lane) : 0;
  op_issue<V>(buf, X, pj, group_cnt(r0), lane);
  int pnext = r0 + 32 + lane < r1 ? __ldg(perm + r0 + 32 + lane) : 0;
  int slot = 0;
  for (i64 g0 = r0; g0 < r1; g0 += 32, slot ^= 1) {
    const int cnt = group_cnt(g0);
    // the next group's rows in flight, then the one after's row ids
    if (g0 + 32 < r1) op_issue<V>(buf + (slot ^ 1) * 32 * d, X, pnext, group_cnt(g0 + 32), lane);
    else cp_async_commit();
    pnext = g0 + 64 + lane < r1 ? __ldg(perm + g0 + 64 + lane) : 0;
    cp_async_wait1();
    __syncwarp();
    const float* sx = buf + slot * 32 * d;
    // row dots: per-lane partials of the 32 rows, butterfly transposition
    // (lane j ends with the full dot of row j)
    float p[16][2];
    const bool up16 = (lane & 16) != 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      float xa[V], xb[V];
      if constexpr (V == 2) {
        const float2 ta = r < cnt ? *reinterpret_cast<const float2*>(sx + r * d + lane * 2)
                                  : make_float2(0.f, 0.f);
        const float2 tb = r + 16 < cnt
                              ? *reinterpret_cast<const float2*>(sx + (r + 16) * d + lane * 2)
                              : make_float2(0.f, 0.f);
        xa[0] = ta.x;
        xa[1] = ta.y;
        xb[0] = tb.x;
        xb[1] = tb.y;
      } else {
        xa[0] = r < cnt ? sx[r * d + lane] : 0.f;
        xb[0] = r + 16 < cnt ? sx[(r + 16) * d + lane] : 0.f;
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float a = xa[0] * w[0][c], bb = xb[0] * w[0][c];
#pragma unroll
        for (int v = 1; v < V; ++v) {
          a += xa[v] * w[v][c];
          bb += xb[v] * w[v][c];
        }
        const float send = up16 ? a : bb;
        const float keep = up16 ? bb : a;
        p[r][c] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      }
    }
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
      const bool upper = (lane & o) != 0;
#pragma unroll
      for (int r = 0; r < o; ++r) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float send = upper ? p[r][c] : p[r + o][c];
          const float keep = upper ? p[r + o][c] : p[r][c];
          p[r][c] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
    }
    // lane j: logits of row j -> softmax (softmax_rows_kernel's order)
    const float z0 = p[0][0] + b0, z1 = p[0][1] + b1;
    const float m = nan_max(z0, z1);
    const float e0 = t_exp<float>(z0 - m), e1 = t_exp<float>(z1 - m);
    const float sum = e0 + e1;
    const float p0 = e0 / sum, p1 = e1 / sum;
    const bool valid = lane < cnt;
    const float q = valid ? p0 * p1 : 0.f;
    const float c0 = valid ? p0 : 0.f, c1 = valid ? p1 : 0.f;
    if (g0 + cnt <= next) {
      // the whole group in the current bag (the common case)
      // the group's 32 terms in float32 (relative error ~1e-7), then one
      // float64 add per group into the bag's accumulator
      float sg[V];
#pragma unroll
      for (int v = 0; v < V; ++v) sg[v] = 0.f;
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        if (j >= cnt) break;  // rows past a short last group: stale buffer contents
        const float qj = __shfl_sync(0xffffffffu, q, j);
        float xj[V];
        if constexpr (V == 2) {
          const float2 t = *reinterpret_cast<const float2*>(sx + j * d + lane * 2);
          xj[0] = t.x;
          xj[1] = t.y;
        } else {
          xj[0] = sx[j * d + lane];
        }
#pragma unroll
        for (int v = 0; v < V; ++v) sg[v] = fmaf(qj, xj[v], sg[v]);
      }
#pragma unroll
      for (int v = 0; v < V; ++v) s[v] += (double)sg[v];
      double t0 = c0, t1 = c1, tq = q;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        t0 += __shfl_xor_sync(0xffffffffu, t0, o);
        t1 += __shfl_xor_sync(0xffffffffu, t1, o);
        tq += __shfl_xor_sync(0xffffffffu, tq, o);
      }
      a0 += t0;
      a1 += t1;
      aq += tq;
      if (g0 + cnt == next && g0 + cnt < r1) {  // the bag ends with this group
        TDP_FLUSH();
        do next = __ldg(offs + (++bag) + 1); while (next <= g0 + cnt);
      }
    } else {
      // a bag boundary inside the group: row by row, flushing at each boundary
      for (int j = 0; j < cnt; ++j) {
        while (g0 + j >= next) {
          TDP_FLUSH();
          next = __ldg(offs + (++bag) + 1);
        }
        const float qj = __shfl_sync(0xffffffffu, q, j);
        const float cj0 = __shfl_sync(0xffffffffu, c0, j), cj1 = __shfl_sync(0xffffffffu, c1, j);
#pragma unroll
        for (int v = 0; v < V; ++v) s[v] = fma((double)qj, (double)sx[j * d + lane * V + v], s[v]);
        a0 += cj0;
        a1 += cj1;
        aq += qj;
      }
    }
    __syncwarp();  // the buffer is refilled two groups later
  }
  TDP_FLUSH();
#undef TDP_FLUSH
}

// out_grid[cell(b, c)] (float64) and stats[b][0 .. d] = Q_b, S_b from the cells
__global__ void llp_onepass_finalize_kernel(const unsigned long long* __restrict__ cells, int B,
                                            int d, i64 bag_stride, i64 dense_stride,
                                            double* __restrict__ grid, double* __restrict__ stats) {
  const i64 total = (i64)B * (3 + d);
  for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (i64)gridDim.x * blockDim.x) {
    const int bag = (int)(t / (3 + d)), j = (int)(t % (3 + d));
    const double v = fixed_value(cells + t * kFixedWords);
    if (j < 2)
      grid[(i64)bag * bag_stride + (i64)j * dense_stride] = v;
    else
      stats[(i64)bag * (1 + d) + (j - 2)] = v;
  }
}

// dW[f][0] = sum_b g_b S_b[f] = -dW[f][1];  db[0] = sum_b g_b Q_b = -db[1]
// (one warp per output, bags in a fixed order: deterministic)
__global__ void llp_onepass_bwd_kernel(const double* __restrict__ stats, int B, int d,
                                       const double* __restrict__ G, i64 bag_stride,
                                       i64 dense_stride, float* __restrict__ dW,
                                       float* __restrict__ db) {
  const int lane = threadIdx.x & 31;
  const int out = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);  // 0..d: feature, d: bias
  if (out > d) return;
  const int col = out < d ? 1 + out : 0;
  double acc = 0.0;
  for (int b = lane; b < B; b += 32) {
    const double g = G[(i64)b * bag_stride] - G[(i64)b * bag_stride + dense_stride];
    acc = fma(g, stats[(i64)b * (1 + d) + col], acc);
  }
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    if (out < d) {
      dW[out * 2] = (float)acc;
      dW[out * 2 + 1] = (float)-acc;
    } else if (db != nullptr) {
      db[0] = (float)acc;
      db[1] = (float)-acc;
    }
  }
}

}  // namespace
}  // namespace tdp

using namespace tdp;

extern "C" {

size_t tdp_llp_onepass_workspace(int32_t bags, int32_t d) {
  return (size_t)bags * (3 + d) * kFixedWords * 8 + 256;
}

int tdp_llp_onepass_fwd(const float* X, int64_t n, int32_t d, const float* W, const float* bias,
                        const int32_t* perm, const int64_t* offs, int32_t bags, int64_t bag_stride,
                        int64_t dense_stride, double* out_grid, double* out_stats, void* ws,
                        size_t ws_bytes, void* stream) {
  TDP_REQUIRE(d == 32 || d == 64, "llp_onepass: d must be 32 or 64 (got %d)", d);
  TDP_REQUIRE(n >= 0 && bags >= 1 && n < ((int64_t)1 << 31), "llp_onepass: bad sizes");
  TDP_REQUIRE(((uintptr_t)X & 15) == 0, "llp_onepass: X must be 16-byte aligned");
  TDP_REQUIRE(ws != nullptr && ws_bytes >= tdp_llp_onepass_workspace(bags, d),
              "llp_onepass: workspace too small");
  cudaStream_t st = as_stream(stream);
  unsigned long long* cells = reinterpret_cast<unsigned long long*>(ws);
  TDP_CUDA_TRY(cudaMemsetAsync(cells, 0, (size_t)bags * (3 + d) * kFixedWords * 8, st));
  if (n > 0) {
    const i64 warps = (i64)sm_count() * kOpCtasPerSm * kOpWarps;
    i64 rpw = ceil_div(n, warps);
    rpw = ceil_div(rpw, 32) * 32;
    const unsigned grid = (unsigned)ceil_div(ceil_div(n, rpw), kOpWarps);
    const size_t smem = (size_t)kOpWarps * 2 * 32 * d * sizeof(float);
    if (d == 64) {
      TDP_CUDA_TRY(cudaFuncSetAttribute(llp_onepass_kernel<2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      llp_onepass_kernel<2><<<grid, kOpThreads, smem, st>>>(X, n, perm, offs, bags, W, bias, rpw,
                                                             cells);
    } else {
      TDP_CUDA_TRY(cudaFuncSetAttribute(llp_onepass_kernel<1>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      llp_onepass_kernel<1><<<grid, kOpThreads, smem, st>>>(X, n, perm, offs, bags, W, bias, rpw,
                                                             cells);
    }
    TDP_LAUNCH_CHECK("llp_onepass_kernel");
  }
  llp_onepass_finalize_kernel<<<stream_grid((i64)bags * (3 + d), 256, 8), 256, 0, st>>>(
      cells, bags, d, bag_stride, dense_stride, out_grid, out_stats);
  TDP_LAUNCH_CHECK("llp_onepass_finalize_kernel");
  return TDP_OK;
}

int tdp_llp_onepass_bwd(const double* stats, int32_t bags, int32_t d, const double* grad_grid,
                        int64_t bag_stride, int64_t dense_stride, float* dW, float* db,
                        void* stream) {
  TDP_REQUIRE(bags >= 1 && d >= 1 && stats != nullptr && grad_grid != nullptr && dW != nullptr,
              "llp_onepass_bwd: bad arguments");
  const unsigned blocks = (unsigned)ceil_div((i64)d + 1, 8);
  llp_onepass_bwd_kernel<<<blocks, 256, 0, as_stream(stream)>>>(stats, bags, d, grad_grid,
                                                                bag_stride, dense_stride, dW, db);
  TDP_LAUNCH_CHECK("llp_onepass_bwd_kernel");
  return TDP_OK;
}

}  // extern "C"
