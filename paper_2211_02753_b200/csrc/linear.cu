// Skinny dense layers of the models embedded in trainable queries:
//   Y[n, k] = X[n, d] . W[d, k]            (tdp_linear_fwd)
//   dW[d, k] = X^T . G,  db[k] = sum_i G   (tdp_linear_wgrad)
// for k <= 8 output classes and d <= 256 features.
//
// Reference: matmul and its VJP, tq/tensor.py:437-454, reached through
// Linear.__call__ (tq/models.py:26-27) inside a classifier TVF.  In the LLP
// query (SURVEY config 4) these two products read the [1e8, 64] feature matrix
// and dominate the step; a general GEMM library treats m = 1e8, n = 2 as a
// tall-skinny problem and runs it far below HBM bandwidth.  Both kernels here
// are pure streaming passes over X (4·d bytes per row), CUDA-core FMAs
// (the arithmetic intensity is ~k/2 flop/byte, far below the tensor-core
// ridge), float64 accumulation.
#include "tdp_common.cuh"

namespace tdp {
namespace {

constexpr int kMaxK = 8;
constexpr int kMaxD = 256;

// One thread per row; X row read with 16-byte vector loads (rows of one warp
// are 4·d bytes apart; the sectors a vector load leaves unused are consumed by
// the thread's next load from L1).  W lives in shared memory, read as
// broadcasts.
template <class T, int K>
__global__ void __launch_bounds__(256)
    linear_fwd_kernel(const T* __restrict__ X, i64 n, int d, const T* __restrict__ W,
                      const T* __restrict__ bias, T* __restrict__ Y) {
  __shared__ T sw[kMaxD * K];
  __shared__ T sb[K];
  for (int t = threadIdx.x; t < d * K; t += blockDim.x) sw[t] = W[t];
  if (threadIdx.x < K) sb[threadIdx.x] = bias ? bias[threadIdx.x] : T(0);
  __syncthreads();
  const bool vec = (sizeof(T) == 4) && (d % 4 == 0) && ((((uintptr_t)X) & 15) == 0);
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    double acc[K];
#pragma unroll
    for (int j = 0; j < K; ++j) acc[j] = 0.0;
    const T* row = X + i * d;
    if (vec) {
      const float4* r4 = reinterpret_cast<const float4*>(row);
      for (int c = 0; c < d / 4; ++c) {
        const float4 v = __ldg(r4 + c);
        const T* w = sw + (c * 4) * K;
#pragma unroll
        for (int j = 0; j < K; ++j) {
          acc[j] += (double)v.x * (double)w[j] + (double)v.y * (double)w[K + j] +
                    (double)v.z * (double)w[2 * K + j] + (double)v.w * (double)w[3 * K + j];
        }
      }
    } else {
      for (int c = 0; c < d; ++c) {
        const double v = (double)__ldg(row + c);
#pragma unroll
        for (int j = 0; j < K; ++j) acc[j] += v * (double)sw[c * K + j];
      }
    }
#pragma unroll
    for (int j = 0; j < K; ++j) Y[i * K + j] = (T)(acc[j] + (double)sb[j]);
  }
}

// Warp per row group: lane l owns features l, l+32, ...; each row's X is one
// coalesced warp load, its G row a broadcast.  Per-CTA partials in float64
// are written to `part` ([gridDim.x][d*K + K]) and reduced in a fixed order.
template <class T, int K>
__global__ void __launch_bounds__(256)
    linear_wgrad_kernel(const T* __restrict__ X, const T* __restrict__ G, i64 n, int d,
                        double* __restrict__ part) {
  constexpr int kF = kMaxD / 32;
  double acc[kF][K];
  double bacc[K];
#pragma unroll
  for (int f = 0; f < kF; ++f)
#pragma unroll
    for (int j = 0; j < K; ++j) acc[f][j] = 0.0;
#pragma unroll
  for (int j = 0; j < K; ++j) bacc[j] = 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 warps = (i64)gridDim.x * (blockDim.x >> 5);
  const int nf = (d + 31) / 32;
  for (i64 i = (i64)blockIdx.x * (blockDim.x >> 5) + warp; i < n; i += warps) {
    double g[K];
#pragma unroll
    for (int j = 0; j < K; ++j) g[j] = (double)__ldg(G + i * K + j);
#pragma unroll
    for (int f = 0; f < kF; ++f) {
      if (f < nf) {
        const int c = f * 32 + lane;
        const double x = c < d ? (double)__ldg(X + i * d + c) : 0.0;
#pragma unroll
        for (int j = 0; j < K; ++j) acc[f][j] += x * g[j];
      }
    }
#pragma unroll
    for (int j = 0; j < K; ++j) bacc[j] += g[j];
  }
  // one partial row per warp; reduced across rows in a fixed order afterwards
  const int W = d * K + K;
  double* out = part + ((i64)blockIdx.x * (blockDim.x >> 5) + warp) * W;
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

template <class T>
int launch_fwd(const T* X, i64 n, int d, int k, const T* W, const T* b, T* Y, cudaStream_t st) {
  const int grid = stream_grid(n, 256, 8);
  switch (k) {
#define TDP_CASE(KK)                                                                      \
  case KK:                                                                                \
    linear_fwd_kernel<T, KK><<<grid, 256, 0, st>>>(X, n, d, W, b, Y);                     \
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
  const int grid = stream_grid(n, 8 * 64, 2);
  const int width = d * k + k;
  const int rows = grid * 8;  // one partial row per warp
  TDP_REQUIRE(ws_bytes >= (size_t)rows * width * sizeof(double), "linear_wgrad workspace too small");
  switch (k) {
#define TDP_CASE(KK)                                                                      \
  case KK:                                                                                \
    linear_wgrad_kernel<T, KK><<<grid, 256, 0, st>>>(X, G, n, d, ws);                     \
    break;
    TDP_CASE(1) TDP_CASE(2) TDP_CASE(3) TDP_CASE(4) TDP_CASE(5) TDP_CASE(6) TDP_CASE(7) TDP_CASE(8)
#undef TDP_CASE
    default:
      return set_error(TDP_EINVAL, "linear: k=%d > %d", k, kMaxK);
  }
  TDP_LAUNCH_CHECK("linear_wgrad_kernel");
  wgrad_reduce_kernel<T><<<(unsigned)ceil_div((i64)width * 32, 256), 256, 0, st>>>(ws, rows, width,
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
  return (size_t)stream_grid(n, 8 * 64, 2) * 8 * (size_t)(d * k + k) * sizeof(double) + 256;
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
