// Differentiable ORDER BY ... [LIMIT k] for trainable queries (SURVEY §8(f)
// rank 4).  The reference rejects Sort / Limit when trainable
// (tq/compiler.py:464-475; learning-to-rank is the paper's stated future
// work), so this is new, opt-in semantics
// (CompileConfig.soft_sort_tau): the NeuralSort relaxation of the sorting
// permutation (Grover et al., ICLR 2019).  For scores s (n rows; descending
// order -- ascending sorts -s) and temperature tau, output rank r of a top-k
// (r < k <= n) is the row-stochastic mixture
//   P[r, i] = softmax_i( ((n + 1 - 2 (r + 1)) s_i - B_i) / tau ),
//   B_i = sum_j |s_i - s_j|,
// which tends to the hard descending permutation as tau -> 0.
//
// Backward (dP given): dlogit = P * (dP - rowsum(P dP)) per row, and
//   ds_m = ( sum_r dlogit[r, m] c_r - sum_j (u_j + u_m) sign(s_m - s_j) ) / tau
// with c_r = n + 1 - 2 (r + 1), u_i = sum_r dlogit[r, i].
// The O(n^2) pair sums (B and the sign term) are tiled through shared
// memory; all arithmetic in float64.
#include "tdp_common.cuh"

namespace tdp {
namespace {

constexpr int kSsThreads = 256;

// B_i = sum_j |s_i - s_j|
__global__ void softsort_abs_sum_kernel(const double* __restrict__ s, i64 n,
                                        double* __restrict__ B) {
  __shared__ double tile[kSsThreads];
  const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  const double si = i < n ? s[i] : 0.0;
  double acc = 0.0;
  for (i64 t0 = 0; t0 < n; t0 += kSsThreads) {
    const i64 j = t0 + threadIdx.x;
    tile[threadIdx.x] = j < n ? s[j] : 0.0;
    __syncthreads();
    const int m = (int)(n - t0 < kSsThreads ? n - t0 : kSsThreads);
    for (int q = 0; q < m; ++q) acc += fabs(si - tile[q]);
    __syncthreads();
  }
  if (i < n) B[i] = acc;
}

// one CTA per output rank r: P[r, :] = softmax of the row's logits
__global__ void softsort_rows_kernel(const double* __restrict__ s, const double* __restrict__ B,
                                     i64 n, double inv_tau, double* __restrict__ P) {
  __shared__ double red[kSsThreads / 32];
  __shared__ double bc;
  const int r = blockIdx.x;
  const double c = (double)(n + 1 - 2 * (r + 1));
  double mx = -INFINITY;
  for (i64 i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, (c * s[i] - B[i]) * inv_tau);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = red[0];
    for (int w = 1; w < kSsThreads / 32; ++w) m = fmax(m, red[w]);
    bc = m;
  }
  __syncthreads();
  const double m = bc;
  double sum = 0.0;
  double* row = P + (i64)r * n;
  for (i64 i = threadIdx.x; i < n; i += blockDim.x) {
    const double e = exp((c * s[i] - B[i]) * inv_tau - m);
    row[i] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kSsThreads / 32; ++w) t += red[w];
    bc = t;
  }
  __syncthreads();
  const double inv = 1.0 / bc;
  for (i64 i = threadIdx.x; i < n; i += blockDim.x) row[i] *= inv;
}

// dlogit[r, :] = P * (dP - <P, dP>) in place of dP (one CTA per row)
__global__ void softsort_dlogit_kernel(const double* __restrict__ P, double* __restrict__ dP,
                                       i64 n) {
  __shared__ double red[kSsThreads / 32];
  __shared__ double bc;
  const int r = blockIdx.x;
  const double* p = P + (i64)r * n;
  double* g = dP + (i64)r * n;
  double dot = 0.0;
  for (i64 i = threadIdx.x; i < n; i += blockDim.x) dot += p[i] * g[i];
  dot = warp_sum(dot);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dot;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kSsThreads / 32; ++w) t += red[w];
    bc = t;
  }
  __syncthreads();
  const double inner = bc;
  for (i64 i = threadIdx.x; i < n; i += blockDim.x) g[i] = p[i] * (g[i] - inner);
}

// u_i = sum_r dlogit[r, i],  v_i = sum_r dlogit[r, i] c_r  (rows in order)
__global__ void softsort_colsum_kernel(const double* __restrict__ dl, i64 n, int k,
                                       double* __restrict__ u, double* __restrict__ v) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    double a = 0.0, b = 0.0;
    for (int r = 0; r < k; ++r) {
      const double x = dl[(i64)r * n + i];
      a += x;
      b += x * (double)(n + 1 - 2 * (r + 1));
    }
    u[i] = a;
    v[i] = b;
  }
}

// ds_m = (v_m - sum_j (u_j + u_m) sign(s_m - s_j)) / tau
__global__ void softsort_ds_kernel(const double* __restrict__ s, const double* __restrict__ u,
                                   const double* __restrict__ v, i64 n, double inv_tau,
                                   double* __restrict__ ds) {
  __shared__ double ts[kSsThreads], tu[kSsThreads];
  const i64 m = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  const double sm = m < n ? s[m] : 0.0, um = m < n ? u[m] : 0.0;
  double acc = 0.0;
  for (i64 t0 = 0; t0 < n; t0 += kSsThreads) {
    const i64 j = t0 + threadIdx.x;
    ts[threadIdx.x] = j < n ? s[j] : 0.0;
    tu[threadIdx.x] = j < n ? u[j] : 0.0;
    __syncthreads();
    const int cnt = (int)(n - t0 < kSsThreads ? n - t0 : kSsThreads);
    for (int q = 0; q < cnt; ++q) {
      const double d = sm - ts[q];
      const double sg = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0);
      acc += (tu[q] + um) * sg;
    }
    __syncthreads();
  }
  if (m < n) ds[m] = (v[m] - acc) * inv_tau;
}

}  // namespace
}  // namespace tdp

using namespace tdp;

extern "C" {

int tdp_softsort_fwd(const double* s, int64_t n, int32_t k, double tau, double* out_P,
                     double* ws, void* stream) {
  TDP_REQUIRE(n >= 1 && k >= 1 && k <= n && tau > 0.0, "softsort: need 1 <= k <= n, tau > 0");
  TDP_REQUIRE(n <= (1 << 20), "softsort: at most 2^20 rows (pairwise terms)");
  cudaStream_t st = as_stream(stream);
  double* B = ws;  // [n]
  softsort_abs_sum_kernel<<<(unsigned)ceil_div(n, kSsThreads), kSsThreads, 0, st>>>(s, n, B);
  TDP_LAUNCH_CHECK("softsort_abs_sum_kernel");
  softsort_rows_kernel<<<(unsigned)k, kSsThreads, 0, st>>>(s, B, n, 1.0 / tau, out_P);
  TDP_LAUNCH_CHECK("softsort_rows_kernel");
  return TDP_OK;
}

int tdp_softsort_bwd(const double* s, int64_t n, int32_t k, double tau, const double* P,
                     double* dP_inout, double* out_ds, double* ws, void* stream) {
  TDP_REQUIRE(n >= 1 && k >= 1 && k <= n && tau > 0.0, "softsort: need 1 <= k <= n, tau > 0");
  cudaStream_t st = as_stream(stream);
  double* u = ws;      // [n]
  double* v = ws + n;  // [n]
  softsort_dlogit_kernel<<<(unsigned)k, kSsThreads, 0, st>>>(P, dP_inout, n);
  TDP_LAUNCH_CHECK("softsort_dlogit_kernel");
  softsort_colsum_kernel<<<stream_grid(n, 256, 8), 256, 0, st>>>(dP_inout, n, k, u, v);
  TDP_LAUNCH_CHECK("softsort_colsum_kernel");
  softsort_ds_kernel<<<(unsigned)ceil_div(n, kSsThreads), kSsThreads, 0, st>>>(s, u, v, n,
                                                                              1.0 / tau, out_ds);
  TDP_LAUNCH_CHECK("softsort_ds_kernel");
  return TDP_OK;
}

}  // extern "C"
