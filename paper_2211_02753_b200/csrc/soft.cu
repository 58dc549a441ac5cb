// Probability encodings and the differentiable (soft) group-by.
//
// Reference (tq = /root/reference/pkg/src/tensorquery):
//   softmax fwd / VJP            tq/tensor.py:515-527 (via pe_encode, tq/encodings.py:143-151)
//   PE validation                tq/encodings.py:94-107
//   pe_decode argmax             tq/encodings.py:154-165
//   one_hot_pe range check       tq/encodings.py:175-183
//   soft_groupby forward         tq/kernels.py:190-229 (n x prod(k) joint, then reduce_sum)
//   soft_groupby backward        VJP chain reduce_sum (tq/tensor.py:474) -> mul (:364-365)
//                                -> reshape (:544)
//
// The reference materialises the n x prod(k) joint probability tensor.  Here
// the joint is never formed: one-hot keys are consumed as int64 codes (the
// compact form of one_hot_pe) and only the dense classes are enumerated per
// row; the grid is accumulated in float64.
#include <math.h>

#include <cstring>

#include "tdp_common.cuh"

namespace tdp {

namespace {

template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T t = __shfl_xor_sync(0xffffffffu, v, o);
    v = (t > v || t != t) ? t : v;
  }
  return v;
}

template <class T>
__global__ void softmax_rows_kernel(const T* __restrict__ x, i64 n, int k, T* __restrict__ y) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const T* row = x + i * k;
    T m = row[0];
    for (int c = 1; c < k; ++c) m = nan_max(m, row[c]);
    T s = 0;
    for (int c = 0; c < k; ++c) s += t_exp<T>(row[c] - m);
    T* out = y + i * k;
    for (int c = 0; c < k; ++c) out[c] = t_exp<T>(row[c] - m) / s;
  }
}

template <class T>
__global__ void softmax_warp_kernel(const T* __restrict__ x, i64 n, i64 k, T* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const i64 warps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 i = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const T* row = x + i * k;
    T m = row[0];
    for (i64 c = lane; c < k; c += 32) m = nan_max(m, row[c]);
    m = warp_max(m);
    T s = 0;
    for (i64 c = lane; c < k; c += 32) s += t_exp<T>(row[c] - m);
    s = warp_sum(s);
    T* out = y + i * k;
    for (i64 c = lane; c < k; c += 32) out[c] = t_exp<T>(row[c] - m) / s;
  }
}

template <class T>
__global__ void softmax_bwd_rows_kernel(const T* __restrict__ p, const T* __restrict__ g, i64 n,
                                        int k, T* __restrict__ dz) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    T inner = 0;
    for (int c = 0; c < k; ++c) inner += g[i * k + c] * p[i * k + c];
    for (int c = 0; c < k; ++c) dz[i * k + c] = p[i * k + c] * (g[i * k + c] - inner);
  }
}

template <class T>
__global__ void softmax_bwd_warp_kernel(const T* __restrict__ p, const T* __restrict__ g, i64 n,
                                        i64 k, T* __restrict__ dz) {
  const int lane = threadIdx.x & 31;
  const i64 warps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 i = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    T inner = 0;
    for (i64 c = lane; c < k; c += 32) inner += g[i * k + c] * p[i * k + c];
    inner = warp_sum(inner);
    for (i64 c = lane; c < k; c += 32) dz[i * k + c] = p[i * k + c] * (g[i * k + c] - inner);
  }
}

// flags: 1 entry outside [-tol, 1+tol] (non-NaN entries), 2 |rowsum-1| > tol
// (non-NaN sums), 4 a NaN entry exists, 8 a NaN row sum exists.
template <class T>
__global__ void pe_validate_kernel(const T* __restrict__ p, i64 n, i64 k, double tol,
                                   int* __restrict__ flags) {
  int f = 0;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    T s = 0;
    for (i64 c = 0; c < k; ++c) {
      const T v = p[i * k + c];
      if (v != v) f |= 4;
      else if ((double)v < -tol || (double)v > 1.0 + tol) f |= 1;
      s += v;
    }
    if (s != s) f |= 8;
    else if (fabs((double)s - 1.0) > tol) f |= 2;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

template <class T>
__device__ __forceinline__ bool arg_better(T v, i64 i, T bv, i64 bi) {
  const bool vn = v != v, bn = bv != bv;
  if (vn != bn) return vn;
  if (vn) return i < bi;
  if (v != bv) return v > bv;
  return i < bi;
}

template <class T>
__global__ void argmax_rows_kernel(const T* __restrict__ p, i64 n, i64 k, i64* __restrict__ out) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    T bv = p[i * k];
    i64 bi = 0;
    for (i64 c = 1; c < k; ++c) {
      const T v = p[i * k + c];
      if (arg_better(v, c, bv, bi)) {
        bv = v;
        bi = c;
      }
    }
    out[i] = bi;
  }
}

template <class T>
__global__ void argmax_warp_kernel(const T* __restrict__ p, i64 n, i64 k, i64* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const i64 warps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 i = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    T bv = p[i * k];
    i64 bi = 0;
    for (i64 c = lane; c < k; c += 32) {
      const T v = p[i * k + c];
      if (arg_better(v, c, bv, bi)) {
        bv = v;
        bi = c;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const T ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const i64 oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (arg_better(ov, oi, bv, bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) out[i] = bi;
  }
}

__global__ void codes_check_kernel(const i64* __restrict__ codes, i64 n, i64 k,
                                   int* __restrict__ flags) {
  int f = 0;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const i64 c = codes[i];
    if (c < 0 || c >= k) f = 1;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

// ---- soft group-by ---------------------------------------------------------
constexpr int kMaxSoftKeys = 8;

struct SoftKeys {
  int nkeys;
  int ndense;
  const void* p[kMaxSoftKeys];
  int kind[kMaxSoftKeys];
  int dt[kMaxSoftKeys];
  i64 k[kMaxSoftKeys];
  i64 stride[kMaxSoftKeys];  // row-major grid stride of each key
  i64 dense_total;           // product of dense k
};

__device__ __forceinline__ double prob_at(const SoftKeys& sk, int j, i64 i, i64 c) {
  if (sk.dt[j] == TDP_F64) return reinterpret_cast<const double*>(sk.p[j])[i * sk.k[j] + c];
  return (double)reinterpret_cast<const float*>(sk.p[j])[i * sk.k[j] + c];
}

__device__ __forceinline__ i64 onehot_base(const SoftKeys& sk, i64 i) {
  i64 base = 0;
  for (int j = 0; j < sk.nkeys; ++j)
    if (sk.kind[j] == TDP_SOFT_ONEHOT) base += reinterpret_cast<const i64*>(sk.p[j])[i] * sk.stride[j];
  return base;
}

// One thread per (row, dense class combination).
__global__ void soft_fwd_kernel(SoftKeys sk, i64 n, const void* __restrict__ values, int vdt,
                                double* __restrict__ grid) {
  const i64 D = sk.dense_total;
  const i64 total = n * D;
  for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (i64)gridDim.x * blockDim.x) {
    const i64 i = t / D;
    i64 rem = t - i * D;
    double prod = values ? load_as_f64(values, vdt, i) : 1.0;
    i64 cell = onehot_base(sk, i);
    for (int j = sk.nkeys - 1; j >= 0; --j) {
      if (sk.kind[j] != TDP_SOFT_DENSE) continue;
      const i64 c = rem % sk.k[j];
      rem /= sk.k[j];
      cell += c * sk.stride[j];
      prod *= prob_at(sk, j, i, c);
    }
    atomicAdd(grid + cell, prod);
  }
}

// Count grid privatised per CTA in shared memory as 64-bit fixed point
// (scale 2^30) split into two 32-bit words, updated with native ATOMS.ADD on
// the low word and a carry into the high word.  Joint probabilities lie in
// [0, 1]: the quantisation error is <= 2^-31 per row-cell (relative error of
// a cell count ~1e-12), and integer addition makes each CTA's partial exact
// and order-independent.  Values outside [0, 3] (NaN, negative PE noise, ...)
// go straight to the float64 grid so they propagate exactly as in the
// reference.  One float64 atomic per cell per CTA merges the partials.
constexpr double kFixScale = 1073741824.0;  // 2^30

__global__ void soft_fwd_count_smem_kernel(SoftKeys sk, i64 n, int cells, double* __restrict__ grid) {
  extern __shared__ unsigned fx[];  // lo[cells] then hi[cells]
  unsigned* lo = fx;
  unsigned* hi = fx + cells;
  for (int c = threadIdx.x; c < 2 * cells; c += blockDim.x) fx[c] = 0u;
  __syncthreads();
  const i64 D = sk.dense_total;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const i64 base = onehot_base(sk, i);
    for (i64 comb = 0; comb < D; ++comb) {
      i64 rem = comb, cell = base;
      double prod = 1.0;
      for (int j = sk.nkeys - 1; j >= 0; --j) {
        if (sk.kind[j] != TDP_SOFT_DENSE) continue;
        const i64 c = rem % sk.k[j];
        rem /= sk.k[j];
        cell += c * sk.stride[j];
        prod *= prob_at(sk, j, i, c);
      }
      if (prod >= 0.0 && prod <= 3.0) {
        const unsigned q = __double2uint_rn(prod * kFixScale);
        const unsigned old = atomicAdd(lo + cell, q);
        if (old > 0xffffffffu - q) atomicAdd(hi + cell, 1u);
      } else {
        atomicAdd(grid + cell, prod);
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < cells; c += blockDim.x) {
    const unsigned l = lo[c], h = hi[c];
    if (l | h) atomicAdd(grid + c, ((double)h * 4294967296.0 + (double)l) / kFixScale);
  }
}

// Single dense key: dP[i, c] = w_i * G[base_i + c * stride]   (thread per element)
template <class T>
__global__ void soft_bwd_single_kernel(SoftKeys sk, int j, i64 n, const void* __restrict__ values,
                                       int vdt, const double* __restrict__ G, T* __restrict__ dP) {
  const i64 k = sk.k[j];
  const i64 total = n * k;
  for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (i64)gridDim.x * blockDim.x) {
    const i64 i = t / k, c = t - i * k;
    double g = G[onehot_base(sk, i) + c * sk.stride[j]];
    if (values) g *= load_as_f64(values, vdt, i);
    dP[t] = (T)g;
  }
}

// General case: thread per row, enumerate the dense combinations.
__global__ void soft_bwd_general_kernel(SoftKeys sk, i64 n, const void* __restrict__ values,
                                        int vdt, const double* __restrict__ G, SoftKeys grads,
                                        void* __restrict__ dvalues, int dvdt) {
  const i64 D = sk.dense_total;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const double w = values ? load_as_f64(values, vdt, i) : 1.0;
    const i64 base = onehot_base(sk, i);
    // zero this row of every requested dense gradient
    for (int j = 0; j < sk.nkeys; ++j) {
      if (sk.kind[j] != TDP_SOFT_DENSE || grads.p[j] == nullptr) continue;
      for (i64 c = 0; c < sk.k[j]; ++c) {
        if (grads.dt[j] == TDP_F64) ((double*)grads.p[j])[i * sk.k[j] + c] = 0.0;
        else ((float*)grads.p[j])[i * sk.k[j] + c] = 0.0f;
      }
    }
    double dw = 0.0;
    for (i64 comb = 0; comb < D; ++comb) {
      i64 digit[kMaxSoftKeys];
      i64 rem = comb, cell = base;
      double full = 1.0;
      for (int j = sk.nkeys - 1; j >= 0; --j) {
        digit[j] = 0;
        if (sk.kind[j] != TDP_SOFT_DENSE) continue;
        digit[j] = rem % sk.k[j];
        rem /= sk.k[j];
        cell += digit[j] * sk.stride[j];
        full *= prob_at(sk, j, i, digit[j]);
      }
      const double g = G[cell];
      dw += g * full;
      for (int j = 0; j < sk.nkeys; ++j) {
        if (sk.kind[j] != TDP_SOFT_DENSE || grads.p[j] == nullptr) continue;
        double others = w * g;
        for (int l = 0; l < sk.nkeys; ++l)
          if (l != j && sk.kind[l] == TDP_SOFT_DENSE) others *= prob_at(sk, l, i, digit[l]);
        const i64 off = i * sk.k[j] + digit[j];
        if (grads.dt[j] == TDP_F64) ((double*)grads.p[j])[off] += others;
        else ((float*)grads.p[j])[off] = (float)((double)((float*)grads.p[j])[off] + others);
      }
    }
    if (dvalues) {
      if (dvdt == TDP_F64) ((double*)dvalues)[i] = dw;
      else ((float*)dvalues)[i] = (float)dw;
    }
  }
}

int make_softkeys(const tdp_soft_key* keys, int32_t nkeys, i64 n, SoftKeys* sk, i64* grid_cells) {
  TDP_REQUIRE(nkeys >= 1 && nkeys <= kMaxSoftKeys, "soft group-by needs 1..%d keys", kMaxSoftKeys);
  std::memset(sk, 0, sizeof(*sk));
  sk->nkeys = nkeys;
  sk->dense_total = 1;
  i64 prod = 1;
  for (int j = nkeys - 1; j >= 0; --j) {
    const tdp_soft_key& k = keys[j];
    TDP_REQUIRE(k.k >= 1, "key %d: k must be >= 1", j);
    TDP_REQUIRE(n == 0 || k.data != nullptr, "key %d: null data", j);
    TDP_REQUIRE(k.kind == TDP_SOFT_DENSE || k.kind == TDP_SOFT_ONEHOT, "key %d: bad kind", j);
    if (k.kind == TDP_SOFT_DENSE) {
      TDP_REQUIRE(k.dtype == TDP_F32 || k.dtype == TDP_F64, "key %d: PE must be float", j);
      sk->ndense++;
      sk->dense_total *= k.k;
    }
    sk->p[j] = k.data;
    sk->kind[j] = k.kind;
    sk->dt[j] = k.dtype;
    sk->k[j] = k.k;
    sk->stride[j] = prod;
    prod *= k.k;
    TDP_REQUIRE(prod <= ((i64)1 << 40), "soft group-by grid too large");
  }
  *grid_cells = prod;
  return TDP_OK;
}

}  // namespace

}  // namespace tdp

using namespace tdp;

#include <cstring>

extern "C" {

int tdp_softmax_fwd(const void* logits, int32_t dtype, int64_t n, int64_t k, void* probs,
                    void* stream) {
  TDP_REQUIRE(n >= 0 && k >= 1, "bad softmax shape");
  if (n == 0) return TDP_OK;
  cudaStream_t st = as_stream(stream);
  if (k <= 32) {
    const int grid = stream_grid(n, 256, 16);
    if (dtype == TDP_F32)
      softmax_rows_kernel<float><<<grid, 256, 0, st>>>((const float*)logits, n, (int)k, (float*)probs);
    else if (dtype == TDP_F64)
      softmax_rows_kernel<double><<<grid, 256, 0, st>>>((const double*)logits, n, (int)k, (double*)probs);
    else
      return set_error(TDP_EINVAL, "softmax requires float input");
  } else {
    const int grid = stream_grid(n, 8, 16);
    if (dtype == TDP_F32)
      softmax_warp_kernel<float><<<grid, 256, 0, st>>>((const float*)logits, n, k, (float*)probs);
    else if (dtype == TDP_F64)
      softmax_warp_kernel<double><<<grid, 256, 0, st>>>((const double*)logits, n, k, (double*)probs);
    else
      return set_error(TDP_EINVAL, "softmax requires float input");
  }
  TDP_LAUNCH_CHECK("softmax_fwd");
  return TDP_OK;
}

int tdp_softmax_bwd(const void* probs, const void* grad_probs, int32_t dtype, int64_t n,
                    int64_t k, void* grad_logits, void* stream) {
  TDP_REQUIRE(n >= 0 && k >= 1, "bad softmax shape");
  if (n == 0) return TDP_OK;
  cudaStream_t st = as_stream(stream);
  if (k <= 32) {
    const int grid = stream_grid(n, 256, 16);
    if (dtype == TDP_F32)
      softmax_bwd_rows_kernel<float><<<grid, 256, 0, st>>>((const float*)probs, (const float*)grad_probs,
                                                           n, (int)k, (float*)grad_logits);
    else if (dtype == TDP_F64)
      softmax_bwd_rows_kernel<double><<<grid, 256, 0, st>>>((const double*)probs,
                                                            (const double*)grad_probs, n, (int)k,
                                                            (double*)grad_logits);
    else
      return set_error(TDP_EINVAL, "softmax requires float input");
  } else {
    const int grid = stream_grid(n, 8, 16);
    if (dtype == TDP_F32)
      softmax_bwd_warp_kernel<float><<<grid, 256, 0, st>>>((const float*)probs, (const float*)grad_probs,
                                                           n, k, (float*)grad_logits);
    else if (dtype == TDP_F64)
      softmax_bwd_warp_kernel<double><<<grid, 256, 0, st>>>((const double*)probs,
                                                            (const double*)grad_probs, n, k,
                                                            (double*)grad_logits);
    else
      return set_error(TDP_EINVAL, "softmax requires float input");
  }
  TDP_LAUNCH_CHECK("softmax_bwd");
  return TDP_OK;
}

int tdp_pe_validate(const void* probs, int32_t dtype, int64_t n, int64_t k, double tol,
                    int32_t* out_flags, void* stream) {
  TDP_REQUIRE(n >= 0 && k >= 1, "bad PE shape");
  if (n == 0) return TDP_OK;
  cudaStream_t st = as_stream(stream);
  const int grid = stream_grid(n, 256, 16);
  if (dtype == TDP_F32)
    pe_validate_kernel<float><<<grid, 256, 0, st>>>((const float*)probs, n, k, tol, out_flags);
  else if (dtype == TDP_F64)
    pe_validate_kernel<double><<<grid, 256, 0, st>>>((const double*)probs, n, k, tol, out_flags);
  else
    return set_error(TDP_EINVAL, "PE must be float");
  TDP_LAUNCH_CHECK("pe_validate_kernel");
  return TDP_OK;
}

int tdp_pe_argmax(const void* probs, int32_t dtype, int64_t n, int64_t k, int64_t* out_codes,
                  void* stream) {
  TDP_REQUIRE(n >= 0 && k >= 1, "bad PE shape");
  if (n == 0) return TDP_OK;
  cudaStream_t st = as_stream(stream);
  if (k <= 32) {
    const int grid = stream_grid(n, 256, 16);
    if (dtype == TDP_F32)
      argmax_rows_kernel<float><<<grid, 256, 0, st>>>((const float*)probs, n, k, (i64*)out_codes);
    else if (dtype == TDP_F64)
      argmax_rows_kernel<double><<<grid, 256, 0, st>>>((const double*)probs, n, k, (i64*)out_codes);
    else
      return set_error(TDP_EINVAL, "PE must be float");
  } else {
    const int grid = stream_grid(n, 8, 16);
    if (dtype == TDP_F32)
      argmax_warp_kernel<float><<<grid, 256, 0, st>>>((const float*)probs, n, k, (i64*)out_codes);
    else if (dtype == TDP_F64)
      argmax_warp_kernel<double><<<grid, 256, 0, st>>>((const double*)probs, n, k, (i64*)out_codes);
    else
      return set_error(TDP_EINVAL, "PE must be float");
  }
  TDP_LAUNCH_CHECK("pe_argmax");
  return TDP_OK;
}

int tdp_codes_check(const int64_t* codes, int64_t n, int64_t k, int32_t* out_flags, void* stream) {
  TDP_REQUIRE(n >= 0, "bad code count");
  if (n == 0) return TDP_OK;
  codes_check_kernel<<<stream_grid(n, 256 * 8, 8), 256, 0, as_stream(stream)>>>((const i64*)codes,
                                                                                n, k, out_flags);
  TDP_LAUNCH_CHECK("codes_check_kernel");
  return TDP_OK;
}

int tdp_soft_groupby_fwd(const tdp_soft_key* keys, int32_t nkeys, int64_t n, const void* values,
                         int32_t values_dtype, double* out_grid, void* stream) {
  TDP_REQUIRE(n >= 0, "negative row count");
  SoftKeys sk;
  i64 cells = 0;
  int rc = make_softkeys(keys, nkeys, n, &sk, &cells);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  TDP_CUDA_TRY(cudaMemsetAsync(out_grid, 0, (size_t)cells * 8, st));
  if (n == 0) return TDP_OK;
  if (values == nullptr && cells <= 8192 && sk.dense_total <= 16) {
    const size_t smem = (size_t)cells * 2 * sizeof(unsigned);
    if (smem > 48 * 1024)
      TDP_CUDA_TRY(cudaFuncSetAttribute(soft_fwd_count_smem_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    soft_fwd_count_smem_kernel<<<stream_grid(n, 256 * 16, 4), 256, smem, st>>>(sk, n, (int)cells,
                                                                               out_grid);
    TDP_LAUNCH_CHECK("soft_fwd_count_smem_kernel");
    return TDP_OK;
  }
  soft_fwd_kernel<<<stream_grid(n * sk.dense_total, 256 * 4, 8), 256, 0, st>>>(
      sk, n, values, values_dtype, out_grid);
  TDP_LAUNCH_CHECK("soft_fwd_kernel");
  return TDP_OK;
}

int tdp_soft_groupby_bwd(const tdp_soft_key* keys, int32_t nkeys, int64_t n, const void* values,
                         int32_t values_dtype, const double* grad_grid, void* const* grad_keys,
                         void* grad_values, void* stream) {
  TDP_REQUIRE(n >= 0, "negative row count");
  SoftKeys sk;
  i64 cells = 0;
  int rc = make_softkeys(keys, nkeys, n, &sk, &cells);
  if (rc) return rc;
  if (n == 0) return TDP_OK;
  cudaStream_t st = as_stream(stream);
  SoftKeys gk;
  std::memset(&gk, 0, sizeof(gk));
  int nreq = 0, only = -1;
  for (int j = 0; j < nkeys; ++j) {
    gk.p[j] = (grad_keys && keys[j].kind == TDP_SOFT_DENSE) ? grad_keys[j] : nullptr;
    gk.dt[j] = keys[j].dtype;
    if (gk.p[j]) {
      ++nreq;
      only = j;
    }
  }
  if (sk.ndense == 1 && nreq == 1 && grad_values == nullptr) {
    const i64 total = n * sk.k[only];
    if (sk.dt[only] == TDP_F32)
      soft_bwd_single_kernel<float><<<stream_grid(total, 256 * 4, 8), 256, 0, st>>>(
          sk, only, n, values, values_dtype, grad_grid, (float*)gk.p[only]);
    else
      soft_bwd_single_kernel<double><<<stream_grid(total, 256 * 4, 8), 256, 0, st>>>(
          sk, only, n, values, values_dtype, grad_grid, (double*)gk.p[only]);
    TDP_LAUNCH_CHECK("soft_bwd_single_kernel");
    return TDP_OK;
  }
  if (nreq == 0 && grad_values == nullptr) return TDP_OK;
  soft_bwd_general_kernel<<<stream_grid(n, 256, 8), 256, 0, st>>>(
      sk, n, values, values_dtype, grad_grid, gk, grad_values, values_dtype);
  TDP_LAUNCH_CHECK("soft_bwd_general_kernel");
  return TDP_OK;
}

}  // extern "C"
