// Predicate filter, order-preserving stream compaction, row gather and the
// gather VJP (scatter-add).
//
// Reference chain replaced (tq = /root/reference/pkg/src/tensorquery):
//   comparison_mask        tq/kernels.py:54-84
//   mask &= ...; nonzero   tq/kernels.py:93-96
//   take_rows / gather     tq/kernels.py:44-51, tq/tensor.py:597-607
//   gather VJP (add.at)    tq/tensor.py:609-612
//
// Compaction is two streaming passes plus a tiny scan:
//   1. filter_bits: each CTA owns kFilterTile rows, evaluates the conjunction
//      for 32 consecutive rows per warp step (coalesced loads), stores one
//      ballot word per 32 rows and the tile's survivor count;
//   2. exclusive scan of tile counts -> tile output offsets;
//   3. write_indices: each warp expands its ballot words into ascending row
//      indices with coalesced stores.
// Only the predicate columns and 1 bit/row move in pass 1; pass 3 reads the
// bits and writes 8 bytes per surviving row.
#include "tdp_common.cuh"

namespace tdp {

namespace {

__global__ void __launch_bounds__(kFilterThreads)
    filter_bits_kernel(PredSet ps, i64 n, unsigned* __restrict__ bits,
                       i64* __restrict__ tile_counts) {
  __shared__ int warp_counts[kFilterThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 tile = blockIdx.x;
  const i64 tile_base = tile * kFilterTile;
  int count = 0;
  constexpr int kPer = kFilterWords / (kFilterThreads / 32);  // words per warp
  constexpr int kBatch = 8;
#pragma unroll
  for (int b = 0; b < kPer; b += kBatch) {
    i64 row[kBatch];
    bool keep[kBatch];
#pragma unroll
    for (int r = 0; r < kBatch; ++r) {
      const int w = warp + (b + r) * (kFilterThreads / 32);
      row[r] = tile_base + (i64)w * 32 + lane;
      keep[r] = row[r] < n;
    }
    eval_batch<kBatch>(ps, row, keep);
#pragma unroll
    for (int r = 0; r < kBatch; ++r) {
      const int w = warp + (b + r) * (kFilterThreads / 32);
      const unsigned word = __ballot_sync(0xffffffffu, keep[r]);
      if (lane == 0) {
        bits[tile * kFilterWords + w] = word;
        count += __popc(word);
      }
    }
  }
  if (lane == 0) warp_counts[warp] = count;
  __syncthreads();
  if (threadIdx.x == 0) {
    int total = 0;
#pragma unroll
    for (int k = 0; k < kFilterThreads / 32; ++k) total += warp_counts[k];
    tile_counts[tile] = total;
  }
}

__global__ void __launch_bounds__(kFilterThreads)
    write_indices_kernel(const unsigned* __restrict__ bits, const i64* __restrict__ tile_offsets,
                         i64 n, i64* __restrict__ out) {
  __shared__ int word_prefix[kFilterWords];
  __shared__ int warp_tot[kFilterWords / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 tile = blockIdx.x;
  // Scan of the tile's word popcounts (threads 0..kFilterWords-1 own one word).
  unsigned myword = 0;
  int pc = 0, incl = 0;
  if (threadIdx.x < kFilterWords) {
    myword = bits[tile * kFilterWords + threadIdx.x];
    pc = __popc(myword);
    incl = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
  }
  __syncthreads();
  if (threadIdx.x < kFilterWords) {
    int add = 0;
    for (int k = 0; k < warp; ++k) add += warp_tot[k];
    word_prefix[threadIdx.x] = add + incl - pc;
  }
  __syncthreads();
  const i64 base = tile_offsets[tile];
  const i64 tile_base = tile * kFilterTile;
  const unsigned lt = lanemask_lt();
  for (int w = warp; w < kFilterWords; w += kFilterThreads / 32) {
    const unsigned word = bits[tile * kFilterWords + w];
    if (word == 0) continue;
    if ((word >> lane) & 1u) {
      const i64 pos = base + word_prefix[w] + __popc(word & lt);
      out[pos] = tile_base + (i64)w * 32 + lane;
    }
  }
}

__global__ void filter_mask_kernel(PredSet ps, i64 n, unsigned char* __restrict__ out) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    out[i] = eval_all(ps, i) ? 1 : 0;
}

// ---- gather --------------------------------------------------------------
struct GatherCol {
  const unsigned char* src;
  unsigned char* dst;
  i64 row_bytes;
  i64 second;  // 1: rows from the second index vector (tdp_gather_rows2)
};
struct GatherSet {
  int ncols;
  int pad;
  GatherCol c[kMaxCols];
};

template <int B>
struct Chunk;
template <>
struct Chunk<8> {
  typedef unsigned long long T;
};
template <>
struct Chunk<4> {
  typedef unsigned T;
};
template <>
struct Chunk<2> {
  typedef unsigned short T;
};
template <>
struct Chunk<1> {
  typedef unsigned char T;
};

template <int B>
__device__ __forceinline__ void copy_elem(const GatherCol& c, i64 src_row, i64 j) {
  typedef typename Chunk<B>::T T;
  reinterpret_cast<T*>(c.dst)[j] = __ldg(reinterpret_cast<const T*>(c.src) + src_row);
}

// Narrow rows (<= 8 bytes): one thread per output row, all columns.
__global__ void gather_narrow_kernel(GatherSet gs, const i64* __restrict__ idx,
                                     const i64* __restrict__ idx2, i64 m) {
  for (i64 j = (i64)blockIdx.x * blockDim.x + threadIdx.x; j < m;
       j += (i64)gridDim.x * blockDim.x) {
    const i64 r1 = __ldg(idx + j);
    const i64 r2 = idx2 != nullptr ? __ldg(idx2 + j) : 0;
    for (int k = 0; k < gs.ncols; ++k) {
      const GatherCol& c = gs.c[k];
      const i64 r = c.second ? r2 : r1;
      switch (c.row_bytes) {
        case 8:
          copy_elem<8>(c, r, j);
          break;
        case 4:
          copy_elem<4>(c, r, j);
          break;
        case 2:
          copy_elem<2>(c, r, j);
          break;
        default:
          copy_elem<1>(c, r, j);
          break;
      }
    }
  }
}

// Wide rows: one warp per output row, lanes stride over 4-byte words.
__global__ void gather_wide_kernel(GatherCol c, const i64* __restrict__ idx, i64 m) {
  const int lane = threadIdx.x & 31;
  const i64 warps = (i64)gridDim.x * (blockDim.x >> 5);
  const i64 words = c.row_bytes / 4;
  for (i64 j = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < m; j += warps) {
    const i64 r = __ldg(idx + j);
    const unsigned* s = reinterpret_cast<const unsigned*>(c.src + r * c.row_bytes);
    unsigned* d = reinterpret_cast<unsigned*>(c.dst + j * c.row_bytes);
    for (i64 w = lane; w < words; w += 32) d[w] = __ldg(s + w);
  }
}

template <class T>
__global__ void scatter_add_kernel(const T* __restrict__ g, i64 width, const i64* __restrict__ idx,
                                   i64 m, T* __restrict__ out) {
  const i64 total = m * width;
  for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (i64)gridDim.x * blockDim.x) {
    const i64 j = t / width, e = t - j * width;
    atomicAdd(out + __ldg(idx + j) * width + e, g[t]);
  }
}

}  // namespace

int filter_bits(const PredSet& ps, int64_t n, unsigned* bits, i64* tile_counts,
                cudaStream_t stream) {
  const i64 tiles = ceil_div(n, kFilterTile);
  if (tiles == 0) return TDP_OK;
  filter_bits_kernel<<<(unsigned)tiles, kFilterThreads, 0, stream>>>(ps, n, bits, tile_counts);
  TDP_LAUNCH_CHECK("filter_bits_kernel");
  return TDP_OK;
}

}  // namespace tdp

using namespace tdp;

extern "C" {

int tdp_filter_mask(const tdp_column* cols, int32_t ncols, const tdp_predicate* preds,
                    int32_t npreds, int64_t n, uint8_t* out_mask, void* stream) {
  TDP_REQUIRE(n >= 0, "negative row count");
  if (n == 0) return TDP_OK;
  TDP_REQUIRE(out_mask != nullptr, "null output mask");
  PredSet ps;
  int rc = make_predset(cols, ncols, preds, npreds, n, &ps);
  if (rc) return rc;
  filter_mask_kernel<<<stream_grid(n, 256 * 8, 8), 256, 0, as_stream(stream)>>>(ps, n, out_mask);
  TDP_LAUNCH_CHECK("filter_mask_kernel");
  return TDP_OK;
}

size_t tdp_filter_workspace(int64_t n) {
  const i64 tiles = ceil_div(n > 0 ? n : 1, kFilterTile);
  return (size_t)tiles * kFilterWords * sizeof(unsigned) + 2 * (size_t)tiles * sizeof(i64) +
         exclusive_scan_workspace(tiles) + 512;
}

int tdp_filter_select(const tdp_column* cols, int32_t ncols, const tdp_predicate* preds,
                      int32_t npreds, int64_t n, int64_t* out_indices, int64_t* out_count,
                      void* ws, size_t ws_bytes, void* stream) {
  TDP_REQUIRE(n >= 0, "negative row count");
  TDP_REQUIRE(out_count != nullptr, "null count output");
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    TDP_CUDA_TRY(cudaMemsetAsync(out_count, 0, sizeof(i64), st));
    return TDP_OK;
  }
  TDP_REQUIRE(ws_bytes >= tdp_filter_workspace(n), "filter workspace too small");
  PredSet ps;
  int rc = make_predset(cols, ncols, preds, npreds, n, &ps);
  if (rc) return rc;
  const i64 tiles = ceil_div(n, kFilterTile);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  unsigned* bits = reinterpret_cast<unsigned*>(p);
  p += ((size_t)tiles * kFilterWords * sizeof(unsigned) + 255) & ~(size_t)255;
  i64* counts = reinterpret_cast<i64*>(p);
  i64* offsets = counts + tiles;
  void* scan_ws = offsets + tiles;
  size_t used = (size_t)((unsigned char*)scan_ws - (unsigned char*)ws);
  rc = filter_bits(ps, n, bits, counts, st);
  if (rc) return rc;
  rc = exclusive_scan_i64(counts, offsets, tiles, out_count, scan_ws, ws_bytes - used, st);
  if (rc) return rc;
  TDP_REQUIRE(out_indices != nullptr, "null index output");
  write_indices_kernel<<<(unsigned)tiles, kFilterThreads, 0, st>>>(bits, offsets, n, out_indices);
  TDP_LAUNCH_CHECK("write_indices_kernel");
  return TDP_OK;
}

}  // extern "C"

namespace tdp {
namespace {

// Columns [0, nfirst) gathered at idx, the rest at idx2 (null: idx for all).
int gather_rows_impl(const tdp_column* src, int32_t ncols, int32_t nfirst, const i64* idx,
                     const i64* idx2, i64 m, void* const* dst, cudaStream_t st) {
  TDP_REQUIRE(ncols >= 0 && ncols <= kMaxCols, "gather of %d columns (max %d)", ncols, kMaxCols);
  TDP_REQUIRE(m >= 0, "negative gather size");
  if (m == 0 || ncols == 0) return TDP_OK;
  TDP_REQUIRE(idx != nullptr && dst != nullptr, "null gather argument");
  GatherSet narrow;
  narrow.ncols = 0;
  narrow.pad = 0;
  for (int k = 0; k < ncols; ++k) {
    const int es = dtype_size(src[k].dtype);
    TDP_REQUIRE(es > 0, "gather column %d: bad dtype", k);
    TDP_REQUIRE(src[k].width >= 1, "gather column %d: bad width", k);
    GatherCol c;
    c.src = reinterpret_cast<const unsigned char*>(src[k].data);
    c.dst = reinterpret_cast<unsigned char*>(dst[k]);
    c.row_bytes = (i64)es * src[k].width;
    c.second = k >= nfirst ? 1 : 0;
    if (c.row_bytes == 8 || c.row_bytes == 4 || c.row_bytes == 2 || c.row_bytes == 1) {
      narrow.c[narrow.ncols++] = c;
    } else {
      TDP_REQUIRE(c.row_bytes % 4 == 0, "gather column %d: row of %lld bytes", k,
                  (long long)c.row_bytes);
      gather_wide_kernel<<<stream_grid(m, 8, 16), 256, 0, st>>>(c, c.second ? idx2 : idx, m);
      TDP_LAUNCH_CHECK("gather_wide_kernel");
    }
  }
  if (narrow.ncols) {
    gather_narrow_kernel<<<stream_grid(m, 256 * 4, 8), 256, 0, st>>>(
        narrow, idx, nfirst < ncols ? idx2 : nullptr, m);
    TDP_LAUNCH_CHECK("gather_narrow_kernel");
  }
  return TDP_OK;
}

}  // namespace
}  // namespace tdp

extern "C" {

int tdp_gather_rows(const tdp_column* src, int32_t ncols, const int64_t* indices, int64_t m,
                    void* const* dst, void* stream) {
  return gather_rows_impl(src, ncols, ncols, indices, nullptr, m, dst, as_stream(stream));
}

int tdp_gather_rows2(const tdp_column* src, int32_t ncols, int32_t nfirst, const int64_t* indices,
                     const int64_t* indices2, int64_t m, void* const* dst, void* stream) {
  TDP_REQUIRE(nfirst >= 0 && nfirst <= ncols, "bad first-column count");
  TDP_REQUIRE(nfirst == ncols || indices2 != nullptr, "null second index vector");
  return gather_rows_impl(src, ncols, nfirst, indices, indices2, m, dst, as_stream(stream));
}

int tdp_scatter_add_rows(const void* grad_out, int32_t dtype, int64_t width,
                         const int64_t* indices, int64_t m, void* grad_in, void* stream) {
  TDP_REQUIRE(m >= 0 && width >= 1, "bad scatter shape");
  if (m == 0) return TDP_OK;
  cudaStream_t st = as_stream(stream);
  const int grid = stream_grid(m * width, 256 * 4, 8);
  if (dtype == TDP_F64) {
    scatter_add_kernel<double><<<grid, 256, 0, st>>>(reinterpret_cast<const double*>(grad_out),
                                                     width, indices, m,
                                                     reinterpret_cast<double*>(grad_in));
  } else if (dtype == TDP_F32) {
    scatter_add_kernel<float><<<grid, 256, 0, st>>>(reinterpret_cast<const float*>(grad_out),
                                                    width, indices, m,
                                                    reinterpret_cast<float*>(grad_in));
  } else {
    return set_error(TDP_EINVAL, "scatter_add needs float32/float64 (got dtype %d)", dtype);
  }
  TDP_LAUNCH_CHECK("scatter_add_kernel");
  return TDP_OK;
}

}  // extern "C"
