// Stable LSD radix sort of 64-bit keys with int64 payload, and the sort-based
// relational primitives built on it.
//
// Reference primitives replaced (tq = /root/reference/pkg/src/tensorquery):
//   np.argsort(+-key, kind="stable")   stable_order, tq/kernels.py:256-264
//   np.unique(key, return_inverse)     groupby_exact, tq/kernels.py:128, :136
//   np.bincount / np.add.at            groupby_exact, tq/kernels.py:138-153
//
// Keys are mapped to unsigned 64-bit images whose unsigned order is numpy's
// order: int64 -> flip the sign bit; float -> IEEE total-order flip with
// -0.0 canonicalised to +0.0 (numpy treats them as equal, so the stable sort
// keeps input order) and every NaN mapped to the all-ones image (NaN sorts last
// in both directions, ties among NaNs keep input order).  DESC sorts the
// negated key exactly like the reference (`-arr`, INT64_MIN wraps).
//
// One pass per 8-bit digit: per-tile digit histograms -> device-wide scan of
// the digit-major [256 x tiles] count matrix -> stable scatter, where each
// warp ranks its keys in input order with __match_any_sync and the CTA adds
// per-warp prefixes.  Digits that are constant across all keys (found with a
// single histogram pre-pass over all 8 digits) are skipped, so int64 keys of
// small range sort in 3-4 passes.
#include <vector>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "tdp_common.cuh"
#include "fixed_acc.cuh"

namespace tdp {

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;  // per thread
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr int kWarpKeys = 32 * kSortItems;
constexpr int kWarps = kSortThreads / 32;

__device__ __forceinline__ u64 image_i64(i64 x, bool desc) {
  const u64 v = desc ? (u64)0 - (u64)x : (u64)x;
  return v ^ 0x8000000000000000ull;
}

__device__ __forceinline__ u64 image_f64(double x, bool desc) {
  if (x != x) return ~0ull;
  if (desc) x = -x;
  if (x == 0.0) x = 0.0;  // -0.0 -> +0.0
  const u64 b = (u64)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ u64 image_f32(float x, bool desc) {
  if (x != x) return 0xffffffffull;
  if (desc) x = -x;
  if (x == 0.0f) x = 0.0f;
  const unsigned b = __float_as_uint(x);
  return (u64)((b & 0x80000000u) ? ~b : (b | 0x80000000u));
}

__global__ void make_keys_kernel(const void* __restrict__ key, int dtype, int desc, i64 n,
                                 u64* __restrict__ out, i64* __restrict__ idx) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    u64 k;
    switch (dtype) {
      case TDP_I64:
        k = image_i64(reinterpret_cast<const i64*>(key)[i], desc);
        break;
      case TDP_I32:
        k = image_i64((i64)reinterpret_cast<const int*>(key)[i], desc);
        break;
      case TDP_F64:
        k = image_f64(reinterpret_cast<const double*>(key)[i], desc);
        break;
      default:
        k = image_f32(reinterpret_cast<const float*>(key)[i], desc);
        break;
    }
    out[i] = k;
    idx[i] = i;
  }
}

// Histograms of all 8 digits at once -> hist[8][256] (global, zeroed).
__global__ void all_digit_hist_kernel(const u64* __restrict__ keys, i64 n,
                                      unsigned long long* __restrict__ hist) {
  __shared__ unsigned h[8][256];
  for (int t = threadIdx.x; t < 8 * 256; t += blockDim.x) (&h[0][0])[t] = 0;
  __syncthreads();
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const u64 k = keys[i];
#pragma unroll
    for (int d = 0; d < 8; ++d) atomicAdd(&h[d][(k >> (8 * d)) & 0xff], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 8 * 256; t += blockDim.x) {
    const unsigned v = (&h[0][0])[t];
    if (v) atomicAdd(hist + t, (unsigned long long)v);
  }
}

__global__ void __launch_bounds__(kSortThreads)
    tile_hist_kernel(const u64* __restrict__ keys, i64 n, int shift, i64 ntiles,
                     i64* __restrict__ counts) {
  __shared__ unsigned h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const i64 base = (i64)blockIdx.x * kSortTile;
#pragma unroll 4
  for (int k = 0; k < kSortItems; ++k) {
    const i64 i = base + (i64)k * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 0xff], 1u);
  }
  __syncthreads();
  counts[(i64)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads)
    scatter_kernel(const u64* __restrict__ keys_in, const i64* __restrict__ idx_in, i64 n,
                   int shift, i64 ntiles, const i64* __restrict__ offsets,
                   u64* __restrict__ keys_out, i64* __restrict__ idx_out) {
  __shared__ unsigned wcount[kWarps][256];
  __shared__ i64 goff[256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = lane; d < 256; d += 32) wcount[warp][d] = 0;
  goff[threadIdx.x] = offsets[(i64)threadIdx.x * ntiles + blockIdx.x];
  __syncwarp();
  const i64 wbase = (i64)blockIdx.x * kSortTile + (i64)warp * kWarpKeys;
  const unsigned lt = lanemask_lt();
  u64 k[kSortItems];
  i64 p[kSortItems];
  unsigned rank[kSortItems];
  int dig[kSortItems];
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const i64 i = wbase + it * 32 + lane;
    const bool valid = i < n;
    k[it] = valid ? keys_in[i] : 0;
    p[it] = valid ? idx_in[i] : 0;
    dig[it] = valid ? (int)((k[it] >> shift) & 0xff) : 256;
  }
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const int d = dig[it];
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    unsigned before = 0;
    if (d < 256) before = wcount[warp][d];
    rank[it] = before + __popc(peers & lt);
    __syncwarp();
    if (d < 256 && (peers & lt) == 0) wcount[warp][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // exclusive prefix over warps for each digit (thread t owns digit t)
  {
    unsigned run = 0;
    const int d = threadIdx.x;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const unsigned c = wcount[w][d];
      wcount[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const int d = dig[it];
    if (d < 256) {
      const i64 pos = goff[d] + wcount[warp][d] + rank[it];
      keys_out[pos] = k[it];
      idx_out[pos] = p[it];
    }
  }
}

struct SortBuffers {
  u64* k0;
  u64* k1;
  i64* i0;
  i64* i1;
  i64* counts;
  i64* offsets;
  unsigned long long* hist;
  void* scan_ws;
  size_t scan_bytes;
};

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// Scans run over the [256 x tiles] digit counts and (unique) over n flags.
i64 scan_extent(i64 n) {
  const i64 ntiles = ceil_div(n > 0 ? n : 1, kSortTile);
  return ntiles * 256 > n ? ntiles * 256 : n;
}

size_t sort_ws_bytes(i64 n) {
  const i64 ntiles = ceil_div(n > 0 ? n : 1, kSortTile);
  return align256(4 * align256((size_t)n * 8) + 2 * align256((size_t)ntiles * 256 * 8) +
                  align256(8 * 256 * 8) + exclusive_scan_workspace(scan_extent(n)) + 1024);
}

SortBuffers carve(void* ws, i64 n) {
  const i64 ntiles = ceil_div(n > 0 ? n : 1, kSortTile);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  SortBuffers b;
  b.k0 = (u64*)p;
  p += align256((size_t)n * 8);
  b.k1 = (u64*)p;
  p += align256((size_t)n * 8);
  b.i0 = (i64*)p;
  p += align256((size_t)n * 8);
  b.i1 = (i64*)p;
  p += align256((size_t)n * 8);
  b.counts = (i64*)p;
  p += align256((size_t)ntiles * 256 * 8);
  b.offsets = (i64*)p;
  p += align256((size_t)ntiles * 256 * 8);
  b.hist = (unsigned long long*)p;
  p += align256(8 * 256 * 8);
  b.scan_ws = p;
  b.scan_bytes = exclusive_scan_workspace(scan_extent(n)) + 512;
  return b;
}

// A replayed sort skips the digit passes its recording run skipped: each of
// them must still be constant (one bin holds all n keys), else trap.
__global__ void sort_passes_check_kernel(const unsigned long long* __restrict__ hist, i64 n,
                                         unsigned passes) {
  __shared__ int constant[8];
  if (threadIdx.x < 8) constant[threadIdx.x] = 0;
  __syncthreads();
  for (int d = 0; d < 8; ++d)
    if (hist[d * 256 + threadIdx.x] == (unsigned long long)n) constant[d] = 1;
  __syncthreads();
  if (threadIdx.x < 8 && !((passes >> threadIdx.x) & 1u) && !constant[threadIdx.x]) {
    printf("tdp: replayed radix sort skips digit %d, which is no longer constant\n",
           (int)threadIdx.x);
    __trap();
  }
}

// Sorts the images in b.k0 / payload b.i0.  On return *keys/*idx point at the
// buffer holding the sorted result.
int radix_sort(SortBuffers& b, i64 n, cudaStream_t st, u64** keys, i64** idx) {
  *keys = b.k0;
  *idx = b.i0;
  if (n <= 1) return TDP_OK;
  const i64 ntiles = ceil_div(n, kSortTile);
  TDP_CUDA_TRY(cudaMemsetAsync(b.hist, 0, 8 * 256 * 8, st));
  all_digit_hist_kernel<<<stream_grid(n, 256 * 16, 4), 256, 0, st>>>(b.k0, n, b.hist);
  TDP_LAUNCH_CHECK("all_digit_hist_kernel");
  // bit d set: digit d is not constant, pass d runs
  unsigned passes = 0;
  if (replay_mode() == 2) {  // graph capture: the recorded decision, checked on the device
    i64 v;
    TDP_REQUIRE(replay_take(&v), "radix sort: replay log exhausted");
    passes = (unsigned)v;
    sort_passes_check_kernel<<<1, 256, 0, st>>>(b.hist, n, passes);
    TDP_LAUNCH_CHECK("sort_passes_check_kernel");
  } else {
    std::vector<unsigned long long> h(8 * 256);
    TDP_CUDA_TRY(cudaMemcpyAsync(h.data(), b.hist, h.size() * 8, cudaMemcpyDeviceToHost, st));
    TDP_CUDA_TRY(cudaStreamSynchronize(st));
    for (int d = 0; d < 8; ++d) {
      bool trivial = false;
      for (int v = 0; v < 256; ++v)
        if (h[d * 256 + v] == (unsigned long long)n) trivial = true;
      if (!trivial) passes |= 1u << d;
    }
    if (replay_mode() == 1) replay_push((i64)passes);
  }
  u64* kin = b.k0;
  u64* kout = b.k1;
  i64* iin = b.i0;
  i64* iout = b.i1;
  for (int d = 0; d < 8; ++d) {
    if (!((passes >> d) & 1u)) continue;
    const int shift = 8 * d;
    tile_hist_kernel<<<(unsigned)ntiles, kSortThreads, 0, st>>>(kin, n, shift, ntiles, b.counts);
    TDP_LAUNCH_CHECK("tile_hist_kernel");
    int rc = exclusive_scan_i64(b.counts, b.offsets, ntiles * 256, nullptr, b.scan_ws,
                                b.scan_bytes, st);
    if (rc) return rc;
    scatter_kernel<<<(unsigned)ntiles, kSortThreads, 0, st>>>(kin, iin, n, shift, ntiles,
                                                              b.offsets, kout, iout);
    TDP_LAUNCH_CHECK("scatter_kernel");
    u64* tk = kin;
    kin = kout;
    kout = tk;
    i64* ti = iin;
    iin = iout;
    iout = ti;
  }
  *keys = kin;
  *idx = iin;
  return TDP_OK;
}

// ---- unique / inverse ----------------------------------------------------
__global__ void boundary_flags_kernel(const u64* __restrict__ sk, i64 n, i64* __restrict__ flags) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || sk[i] != sk[i - 1]) ? 1 : 0;
}

// rank of sorted position i = (#boundaries at or before i) - 1 = excl[i] + flag[i] - 1
__global__ void unique_scatter_kernel(const u64* __restrict__ sk, const i64* __restrict__ order,
                                      const i64* __restrict__ flags, const i64* __restrict__ excl,
                                      i64 n, i64* __restrict__ uniques, i64* __restrict__ inverse) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const i64 r = excl[i] + flags[i] - 1;
    inverse[order[i]] = r;
    if (flags[i]) uniques[r] = (i64)(sk[i] ^ 0x8000000000000000ull);
  }
}

// ---- grouped aggregation over dense codes ----------------------------------
struct ValSet {
  int naggs;
  int nfixed;     // float SUM aggregates: fixed-point cells (fixed_acc.cuh)
  const void* p[32];
  int dt[32];
  int kind[32];
  int fidx[32];   // aggregate -> fixed-point cell block (float SUMs), else -1
  unsigned avg;   // emit: aggregates written as double(sum) / double(count)
};

// Emit kinds: TDP_AGG_AVG_BIT moved into vs->avg, the kinds themselves plain.
inline int emit_kinds(const int32_t* agg_kinds, int32_t naggs, ValSet* vs) {
  TDP_REQUIRE(naggs >= 0 && naggs <= 32, "at most 32 aggregates");
  std::memset(vs, 0, sizeof(*vs));
  vs->naggs = naggs;
  for (int a = 0; a < naggs; ++a) {
    const int k = agg_kinds[a] & ~TDP_AGG_AVG_BIT;
    TDP_REQUIRE(k >= TDP_AGG_COUNT && k <= TDP_AGG_SUM_I64, "agg %d: bad kind", a);
    TDP_REQUIRE(!(agg_kinds[a] & TDP_AGG_AVG_BIT) || k != TDP_AGG_COUNT,
                "agg %d: AVG of a count", a);
    vs->kind[a] = k;
    if (agg_kinds[a] & TDP_AGG_AVG_BIT) vs->avg |= 1u << a;
  }
  return TDP_OK;
}

// One emitted aggregate value (8 bytes): the mean when the AVG bit is set.
__device__ __forceinline__ u64 emit_value(const ValSet& vs, int a, u64 raw, u64 cnt) {
  if (!((vs.avg >> a) & 1u)) return raw;
  const double s = vs.kind[a] == TDP_AGG_SUM_F64 ? __longlong_as_double((i64)raw) : (double)(i64)raw;
  return (u64)__double_as_longlong(s / (double)cnt);
}

inline void number_fixed(ValSet* vs) {
  vs->nfixed = 0;
  for (int a = 0; a < vs->naggs; ++a)
    vs->fidx[a] = vs->kind[a] == TDP_AGG_SUM_F64 ? vs->nfixed++ : -1;
}

// fixed-point cells -> the double bits of the float sums: sums[a][slot]
// (stride `sstride` per aggregate), cells [fidx][slot][kFixedWords]
__global__ void fixed_finalize_kernel(const unsigned long long* __restrict__ fx, i64 slots,
                                      ValSet vs, unsigned long long* __restrict__ sums,
                                      i64 sstride) {
  for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < slots * vs.naggs;
       t += (i64)gridDim.x * blockDim.x) {
    const int a = (int)(t / slots);
    const i64 s = t - (i64)a * slots;
    if (vs.fidx[a] < 0) continue;
    const double v = fixed_value(fx + ((i64)vs.fidx[a] * slots + s) * kFixedWords);
    sums[(i64)a * sstride + s] = (unsigned long long)__double_as_longlong(v);
  }
}

__global__ void groupby_codes_kernel(const i64* __restrict__ codes, i64 n, i64 slots, ValSet vs,
                                     unsigned long long* __restrict__ counts,
                                     unsigned long long* __restrict__ sums,
                                     unsigned long long* __restrict__ fx) {
  const int lane = threadIdx.x & 31;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 base = (i64)blockIdx.x * blockDim.x; base < n; base += stride) {
    const i64 i = base + threadIdx.x;
    const bool valid = i < n;
    const i64 c = valid ? codes[i] : -1;
    const i64 c0 = __shfl_sync(0xffffffffu, c, 0);
    const bool uniform = __all_sync(0xffffffffu, c == c0) && c0 >= 0;
    if (uniform) {
      // whole warp in one group (typical after sorting / small key spaces)
      const unsigned long long cnt = warp_sum(1ull);
      if (lane == 0) atomicAdd(counts + c0, cnt);
      for (int a = 0; a < vs.naggs; ++a) {
        if (vs.kind[a] == TDP_AGG_COUNT) continue;
        if (vs.kind[a] == TDP_AGG_SUM_F64) {
          // fixed lane order -> the same warp sum every run; integer cells
          const double v = warp_sum(load_as_f64(vs.p[a], vs.dt[a], i));
          if (lane == 0) fixed_add(fx + ((i64)vs.fidx[a] * slots + c0) * kFixedWords, v);
        } else {
          const unsigned long long v = warp_sum((unsigned long long)load_as_i64(vs.p[a], vs.dt[a], i));
          if (lane == 0) atomicAdd(sums + (i64)a * slots + c0, v);
        }
      }
    } else if (valid) {
      atomicAdd(counts + c, 1ull);
      for (int a = 0; a < vs.naggs; ++a) {
        if (vs.kind[a] == TDP_AGG_COUNT) continue;
        if (vs.kind[a] == TDP_AGG_SUM_F64)
          fixed_add(fx + ((i64)vs.fidx[a] * slots + c) * kFixedWords,
                    load_as_f64(vs.p[a], vs.dt[a], i));
        else
          atomicAdd(sums + (i64)a * slots + c,
                    (unsigned long long)load_as_i64(vs.p[a], vs.dt[a], i));
      }
    }
  }
}

__global__ void copy_counts_kernel(const unsigned long long* __restrict__ counts, i64 slots,
                                   ValSet vs, unsigned long long* __restrict__ sums) {
  for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < slots * vs.naggs;
       t += (i64)gridDim.x * blockDim.x) {
    const int a = (int)(t / slots);
    if (vs.kind[a] == TDP_AGG_COUNT) sums[t] = counts[t - (i64)a * slots];
  }
}

}  // namespace


// ---------------------------------------------------------------------------
// top-k of a stable order (ORDER BY ... LIMIT k, tq/kernels.py:267-273): the k
// smallest (key image, row) pairs.  Each CTA bitonic-sorts a chunk of
// `chunk` pairs (a power of two <= kTopkChunk) in shared memory and keeps its
// first k; the survivors are reduced the same way until one CTA remains.
// Chunks are sized per round: the smallest power of two >= 2k that still
// gives at most two CTAs per SM, so a round is a short sort on many SMs
// rather than a 2048-wide one on few.  Ties keep row order because the row
// index is the second sort key, exactly as the stable radix sort orders.
// ---------------------------------------------------------------------------
constexpr int kTopkChunk = 2048;
constexpr int kTopkMax = 1024;

// Key images of the first round are made while loading (no separate pass).
struct TopkRaw {
  const void* key;  // null: read (image, row) pairs of an earlier round
  int dtype;
  int desc;
};

__device__ __forceinline__ u64 topk_image(const TopkRaw& r, i64 i) {
  switch (r.dtype) {
    case TDP_I64:
      return image_i64(__ldg(reinterpret_cast<const i64*>(r.key) + i), r.desc);
    case TDP_I32:
      return image_i64((i64)__ldg(reinterpret_cast<const int*>(r.key) + i), r.desc);
    case TDP_F64:
      return image_f64(__ldg(reinterpret_cast<const double*>(r.key) + i), r.desc);
    default:
      return image_f32(__ldg(reinterpret_cast<const float*>(r.key) + i), r.desc);
  }
}

// Ascending bitonic sort of n (a power of two) (image, row) pairs in shared memory.
__device__ __forceinline__ void topk_bitonic(u64* sk, i64* si, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < n / 2; t += blockDim.x) {
        const int a = 2 * t - (t & (stride - 1));
        const int b = a + stride;
        const bool up = (a & size) == 0;
        const u64 ka = sk[a], kb = sk[b];
        const i64 ia = si[a], ib = si[b];
        const bool gt = ka > kb || (ka == kb && ia > ib);
        if (gt == up) {
          sk[a] = kb;
          sk[b] = ka;
          si[a] = ib;
          si[b] = ia;
        }
      }
    }
  }
  __syncthreads();
}

// One round: every CTA sorts `chunk` pairs and keeps its first k (the first
// round reads the key column itself); final_idx: a single CTA, the answer.
// (A last-CTA-finishes-the-job variant of the second-to-last round measured
// slower: one CTA sorting 2048 survivors takes longer than a launch.)
__global__ void __launch_bounds__(kTopkChunk / 2)
    topk_chunk_kernel(TopkRaw raw, const u64* __restrict__ keys, const i64* __restrict__ idx,
                      i64 m, int k, int chunk, u64* __restrict__ out_keys,
                      i64* __restrict__ out_idx, i64* __restrict__ final_idx, i64 final_count) {
  __shared__ u64 sk[kTopkChunk];
  __shared__ i64 si[kTopkChunk];
  const i64 base = (i64)blockIdx.x * chunk;
  for (int t = threadIdx.x; t < chunk; t += blockDim.x) {
    const i64 g = base + t;
    const bool ok = g < m;
    if (raw.key != nullptr) {
      sk[t] = ok ? topk_image(raw, g) : ~0ull;
      si[t] = ok ? g : LLONG_MAX;
    } else {
      sk[t] = ok ? keys[g] : ~0ull;
      si[t] = ok ? idx[g] : LLONG_MAX;  // sentinel sorts after every real pair
    }
  }
  topk_bitonic(sk, si, chunk);
  if (final_idx != nullptr) {  // last round: one CTA, the answer
    for (int t = threadIdx.x; t < final_count; t += blockDim.x) final_idx[t] = si[t];
    return;
  }
  for (int t = threadIdx.x; t < k; t += blockDim.x) {
    out_keys[(i64)blockIdx.x * k + t] = sk[t];
    out_idx[(i64)blockIdx.x * k + t] = si[t];
  }
}

// ---------------------------------------------------------------------------
// Large inputs (n >= kSelMinRows): radix select instead of sorting chunks.
// The k smallest (image, row) pairs are found digit by digit -- 11 bits of the
// 64-bit key image per pass (6 passes), then 11 bits of the row index (4
// passes: ties resolved to the lowest rows, the stable order) -- each pass a
// histogram of the candidates' next digit, a one-CTA pick of the bucket that
// holds the k-th pair, and a compaction that sets aside every pair below it
// ("sure") and keeps the bucket's pairs as the next candidates.  Candidates
// are rows of the key column re-read with the prefix as a filter ("virtual")
// until a bucket holds <= kSelCompact pairs, then a materialised buffer.  The
// want <= 1024 selected pairs are finally sorted in one CTA.  Everything is
// decided on the device (no host read); a virtual pass costs two reads of the
// key column, typically two such passes, then microseconds.
// ---------------------------------------------------------------------------
constexpr int kSelBits = 11, kSelBins = 1 << kSelBits;
constexpr int kSelPasses = 10;            // 6 over the image, 4 over the row (< 2^44)
constexpr i64 kSelMinRows = 1 << 20;
constexpr i64 kSelCompact = 1 << 16;

struct SelPass {
  int phase;  // 0: image bits, 1: row bits
  int shift;
  int bits;
};

struct SelPlan {
  SelPass p[kSelPasses];
};

// per pass p (filled by the pick kernel of pass p - 1; pass 0 by the host):
//   prefix[p]: the processed high bits the candidates share (phase 0: image
//   bits above shift + bits; phase 1: the whole image is img_eq and the row's
//   high bits match), krem[p] pairs still to take, mat[p]/nbuf[p] whether the
//   candidates are materialised (buf[p & 1]) and how many, done[p]
struct SelState {
  unsigned long long prefix[kSelPasses + 1];
  long long krem[kSelPasses + 1];
  long long nbuf[kSelPasses + 1];
  int mat[kSelPasses + 1];
  int done[kSelPasses + 1];
  int bucket[kSelPasses];
  int take_bucket[kSelPasses];  // last pass: the bucket's pairs are selected too
  long long below[kSelPasses];  // candidates below the picked bucket (selected)
  unsigned long long img_eq;    // phase 1: the threshold image
  unsigned long long nsure;     // pairs selected so far
};

struct SelWs {
  SelState* st;
  unsigned long long* hist;  // [kSelBins]
  u64* sure_k;               // [kTopkMax]
  i64* sure_i;
  u64* buf_k[2];             // [kSelCompact]
  i64* buf_i[2];
};

__device__ __forceinline__ bool sel_candidate(const SelState& st, const SelPass& ps, int p, u64 img,
                                              i64 row, unsigned* digit) {
  if (ps.phase == 0) {
    const int hi = ps.shift + ps.bits;  // bits above this digit
    if (hi < 64 && (img >> hi) != st.prefix[p]) return false;
    *digit = (unsigned)((img >> ps.shift) & ((1u << ps.bits) - 1u));
    return true;
  }
  if (img != st.img_eq) return false;
  const int hi = ps.shift + ps.bits;
  const u64 r = (u64)row;
  if (hi < 64 && (r >> hi) != st.prefix[p]) return false;
  *digit = (unsigned)((r >> ps.shift) & ((1u << ps.bits) - 1u));
  return true;
}

__global__ void __launch_bounds__(256)
    sel_hist_kernel(TopkRaw raw, i64 n, SelWs w, SelPlan plan, int p) {
  const SelState& st = *w.st;
  if (st.done[p]) return;
  __shared__ unsigned h[kSelBins];
  for (int b = threadIdx.x; b < kSelBins; b += blockDim.x) h[b] = 0u;
  __syncthreads();
  const SelPass ps = plan.p[p];
  const bool mat = st.mat[p] != 0;
  const i64 m = mat ? (i64)st.nbuf[p] : n;
  const u64* bk = w.buf_k[p & 1];
  const i64* bi = w.buf_i[p & 1];
  const i64 stride = (i64)gridDim.x * blockDim.x;
  i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (!mat) {  // four rows' loads in flight per thread
    for (; i + 3 * stride < m; i += 4 * stride) {
      u64 img[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) img[u] = topk_image(raw, i + u * stride);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        unsigned d;
        if (sel_candidate(st, ps, p, img[u], i + u * stride, &d)) atomicAdd(&h[d], 1u);
      }
    }
  }
  for (; i < m; i += stride) {
    const u64 img = mat ? bk[i] : topk_image(raw, i);
    const i64 row = mat ? bi[i] : i;
    unsigned d;
    if (sel_candidate(st, ps, p, img, row, &d)) atomicAdd(&h[d], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kSelBins; b += blockDim.x)
    if (h[b]) atomicAdd(w.hist + b, (unsigned long long)h[b]);
}

// One CTA of 1024 threads: the bucket holding the krem-th candidate.
__global__ void __launch_bounds__(1024) sel_pick_kernel(SelWs w, SelPlan plan, int p) {
  SelState& st = *w.st;
  __shared__ unsigned long long part[1024];
  __shared__ int pick;
  if (st.done[p]) {
    if (threadIdx.x == 0) {
      st.done[p + 1] = 1;
      st.krem[p + 1] = 0;
    }
    return;
  }
  // two bins per thread, inclusive scan over the 1024 partial sums
  const int t = threadIdx.x;
  const unsigned long long a = w.hist[2 * t], b = w.hist[2 * t + 1];
  part[t] = a + b;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const unsigned long long v = t >= o ? part[t - o] : 0ull;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  const long long krem = st.krem[p];
  if (t == 0) pick = -1;
  __syncthreads();
  const unsigned long long before = t ? part[t - 1] : 0ull;
  if ((long long)before < krem && (long long)part[t] >= krem)  // the k-th lies in bins 2t, 2t+1
    pick = (long long)(before + a) >= krem ? 2 * t : 2 * t + 1;
  __syncthreads();
  if (t == 0) {
    const SelPass ps = plan.p[p];
    const int bk = pick < 0 ? 0 : pick;
    unsigned long long below = 0;
    for (int q = 0; q < bk; ++q) below += w.hist[q];
    const unsigned long long inb = w.hist[bk];
    st.bucket[p] = bk;
    st.below[p] = (long long)below;
    const long long left = krem - (long long)below;  // to take from the bucket
    const bool last = p == kSelPasses - 1;
    st.take_bucket[p] = last && left > 0;
    st.krem[p + 1] = left;
    st.done[p + 1] = pick < 0 || left <= 0 || last;
    if (p + 1 < kSelPasses) {
      const SelPass nx = plan.p[p + 1];
      if (ps.phase == 0 && nx.phase == 1) {  // the image is now fully known
        st.img_eq = (ps.shift + ps.bits >= 64 ? 0ull : (st.prefix[p] << ps.bits)) | (u64)bk;
        st.img_eq = (st.img_eq << ps.shift);
        st.prefix[p + 1] = 0ull;
      } else {
        st.prefix[p + 1] = (st.prefix[p] << ps.bits) | (u64)bk;
      }
      st.mat[p + 1] = st.mat[p] || (long long)inb <= kSelCompact;
      st.nbuf[p + 1] = 0;
    }
  }
  __syncthreads();
  w.hist[2 * t] = 0ull;  // ready for the next pass
  w.hist[2 * t + 1] = 0ull;
}

// One candidate of the compaction: selected (below the bucket, or the
// bucket's pairs in the last pass) or kept as a next-pass candidate.
__device__ __forceinline__ void sel_place(SelState& st, const SelWs& w, unsigned d,
                                          unsigned bsel, bool take_bucket, bool keep_next,
                                          u64 img, i64 row, u64* nk, i64* ni, int p) {
  if (d < bsel || (d == bsel && take_bucket)) {
    const unsigned long long at = atomicAdd(&st.nsure, 1ull);
    if (at < (unsigned long long)kTopkMax) {
      w.sure_k[at] = img;
      w.sure_i[at] = row;
    }
  } else if (d == bsel && keep_next) {
    const unsigned long long at = atomicAdd((unsigned long long*)&st.nbuf[p + 1], 1ull);
    if (at < (unsigned long long)kSelCompact) {
      nk[at] = img;
      ni[at] = row;
    }
  }
}

// Pairs below the picked bucket are selected; the bucket's pairs become the
// next candidates when they are materialised (or, in the last pass, selected).
__global__ void __launch_bounds__(256)
    sel_compact_kernel(TopkRaw raw, i64 n, SelWs w, SelPlan plan, int p) {
  SelState& st = *w.st;
  if (st.done[p]) return;
  const SelPass ps = plan.p[p];
  const bool mat = st.mat[p] != 0;
  const bool keep_next = p + 1 < kSelPasses && st.mat[p + 1] && !st.done[p + 1];
  const bool take_bucket = st.take_bucket[p] != 0;
  const unsigned bsel = (unsigned)st.bucket[p];
  if (st.below[p] == 0 && !keep_next && !take_bucket) return;  // nothing to place
  const i64 m = mat ? (i64)st.nbuf[p] : n;
  const u64* bk = w.buf_k[p & 1];
  const i64* bi = w.buf_i[p & 1];
  u64* nk = w.buf_k[(p + 1) & 1];
  i64* ni = w.buf_i[(p + 1) & 1];
  const i64 stride = (i64)gridDim.x * blockDim.x;
  i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (!mat) {  // four rows' loads in flight; rows with no action skip the slow path
    for (; i + 3 * stride < m; i += 4 * stride) {
      u64 img[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) img[u] = topk_image(raw, i + u * stride);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        unsigned d;
        if (!sel_candidate(st, ps, p, img[u], i + u * stride, &d)) continue;
        sel_place(st, w, d, bsel, take_bucket, keep_next, img[u], i + u * stride, nk, ni, p);
      }
    }
  }
  for (; i < m; i += stride) {
    const u64 img = mat ? bk[i] : topk_image(raw, i);
    const i64 row = mat ? bi[i] : i;
    unsigned d;
    if (!sel_candidate(st, ps, p, img, row, &d)) continue;
    sel_place(st, w, d, bsel, take_bucket, keep_next, img, row, nk, ni, p);
  }
}


__global__ void sel_init_kernel(SelState* st, i64 want) {
  unsigned* w = reinterpret_cast<unsigned*>(st);
  for (int t = threadIdx.x; t < (int)(sizeof(SelState) / 4); t += blockDim.x) w[t] = 0u;
  __syncthreads();
  if (threadIdx.x == 0) st->krem[0] = want;
}

// The selected pairs (want of them) in ascending (image, row) order.
__global__ void __launch_bounds__(1024)
    sel_final_kernel(SelWs w, i64 want, i64* __restrict__ out_order) {
  __shared__ u64 sk[kTopkMax];
  __shared__ i64 si[kTopkMax];
  const int nsel = (int)(w.st->nsure < (unsigned long long)kTopkMax ? w.st->nsure : kTopkMax);
  for (int t = threadIdx.x; t < kTopkMax; t += blockDim.x) {
    sk[t] = t < nsel ? w.sure_k[t] : ~0ull;
    si[t] = t < nsel ? w.sure_i[t] : LLONG_MAX;
  }
  topk_bitonic(sk, si, kTopkMax);
  for (int t = threadIdx.x; t < want; t += blockDim.x) out_order[t] = si[t];
}

int topk_round_chunk(i64 m, i64 k) {
  int c = 64;
  while (c < 2 * k) c <<= 1;
  while (c < kTopkChunk && ceil_div(m, c) > 2 * (i64)sm_count()) c <<= 1;
  return c;
}

int pow2_at_least(i64 m) {
  int c = 2;
  while (c < m) c <<= 1;
  return c;
}

}  // namespace tdp

using namespace tdp;

extern "C" {

size_t tdp_sort_workspace(int64_t n) { return sort_ws_bytes(n); }

size_t tdp_topk_workspace(int64_t n, int64_t k) {
  // first round: chunks of at least 64 pairs (and >= 2k), k survivors each
  const i64 m1 = ceil_div(n > 0 ? n : 1, 64) * (k > 0 ? k : 1);
  return 2 * align256((size_t)(n > 0 ? n : 1) * 8) + 4 * align256((size_t)m1 * 8) + 256;
}

int tdp_topk_order(const tdp_column* key, int32_t descending, int64_t n, int64_t k,
                   int64_t* out_order, void* ws, size_t ws_bytes, void* stream) {
  TDP_REQUIRE(key != nullptr && n >= 0, "bad top-k arguments");
  TDP_REQUIRE(k >= 1 && k <= kTopkMax, "top-k needs 1 <= k <= %d (got %lld)", kTopkMax,
              (long long)k);
  TDP_REQUIRE(key->width == 1, "sort keys must be scalar columns");
  TDP_REQUIRE(key->dtype == TDP_I64 || key->dtype == TDP_F64 || key->dtype == TDP_F32 ||
                  key->dtype == TDP_I32,
              "sort key dtype %d not supported", key->dtype);
  TDP_REQUIRE(key->rows >= n, "short key column");
  if (n == 0) return TDP_OK;
  TDP_REQUIRE(ws_bytes >= tdp_topk_workspace(n, k), "top-k workspace too small");
  cudaStream_t st = as_stream(stream);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  u64* k0 = (u64*)p;
  p += align256((size_t)n * 8);
  i64* i0 = (i64*)p;
  p += align256((size_t)n * 8);
  const i64 m1 = ceil_div(n, 64) * k;
  u64* ka = (u64*)p;
  p += align256((size_t)m1 * 8);
  i64* ia = (i64*)p;
  p += align256((size_t)m1 * 8);
  u64* kb = (u64*)p;
  p += align256((size_t)m1 * 8);
  i64* ib = (i64*)p;
  (void)k0;
  (void)i0;
  TopkRaw raw{key->data, key->dtype, descending ? 1 : 0};
  const TopkRaw none{nullptr, 0, 0};
  const i64 want = k < n ? k : n;
  if (n >= kSelMinRows) {  // radix select (see above)
    unsigned char* q = reinterpret_cast<unsigned char*>(ws);
    SelWs w;
    w.st = reinterpret_cast<SelState*>(q);
    q += align256(sizeof(SelState));
    w.hist = reinterpret_cast<unsigned long long*>(q);
    q += align256(kSelBins * 8);
    w.sure_k = reinterpret_cast<u64*>(q);
    q += align256(kTopkMax * 8);
    w.sure_i = reinterpret_cast<i64*>(q);
    q += align256(kTopkMax * 8);
    for (int b = 0; b < 2; ++b) {
      w.buf_k[b] = reinterpret_cast<u64*>(q);
      q += align256(kSelCompact * 8);
      w.buf_i[b] = reinterpret_cast<i64*>(q);
      q += align256(kSelCompact * 8);
    }
    TDP_REQUIRE((size_t)(q - reinterpret_cast<unsigned char*>(ws)) <= ws_bytes,
                "top-k workspace too small for the radix select");
    SelPlan plan;
    const int img_shifts[6] = {53, 42, 31, 20, 9, 0};
    const int img_bits[6] = {11, 11, 11, 11, 11, 9};
    for (int i = 0; i < 6; ++i) plan.p[i] = SelPass{0, img_shifts[i], img_bits[i]};
    for (int i = 0; i < 4; ++i) plan.p[6 + i] = SelPass{1, 33 - 11 * i, 11};
    sel_init_kernel<<<1, 128, 0, st>>>(w.st, want);  // no host copy: graph-capturable
    TDP_CUDA_TRY(cudaMemsetAsync(w.hist, 0, kSelBins * 8, st));
    const int grid = stream_grid(n, 256 * 8, 8);
    for (int p = 0; p < kSelPasses; ++p) {
      sel_hist_kernel<<<grid, 256, 0, st>>>(raw, n, w, plan, p);
      sel_pick_kernel<<<1, 1024, 0, st>>>(w, plan, p);
      sel_compact_kernel<<<grid, 256, 0, st>>>(raw, n, w, plan, p);
    }
    TDP_LAUNCH_CHECK("sel kernels");
    sel_final_kernel<<<1, 1024, 0, st>>>(w, want, out_order);
    TDP_LAUNCH_CHECK("sel_final_kernel");
    return TDP_OK;
  }
  if (n <= kTopkChunk) {  // one CTA: the answer
    const int last = pow2_at_least(n);
    topk_chunk_kernel<<<1, last / 2 > 32 ? last / 2 : 32, 0, st>>>(
        raw, nullptr, nullptr, n, (int)k, last, nullptr, nullptr, out_order, want);
    TDP_LAUNCH_CHECK("topk_chunk_kernel");
    return TDP_OK;
  }
  const u64* sk = nullptr;
  const i64* si = nullptr;
  i64 m = n;
  bool use_a = true;
  for (;;) {
    const int chunk = topk_round_chunk(m, k);
    const i64 blocks = ceil_div(m, chunk);
    u64* dk = use_a ? ka : kb;
    i64* di = use_a ? ia : ib;
    topk_chunk_kernel<<<(unsigned)blocks, chunk / 2, 0, st>>>(sk == nullptr ? raw : none, sk, si,
                                                              m, (int)k, chunk, dk, di, nullptr,
                                                              0);
    TDP_LAUNCH_CHECK("topk_chunk_kernel");
    sk = dk;
    si = di;
    m = blocks * k;
    use_a = !use_a;
    if (m <= kTopkChunk) {
      const int last = pow2_at_least(m);
      topk_chunk_kernel<<<1, last / 2 > 32 ? last / 2 : 32, 0, st>>>(
          none, sk, si, m, (int)k, last, nullptr, nullptr, out_order, want);
      TDP_LAUNCH_CHECK("topk_chunk_kernel");
      return TDP_OK;
    }
  }
}

int tdp_sort_order(const tdp_column* key, int32_t descending, int64_t n, int64_t* out_order,
                   void* ws, size_t ws_bytes, void* stream) {
  TDP_REQUIRE(key != nullptr && n >= 0, "bad sort arguments");
  TDP_REQUIRE(key->width == 1, "sort keys must be scalar columns");
  TDP_REQUIRE(key->dtype == TDP_I64 || key->dtype == TDP_F64 || key->dtype == TDP_F32 ||
                  key->dtype == TDP_I32,
              "sort key dtype %d not supported", key->dtype);
  TDP_REQUIRE(key->rows >= n, "short key column");
  if (n == 0) return TDP_OK;
  TDP_REQUIRE(ws_bytes >= sort_ws_bytes(n), "sort workspace too small");
  cudaStream_t st = as_stream(stream);
  SortBuffers b = carve(ws, n);
  make_keys_kernel<<<stream_grid(n, 256 * 8, 8), 256, 0, st>>>(key->data, key->dtype,
                                                                descending ? 1 : 0, n, b.k0, b.i0);
  TDP_LAUNCH_CHECK("make_keys_kernel");
  u64* sk;
  i64* order;
  int rc = radix_sort(b, n, st, &sk, &order);
  if (rc) return rc;
  TDP_CUDA_TRY(cudaMemcpyAsync(out_order, order, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
  return TDP_OK;
}

int tdp_unique_inverse(const int64_t* key, int64_t n, int64_t* out_uniques, int64_t* out_inverse,
                       int64_t* out_nunique, void* ws, size_t ws_bytes, void* stream) {
  TDP_REQUIRE(n >= 0, "negative length");
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    TDP_CUDA_TRY(cudaMemsetAsync(out_nunique, 0, 8, st));
    return TDP_OK;
  }
  TDP_REQUIRE(ws_bytes >= sort_ws_bytes(n) + 2 * align256((size_t)n * 8),
              "unique workspace too small");
  SortBuffers b = carve(ws, n);
  unsigned char* extra = reinterpret_cast<unsigned char*>(ws) + sort_ws_bytes(n);
  i64* flags = reinterpret_cast<i64*>(extra);
  i64* excl = reinterpret_cast<i64*>(extra + align256((size_t)n * 8));
  make_keys_kernel<<<stream_grid(n, 256 * 8, 8), 256, 0, st>>>(key, TDP_I64, 0, n, b.k0, b.i0);
  TDP_LAUNCH_CHECK("make_keys_kernel");
  u64* sk;
  i64* order;
  int rc = radix_sort(b, n, st, &sk, &order);
  if (rc) return rc;
  boundary_flags_kernel<<<stream_grid(n, 256 * 8, 8), 256, 0, st>>>(sk, n, flags);
  TDP_LAUNCH_CHECK("boundary_flags_kernel");
  rc = exclusive_scan_i64(flags, excl, n, out_nunique, b.scan_ws, b.scan_bytes, st);
  if (rc) return rc;
  unique_scatter_kernel<<<stream_grid(n, 256 * 8, 8), 256, 0, st>>>(sk, order, flags, excl, n,
                                                                     out_uniques, out_inverse);
  TDP_LAUNCH_CHECK("unique_scatter_kernel");
  return TDP_OK;
}

size_t tdp_groupby_codes_workspace(int64_t slots, int32_t naggs) {
  return (size_t)(slots > 0 ? slots : 1) * (size_t)(naggs > 0 ? naggs : 0) * kFixedWords * 8 + 256;
}

int tdp_groupby_codes(const int64_t* codes, int64_t n, int64_t slots, const tdp_column* vals,
                      const int32_t* agg_kinds, int32_t naggs, int64_t* out_counts,
                      void* out_sums, void* ws, size_t ws_bytes, void* stream) {
  TDP_REQUIRE(n >= 0 && slots >= 1, "bad group-by shape");
  TDP_REQUIRE(naggs >= 0 && naggs <= 32, "at most 32 aggregates");
  ValSet vs;
  std::memset(&vs, 0, sizeof(vs));
  vs.naggs = naggs;
  for (int a = 0; a < naggs; ++a) {
    vs.kind[a] = agg_kinds[a];
    TDP_REQUIRE(agg_kinds[a] >= TDP_AGG_COUNT && agg_kinds[a] <= TDP_AGG_SUM_I64,
                "agg %d: bad kind", a);
    if (agg_kinds[a] == TDP_AGG_COUNT) {
      vs.p[a] = nullptr;
      vs.dt[a] = TDP_I64;
      continue;
    }
    TDP_REQUIRE(vals != nullptr && vals[a].rows >= n && vals[a].width == 1,
                "agg %d: value column must be scalar with >= n rows", a);
    vs.p[a] = vals[a].data;
    vs.dt[a] = vals[a].dtype;
  }
  number_fixed(&vs);
  const size_t fx_bytes = (size_t)slots * vs.nfixed * kFixedWords * 8;
  TDP_REQUIRE(vs.nfixed == 0 || (ws != nullptr && ws_bytes >= fx_bytes),
              "group-by workspace too small (%zu < %zu)", ws_bytes, fx_bytes);
  unsigned long long* fx = reinterpret_cast<unsigned long long*>(ws);
  cudaStream_t st = as_stream(stream);
  TDP_CUDA_TRY(cudaMemsetAsync(out_counts, 0, (size_t)slots * 8, st));
  if (naggs) TDP_CUDA_TRY(cudaMemsetAsync(out_sums, 0, (size_t)slots * naggs * 8, st));
  if (vs.nfixed) TDP_CUDA_TRY(cudaMemsetAsync(fx, 0, fx_bytes, st));
  if (n > 0) {
    groupby_codes_kernel<<<stream_grid(n, 256 * 4, 8), 256, 0, st>>>(
        codes, n, slots, vs, reinterpret_cast<unsigned long long*>(out_counts),
        reinterpret_cast<unsigned long long*>(out_sums), fx);
    TDP_LAUNCH_CHECK("groupby_codes_kernel");
  }
  if (vs.nfixed) {
    fixed_finalize_kernel<<<stream_grid(slots * naggs, 256, 4), 256, 0, st>>>(
        fx, slots, vs, reinterpret_cast<unsigned long long*>(out_sums), slots);
    TDP_LAUNCH_CHECK("fixed_finalize_kernel");
  }
  if (naggs) {
    copy_counts_kernel<<<stream_grid(slots * naggs, 256, 4), 256, 0, st>>>(
        reinterpret_cast<unsigned long long*>(out_counts), slots, vs,
        reinterpret_cast<unsigned long long*>(out_sums));
    TDP_LAUNCH_CHECK("copy_counts_kernel");
  }
  return TDP_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// equi-join.  Build: an open-addressing hash table over the distinct build
// keys (16-byte slots {key ^ INT64_MIN (0 = empty), packed run}, one vector
// load per probe) plus a split-block Bloom filter (~16 bits per key, L2-
// resident).  The build first inserts every row in input order, which is the
// whole build when the keys are unique (the primary-key side of a PK-FK join:
// no sort, run start = the row itself).  Only if a key repeats does it fall
// back to a stable radix sort of the build keys and insert one run per
// distinct key (key -> [start, count) in sorted order).
//
// Probe: pass 1 (count) evaluates the optional probe-side filter on the base
// columns, the Bloom filter and the table, and writes one match bit per row,
// per-word pair counts and per-tile pair counts; a scan gives tile offsets.
// Pass 2 (emit) writes the pairs: probe row order (base row ids), ascending
// build row within a probe row.  Unique keys emit in two fully parallel
// steps (expand match bits -> probe rows, then one thread per pair); runs use
// a warp-per-word re-probe with a warp scan of the run lengths.
// ---------------------------------------------------------------------------
namespace tdp {
namespace {

constexpr int kJoinThreads = 256;
constexpr int kJoinTile = 2048;  // probe rows per tile
constexpr int kJoinWords = kJoinTile / 32;
constexpr int kJoinPer = kJoinTile / kJoinThreads;
constexpr int kJoinWarps = kJoinThreads / 32;

// Tile-per-CTA probe / build passes prefetch a later tile's columns into L2
// with one bulk instruction per column (l2_prefetch_range): the HBM stream
// runs a wave ahead of the CTAs' dependent bitmap / Bloom / slot lookups
// (Q3 SF10 lineitem probe 0.182 -> 0.153 ms, 0.81 -> 0.96 of the copy peak).
// The CTA of tile `tile` asks L2 for the rows of tile `tile + ahead`.
__device__ __forceinline__ void join_prefetch_ahead(i64 ahead, i64 tile, const i64* keys, i64 n,
                                                     const PredSet& ps, bool filtered) {
  if (ahead <= 0 || threadIdx.x != 0) return;
  const i64 r0 = (tile + ahead) * kJoinTile;
  if (r0 >= n) return;
  const i64 rows = n - r0 < kJoinTile ? n - r0 : kJoinTile;
  l2_prefetch_range(keys + r0, rows * 8);
  if (filtered) prefetch_predset_l2(ps, r0, rows);
}

// L2 prefetch distance in tiles: resident CTAs of a wave x TDP_L2_AHEAD
// (measurements; default 1, 0 disables)
inline i64 join_ahead(int ctas_per_sm) {
  static const double mult = [] {
    const char* e = getenv("TDP_L2_AHEAD");
    return e ? atof(e) : 1.0;
  }();
  return (i64)(mult * sm_count() * ctas_per_sm);
}
constexpr i64 kMinKey = (i64)0x8000000000000000ull;

// slot.y packs (start + 1) << 24 | min(run length, kCountSat); a saturated
// length is read from count[] (runs of >= 16M equal build keys only).
constexpr i64 kCountSat = (1 << 24) - 1;

// One 64-bit multiply + xor-shift (the probe pass is instruction-bound at
// 8-16 B/row); the table index, the Bloom block and its bit salts use
// different bits.
__device__ __forceinline__ u64 join_hash(i64 key) {
  u64 h = (u64)key * 0x9E3779B97F4A7C15ull;
  return h ^ (h >> 29);
}

struct HashTable {
  longlong2* slot;   // [cap]
  i64* count;        // [cap] run length (read only when saturated)
  u64 mask;
  unsigned* bloom;   // [nwords]
  unsigned bmask;    // nwords - 1
  i64* side;         // run of the key INT64_MIN (its image is the empty marker): {start+1, count}
  int* flags;        // [0] a key repeats, [1] build is sorted (runs), else unique
  const i64* order;  // sorted build row ids (sorted mode)
  i64 ahead;         // probe: tiles ahead prefetched into L2 (join_prefetch_ahead)
};

// Register-blocked Bloom filter: one 32-bit word per key, 3 bits from 5-bit
// fields of the hash (the table index uses the low bits of the full hash, the
// word index bits 40+).  ~16 bits per key: a few MB, L2-resident, one 4-byte
// load and a handful of 32-bit ops per probe; false positives ~1%.
__device__ __forceinline__ unsigned bloom_mask(u64 h) {
  const unsigned x = (unsigned)(h >> 16);
  return (1u << (x & 31)) | (1u << ((x >> 5) & 31)) | (1u << ((x >> 10) & 31));
}

__device__ __forceinline__ const unsigned* bloom_word(const HashTable& ht, u64 h) {
  return ht.bloom + ((unsigned)(h >> 40) & ht.bmask);
}

__device__ __forceinline__ i64 pack_run(i64 start, i64 cnt) {
  return ((start + 1) << 24) | (cnt < kCountSat ? cnt : kCountSat);
}

// Insert key -> run; false if the key is already present.
__device__ bool ht_insert(const HashTable& ht, i64 key, i64 start, i64 cnt) {
  if (key == kMinKey) {
    const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(ht.side), 0ull,
                                              (unsigned long long)(start + 1));
    if (prev != 0ull) return false;
    ht.side[1] = cnt;
    return true;
  }
  const u64 hk = join_hash(key);
  const i64 kx = key ^ kMinKey;
  u64 h = hk & ht.mask;
  for (;;) {
    const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(&ht.slot[h].x),
                                              0ull, (unsigned long long)kx);
    if (prev == 0ull) {
      ht.slot[h].y = pack_run(start, cnt);
      if (cnt >= kCountSat) ht.count[h] = cnt;
      atomicOr(ht.bloom + ((unsigned)(hk >> 40) & ht.bmask), bloom_mask(hk));
      return true;
    }
    if ((i64)prev == kx) return false;
    h = (h + 1) & ht.mask;
  }
}

// Build rows failing the optional build predicates are skipped (a filtered
// build relation read straight from its base columns; run starts are then
// base row ids).
template <bool kFiltered>
__global__ void join_build_unique_kernel(const i64* __restrict__ keys, i64 nb, HashTable ht,
                                         PredSet bps) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (i64)gridDim.x * blockDim.x) {
    if (kFiltered && !eval_all(bps, i)) continue;
    if (!ht_insert(ht, __ldg(keys + i), i, 1)) ht.flags[0] = 1;
  }
}

__global__ void join_build_runs_kernel(const u64* __restrict__ sk, i64 nb, HashTable ht) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (i64)gridDim.x * blockDim.x) {
    if (i > 0 && sk[i] == sk[i - 1]) continue;  // only run starts insert
    i64 e = i + 1;
    while (e < nb && sk[e] == sk[i]) ++e;
    ht_insert(ht, (i64)(sk[i] ^ 0x8000000000000000ull), i, e - i);
  }
}

__device__ __forceinline__ void unpack_run(const HashTable& ht, i64 y, u64 h, i64* start, i64* cnt) {
  *start = (y >> 24) - 1;
  const i64 c = y & kCountSat;
  *cnt = c < kCountSat ? c : ht.count[h];
}

// Full lookup (collision chains, the INT64_MIN side slot).
__device__ __noinline__ void join_lookup_slow(const HashTable& ht, i64 key, i64* start, i64* cnt) {
  *start = 0;
  *cnt = 0;
  if (key == kMinKey) {
    const i64 y = ht.side[0];
    if (y != 0) {
      *start = y - 1;
      *cnt = ht.side[1];
    }
    return;
  }
  const i64 kx = key ^ kMinKey;
  u64 h = join_hash(key) & ht.mask;
  for (;;) {
    const longlong2 e = ht.slot[h];
    if (e.x == 0) return;
    if (e.x == kx) {
      unpack_run(ht, e.y, h, start, cnt);
      return;
    }
    h = (h + 1) & ht.mask;
  }
}

// First slot inline; chains and INT64_MIN go to the slow path.
__device__ __forceinline__ void join_resolve(const HashTable& ht, i64 key, u64 hm, longlong2 e,
                                             i64* start, i64* cnt) {
  if (key != kMinKey && e.x == (key ^ kMinKey)) {
    unpack_run(ht, e.y, hm, start, cnt);
  } else if (key != kMinKey && e.x == 0) {
    *start = 0;
    *cnt = 0;
  } else {
    join_lookup_slow(ht, key, start, cnt);
  }
}

__device__ __forceinline__ void join_lookup(const HashTable& ht, i64 key, i64* start, i64* cnt) {
  const u64 hm = join_hash(key) & ht.mask;
  join_resolve(ht, key, hm, ht.slot[hm], start, cnt);
}

// Item k of a thread: rows k*256 .. k*256+255 of the tile form the match
// words k*8 .. k*8+7 (warp w owns word k*8+w, lane = bit).
__device__ __forceinline__ i64 join_row(i64 tile, int k) {
  return tile * kJoinTile + (i64)k * kJoinThreads + threadIdx.x;
}

// tile_counts must be zeroed: every warp adds its pair count (no CTA barrier,
// so a warp leaves as soon as its own lookups are done).  Three batched
// rounds of loads per thread (keys + predicate columns, Bloom words, table
// slots), 8 rows each; with unique build keys only the slot keys are read.
template <bool kFiltered, bool kUnique>
__global__ void __launch_bounds__(kJoinThreads, kUnique ? 4 : 3)
    join_count_kernel(HashTable ht, const i64* __restrict__ probe, i64 np, PredSet ps,
                      unsigned* __restrict__ match_bits, i64* __restrict__ word_counts,
                      i64* __restrict__ tile_counts) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 tile = blockIdx.x;
  join_prefetch_ahead(ht.ahead, tile, probe, np, ps, kFiltered);
  bool act[kJoinPer];
  i64 row[kJoinPer], key[kJoinPer];
#pragma unroll
  for (int k = 0; k < kJoinPer; ++k) {
    row[k] = join_row(tile, k);
    act[k] = row[k] < np;
  }
  // keys are loaded together with the predicate columns (a selective filter
  // still touches nearly every sector, so this costs no DRAM traffic and
  // saves a dependent round trip)
#pragma unroll
  for (int k = 0; k < kJoinPer; ++k) key[k] = act[k] ? __ldcs(probe + row[k]) : 0;
  if (kFiltered) eval_batch<kJoinPer>(ps, row, act);
  unsigned bw[kJoinPer];
#pragma unroll
  for (int k = 0; k < kJoinPer; ++k)
    bw[k] = act[k] ? *bloom_word(ht, join_hash(key[k])) : 0u;
  unsigned slot[kJoinPer];
  i64 ex[kJoinPer], ey[kJoinPer];
#pragma unroll
  for (int k = 0; k < kJoinPer; ++k) {
    const u64 h = join_hash(key[k]);
    const unsigned m = bloom_mask(h);
    act[k] = act[k] && (key[k] == kMinKey || (bw[k] & m) == m);
    slot[k] = (unsigned)(h & ht.mask);
    ex[k] = 0;
    ey[k] = 0;
    if (act[k]) {
      if (kUnique) {
        ex[k] = ht.slot[slot[k]].x;
      } else {
        const longlong2 e = ht.slot[slot[k]];
        ex[k] = e.x;
        ey[k] = e.y;
      }
    }
  }
  i64 local = 0;
#pragma unroll
  for (int k = 0; k < kJoinPer; ++k) {
    i64 c = 0;
    if (act[k]) {
      if (kUnique && key[k] != kMinKey && ex[k] == (key[k] ^ kMinKey)) {
        c = 1;
      } else if (key[k] != kMinKey && ex[k] == 0) {
        c = 0;
      } else {
        i64 st;
        join_resolve(ht, key[k], slot[k], make_longlong2(ex[k], kUnique ? ht.slot[slot[k]].y : ey[k]),
                     &st, &c);
      }
    }
    const unsigned word = __ballot_sync(0xffffffffu, c > 0);
    const i64 wc = kUnique ? (i64)__popc(word) : (word ? warp_sum(c) : 0);
    if (lane == 0) {
      match_bits[tile * kJoinWords + k * kJoinWarps + warp] = word;
      word_counts[tile * kJoinWords + k * kJoinWarps + warp] = wc;
    }
    local += wc;
  }
  if (lane == 0 && local != 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(tile_counts + tile), (unsigned long long)local);
}

// Exclusive prefix of a tile's 64 word pair counts, per warp (lane l holds
// words 2l, 2l+1); word_offset(j) reads it back for word j.
struct WordPrefix {
  i64 excl, w0;
  __device__ __forceinline__ WordPrefix(const i64* wc, int lane) {
    w0 = wc[2 * lane];
    const i64 w1 = wc[2 * lane + 1];
    i64 incl = w0 + w1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const i64 t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    excl = incl - w0 - w1;
  }
  __device__ __forceinline__ i64 word_offset(int j) const {
    const i64 pe = __shfl_sync(0xffffffffu, excl, j >> 1);
    const i64 p0 = __shfl_sync(0xffffffffu, w0, j >> 1);
    return pe + ((j & 1) ? p0 : 0);
  }
};

// Runs (a key repeats): every warp places its own words, its 8 lookups in
// flight together, a warp scan of the run lengths per word.  Persistent CTAs
// walk the tiles.
__global__ void __launch_bounds__(kJoinThreads)
    join_emit_runs_kernel(HashTable ht, const i64* __restrict__ probe, i64 tiles,
                          const unsigned* __restrict__ match_bits,
                          const i64* __restrict__ word_counts, const i64* __restrict__ tile_counts,
                          const i64* __restrict__ tile_offsets, i64* __restrict__ out_probe,
                          i64* __restrict__ out_build) {
  if (ht.flags[1] == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (i64 tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    if (tile_counts[tile] == 0) continue;
    const WordPrefix wp(word_counts + tile * kJoinWords, lane);
    const i64 base = tile_offsets[tile];
    unsigned bits[kJoinPer];
    i64 s[kJoinPer], c[kJoinPer];
#pragma unroll
    for (int k = 0; k < kJoinPer; ++k) bits[k] = match_bits[tile * kJoinWords + k * kJoinWarps + warp];
#pragma unroll
    for (int k = 0; k < kJoinPer; ++k) {
      s[k] = 0;
      c[k] = 0;
      if ((bits[k] >> lane) & 1u) join_lookup(ht, __ldg(probe + join_row(tile, k)), &s[k], &c[k]);
    }
#pragma unroll
    for (int k = 0; k < kJoinPer; ++k) {
      if (bits[k] == 0u) continue;  // warp-uniform
      const i64 word_off = base + wp.word_offset(k * kJoinWarps + warp);
      i64 ci = c[k];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const i64 t = __shfl_up_sync(0xffffffffu, ci, o);
        if (lane >= o) ci += t;
      }
      const i64 pos = word_off + ci - c[k];
      const i64 i = join_row(tile, k);
      for (i64 m = 0; m < c[k]; ++m) {
        out_probe[pos + m] = i;
        out_build[pos + m] = ht.order[s[k] + m];
      }
    }
  }
}

// Unique keys: expand the match bits into probe rows (no lookups), one warp
// per tile (one DRAM round trip per tile, thousands of tiles in flight):
// lane l owns words 2l, 2l+1 = rows 64l .. 64l+63 of the tile ...
__global__ void __launch_bounds__(kJoinThreads)
    join_expand_unique_kernel(HashTable ht, i64 tiles, const unsigned* __restrict__ match_bits,
                              const i64* __restrict__ word_counts,
                              const i64* __restrict__ tile_counts,
                              const i64* __restrict__ tile_offsets, i64* __restrict__ out_probe) {
  if (ht.flags[1] != 0) return;
  const int lane = threadIdx.x & 31;
  const i64 tile = (i64)blockIdx.x * kJoinWarps + (threadIdx.x >> 5);
  if (tile >= tiles || tile_counts[tile] == 0) return;  // warp-uniform
  const i64* wc = word_counts + tile * kJoinWords;
  const unsigned* mb = match_bits + tile * kJoinWords;
  const i64 w0 = wc[2 * lane], w1 = wc[2 * lane + 1];
  unsigned b0 = mb[2 * lane], b1 = mb[2 * lane + 1];
  i64 incl = w0 + w1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const i64 t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  i64 pos = tile_offsets[tile] + incl - w0 - w1;
  const i64 row0 = tile * kJoinTile + (i64)lane * 64;
  while (b0) {
    out_probe[pos++] = row0 + __ffs(b0) - 1;
    b0 &= b0 - 1;
  }
  while (b1) {
    out_probe[pos++] = row0 + 32 + __ffs(b1) - 1;
    b1 &= b1 - 1;
  }
}

// ... then one thread per pair re-probes (all lookups independent).
__global__ void join_pairs_unique_kernel(HashTable ht, const i64* __restrict__ probe,
                                         const i64* __restrict__ tile_counts,
                                         const i64* __restrict__ tile_offsets, i64 tiles,
                                         const i64* __restrict__ out_probe,
                                         i64* __restrict__ out_build) {
  if (ht.flags[1] != 0) return;
  const i64 total = tile_offsets[tiles - 1] + tile_counts[tiles - 1];
  for (i64 m = (i64)blockIdx.x * blockDim.x + threadIdx.x; m < total;
       m += (i64)gridDim.x * blockDim.x) {
    i64 s, c;
    join_lookup(ht, __ldg(probe + out_probe[m]), &s, &c);
    out_build[m] = s;
  }
}

u64 table_capacity(i64 nb) {
  u64 cap = 1024;
  while (cap < (u64)(2 * (nb > 0 ? nb : 1))) cap <<= 1;
  return cap;
}

// Bloom words (32-bit): power of two >= nb * per_key_x2 / 2.
// Default half a word (16 bits) per key: Q3's probes measured 0.863 ms at
// 64 bits/key, 0.846 at 32, 0.841 at 16 (a smaller filter stays in L2 and
// clears faster; the extra false positives cost one slot read each).
u64 bloom_blocks(i64 nb) {
  static const int per_key_x2 = [] {  // words per key x 2 (measurements only)
    const char* e = getenv("TDP_BLOOM_WORDS_X2");
    return e ? atoi(e) : 1;
  }();
  u64 b = 64;
  while (b * 2 < (u64)per_key_x2 * (u64)(nb > 0 ? nb : 1)) b <<= 1;
  return b;
}

struct JoinWs {
  SortBuffers sb;
  HashTable ht;
  unsigned* match_bits;
  i64* word_counts;
  i64* tile_counts;
  i64* tile_offsets;
  void* scan_ws;
  size_t scan_bytes;
};

size_t join_ws_bytes(i64 nb, i64 np) {
  const u64 cap = table_capacity(nb);
  const i64 tiles = ceil_div(np > 0 ? np : 1, kJoinTile);
  return sort_ws_bytes(nb) + align256(cap * 16) + align256(cap * 8) +
         align256(bloom_blocks(nb) * 4) + 512 +
         align256((size_t)tiles * kJoinWords * 4) + align256((size_t)tiles * kJoinWords * 8) +
         2 * align256((size_t)tiles * 8) + exclusive_scan_workspace(tiles) + 2048;
}

JoinWs carve_join(void* ws, i64 nb, i64 np) {
  JoinWs j;
  j.sb = carve(ws, nb);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws) + sort_ws_bytes(nb);
  const u64 cap = table_capacity(nb);
  const i64 tiles = ceil_div(np > 0 ? np : 1, kJoinTile);
  j.ht.slot = (longlong2*)p;
  p += align256(cap * 16);
  j.ht.count = (i64*)p;
  p += align256(cap * 8);
  j.ht.mask = cap - 1;
  j.ht.ahead = 0;
  j.ht.bloom = (unsigned*)p;
  p += align256(bloom_blocks(nb) * 4);
  j.ht.bmask = (unsigned)(bloom_blocks(nb) - 1);
  j.ht.side = (i64*)p;
  j.ht.flags = (int*)(p + 256);
  p += 512;
  j.ht.order = j.sb.i0;
  j.match_bits = (unsigned*)p;
  p += align256((size_t)tiles * kJoinWords * 4);
  j.word_counts = (i64*)p;
  p += align256((size_t)tiles * kJoinWords * 8);
  j.tile_counts = (i64*)p;
  p += align256((size_t)tiles * 8);
  j.tile_offsets = (i64*)p;
  p += align256((size_t)tiles * 8);
  j.scan_ws = p;
  j.scan_bytes = exclusive_scan_workspace(tiles) + 1024;
  return j;
}

int clear_table(const JoinWs& j, cudaStream_t st) {
  TDP_CUDA_TRY(cudaMemsetAsync(j.ht.slot, 0, (j.ht.mask + 1) * 16, st));
  TDP_CUDA_TRY(cudaMemsetAsync(j.ht.bloom, 0, ((size_t)j.ht.bmask + 1) * 4, st));
  TDP_CUDA_TRY(cudaMemsetAsync(j.ht.side, 0, 512, st));
  return TDP_OK;
}

// mode 0 (optimistic): hash the (filtered) build rows in input order as if
// the keys were unique; out_info[1] = 1 reports a repeated key, in which case
// the pair count in out_info[0] is not valid and mode 1 must follow.
// mode 1 (runs): stable radix sort of the build keys, one table entry per run
// (no build predicates).  Neither mode synchronises with the host.
int join_prepare_mode(const int64_t* build_keys, int64_t n_build, const PredSet* bps,
                      const int64_t* probe_keys, int64_t n_probe, const PredSet* ps, int mode,
                      int64_t* out_info, void* ws, size_t ws_bytes, cudaStream_t st) {
  TDP_REQUIRE(n_build >= 0 && n_probe >= 0, "negative join sizes");
  TDP_REQUIRE(out_info != nullptr, "null join info output");
  TDP_REQUIRE(mode == 0 || mode == 1, "join mode must be 0 (optimistic) or 1 (runs)");
  TDP_REQUIRE(ws_bytes >= join_ws_bytes(n_build, n_probe), "join workspace too small");
  const bool bfilt = bps != nullptr && bps->npreds > 0;
  TDP_REQUIRE(!(bfilt && mode == 1), "build predicates need unique build keys (mode 0)");
  JoinWs j = carve_join(ws, n_build, n_probe);
  const i64 tiles = ceil_div(n_probe, kJoinTile);
  TDP_CUDA_TRY(cudaMemsetAsync(out_info, 0, 2 * sizeof(i64), st));
  if (n_build == 0 || n_probe == 0) return TDP_OK;
  int rc = clear_table(j, st);
  if (rc) return rc;
  PredSet none;
  none.npreds = 0;
  none.pad = 0;
  if (mode == 0) {
    if (bfilt)
      join_build_unique_kernel<true><<<stream_grid(n_build, 256 * 4, 8), 256, 0, st>>>(
          build_keys, n_build, j.ht, *bps);
    else
      join_build_unique_kernel<false><<<stream_grid(n_build, 256 * 4, 8), 256, 0, st>>>(
          build_keys, n_build, j.ht, none);
    TDP_LAUNCH_CHECK("join_build_unique_kernel");
    // report a repeated key (int flag into the low half of out_info[1])
    TDP_CUDA_TRY(cudaMemcpyAsync(out_info + 1, j.ht.flags, sizeof(int), cudaMemcpyDeviceToDevice,
                                 st));
  } else {
    // flags[0] (keys repeat), flags[1] (runs mode): nonzero, no host source
    TDP_CUDA_TRY(cudaMemsetAsync(j.ht.flags, 1, 2 * sizeof(int), st));
    make_keys_kernel<<<stream_grid(n_build, 256 * 8, 8), 256, 0, st>>>(
        build_keys, TDP_I64, 0, n_build, j.sb.k0, j.sb.i0);
    TDP_LAUNCH_CHECK("make_keys_kernel");
    u64* sk;
    i64* order;
    rc = radix_sort(j.sb, n_build, st, &sk, &order);
    if (rc) return rc;
    if (sk != j.sb.k0) {  // keep the sorted result in the k0/i0 slots for tdp_join_emit
      TDP_CUDA_TRY(cudaMemcpyAsync(j.sb.k0, sk, (size_t)n_build * 8, cudaMemcpyDeviceToDevice, st));
      TDP_CUDA_TRY(cudaMemcpyAsync(j.sb.i0, order, (size_t)n_build * 8, cudaMemcpyDeviceToDevice, st));
    }
    join_build_runs_kernel<<<stream_grid(n_build, 256 * 4, 8), 256, 0, st>>>(j.sb.k0, n_build,
                                                                             j.ht);
    TDP_LAUNCH_CHECK("join_build_runs_kernel");
  }
  TDP_CUDA_TRY(cudaMemsetAsync(j.tile_counts, 0, (size_t)tiles * sizeof(i64), st));
  const bool filtered = ps != nullptr && ps->npreds > 0;
  const PredSet& pp = filtered ? *ps : none;
  const bool runs = mode == 1;
  auto kernel = filtered ? (runs ? join_count_kernel<true, false> : join_count_kernel<true, true>)
                         : (runs ? join_count_kernel<false, false> : join_count_kernel<false, true>);
  j.ht.ahead = join_ahead(runs ? 3 : 4);
  cudaEvent_t t0 = timer_begin(2, st);
  kernel<<<(unsigned)tiles, kJoinThreads, 0, st>>>(j.ht, probe_keys, n_probe, pp, j.match_bits,
                                                   j.word_counts, j.tile_counts);
  TDP_LAUNCH_CHECK("join_count_kernel");
  timer_end(t0, st);
  return exclusive_scan_i64(j.tile_counts, j.tile_offsets, tiles, out_info, j.scan_ws,
                            j.scan_bytes, st);
}

// Legacy single-call form: optimistic pass, one host check, runs if needed.
int join_prepare(const int64_t* build_keys, int64_t n_build, const int64_t* probe_keys,
                 int64_t n_probe, const PredSet* ps, int64_t* out_count, void* ws,
                 size_t ws_bytes, cudaStream_t st) {
  TDP_REQUIRE(out_count != nullptr, "null join count output");
  i64* info = nullptr;
  TDP_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&info), 2 * sizeof(i64), st));
  int rc = join_prepare_mode(build_keys, n_build, nullptr, probe_keys, n_probe, ps, 0, info, ws,
                             ws_bytes, st);
  i64 host[2] = {0, 0};
  if (!rc) {
    TDP_CUDA_TRY(cudaMemcpyAsync(host, info, sizeof(host), cudaMemcpyDeviceToHost, st));
    TDP_CUDA_TRY(cudaStreamSynchronize(st));
    if (host[1] & 0xffffffff)
      rc = join_prepare_mode(build_keys, n_build, nullptr, probe_keys, n_probe, ps, 1, info, ws,
                             ws_bytes, st);
  }
  if (!rc) TDP_CUDA_TRY(cudaMemcpyAsync(out_count, info, sizeof(i64), cudaMemcpyDeviceToDevice, st));
  cudaFreeAsync(info, st);
  return rc;
}

}  // namespace
}  // namespace tdp

extern "C" {

size_t tdp_join_workspace(int64_t n_build, int64_t n_probe) { return join_ws_bytes(n_build, n_probe); }

int tdp_join_prepare(const int64_t* build_keys, int64_t n_build, const int64_t* probe_keys,
                     int64_t n_probe, int64_t* out_count, void* ws, size_t ws_bytes,
                     void* stream) {
  return join_prepare(build_keys, n_build, probe_keys, n_probe, nullptr, out_count, ws, ws_bytes,
                      as_stream(stream));
}

int tdp_join_prepare_filtered(const int64_t* build_keys, int64_t n_build,
                              const int64_t* probe_keys, int64_t n_probe, const tdp_column* cols,
                              int32_t ncols, const tdp_predicate* preds, int32_t npreds,
                              int64_t* out_count, void* ws, size_t ws_bytes, void* stream) {
  PredSet ps;
  int rc = make_predset(cols, ncols, preds, npreds, n_probe, &ps);
  if (rc) return rc;
  return join_prepare(build_keys, n_build, probe_keys, n_probe, &ps, out_count, ws, ws_bytes,
                      as_stream(stream));
}

int tdp_join_prepare_ex(const int64_t* build_keys, int64_t n_build, const tdp_column* bcols,
                        int32_t nbcols, const tdp_predicate* bpreds, int32_t nbpreds,
                        const int64_t* probe_keys, int64_t n_probe, const tdp_column* pcols,
                        int32_t npcols, const tdp_predicate* ppreds, int32_t nppreds,
                        int32_t mode, int64_t* out_info, void* ws, size_t ws_bytes,
                        void* stream) {
  PredSet bps, pps;
  int rc = make_predset(bcols, nbcols, bpreds, nbpreds, n_build, &bps);
  if (rc) return rc;
  rc = make_predset(pcols, npcols, ppreds, nppreds, n_probe, &pps);
  if (rc) return rc;
  return join_prepare_mode(build_keys, n_build, &bps, probe_keys, n_probe, &pps, mode, out_info,
                           ws, ws_bytes, as_stream(stream));
}

int tdp_join_emit(const int64_t* probe_keys, int64_t n_build, int64_t n_probe,
                  int64_t* out_probe_idx, int64_t* out_build_idx, void* ws, size_t ws_bytes,
                  void* stream) {
  TDP_REQUIRE(ws_bytes >= join_ws_bytes(n_build, n_probe), "join workspace too small");
  if (n_build == 0 || n_probe == 0) return TDP_OK;
  cudaStream_t st = as_stream(stream);
  JoinWs j = carve_join(ws, n_build, n_probe);
  const i64 tiles = ceil_div(n_probe, kJoinTile);
  const unsigned grid = (unsigned)(tiles < (i64)sm_count() * 8 ? tiles : (i64)sm_count() * 8);
  join_emit_runs_kernel<<<grid, kJoinThreads, 0, st>>>(
      j.ht, probe_keys, tiles, j.match_bits, j.word_counts, j.tile_counts, j.tile_offsets,
      out_probe_idx, out_build_idx);
  TDP_LAUNCH_CHECK("join_emit_runs_kernel");
  join_expand_unique_kernel<<<(unsigned)ceil_div(tiles, kJoinWarps), kJoinThreads, 0, st>>>(
      j.ht, tiles, j.match_bits, j.word_counts, j.tile_counts, j.tile_offsets, out_probe_idx);
  TDP_LAUNCH_CHECK("join_expand_unique_kernel");
  join_pairs_unique_kernel<<<(unsigned)(sm_count() * 8), 256, 0, st>>>(
      j.ht, probe_keys, j.tile_counts, j.tile_offsets, tiles, out_probe_idx, out_build_idx);
  TDP_LAUNCH_CHECK("join_pairs_unique_kernel");
  return TDP_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// hash group-by for one high-cardinality int64 key (groupby_exact's general
// path, tq/kernels.py:108-167, when the key range is too wide for dense
// slots).  prepare: one pass inserts every row's key into an open-addressing
// table (CAS on the key image, INT64_MIN in a side slot) and adds its count /
// sums into the slot's accumulators with global atomics -- lanes of a warp
// holding the same key are combined first (__match_any_sync + shuffle sums),
// so a hot key costs one atomic per warp; occupied slots are then compacted
// into (key image, slot) pairs and counted.  emit: a stable radix sort of the
// m distinct keys (not of the n rows) and a gather of the accumulators, so
// groups come out in ascending key order as np.unique orders them.
// ---------------------------------------------------------------------------
namespace tdp {
namespace {

// A distinct key owns a *cell* (claimed on first insertion, zeroed by its
// claimer and then published through cidx): image, count, integer sums and
// the float SUMs' fixed-point words.  Only the key table (8 B per slot) and
// the cell indices (4 B) are cleared per call -- not a full set of per-slot
// accumulators -- and the m claimed cells are the groups directly.
struct HashAgg {
  u64* slot;                 // [cap]      key image (0 = empty)
  unsigned* cidx;            // [cap + 1]  published cell + 1; [cap]: INT64_MIN (image 0)
  unsigned long long* misc;  // [0] cells claimed (= groups m), [1] INT64_MIN claimed
  u64* cells;                // [ncap][cw]
  i64 ncap;
  int cw;                    // image, count, naggs sums, kFixedWords per float SUM
  int naggs;
  u64 mask;
  i64 cap;                   // power of two
};

constexpr int kCellImg = 0, kCellCnt = 1, kCellAcc = 2;

int cell_words(int naggs, int nfixed) { return kCellAcc + naggs + kFixedWords * nfixed; }

size_t hashagg_ws_bytes(i64 n, int naggs) {
  const i64 cap = (i64)table_capacity(n);
  const i64 ncap = n > 0 ? n : 1;
  const int na = naggs > 0 ? naggs : 0;
  return sort_ws_bytes(n) + align256((size_t)cap * 8) + align256((size_t)(cap + 1) * 4) + 256 +
         align256((size_t)ncap * cell_words(na, na) * 8) + 1024;
}

HashAgg carve_hashagg(void* ws, i64 n, const ValSet& vs) {
  HashAgg h;
  h.cap = (i64)table_capacity(n);
  h.mask = (u64)h.cap - 1;
  h.ncap = n > 0 ? n : 1;
  h.naggs = vs.naggs;
  h.cw = cell_words(vs.naggs, vs.nfixed);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws) + sort_ws_bytes(n);
  h.slot = (u64*)p;
  p += align256((size_t)h.cap * 8);
  h.cidx = (unsigned*)p;
  p += align256((size_t)(h.cap + 1) * 4);
  h.misc = (unsigned long long*)p;
  p += 256;
  h.cells = (u64*)p;
  return h;
}

template <class V>
__device__ __forceinline__ V group_sum(V v, unsigned peers, int lane) {
  // sum of v over the lanes in `peers` (lanes holding the same key): lane
  // order within the group is fixed (ascending), so the result is reproducible
  V total = 0;
  unsigned m = peers;
  while (m) {
    const int src = __ffs(m) - 1;
    total += __shfl_sync(peers, v, src);
    m &= m - 1;
  }
  (void)lane;
  return total;
}

// A new key's cell: zero it, then publish its index (release).
__device__ __forceinline__ void init_cell(const HashAgg& h, i64 id, u64 img, unsigned* pub) {
  u64* c = h.cells + id * h.cw;
  c[kCellImg] = img;
  for (int w = 1; w < h.cw; ++w) c[w] = 0ull;
  __threadfence();
  atomicExch(pub, (unsigned)(id + 1));
}

// A key another warp inserted: wait for its cell index (the claimer is
// running: it won the slot's CAS, and it is never in this warp -- a warp's
// lanes with one key are a single peer group with one leader).
__device__ __forceinline__ i64 wait_cell(const unsigned* pub) {
  unsigned v;
  while ((v = *(volatile const unsigned*)pub) == 0u) {
  }
  __threadfence();
  return (i64)v - 1;
}

__global__ void hashagg_kernel(const i64* __restrict__ keys, i64 n, HashAgg h, ValSet vs) {
  const int lane = threadIdx.x & 31;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 base = (i64)blockIdx.x * blockDim.x; base < n; base += stride) {
    const i64 i = base + threadIdx.x;
    const bool valid = i < n;
    const unsigned active = __ballot_sync(0xffffffffu, valid);
    if (!valid) continue;
    const i64 k = keys[i];
    const unsigned peers = __match_any_sync(active, k);
    const int leader = __ffs(peers) - 1;
    const u64 img = (u64)k ^ 0x8000000000000000ull;
    // the leader finds or inserts the key's slot ...
    unsigned* pub = nullptr;
    bool inserted = false;
    if (lane == leader) {
      if (img == 0ull) {
        pub = h.cidx + h.cap;
        inserted = atomicCAS(h.misc + 1, 0ull, 1ull) == 0ull;
      } else {
        u64 s = join_hash(k) & h.mask;
        unsigned long long* slots = reinterpret_cast<unsigned long long*>(h.slot);
        for (;;) {
          // a plain (L2) read first: a slot only ever goes 0 -> key, so a key
          // seen is final and only an empty slot needs the CAS (most rows of a
          // repeated key then do no atomic here)
          const unsigned long long cur = __ldcg(slots + s);
          if (cur == img) break;
          if (cur == 0ull) {
            const unsigned long long prev = atomicCAS(slots + s, 0ull, (unsigned long long)img);
            if (prev == 0ull || prev == img) {
              inserted = prev == 0ull;
              break;
            }
          }
          s = (s + 1) & h.mask;
        }
        pub = h.cidx + s;
      }
    }
    // ... the warp's new keys take consecutive cells with one counter atomic
    const unsigned claims = __ballot_sync(active, inserted);
    unsigned long long first = 0;
    if (claims) {
      const int src = __ffs(claims) - 1;
      if (lane == src) first = atomicAdd(h.misc, (unsigned long long)__popc(claims));
      first = __shfl_sync(active, first, src);
    }
    i64 cell = 0;
    if (inserted) {
      cell = (i64)first + __popc(claims & lanemask_lt());
      init_cell(h, cell, img, pub);
    } else if (lane == leader) {
      cell = wait_cell(pub);
    }
    cell = __shfl_sync(peers, cell, leader);
    unsigned long long* c = reinterpret_cast<unsigned long long*>(h.cells + cell * h.cw);
    if (lane == leader) atomicAdd(c + kCellCnt, (unsigned long long)__popc(peers));
    for (int a = 0; a < vs.naggs; ++a) {
      if (vs.kind[a] == TDP_AGG_COUNT) continue;
      if (vs.kind[a] == TDP_AGG_SUM_F64) {
        // the peers' sum in fixed lane order, then order-free integer words
        const double v = group_sum(load_as_f64(vs.p[a], vs.dt[a], i), peers, lane);
        if (lane == leader) fixed_add(c + kCellAcc + vs.naggs + kFixedWords * vs.fidx[a], v);
      } else {
        const unsigned long long v =
            group_sum((unsigned long long)load_as_i64(vs.p[a], vs.dt[a], i), peers, lane);
        if (lane == leader) atomicAdd(c + kCellAcc + a, v);
      }
    }
  }
}

// Per claimed cell: float SUMs -> double bits in the cell's sum word; the key
// image and cell id into the sort input; the images' [min, max] into range.
__global__ void hashagg_cells_kernel(HashAgg h, ValSet vs, u64* __restrict__ out_img,
                                     i64* __restrict__ out_cell,
                                     unsigned long long* __restrict__ range) {
  const i64 m = (i64)h.misc[0];
  unsigned long long lo = ~0ull, hi = 0ull;
  for (i64 id = (i64)blockIdx.x * blockDim.x + threadIdx.x; id < m;
       id += (i64)gridDim.x * blockDim.x) {
    unsigned long long* c = reinterpret_cast<unsigned long long*>(h.cells + id * h.cw);
    for (int a = 0; a < vs.naggs; ++a)
      if (vs.kind[a] == TDP_AGG_SUM_F64)
        c[kCellAcc + a] = (unsigned long long)__double_as_longlong(
            fixed_value(c + kCellAcc + vs.naggs + kFixedWords * vs.fidx[a]));
    const u64 img = c[kCellImg];  // key images sort like the keys
    out_img[id] = img;
    out_cell[id] = id;
    lo = img < lo ? img : lo;
    hi = img > hi ? img : hi;
  }
  if (range == nullptr) return;
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    const unsigned long long h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
  }
  if ((threadIdx.x & 31) == 0 && lo <= hi) {
    atomicMin(range + 1, lo);
    atomicMax(range + 2, hi);
  }
}

__global__ void info_init_kernel(unsigned long long* info) {
  info[1] = ~0ull;
  info[2] = 0ull;
}

// Rank of each distinct key by a bitmap over its range (instead of a radix
// sort of the m keys: a handful of bandwidth-bound passes over range/8 bytes
// rather than four latency-bound sort passes).
__global__ void rank_bits_kernel(const u64* __restrict__ img, i64 m, u64 lo,
                                 unsigned* __restrict__ bits) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (i64)gridDim.x * blockDim.x) {
    const u64 d = img[i] - lo;
    atomicOr(bits + (d >> 5), 1u << (d & 31));
  }
}

// One warp per 1024-bit block of the bitmap: its population, and per word
// the set bits of the block's earlier words (u16, <= 992).
__global__ void rank_popc_kernel(const unsigned* __restrict__ bits, i64 words, i64 blocks,
                                 i64* __restrict__ counts, unsigned short* __restrict__ wpre) {
  const int lane = threadIdx.x & 31;
  const i64 warps = (i64)gridDim.x * (blockDim.x >> 5);
  for (i64 blk = (i64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); blk < blocks;
       blk += warps) {
    const i64 w = blk * 32 + lane;
    const int c = w < words ? __popc(bits[w]) : 0;
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (w < words) wpre[w] = (unsigned short)(incl - c);
    if (lane == 31) counts[blk] = incl;
  }
}

// rank = keys in earlier blocks + earlier words of the block + bits below
__global__ void rank_place_kernel(const u64* __restrict__ img, const i64* __restrict__ slot, i64 m,
                                  u64 lo, const unsigned* __restrict__ bits,
                                  const unsigned short* __restrict__ wpre,
                                  const i64* __restrict__ offs, u64* __restrict__ img_out,
                                  i64* __restrict__ slot_out) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (i64)gridDim.x * blockDim.x) {
    const u64 d = img[i] - lo;
    const i64 word = (i64)(d >> 5);
    const i64 r = offs[d >> 10] + wpre[word] + __popc(bits[word] & ((1u << (d & 31)) - 1u));
    img_out[r] = img[i];
    slot_out[r] = slot[i];
  }
}

i64 rank_words(i64 range) { return (range + 31) / 32; }
i64 rank_blocks(i64 range) { return (range + 1023) / 1024; }

size_t rank_ws_bytes(i64 range) {
  const i64 r = range > 0 ? range : 1;
  const i64 b = rank_blocks(r);
  return align256((size_t)rank_words(r) * 4) + align256((size_t)rank_words(r) * 2) +
         2 * align256((size_t)b * 8) + exclusive_scan_workspace(b) + 1024;
}

__global__ void hashagg_gather_kernel(HashAgg h, const u64* __restrict__ img,
                                      const i64* __restrict__ cell, i64 m, ValSet vs,
                                      i64* __restrict__ out_keys, i64* __restrict__ out_counts,
                                      u64* __restrict__ out_sums) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (i64)gridDim.x * blockDim.x) {
    const u64* c = h.cells + cell[i] * h.cw;
    out_keys[i] = (i64)(img[i] ^ 0x8000000000000000ull);
    const u64 cnt = c[kCellCnt];
    out_counts[i] = (i64)cnt;
    for (int a = 0; a < vs.naggs; ++a)
      out_sums[(i64)a * m + i] =
          vs.kind[a] == TDP_AGG_COUNT ? cnt : emit_value(vs, a, c[kCellAcc + a], cnt);
  }
}

int make_valset(const tdp_column* vals, const int32_t* agg_kinds, int32_t naggs, i64 n,
                ValSet* vs) {
  TDP_REQUIRE(naggs >= 0 && naggs <= 32, "at most 32 aggregates");
  std::memset(vs, 0, sizeof(*vs));
  vs->naggs = naggs;
  for (int a = 0; a < naggs; ++a) {
    vs->kind[a] = agg_kinds[a];
    TDP_REQUIRE(agg_kinds[a] >= TDP_AGG_COUNT && agg_kinds[a] <= TDP_AGG_SUM_I64,
                "agg %d: bad kind", a);
    if (agg_kinds[a] == TDP_AGG_COUNT) {
      vs->dt[a] = TDP_I64;
      continue;
    }
    TDP_REQUIRE(vals != nullptr && vals[a].rows >= n && vals[a].width == 1,
                "agg %d: value column must be scalar with >= n rows", a);
    vs->p[a] = vals[a].data;
    vs->dt[a] = vals[a].dtype;
  }
  number_fixed(vs);
  return TDP_OK;
}

}  // namespace
}  // namespace tdp

extern "C" {

size_t tdp_groupby_hash_workspace(int64_t n, int32_t naggs) { return hashagg_ws_bytes(n, naggs); }

static int hash_prepare(const int64_t* keys, int64_t n, const tdp_column* vals,
                        const int32_t* agg_kinds, int32_t naggs, int64_t* out_ngroups,
                        void* ws, size_t ws_bytes, void* stream, unsigned long long* range);

int tdp_groupby_hash_prepare(const int64_t* keys, int64_t n, const tdp_column* vals,
                             const int32_t* agg_kinds, int32_t naggs, int64_t* out_ngroups,
                             void* ws, size_t ws_bytes, void* stream) {
  return hash_prepare(keys, n, vals, agg_kinds, naggs, out_ngroups, ws, ws_bytes, stream, nullptr);
}

static int hash_prepare(const int64_t* keys, int64_t n, const tdp_column* vals,
                        const int32_t* agg_kinds, int32_t naggs, int64_t* out_ngroups,
                        void* ws, size_t ws_bytes, void* stream, unsigned long long* range) {
  TDP_REQUIRE(n >= 0 && out_ngroups != nullptr, "bad hash group-by arguments");
  TDP_REQUIRE(ws_bytes >= hashagg_ws_bytes(n, naggs), "hash group-by workspace too small");
  ValSet vs;
  int rc = make_valset(vals, agg_kinds, naggs, n, &vs);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    TDP_CUDA_TRY(cudaMemsetAsync(out_ngroups, 0, 8, st));
    return TDP_OK;
  }
  HashAgg h = carve_hashagg(ws, n, vs);
  TDP_CUDA_TRY(cudaMemsetAsync(h.slot, 0, (size_t)h.cap * 8, st));
  TDP_CUDA_TRY(cudaMemsetAsync(h.cidx, 0, (size_t)(h.cap + 1) * 4, st));
  TDP_CUDA_TRY(cudaMemsetAsync(h.misc, 0, 16, st));
  // one row per thread: the pass is latency-bound (CAS, dependent atomics of the
  // fixed-point cells), so keep every row's chain in flight at once
  hashagg_kernel<<<stream_grid(n, 256, 32), 256, 0, st>>>(keys, n, h, vs);
  TDP_LAUNCH_CHECK("hashagg_kernel");
  SortBuffers b = carve(ws, n);
  hashagg_cells_kernel<<<stream_grid(n, 256, 32), 256, 0, st>>>(h, vs, b.k0, b.i0, range);
  TDP_LAUNCH_CHECK("hashagg_cells_kernel");
  TDP_CUDA_TRY(cudaMemcpyAsync(out_ngroups, h.misc, 8, cudaMemcpyDeviceToDevice, st));
  return TDP_OK;
}

int tdp_groupby_hash_prepare_ex(const int64_t* keys, int64_t n, const tdp_column* vals,
                                const int32_t* agg_kinds, int32_t naggs, int64_t* out_info,
                                void* ws, size_t ws_bytes, void* stream) {
  TDP_REQUIRE(out_info != nullptr, "null group-by info output");
  unsigned long long* info = reinterpret_cast<unsigned long long*>(out_info);
  info_init_kernel<<<1, 1, 0, as_stream(stream)>>>(info);
  TDP_LAUNCH_CHECK("info_init_kernel");
  return hash_prepare(keys, n, vals, agg_kinds, naggs, out_info, ws, ws_bytes, stream, info);
}

size_t tdp_groupby_hash_rank_workspace(int64_t key_range) { return rank_ws_bytes(key_range); }

int tdp_groupby_hash_emit_ranked(int64_t n, const int32_t* agg_kinds, int32_t naggs, int64_t m,
                                 int64_t min_key, int64_t key_range, int64_t* out_keys,
                                 int64_t* out_counts, void* out_sums, void* ws, size_t ws_bytes,
                                 void* rank_ws, size_t rank_ws_bytes_, void* stream) {
  TDP_REQUIRE(m >= 0 && m <= (n > 0 ? n : 0), "bad group count");
  TDP_REQUIRE(ws_bytes >= hashagg_ws_bytes(n, naggs), "hash group-by workspace too small");
  TDP_REQUIRE(m == 0 || (key_range >= m && key_range <= ((int64_t)1 << 36)),
              "key range %lld cannot hold %lld distinct keys", (long long)key_range, (long long)m);
  TDP_REQUIRE(m == 0 || rank_ws_bytes_ >= rank_ws_bytes(key_range), "rank workspace too small");
  if (m == 0) return TDP_OK;
  ValSet vs;
  int rc = emit_kinds(agg_kinds, naggs, &vs);  // kinds only (+ AVG bits)
  if (rc) return rc;
  number_fixed(&vs);
  cudaStream_t st = as_stream(stream);
  HashAgg h = carve_hashagg(ws, n, vs);
  SortBuffers b = carve(ws, n);
  const i64 words = rank_words(key_range), blocks = rank_blocks(key_range);
  unsigned char* p = reinterpret_cast<unsigned char*>(rank_ws);
  unsigned* bits = (unsigned*)p;
  p += align256((size_t)words * 4);
  unsigned short* wpre = (unsigned short*)p;
  p += align256((size_t)words * 2);
  i64* counts = (i64*)p;
  p += align256((size_t)blocks * 8);
  i64* offs = (i64*)p;
  p += align256((size_t)blocks * 8);
  const u64 lo = (u64)min_key ^ 0x8000000000000000ull;
  TDP_CUDA_TRY(cudaMemsetAsync(bits, 0, (size_t)words * 4, st));
  rank_bits_kernel<<<stream_grid(m, 256 * 4, 8), 256, 0, st>>>(b.k0, m, lo, bits);
  TDP_LAUNCH_CHECK("rank_bits_kernel");
  rank_popc_kernel<<<stream_grid(blocks, 8, 8), 256, 0, st>>>(bits, words, blocks, counts, wpre);
  TDP_LAUNCH_CHECK("rank_popc_kernel");
  rc = exclusive_scan_i64(counts, offs, blocks, nullptr, p, exclusive_scan_workspace(blocks) + 512,
                          st);
  if (rc) return rc;
  rank_place_kernel<<<stream_grid(m, 256 * 4, 8), 256, 0, st>>>(b.k0, b.i0, m, lo, bits, wpre,
                                                                  offs, b.k1, b.i1);
  TDP_LAUNCH_CHECK("rank_place_kernel");
  hashagg_gather_kernel<<<stream_grid(m, 256 * 4, 8), 256, 0, st>>>(
      h, b.k1, b.i1, m, vs, out_keys, out_counts, reinterpret_cast<u64*>(out_sums));
  TDP_LAUNCH_CHECK("hashagg_gather_kernel");
  return TDP_OK;
}

int tdp_groupby_hash_emit(int64_t n, const int32_t* agg_kinds, int32_t naggs, int64_t m,
                          int64_t* out_keys, int64_t* out_counts, void* out_sums, void* ws,
                          size_t ws_bytes, void* stream) {
  TDP_REQUIRE(m >= 0 && m <= (n > 0 ? n : 0), "bad group count");
  TDP_REQUIRE(ws_bytes >= hashagg_ws_bytes(n, naggs), "hash group-by workspace too small");
  if (m == 0) return TDP_OK;
  ValSet vs;
  int rc = emit_kinds(agg_kinds, naggs, &vs);  // kinds only (+ AVG bits)
  if (rc) return rc;
  number_fixed(&vs);
  cudaStream_t st = as_stream(stream);
  HashAgg h = carve_hashagg(ws, n, vs);
  SortBuffers b = carve(ws, n);
  u64* sk;
  i64* order;
  rc = radix_sort(b, m, st, &sk, &order);
  if (rc) return rc;
  hashagg_gather_kernel<<<stream_grid(m, 256 * 4, 8), 256, 0, st>>>(
      h, sk, order, m, vs, out_keys, out_counts, reinterpret_cast<u64*>(out_sums));
  TDP_LAUNCH_CHECK("hashagg_gather_kernel");
  return TDP_OK;
}

}  // extern "C"


// ---------------------------------------------------------------------------
// Dense-range equi-join (unique build keys within a known range [lo, lo+R)):
// the build sets one bit per key in a bitmap of R bits (atomicOr; a bit seen
// twice = repeated key -> the caller falls back to the hash join), the probe
// tests one bit per row -- no hashing, no Bloom filter, no slot compare, and
// no false positives.  A build row is found again by its key's rank among the
// set bits (per-1024-bit block offsets + per-word u16 prefixes, the bitmap
// rank of the hash group-by), and rank order is ascending key order.  Used
// when R is small next to the build (TPC-H keys: c_custkey R = rows, o_orderkey
// R = 4 x rows); the bitmap (R/8 bytes) and rank words stay L2-resident.
// ---------------------------------------------------------------------------
namespace tdp {
namespace {

struct DenseJoin {
  unsigned* bits;        // [words]
  unsigned short* wpre;  // [words]  set bits of the block's earlier words
  i64* bcount;           // [blocks]
  i64* boffs;            // [blocks]  set bits of earlier blocks
  i64* rank_row;         // [nb]      build row of each rank (need_rows, rank mode)
  int* row_of;           // [R]       build row of each key offset (need_rows, direct mode)
  int* flags;            // [0] repeated key, [1] key outside [lo, lo+R), [2] zero (expand)
  u64 lo;
  i64 range;
  // [0] build rows set, [1] set bits, [2] CTAs done (dense_dup_check_kernel);
  // null: repeats are detected from the atomics' return values instead
  unsigned long long* cnt;
  // tiles ahead of its own whose columns a build / probe CTA prefetches into
  // L2 (about one wave of resident CTAs; 0: none)
  i64 ahead;
};


// Build rows by key offset in a plain int32 array of R entries (no clearing:
// only offsets whose bit is set are read) while R <= 8 x the build rows;
// beyond, by rank among the set bits.
inline bool dense_direct(i64 range, i64 nb) {
  return range <= 8 * (nb > (1 << 20) ? nb : (1 << 20)) && nb < ((i64)1 << 31);
}

__device__ __forceinline__ i64 dense_rank(const DenseJoin& dj, u64 d) {
  const i64 w = (i64)(d >> 5);
  return dj.boffs[d >> 10] + dj.wpre[w] + __popc(dj.bits[w] & ((1u << (d & 31)) - 1u));
}

// Build pass, tiled like the probe (kJoinPer rows per thread, their
// predicate loads batched): a filtered build reads its predicate columns
// once per row with R independent loads in flight.
constexpr int kBuildThreads = 512, kBuildPer = kJoinTile / kBuildThreads;

template <bool kFiltered>
__global__ void __launch_bounds__(kBuildThreads, 2)
    dense_build_kernel(const i64* __restrict__ keys, i64 nb, DenseJoin dj, PredSet bps) {
  const i64 tile = blockIdx.x;
  join_prefetch_ahead(dj.ahead, tile, keys, nb, bps, kFiltered);
  bool act[kBuildPer];
  i64 row[kBuildPer], key[kBuildPer];
#pragma unroll
  for (int k = 0; k < kBuildPer; ++k) {
    row[k] = tile * kJoinTile + (i64)k * kBuildThreads + threadIdx.x;
    act[k] = row[k] < nb;
  }
  // keys with the predicate columns: one round of independent loads (a
  // selective build filter still touches most key sectors)
#pragma unroll
  for (int k = 0; k < kBuildPer; ++k) key[k] = act[k] ? __ldg(keys + row[k]) : 0;
  if (kFiltered) eval_batch_upfront<kBuildPer>(bps, row, act);
  unsigned built = 0;
#pragma unroll
  for (int k = 0; k < kBuildPer; ++k) {
    if (!act[k]) continue;
    const u64 x = (u64)key[k] - dj.lo;
    if (x >= (u64)dj.range) {
      dj.flags[1] = 1;
      continue;
    }
    const unsigned bit = 1u << (x & 31);
    if (dj.cnt != nullptr) {
      // fire-and-forget OR (the CTA does not wait for L2): a repeated key
      // shows as fewer set bits than rows set (dense_dup_check_kernel)
      atomicOr(dj.bits + (x >> 5), bit);
      ++built;
    } else if (atomicOr(dj.bits + (x >> 5), bit) & bit) {
      dj.flags[0] = 1;
    }
    if (dj.row_of != nullptr) dj.row_of[x] = (int)row[k];
  }
  if (dj.cnt != nullptr) {  // one global atomic per CTA (a single counter: avoid contention)
    __shared__ unsigned cta_built;
    if (threadIdx.x == 0) cta_built = 0;
    __syncthreads();
    const unsigned w = warp_sum(built);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(&cta_built, w);
    __syncthreads();
    if (threadIdx.x == 0 && cta_built) atomicAdd(dj.cnt, (unsigned long long)cta_built);
  }
}

// After the build: set bits vs rows set -> flags[0] (a repeated key).  The
// last CTA to finish compares (order-free integer sums).
__global__ void dense_dup_check_kernel(DenseJoin dj, i64 words) {
  __shared__ unsigned long long part[32];
  unsigned long long s = 0;
  for (i64 w = (i64)blockIdx.x * blockDim.x + threadIdx.x; w < words;
       w += (i64)gridDim.x * blockDim.x)
    s += __popc(dj.bits[w]);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += part[k];
    atomicAdd(dj.cnt + 1, t);
    __threadfence();
    if (atomicAdd(dj.cnt + 2, 1ull) == gridDim.x - 1) {
      __threadfence();
      const unsigned long long set = atomicAdd(dj.cnt + 1, 0ull);
      if (set != atomicAdd(dj.cnt, 0ull)) dj.flags[0] = 1;
    }
  }
}

template <bool kFiltered>
__global__ void dense_place_kernel(const i64* __restrict__ keys, i64 nb, DenseJoin dj,
                                   PredSet bps) {
  if (dj.flags[0] | dj.flags[1]) return;  // falls back to the hash join
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (i64)gridDim.x * blockDim.x) {
    if (kFiltered && !eval_all(bps, i)) continue;
    dj.rank_row[dense_rank(dj, (u64)__ldg(keys + i) - dj.lo)] = i;
  }
}

// Probe pass: the tile / word layout of join_count_kernel (so the unique-key
// expansion is shared), one bitmap word per row instead of Bloom + slot.
template <bool kFiltered>
__global__ void __launch_bounds__(kJoinThreads, 4)
    dense_count_kernel(DenseJoin dj, const i64* __restrict__ probe, i64 np, PredSet ps,
                       unsigned* __restrict__ match_bits, i64* __restrict__ word_counts,
                       i64* __restrict__ tile_counts) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 tile = blockIdx.x;
  join_prefetch_ahead(dj.ahead, tile, probe, np, ps, kFiltered);
  bool act[kJoinPer];
  i64 row[kJoinPer], key[kJoinPer];
#pragma unroll
  for (int k = 0; k < kJoinPer; ++k) {
    row[k] = join_row(tile, k);
    act[k] = row[k] < np;
  }
#pragma unroll
  for (int k = 0; k < kJoinPer; ++k) key[k] = act[k] ? __ldcs(probe + row[k]) : 0;
  if (kFiltered) eval_batch<kJoinPer>(ps, row, act);
  unsigned w[kJoinPer];
  u64 d[kJoinPer];
#pragma unroll
  for (int k = 0; k < kJoinPer; ++k) {
    d[k] = (u64)key[k] - dj.lo;
    act[k] = act[k] && d[k] < (u64)dj.range;
    w[k] = act[k] ? __ldg(dj.bits + (d[k] >> 5)) : 0u;
  }
  i64 local = 0;
#pragma unroll
  for (int k = 0; k < kJoinPer; ++k) {
    const bool hit = act[k] && ((w[k] >> (d[k] & 31)) & 1u);
    const unsigned word = __ballot_sync(0xffffffffu, hit);
    const i64 wc = (i64)__popc(word);
    if (lane == 0) {
      match_bits[tile * kJoinWords + k * kJoinWarps + warp] = word;
      word_counts[tile * kJoinWords + k * kJoinWarps + warp] = wc;
    }
    local += wc;
  }
  if (lane == 0 && local != 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(tile_counts + tile), (unsigned long long)local);
}

// Expansion of the match words (join_expand_unique_kernel's layout) that also
// writes each pair's build row: the probe keys of up to four matches are
// loaded together, then their build rows -- one launch instead of expand +
// dense_pairs_kernel (a selective probe has few matches per lane).
__global__ void dense_expand_pairs_kernel(DenseJoin dj, const i64* __restrict__ probe, i64 tiles,
                                          const unsigned* __restrict__ match_bits,
                                          const i64* __restrict__ word_counts,
                                          const i64* __restrict__ tile_counts,
                                          const i64* __restrict__ tile_offsets,
                                          i64* __restrict__ out_probe,
                                          i64* __restrict__ out_build) {
  const int lane = threadIdx.x & 31;
  const i64 tile = (i64)blockIdx.x * kJoinWarps + (threadIdx.x >> 5);
  if (tile >= tiles || tile_counts[tile] == 0) return;  // warp-uniform
  const i64* wc = word_counts + tile * kJoinWords;
  const unsigned* mb = match_bits + tile * kJoinWords;
  const i64 w0 = wc[2 * lane], w1 = wc[2 * lane + 1];
  u64 bits = (u64)mb[2 * lane] | ((u64)mb[2 * lane + 1] << 32);
  i64 incl = w0 + w1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const i64 t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  i64 pos = tile_offsets[tile] + incl - w0 - w1;
  const i64 row0 = tile * kJoinTile + (i64)lane * 64;
  while (bits) {
    i64 r[4], key[4];
    int c = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      r[u] = row0 + (bits ? __ffsll((long long)bits) - 1 : 0);
      c += bits ? 1 : 0;
      bits &= bits - 1;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) key[u] = u < c ? __ldg(probe + r[u]) : 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u >= c) break;
      const u64 d = (u64)key[u] - dj.lo;
      out_probe[pos + u] = r[u];
      out_build[pos + u] = dj.row_of != nullptr ? (i64)dj.row_of[d] : dj.rank_row[dense_rank(dj, d)];
    }
    pos += c;
  }
}

struct DenseWs {
  DenseJoin dj;
  unsigned* match_bits;
  i64* word_counts;
  i64* tile_counts;
  i64* tile_offsets;
  void* scan_ws;
  size_t scan_bytes;
  void* bscan_ws;
  size_t bscan_bytes;
};

size_t dense_ws_bytes(i64 range, i64 nb, i64 np) {
  const i64 r = range > 0 ? range : 1;
  const i64 words = rank_words(r), blocks = rank_blocks(r);
  const i64 tiles = ceil_div(np > 0 ? np : 1, kJoinTile);
  return align256((size_t)words * 4) + align256((size_t)words * 2) + 2 * align256((size_t)blocks * 8) +
         align256((size_t)(nb > 0 ? nb : 1) * 8) + (dense_direct(r, nb) ? align256((size_t)r * 4) : 0) +
         256 + align256((size_t)tiles * kJoinWords * 4) +
         align256((size_t)tiles * kJoinWords * 8) + 2 * align256((size_t)tiles * 8) +
         exclusive_scan_workspace(tiles) + exclusive_scan_workspace(blocks) + 4096;
}

DenseWs carve_dense(void* ws, i64 range, i64 lo, i64 nb, i64 np, bool need_rows) {
  DenseWs w;
  const i64 r = range > 0 ? range : 1;
  const i64 words = rank_words(r), blocks = rank_blocks(r);
  const i64 tiles = ceil_div(np > 0 ? np : 1, kJoinTile);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  w.dj.bits = (unsigned*)p;
  p += align256((size_t)words * 4);
  w.dj.wpre = (unsigned short*)p;
  p += align256((size_t)words * 2);
  w.dj.bcount = (i64*)p;
  p += align256((size_t)blocks * 8);
  w.dj.boffs = (i64*)p;
  p += align256((size_t)blocks * 8);
  w.dj.rank_row = (i64*)p;
  p += align256((size_t)(nb > 0 ? nb : 1) * 8);
  w.dj.row_of = nullptr;
  if (dense_direct(r, nb)) {
    if (need_rows) w.dj.row_of = (int*)p;
    p += align256((size_t)r * 4);
  }
  w.dj.flags = (int*)p;
  w.dj.cnt = reinterpret_cast<unsigned long long*>(p + 32);
  p += 256;
  w.dj.lo = (u64)lo;
  w.dj.ahead = 0;
  w.dj.range = r;
  w.match_bits = (unsigned*)p;
  p += align256((size_t)tiles * kJoinWords * 4);
  w.word_counts = (i64*)p;
  p += align256((size_t)tiles * kJoinWords * 8);
  w.tile_counts = (i64*)p;
  p += align256((size_t)tiles * 8);
  w.tile_offsets = (i64*)p;
  p += align256((size_t)tiles * 8);
  w.scan_ws = p;
  w.scan_bytes = exclusive_scan_workspace(tiles);
  p += exclusive_scan_workspace(tiles);
  w.bscan_ws = p;
  w.bscan_bytes = exclusive_scan_workspace(blocks) + 1024;
  return w;
}

}  // namespace
}  // namespace tdp

extern "C" {

size_t tdp_join_dense_workspace(int64_t key_range, int64_t n_build, int64_t n_probe) {
  return dense_ws_bytes(key_range, n_build, n_probe);
}

int tdp_join_dense_prepare(const int64_t* build_keys, int64_t n_build, const tdp_column* bcols,
                           int32_t nbcols, const tdp_predicate* bpreds, int32_t nbpreds,
                           const int64_t* probe_keys, int64_t n_probe, const tdp_column* pcols,
                           int32_t npcols, const tdp_predicate* ppreds, int32_t nppreds,
                           int64_t lo, int64_t key_range, int32_t need_rows, int64_t* out_info,
                           void* ws, size_t ws_bytes, void* stream) {
  TDP_REQUIRE(n_build >= 0 && n_probe >= 0, "negative join sizes");
  TDP_REQUIRE(out_info != nullptr, "null join info output");
  TDP_REQUIRE(key_range >= 1 && key_range <= ((int64_t)1 << 34),
              "dense join key range %lld outside [1, 2^34]", (long long)key_range);
  TDP_REQUIRE(ws_bytes >= dense_ws_bytes(key_range, n_build, n_probe), "join workspace too small");
  PredSet bps, pps;
  int rc = make_predset(bcols, nbcols, bpreds, nbpreds, n_build, &bps);
  if (rc) return rc;
  rc = make_predset(pcols, npcols, ppreds, nppreds, n_probe, &pps);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  DenseWs w = carve_dense(ws, key_range, lo, n_build, n_probe, need_rows != 0);
  const i64 tiles = ceil_div(n_probe, kJoinTile);
  const i64 words = rank_words(key_range), blocks = rank_blocks(key_range);
  TDP_CUDA_TRY(cudaMemsetAsync(out_info, 0, 2 * sizeof(i64), st));
  if (n_build == 0 || n_probe == 0) return TDP_OK;
  TDP_CUDA_TRY(cudaMemsetAsync(w.dj.bits, 0, (size_t)words * 4, st));
  TDP_CUDA_TRY(cudaMemsetAsync(w.dj.flags, 0, 64, st));  // flags + the dup-check counters
  TDP_CUDA_TRY(cudaMemsetAsync(w.tile_counts, 0, (size_t)tiles * sizeof(i64), st));
  const bool bfilt = bps.npreds > 0, pfilt = pps.npreds > 0;
  const unsigned btiles = (unsigned)ceil_div(n_build, kJoinTile);
  w.dj.ahead = join_ahead(2);
  if (bfilt)
    dense_build_kernel<true><<<btiles, kBuildThreads, 0, st>>>(build_keys, n_build, w.dj, bps);
  else
    dense_build_kernel<false><<<btiles, kBuildThreads, 0, st>>>(build_keys, n_build, w.dj, bps);
  TDP_LAUNCH_CHECK("dense_build_kernel");
  dense_dup_check_kernel<<<stream_grid(words, 256 * 8, 4), 256, 0, st>>>(w.dj, words);
  TDP_LAUNCH_CHECK("dense_dup_check_kernel");
  if (need_rows && w.dj.row_of == nullptr) {
    rank_popc_kernel<<<stream_grid(blocks, 8, 8), 256, 0, st>>>(w.dj.bits, words, blocks,
                                                                 w.dj.bcount, w.dj.wpre);
    TDP_LAUNCH_CHECK("rank_popc_kernel");
    rc = exclusive_scan_i64(w.dj.bcount, w.dj.boffs, blocks, nullptr, w.bscan_ws, w.bscan_bytes, st);
    if (rc) return rc;
    if (bfilt)
      dense_place_kernel<true><<<stream_grid(n_build, 256 * 4, 8), 256, 0, st>>>(
          build_keys, n_build, w.dj, bps);
    else
      dense_place_kernel<false><<<stream_grid(n_build, 256 * 4, 8), 256, 0, st>>>(
          build_keys, n_build, w.dj, bps);
    TDP_LAUNCH_CHECK("dense_place_kernel");
  }
  // out_info[1] = repeated key | key outside the range (two ints): fall back
  TDP_CUDA_TRY(cudaMemcpyAsync(out_info + 1, w.dj.flags, 2 * sizeof(int), cudaMemcpyDeviceToDevice,
                               st));
  auto kernel = pfilt ? dense_count_kernel<true> : dense_count_kernel<false>;
  w.dj.ahead = join_ahead(4);
  cudaEvent_t t0 = timer_begin(2, st);
  kernel<<<(unsigned)tiles, kJoinThreads, 0, st>>>(w.dj, probe_keys, n_probe, pps, w.match_bits,
                                                   w.word_counts, w.tile_counts);
  TDP_LAUNCH_CHECK("dense_count_kernel");
  timer_end(t0, st);
  return exclusive_scan_i64(w.tile_counts, w.tile_offsets, tiles, out_info, w.scan_ws,
                            w.scan_bytes, st);
}

int tdp_join_dense_bitmap(const int64_t* build_keys, int64_t n_build, const tdp_column* bcols,
                          int32_t nbcols, const tdp_predicate* bpreds, int32_t nbpreds, int64_t lo,
                          int64_t key_range, uint32_t* out_bits, int32_t* out_flags, void* stream) {
  TDP_REQUIRE(n_build >= 0 && out_bits != nullptr && out_flags != nullptr, "bad bitmap arguments");
  TDP_REQUIRE(key_range >= 1 && key_range <= ((int64_t)1 << 34),
              "dense join key range %lld outside [1, 2^34]", (long long)key_range);
  PredSet bps;
  int rc = make_predset(bcols, nbcols, bpreds, nbpreds, n_build, &bps);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  TDP_CUDA_TRY(cudaMemsetAsync(out_bits, 0, (size_t)rank_words(key_range) * 4, st));
  TDP_CUDA_TRY(cudaMemsetAsync(out_flags, 0, 2 * sizeof(int32_t), st));
  if (n_build == 0) return TDP_OK;
  DenseJoin dj;
  std::memset(&dj, 0, sizeof(dj));
  dj.bits = out_bits;
  dj.flags = out_flags;
  dj.lo = (u64)lo;
  dj.range = key_range;
  dj.ahead = join_ahead(2);
  const unsigned btiles = (unsigned)ceil_div(n_build, kJoinTile);
  if (bps.npreds > 0)
    dense_build_kernel<true><<<btiles, kBuildThreads, 0, st>>>(build_keys, n_build, dj, bps);
  else
    dense_build_kernel<false><<<btiles, kBuildThreads, 0, st>>>(build_keys, n_build, dj, bps);
  TDP_LAUNCH_CHECK("dense_build_kernel");
  return TDP_OK;
}

int tdp_join_dense_emit(const int64_t* probe_keys, int64_t n_build, int64_t n_probe, int64_t lo,
                        int64_t key_range, int32_t need_rows, int64_t* out_probe_idx,
                        int64_t* out_build_idx, void* ws, size_t ws_bytes, void* stream) {
  TDP_REQUIRE(ws_bytes >= dense_ws_bytes(key_range, n_build, n_probe), "join workspace too small");
  TDP_REQUIRE(!need_rows || out_build_idx != nullptr, "null build row output");
  if (n_build == 0 || n_probe == 0) return TDP_OK;
  cudaStream_t st = as_stream(stream);
  DenseWs w = carve_dense(ws, key_range, lo, n_build, n_probe, need_rows != 0);
  const i64 tiles = ceil_div(n_probe, kJoinTile);
  HashTable none;  // the expansion only reads flags[1] (runs mode): the zero flag
  std::memset(&none, 0, sizeof(none));
  none.flags = w.dj.flags + 2;
  if (need_rows) {
    dense_expand_pairs_kernel<<<(unsigned)ceil_div(tiles, kJoinWarps), kJoinThreads, 0, st>>>(
        w.dj, probe_keys, tiles, w.match_bits, w.word_counts, w.tile_counts, w.tile_offsets,
        out_probe_idx, out_build_idx);
    TDP_LAUNCH_CHECK("dense_expand_pairs_kernel");
    return TDP_OK;
  }
  join_expand_unique_kernel<<<(unsigned)ceil_div(tiles, kJoinWarps), kJoinThreads, 0, st>>>(
      none, tiles, w.match_bits, w.word_counts, w.tile_counts, w.tile_offsets, out_probe_idx);
  TDP_LAUNCH_CHECK("join_expand_unique_kernel");
  return TDP_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Bitmap group-by: one int64 key whose range R (from the scan's min/max) is at
// most ~1024 values per row.  The distinct keys are the set bits of an R-bit
// map, their rank among the set bits is the group id in ascending key order
// (np.unique's order, tq/kernels.py:128-136), so rows accumulate straight
// into dense cells [0, m) -- no hash table, no CAS chains, no sort of the
// distinct keys.  Passes: set bits (rows) -> popcount prefix (R/32 words) ->
// accumulate (rows) -> emit (m groups).
// ---------------------------------------------------------------------------
namespace tdp {
namespace {

struct BitmapAgg {
  unsigned* bits;
  unsigned short* wpre;
  i64* bcount;
  i64* boffs;
  unsigned long long* m;  // [1] group count (device)
  u64* cells;             // [n][cw]  image, count, sums, fixed words
  void* scan_ws;
  size_t scan_bytes;
  u64 lo;
  i64 range;
  int cw;
  // partitioned accumulation (part_ws_bytes; null below kPartMinRows)
  unsigned short* pslot;  // [n] group within its partition
  unsigned* pgroup;       // [n] group of each row (part_hist_kernel)
  u64* prw;               // [words] bits | in-block prefix << 32: one load per rank
  u64* pval;              // [naggs][n] value bits in partition order
  i64* phist;             // [P] rows per partition
  i64* poffs;             // [P] partition starts
  unsigned long long* pcur;  // [P] scatter cursors
  void* pscan_ws;
  size_t pscan_bytes;
};

// Partitioned accumulation (large inputs): rows are scattered by group into
// partitions of G groups whose cells fit one CTA's shared memory, then each
// partition is aggregated with shared-memory atomics and written out once --
// instead of 3-5 L2 atomics per row into a cell array of n x cw words.
constexpr i64 kPartMinRows = (i64)1 << 22;
constexpr int kPartMaxParts = 4096;
constexpr int kPartSmem = 200 * 1024;
constexpr int kPartMinGroups = 256;  // G below this: the unpartitioned kernel
constexpr int kPartTileRows = 12288;  // scatter tile: 1024 threads x 12 rows

size_t part_ws_bytes(i64 n, i64 range, int naggs) {
  if (n < kPartMinRows) return 0;
  return align256((size_t)n * 2) + align256((size_t)n * 4) +
         (size_t)(naggs > 0 ? naggs : 0) * align256((size_t)n * 8) +
         align256((size_t)rank_words(range) * 8) +
         3 * align256((size_t)(kPartMaxParts + 1) * 8) +
         align256(exclusive_scan_workspace(kPartMaxParts) + 1024);
}

size_t bitmap_agg_ws_bytes(i64 n, i64 range, int naggs) {
  const i64 r = range > 0 ? range : 1;
  const i64 words = rank_words(r), blocks = rank_blocks(r);
  const int na = naggs > 0 ? naggs : 0;
  return align256((size_t)words * 4) + align256((size_t)words * 2) + 2 * align256((size_t)blocks * 8) +
         256 + align256((size_t)(n > 0 ? n : 1) * cell_words(na, na) * 8) +
         align256(exclusive_scan_workspace(blocks)) + 2048 + part_ws_bytes(n, r, na);
}

BitmapAgg carve_bitmap_agg(void* ws, i64 n, i64 range, i64 lo, const ValSet& vs) {
  BitmapAgg b;
  const i64 r = range > 0 ? range : 1;
  const i64 words = rank_words(r), blocks = rank_blocks(r);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  b.bits = (unsigned*)p;
  p += align256((size_t)words * 4);
  b.wpre = (unsigned short*)p;
  p += align256((size_t)words * 2);
  b.bcount = (i64*)p;
  p += align256((size_t)blocks * 8);
  b.boffs = (i64*)p;
  p += align256((size_t)blocks * 8);
  b.m = (unsigned long long*)p;
  p += 256;
  b.cw = cell_words(vs.naggs, vs.nfixed);
  b.cells = (u64*)p;
  p += align256((size_t)(n > 0 ? n : 1) * cell_words(vs.naggs, vs.naggs) * 8);
  b.scan_ws = p;
  b.scan_bytes = exclusive_scan_workspace(blocks) + 1024;
  p += align256(exclusive_scan_workspace(blocks)) + 2048;
  b.lo = (u64)lo;
  b.range = r;
  b.pslot = nullptr;
  if (n >= kPartMinRows) {
    b.pslot = (unsigned short*)p;
    p += align256((size_t)n * 2);
    b.pgroup = (unsigned*)p;
    p += align256((size_t)n * 4);
    b.pval = (u64*)p;
    p += (size_t)vs.naggs * align256((size_t)n * 8);
    b.phist = (i64*)p;
    p += align256((size_t)(kPartMaxParts + 1) * 8);
    b.poffs = (i64*)p;
    p += align256((size_t)(kPartMaxParts + 1) * 8);
    b.pcur = (unsigned long long*)p;
    p += align256((size_t)(kPartMaxParts + 1) * 8);
    b.pscan_ws = p;
    b.pscan_bytes = exclusive_scan_workspace(kPartMaxParts) + 1024;
    p += align256(exclusive_scan_workspace(kPartMaxParts) + 1024);
    b.prw = (u64*)p;
  }
  return b;
}

__global__ void bm_set_kernel(const i64* __restrict__ keys, i64 n, BitmapAgg b) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const u64 d = (u64)__ldg(keys + i) - b.lo;
    atomicOr(b.bits + (d >> 5), 1u << (d & 31));
  }
}

// zero the m cells (m from the scan, on the device)
__global__ void bm_clear_kernel(BitmapAgg b) {
  const i64 words = (i64)*b.m * b.cw;
  for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < words;
       t += (i64)gridDim.x * blockDim.x)
    b.cells[t] = 0ull;
}

__global__ void bm_accum_kernel(const i64* __restrict__ keys, i64 n, BitmapAgg b, ValSet vs) {
  const int lane = threadIdx.x & 31;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 base = (i64)blockIdx.x * blockDim.x; base < n; base += stride) {
    const i64 i = base + threadIdx.x;
    const bool valid = i < n;
    const unsigned active = __ballot_sync(0xffffffffu, valid);
    if (!valid) continue;
    const i64 k = __ldg(keys + i);
    const unsigned peers = __match_any_sync(active, k);  // equal keys of the warp combine
    const int leader = __ffs(peers) - 1;
    const u64 d = (u64)k - b.lo;
    const i64 w = (i64)(d >> 5);
    const i64 g = b.boffs[d >> 10] + b.wpre[w] + __popc(b.bits[w] & ((1u << (d & 31)) - 1u));
    unsigned long long* c = reinterpret_cast<unsigned long long*>(b.cells + g * b.cw);
    if (lane == leader) {
      c[kCellImg] = (unsigned long long)k ^ 0x8000000000000000ull;  // same value from every writer
      atomicAdd(c + kCellCnt, (unsigned long long)__popc(peers));
    }
    for (int a = 0; a < vs.naggs; ++a) {
      if (vs.kind[a] == TDP_AGG_COUNT) continue;
      if (vs.kind[a] == TDP_AGG_SUM_F64) {
        const double v = group_sum(load_as_f64(vs.p[a], vs.dt[a], i), peers, lane);
        if (lane == leader) fixed_add(c + kCellAcc + vs.naggs + kFixedWords * vs.fidx[a], v);
      } else {
        const unsigned long long v =
            group_sum((unsigned long long)load_as_i64(vs.p[a], vs.dt[a], i), peers, lane);
        if (lane == leader) atomicAdd(c + kCellAcc + a, v);
      }
    }
  }
}

__global__ void bm_emit_kernel(BitmapAgg b, i64 m, ValSet vs, i64* __restrict__ out_keys,
                               i64* __restrict__ out_counts, u64* __restrict__ out_sums) {
  for (i64 g = (i64)blockIdx.x * blockDim.x + threadIdx.x; g < m;
       g += (i64)gridDim.x * blockDim.x) {
    const unsigned long long* c = reinterpret_cast<const unsigned long long*>(b.cells + g * b.cw);
    out_keys[g] = (i64)(c[kCellImg] ^ 0x8000000000000000ull);
    const u64 cnt = c[kCellCnt];
    out_counts[g] = (i64)cnt;
    for (int a = 0; a < vs.naggs; ++a) {
      u64 v;
      if (vs.kind[a] == TDP_AGG_COUNT)
        v = cnt;
      else if (vs.kind[a] == TDP_AGG_SUM_F64)
        v = (u64)__double_as_longlong(fixed_value(c + kCellAcc + vs.naggs + kFixedWords * vs.fidx[a]));
      else
        v = c[kCellAcc + a];
      out_sums[(i64)a * m + g] = vs.kind[a] == TDP_AGG_COUNT ? v : emit_value(vs, a, v, cnt);
    }
  }
}

__device__ __forceinline__ i64 bm_rank(const BitmapAgg& b, u64 d) {
  const i64 w = (i64)(d >> 5);
  return __ldg(b.boffs + (d >> 10)) + __ldg(b.wpre + w) +
         __popc(__ldg(b.bits + w) & ((1u << (d & 31)) - 1u));
}

// Key images of the m groups straight from the bitmap (group g = the g-th
// set bit): one thread per bitmap word, no pass over the rows.
__global__ void bm_keys_kernel(BitmapAgg b, i64 words) {
  for (i64 w = (i64)blockIdx.x * blockDim.x + threadIdx.x; w < words;
       w += (i64)gridDim.x * blockDim.x) {
    unsigned bits = b.bits[w];
    if (!bits) continue;
    i64 g = b.boffs[w >> 5] + b.wpre[w];
    while (bits) {
      const int bit = __ffs(bits) - 1;
      bits &= bits - 1;
      const u64 k = b.lo + (u64)w * 32 + (u64)bit;
      b.cells[g * b.cw + kCellImg] = k ^ 0x8000000000000000ull;
      ++g;
    }
  }
}

__global__ void rank_pack_kernel(BitmapAgg b, i64 words) {
  for (i64 w = (i64)blockIdx.x * blockDim.x + threadIdx.x; w < words;
       w += (i64)gridDim.x * blockDim.x)
    b.prw[w] = (u64)b.bits[w] | (u64)b.wpre[w] << 32;
}

// Rows per partition (partition = group >> gshift): shared counters, one
// global add per CTA and partition.
__global__ void part_hist_kernel(const i64* __restrict__ keys, i64 n, BitmapAgg b, int gshift,
                                 int parts) {
  extern __shared__ unsigned ph_cnt[];
  for (int p = threadIdx.x; p < parts; p += blockDim.x) ph_cnt[p] = 0u;
  __syncthreads();
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const u64 d = (u64)__ldg(keys + i) - b.lo;
    const u64 rw = __ldg(b.prw + (d >> 5));
    const i64 g = __ldg(b.boffs + (d >> 10)) + (i64)(rw >> 32) +
                  __popc((unsigned)rw & ((1u << (d & 31)) - 1u));
    b.pgroup[i] = (unsigned)g;
    atomicAdd(ph_cnt + (g >> gshift), 1u);
  }
  __syncthreads();
  for (int p = threadIdx.x; p < parts; p += blockDim.x)
    if (ph_cnt[p])
      atomicAdd(reinterpret_cast<unsigned long long*>(b.phist) + p, (unsigned long long)ph_cnt[p]);
}

// Scatter rows into their partitions, 12288-row tiles of 1024 threads: count
// per partition in shared memory (each row's place in its partition's run),
// a block scan of the counts (the tile's rows staged in partition order),
// one global add per partition and tile to reserve the runs, then the staged
// rows -- group-in-partition and each aggregate value (8 B) -- written out
// in staging order, so consecutive threads write consecutive addresses of a
// run (a row-order write would touch one sector per row).  Row order inside
// a partition is not fixed; every accumulation downstream is
// order-independent (integer and fixed-point adds).
constexpr int kScatterThreads = 1024;
constexpr int kScatterRows = kPartTileRows / kScatterThreads;

__global__ void __launch_bounds__(kScatterThreads)
    part_scatter_kernel(i64 n, BitmapAgg b, ValSet vs, int gshift, int parts) {
  extern __shared__ unsigned ps_sm[];
  unsigned* cnt = ps_sm;                      // [kPartMaxParts] rows per partition in the tile
  unsigned* tpre = cnt + kPartMaxParts;       // [kPartMaxParts] staged start
  unsigned* base = tpre + kPartMaxParts;      // [kPartMaxParts] reserved global start
  unsigned* wsum = base + kPartMaxParts;      // [32]
  u64* sval = reinterpret_cast<u64*>(wsum + 32);                                   // [tile]
  unsigned short* sslot = reinterpret_cast<unsigned short*>(sval + kPartTileRows);  // [tile]
  unsigned short* spart = sslot + kPartTileRows;                                   // [tile]
  const unsigned gmask = (1u << gshift) - 1u;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int p = tid; p < parts; p += kScatterThreads) cnt[p] = 0u;
  __syncthreads();
  for (i64 t0 = (i64)blockIdx.x * kPartTileRows; t0 < n; t0 += (i64)gridDim.x * kPartTileRows) {
    unsigned pp[kScatterRows], gg[kScatterRows];
#pragma unroll
    for (int r = 0; r < kScatterRows; ++r) {
      const i64 i = t0 + r * kScatterThreads + tid;
      pp[r] = 0xffffffffu;
      if (i < n) {
        const unsigned g = __ldcs(b.pgroup + i);
        gg[r] = g;
        pp[r] = g >> gshift;
      }
    }
#pragma unroll
    for (int r = 0; r < kScatterRows; ++r)
      if (pp[r] != 0xffffffffu) gg[r] = (gg[r] & gmask) | atomicAdd(cnt + pp[r], 1u) << 16;
    __syncthreads();
    // block exclusive scan of cnt[0, parts): 4 consecutive per thread
    unsigned c4[4], t = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int p = tid * 4 + j;
      c4[j] = p < parts ? cnt[p] : 0u;
      t += c4[j];
    }
    unsigned incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      unsigned w = wsum[lane], wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += v;
      }
      wsum[lane] = wi - w;
    }
    __syncthreads();
    unsigned run = wsum[warp] + incl - t;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int p = tid * 4 + j;
      if (p < parts) {
        tpre[p] = run;
        if (c4[j]) base[p] = (unsigned)atomicAdd(b.pcur + p, (unsigned long long)c4[j]);
        cnt[p] = 0u;
      }
      run += c4[j];
    }
    __syncthreads();
    // stage: slots and partitions, then one aggregate's values at a time
    unsigned sidx[kScatterRows];
#pragma unroll
    for (int r = 0; r < kScatterRows; ++r) {
      if (pp[r] != 0xffffffffu) {
        sidx[r] = tpre[pp[r]] + (gg[r] >> 16);
        sslot[sidx[r]] = (unsigned short)(gg[r] & 0xffffu);
        spart[sidx[r]] = (unsigned short)pp[r];
      }
    }
    const int tile = (int)min((i64)kPartTileRows, n - t0);
    __syncthreads();
    for (int s2 = tid; s2 < tile; s2 += kScatterThreads) {
      const unsigned p = spart[s2];
      b.pslot[(i64)base[p] + (s2 - tpre[p])] = sslot[s2];
    }
    for (int a = 0; a < vs.naggs; ++a) {
      if (vs.kind[a] == TDP_AGG_COUNT) continue;
      const bool f = vs.kind[a] == TDP_AGG_SUM_F64;
#pragma unroll
      for (int r = 0; r < kScatterRows; ++r) {
        const i64 i = t0 + r * kScatterThreads + tid;
        if (pp[r] != 0xffffffffu)
          sval[sidx[r]] = f ? (u64)__double_as_longlong(load_as_f64(vs.p[a], vs.dt[a], i))
                            : (u64)load_as_i64(vs.p[a], vs.dt[a], i);
      }
      __syncthreads();
      for (int s2 = tid; s2 < tile; s2 += kScatterThreads) {
        const unsigned p = spart[s2];
        b.pval[(i64)a * n + (i64)base[p] + (s2 - tpre[p])] = sval[s2];
      }
      __syncthreads();
    }
    __syncthreads();
  }
}

// One CTA per partition: its groups' cells (the cell layout minus the key
// image, `cw - 1` words each) in shared memory, shared-memory atomics per
// row, then one coalesced write of the cells.
__global__ void __launch_bounds__(1024)
    part_agg_kernel(BitmapAgg b, i64 n, ValSet vs, int gshift) {
  extern __shared__ unsigned long long pa_sm[];
  const int sw = b.cw - 1;
  const i64 p = blockIdx.x;
  const i64 g0 = p << gshift;
  const i64 m = (i64)*b.m;
  if (g0 >= m) return;
  const i64 ng = min((i64)1 << gshift, m - g0);
  for (i64 w = threadIdx.x; w < ng * sw; w += blockDim.x) pa_sm[w] = 0ull;
  __syncthreads();
  const i64 lo = b.poffs[p], hi = lo + b.phist[p];
  for (i64 i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    unsigned long long* c = pa_sm + (i64)b.pslot[i] * sw;  // c[w] = cell word w + 1
    atomicAdd(reinterpret_cast<unsigned*>(c + (kCellCnt - 1)), 1u);  // low half: < 2^31 rows
    for (int a = 0; a < vs.naggs; ++a) {
      if (vs.kind[a] == TDP_AGG_COUNT) continue;
      const u64 v = b.pval[(i64)a * n + i];
      if (vs.kind[a] == TDP_AGG_SUM_F64)
        fixed_add_shared(c + (kCellAcc - 1) + vs.naggs + kFixedWords * vs.fidx[a],
                         __longlong_as_double((long long)v));
      else
        split_add64(c + (kCellAcc - 1) + a, (unsigned long long)v);
    }
  }
  __syncthreads();
  u64* out = b.cells + g0 * b.cw;
  for (i64 w = threadIdx.x; w < ng * sw; w += blockDim.x) {
    const i64 g = w / sw;
    out[g * b.cw + 1 + (w - g * sw)] = pa_sm[w];
  }
}

}  // namespace
}  // namespace tdp

extern "C" {

size_t tdp_groupby_bitmap_workspace(int64_t n, int64_t key_range, int32_t naggs) {
  return bitmap_agg_ws_bytes(n, key_range, naggs);
}

int tdp_groupby_bitmap_prepare(const int64_t* keys, int64_t n, int64_t lo, int64_t key_range,
                               const tdp_column* vals, const int32_t* agg_kinds, int32_t naggs,
                               int64_t* out_ngroups, void* ws, size_t ws_bytes, void* stream) {
  TDP_REQUIRE(n >= 0 && out_ngroups != nullptr, "bad bitmap group-by arguments");
  TDP_REQUIRE(key_range >= 1 && key_range <= ((int64_t)1 << 34),
              "bitmap group-by key range %lld outside [1, 2^34]", (long long)key_range);
  TDP_REQUIRE(ws_bytes >= bitmap_agg_ws_bytes(n, key_range, naggs),
              "bitmap group-by workspace too small");
  ValSet vs;
  int rc = make_valset(vals, agg_kinds, naggs, n, &vs);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    TDP_CUDA_TRY(cudaMemsetAsync(out_ngroups, 0, 8, st));
    return TDP_OK;
  }
  BitmapAgg b = carve_bitmap_agg(ws, n, key_range, lo, vs);
  const i64 words = rank_words(key_range), blocks = rank_blocks(key_range);
  TDP_CUDA_TRY(cudaMemsetAsync(b.bits, 0, (size_t)words * 4, st));
  bm_set_kernel<<<stream_grid(n, 256 * 4, 16), 256, 0, st>>>(keys, n, b);
  TDP_LAUNCH_CHECK("bm_set_kernel");
  rank_popc_kernel<<<stream_grid(blocks, 8, 8), 256, 0, st>>>(b.bits, words, blocks, b.bcount,
                                                               b.wpre);
  TDP_LAUNCH_CHECK("rank_popc_kernel");
  rc = exclusive_scan_i64(b.bcount, b.boffs, blocks, reinterpret_cast<i64*>(b.m), b.scan_ws,
                          b.scan_bytes, st);
  if (rc) return rc;
  // partitioned accumulation: G groups per partition (a power of two whose
  // cells fit kPartSmem), P partitions over the <= min(n, range) groups
  int gshift = 15;
  while (gshift > 0 && ((size_t)1 << gshift) * (size_t)(b.cw - 1) * 8 > (size_t)kPartSmem) --gshift;
  const i64 gbound = n < key_range ? n : key_range;
  const i64 parts = (gbound + ((i64)1 << gshift) - 1) >> gshift;
  const char* part_env = getenv("TDP_GROUPBY_PARTITION");  // A/B tests and measurements
  const bool part_on = !(part_env && part_env[0] == '0');
  if (part_on && b.pslot != nullptr && n < ((i64)1 << 31) && ((i64)1 << gshift) >= kPartMinGroups &&
      parts <= kPartMaxParts) {
    bm_keys_kernel<<<stream_grid(words, 256, 8), 256, 0, st>>>(b, words);
    TDP_LAUNCH_CHECK("bm_keys_kernel");
    rank_pack_kernel<<<stream_grid(words, 256, 8), 256, 0, st>>>(b, words);
    TDP_LAUNCH_CHECK("rank_pack_kernel");
    TDP_CUDA_TRY(cudaMemsetAsync(b.phist, 0, (size_t)parts * 8, st));
    part_hist_kernel<<<stream_grid(n, 256 * 16, 8), 256, (size_t)parts * 4, st>>>(keys, n, b, gshift,
                                                                                  (int)parts);
    TDP_LAUNCH_CHECK("part_hist_kernel");
    rc = exclusive_scan_i64(b.phist, b.poffs, parts, nullptr, b.pscan_ws, b.pscan_bytes, st);
    if (rc) return rc;
    TDP_CUDA_TRY(cudaMemcpyAsync(b.pcur, b.poffs, (size_t)parts * 8, cudaMemcpyDeviceToDevice, st));
    const size_t ssm = (size_t)kPartMaxParts * 12 + 128 + (size_t)kPartTileRows * 12;
    TDP_CUDA_TRY(cudaFuncSetAttribute(part_scatter_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)ssm));
    TDP_CUDA_TRY(cudaFuncSetAttribute(part_agg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kPartSmem));
    part_scatter_kernel<<<stream_grid(n, kPartTileRows, 1), kScatterThreads, ssm, st>>>(
        n, b, vs, gshift, (int)parts);
    TDP_LAUNCH_CHECK("part_scatter_kernel");
    const size_t asm_ = ((size_t)1 << gshift) * (size_t)(b.cw - 1) * 8;
    part_agg_kernel<<<(unsigned)parts, 1024, asm_, st>>>(b, n, vs, gshift);
    TDP_LAUNCH_CHECK("part_agg_kernel");
  } else {
    bm_clear_kernel<<<stream_grid(n * b.cw, 256 * 4, 8), 256, 0, st>>>(b);
    TDP_LAUNCH_CHECK("bm_clear_kernel");
    bm_accum_kernel<<<stream_grid(n, 256, 32), 256, 0, st>>>(keys, n, b, vs);
    TDP_LAUNCH_CHECK("bm_accum_kernel");
  }
  TDP_CUDA_TRY(cudaMemcpyAsync(out_ngroups, b.m, 8, cudaMemcpyDeviceToDevice, st));
  return TDP_OK;
}

int tdp_groupby_bitmap_emit(int64_t n, int64_t lo, int64_t key_range, const int32_t* agg_kinds,
                            int32_t naggs, int64_t m, int64_t* out_keys, int64_t* out_counts,
                            void* out_sums, void* ws, size_t ws_bytes, void* stream) {
  TDP_REQUIRE(m >= 0 && m <= (n > 0 ? n : 0), "bad group count");
  TDP_REQUIRE(ws_bytes >= bitmap_agg_ws_bytes(n, key_range, naggs),
              "bitmap group-by workspace too small");
  if (m == 0) return TDP_OK;
  ValSet vs;
  int rc = emit_kinds(agg_kinds, naggs, &vs);  // kinds only (+ AVG bits)
  if (rc) return rc;
  number_fixed(&vs);
  BitmapAgg b = carve_bitmap_agg(ws, n, key_range, lo, vs);
  cudaStream_t st = as_stream(stream);
  bm_emit_kernel<<<stream_grid(m, 256, 16), 256, 0, st>>>(b, m, vs, out_keys, out_counts,
                                                           reinterpret_cast<u64*>(out_sums));
  TDP_LAUNCH_CHECK("bm_emit_kernel");
  return TDP_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Sorted-runs group-by: one int64 key column that is non-decreasing with runs
// of at most kRunLen equal keys (tdp_scan_minmax_runs checks both) -- e.g. a
// join's output in probe-row order over a clustered key (TPC-H lineitem by
// l_orderkey).  Groups are the runs: a count pass over 2048-row tiles (run
// starts per tile), a scan of the tile counts (group offsets, m), and an emit
// pass in which the thread at each run start writes its group: the key, the
// run length and every sum over the run's rows in row order -- the order of
// np.add.at (tq/kernels.py:153-158), so float sums are bit-identical to the
// reference's; no hash table, no bitmap, no atomics.
// ---------------------------------------------------------------------------
namespace tdp {
namespace {

constexpr int kRunTile = 256;  // rows per CTA, one per thread
constexpr int kRunLen = 32;    // = kRunMax of tdp_scan_minmax_runs

__global__ void __launch_bounds__(kRunTile)
    runs_count_kernel(const i64* __restrict__ keys, i64 n, i64* __restrict__ tile_counts) {
  __shared__ int wsum[kRunTile / 32];
  const i64 i = (i64)blockIdx.x * kRunTile + threadIdx.x;
  const bool start = i < n && (i == 0 || __ldg(keys + i) != __ldg(keys + i - 1));
  const int c = __popc(__ballot_sync(0xffffffffu, start));
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    i64 t = 0;
    for (int w = 0; w < kRunTile / 32; ++w) t += wsum[w];
    tile_counts[blockIdx.x] = t;
  }
}

// One row per thread; the thread at a run start writes the group.  The run's
// end is the next start bit of the tile (shared ballot words), else the run
// continues past the tile (<= kRunLen rows, read on).  Value loads of a run
// are issued four rows at a time, the adds stay in row order.
__global__ void __launch_bounds__(kRunTile)
    runs_emit_kernel(const i64* __restrict__ keys, i64 n, const i64* __restrict__ tile_offsets,
                     ValSet vs, i64 m, i64* __restrict__ out_keys, i64* __restrict__ out_counts,
                     u64* __restrict__ out_sums) {
  __shared__ unsigned sbits[kRunTile / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 row0 = (i64)blockIdx.x * kRunTile;
  const i64 i = row0 + threadIdx.x;
  i64 key = 0;
  bool start = false;
  if (i < n) {
    key = __ldg(keys + i);
    start = i == 0 || key != __ldg(keys + i - 1);
  }
  const unsigned bal = __ballot_sync(0xffffffffu, start);
  if (lane == 0) sbits[warp] = bal;
  __syncthreads();
  if (!start) return;
  int before = __popc(bal & lanemask_lt());
  for (int w = 0; w < warp; ++w) before += __popc(sbits[w]);
  const i64 g = tile_offsets[blockIdx.x] + before;
  // run end: the next start in this tile, else the tile's end and beyond
  const int rows_here = (int)(n - row0 < kRunTile ? n - row0 : kRunTile);
  int end = -1;
  const int t = threadIdx.x + 1;
  if (t < kRunTile) {
    int w = t >> 5;
    unsigned b = sbits[w] & (0xffffffffu << (t & 31));
    for (;;) {
      if (b) {
        end = w * 32 + __ffs(b) - 1;
        break;
      }
      if (++w >= kRunTile / 32) break;
      b = sbits[w];
    }
  }
  int len;
  if (end >= 0) {
    len = end - threadIdx.x;
  } else {
    len = rows_here - threadIdx.x;
    while (len < kRunLen && i + len < n && __ldg(keys + i + len) == key) ++len;
  }
  out_keys[g] = key;
  out_counts[g] = len;
  for (int a = 0; a < vs.naggs; ++a) {
    if (vs.kind[a] == TDP_AGG_COUNT) {
      out_sums[(i64)a * m + g] = (u64)len;
      continue;
    }
    u64 raw;
    if (vs.kind[a] == TDP_AGG_SUM_F64) {
      double acc = 0.0;  // np.add.at into zeros, in row order
      for (int r = 0; r < len; r += 4) {
        double x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          x[u] = r + u < len ? load_as_f64(vs.p[a], vs.dt[a], i + r + u) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (r + u < len) acc = __dadd_rn(acc, x[u]);
      }
      raw = (u64)__double_as_longlong(acc);
    } else {
      u64 acc = 0;
      for (int r = 0; r < len; ++r) acc += (u64)load_as_i64(vs.p[a], vs.dt[a], i + r);
      raw = acc;
    }
    out_sums[(i64)a * m + g] = emit_value(vs, a, raw, (u64)len);
  }
}

struct RunsWs {
  i64* tile_counts;
  i64* tile_offsets;
  void* scan_ws;
  size_t scan_bytes;
};

size_t runs_ws_bytes(i64 n) {
  const i64 tiles = ceil_div(n > 0 ? n : 1, kRunTile);
  return 2 * align256((size_t)tiles * 8) + exclusive_scan_workspace(tiles) + 256;
}

RunsWs carve_runs(void* ws, i64 n) {
  const i64 tiles = ceil_div(n > 0 ? n : 1, kRunTile);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  RunsWs w;
  w.tile_counts = (i64*)p;
  p += align256((size_t)tiles * 8);
  w.tile_offsets = (i64*)p;
  p += align256((size_t)tiles * 8);
  w.scan_ws = p;
  w.scan_bytes = exclusive_scan_workspace(tiles) + 256;
  return w;
}

}  // namespace
}  // namespace tdp

extern "C" {

size_t tdp_groupby_runs_workspace(int64_t n) { return runs_ws_bytes(n); }

int tdp_groupby_runs_prepare(const int64_t* keys, int64_t n, int64_t* out_ngroups, void* ws,
                             size_t ws_bytes, void* stream) {
  TDP_REQUIRE(n >= 0 && out_ngroups != nullptr, "bad sorted-runs group-by arguments");
  TDP_REQUIRE(ws_bytes >= runs_ws_bytes(n), "sorted-runs group-by workspace too small");
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    TDP_CUDA_TRY(cudaMemsetAsync(out_ngroups, 0, sizeof(i64), st));
    return TDP_OK;
  }
  RunsWs w = carve_runs(ws, n);
  const i64 tiles = ceil_div(n, kRunTile);
  runs_count_kernel<<<(unsigned)tiles, kRunTile, 0, st>>>(keys, n, w.tile_counts);
  TDP_LAUNCH_CHECK("runs_count_kernel");
  return exclusive_scan_i64(w.tile_counts, w.tile_offsets, tiles, out_ngroups, w.scan_ws,
                            w.scan_bytes, st);
}

int tdp_groupby_runs_emit(const int64_t* keys, int64_t n, const tdp_column* vals,
                          const int32_t* agg_kinds, int32_t naggs, int64_t m, int64_t* out_keys,
                          int64_t* out_counts, void* out_sums, void* ws, size_t ws_bytes,
                          void* stream) {
  TDP_REQUIRE(m >= 0 && m <= (n > 0 ? n : 0), "bad group count");
  TDP_REQUIRE(ws_bytes >= runs_ws_bytes(n), "sorted-runs group-by workspace too small");
  TDP_REQUIRE(naggs >= 0 && naggs <= 32, "at most 32 aggregates");
  if (m == 0) return TDP_OK;
  int32_t plain[32];
  unsigned avg = 0;
  for (int a = 0; a < naggs; ++a) {
    plain[a] = agg_kinds[a] & ~TDP_AGG_AVG_BIT;
    if (agg_kinds[a] & TDP_AGG_AVG_BIT) avg |= 1u << a;
  }
  ValSet vs;
  int rc = make_valset(vals, plain, naggs, n, &vs);
  if (rc) return rc;
  vs.avg = avg;
  RunsWs w = carve_runs(ws, n);
  cudaStream_t st = as_stream(stream);
  runs_emit_kernel<<<(unsigned)ceil_div(n, kRunTile), kRunTile, 0, st>>>(
      keys, n, w.tile_offsets, vs, m, out_keys, out_counts, reinterpret_cast<u64*>(out_sums));
  TDP_LAUNCH_CHECK("runs_emit_kernel");
  return TDP_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// sort / searchsorted equi-join (the algorithm north_star names; the default
// planner prefers the dense-range and hash joins, which read the probe side
// once with one table lookup per row -- tdp_join_sorted_* is kept as the
// measured alternative and for callers that want it).
//   prepare: stable LSD radix sort of the build key images with their row ids
//            (ascending row within equal keys), then every probe key searches
//            the sorted images: a top level of <= kTopFences fence keys held
//            in shared memory by persistent CTAs, then a binary search of the
//            fence interval in global memory (L2-resident for build sides up
//            to ~10^7 keys; sorted probe columns hit L1).  Match bits + per
//            word pair counts per 2048-row tile, as the hash join's.
//   emit:    matched rows search again and write (probe row, build row)
//            pairs: by probe row, then ascending build row.
// ---------------------------------------------------------------------------
namespace tdp {
namespace {

constexpr int kTopFences = 4096;

struct SortedJoin {
  const u64* sk;     // sorted build key images [m]
  const i64* order;  // build row of each sorted key [m]
  i64 m;
  i64 stride;        // top[j] = sk[j * stride], j < ntop
  int ntop;
};

__device__ __forceinline__ void sj_load_top(const SortedJoin& sj, u64* top) {
  for (int j = threadIdx.x; j < sj.ntop; j += blockDim.x) top[j] = __ldg(sj.sk + (i64)j * sj.stride);
  __syncthreads();
}

// First index of sk with image >= k (m if none).
__device__ __forceinline__ i64 sj_lower(const SortedJoin& sj, const u64* top, u64 k) {
  int a = 0, b = sj.ntop;  // first fence >= k
  while (a < b) {
    const int mid = (a + b) >> 1;
    if (top[mid] < k) a = mid + 1;
    else b = mid;
  }
  // sk[(a-1)*stride] < k <= sk[a*stride]: the answer lies in ((a-1)*stride, a*stride]
  i64 lo = a > 0 ? (i64)(a - 1) * sj.stride + 1 : 0;
  i64 hi = (i64)a * sj.stride;
  if (hi > sj.m) hi = sj.m;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (__ldg(sj.sk + mid) < k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Number of build keys equal to image k; *first = their first sorted index.
__device__ __forceinline__ i64 sj_count(const SortedJoin& sj, const u64* top, u64 k, i64* first) {
  const i64 lo = sj_lower(sj, top, k);
  *first = lo;
  if (lo >= sj.m || __ldg(sj.sk + lo) != k) return 0;
  if (lo + 1 >= sj.m || __ldg(sj.sk + lo + 1) != k) return 1;
  // a run: galloping, then bisection for the first image > k
  i64 a = lo + 1, step = 2;
  while (a + step < sj.m && __ldg(sj.sk + a + step) == k) {
    a += step;
    step <<= 1;
  }
  i64 b = a + step < sj.m ? a + step : sj.m;  // sk[a] == k, sk[b] > k or b == m
  while (a + 1 < b) {
    const i64 mid = (a + b) >> 1;
    if (__ldg(sj.sk + mid) == k) a = mid;
    else b = mid;
  }
  return b - lo;
}

// tile_counts zeroed; persistent CTAs walk the 2048-row tiles.
template <bool kFiltered>
__global__ void __launch_bounds__(kJoinThreads)
    sorted_count_kernel(SortedJoin sj, const i64* __restrict__ probe, i64 np, i64 tiles,
                        PredSet ps, unsigned* __restrict__ match_bits,
                        i64* __restrict__ word_counts, i64* __restrict__ tile_counts) {
  __shared__ u64 top[kTopFences];
  sj_load_top(sj, top);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (i64 tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    bool act[kJoinPer];
    i64 row[kJoinPer];
    u64 key[kJoinPer];
#pragma unroll
    for (int k = 0; k < kJoinPer; ++k) {
      row[k] = join_row(tile, k);
      act[k] = row[k] < np;
      key[k] = act[k] ? image_i64(__ldcs(probe + row[k]), 0) : 0;
    }
    if (kFiltered) eval_batch<kJoinPer>(ps, row, act);
    i64 local = 0;
#pragma unroll
    for (int k = 0; k < kJoinPer; ++k) {
      i64 first, c = act[k] ? sj_count(sj, top, key[k], &first) : 0;
      const unsigned word = __ballot_sync(0xffffffffu, c > 0);
      const i64 wc = word ? warp_sum(c) : 0;
      if (lane == 0) {
        match_bits[tile * kJoinWords + k * kJoinWarps + warp] = word;
        word_counts[tile * kJoinWords + k * kJoinWarps + warp] = wc;
      }
      local += wc;
    }
    if (lane == 0 && local != 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(tile_counts + tile), (unsigned long long)local);
  }
}

__global__ void __launch_bounds__(kJoinThreads)
    sorted_emit_kernel(SortedJoin sj, const i64* __restrict__ probe, i64 tiles,
                       const unsigned* __restrict__ match_bits,
                       const i64* __restrict__ word_counts, const i64* __restrict__ tile_counts,
                       const i64* __restrict__ tile_offsets, i64* __restrict__ out_probe,
                       i64* __restrict__ out_build) {
  __shared__ u64 top[kTopFences];
  sj_load_top(sj, top);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (i64 tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    if (tile_counts[tile] == 0) continue;  // CTA-uniform
    const WordPrefix wp(word_counts + tile * kJoinWords, lane);
    const i64 base = tile_offsets[tile];
    unsigned bits[kJoinPer];
    i64 s[kJoinPer], c[kJoinPer];
#pragma unroll
    for (int k = 0; k < kJoinPer; ++k) bits[k] = match_bits[tile * kJoinWords + k * kJoinWarps + warp];
#pragma unroll
    for (int k = 0; k < kJoinPer; ++k) {
      s[k] = 0;
      c[k] = 0;
      if ((bits[k] >> lane) & 1u)
        c[k] = sj_count(sj, top, image_i64(__ldg(probe + join_row(tile, k)), 0), &s[k]);
    }
#pragma unroll
    for (int k = 0; k < kJoinPer; ++k) {
      if (bits[k] == 0u) continue;  // warp-uniform
      const i64 word_off = base + wp.word_offset(k * kJoinWarps + warp);
      i64 ci = c[k];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const i64 t = __shfl_up_sync(0xffffffffu, ci, o);
        if (lane >= o) ci += t;
      }
      const i64 pos = word_off + ci - c[k];
      const i64 i = join_row(tile, k);
      for (i64 m = 0; m < c[k]; ++m) {
        out_probe[pos + m] = i;
        out_build[pos + m] = __ldg(sj.order + s[k] + m);
      }
    }
  }
}

struct SortedWs {
  SortBuffers sb;
  unsigned* match_bits;
  i64* word_counts;
  i64* tile_counts;
  i64* tile_offsets;
  void* scan_ws;
  size_t scan_bytes;
};

size_t sorted_ws_bytes(i64 nb, i64 np) {
  const i64 tiles = ceil_div(np > 0 ? np : 1, kJoinTile);
  return sort_ws_bytes(nb) + align256((size_t)tiles * kJoinWords * 4) +
         align256((size_t)tiles * kJoinWords * 8) + 2 * align256((size_t)tiles * 8) +
         exclusive_scan_workspace(tiles) + 2048;
}

SortedWs carve_sorted(void* ws, i64 nb, i64 np) {
  SortedWs j;
  j.sb = carve(ws, nb);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws) + sort_ws_bytes(nb);
  const i64 tiles = ceil_div(np > 0 ? np : 1, kJoinTile);
  j.match_bits = (unsigned*)p;
  p += align256((size_t)tiles * kJoinWords * 4);
  j.word_counts = (i64*)p;
  p += align256((size_t)tiles * kJoinWords * 8);
  j.tile_counts = (i64*)p;
  p += align256((size_t)tiles * 8);
  j.tile_offsets = (i64*)p;
  p += align256((size_t)tiles * 8);
  j.scan_ws = p;
  j.scan_bytes = exclusive_scan_workspace(tiles) + 1024;
  return j;
}

SortedJoin sorted_view(const SortedWs& j, i64 nb) {
  SortedJoin sj;
  sj.sk = j.sb.k0;
  sj.order = j.sb.i0;
  sj.m = nb;
  sj.stride = ceil_div(nb > 0 ? nb : 1, kTopFences);
  sj.ntop = (int)ceil_div(nb, sj.stride);
  return sj;
}

int persistent_grid(i64 tiles) {
  const i64 g = (i64)sm_count() * 4;
  return (int)(tiles < g ? (tiles > 0 ? tiles : 1) : g);
}

}  // namespace
}  // namespace tdp

extern "C" {

size_t tdp_join_sorted_workspace(int64_t n_build, int64_t n_probe) {
  return sorted_ws_bytes(n_build, n_probe);
}

int tdp_join_sorted_prepare(const int64_t* build_keys, int64_t n_build, const int64_t* probe_keys,
                            int64_t n_probe, const tdp_column* pcols, int32_t npcols,
                            const tdp_predicate* ppreds, int32_t nppreds, int64_t* out_count,
                            void* ws, size_t ws_bytes, void* stream) {
  TDP_REQUIRE(n_build >= 0 && n_probe >= 0, "negative join sizes");
  TDP_REQUIRE(out_count != nullptr, "null join count output");
  TDP_REQUIRE(ws_bytes >= sorted_ws_bytes(n_build, n_probe), "sorted join workspace too small");
  PredSet pps;
  int rc = make_predset(pcols, npcols, ppreds, nppreds, n_probe, &pps);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  SortedWs j = carve_sorted(ws, n_build, n_probe);
  TDP_CUDA_TRY(cudaMemsetAsync(out_count, 0, sizeof(i64), st));
  if (n_build == 0 || n_probe == 0) return TDP_OK;
  make_keys_kernel<<<stream_grid(n_build, 256 * 8, 8), 256, 0, st>>>(build_keys, TDP_I64, 0,
                                                                     n_build, j.sb.k0, j.sb.i0);
  TDP_LAUNCH_CHECK("make_keys_kernel");
  u64* sk;
  i64* order;
  rc = radix_sort(j.sb, n_build, st, &sk, &order);
  if (rc) return rc;
  if (sk != j.sb.k0) {  // keep the sorted build in k0 / i0 for tdp_join_sorted_emit
    TDP_CUDA_TRY(cudaMemcpyAsync(j.sb.k0, sk, (size_t)n_build * 8, cudaMemcpyDeviceToDevice, st));
    TDP_CUDA_TRY(cudaMemcpyAsync(j.sb.i0, order, (size_t)n_build * 8, cudaMemcpyDeviceToDevice, st));
  }
  const i64 tiles = ceil_div(n_probe, kJoinTile);
  TDP_CUDA_TRY(cudaMemsetAsync(j.tile_counts, 0, (size_t)tiles * sizeof(i64), st));
  const SortedJoin sj = sorted_view(j, n_build);
  const int grid = persistent_grid(tiles);
  cudaEvent_t t0 = timer_begin(2, st);
  if (pps.npreds > 0)
    sorted_count_kernel<true><<<grid, kJoinThreads, 0, st>>>(
        sj, probe_keys, n_probe, tiles, pps, j.match_bits, j.word_counts, j.tile_counts);
  else
    sorted_count_kernel<false><<<grid, kJoinThreads, 0, st>>>(
        sj, probe_keys, n_probe, tiles, pps, j.match_bits, j.word_counts, j.tile_counts);
  TDP_LAUNCH_CHECK("sorted_count_kernel");
  timer_end(t0, st);
  return exclusive_scan_i64(j.tile_counts, j.tile_offsets, tiles, out_count, j.scan_ws,
                            j.scan_bytes, st);
}

int tdp_join_sorted_emit(const int64_t* probe_keys, int64_t n_build, int64_t n_probe,
                         int64_t* out_probe_idx, int64_t* out_build_idx, void* ws,
                         size_t ws_bytes, void* stream) {
  TDP_REQUIRE(ws_bytes >= sorted_ws_bytes(n_build, n_probe), "sorted join workspace too small");
  if (n_build == 0 || n_probe == 0) return TDP_OK;
  cudaStream_t st = as_stream(stream);
  SortedWs j = carve_sorted(ws, n_build, n_probe);
  const i64 tiles = ceil_div(n_probe, kJoinTile);
  sorted_emit_kernel<<<persistent_grid(tiles), kJoinThreads, 0, st>>>(
      sorted_view(j, n_build), probe_keys, tiles, j.match_bits, j.word_counts, j.tile_counts,
      j.tile_offsets, out_probe_idx, out_build_idx);
  TDP_LAUNCH_CHECK("sorted_emit_kernel");
  return TDP_OK;
}

}  // extern "C"
