// Device-wide exclusive prefix sum over int64 counts (tile counts of the
// filter compaction, radix-sort digit histograms, join match counts).
// One launch: up to kChunk values are scanned by one CTA; beyond that every
// CTA scans a chunk and finds its offset by decoupled look-back over its
// predecessors' published aggregates / inclusive prefixes (one 64-bit status
// word per chunk: 2 flag bits + a 62-bit value), so no second pass over the
// data and no recursion.  Counts are non-negative and below 2^62.
#include "tdp_common.cuh"

namespace tdp {

namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;
constexpr int kChunk = kScanThreads * kScanItems;

// Block-wide exclusive scan of one value per thread; returns the block total
// through *total.
__device__ __forceinline__ i64 block_exclusive_scan(i64 v, i64* total) {
  __shared__ i64 warp_tot[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  i64 incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    i64 t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    i64 w = lane < (kScanThreads / 32) ? warp_tot[lane] : 0;
    i64 wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      i64 t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < (kScanThreads / 32)) warp_tot[lane] = wi - w;
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  i64 out = warp_tot[warp] + incl - v;
  return out;
}

__global__ void __launch_bounds__(kScanThreads) chunk_scan_kernel(const i64* __restrict__ in,
                                                                  i64* __restrict__ out, i64 n,
                                                                  i64* __restrict__ total) {
  __shared__ i64 s_total;
  const i64 base = (i64)blockIdx.x * kChunk + (i64)threadIdx.x * kScanItems;
  i64 v[kScanItems];
  i64 local = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    i64 idx = base + k;
    v[k] = idx < n ? in[idx] : 0;
    local += v[k];
  }
  i64 pre = block_exclusive_scan(local, &s_total);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    i64 idx = base + k;
    if (idx < n) out[idx] = pre;
    pre += v[k];
  }
  if (threadIdx.x == 0 && total != nullptr) *total = s_total;
}

constexpr u64 kFlagAgg = 1ull << 62;   // value = this chunk's sum
constexpr u64 kFlagPre = 2ull << 62;   // value = inclusive prefix through this chunk
constexpr u64 kValMask = kFlagAgg - 1;

__device__ __forceinline__ u64 load_status(const u64* p) {
  return *reinterpret_cast<const volatile u64*>(p);
}

// status[nchunks] and the chunk ticket (status[nchunks]) must be zero.
__global__ void __launch_bounds__(kScanThreads)
    lookback_scan_kernel(const i64* __restrict__ in, i64* __restrict__ out, i64 n,
                         u64* __restrict__ status, i64 nchunks, i64* __restrict__ total) {
  __shared__ i64 s_total;
  __shared__ i64 s_prefix;
  __shared__ unsigned s_chunk;
  if (threadIdx.x == 0)  // chunks in dispatch order: predecessors are running or done
    s_chunk = atomicAdd(reinterpret_cast<unsigned*>(status + nchunks), 1u);
  __syncthreads();
  const i64 chunk = s_chunk;
  const i64 base = chunk * kChunk + (i64)threadIdx.x * kScanItems;
  i64 v[kScanItems];
  i64 local = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const i64 idx = base + k;
    v[k] = idx < n ? __ldg(in + idx) : 0;
    local += v[k];
  }
  i64 pre = block_exclusive_scan(local, &s_total);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const i64 agg = s_total;
    i64 excl = 0;
    if (chunk == 0) {
      if (lane == 0) atomicExch(reinterpret_cast<unsigned long long*>(status), kFlagPre | (u64)agg);
    } else {
      if (lane == 0)
        atomicExch(reinterpret_cast<unsigned long long*>(status + chunk), kFlagAgg | (u64)agg);
      for (i64 p = chunk - 1;; p -= 32) {
        const i64 idx = p - lane;  // lane 0 = nearest predecessor
        u64 st = idx >= 0 ? load_status(status + idx) : kFlagPre;
        while (__any_sync(0xffffffffu, (st >> 62) == 0))
          if ((st >> 62) == 0) st = load_status(status + idx);
        const unsigned prefixed = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        const int stop = prefixed ? __ffs(prefixed) - 1 : 31;
        i64 c = lane <= stop ? (i64)(st & kValMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        excl += c;
        if (prefixed) break;
      }
      if (lane == 0)
        atomicExch(reinterpret_cast<unsigned long long*>(status + chunk),
                   kFlagPre | (u64)(excl + agg));
    }
    if (lane == 0) s_prefix = excl;
  }
  __syncthreads();
  pre += s_prefix;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const i64 idx = base + k;
    if (idx < n) out[idx] = pre;
    pre += v[k];
  }
  if (total != nullptr && chunk == nchunks - 1 && threadIdx.x == 0) *total = s_prefix + s_total;
}

}  // namespace

size_t exclusive_scan_workspace(i64 n) {
  // a multiple of 256 bytes: callers carve further buffers behind it
  const size_t b = (size_t)(ceil_div(n > 0 ? n : 1, kChunk) + 1) * sizeof(u64) + 256;
  return (b + 255) & ~(size_t)255;
}

int exclusive_scan_i64(const i64* in, i64* out, i64 n, i64* total, void* ws, size_t ws_bytes,
                       cudaStream_t stream) {
  if (n <= 0) {
    if (total) TDP_CUDA_TRY(cudaMemsetAsync(total, 0, sizeof(i64), stream));
    return TDP_OK;
  }
  if (n <= kChunk) {
    chunk_scan_kernel<<<1, kScanThreads, 0, stream>>>(in, out, n, total);
    TDP_LAUNCH_CHECK("chunk_scan_kernel");
    return TDP_OK;
  }
  const i64 nchunks = ceil_div(n, kChunk);
  TDP_REQUIRE(ws != nullptr && ws_bytes >= exclusive_scan_workspace(n), "scan workspace too small");
  u64* status = reinterpret_cast<u64*>(ws);
  TDP_CUDA_TRY(cudaMemsetAsync(status, 0, (size_t)(nchunks + 1) * sizeof(u64), stream));
  lookback_scan_kernel<<<(unsigned)nchunks, kScanThreads, 0, stream>>>(in, out, n, status, nchunks,
                                                                      total);
  TDP_LAUNCH_CHECK("lookback_scan_kernel");
  return TDP_OK;
}

}  // namespace tdp
