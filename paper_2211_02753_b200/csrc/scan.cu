// Device-wide exclusive prefix sum over int64 counts (tile counts of the
// filter compaction, radix-sort digit histograms, join match counts).
// Reduce-then-scan: each CTA scans a chunk of kChunk values, the chunk totals
// are scanned recursively, then chunk offsets are added back.
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
                                                                  i64* __restrict__ chunk_sums) {
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
  if (threadIdx.x == 0 && chunk_sums != nullptr) chunk_sums[blockIdx.x] = s_total;
}

__global__ void add_offsets_kernel(i64* __restrict__ out, i64 n, const i64* __restrict__ offs) {
  const i64 chunk = blockIdx.x;
  const i64 add = offs[chunk];
  const i64 start = chunk * kChunk;
  for (int t = threadIdx.x; t < kChunk; t += blockDim.x) {
    i64 idx = start + t;
    if (idx < n) out[idx] += add;
  }
}

// total = out[n-1] + in[n-1] (or 0 when n == 0)
__global__ void write_total_kernel(const i64* in, const i64* out, i64 n, i64* total) {
  *total = n > 0 ? out[n - 1] + in[n - 1] : 0;
}

}  // namespace

size_t exclusive_scan_workspace(i64 n) {
  size_t bytes = 0;
  i64 level = n;
  while (level > kChunk) {
    level = ceil_div(level, kChunk);
    bytes += 2 * (size_t)level * sizeof(i64);
  }
  return bytes + 256;
}

int exclusive_scan_i64(const i64* in, i64* out, i64 n, i64* total, void* ws, size_t ws_bytes,
                       cudaStream_t stream) {
  if (n <= 0) {
    if (total) TDP_CUDA_TRY(cudaMemsetAsync(total, 0, sizeof(i64), stream));
    return TDP_OK;
  }
  if (n <= kChunk) {
    chunk_scan_kernel<<<1, kScanThreads, 0, stream>>>(in, out, n, nullptr);
    TDP_LAUNCH_CHECK("chunk_scan_kernel");
  } else {
    const i64 nchunks = ceil_div(n, kChunk);
    TDP_REQUIRE(ws_bytes >= exclusive_scan_workspace(n), "scan workspace too small");
    i64* sums = reinterpret_cast<i64*>(ws);
    i64* offs = sums + nchunks;
    chunk_scan_kernel<<<(unsigned)nchunks, kScanThreads, 0, stream>>>(in, out, n, sums);
    TDP_LAUNCH_CHECK("chunk_scan_kernel");
    int rc = exclusive_scan_i64(sums, offs, nchunks, nullptr, offs + nchunks,
                                ws_bytes - 2 * nchunks * sizeof(i64), stream);
    if (rc != TDP_OK) return rc;
    add_offsets_kernel<<<(unsigned)nchunks, 256, 0, stream>>>(out, n, offs);
    TDP_LAUNCH_CHECK("add_offsets_kernel");
  }
  if (total) {
    write_total_kernel<<<1, 1, 0, stream>>>(in, out, n, total);
    TDP_LAUNCH_CHECK("write_total_kernel");
  }
  return TDP_OK;
}

}  // namespace tdp
