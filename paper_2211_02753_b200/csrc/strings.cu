// Dictionary encoding of a string column on the device (
// tq/encodings.py:127-133 dict_encode: codes are the strings' ranks in the
// sorted set of distinct strings).
//
// The strings arrive as one UTF-8 byte buffer with int64 offsets (byte-wise
// order of UTF-8 equals code-point order, Python's str order).  Per string a
// 64-bit hash; equal hashes are grouped with the radix-sort unique
// (tdp_unique_inverse); every string is then compared byte for byte with its
// group's first string, so a hash collision between different strings is
// detected (flag) rather than merging them.  The host sorts only the m
// distinct strings and uploads each group's rank; the codes are a gather.
#include "tdp_common.cuh"

namespace tdp {
namespace {

__device__ __forceinline__ u64 mix64(u64 x) {  // splitmix64 finaliser
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// FNV-1a over the bytes, 8 at a time where aligned, then a finaliser;
// the length is part of the hash.
__global__ void string_hash_kernel(const unsigned char* __restrict__ bytes,
                                   const i64* __restrict__ offs, i64 n, i64* __restrict__ out) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const i64 b = offs[i], e = offs[i + 1];
    u64 h = 0xcbf29ce484222325ull ^ (u64)(e - b);
    for (i64 p = b; p < e; ++p) {
      h ^= bytes[p];
      h *= 0x100000001b3ull;
    }
    out[i] = (i64)mix64(h);
  }
}

__global__ void group_first_kernel(const i64* __restrict__ inverse, i64 n,
                                   unsigned long long* __restrict__ first) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    atomicMin(first + inverse[i], (unsigned long long)i);
}

__global__ void string_group_check_kernel(const unsigned char* __restrict__ bytes,
                                          const i64* __restrict__ offs,
                                          const i64* __restrict__ inverse,
                                          const unsigned long long* __restrict__ first, i64 n,
                                          int* __restrict__ flag) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    const i64 r = (i64)first[inverse[i]];
    if (r == i) continue;
    const i64 b = offs[i], e = offs[i + 1], rb = offs[r], re = offs[r + 1];
    bool same = (e - b) == (re - rb);
    for (i64 p = 0; same && p < e - b; ++p) same = bytes[b + p] == bytes[rb + p];
    if (!same) *flag = 1;
  }
}

__global__ void fill_u64_kernel(unsigned long long* p, i64 n, unsigned long long v) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace
}  // namespace tdp

using namespace tdp;

extern "C" {

int tdp_string_hash(const uint8_t* bytes, const int64_t* offsets, int64_t n, int64_t* out_hash,
                    void* stream) {
  TDP_REQUIRE(n >= 0 && offsets != nullptr && out_hash != nullptr, "bad string hash arguments");
  if (n == 0) return TDP_OK;
  string_hash_kernel<<<stream_grid(n, 256, 16), 256, 0, as_stream(stream)>>>(bytes, offsets, n,
                                                                             out_hash);
  TDP_LAUNCH_CHECK("string_hash_kernel");
  return TDP_OK;
}

int tdp_string_groups(const uint8_t* bytes, const int64_t* offsets, int64_t n,
                      const int64_t* inverse, int64_t m, int64_t* out_first, int32_t* out_flag,
                      void* stream) {
  TDP_REQUIRE(n >= 0 && m >= 0 && m <= n, "bad string group arguments");
  cudaStream_t st = as_stream(stream);
  TDP_CUDA_TRY(cudaMemsetAsync(out_flag, 0, sizeof(int32_t), st));
  if (n == 0) return TDP_OK;
  unsigned long long* first = reinterpret_cast<unsigned long long*>(out_first);
  fill_u64_kernel<<<stream_grid(m, 256, 8), 256, 0, st>>>(first, m, ~0ull);
  TDP_LAUNCH_CHECK("fill_u64_kernel");
  group_first_kernel<<<stream_grid(n, 256, 16), 256, 0, st>>>(inverse, n, first);
  TDP_LAUNCH_CHECK("group_first_kernel");
  string_group_check_kernel<<<stream_grid(n, 256, 16), 256, 0, st>>>(bytes, offsets, inverse,
                                                                     first, n, out_flag);
  TDP_LAUNCH_CHECK("string_group_check_kernel");
  return TDP_OK;
}

}  // extern "C"
