// Shared infrastructure of libtdp_kernels: error reporting, dtype access,
// predicate evaluation, grid sizing.  Device code targets sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/tdp_kernels.h"

namespace tdp {

typedef int64_t i64;
typedef uint64_t u64;

// ---------------------------------------------------------------------------
// host-side error plumbing (thread-local message, returned by tdp_last_error)
// ---------------------------------------------------------------------------
int set_error(int code, const char* fmt, ...);
const char* last_error();

#define TDP_CUDA_TRY(expr)                                                              \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return ::tdp::set_error(TDP_ECUDA, "%s failed: %s (%s:%d)", #expr,                \
                              cudaGetErrorString(_e), __FILE__, __LINE__);              \
  } while (0)

// Counts every kernel this library launches (tdp_launch_count) so benchmarks
// can report how many of their launches were ours.
void count_launch();

// Replay log of host decisions taken inside the library from device data
// (the radix sort's skipped digit passes).  Mode 1 records every decision;
// mode 2 (a CUDA-graph capture) takes them from the log instead of
// synchronising -- the caller enqueues a device check of each.  Thread-local.
int replay_mode();
void replay_push(i64 v);
bool replay_take(i64* v);

#define TDP_LAUNCH_CHECK(name)                                                          \
  do {                                                                                  \
    cudaError_t _e = cudaGetLastError();                                                \
    if (_e != cudaSuccess)                                                              \
      return ::tdp::set_error(TDP_ECUDA, "launch of %s failed: %s", name,               \
                              cudaGetErrorString(_e));                                  \
    ::tdp::count_launch();                                                              \
  } while (0)

#define TDP_REQUIRE(cond, ...)                                                          \
  do {                                                                                  \
    if (!(cond)) return ::tdp::set_error(TDP_EINVAL, __VA_ARGS__);                      \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Number of SMs of the current device (cached per device ordinal).
int sm_count();
// benchmark timer (tdp_kernel_timer_enable): events around launches of `kind`
cudaEvent_t timer_begin(int kind, cudaStream_t st);
void timer_end(cudaEvent_t a, cudaStream_t st);

__host__ __device__ inline int dtype_size(int dt) {
  switch (dt) {
    case TDP_I64:
    case TDP_F64:
      return 8;
    case TDP_F32:
    case TDP_I32:
      return 4;
    case TDP_I16:
      return 2;
    case TDP_BOOL:
    case TDP_I8:
    case TDP_U8:
      return 1;
    default:
      return 0;
  }
}

inline i64 ceil_div(i64 a, i64 b) { return (a + b - 1) / b; }

// Grid for a grid-stride streaming kernel: enough CTAs to cover the work,
// capped at `per_sm` resident CTAs on every SM.
inline int stream_grid(i64 work_items, int items_per_cta, int per_sm) {
  i64 want = ceil_div(work_items > 0 ? work_items : 1, items_per_cta);
  i64 cap = (i64)sm_count() * per_sm;
  return (int)(want < cap ? want : cap);
}

// ---------------------------------------------------------------------------
// device-side column access
// ---------------------------------------------------------------------------
constexpr int kMaxPreds = 16;
constexpr int kMaxCols = 32;

struct DevPred {
  const void* ptr;
  int dtype;
  int op;
  int cmp;
  int pad;
  i64 li;
  double lf;
  const unsigned* bits;  // TDP_CMP_BITMAP: the semi-join bitmap
};

struct PredSet {
  int npreds;
  int pad;
  DevPred p[kMaxPreds];
};

// Bulk prefetch of [p, p + bytes) into L2 by the TMA engine (no registers,
// no shared memory): a tile-per-CTA streaming kernel asks for a tile the next
// wave of CTAs will read, so its HBM traffic no longer waits for the CTAs of
// this wave to finish their dependent (L2-latency) phase.  The range is
// widened to 16-byte bounds, which stay inside the allocation's last chunk.
__device__ __forceinline__ void l2_prefetch_range(const void* p, i64 bytes) {
  if (p == nullptr || bytes <= 0) return;
  const unsigned long long a = (unsigned long long)p & ~15ull;
  const unsigned long long e = ((unsigned long long)p + (unsigned long long)bytes + 15ull) & ~15ull;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(e - a))
               : "memory");
}

__device__ __forceinline__ i64 load_as_i64(const void* base, int dt, i64 i) {
  switch (dt) {
    case TDP_I64:
      return __ldg(reinterpret_cast<const i64*>(base) + i);
    case TDP_I32:
      return (i64)__ldg(reinterpret_cast<const int*>(base) + i);
    case TDP_I16:
      return (i64)__ldg(reinterpret_cast<const short*>(base) + i);
    case TDP_I8:
      return (i64)__ldg(reinterpret_cast<const signed char*>(base) + i);
    case TDP_BOOL:
    case TDP_U8:
      return (i64)reinterpret_cast<const unsigned char*>(base)[i];
    case TDP_F64:
      return (i64)__ldg(reinterpret_cast<const double*>(base) + i);
    default:
      return (i64)__ldg(reinterpret_cast<const float*>(base) + i);
  }
}

__device__ __forceinline__ double load_as_f64(const void* base, int dt, i64 i) {
  switch (dt) {
    case TDP_F64:
      return __ldg(reinterpret_cast<const double*>(base) + i);
    case TDP_F32:
      return (double)__ldg(reinterpret_cast<const float*>(base) + i);
    case TDP_I64:
      return (double)__ldg(reinterpret_cast<const i64*>(base) + i);
    case TDP_I32:
      return (double)__ldg(reinterpret_cast<const int*>(base) + i);
    case TDP_I16:
      return (double)__ldg(reinterpret_cast<const short*>(base) + i);
    case TDP_I8:
      return (double)__ldg(reinterpret_cast<const signed char*>(base) + i);
    default:
      return (double)reinterpret_cast<const unsigned char*>(base)[i];
  }
}

__device__ __forceinline__ float load_as_f32(const void* base, int dt, i64 i) {
  switch (dt) {
    case TDP_F32:
      return __ldg(reinterpret_cast<const float*>(base) + i);
    case TDP_F64:
      return (float)__ldg(reinterpret_cast<const double*>(base) + i);
    case TDP_I64:
      return (float)__ldg(reinterpret_cast<const i64*>(base) + i);
    case TDP_I32:
      return (float)__ldg(reinterpret_cast<const int*>(base) + i);
    default:
      return (float)reinterpret_cast<const unsigned char*>(base)[i];
  }
}

template <class T>
__device__ __forceinline__ bool compare(T x, T y, int op) {
  switch (op) {
    case TDP_EQ:
      return x == y;
    case TDP_NE:
      return x != y;
    case TDP_LT:
      return x < y;
    case TDP_GT:
      return x > y;
    case TDP_LE:
      return x <= y;
    default:
      return x >= y;
  }
}

// One comparison with the promotion the host resolved (numpy NEP 50 rules).
__device__ __forceinline__ bool eval_pred(const DevPred& p, i64 i) {
  switch (p.cmp) {
    case TDP_CMP_I64:
      return compare<i64>(load_as_i64(p.ptr, p.dtype, i), p.li, p.op);
    case TDP_CMP_F64:
      return compare<double>(load_as_f64(p.ptr, p.dtype, i), p.lf, p.op);
    case TDP_CMP_F32:
      return compare<float>(load_as_f32(p.ptr, p.dtype, i), (float)p.lf, p.op);
    case TDP_CMP_DEC:
      return compare<double>((double)load_as_i64(p.ptr, p.dtype, i) / (double)p.li, p.lf, p.op);
    case TDP_CMP_NONE:
      return false;
    case TDP_CMP_BITMAP: {
      const unsigned long long x = (unsigned long long)load_as_i64(p.ptr, p.dtype, i) -
                                   (unsigned long long)p.li;
      return x < (unsigned long long)(i64)p.lf && ((__ldg(p.bits + (x >> 5)) >> (x & 31)) & 1u);
    }
    default:
      return true;
  }
}

__device__ __forceinline__ bool eval_all(const PredSet& ps, i64 i) {
  bool keep = true;
  for (int k = 0; k < ps.npreds; ++k) keep &= eval_pred(ps.p[k], i);
  return keep;
}

// Branch-free comparison (numpy semantics: every comparison with NaN is false
// except <>, which is true).
template <class T>
__device__ __forceinline__ bool compare_nb(T x, T y, int op) {
  const bool lt = x < y, gt = x > y, eq = x == y;
  return (op == TDP_EQ && eq) | (op == TDP_NE && !eq) | (op == TDP_LT && lt) |
         (op == TDP_GT && gt) | (op == TDP_LE && (lt | eq)) | (op == TDP_GE && (gt | eq));
}

// keep[r] &= v[r] <op> lit with the operator resolved once, outside the
// row loop (two compares per 64-bit row instead of a six-way select).
template <int R, class T>
__device__ __forceinline__ void cmp_rows(const T (&v)[R], T lit, int op, bool (&keep)[R]) {
  switch (op) {
    case TDP_EQ:
#pragma unroll
      for (int r = 0; r < R; ++r) keep[r] = keep[r] && v[r] == lit;
      break;
    case TDP_NE:
#pragma unroll
      for (int r = 0; r < R; ++r) keep[r] = keep[r] && !(v[r] == lit);
      break;
    case TDP_LT:
#pragma unroll
      for (int r = 0; r < R; ++r) keep[r] = keep[r] && v[r] < lit;
      break;
    case TDP_GT:
#pragma unroll
      for (int r = 0; r < R; ++r) keep[r] = keep[r] && v[r] > lit;
      break;
    case TDP_LE:
#pragma unroll
      for (int r = 0; r < R; ++r) keep[r] = keep[r] && v[r] <= lit;
      break;
    default:
#pragma unroll
      for (int r = 0; r < R; ++r) keep[r] = keep[r] && v[r] >= lit;
      break;
  }
}

// Predicate-major evaluation of the conjunction over R rows of one thread:
// for each predicate, the loads of all still-selected rows are issued
// together (R independent loads in flight instead of one row's dependent
// chain of switches).  row[r] must be a valid row wherever keep[r] is true.
template <int R>
__device__ __forceinline__ void eval_batch(const PredSet& ps, const i64 (&row)[R], bool (&keep)[R]) {
  // the later predicates' loads depend on the earlier ones' outcome: start
  // their lines towards L2 now, so each later round waits on L2, not DRAM
  for (int k = 1; k < ps.npreds; ++k) {
    const int es = dtype_size(ps.p[k].dtype);
    const char* base = reinterpret_cast<const char*>(ps.p[k].ptr);
    if (base == nullptr || es == 0) continue;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (keep[r]) asm volatile("prefetch.global.L2 [%0];" ::"l"(base + row[r] * es));
  }
  for (int k = 0; k < ps.npreds; ++k) {
    const int cmp = ps.p[k].cmp, dt = ps.p[k].dtype, op = ps.p[k].op;
    const void* ptr = ps.p[k].ptr;
    if (cmp == TDP_CMP_NONE) {
#pragma unroll
      for (int r = 0; r < R; ++r) keep[r] = false;
    } else if (cmp == TDP_CMP_ALL) {
      continue;
    } else if (cmp == TDP_CMP_I64 && dt == TDP_I64) {
      const i64* c = reinterpret_cast<const i64*>(ptr);
      i64 v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = keep[r] ? __ldg(c + row[r]) : 0;
      cmp_rows<R, i64>(v, ps.p[k].li, op, keep);
    } else if (cmp == TDP_CMP_F64 && dt == TDP_F64) {
      const double* c = reinterpret_cast<const double*>(ptr);
      double v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = keep[r] ? __ldg(c + row[r]) : 0.0;
      cmp_rows<R, double>(v, ps.p[k].lf, op, keep);
    } else if (cmp == TDP_CMP_BITMAP && dt == TDP_I64) {
      // semi-join membership: R key loads, then R bitmap-word loads in flight
      const i64* c = reinterpret_cast<const i64*>(ptr);
      unsigned long long x[R];
      unsigned w[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        x[r] = keep[r] ? (unsigned long long)__ldg(c + row[r]) - (unsigned long long)ps.p[k].li : 0ull;
        keep[r] = keep[r] && x[r] < (unsigned long long)(i64)ps.p[k].lf;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) w[r] = keep[r] ? __ldg(ps.p[k].bits + (x[r] >> 5)) : 0u;
#pragma unroll
      for (int r = 0; r < R; ++r) keep[r] = keep[r] && ((w[r] >> (x[r] & 31)) & 1u);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) keep[r] = keep[r] && eval_pred(ps.p[k], row[r]);
    }
  }
}

// L2 prefetch of rows [row0, row0 + rows) of every predicate column
__device__ __forceinline__ void prefetch_predset_l2(const PredSet& ps, i64 row0, i64 rows) {
  for (int k = 0; k < ps.npreds; ++k) {
    const int es = dtype_size(ps.p[k].dtype);
    if (ps.p[k].cmp == TDP_CMP_NONE || ps.p[k].cmp == TDP_CMP_ALL || es == 0) continue;
    l2_prefetch_range(reinterpret_cast<const char*>(ps.p[k].ptr) + row0 * es, rows * es);
  }
}

// eval_batch with every predicate's column loaded for all R rows up front
// (one round of independent loads instead of one per predicate; a bitmap
// membership test adds one dependent round for its words) when the set is
// at most kUpfront predicates on 8-byte columns; else eval_batch.
constexpr int kUpfront = 3;

template <int R>
__device__ __forceinline__ void eval_batch_upfront(const PredSet& ps, const i64 (&row)[R],
                                                   bool (&keep)[R]) {
  bool simple = ps.npreds <= kUpfront;
  for (int k = 0; k < ps.npreds && simple; ++k) {
    const int cmp = ps.p[k].cmp, dt = ps.p[k].dtype;
    simple = (cmp == TDP_CMP_I64 && dt == TDP_I64) || (cmp == TDP_CMP_F64 && dt == TDP_F64) ||
             (cmp == TDP_CMP_BITMAP && dt == TDP_I64);
  }
  if (!simple) {
    eval_batch<R>(ps, row, keep);
    return;
  }
  i64 v[kUpfront][R];
#pragma unroll
  for (int k = 0; k < kUpfront; ++k)
    if (k < ps.npreds) {
      const i64* c = reinterpret_cast<const i64*>(ps.p[k].ptr);
#pragma unroll
      for (int r = 0; r < R; ++r) v[k][r] = keep[r] ? __ldg(c + row[r]) : 0;
    }
#pragma unroll
  for (int k = 0; k < kUpfront; ++k) {
    if (k >= ps.npreds) break;
    const DevPred& p = ps.p[k];
    if (p.cmp == TDP_CMP_I64) {
      cmp_rows<R, i64>(v[k], p.li, p.op, keep);
    } else if (p.cmp == TDP_CMP_F64) {
      double f[R];
#pragma unroll
      for (int r = 0; r < R; ++r) f[r] = __longlong_as_double(v[k][r]);
      cmp_rows<R, double>(f, p.lf, p.op, keep);
    } else {  // bitmap membership
      unsigned w[R];
      unsigned long long x[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        x[r] = (unsigned long long)v[k][r] - (unsigned long long)p.li;
        keep[r] = keep[r] && x[r] < (unsigned long long)(i64)p.lf;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) w[r] = keep[r] ? __ldg(p.bits + (x[r] >> 5)) : 0u;
#pragma unroll
      for (int r = 0; r < R; ++r) keep[r] = keep[r] && ((w[r] >> (x[r] & 31)) & 1u);
    }
  }
}

// Host: translate public descriptors into the device predicate set.
int make_predset(const tdp_column* cols, int32_t ncols, const tdp_predicate* preds,
                 int32_t npreds, int64_t n, PredSet* out);

// ---------------------------------------------------------------------------
// warp / block helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// mbarrier + bulk async copy (TMA engine) helpers for shared-memory rings
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "TDP_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra TDP_DONE;\n"
      "bra TDP_WAIT;\n"
      "TDP_DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// global -> shared bulk copy; bytes and both addresses 16-byte aligned
__device__ __forceinline__ void bulk_load(unsigned dst, const void* src, unsigned bytes,
                                          unsigned bar, unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}

// Exclusive scan of int64 block counts; writes offsets and the total.
// Lives in scan.cu; used by filter compaction, sort and join.
int exclusive_scan_i64(const i64* in, i64* out, i64 n, i64* total, void* ws, size_t ws_bytes,
                       cudaStream_t stream);
size_t exclusive_scan_workspace(i64 n);

// Filter tiling shared by compaction and the JIT projection pass: a CTA of
// kFilterThreads threads owns kFilterTile consecutive rows, evaluated as
// kFilterTile/32 ballot words in row order.
constexpr int kFilterThreads = 256;
constexpr int kFilterTile = 4096;
constexpr int kFilterWords = kFilterTile / 32;

// mask pass: bitmask words + per-tile counts (internal to filter.cu).
int filter_bits(const PredSet& ps, int64_t n, unsigned* bits, i64* tile_counts,
                cudaStream_t stream);

// ---------------------------------------------------------------------------
// softmax helpers (soft.cu, llp.cu)
// ---------------------------------------------------------------------------
template <class T>
__device__ __forceinline__ T t_exp(T x);
template <>
__device__ __forceinline__ float t_exp<float>(float x) {
  return expf(x);
}
template <>
__device__ __forceinline__ double t_exp<double>(double x) {
  return exp(x);
}

// numpy max propagates NaN; keep that so exp(x - NaN) poisons the row as in
// the reference.
template <class T>
__device__ __forceinline__ T nan_max(T a, T b) {
  return (b > a || b != b) ? b : a;
}

}  // namespace tdp
