// Library-level C ABI: error strings, version, device properties, and the
// host translation of predicate descriptors.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <mutex>
#include <vector>

#include "tdp_common.cuh"

namespace tdp {

static thread_local std::string g_error;
static std::atomic<unsigned long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static thread_local int g_replay_mode = 0;
static thread_local std::vector<i64> g_replay_log;
static thread_local size_t g_replay_pos = 0;

int replay_mode() { return g_replay_mode; }
void replay_push(i64 v) { g_replay_log.push_back(v); }
bool replay_take(i64* v) {
  if (g_replay_pos >= g_replay_log.size()) return false;
  *v = g_replay_log[g_replay_pos++];
  return true;
}

int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_error = buf;
  return code;
}

const char* last_error() { return g_error.c_str(); }

int sm_count() {
  static std::mutex mu;
  static std::vector<int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lock(mu);
  if ((int)cache.size() <= dev) cache.resize(dev + 1, 0);
  if (cache[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cache[dev] = v;
  }
  return cache[dev];
}

int make_predset(const tdp_column* cols, int32_t ncols, const tdp_predicate* preds,
                 int32_t npreds, int64_t n, PredSet* out) {
  TDP_REQUIRE(npreds >= 0 && npreds <= kMaxPreds, "at most %d predicates per filter (got %d)",
              kMaxPreds, npreds);
  TDP_REQUIRE(npreds == 0 || preds != nullptr, "null predicate array");
  out->npreds = npreds;
  out->pad = 0;
  for (int k = 0; k < npreds; ++k) {
    const tdp_predicate& p = preds[k];
    TDP_REQUIRE(p.op >= TDP_EQ && p.op <= TDP_GE, "predicate %d: bad operator %d", k, p.op);
    TDP_REQUIRE(p.cmp >= TDP_CMP_I64 && p.cmp <= TDP_CMP_BITMAP, "predicate %d: bad compare kind",
                k);
    TDP_REQUIRE(p.cmp != TDP_CMP_DEC || p.lit_i > 0, "predicate %d: decimal divisor must be > 0", k);
    DevPred& d = out->p[k];
    d.op = p.op;
    d.cmp = p.cmp;
    d.li = p.lit_i;
    d.lf = p.lit_f;
    d.pad = 0;
    d.bits = nullptr;
    if (p.cmp == TDP_CMP_BITMAP) {
      TDP_REQUIRE(p.reserved >= 0 && p.reserved < ncols, "predicate %d: bitmap column %d out of range",
                  k, p.reserved);
      TDP_REQUIRE(p.lit_f >= 1.0 && (double)cols[p.reserved].rows * 32.0 >= p.lit_f,
                  "predicate %d: bitmap shorter than its key range", k);
      d.bits = reinterpret_cast<const unsigned*>(cols[p.reserved].data);
    }
    if (p.cmp == TDP_CMP_NONE || p.cmp == TDP_CMP_ALL) {
      d.ptr = nullptr;
      d.dtype = TDP_I64;
      continue;
    }
    TDP_REQUIRE(p.column >= 0 && p.column < ncols, "predicate %d: column %d out of range", k,
                p.column);
    const tdp_column& c = cols[p.column];
    TDP_REQUIRE(c.width == 1, "predicate %d: filters require scalar columns", k);
    TDP_REQUIRE(c.rows >= n, "predicate %d: column has %lld rows < %lld", k, (long long)c.rows,
                (long long)n);
    TDP_REQUIRE(dtype_size(c.dtype) > 0, "predicate %d: bad column dtype %d", k, c.dtype);
    TDP_REQUIRE(n == 0 || c.data != nullptr, "predicate %d: null column", k);
    TDP_REQUIRE(p.cmp != TDP_CMP_DEC || c.dtype == TDP_I64 || c.dtype == TDP_I32 ||
                    c.dtype == TDP_I16 || c.dtype == TDP_I8 || c.dtype == TDP_U8,
                "predicate %d: decimal compare needs an integer column", k);
    d.ptr = c.data;
    d.dtype = c.dtype;
  }
  return TDP_OK;
}

constexpr int kMaxExpected = 16;  // a dense group-by's key ranges: 2 per key, <= 8 keys

struct Expected {
  i64 v[kMaxExpected];
};

// One thread per value: a replayed plan's device-computed integer must equal
// the value its buffers were sized from; anything else aborts the replay.
__global__ void expect_values_kernel(const void* got, int esize, int n, Expected e) {
  const int i = threadIdx.x;
  if (i >= n) return;
  const i64 v = esize == 8 ? reinterpret_cast<const i64*>(got)[i]
                           : (i64) reinterpret_cast<const int*>(got)[i];
  if (v != e.v[i]) {
    printf("tdp: replayed plan read %lld where %lld was recorded (catalog changed behind "
           "the replay signature)\n", (long long)v, (long long)e.v[i]);
    __trap();
  }
}

}  // namespace tdp

extern "C" {

int tdp_replay_log_begin(int32_t mode, const int64_t* values, int64_t n) {
  TDP_REQUIRE(mode >= 0 && mode <= 2, "replay log mode must be 0, 1 or 2");
  TDP_REQUIRE(n >= 0 && (n == 0 || values != nullptr), "bad replay log values");
  tdp::g_replay_mode = mode;
  tdp::g_replay_log.assign(values, values + (mode == 2 ? n : 0));
  tdp::g_replay_pos = 0;
  return TDP_OK;
}

int64_t tdp_replay_log_size(void) {
  return tdp::g_replay_mode == 2 ? (int64_t)tdp::g_replay_pos : (int64_t)tdp::g_replay_log.size();
}

int tdp_replay_log_end(int64_t* out, int64_t cap) {
  const int64_t n = (int64_t)tdp::g_replay_log.size();
  TDP_REQUIRE(cap >= n || tdp::g_replay_mode == 2, "replay log output too small");
  if (tdp::g_replay_mode == 1 && n) std::copy(tdp::g_replay_log.begin(), tdp::g_replay_log.end(), out);
  tdp::g_replay_mode = 0;
  tdp::g_replay_log.clear();
  tdp::g_replay_pos = 0;
  return TDP_OK;
}

int tdp_expect_values(const void* got, int32_t esize, int32_t n, const int64_t* expected,
                      void* stream) {
  TDP_REQUIRE(n >= 0 && n <= tdp::kMaxExpected, "tdp_expect_values: at most %d values (got %d)",
              tdp::kMaxExpected, n);
  TDP_REQUIRE(esize == 4 || esize == 8, "tdp_expect_values: element size must be 4 or 8");
  TDP_REQUIRE(n == 0 || (got != nullptr && expected != nullptr), "tdp_expect_values: null pointer");
  if (n == 0) return TDP_OK;
  tdp::Expected e;
  for (int i = 0; i < tdp::kMaxExpected; ++i) e.v[i] = i < n ? expected[i] : 0;
  tdp::expect_values_kernel<<<1, 32, 0, tdp::as_stream(stream)>>>(got, esize, n, e);
  TDP_LAUNCH_CHECK("expect_values_kernel");
  return TDP_OK;
}

const char* tdp_last_error(void) { return tdp::last_error(); }

const char* tdp_version(void) { return "tdp-b200 0.1.0 (sm_100a)"; }

int tdp_device_sm_count(void) { return tdp::sm_count(); }

uint64_t tdp_launch_count(void) { return tdp::g_launches.load(std::memory_order_relaxed); }

int tdp_clear_error(void) { return (int)cudaGetLastError(); }

void tdp_count_graph_launches(uint64_t n) {
  tdp::g_launches.fetch_add(n, std::memory_order_relaxed);
}

int tdp_stream_wait_event(void* stream, void* event) {
  TDP_REQUIRE(event != nullptr, "null event");
  TDP_CUDA_TRY(cudaStreamWaitEvent(tdp::as_stream(stream), reinterpret_cast<cudaEvent_t>(event), 0));
  return TDP_OK;
}

int tdp_replay_done(void* event, void* stream, uint64_t graph_launches) {
  TDP_REQUIRE(event != nullptr, "null event");
  tdp::g_launches.fetch_add(graph_launches, std::memory_order_relaxed);
  TDP_CUDA_TRY(cudaEventRecord(reinterpret_cast<cudaEvent_t>(event), tdp::as_stream(stream)));
  return TDP_OK;
}

}  // extern "C"
