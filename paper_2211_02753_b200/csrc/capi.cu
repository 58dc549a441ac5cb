// Library-level C ABI: error strings, version, device properties, and the
// host translation of predicate descriptors.
#include <atomic>
#include <mutex>
#include <vector>

#include "tdp_common.cuh"

namespace tdp {

static thread_local std::string g_error;
static std::atomic<unsigned long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

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
    TDP_REQUIRE(p.cmp >= TDP_CMP_I64 && p.cmp <= TDP_CMP_DEC, "predicate %d: bad compare kind",
                k);
    TDP_REQUIRE(p.cmp != TDP_CMP_DEC || p.lit_i > 0, "predicate %d: decimal divisor must be > 0", k);
    DevPred& d = out->p[k];
    d.op = p.op;
    d.cmp = p.cmp;
    d.li = p.lit_i;
    d.lf = p.lit_f;
    d.pad = 0;
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

}  // namespace tdp

extern "C" {

const char* tdp_last_error(void) { return tdp::last_error(); }

const char* tdp_version(void) { return "tdp-b200 0.1.0 (sm_100a)"; }

int tdp_device_sm_count(void) { return tdp::sm_count(); }

uint64_t tdp_launch_count(void) { return tdp::g_launches.load(std::memory_order_relaxed); }

int tdp_clear_error(void) { return (int)cudaGetLastError(); }

void tdp_count_graph_launches(uint64_t n) {
  tdp::g_launches.fetch_add(n, std::memory_order_relaxed);
}

}  // extern "C"
