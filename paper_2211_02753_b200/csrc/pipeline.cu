// Fused scan -> filter -> elementwise expression -> dense grouped aggregate.
//
// Replaces, in ONE pass over the base columns, the reference's operator-at-a-
// time chain (tq = /root/reference/pkg/src/tensorquery):
//   FilterOp  -> filter_exact        tq/compiler.py:146-150, tq/kernels.py:87-97
//   TvfOp     -> elementwise UDF     tq/compiler.py:114-122 (add/sub/mul/... tq/tensor.py:330-412)
//   GroupAggExactOp -> groupby_exact tq/compiler.py:176-203, tq/kernels.py:108-167
//                   or _global_aggregate tq/compiler.py:206-215
// The reference moves every surviving row of every column through three
// materialisations; here the base columns are read once and nothing per-row is
// written.
//
// The query-specific part (column loads, predicate conjunction, the SSA
// expression program, the key -> slot map and the aggregate inputs) is emitted
// as CUDA C++ and compiled once per distinct program by NVRTC for sm_100a; the
// kernel body is the hand-written skeleton in pipeline_skeleton.cuh.  Literals
// and constants are kernel parameters, so only the program SHAPE keys the cache.
#include <cuda.h>
#include <nvrtc.h>

#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <vector>

#include "tdp_common.cuh"

namespace tdp {

namespace {

#include "pipeline_skeleton.inc"  // static const char* kSkeleton

constexpr int kThreads = 256;
constexpr int kUnroll = 4;
constexpr int kMaxInstr = 64;
constexpr int kMaxKeys = 8;
constexpr int kMaxOuts = 16;
constexpr int kMaxRegCells = 64;
constexpr i64 kMaxSlots = 1 << 20;
constexpr int kConsWarps = 8;               // consumer warps of the ring kernel
constexpr i64 kStageBudget = 64 * 1024;     // max bytes of one ring stage
// bytes of shared memory for the ring + accumulators of one CTA
// (env TDP_RING_BUDGET_KB overrides, for measurements)
static i64 ring_budget() {
  static const i64 v = [] {
    const char* e = getenv("TDP_RING_BUDGET_KB");
    return e ? (i64)atoll(e) * 1024 : (i64)200 * 1024;
  }();
  return v;
}
#define kRingBudget ring_budget()
constexpr i64 kTwoCtaBudget = 110 * 1024;   // ring + accumulators per CTA at 2 CTAs/SM
// rows up to this many bytes prefer two CTAs per SM (env TDP_TWO_CTA_ROW_BYTES
// overrides, for measurements)
static i64 two_cta_row_bytes() {
  static const i64 v = [] {
    const char* e = getenv("TDP_TWO_CTA_ROW_BYTES");
    return e ? (i64)atoll(e) : (i64)32;
  }();
  return v;
}
#define kTwoCtaRowBytes two_cta_row_bytes()
constexpr i64 kMaxSmemCells = 48;           // shared-memory accumulator mode limit
constexpr int kAccThreads = 256;            // accumulator columns (TDP_ACC_THREADS)
constexpr int kMaxPackWords = 8;            // packed per-thread accumulator words
constexpr int kMaxIvals = 32;               // integer accumulators (<= aggregates)

// Must match the TdpParams emitted below, field for field.
struct HostParams {
  const void* col[kMaxCols];
  void* out[kMaxOuts];
  i64 n;
  i64 pli[kMaxPreds];
  double plf[kMaxPreds];
  i64 imi[kMaxInstr];
  double imf[kMaxInstr];
  i64 klo[kMaxKeys];
  void* acc;
  const unsigned* bits;
  const i64* tile_off;
  i64 plo[kMaxIvals];     // per integer accumulator: bias of its packed field
};

// ---------------------------------------------------------------------------
// driver API through the runtime's entry-point query (no libcuda link, so the
// library also loads on hosts without a driver)
// ---------------------------------------------------------------------------
typedef CUresult (*PFN_ModuleLoadData)(CUmodule*, const void*);
typedef CUresult (*PFN_ModuleGetFunction)(CUfunction*, CUmodule, const char*);
typedef CUresult (*PFN_LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned,
                                     unsigned, unsigned, CUstream, void**, void**);
typedef CUresult (*PFN_Occupancy)(int*, CUfunction, int, size_t);
typedef CUresult (*PFN_GetErrorString)(CUresult, const char**);
typedef CUresult (*PFN_FuncSetAttribute)(CUfunction, CUfunction_attribute, int);

struct Driver {
  PFN_ModuleLoadData load = nullptr;
  PFN_ModuleGetFunction getfn = nullptr;
  PFN_LaunchKernel launch = nullptr;
  PFN_Occupancy occupancy = nullptr;
  PFN_GetErrorString errstr = nullptr;
  PFN_FuncSetAttribute setattr = nullptr;
  bool ok = false;
};

int get_driver(Driver** out) {
  static Driver d;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    auto q = [](const char* sym, void** fp) -> bool {
      cudaDriverEntryPointQueryResult st;
      cudaError_t e = cudaGetDriverEntryPoint(sym, fp, cudaEnableDefault, &st);
      return e == cudaSuccess && st == cudaDriverEntryPointSuccess && *fp != nullptr;
    };
    bool ok = q("cuModuleLoadData", (void**)&d.load) &&
              q("cuModuleGetFunction", (void**)&d.getfn) &&
              q("cuLaunchKernel", (void**)&d.launch) &&
              q("cuOccupancyMaxActiveBlocksPerMultiprocessor", (void**)&d.occupancy) &&
              q("cuGetErrorString", (void**)&d.errstr) &&
              q("cuFuncSetAttribute", (void**)&d.setattr);
    d.ok = ok;
    if (!ok) err = "driver entry points unavailable";
  });
  if (!d.ok) return set_error(TDP_ECUDA, "%s", err.c_str());
  *out = &d;
  return TDP_OK;
}

int cu_check(Driver* d, CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return TDP_OK;
  const char* s = "?";
  if (d && d->errstr) d->errstr(r, &s);
  return set_error(TDP_ECUDA, "%s failed: %s", what, s);
}

// ---------------------------------------------------------------------------
// code generation
// ---------------------------------------------------------------------------
const char* ctype_of(int dt) {
  switch (dt) {
    case TDP_I64:
      return "i64";
    case TDP_F64:
      return "double";
    case TDP_F32:
      return "float";
    case TDP_I32:
      return "int";
    case TDP_I16:
      return "short";
    case TDP_I8:
      return "signed char";
    default:
      return "unsigned char";
  }
}

const char* op_sym(int op) {
  switch (op) {
    case TDP_EQ:
      return "==";
    case TDP_NE:
      return "!=";
    case TDP_LT:
      return "<";
    case TDP_GT:
      return ">";
    case TDP_LE:
      return "<=";
    default:
      return ">=";
  }
}

// Internal aggregate kind (never passed in by callers): SUM of a float64 value
// that the program computes exactly as scaled integers (decimal columns kept
// as integers by compact storage, exact decimal constants, + - *): the sum is
// accumulated exactly in integers and converted once, sum / scale, at the end.
constexpr int kAggSumDec = 3;

// Closed interval of an int64 program value, when it provably never wraps.
struct Range {
  bool ok = false;
  i64 lo = 0, hi = 0;
};

// One accumulator packed into a 64-bit per-thread word (shared-memory mode):
// the word receives (v - lo) << off per kept row, so every field stays
// non-negative and fields never borrow from each other.
struct Field {
  int acc;   // -1: the row count, else an integer accumulator (ival index)
  int word;
  int off;
  int bits;   // field width: the sum of up to rows-per-thread values
  i64 lo;     // bias subtracted from every value (min(range lo, 0))
  int rbits;  // width of one biased value
};

struct Spec {
  // inputs
  std::vector<int> col_dtype;  // per column
  std::vector<tdp_predicate> preds;
  std::vector<tdp_instr> prog;
  std::vector<tdp_key> keys;
  std::vector<tdp_agg> aggs;
  std::vector<int> outs;
  // derived
  std::vector<int> used_cols;
  std::vector<int> fvals, ivals;  // accumulator -> program value
  std::vector<int> agg_acc;       // agg -> accumulator index (-1 for count)
  std::vector<double> agg_scale;  // per agg: decimal scale of a kAggSumDec sum, else 0
  std::vector<double> iscale;     // per ival: 0 (plain SUM_I64) or the decimal scale
  i64 slots = 1;
  int accmode = 0;       // 0 registers, 1 shared-memory columns, 2 global atomics
  bool regacc = true;    // per-CTA partial rows (modes 0 and 1)
  i64 acc_smem = 0;      // bytes of shared-memory accumulators (mode 1)
  // shared-memory mode: packed per-thread words (count + bounded integer sums)
  std::vector<Field> fields;
  int pwords = 0;
  std::vector<int> iu;   // per ival: unpacked cell index, or -1 when packed
  i64 sm_rows = 0;       // u64 rows of TDP_ACC_THREADS words
};

// ---------------------------------------------------------------------------
// exact decimal aggregation
// ---------------------------------------------------------------------------
constexpr i64 kRangeLimit = (i64)1 << 62;

Range type_range(int dt) {
  Range r;
  r.ok = true;
  switch (dt) {
    case TDP_I8: r.lo = -128; r.hi = 127; break;
    case TDP_U8: r.lo = 0; r.hi = 255; break;
    case TDP_BOOL: r.lo = 0; r.hi = 1; break;
    case TDP_I16: r.lo = -32768; r.hi = 32767; break;
    case TDP_I32: r.lo = INT32_MIN; r.hi = INT32_MAX; break;
    default: r.ok = false;
  }
  return r;
}

Range make_range(__int128 lo, __int128 hi) {
  Range r;
  r.ok = lo >= -(__int128)kRangeLimit && hi <= (__int128)kRangeLimit;
  r.lo = r.ok ? (i64)lo : 0;
  r.hi = r.ok ? (i64)hi : 0;
  return r;
}

// Interval of every int64 program value (others: !ok).  A LOAD with b == 1
// carries the caller's promise that the stored values lie in [imm_i, imm_f]
// (compact storage measures it at ingestion).
std::vector<Range> value_ranges(const Spec& s) {
  std::vector<Range> R(s.prog.size());
  for (size_t j = 0; j < s.prog.size(); ++j) {
    const tdp_instr& in = s.prog[j];
    if (in.dtype != TDP_I64) continue;
    const Range a = in.a >= 0 && in.a < (int)j ? R[in.a] : Range();
    const Range b = in.b >= 0 && in.b < (int)j ? R[in.b] : Range();
    switch (in.op) {
      case TDP_OP_LOAD: {
        Range t = type_range(s.col_dtype[in.a]);
        if (in.b == 1) {
          const i64 hlo = in.imm_i, hhi = (i64)in.imm_f;
          if (!t.ok) t = make_range(hlo, hhi);
          else if (hlo >= t.lo && hhi <= t.hi && hlo <= hhi) t = make_range(hlo, hhi);
        }
        R[j] = t;
        break;
      }
      case TDP_OP_CONST: R[j] = make_range(in.imm_i, in.imm_i); break;
      case TDP_OP_CAST: R[j] = s.prog[in.a].dtype == TDP_I64 ? a : Range(); break;
      case TDP_OP_ADD:
        if (a.ok && b.ok) R[j] = make_range((__int128)a.lo + b.lo, (__int128)a.hi + b.hi);
        break;
      case TDP_OP_SUB:
        if (a.ok && b.ok) R[j] = make_range((__int128)a.lo - b.hi, (__int128)a.hi - b.lo);
        break;
      case TDP_OP_MUL:
        if (a.ok && b.ok) {
          const __int128 p[4] = {(__int128)a.lo * b.lo, (__int128)a.lo * b.hi,
                                 (__int128)a.hi * b.lo, (__int128)a.hi * b.hi};
          __int128 lo = p[0], hi = p[0];
          for (int k = 1; k < 4; ++k) {
            lo = p[k] < lo ? p[k] : lo;
            hi = p[k] > hi ? p[k] : hi;
          }
          R[j] = make_range(lo, hi);
        }
        break;
      case TDP_OP_NEG:
        if (a.ok) R[j] = make_range(-(__int128)a.hi, -(__int128)a.lo);
        break;
      case TDP_OP_SQUARE:
        if (a.ok) {
          const __int128 l2 = (__int128)a.lo * a.lo, h2 = (__int128)a.hi * a.hi;
          const __int128 mx = l2 > h2 ? l2 : h2;
          R[j] = a.lo >= 0 ? make_range(l2, h2) : a.hi <= 0 ? make_range(h2, l2) : make_range(0, mx);
        }
        break;
      case TDP_OP_RELU:
        if (a.ok) R[j] = make_range(a.lo > 0 ? a.lo : 0, a.hi > 0 ? a.hi : 0);
        break;
      default:
        break;
    }
  }
  return R;
}

struct Exact {
  int v = -1;     // int64 program value
  i64 scale = 0;  // value of the float64 = v / scale, exactly
};

int push_instr(Spec& s, int op, int a, int b, i64 imm_i) {
  if ((int)s.prog.size() >= kMaxInstr) return -1;
  tdp_instr in;
  in.op = op;
  in.dtype = TDP_I64;
  in.a = a;
  in.b = b;
  in.imm_i = imm_i;
  in.imm_f = 0.0;
  s.prog.push_back(in);
  return (int)s.prog.size() - 1;
}

// Exact scaled decimal of a small-magnitude float constant: m / 10^k == c.
bool exact_const(double c, i64* m, i64* scale) {
  i64 p = 1;
  for (int k = 0; k <= 6; ++k, p *= 10) {
    const double x = c * (double)p;
    if (!(x > -9.0e15 && x < 9.0e15)) return false;
    const double r = nearbyint(x);
    if ((double)(i64)r / (double)p == c) {
      *m = (i64)r;
      *scale = p;
      return true;
    }
  }
  return false;
}

// The float64 program value `v` restated over int64 values with a scale, or
// false.  Emits the integer instructions it needs (memoised per value).
bool exact_of(Spec& s, int v, std::map<int, Exact>& memo, Exact* out) {
  auto it = memo.find(v);
  if (it != memo.end()) {
    *out = it->second;
    return out->v >= 0;
  }
  memo[v] = Exact();  // in progress / failed
  const tdp_instr in = s.prog[v];
  Exact e;
  if (in.dtype != TDP_F64) return false;
  switch (in.op) {
    case TDP_OP_DECIMAL: {
      const double d = in.imm_f;
      if (!(d >= 1.0 && d <= 1e9 && d == nearbyint(d))) return false;
      e.v = in.a;
      e.scale = (i64)d;
      break;
    }
    case TDP_OP_CAST:
      if (s.prog[in.a].dtype != TDP_I64) return false;
      e.v = in.a;
      e.scale = 1;
      break;
    case TDP_OP_CONST: {
      i64 m = 0, sc = 1;
      if (!exact_const(in.imm_f, &m, &sc)) return false;
      e.v = push_instr(s, TDP_OP_CONST, 0, 0, m);
      e.scale = sc;
      break;
    }
    case TDP_OP_NEG:
    case TDP_OP_SQUARE: {
      Exact a;
      if (!exact_of(s, in.a, memo, &a)) return false;
      if (in.op == TDP_OP_SQUARE && a.scale > ((i64)1 << 26)) return false;
      e.v = push_instr(s, in.op, a.v, 0, 0);
      e.scale = in.op == TDP_OP_SQUARE ? a.scale * a.scale : a.scale;
      break;
    }
    case TDP_OP_ADD:
    case TDP_OP_SUB:
    case TDP_OP_MUL: {
      Exact a, b;
      if (!exact_of(s, in.a, memo, &a) || !exact_of(s, in.b, memo, &b)) return false;
      if (in.op == TDP_OP_MUL) {
        if ((__int128)a.scale * b.scale > ((i64)1 << 53)) return false;
        e.v = push_instr(s, TDP_OP_MUL, a.v, b.v, 0);
        e.scale = a.scale * b.scale;
        break;
      }
      // common scale: one scale must divide the other (powers of ten do)
      const i64 hi = a.scale > b.scale ? a.scale : b.scale;
      if (hi % a.scale || hi % b.scale) return false;
      // x * factor (a constant operand is folded: no per-row multiply)
      auto rescale = [&s](int v, i64 factor) -> int {
        if (factor == 1) return v;
        const tdp_instr& c = s.prog[v];
        if (c.op == TDP_OP_CONST && c.dtype == TDP_I64) {
          const __int128 m = (__int128)c.imm_i * factor;
          if (m > -(__int128)kRangeLimit && m < (__int128)kRangeLimit)
            return push_instr(s, TDP_OP_CONST, 0, 0, (i64)m);
        }
        const int f = push_instr(s, TDP_OP_CONST, 0, 0, factor);
        return f < 0 ? -1 : push_instr(s, TDP_OP_MUL, v, f, 0);
      };
      const int av = rescale(a.v, hi / a.scale);
      const int bv = av < 0 ? -1 : rescale(b.v, hi / b.scale);
      if (av < 0 || bv < 0) return false;
      e.v = push_instr(s, in.op, av, bv, 0);
      e.scale = hi;
      break;
    }
    default:
      return false;
  }
  if (e.v < 0) return false;
  memo[v] = e;
  *out = e;
  return true;
}

i64 ceil_pow2(i64 x) {
  i64 p = 1;
  while (p < x) p <<= 1;
  return p;
}

int bits_for(unsigned __int128 x) {  // bits of the largest value a field must hold
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b > 0 ? b : 1;
}

// Rows one accumulating thread can see: every kernel variant runs 256
// accumulating threads per CTA and at least one CTA per SM (or <= 4 rows per
// thread when the grid is smaller), so n / (256 * SMs) plus a tile's rows;
// rounded up to a power of two so the packing (part of the kernel's cache
// key) changes only when n doubles.
i64 rows_per_thread_bound(i64 n) {
  const i64 sms = sm_count() > 0 ? sm_count() : 148;
  return ceil_pow2(n / (256 * sms) + 16);
}

// SUM over a float64 value computed exactly from scaled integers -> exact
// integer accumulation (kAggSumDec), when the integer program cannot wrap and
// a CTA's partial sum fits int64.  Changes no result beyond the rounding of
// the float path (the sum of the exact row values, rounded once).
void convert_decimal_sums(Spec& s, i64 n) {
  std::map<int, Exact> memo;
  const size_t keep = s.prog.size();
  std::vector<std::pair<int, Exact>> conv;  // agg -> exact
  for (size_t a = 0; a < s.aggs.size(); ++a) {
    if (s.aggs[a].kind != TDP_AGG_SUM_F64) continue;
    Exact e;
    if (exact_of(s, s.aggs[a].value, memo, &e)) conv.emplace_back((int)a, e);
  }
  if (conv.empty()) {
    s.prog.resize(keep);
    return;
  }
  const std::vector<Range> R = value_ranges(s);
  const i64 per_cta = s.accmode == 2 ? (n > 0 ? n : 1) : rows_per_thread_bound(n) * 256;
  bool any = false;
  for (auto& ce : conv) {
    const Range& r = R[ce.second.v];
    if (!r.ok) continue;
    const i64 mag = r.hi > -r.lo ? r.hi : -r.lo;
    if ((__int128)mag * per_cta >= ((__int128)1 << 63)) continue;
    s.aggs[ce.first].kind = kAggSumDec;
    s.aggs[ce.first].value = ce.second.v;
    any = true;
  }
  if (!any) s.prog.resize(keep);
  s.agg_scale.assign(s.aggs.size(), 0.0);
  for (auto& ce : conv)
    if (s.aggs[ce.first].kind == kAggSumDec) s.agg_scale[ce.first] = (double)ce.second.scale;
}

// Shared-memory accumulators: pack the row count and every bounded integer
// sum into as few per-thread 64-bit words as their ranges allow (first fit,
// widest first).  Q1 on compact storage: count + 5 sums in 3 words instead of
// a 32-bit count and five 64-bit cells (48 instead of 88 bytes of shared-memory
// read-modify-write per row).
void pack_fields(Spec& s, i64 n) {
  s.fields.clear();
  s.pwords = 0;
  s.iu.assign(s.ivals.size(), -1);
  const std::vector<Range> R = value_ranges(s);
  const unsigned __int128 rows = (unsigned __int128)rows_per_thread_bound(n);
  std::vector<Field> cand;
  cand.push_back(Field{-1, 0, 0, bits_for(rows), 0, 1});
  for (size_t k = 0; k < s.ivals.size(); ++k) {
    const Range& r = R[s.ivals[k]];
    if (!r.ok) continue;
    // biased by min(lo, 0): non-negative ranges need no per-row subtract
    const i64 bias = r.lo < 0 ? r.lo : 0;
    const unsigned __int128 span = (unsigned __int128)((__int128)r.hi - bias);
    const int b = bits_for(span * rows);
    if (b <= 62) cand.push_back(Field{(int)k, 0, 0, b, bias, bits_for(span)});
  }
  std::vector<int> order(cand.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int x, int y) { return cand[x].bits > cand[y].bits; });
  std::vector<int> used;
  for (int i : order) {
    Field f = cand[i];
    int w = 0;
    while (w < (int)used.size() && used[w] + f.bits > 64) ++w;
    if (w == (int)used.size()) {
      if ((int)used.size() == kMaxPackWords) continue;
      used.push_back(0);
    }
    f.word = w;
    f.off = used[w];
    used[w] += f.bits;
    s.fields.push_back(f);
  }
  bool count_packed = false;
  for (const Field& f : s.fields) count_packed |= f.acc < 0;
  // worth it only when some word holds two fields
  if (!count_packed || used.size() >= s.fields.size()) {
    // not packed: every integer sum keeps its own cell (iu[k] = k), as
    // without packing -- not -1, which would mean "in a packed word"
    s.fields.clear();
    for (size_t k = 0; k < s.ivals.size(); ++k) s.iu[k] = (int)k;
    return;
  }
  s.pwords = (int)used.size();
  std::vector<char> packed(s.ivals.size(), 0);
  for (const Field& f : s.fields)
    if (f.acc >= 0) packed[f.acc] = 1;
  int nu = 0;
  for (size_t k = 0; k < s.ivals.size(); ++k) s.iu[k] = packed[k] ? -1 : nu++;
}

// agg -> accumulator lists (deduplicated by value and scale)
void list_accumulators(Spec& s) {
  s.fvals.clear();
  s.ivals.clear();
  s.iscale.clear();
  s.agg_acc.clear();
  for (size_t a = 0; a < s.aggs.size(); ++a) {
    const tdp_agg& g = s.aggs[a];
    if (g.kind == TDP_AGG_COUNT) {
      s.agg_acc.push_back(-1);
      continue;
    }
    const bool isf = g.kind == TDP_AGG_SUM_F64;
    const double sc = s.agg_scale[a];
    std::vector<int>& lst = isf ? s.fvals : s.ivals;
    int idx = -1;
    for (size_t t = 0; t < lst.size(); ++t)
      if (lst[t] == g.value && (isf || s.iscale[t] == sc)) idx = (int)t;
    if (idx < 0) {
      idx = (int)lst.size();
      lst.push_back(g.value);
      if (!isf) s.iscale.push_back(sc);
    }
    s.agg_acc.push_back(idx);
  }
}

int validate_and_derive(Spec& s, const tdp_column* cols, int ncols, i64 n) {
  TDP_REQUIRE(ncols >= 0 && ncols <= kMaxCols, "at most %d columns (got %d)", kMaxCols, ncols);
  TDP_REQUIRE((int)s.prog.size() <= kMaxInstr, "program longer than %d instructions",
              kMaxInstr);
  TDP_REQUIRE((int)s.keys.size() <= kMaxKeys, "at most %d keys", kMaxKeys);
  TDP_REQUIRE((int)s.preds.size() <= kMaxPreds, "at most %d predicates", kMaxPreds);
  TDP_REQUIRE((int)s.outs.size() <= kMaxOuts, "at most %d outputs", kMaxOuts);
  std::vector<char> used(ncols, 0);
  for (int c = 0; c < ncols; ++c) {
    TDP_REQUIRE(dtype_size(cols[c].dtype) > 0, "column %d: bad dtype", c);
    TDP_REQUIRE(cols[c].width == 1, "column %d: scalar columns only", c);
    s.col_dtype.push_back(cols[c].dtype);
  }
  for (size_t k = 0; k < s.preds.size(); ++k) {
    const tdp_predicate& p = s.preds[k];
    TDP_REQUIRE(p.op >= TDP_EQ && p.op <= TDP_GE, "predicate %zu: bad op", k);
    TDP_REQUIRE(p.cmp >= TDP_CMP_I64 && p.cmp <= TDP_CMP_BITMAP, "predicate %zu: bad compare", k);
    TDP_REQUIRE(p.cmp != TDP_CMP_DEC || p.lit_i > 0, "predicate %zu: bad decimal divisor", k);
    if (p.cmp == TDP_CMP_BITMAP)  // the bitmap is read by address, never streamed
      TDP_REQUIRE(p.reserved >= 0 && p.reserved < ncols && p.lit_f >= 1.0 &&
                      (double)cols[p.reserved].rows * 32.0 >= p.lit_f,
                  "predicate %zu: bad bitmap operand", k);
    if (p.cmp <= TDP_CMP_F32 || p.cmp == TDP_CMP_DEC || p.cmp == TDP_CMP_BITMAP) {
      TDP_REQUIRE(p.column >= 0 && p.column < ncols, "predicate %zu: bad column", k);
      used[p.column] = 1;
    }
  }
  for (size_t j = 0; j < s.prog.size(); ++j) {
    const tdp_instr& in = s.prog[j];
    TDP_REQUIRE(in.dtype == TDP_I64 || in.dtype == TDP_F64 || in.dtype == TDP_F32,
                "instr %zu: result dtype must be int64/float64/float32", j);
    switch (in.op) {
      case TDP_OP_LOAD:
        TDP_REQUIRE(in.a >= 0 && in.a < ncols, "instr %zu: bad column", j);
        TDP_REQUIRE(in.b == 0 || (in.b == 1 && in.dtype == TDP_I64 && (double)in.imm_i <= in.imm_f),
                    "instr %zu: bad value-range hint", j);
        used[in.a] = 1;
        break;
      case TDP_OP_CONST:
        break;
      case TDP_OP_ADD:
      case TDP_OP_SUB:
      case TDP_OP_MUL:
      case TDP_OP_DIV:
        TDP_REQUIRE(in.b >= 0 && in.b < (int)j, "instr %zu: bad operand b", j);
        TDP_REQUIRE(s.prog[in.b].dtype == in.dtype, "instr %zu: operand b type mismatch", j);
        // fallthrough
      case TDP_OP_NEG:
      case TDP_OP_SQUARE:
      case TDP_OP_LOG:
      case TDP_OP_EXP:
      case TDP_OP_RELU:
        TDP_REQUIRE(in.a >= 0 && in.a < (int)j, "instr %zu: bad operand a", j);
        TDP_REQUIRE(s.prog[in.a].dtype == in.dtype, "instr %zu: operand a type mismatch", j);
        if (in.op == TDP_OP_DIV || in.op == TDP_OP_LOG || in.op == TDP_OP_EXP)
          TDP_REQUIRE(in.dtype != TDP_I64, "instr %zu: float-only op on int64", j);
        break;
      case TDP_OP_DECIMAL:
        TDP_REQUIRE(in.a >= 0 && in.a < (int)j, "instr %zu: bad decimal operand", j);
        TDP_REQUIRE(in.dtype == TDP_F64 && s.prog[in.a].dtype == TDP_I64,
                    "instr %zu: decimal decodes int64 to float64", j);
        TDP_REQUIRE(in.imm_f > 0.0, "instr %zu: decimal divisor must be > 0", j);
        break;
      case TDP_OP_CAST:
        TDP_REQUIRE(in.a >= 0 && in.a < (int)j, "instr %zu: bad cast operand", j);
        TDP_REQUIRE(!(in.dtype == TDP_I64 && s.prog[in.a].dtype != TDP_I64),
                    "instr %zu: float -> int cast not supported", j);
        break;
      default:
        return set_error(TDP_EINVAL, "instr %zu: unknown opcode %d", j, in.op);
    }
  }
  for (size_t j = 0; j < s.keys.size(); ++j) {
    const tdp_key& k = s.keys[j];
    TDP_REQUIRE(k.value >= 0 && k.value < (int)s.prog.size(), "key %zu: bad value", j);
    TDP_REQUIRE(s.prog[k.value].dtype == TDP_I64, "key %zu: keys must be int64 values", j);
    TDP_REQUIRE(k.span >= 1, "key %zu: span must be >= 1", j);
    TDP_REQUIRE(s.slots <= kMaxSlots / k.span, "dense key space exceeds %lld slots",
                (long long)kMaxSlots);
    s.slots *= k.span;
  }
  for (size_t a = 0; a < s.aggs.size(); ++a) {
    const tdp_agg& g = s.aggs[a];
    if (g.kind == TDP_AGG_COUNT) continue;
    TDP_REQUIRE(g.kind == TDP_AGG_SUM_F64 || g.kind == TDP_AGG_SUM_I64, "agg %zu: bad kind", a);
    TDP_REQUIRE(g.value >= 0 && g.value < (int)s.prog.size(), "agg %zu: bad value", a);
    if (g.kind == TDP_AGG_SUM_I64)
      TDP_REQUIRE(s.prog[g.value].dtype == TDP_I64, "agg %zu: SUM_I64 over a float value", a);
  }
  s.agg_scale.assign(s.aggs.size(), 0.0);
  list_accumulators(s);
  for (size_t o = 0; o < s.outs.size(); ++o)
    TDP_REQUIRE(s.outs[o] >= 0 && s.outs[o] < (int)s.prog.size(), "output %zu: bad value", o);
  for (int c = 0; c < ncols; ++c)
    if (used[c]) {
      TDP_REQUIRE(cols[c].rows >= n, "column %d has %lld rows < %lld", c, (long long)cols[c].rows,
                  (long long)n);
      TDP_REQUIRE(n == 0 || cols[c].data != nullptr, "column %d: null data", c);
      s.used_cols.push_back(c);
    }
  const i64 cells = s.slots * (i64)(1 + s.fvals.size() + s.ivals.size());
  // registers when the per-row select-and-add over all slots is cheap, private
  // shared-memory columns (one add per aggregate per row) for up to
  // kMaxSmemCells cells, global atomics beyond.
  if (s.slots == 1 || cells <= 8) s.accmode = 0;
  else if (cells <= kMaxSmemCells) s.accmode = 1;
  else s.accmode = 2;
  s.regacc = s.accmode != 2;
  if (!s.aggs.empty() && s.outs.empty()) {
    convert_decimal_sums(s, n);
    list_accumulators(s);
  }
  s.iu.assign(s.ivals.size(), -1);
  for (size_t k = 0; k < s.ivals.size(); ++k) s.iu[k] = (int)k;
  s.fields.clear();
  s.pwords = 0;
  if (s.accmode == 1) pack_fields(s, n);
  // shared-memory rows: packed words [pwords][G], 32-bit counts (when not
  // packed) [G] (G/2 rows of u64), float cells [NF][G], unpacked int cells
  int niu = 0;
  for (int k : s.iu) niu += k >= 0 ? 1 : 0;
  // one extra slot row per cell takes the rows that fail the predicates
  // (branch-free updates)
  s.sm_rows = (s.slots + 1) * ((i64)s.pwords + (i64)s.fvals.size() + niu) +
              (s.pwords > 0 ? 0 : (s.slots + 2) / 2);
  s.acc_smem = s.accmode == 1 ? s.sm_rows * kAccThreads * 8 : 0;
  return TDP_OK;
}

bool fits32(const Range& r) { return r.ok && r.lo >= INT32_MIN && r.hi <= INT32_MAX; }

// integer compares on <= 16-bit columns run in 32 bits (fill_params clamps the literal)
bool narrow_cmp(int dt) { return dt == TDP_I8 || dt == TDP_I16 || dt == TDP_U8 || dt == TDP_BOOL; }

void emit_program(std::ostringstream& o, const Spec& s) {
  // int64 values whose range provably fits 32 bits are computed in 32-bit
  // arithmetic (mod 2^32, exact because the result fits); 32 x 32 -> 64-bit
  // products are one wide multiply
  const std::vector<Range> R = value_ranges(s);
  for (size_t j = 0; j < s.prog.size(); ++j) {
    const tdp_instr& in = s.prog[j];
    const char* T = ctype_of(in.dtype);
    const bool isint = in.dtype == TDP_I64;
    const bool isf32 = in.dtype == TDP_F32;
    o << "  const " << T << " v" << j << " = ";
    const std::string a = "v" + std::to_string(in.a), b = "v" + std::to_string(in.b);
    if (isint && fits32(R[j]) &&
        (in.op == TDP_OP_ADD || in.op == TDP_OP_SUB || in.op == TDP_OP_MUL ||
         in.op == TDP_OP_NEG || in.op == TDP_OP_SQUARE)) {
      const std::string ua = "(unsigned)" + a, ub = "(unsigned)" + b;
      o << "(i64)(int)(";
      switch (in.op) {
        case TDP_OP_ADD: o << ua << " + " << ub; break;
        case TDP_OP_SUB: o << ua << " - " << ub; break;
        case TDP_OP_MUL: o << ua << " * " << ub; break;
        case TDP_OP_NEG: o << "0u - " << ua; break;
        default: o << ua << " * " << ua; break;
      }
      o << ");\n";
      continue;
    }
    if (isint && in.op == TDP_OP_MUL && fits32(R[in.a]) && fits32(R[in.b])) {
      o << "(i64)(int)" << a << " * (i64)(int)" << b << ";\n";
      continue;
    }
    switch (in.op) {
      case TDP_OP_LOAD:
        o << "(" << T << ")r.c" << in.a;
        break;
      case TDP_OP_CONST:
        if (isint) o << "P.imi[" << j << "]";
        else o << "(" << T << ")P.imf[" << j << "]";
        break;
      case TDP_OP_CAST:
        o << "(" << T << ")" << a;
        break;
      case TDP_OP_DECIMAL:
        o << "tdp_decimal((double)" << a << ", P.imf[" << j << "], __longlong_as_double(P.imi[" << j
          << "]))";
        break;
      case TDP_OP_ADD:
        if (isint) o << "(i64)((u64)" << a << " + (u64)" << b << ")";
        else o << a << " + " << b;
        break;
      case TDP_OP_SUB:
        if (isint) o << "(i64)((u64)" << a << " - (u64)" << b << ")";
        else o << a << " - " << b;
        break;
      case TDP_OP_MUL:
        if (isint) o << "(i64)((u64)" << a << " * (u64)" << b << ")";
        else o << a << " * " << b;
        break;
      case TDP_OP_DIV:
        o << a << " / " << b;
        break;
      case TDP_OP_NEG:
        if (isint) o << "(i64)(0ull - (u64)" << a << ")";
        else o << "-" << a;
        break;
      case TDP_OP_SQUARE:
        if (isint) o << "(i64)((u64)" << a << " * (u64)" << a << ")";
        else o << a << " * " << a;
        break;
      case TDP_OP_LOG:
        o << (isf32 ? "logf(" : "log(") << a << ")";
        break;
      case TDP_OP_EXP:
        o << (isf32 ? "expf(" : "exp(") << a << ")";
        break;
      case TDP_OP_RELU:
        o << "(" << a << " > (" << T << ")0 ? " << a << " : (" << T << ")0)";
        break;
    }
    o << ";\n";
  }
}

// Shared-memory accumulator columns (TDP_ACCMODE 1): one TDP_ACC_THREADS-wide
// row of u64 per cell, each thread owning one column of every row.  Rows:
// packed words [NW][G] | 32-bit counts [G] (only when the count is not
// packed; G/2 rows) | float cells [NF][G] | unpacked integer cells [..][G].
void emit_smem_acc(std::ostringstream& o, const Spec& s) {
  const i64 G = s.slots + 1, NW = s.pwords, NF = (i64)s.fvals.size();  // + the reject slot
  const i64 FB = NW * G + (NW > 0 ? 0 : (G + 1) / 2);
  const i64 IB = FB + NF * G;
  const Field* cnt = nullptr;
  std::vector<const Field*> fof(s.ivals.size(), nullptr);
  for (const Field& f : s.fields) {
    if (f.acc < 0) cnt = &f;
    else fof[f.acc] = &f;
  }
  // `mine` = this thread's column (sm + col); rows failing the predicates go
  // to slot TDP_G, which the flush ignores
  o << "__device__ __forceinline__ void tdp_smem_add(u64* mine, int slot, const double* f, "
       "const i64* q, const TdpParams& P) {\n";
  o << "  (void)f; (void)q; (void)P;\n  u64* p = mine + slot * TDP_ACC_THREADS;\n";
  // per word: the biased field values x = q - bias (0 <= x < 2^bits) occupy
  // disjoint bit ranges, so the word is assembled from two 32-bit halves
  // without carries (one shift per field; 64-bit only for > 32-bit fields)
  for (int w = 0; w < NW; ++w) {
    u64 konst = 0;
    std::ostringstream lo32, hi32, w64;
    for (const Field& f : s.fields) {
      if (f.word != w) continue;
      if (f.acc < 0) {
        konst += (u64)1 << f.off;
        continue;
      }
      std::ostringstream x;
      if (f.rbits <= 32) {
        x << "((unsigned)q[" << f.acc << "]";
        if (f.lo != 0) x << " - (unsigned)P.plo[" << f.acc << "]";
        x << ")";
        if (f.off + f.rbits <= 32) {
          lo32 << " + (" << x.str() << " << " << f.off << ")";
        } else if (f.off >= 32) {
          hi32 << " + (" << x.str() << " << " << f.off - 32 << ")";
        } else {
          lo32 << " + (" << x.str() << " << " << f.off << ")";
          hi32 << " + (" << x.str() << " >> " << 32 - f.off << ")";
        }
      } else {
        w64 << " + ((u64)(q[" << f.acc << "]";
        if (f.lo != 0) w64 << " - P.plo[" << f.acc << "]";
        w64 << ") << " << f.off << ")";
      }
    }
    o << "  {\n    const unsigned lo = " << (unsigned)(konst & 0xffffffffu) << "u" << lo32.str()
      << ";\n    const unsigned hi = " << (unsigned)(konst >> 32) << "u" << hi32.str() << ";\n";
    o << "    p[" << w * G << " * TDP_ACC_THREADS] += (((u64)hi << 32) | lo)" << w64.str()
      << ";\n  }\n";
  }
  if (NW == 0)  // 32-bit counts [G][256] at the start (col == threadIdx.x)
    o << "  reinterpret_cast<unsigned*>(mine - threadIdx.x)[slot * TDP_ACC_THREADS + threadIdx.x] "
         "+= 1u;\n";
  for (i64 a = 0; a < NF; ++a)
    o << "  *reinterpret_cast<double*>(p + " << FB + a * G << " * TDP_ACC_THREADS) += f[" << a
      << "];\n";
  for (size_t k = 0; k < s.iu.size(); ++k)
    if (s.iu[k] >= 0)
      o << "  p[" << IB + (i64)s.iu[k] * G << " * TDP_ACC_THREADS] += (u64)q[" << k << "];\n";
  o << "}\n";
  // per-CTA partial row, cell-major (acc[cell * gridDim.x + cta]); fixed order
  auto field_sum = [&](const Field& f, const char* v) {
    o << "      const u64* row = sm + (" << (i64)f.word * G << " + slot) * TDP_ACC_THREADS;\n"
      << "      for (int t = 0; t < TDP_ACC_THREADS; ++t) " << v << " += (row[t] >> " << f.off
      << ") & " << (((u64)1 << f.bits) - 1) << "ull;\n";
  };
  o << "__device__ __forceinline__ void tdp_smem_flush(const u64* sm, const TdpParams& P) {\n"
       "  u64* out = reinterpret_cast<u64*>(P.acc) + blockIdx.x;\n"
       "  for (int c = threadIdx.x; c < TDP_CELLS; c += blockDim.x) {\n"
       "    const int grp = c / TDP_G, slot = c % TDP_G;\n"
       "    u64 v = 0;\n"
       "    switch (grp) {\n";
  o << "    case 0: {\n";
  if (cnt) {
    field_sum(*cnt, "v");
  } else {
    o << "      const unsigned* row = reinterpret_cast<const unsigned*>(sm) + slot * "
         "TDP_ACC_THREADS;\n      for (int t = 0; t < TDP_ACC_THREADS; ++t) v += row[t];\n";
  }
  o << "      break;\n    }\n";
  for (i64 a = 0; a < NF; ++a)
    o << "    case " << 1 + a << ": {\n      const double* row = reinterpret_cast<const double*>(sm) + ("
      << FB + a * G << " + slot) * TDP_ACC_THREADS;\n      double d = 0.0;\n"
      << "      for (int t = 0; t < TDP_ACC_THREADS; ++t) d += row[t];\n"
      << "      v = (u64)__double_as_longlong(d);\n      break;\n    }\n";
  for (size_t k = 0; k < s.ivals.size(); ++k) {
    o << "    case " << 1 + NF + (i64)k << ": {\n";
    if (fof[k]) {
      // biased field sums + lo * (rows counted by this CTA for the slot)
      o << "      u64 cn = 0;\n      {\n";
      field_sum(*cnt, "cn");
      o << "      }\n";
      field_sum(*fof[k], "v");
      o << "      v += (u64)P.plo[" << k << "] * cn;\n";
    } else {
      o << "      const u64* row = sm + (" << IB + (i64)s.iu[k] * G
        << " + slot) * TDP_ACC_THREADS;\n      for (int t = 0; t < TDP_ACC_THREADS; ++t) v += "
           "row[t];\n";
    }
    o << "      break;\n    }\n";
  }
  o << "    default: break;\n    }\n    out[(i64)c * gridDim.x] = v;\n  }\n}\n";
}

// Shape of the bulk-copy ring for the columns a program reads.
struct Ring {
  int pu = 4;            // rows per consumer thread per tile
  int ptile = 0;         // rows per tile
  i64 stage_bytes = 0;   // bytes of one ring stage (all columns of one tile)
  int stages = 0;
};

Ring ring_shape(const Spec& s) {
  Ring r;
  i64 row_bytes = 0;
  for (int c : s.used_cols) row_bytes += dtype_size(s.col_dtype[c]);
  if (row_bytes == 0) row_bytes = 1;
  // private accumulator columns read each column with one vector load per
  // thread: 8 rows per thread halve the per-tile loop overhead per row
  static const int vec_pu = [] {  // measurements only
    const char* e = getenv("TDP_VEC_PU");
    const int v = e ? atoi(e) : 8;
    return v == 4 ? 4 : 8;
  }();
  r.pu = s.accmode == 1 ? vec_pu : 4;
  const i64 budget = kRingBudget - s.acc_smem;
  static const i64 min_stages = [] {
    const char* e = getenv("TDP_RING_MIN_STAGES");  // measurements only
    return e ? (i64)atoll(e) : (i64)4;
  }();
  while (r.pu > 1 && (i64)kConsWarps * 32 * r.pu * row_bytes * min_stages > budget) r.pu >>= 1;
  r.ptile = kConsWarps * 32 * r.pu;
  r.stage_bytes = (i64)r.ptile * row_bytes;
  i64 st = (kRingBudget - s.acc_smem) / r.stage_bytes;
  // Narrow rows (compact storage) make the per-row arithmetic, not the bytes,
  // the limit: then prefer two CTAs per SM (twice the consumer warps to hide
  // FP64 / shared-memory latency) over a deeper ring, when two fit.
  static const int narrow_ctas = [] {  // CTAs per SM for narrow rows (measurements)
    const char* e = getenv("TDP_NARROW_CTAS");
    const int v = e ? atoi(e) : 2;
    return v < 2 ? 2 : (v > 4 ? 4 : v);
  }();
  const i64 per_cta = narrow_ctas == 2 ? kTwoCtaBudget : (i64)233472 / narrow_ctas - 2048;
  const i64 half = per_cta - s.acc_smem;
  if (row_bytes <= kTwoCtaRowBytes && half >= 2 * r.stage_bytes) st = half / r.stage_bytes;
  r.stages = (int)(st < 2 ? 2 : (st > 8 ? 8 : st));
  return r;
}

std::string generate(const Spec& s) {
  std::ostringstream o;
  const Ring ring = ring_shape(s);
  o << "typedef long long i64;\ntypedef unsigned long long u64;\n";
  o << "__device__ __forceinline__ double tdp_decimal(double x, double d, double inv) {\n"
       "  const double q = x * inv;\n  return fma(fma(-q, d, x), inv, q);\n}\n";
  o << "#define TDP_THREADS " << kThreads << "\n#define TDP_U " << kUnroll << "\n";
  o << "#define TDP_CONS_WARPS " << kConsWarps << "\n#define TDP_PU " << ring.pu
    << "\n#define TDP_PTILE " << ring.ptile << "\n#define TDP_STAGE_BYTES " << ring.stage_bytes
    << "\n#define TDP_STAGES " << ring.stages << "\n";
  // per-thread contiguous rows + vector loads when shared-memory wavefronts
  // are the limit (private accumulator columns: Q1 on narrow columns 0.261 ->
  // 0.236 ms); register accumulators keep the interleaved scalar loads (Q6
  // narrow: 0.112 vs 0.130 ms vectorised)
  o << "#define TDP_VEC_RING " << (s.accmode == 1 ? 1 : 0) << "\n";
  o << "#define TDP_G " << s.slots << "\n#define TDP_NF " << s.fvals.size() << "\n";
  o << "#define TDP_NI " << s.ivals.size() << "\n#define TDP_ACCMODE " << s.accmode
    << "\n";
  o << "#define TDP_CELLS (TDP_G * (1 + TDP_NF + TDP_NI))\n#define TDP_ACC_THREADS " << kAccThreads
    << "\n";
  o << "#define TDP_SM_ROWS " << (s.accmode == 1 ? s.sm_rows : 0) << "\n#define TDP_NW "
    << s.pwords << "\n";
  o << "#define TDP_FTILE " << kFilterTile << "\n#define TDP_FWORDS " << kFilterWords << "\n";
  o << "struct TdpParams {\n  const void* col[" << kMaxCols << "];\n  void* out[" << kMaxOuts
    << "];\n  i64 n;\n  i64 pli[" << kMaxPreds << "];\n  double plf[" << kMaxPreds
    << "];\n  i64 imi[" << kMaxInstr << "];\n  double imf[" << kMaxInstr << "];\n  i64 klo["
    << kMaxKeys << "];\n  void* acc;\n  const unsigned* bits;\n  const i64* tile_off;\n"
    << "  i64 plo[" << kMaxIvals << "];\n};\n";
  // row of loaded columns
  o << "struct TdpRow {\n  int pad_;\n";
  for (int c : s.used_cols) o << "  " << ctype_of(s.col_dtype[c]) << " c" << c << ";\n";
  o << "};\n";
  o << "__device__ __forceinline__ void tdp_zero(TdpRow& r) {\n  r.pad_ = 0;\n";
  for (int c : s.used_cols) o << "  r.c" << c << " = 0;\n";
  o << "}\n";
  o << "__device__ __forceinline__ void tdp_load(TdpRow& r, const TdpParams& P, i64 i) {\n"
       "  r.pad_ = 0;\n";
  for (int c : s.used_cols) {
    const char* T = ctype_of(s.col_dtype[c]);
    if (s.col_dtype[c] == TDP_BOOL)
      o << "  r.c" << c << " = ((const " << T << "*)P.col[" << c << "])[i];\n";
    else
      o << "  r.c" << c << " = __ldg((const " << T << "*)P.col[" << c << "] + i);\n";
  }
  o << "}\n";
  // ring stage layout: column tiles back to back, each PTILE elements
  {
    std::ostringstream ld, is;
    i64 off = 0;
    for (int c : s.used_cols) {
      const int es = dtype_size(s.col_dtype[c]);
      const char* T = ctype_of(s.col_dtype[c]);
      ld << "  r.c" << c << " = ((const " << T << "*)(sb + " << off << "))[lr];\n";
      is << "  tdp_bulk_load(sb + " << off << "u, (const unsigned char*)P.col[" << c
         << "] + row0 * " << es << ", " << (i64)ring.ptile * es << "u, bar, policy);\n";
      off += (i64)ring.ptile * es;
    }
    o << "__device__ __forceinline__ void tdp_load_smem(TdpRow& r, const unsigned char* sb, int lr) {\n"
         "  r.pad_ = 0;\n"
      << ld.str() << "}\n";
    // consumer thread t owns rows t*PU .. t*PU+PU-1 of a tile: one vector
    // load per column (a 1-byte column of 4 rows is one 32-bit load, i.e. a
    // quarter of the shared-memory wavefronts of four scalar loads)
    o << "__device__ __forceinline__ void tdp_load_smem_pu(TdpRow (&r)[TDP_PU], const unsigned "
         "char* sb, int t) {\n";
    o << "#pragma unroll\n  for (int u = 0; u < TDP_PU; ++u) r[u].pad_ = 0;\n";
    off = 0;
    for (int c : s.used_cols) {
      const int es = dtype_size(s.col_dtype[c]);
      const char* T = ctype_of(s.col_dtype[c]);
      const int bytes = ring.pu * es;
      o << "  {\n    __align__(16) " << T << " v[TDP_PU];\n";
      const char* V = bytes == 1 ? "unsigned char" : bytes == 2 ? "unsigned short"
                      : bytes == 4 ? "unsigned" : bytes == 8 ? "unsigned long long" : "uint4";
      const int nv = bytes <= 16 ? 1 : bytes / 16;
      o << "    const " << V << "* src = (const " << V << "*)(sb + " << off << ") + (i64)t * " << nv
        << ";\n";
      for (int k = 0; k < nv; ++k) o << "    ((" << V << "*)v)[" << k << "] = src[" << k << "];\n";
      o << "#pragma unroll\n    for (int u = 0; u < TDP_PU; ++u) r[u].c" << c << " = v[u];\n  }\n";
      off += (i64)ring.ptile * es;
    }
    o << "}\n";
    o << "__device__ __forceinline__ void tdp_bulk_load(unsigned, const void*, unsigned, unsigned, u64);\n";
    o << "__device__ __forceinline__ void tdp_issue_tile(const TdpParams& P, unsigned sb, i64 row0, "
         "unsigned bar, u64 policy) {\n"
      << is.str() << "}\n";
  }
  // predicate conjunction + program + keys + aggregate inputs
  o << "__device__ __forceinline__ bool tdp_eval(const TdpRow& r, const TdpParams& P, int& "
       "slot, double* f, i64* q) {\n";
  o << "  bool keep = true;\n";
  for (size_t k = 0; k < s.preds.size(); ++k) {
    const tdp_predicate& p = s.preds[k];
    switch (p.cmp) {
      case TDP_CMP_I64:
        if (narrow_cmp(s.col_dtype[p.column]))  // literal clamped to the type range +- 1
          o << "  keep &= ((int)r.c" << p.column << " " << op_sym(p.op) << " (int)P.pli[" << k
            << "]);\n";
        else
          o << "  keep &= ((i64)r.c" << p.column << " " << op_sym(p.op) << " P.pli[" << k
            << "]);\n";
        break;
      case TDP_CMP_F64:
        o << "  keep &= ((double)r.c" << p.column << " " << op_sym(p.op) << " P.plf[" << k
          << "]);\n";
        break;
      case TDP_CMP_F32:
        o << "  keep &= ((float)r.c" << p.column << " " << op_sym(p.op) << " (float)P.plf[" << k
          << "]);\n";
        break;
      case TDP_CMP_DEC:
        o << "  keep &= ((double)r.c" << p.column << " / (double)P.pli[" << k << "] "
          << op_sym(p.op) << " P.plf[" << k << "]);\n";
        break;
      case TDP_CMP_NONE:
        o << "  keep = false;\n";
        break;
      case TDP_CMP_BITMAP:
        o << "  { const u64 x = (u64)(i64)r.c" << p.column << " - (u64)P.pli[" << k
          << "]; keep &= x < (u64)(i64)P.plf[" << k << "] && ((__ldg((const unsigned*)P.col["
          << p.reserved << "] + (x >> 5)) >> (x & 31)) & 1u); }\n";
        break;
      default:
        break;
    }
  }
  emit_program(o, s);
  // slots < 2^20: the mixed-radix slot in 32-bit arithmetic
  o << "  int sl = 0;\n";
  for (size_t j = 0; j < s.keys.size(); ++j)
    o << "  sl = sl * " << s.keys[j].span << " + (int)((unsigned)v" << s.keys[j].value
      << " - (unsigned)P.klo[" << j << "]);\n";
  o << "  slot = sl;\n";
  for (size_t a = 0; a < s.fvals.size(); ++a) o << "  f[" << a << "] = (double)v" << s.fvals[a] << ";\n";
  for (size_t a = 0; a < s.ivals.size(); ++a) o << "  q[" << a << "] = (i64)v" << s.ivals[a] << ";\n";
  o << "  return keep;\n}\n";
  if (s.accmode == 1) emit_smem_acc(o, s);
  // projection
  o << "__device__ __forceinline__ void tdp_project(const TdpRow& r, const TdpParams& P, i64 "
       "pos) {\n";
  emit_program(o, s);
  for (size_t k = 0; k < s.outs.size(); ++k) {
    const int v = s.outs[k];
    o << "  ((" << ctype_of(s.prog[v].dtype) << "*)P.out[" << k << "])[pos] = v" << v << ";\n";
  }
  o << "}\n";
  o << kSkeleton;
  return o.str();
}

// ---------------------------------------------------------------------------
// NVRTC compile + module cache
// ---------------------------------------------------------------------------
struct Kernel {
  CUmodule mod = nullptr;
  CUfunction agg = nullptr;      // bulk-copy ring kernel
  CUfunction agg_ldg = nullptr;  // register-staged kernel
  CUfunction proj = nullptr;
  int agg_occ = 1;
  int ldg_occ = 1;
  Ring ring;
  size_t ring_smem = 0;   // ring + accumulators
  size_t ldg_smem = 0;    // accumulators
};

std::mutex g_cache_mu;
std::map<std::pair<int, std::string>, std::shared_ptr<Kernel>> g_cache;

// Source -> sm_100a CUBIN.  Needs no device (usable on build hosts).
int nvrtc_compile(const std::string& src, std::vector<char>* cubin) {
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "tdp_pipeline.cu", 0, nullptr, nullptr) !=
      NVRTC_SUCCESS)
    return set_error(TDP_EJIT, "nvrtcCreateProgram failed");
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-fmad=false",
                        "-lineinfo", "--device-as-default-execution-space"};
  nvrtcResult cr = nvrtcCompileProgram(prog, 5, opts);
  if (cr != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    if (n) nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    return set_error(TDP_EJIT, "NVRTC: %s\n%s", nvrtcGetErrorString(cr), log.c_str());
  }
  size_t cubin_size = 0;
  nvrtcGetCUBINSize(prog, &cubin_size);
  cubin->resize(cubin_size);
  nvrtcGetCUBIN(prog, cubin->data());
  nvrtcDestroyProgram(&prog);
  return TDP_OK;
}

// Everything the generated source depends on (literals and constants are
// kernel parameters), as a compact cache key; the source is only generated on
// a miss.
std::string signature(const Spec& s) {
  std::string k;
  auto put = [&k](long long v) {
    k.append(reinterpret_cast<const char*>(&v), sizeof(v));
  };
  put((long long)s.col_dtype.size());
  for (int d : s.col_dtype) put(d);
  put((long long)s.preds.size());
  for (const auto& p : s.preds)
    put(((long long)p.reserved << 40) | ((long long)p.column << 16) | (p.op << 8) | p.cmp);
  put((long long)s.prog.size());
  for (const auto& in : s.prog) put(((long long)in.op << 48) ^ ((long long)in.dtype << 40) ^ ((long long)in.a << 20) ^ in.b);
  put((long long)s.keys.size());
  for (const auto& kk : s.keys) {
    put(kk.value);
    put(kk.span);
  }
  put((long long)s.aggs.size());
  for (const auto& a : s.aggs) put(((long long)a.kind << 32) | (unsigned)a.value);
  put((long long)s.outs.size());
  for (int o : s.outs) put(o);
  put((long long)s.prog.size());  // incl. the integer restatement of decimal sums
  put(s.pwords);
  for (const auto& f : s.fields)
    put(((long long)(f.acc + 1) << 32) | ((long long)f.word << 16) | (f.off << 8) | f.bits);
  return k;
}

int compile(const Spec& s, const Ring& ring, i64 acc_smem, std::shared_ptr<Kernel>* out) {
  int dev = 0;
  TDP_CUDA_TRY(cudaGetDevice(&dev));
  const std::string key = signature(s);
  {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    auto it = g_cache.find({dev, key});
    if (it != g_cache.end()) {
      *out = it->second;
      return TDP_OK;
    }
  }
  Driver* d = nullptr;
  int rc = get_driver(&d);
  if (rc) return rc;
  const std::string src = generate(s);
  std::vector<char> cubin;
  rc = nvrtc_compile(src, &cubin);
  if (rc) return rc;
  if (const char* dir = getenv("TDP_DUMP_CUBIN_DIR")) {  // SASS evidence (cuobjdump -sass)
    const std::string base = std::string(dir) + "/tdp_scan_" +
                             std::to_string(std::hash<std::string>{}(key) & 0xffffffu);
    if (FILE* f = fopen((base + ".cubin").c_str(), "wb")) {
      fwrite(cubin.data(), 1, cubin.size(), f);
      fclose(f);
    }
    if (FILE* f = fopen((base + ".cu").c_str(), "wb")) {
      fwrite(src.data(), 1, src.size(), f);
      fclose(f);
    }
  }
  TDP_CUDA_TRY(cudaFree(0));  // make the primary context current on this thread
  auto k = std::make_shared<Kernel>();
  rc = cu_check(d, d->load(&k->mod, cubin.data()), "cuModuleLoadData");
  if (rc) return rc;
  rc = cu_check(d, d->getfn(&k->agg, k->mod, "tdp_scan_agg"), "cuModuleGetFunction(agg)");
  if (rc) return rc;
  rc = cu_check(d, d->getfn(&k->agg_ldg, k->mod, "tdp_scan_agg_ldg"), "cuModuleGetFunction(ldg)");
  if (rc) return rc;
  rc = cu_check(d, d->getfn(&k->proj, k->mod, "tdp_scan_project"), "cuModuleGetFunction(proj)");
  if (rc) return rc;
  k->ring = ring;
  k->ring_smem = (size_t)ring.stages * (size_t)ring.stage_bytes + (size_t)acc_smem;
  k->ldg_smem = (size_t)acc_smem;
  rc = cu_check(d, d->setattr(k->agg, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                              (int)k->ring_smem),
                "cuFuncSetAttribute(max dynamic smem)");
  if (rc) return rc;
  rc = cu_check(d, d->setattr(k->agg_ldg, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                              (int)k->ldg_smem),
                "cuFuncSetAttribute(max dynamic smem, ldg)");
  if (rc) return rc;
  int occ = 1;
  if (d->occupancy(&occ, k->agg, (kConsWarps + 1) * 32, k->ring_smem) != CUDA_SUCCESS || occ < 1)
    occ = 1;
  k->agg_occ = occ;
  occ = 1;
  if (d->occupancy(&occ, k->agg_ldg, kThreads, k->ldg_smem) != CUDA_SUCCESS || occ < 1) occ = 1;
  k->ldg_occ = occ;
  std::lock_guard<std::mutex> lock(g_cache_mu);
  g_cache[{dev, key}] = k;
  *out = k;
  return TDP_OK;
}

void fill_params(HostParams& hp, const Spec& s, const tdp_column* cols, int ncols, i64 n) {
  std::memset(&hp, 0, sizeof(hp));
  for (int c = 0; c < ncols; ++c) hp.col[c] = cols[c].data;
  hp.n = n;
  for (size_t k = 0; k < s.preds.size(); ++k) {
    hp.pli[k] = s.preds[k].lit_i;
    hp.plf[k] = s.preds[k].lit_f;
    const tdp_predicate& p = s.preds[k];
    if (p.cmp == TDP_CMP_I64 && p.column >= 0 && p.column < (int)s.col_dtype.size() &&
        narrow_cmp(s.col_dtype[p.column])) {
      // every comparison of a value in [lo, hi] with L equals the comparison
      // with clamp(L, lo - 1, hi + 1), which fits 32 bits
      const Range t = type_range(s.col_dtype[p.column]);
      hp.pli[k] = p.lit_i < t.lo - 1 ? t.lo - 1 : (p.lit_i > t.hi + 1 ? t.hi + 1 : p.lit_i);
    }
  }
  for (size_t j = 0; j < s.prog.size(); ++j) {
    hp.imi[j] = s.prog[j].imm_i;
    hp.imf[j] = s.prog[j].imm_f;
  }
  for (size_t j = 0; j < s.keys.size(); ++j) hp.klo[j] = s.keys[j].lo;
  for (const Field& f : s.fields)
    if (f.acc >= 0) hp.plo[f.acc] = f.lo;
}

// ---------------------------------------------------------------------------
// AOT helpers: deterministic reduction of partial rows, finalize, min/max
// ---------------------------------------------------------------------------
struct AggMap {
  int naggs;
  int nf;
  int ni;
  int pad;
  int kind[32];
  int acc[32];
  double scale[32];  // kAggSumDec: the sum is exact integers / scale
};

// One warp per output item; lanes stride over the partial rows in a fixed
// order and combine with a fixed shuffle tree -> bitwise deterministic.
__device__ __forceinline__ void reduce_items(const u64* __restrict__ part, int rows, int slots,
                                             const AggMap& m, i64* __restrict__ out_counts,
                                             u64* __restrict__ out_sums, i64 first_warp,
                                             i64 nwarps) {
  const int lane = threadIdx.x & 31;
  const i64 items = (i64)slots * (1 + m.naggs);
  const i64 cells = (i64)slots * (1 + m.nf + m.ni);
  for (i64 it = first_warp; it < items; it += nwarps) {
    i64 cell;
    bool is_f = false;
    double dec = 0.0;  // > 0: exact integer cells of a decimal sum
    if (it < slots) {
      cell = it;
    } else {
      const int a = (int)((it - slots) / slots);
      const i64 g = (it - slots) % slots;
      if (m.kind[a] == TDP_AGG_COUNT) {
        cell = g;
      } else if (m.kind[a] == TDP_AGG_SUM_F64) {
        cell = (i64)slots * (1 + m.acc[a]) + g;
        is_f = true;
      } else {
        cell = (i64)slots * (1 + m.nf + m.acc[a]) + g;
        if (m.kind[a] == kAggSumDec) dec = m.scale[a];
      }
    }
    // partial rows are cell-major: part[cell * rows + r] (coalesced per warp);
    // four accumulators per lane keep several loads in flight, combined in a
    // fixed order -> bitwise deterministic
    const u64* src = part + cell * (i64)rows;
    u64 bits;
    if (is_f) {
      double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
      int r = lane;
      for (; r + 96 < rows; r += 128) {
        v0 += __longlong_as_double((i64)src[r]);
        v1 += __longlong_as_double((i64)src[r + 32]);
        v2 += __longlong_as_double((i64)src[r + 64]);
        v3 += __longlong_as_double((i64)src[r + 96]);
      }
      for (; r < rows; r += 32) v0 += __longlong_as_double((i64)src[r]);
      double v = warp_sum((v0 + v1) + (v2 + v3));
      bits = (u64)__double_as_longlong(v);
    } else if (dec > 0.0) {
      // per-CTA partials are exact int64; their sum is kept in 128 bits and
      // rounded once: double(sum) / scale
      __int128 v = 0;
      for (int r = lane; r < rows; r += 32) v += (__int128)(i64)src[r];
      u64 lo = (u64)v;
      i64 hi = (i64)(v >> 64);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const u64 tlo = __shfl_xor_sync(0xffffffffu, lo, o);
        const i64 thi = __shfl_xor_sync(0xffffffffu, hi, o);
        const u64 nlo = lo + tlo;
        hi = hi + thi + (nlo < lo ? 1 : 0);
        lo = nlo;
      }
      const bool fits = hi == ((i64)lo >> 63);
      const double sum = fits ? (double)(i64)lo
                              : fma((double)hi, 18446744073709551616.0, (double)lo);
      bits = (u64)__double_as_longlong(sum / dec);
    } else {
      u64 v = 0;
      for (int r = lane; r < rows; r += 32) v += src[r];
      bits = warp_sum(v);
    }
    (void)cells;
    if (lane == 0) {
      if (it < slots) out_counts[it] = (i64)bits;
      else out_sums[it - slots] = bits;
    }
  }
}

__global__ void agg_reduce_kernel(const u64* __restrict__ part, int rows, int slots, AggMap m,
                                  i64* __restrict__ out_counts, u64* __restrict__ out_sums) {
  reduce_items(part, rows, slots, m, out_counts, out_sums,
               ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5,
               ((i64)gridDim.x * blockDim.x) >> 5);
}

struct KeyDigits {
  int nkeys;
  int pad;
  i64 lo[kMaxKeys];
  i64 span[kMaxKeys];
  i64 stride[kMaxKeys];
};

// Single CTA: compact occupied slots in ascending slot order.
__device__ __forceinline__ void finalize_block(const i64* __restrict__ counts,
                                               const u64* __restrict__ sums, i64 slots,
                                               const KeyDigits& kd, const AggMap& m,
                                               unsigned long long avg_mask,
                                               i64* __restrict__ out_keys,
                                               i64* __restrict__ out_counts,
                                               u64* __restrict__ out_aggs,
                                               i64* __restrict__ out_groups) {
  __shared__ int warp_tot[32];
  __shared__ i64 running;
  if (threadIdx.x == 0) running = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (i64 base = 0; base < slots; base += blockDim.x) {
    const i64 s = base + threadIdx.x;
    const i64 c = s < slots ? counts[s] : 0;
    const int occ = c > 0 ? 1 : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, occ);
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (w < warp) before += warp_tot[w];
      total += warp_tot[w];
    }
    const i64 pos = running + before + __popc(bal & lanemask_lt());
    if (occ) {
      for (int j = 0; j < kd.nkeys; ++j) {
        const i64 digit = (s / kd.stride[j]) % kd.span[j];
        out_keys[(i64)j * slots + pos] = kd.lo[j] + digit;
      }
      out_counts[pos] = c;
      for (int a = 0; a < m.naggs; ++a) {
        const u64 raw = sums[(i64)a * slots + s];
        u64 v = raw;
        if ((avg_mask >> a) & 1ull) {
          double sum;
          if (m.kind[a] == TDP_AGG_SUM_F64 || m.kind[a] == kAggSumDec)
            sum = __longlong_as_double((i64)raw);
          else sum = (double)(i64)raw;
          v = (u64)__double_as_longlong(sum / (double)c);
        }
        out_aggs[(i64)a * slots + pos] = v;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) running += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *out_groups = running;
}

__global__ void __launch_bounds__(1024)
    finalize_kernel(const i64* __restrict__ counts, const u64* __restrict__ sums, i64 slots,
                    KeyDigits kd, AggMap m, unsigned long long avg_mask,
                    i64* __restrict__ out_keys, i64* __restrict__ out_counts,
                    u64* __restrict__ out_aggs, i64* __restrict__ out_groups) {
  finalize_block(counts, sums, slots, kd, m, avg_mask, out_keys, out_counts, out_aggs, out_groups);
}

// Small group spaces: the partial-row reduction and the finalisation in one
// CTA (one launch after the scan instead of two).
constexpr i64 kFusedTailItems = 4096;
__global__ void __launch_bounds__(1024)
    reduce_finalize_kernel(const u64* __restrict__ part, int rows, int slots, AggMap m,
                           i64* __restrict__ red_counts, u64* __restrict__ red_sums,
                           KeyDigits kd, unsigned long long avg_mask, i64* __restrict__ out_keys,
                           i64* __restrict__ out_counts, u64* __restrict__ out_aggs,
                           i64* __restrict__ out_groups) {
  reduce_items(part, rows, slots, m, red_counts, red_sums, threadIdx.x >> 5, blockDim.x >> 5);
  __syncthreads();  // the CTA's global writes are visible to the CTA
  finalize_block(red_counts, red_sums, slots, kd, m, avg_mask, out_keys, out_counts, out_aggs,
                 out_groups);
}

struct KeyCols {
  const void* p[kMaxKeys];
  int dt[kMaxKeys];
};

// runs (nullable; one key, no predicates): runs[0] = 1 if the key column is
// not non-decreasing, runs[1] = 1 if some run of equal keys is longer than
// kRunMax rows (sorted: key[i] == key[i - kRunMax]) -- the sorted-runs
// group-by's preconditions, read with the range in one host read
constexpr int kRunMax = 32;

__global__ void scan_minmax_kernel(PredSet ps, i64 n, KeyCols kc, int nkeys,
                                   i64* __restrict__ out, i64* __restrict__ runs) {
  bool unsorted = false, longrun = false;
  i64 mn[kMaxKeys], mx[kMaxKeys];
#pragma unroll
  for (int j = 0; j < kMaxKeys; ++j) {
    mn[j] = LLONG_MAX;
    mx[j] = LLONG_MIN;
  }
  const i64 stride = (i64)gridDim.x * blockDim.x;
  i64 i0 = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (ps.npreds == 0 && nkeys == 1 && kc.dt[0] == TDP_I64) {
    // one unfiltered int64 key (group-by planning, column statistics): four
    // rows' loads in flight per thread
    const i64* __restrict__ key = reinterpret_cast<const i64*>(kc.p[0]);
    for (; i0 + 3 * stride < n; i0 += 4 * stride) {
      i64 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(key + i0 + u * stride);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const i64 i = i0 + u * stride;
        mn[0] = v[u] < mn[0] ? v[u] : mn[0];
        mx[0] = v[u] > mx[0] ? v[u] : mx[0];
        if (runs != nullptr && i > 0) {
          unsorted |= v[u] < __ldg(key + i - 1);
          if (i >= kRunMax) longrun |= v[u] == __ldg(key + i - kRunMax);
        }
      }
    }
  }
  for (i64 i = i0; i < n; i += stride) {
    if (!eval_all(ps, i)) continue;
#pragma unroll
    for (int j = 0; j < kMaxKeys; ++j) {
      if (j < nkeys) {
        const i64 v = load_as_i64(kc.p[j], kc.dt[j], i);
        mn[j] = v < mn[j] ? v : mn[j];
        mx[j] = v > mx[j] ? v : mx[j];
        if (j == 0 && runs != nullptr && i > 0) {
          unsorted |= v < load_as_i64(kc.p[0], kc.dt[0], i - 1);
          if (i >= kRunMax) longrun |= v == load_as_i64(kc.p[0], kc.dt[0], i - kRunMax);
        }
      }
    }
  }
  if (runs != nullptr) {
    if (__any_sync(0xffffffffu, unsorted) && (threadIdx.x & 31) == 0) runs[0] = 1;
    if (__any_sync(0xffffffffu, longrun) && (threadIdx.x & 31) == 0) runs[1] = 1;
  }
#pragma unroll
  for (int j = 0; j < kMaxKeys; ++j) {
    if (j < nkeys) {
      i64 a = mn[j], b = mx[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const i64 ta = __shfl_xor_sync(0xffffffffu, a, o);
        const i64 tb = __shfl_xor_sync(0xffffffffu, b, o);
        a = ta < a ? ta : a;
        b = tb > b ? tb : b;
      }
      if ((threadIdx.x & 31) == 0) {
        atomicMin(reinterpret_cast<long long*>(out) + 2 * j, a);
        atomicMax(reinterpret_cast<long long*>(out) + 2 * j + 1, b);
      }
    }
  }
}

__global__ void set_i64_kernel(i64* out, i64 v) { *out = v; }

__global__ void init_minmax_kernel(i64* out, int nkeys) {
  const int j = threadIdx.x;
  if (j < nkeys) {
    out[2 * j] = LLONG_MAX;
    out[2 * j + 1] = LLONG_MIN;
  }
}

int build_spec(Spec& s, const tdp_column* cols, int32_t ncols, int64_t n,
               const tdp_predicate* preds, int32_t npreds, const tdp_instr* prog, int32_t nprog,
               const tdp_key* keys, int32_t nkeys, const tdp_agg* aggs, int32_t naggs,
               const int32_t* outs, int32_t nouts) {
  TDP_REQUIRE(n >= 0, "negative row count");
  TDP_REQUIRE(npreds >= 0 && nprog >= 0 && nkeys >= 0 && naggs >= 0 && nouts >= 0,
              "negative descriptor count");
  TDP_REQUIRE(naggs <= 32, "at most 32 aggregates");
  s.preds.assign(preds, preds + npreds);
  s.prog.assign(prog, prog + nprog);
  s.keys.assign(keys, keys + nkeys);
  s.aggs.assign(aggs, aggs + naggs);
  s.outs.assign(outs, outs + nouts);
  return validate_and_derive(s, cols, ncols, n);
}

AggMap make_map(const Spec& s) {
  AggMap m;
  std::memset(&m, 0, sizeof(m));
  m.naggs = (int)s.aggs.size();
  m.nf = (int)s.fvals.size();
  m.ni = (int)s.ivals.size();
  for (int a = 0; a < m.naggs; ++a) {
    m.kind[a] = s.aggs[a].kind;
    m.acc[a] = s.agg_acc[a];
    m.scale[a] = s.aggs[a].kind == kAggSumDec ? s.iscale[s.agg_acc[a]] : 0.0;
  }
  return m;
}

i64 cells_of(const Spec& s) { return s.slots * (i64)(1 + s.fvals.size() + s.ivals.size()); }

}  // namespace

// ---- kernel timer (benchmarks) ---------------------------------------------
// kind 1: the fused scan kernels; kind 2: the join probe kernels
std::mutex g_timer_mu;
int g_timer_on = 0;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_timer_events;

cudaEvent_t timer_begin(int kind, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(g_timer_mu);
  if (g_timer_on != kind) return nullptr;
  cudaEvent_t a = nullptr;
  if (cudaEventCreate(&a) != cudaSuccess) return nullptr;
  cudaEventRecord(a, st);
  return a;
}

void timer_end(cudaEvent_t a, cudaStream_t st) {
  if (!a) return;
  cudaEvent_t b = nullptr;
  if (cudaEventCreate(&b) != cudaSuccess) return;
  cudaEventRecord(b, st);
  std::lock_guard<std::mutex> lock(g_timer_mu);
  g_timer_events.emplace_back(a, b);
}

}  // namespace tdp

using namespace tdp;

extern "C" {

int tdp_pipeline_codegen(const tdp_column* cols, int32_t ncols, int64_t n,
                         const tdp_predicate* preds, int32_t npreds, const tdp_instr* prog,
                         int32_t nprog, const tdp_key* keys, int32_t nkeys, const tdp_agg* aggs,
                         int32_t naggs, const int32_t* outs, int32_t nouts, int32_t compile,
                         char* out_src, size_t cap) {
  Spec s;
  int rc = build_spec(s, cols, ncols, n, preds, npreds, prog, nprog, keys, nkeys, aggs, naggs,
                      outs, nouts);
  if (rc) return rc;
  const std::string src = generate(s);
  if (out_src && cap) {
    const size_t m = src.size() < cap - 1 ? src.size() : cap - 1;
    std::memcpy(out_src, src.data(), m);
    out_src[m] = '\0';
  }
  if (compile) {
    std::vector<char> cubin;
    rc = nvrtc_compile(src, &cubin);
    if (rc) return rc;
  }
  return (int)(src.size() > 0x7fffffff ? 0x7fffffff : src.size());
}

int tdp_kernel_timer_enable(int32_t on) {
  std::lock_guard<std::mutex> lock(g_timer_mu);
  g_timer_on = on;
  return TDP_OK;
}

int tdp_kernel_timer_read(double* total_ms, int64_t* launches) {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs;
  {
    std::lock_guard<std::mutex> lock(g_timer_mu);
    evs.swap(g_timer_events);
  }
  double total = 0.0;
  for (auto& e : evs) {
    float ms = 0.f;
    TDP_CUDA_TRY(cudaEventSynchronize(e.second));
    TDP_CUDA_TRY(cudaEventElapsedTime(&ms, e.first, e.second));
    total += ms;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  if (total_ms) *total_ms = total;
  if (launches) *launches = (int64_t)evs.size();
  return TDP_OK;
}

size_t tdp_scan_aggregate_workspace(int64_t n, int64_t slots, int32_t naggs) {
  (void)n;
  const i64 cells = (slots > 0 ? slots : 1) * (i64)(1 + (naggs > 0 ? naggs : 0));
  const i64 reg_rows = (i64)sm_count() * 32;
  const i64 reg = reg_rows * (cells < kMaxRegCells ? cells : kMaxRegCells);
  return (size_t)((reg > cells ? reg : cells) * 8 + 256);
}

}  // extern "C"

namespace tdp {
namespace {
struct GroupOut {  // finalisation outputs (tdp_scan_aggregate_grouped)
  unsigned long long avg_mask;
  int64_t* keys;
  int64_t* counts;
  void* aggs;
  int64_t* groups;
};

int key_digits(const tdp_key* keys, int nkeys, i64 slots, KeyDigits* kd) {
  TDP_REQUIRE(nkeys >= 0 && nkeys <= kMaxKeys, "bad key count");
  std::memset(kd, 0, sizeof(*kd));
  kd->nkeys = nkeys;
  i64 prod = 1;
  for (int j = nkeys - 1; j >= 0; --j) {
    TDP_REQUIRE(keys[j].span >= 1, "key %d: bad span", j);
    kd->lo[j] = keys[j].lo;
    kd->span[j] = keys[j].span;
    kd->stride[j] = prod;
    prod *= keys[j].span;
  }
  TDP_REQUIRE(prod == slots, "slots %lld != product of key spans %lld", (long long)slots,
              (long long)prod);
  return TDP_OK;
}

int scan_aggregate_impl(const tdp_column* cols, int32_t ncols, int64_t n,
                        const tdp_predicate* preds, int32_t npreds, const tdp_instr* prog,
                        int32_t nprog, const tdp_key* keys, int32_t nkeys, const tdp_agg* aggs,
                        int32_t naggs, int64_t* out_counts, void* out_sums, void* ws,
                        size_t ws_bytes, void* stream, const GroupOut* fin) {
  Spec s;
  int rc = build_spec(s, cols, ncols, n, preds, npreds, prog, nprog, keys, nkeys, aggs, naggs,
                      nullptr, 0);
  if (rc) return rc;
  TDP_REQUIRE(out_counts != nullptr, "null count output");
  TDP_REQUIRE(naggs == 0 || out_sums != nullptr, "null sums output");
  cudaStream_t st = as_stream(stream);
  const i64 cells = cells_of(s);
  const Ring ring = ring_shape(s);
  std::shared_ptr<Kernel> k;
  rc = compile(s, ring, s.acc_smem, &k);
  if (rc) return rc;
  Driver* d = nullptr;
  rc = get_driver(&d);
  if (rc) return rc;
  // The bulk-copy ring needs 16-byte aligned column bases and at least one
  // full tile per CTA to be worth its setup; otherwise use the register path.
  bool aligned = true;
  for (int c : s.used_cols) aligned &= ((uintptr_t)cols[c].data & 15) == 0;
  const i64 ntiles = n / ring.ptile;
  const bool use_ring = aligned && ntiles >= (i64)sm_count();
  const i64 max_rows = (i64)sm_count() * 32;
  i64 grid;
  unsigned threads;
  size_t smem;
  CUfunction fn;
  if (use_ring) {
    grid = ntiles < (i64)sm_count() * k->agg_occ ? ntiles : (i64)sm_count() * k->agg_occ;
    threads = (kConsWarps + 1) * 32;
    smem = k->ring_smem;
    fn = k->agg;
  } else {
    grid = ceil_div(n > 0 ? n : 1, (i64)kThreads * kUnroll);
    const i64 cap = (i64)sm_count() * (s.regacc ? k->ldg_occ : 2 * k->ldg_occ);
    if (grid > cap) grid = cap;
    threads = kThreads;
    smem = k->ldg_smem;
    fn = k->agg_ldg;
  }
  if (grid > max_rows) grid = max_rows;
  const i64 rows = s.regacc ? grid : 1;
  TDP_REQUIRE(ws != nullptr && ws_bytes >= (size_t)(rows * cells * 8),
              "scan_aggregate workspace too small (%zu < %lld)", ws_bytes,
              (long long)(rows * cells * 8));
  if (!s.regacc) TDP_CUDA_TRY(cudaMemsetAsync(ws, 0, (size_t)cells * 8, st));
  if (n > 0 || s.regacc) {
    HostParams hp;
    fill_params(hp, s, cols, ncols, n);
    hp.acc = ws;
    void* args[] = {&hp};
    cudaEvent_t t0 = timer_begin(1, st);
    rc = cu_check(d,
                  d->launch(fn, (unsigned)grid, 1, 1, threads, 1, 1, (unsigned)smem, (CUstream)st,
                            args, nullptr),
                  use_ring ? "cuLaunchKernel(tdp_scan_agg)" : "cuLaunchKernel(tdp_scan_agg_ldg)");
    if (rc) return rc;
    timer_end(t0, st);
    count_launch();
  }
  AggMap m = make_map(s);
  const i64 items = s.slots * (1 + naggs);
  if (fin != nullptr) {
    KeyDigits kd;
    rc = key_digits(keys, nkeys, s.slots, &kd);
    if (rc) return rc;
    if (items <= kFusedTailItems) {
      reduce_finalize_kernel<<<1, 1024, 0, st>>>(
          reinterpret_cast<const u64*>(ws), (int)rows, (int)s.slots, m, out_counts,
          reinterpret_cast<u64*>(out_sums), kd, fin->avg_mask, fin->keys, fin->counts,
          reinterpret_cast<u64*>(fin->aggs), fin->groups);
      TDP_LAUNCH_CHECK("reduce_finalize_kernel");
      return TDP_OK;
    }
    agg_reduce_kernel<<<(unsigned)ceil_div(items * 32, 256), 256, 0, st>>>(
        reinterpret_cast<const u64*>(ws), (int)rows, (int)s.slots, m, out_counts,
        reinterpret_cast<u64*>(out_sums));
    TDP_LAUNCH_CHECK("agg_reduce_kernel");
    finalize_kernel<<<1, 1024, 0, st>>>(out_counts, reinterpret_cast<const u64*>(out_sums),
                                        s.slots, kd, m, fin->avg_mask, fin->keys, fin->counts,
                                        reinterpret_cast<u64*>(fin->aggs), fin->groups);
    TDP_LAUNCH_CHECK("finalize_kernel");
    return TDP_OK;
  }
  agg_reduce_kernel<<<(unsigned)ceil_div(items * 32, 256), 256, 0, st>>>(
      reinterpret_cast<const u64*>(ws), (int)rows, (int)s.slots, m, out_counts,
      reinterpret_cast<u64*>(out_sums));
  TDP_LAUNCH_CHECK("agg_reduce_kernel");
  return TDP_OK;
}
}  // namespace
}  // namespace tdp

extern "C" {

int tdp_scan_aggregate(const tdp_column* cols, int32_t ncols, int64_t n,
                       const tdp_predicate* preds, int32_t npreds, const tdp_instr* prog,
                       int32_t nprog, const tdp_key* keys, int32_t nkeys, const tdp_agg* aggs,
                       int32_t naggs, int64_t* out_counts, void* out_sums, void* ws,
                       size_t ws_bytes, void* stream) {
  return scan_aggregate_impl(cols, ncols, n, preds, npreds, prog, nprog, keys, nkeys, aggs, naggs,
                             out_counts, out_sums, ws, ws_bytes, stream, nullptr);
}

int tdp_scan_aggregate_grouped(const tdp_column* cols, int32_t ncols, int64_t n,
                               const tdp_predicate* preds, int32_t npreds, const tdp_instr* prog,
                               int32_t nprog, const tdp_key* keys, int32_t nkeys,
                               const tdp_agg* aggs, int32_t naggs, int64_t* out_counts,
                               void* out_sums, void* ws, size_t ws_bytes, uint64_t avg_mask,
                               int64_t* out_keys, int64_t* out_group_counts, void* out_aggs,
                               int64_t* out_groups, void* stream) {
  TDP_REQUIRE(out_keys != nullptr && out_group_counts != nullptr && out_groups != nullptr &&
                  (naggs == 0 || out_aggs != nullptr),
              "null finalisation output");
  GroupOut fin{(unsigned long long)avg_mask, out_keys, out_group_counts, out_aggs, out_groups};
  return scan_aggregate_impl(cols, ncols, n, preds, npreds, prog, nprog, keys, nkeys, aggs, naggs,
                             out_counts, out_sums, ws, ws_bytes, stream, &fin);
}

int tdp_scan_project(const tdp_column* cols, int32_t ncols, int64_t n,
                     const tdp_predicate* preds, int32_t npreds, const tdp_instr* prog,
                     int32_t nprog, const int32_t* outs, int32_t nouts, void* const* out_ptrs,
                     int64_t* out_count, void* ws, size_t ws_bytes, void* stream) {
  Spec s;
  int rc = build_spec(s, cols, ncols, n, preds, npreds, prog, nprog, nullptr, 0, nullptr, 0,
                      outs, nouts);
  if (rc) return rc;
  TDP_REQUIRE(out_count != nullptr, "null count output");
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    TDP_CUDA_TRY(cudaMemsetAsync(out_count, 0, sizeof(i64), st));
    return TDP_OK;
  }
  std::shared_ptr<Kernel> k;
  rc = compile(s, ring_shape(s), s.acc_smem, &k);
  if (rc) return rc;
  Driver* d = nullptr;
  rc = get_driver(&d);
  if (rc) return rc;
  HostParams hp;
  fill_params(hp, s, cols, ncols, n);
  for (int o = 0; o < nouts; ++o) hp.out[o] = out_ptrs[o];
  unsigned grid;
  if (npreds > 0) {
    TDP_REQUIRE(ws_bytes >= tdp_filter_workspace(n), "project workspace too small");
    PredSet ps;
    rc = make_predset(cols, ncols, preds, npreds, n, &ps);
    if (rc) return rc;
    const i64 tiles = ceil_div(n, kFilterTile);
    unsigned char* p = reinterpret_cast<unsigned char*>(ws);
    unsigned* bits = reinterpret_cast<unsigned*>(p);
    p += ((size_t)tiles * kFilterWords * sizeof(unsigned) + 255) & ~(size_t)255;
    i64* counts = reinterpret_cast<i64*>(p);
    i64* offsets = counts + tiles;
    void* scan_ws = offsets + tiles;
    const size_t used = (size_t)((unsigned char*)scan_ws - (unsigned char*)ws);
    rc = filter_bits(ps, n, bits, counts, st);
    if (rc) return rc;
    rc = exclusive_scan_i64(counts, offsets, tiles, out_count, scan_ws, ws_bytes - used, st);
    if (rc) return rc;
    hp.bits = bits;
    hp.tile_off = offsets;
    grid = (unsigned)tiles;
  } else {
    set_i64_kernel<<<1, 1, 0, st>>>(out_count, n);
    TDP_LAUNCH_CHECK("set_i64_kernel");
    grid = (unsigned)stream_grid(n, 256 * 4, 8);
  }
  void* args[] = {&hp};
  rc = cu_check(d, d->launch(k->proj, grid, 1, 1, 256, 1, 1, 0, (CUstream)st, args, nullptr),
                "cuLaunchKernel(tdp_scan_project)");
  if (rc) return rc;
  count_launch();
  return TDP_OK;
}

int tdp_groupby_finalize(const int64_t* counts, const void* sums, int64_t slots,
                         const tdp_key* keys, int32_t nkeys, const tdp_agg* aggs, int32_t naggs,
                         uint64_t avg_mask, int64_t* out_keys, int64_t* out_counts,
                         void* out_aggs, int64_t* out_groups, void* stream) {
  TDP_REQUIRE(slots >= 1, "slots must be >= 1");
  TDP_REQUIRE(nkeys >= 0 && nkeys <= kMaxKeys, "bad key count");
  TDP_REQUIRE(naggs >= 0 && naggs <= 32, "bad aggregate count");
  KeyDigits kd;
  std::memset(&kd, 0, sizeof(kd));
  kd.nkeys = nkeys;
  i64 prod = 1;
  for (int j = nkeys - 1; j >= 0; --j) {
    TDP_REQUIRE(keys[j].span >= 1, "key %d: bad span", j);
    kd.lo[j] = keys[j].lo;
    kd.span[j] = keys[j].span;
    kd.stride[j] = prod;
    prod *= keys[j].span;
  }
  TDP_REQUIRE(prod == slots, "slots %lld != product of key spans %lld", (long long)slots,
              (long long)prod);
  AggMap m;
  std::memset(&m, 0, sizeof(m));
  m.naggs = naggs;
  for (int a = 0; a < naggs; ++a) m.kind[a] = aggs[a].kind;
  finalize_kernel<<<1, 1024, 0, as_stream(stream)>>>(
      counts, reinterpret_cast<const u64*>(sums), slots, kd, m,
      (unsigned long long)avg_mask, out_keys, out_counts, reinterpret_cast<u64*>(out_aggs),
      out_groups);
  TDP_LAUNCH_CHECK("finalize_kernel");
  return TDP_OK;
}

int tdp_scan_minmax_runs(const tdp_column* cols, int32_t ncols, int64_t n,
                         const tdp_predicate* preds, int32_t npreds, const int32_t* key_cols,
                         int32_t nkeys, int64_t* out_minmax, int64_t* out_runs, void* stream) {
  TDP_REQUIRE(nkeys >= 1 && nkeys <= kMaxKeys, "bad key count");
  TDP_REQUIRE(out_runs == nullptr || (nkeys == 1 && npreds == 0),
              "run detection needs one key and no predicates");
  PredSet ps;
  int rc = make_predset(cols, ncols, preds, npreds, n, &ps);
  if (rc) return rc;
  KeyCols kc;
  std::memset(&kc, 0, sizeof(kc));
  for (int j = 0; j < nkeys; ++j) {
    TDP_REQUIRE(key_cols[j] >= 0 && key_cols[j] < ncols, "key %d: bad column", j);
    const tdp_column& c = cols[key_cols[j]];
    TDP_REQUIRE(c.dtype == TDP_I64 || c.dtype == TDP_I32 || c.dtype == TDP_BOOL,
                "key %d: integer column required", j);
    TDP_REQUIRE(c.rows >= n, "key %d: short column", j);
    kc.p[j] = c.data;
    kc.dt[j] = c.dtype;
  }
  cudaStream_t st = as_stream(stream);
  if (out_runs != nullptr) TDP_CUDA_TRY(cudaMemsetAsync(out_runs, 0, 2 * sizeof(i64), st));
  init_minmax_kernel<<<1, 32, 0, st>>>(out_minmax, nkeys);
  TDP_LAUNCH_CHECK("init_minmax_kernel");
  if (n == 0) return TDP_OK;
  scan_minmax_kernel<<<stream_grid(n, 256 * 8, 8), 256, 0, st>>>(ps, n, kc, nkeys, out_minmax,
                                                                  out_runs);
  TDP_LAUNCH_CHECK("scan_minmax_kernel");
  return TDP_OK;
}

int tdp_scan_minmax(const tdp_column* cols, int32_t ncols, int64_t n,
                    const tdp_predicate* preds, int32_t npreds, const int32_t* key_cols,
                    int32_t nkeys, int64_t* out_minmax, void* stream) {
  return tdp_scan_minmax_runs(cols, ncols, n, preds, npreds, key_cols, nkeys, out_minmax, nullptr,
                              stream);
}

}  // extern "C"
