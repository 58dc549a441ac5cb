// Device CSV ingestion ("register_csv onto device";
// tq/storage.py:190-249 register_csv / read_csv).
//
// The reference reads a comma-separated, double-quoted UTF-8 file with
// Python's csv module (excel dialect) and converts each cell with int() /
// float() / dict_encode on the host.  Here the file's bytes are uploaded once
// and tokenised on the device:
//
//   1. structure, speculatively per 512-byte chunk: quote count and the
//      delimiters / record ends outside quotes assuming the chunk starts
//      outside quotes (the other hypothesis is the complement); a scan of the
//      quote counts fixes every chunk's real starting state, scans of the
//      chosen counts give each chunk its first field / record index;
//   2. a second pass per chunk writes the byte position of every field end
//      and, per record, the index of its last field, and rejects what the
//      fast path does not model (a quote that neither opens a field nor
//      closes one / escapes a quote, an empty line, malformed UTF-8) -- the
//      caller then falls back to the host reader, which reproduces the
//      reference's result or error exactly;
//   3. per column: int64 (Python int(): sign, digits, single underscores
//      between digits, surrounding ASCII whitespace) and float64 (Python
//      float(): decimal / exponent / inf / nan forms) parsed per cell; a
//      float is produced on the device only when it is exact there -- at most
//      19 significant digits, mantissa < 2^53 and |10-exponent| <= 22, where
//      one IEEE multiply or divide of two exact values is correctly rounded
//      (Clinger's fast path) -- other cells are marked for the host's float();
//      string columns are unquoted / unescaped into one byte buffer for the
//      device dictionary encoder (strings.cu).
#include <math_constants.h>

#include "tdp_common.cuh"

namespace tdp {
namespace {

constexpr int kCsvChunk = 512;

// per-chunk structure counts (hypothesis A: the chunk starts outside quotes)
struct CsvChunk {
  unsigned quotes, fields_a, recs_a, fields_all, recs_all;
};

__device__ __forceinline__ bool csv_record_end(const unsigned char* b, i64 i) {
  const unsigned char c = b[i];
  if (c == '\r') return true;
  return c == '\n' && (i == 0 || b[i - 1] != '\r');
}

__global__ void csv_chunk_kernel(const unsigned char* __restrict__ b, i64 n, i64 nchunks,
                                 CsvChunk* __restrict__ out) {
  for (i64 c = (i64)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks;
       c += (i64)gridDim.x * blockDim.x) {
    const i64 lo = c * kCsvChunk, hi = lo + kCsvChunk < n ? lo + kCsvChunk : n;
    unsigned p = 0, q = 0, fa = 0, ra = 0, ft = 0, rt = 0;
    for (i64 i = lo; i < hi; ++i) {
      const unsigned char ch = b[i];
      if (ch == '"') {
        p ^= 1u;
        ++q;
        continue;
      }
      const bool rec = csv_record_end(b, i);
      if (ch == ',' || rec) {
        ++ft;
        fa += p ^ 1u;
        if (rec) {
          ++rt;
          ra += p ^ 1u;
        }
      }
    }
    out[c] = CsvChunk{q, fa, ra, ft, rt};
  }
}

// chosen counts per chunk from the scanned quote parity
__global__ void csv_choose_kernel(const CsvChunk* __restrict__ st, const i64* __restrict__ qpre,
                                  i64 nchunks, i64* __restrict__ fields, i64* __restrict__ recs) {
  for (i64 c = (i64)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks;
       c += (i64)gridDim.x * blockDim.x) {
    const bool inside = qpre[c] & 1;
    const CsvChunk s = st[c];
    fields[c] = inside ? s.fields_all - s.fields_a : s.fields_a;
    recs[c] = inside ? s.recs_all - s.recs_a : s.recs_a;
  }
}

__device__ __forceinline__ bool utf8_cont(unsigned char c) { return (c & 0xC0) == 0x80; }

// Well-formed UTF-8 at byte i (lead bytes check their continuation bytes,
// continuation bytes only that a lead byte within 3 bytes claims them).
__device__ __forceinline__ bool utf8_ok(const unsigned char* b, i64 n, i64 i) {
  const unsigned char c = b[i];
  if (c < 0x80) return true;
  if (utf8_cont(c)) {
    for (int k = 1; k <= 3 && i - k >= 0; ++k) {
      const unsigned char l = b[i - k];
      if (utf8_cont(l)) continue;
      const int len = l >= 0xF0 ? 4 : l >= 0xE0 ? 3 : l >= 0xC0 ? 2 : 1;
      return k < len;
    }
    return false;
  }
  int len;
  unsigned cp;
  if (c >= 0xC2 && c <= 0xDF) {
    len = 2;
    cp = c & 0x1F;
  } else if (c >= 0xE0 && c <= 0xEF) {
    len = 3;
    cp = c & 0x0F;
  } else if (c >= 0xF0 && c <= 0xF4) {
    len = 4;
    cp = c & 0x07;
  } else {
    return false;
  }
  if (i + len > n) return false;
  for (int k = 1; k < len; ++k) {
    if (!utf8_cont(b[i + k])) return false;
    cp = (cp << 6) | (b[i + k] & 0x3F);
  }
  if (len == 3 && (cp < 0x800 || (cp >= 0xD800 && cp <= 0xDFFF))) return false;
  if (len == 4 && (cp < 0x10000 || cp > 0x10FFFF)) return false;
  return true;
}

// Field ends, record ends, anomalies.  flags: [0] anomaly (host path).
__global__ void csv_write_kernel(const unsigned char* __restrict__ b, i64 n, i64 nchunks,
                                 const i64* __restrict__ qpre, const i64* __restrict__ fpre,
                                 const i64* __restrict__ rpre, i64* __restrict__ fend,
                                 i64* __restrict__ rend, int* __restrict__ flags) {
  for (i64 c = (i64)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks;
       c += (i64)gridDim.x * blockDim.x) {
    const i64 lo = c * kCsvChunk, hi = lo + kCsvChunk < n ? lo + kCsvChunk : n;
    unsigned p = (unsigned)(qpre[c] & 1);
    i64 fi = fpre[c], ri = rpre[c];
    bool bad = false;
    for (i64 i = lo; i < hi; ++i) {
      const unsigned char ch = b[i];
      bad |= !utf8_ok(b, n, i);
      if (ch == '"') {
        if (p == 0) {  // opens: at a field start, or the second quote of a "" escape
          const unsigned char pr = i > 0 ? b[i - 1] : ',';
          bad |= !(pr == ',' || pr == '\n' || pr == '\r' || pr == '"');
        } else {  // closes: before a delimiter, a record end or an escaped quote
          const unsigned char nx = i + 1 < n ? b[i + 1] : '\n';
          bad |= !(nx == ',' || nx == '\n' || nx == '\r' || nx == '"');
        }
        p ^= 1u;
        continue;
      }
      if (p) continue;
      const bool rec = csv_record_end(b, i);
      if (ch != ',' && !rec) continue;
      fend[fi] = i;
      if (rec) {
        // an empty line (csv.reader yields [] for it) is left to the host
        if (i == 0 || b[i - 1] == '\n' || b[i - 1] == '\r') bad = true;
        rend[ri++] = fi;
      }
      ++fi;
    }
    if (bad) atomicOr(flags, 1);
  }
}

// A record whose field count differs from ncols (the host raises the exact
// StorageError): the smallest such record index into flags[1] (init INT_MAX).
__global__ void csv_check_kernel(const i64* __restrict__ rend, i64 nrec, int ncols,
                                 int* __restrict__ flags) {
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < nrec;
       r += (i64)gridDim.x * blockDim.x) {
    const i64 prev = r ? rend[r - 1] : -1;
    if (rend[r] - prev != ncols) atomicMin(flags + 1, (int)(r < 0x7fffffff ? r : 0x7fffffff));
  }
}

__device__ __forceinline__ i64 csv_field_start(const unsigned char* b, const i64* fend, i64 fi) {
  if (fi == 0) return 0;
  const i64 e = fend[fi - 1];
  return e + 1 + ((b[e] == '\r' && b[e + 1] == '\n') ? 1 : 0);
}

__device__ __forceinline__ bool csv_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f';
}

__device__ __forceinline__ bool lower_eq(const unsigned char* s, i64 len, const char* w) {
  i64 k = 0;
  for (; w[k]; ++k)
    if (k >= len || (s[k] | 0x20) != (unsigned char)w[k]) return false;
  return k == len;
}

// status: 0 ok, 1 the host converts this cell (exactness), 2 invalid (the
// host reader raises the reference's error)
constexpr int kCellOk = 0, kCellHost = 1, kCellBad = 2;

__device__ int csv_parse_int(const unsigned char* s, i64 len, i64* out) {
  i64 k = 0;
  bool neg = false;
  if (k < len && (s[k] == '+' || s[k] == '-')) neg = s[k++] == '-';
  if (k >= len) return kCellBad;
  unsigned long long v = 0;
  bool digit_before = false, over = false;
  for (; k < len; ++k) {
    const unsigned char c = s[k];
    if (c == '_') {  // single underscores between digits
      if (!digit_before || k + 1 >= len || s[k + 1] < '0' || s[k + 1] > '9') return kCellBad;
      digit_before = false;
      continue;
    }
    if (c < '0' || c > '9') return c >= 0x80 ? kCellHost : kCellBad;
    digit_before = true;
    if (v > (~0ull - 9) / 10) over = true;
    v = v * 10 + (c - '0');
  }
  // beyond int64: np.asarray raises OverflowError on the host
  if (over || v > (neg ? 0x8000000000000000ull : 0x7fffffffffffffffull)) return kCellHost;
  *out = neg ? (i64)(0ull - v) : (i64)v;
  return kCellOk;
}

__device__ int csv_parse_float(const unsigned char* s, i64 len, double* out) {
  i64 k = 0;
  bool neg = false;
  if (k < len && (s[k] == '+' || s[k] == '-')) neg = s[k++] == '-';
  const unsigned char* t = s + k;
  const i64 tl = len - k;
  if (lower_eq(t, tl, "inf") || lower_eq(t, tl, "infinity")) {
    *out = neg ? -CUDART_INF : CUDART_INF;
    return kCellOk;
  }
  if (lower_eq(t, tl, "nan")) {  // Python's NaN bits: 0x7ff8..., sign set for "-nan"
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    *out = neg ? -qnan : qnan;
    return kCellOk;
  }
  unsigned long long m = 0;
  int sig = 0;         // significant digits kept in m
  i64 e10 = 0;         // decimal exponent adjustment
  bool any = false, dropped = false, digit_before = false;
  // integer part
  for (; k < len; ++k) {
    const unsigned char c = s[k];
    if (c == '_') {
      if (!digit_before || k + 1 >= len || s[k + 1] < '0' || s[k + 1] > '9') return kCellBad;
      digit_before = false;
      continue;
    }
    if (c < '0' || c > '9') break;
    any = digit_before = true;
    if (m == 0 && c == '0') continue;
    if (sig < 19) {
      m = m * 10 + (c - '0');
      ++sig;
    } else {
      ++e10;
      dropped |= c != '0';
    }
  }
  if (k < len && s[k] == '.') {
    ++k;
    digit_before = false;
    for (; k < len; ++k) {
      const unsigned char c = s[k];
      if (c == '_') {
        if (!digit_before || k + 1 >= len || s[k + 1] < '0' || s[k + 1] > '9') return kCellBad;
        digit_before = false;
        continue;
      }
      if (c < '0' || c > '9') break;
      any = digit_before = true;
      if (m == 0 && c == '0') {
        --e10;
        continue;
      }
      if (sig < 19) {
        m = m * 10 + (c - '0');
        ++sig;
        --e10;
      } else {
        dropped |= c != '0';
      }
    }
  }
  if (!any) return kCellBad;
  if (k < len && (s[k] == 'e' || s[k] == 'E')) {
    ++k;
    bool eneg = false;
    if (k < len && (s[k] == '+' || s[k] == '-')) eneg = s[k++] == '-';
    i64 ev = 0;
    bool edig = false;
    digit_before = false;
    for (; k < len; ++k) {
      const unsigned char c = s[k];
      if (c == '_') {
        if (!digit_before || k + 1 >= len || s[k + 1] < '0' || s[k + 1] > '9') return kCellBad;
        digit_before = false;
        continue;
      }
      if (c < '0' || c > '9') break;
      edig = digit_before = true;
      if (ev < 100000) ev = ev * 10 + (c - '0');
    }
    if (!edig) return kCellBad;
    e10 += eneg ? -ev : ev;
  }
  if (k != len) return s[k] >= 0x80 ? kCellHost : kCellBad;
  if (m == 0) {
    *out = neg ? -0.0 : 0.0;
    return kCellOk;
  }
  if (dropped || m >= (1ull << 53) || e10 < -22 || e10 > 22) return kCellHost;
  double p10 = 1.0;
  for (i64 j = 0; j < (e10 < 0 ? -e10 : e10); ++j) p10 *= 10.0;  // exact up to 1e22
  const double v = e10 < 0 ? __ddiv_rn((double)m, p10) : __dmul_rn((double)m, p10);
  *out = neg ? -v : v;
  return kCellOk;
}

// One thread per data row: cell (row + 1, col) as int64 (kind 0) or float64.
__global__ void csv_numeric_kernel(const unsigned char* __restrict__ b,
                                   const i64* __restrict__ fend, int ncols, int col, i64 nrows,
                                   int kind, void* __restrict__ out,
                                   unsigned char* __restrict__ status) {
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < nrows;
       r += (i64)gridDim.x * blockDim.x) {
    const i64 fi = (r + 1) * ncols + col;
    i64 s = csv_field_start(b, fend, fi), e = fend[fi];
    if (e > s && b[s] == '"') {  // quoted: the value inside (a quote inside is no number)
      if (e - s < 2 || b[e - 1] != '"') {
        status[r] = kCellBad;
        continue;
      }
      ++s;
      --e;
      bool q = false;
      for (i64 i = s; i < e; ++i) q |= b[i] == '"';
      if (q) {
        status[r] = kCellBad;
        continue;
      }
    }
    while (s < e && csv_space(b[s])) ++s;
    while (e > s && csv_space(b[e - 1])) --e;
    int st;
    if (e == s) {
      st = kCellBad;  // empty cell
    } else if (kind == 0) {
      i64 v = 0;
      st = csv_parse_int(b + s, e - s, &v);
      reinterpret_cast<i64*>(out)[r] = v;
    } else {
      double v = 0.0;
      st = csv_parse_float(b + s, e - s, &v);
      reinterpret_cast<double*>(out)[r] = v;
    }
    // non-ASCII around the value (Unicode whitespace) is the host's to judge
    if (st == kCellBad)
      for (i64 i = s; i < e; ++i)
        if (b[i] >= 0x80) st = kCellHost;
    status[r] = (unsigned char)st;
  }
}

// String column: unescaped byte length of each cell (quoted cells lose their
// quotes, "" becomes ").
__global__ void csv_str_len_kernel(const unsigned char* __restrict__ b,
                                   const i64* __restrict__ fend, int ncols, int col, i64 nrows,
                                   i64* __restrict__ lens) {
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < nrows;
       r += (i64)gridDim.x * blockDim.x) {
    const i64 fi = (r + 1) * ncols + col;
    const i64 s = csv_field_start(b, fend, fi), e = fend[fi];
    i64 len = e - s;
    if (len >= 2 && b[s] == '"') {
      len = 0;
      for (i64 i = s + 1; i < e - 1; ++i) {
        ++len;
        if (b[i] == '"') ++i;  // "" -> "
      }
    }
    lens[r] = len;
  }
}

__global__ void csv_str_copy_kernel(const unsigned char* __restrict__ b,
                                    const i64* __restrict__ fend, int ncols, int col, i64 nrows,
                                    const i64* __restrict__ offs, unsigned char* __restrict__ dst) {
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < nrows;
       r += (i64)gridDim.x * blockDim.x) {
    const i64 fi = (r + 1) * ncols + col;
    const i64 s = csv_field_start(b, fend, fi), e = fend[fi];
    i64 o = offs[r];
    if (e - s >= 2 && b[s] == '"') {
      for (i64 i = s + 1; i < e - 1; ++i) {
        dst[o++] = b[i];
        if (b[i] == '"') ++i;
      }
    } else {
      for (i64 i = s; i < e; ++i) dst[o++] = b[i];
    }
  }
}

size_t csv_ws_bytes(i64 n) {
  const i64 nch = ceil_div(n > 0 ? n : 1, kCsvChunk);
  const size_t a = (size_t)nch * sizeof(CsvChunk);
  return ((a + 255) & ~(size_t)255) + 6 * (((size_t)nch * 8 + 255) & ~(size_t)255) +
         exclusive_scan_workspace(nch) + 1024;
}

struct CsvWs {
  CsvChunk* st;
  i64 *q, *qpre, *f, *fpre, *r, *rpre;
  void* scan_ws;
  size_t scan_bytes;
};

CsvWs carve_csv(void* ws, i64 n) {
  const i64 nch = ceil_div(n > 0 ? n : 1, kCsvChunk);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  CsvWs w;
  w.st = (CsvChunk*)p;
  p += ((size_t)nch * sizeof(CsvChunk) + 255) & ~(size_t)255;
  i64** arrs[6] = {&w.q, &w.qpre, &w.f, &w.fpre, &w.r, &w.rpre};
  for (auto a : arrs) {
    *a = (i64*)p;
    p += ((size_t)nch * 8 + 255) & ~(size_t)255;
  }
  w.scan_ws = p;
  w.scan_bytes = exclusive_scan_workspace(nch) + 512;
  return w;
}

__global__ void csv_quotes_kernel(const CsvChunk* __restrict__ st, i64 nch, i64* __restrict__ q) {
  for (i64 c = (i64)blockIdx.x * blockDim.x + threadIdx.x; c < nch;
       c += (i64)gridDim.x * blockDim.x)
    q[c] = st[c].quotes;
}

}  // namespace
}  // namespace tdp

using namespace tdp;

extern "C" {

size_t tdp_csv_workspace(int64_t nbytes) { return csv_ws_bytes(nbytes); }

size_t tdp_csv_string_workspace(int64_t nrows) {
  return (((size_t)(nrows > 0 ? nrows : 1) * 8 + 255) & ~(size_t)255) +
         exclusive_scan_workspace(nrows + 1) + 1024;
}


int tdp_csv_index(const uint8_t* bytes, int64_t nbytes, int64_t* out_counts, void* ws,
                  size_t ws_bytes, void* stream) {
  TDP_REQUIRE(nbytes > 0 && bytes != nullptr && out_counts != nullptr, "bad csv index arguments");
  TDP_REQUIRE(ws_bytes >= csv_ws_bytes(nbytes), "csv workspace too small");
  cudaStream_t st = as_stream(stream);
  const i64 nch = ceil_div(nbytes, kCsvChunk);
  CsvWs w = carve_csv(ws, nbytes);
  const unsigned grid = (unsigned)stream_grid(nch, 256, 8);
  csv_chunk_kernel<<<grid, 256, 0, st>>>(bytes, nbytes, nch, w.st);
  TDP_LAUNCH_CHECK("csv_chunk_kernel");
  csv_quotes_kernel<<<grid, 256, 0, st>>>(w.st, nch, w.q);
  TDP_LAUNCH_CHECK("csv_quotes_kernel");
  // counts: [0] fields, [1] records, [2] quotes (odd: an unterminated quoted field)
  int rc = exclusive_scan_i64(w.q, w.qpre, nch, out_counts + 2, w.scan_ws, w.scan_bytes, st);
  if (rc) return rc;
  csv_choose_kernel<<<grid, 256, 0, st>>>(w.st, w.qpre, nch, w.f, w.r);
  TDP_LAUNCH_CHECK("csv_choose_kernel");
  rc = exclusive_scan_i64(w.f, w.fpre, nch, out_counts, w.scan_ws, w.scan_bytes, st);
  if (rc) return rc;
  return exclusive_scan_i64(w.r, w.rpre, nch, out_counts + 1, w.scan_ws, w.scan_bytes, st);
}

int tdp_csv_fields(const uint8_t* bytes, int64_t nbytes, int32_t ncols, int64_t nrecords,
                   int64_t* out_field_ends, int64_t* out_record_ends, int32_t* out_flags,
                   void* ws, size_t ws_bytes, void* stream) {
  TDP_REQUIRE(nbytes > 0 && ncols >= 1 && nrecords >= 0, "bad csv field arguments");
  TDP_REQUIRE(ws_bytes >= csv_ws_bytes(nbytes), "csv workspace too small");
  cudaStream_t st = as_stream(stream);
  const i64 nch = ceil_div(nbytes, kCsvChunk);
  CsvWs w = carve_csv(ws, nbytes);
  const int init[2] = {0, 0x7fffffff};
  TDP_CUDA_TRY(cudaMemcpyAsync(out_flags, init, sizeof(init), cudaMemcpyHostToDevice, st));
  csv_write_kernel<<<(unsigned)stream_grid(nch, 256, 8), 256, 0, st>>>(
      bytes, nbytes, nch, w.qpre, w.fpre, w.rpre, out_field_ends, out_record_ends, out_flags);
  TDP_LAUNCH_CHECK("csv_write_kernel");
  if (nrecords > 0) {
    csv_check_kernel<<<(unsigned)stream_grid(nrecords, 256, 8), 256, 0, st>>>(
        out_record_ends, nrecords, ncols, out_flags);
    TDP_LAUNCH_CHECK("csv_check_kernel");
  }
  return TDP_OK;
}

int tdp_csv_parse_column(const uint8_t* bytes, const int64_t* field_ends, int32_t ncols,
                         int32_t col, int64_t nrows, int32_t kind, void* out_values,
                         uint8_t* out_status, void* stream) {
  TDP_REQUIRE(ncols >= 1 && col >= 0 && col < ncols && nrows >= 0, "bad csv column arguments");
  TDP_REQUIRE(kind == 0 || kind == 1, "csv column kind must be 0 (int64) or 1 (float64)");
  if (nrows == 0) return TDP_OK;
  csv_numeric_kernel<<<(unsigned)stream_grid(nrows, 256, 16), 256, 0, as_stream(stream)>>>(
      bytes, field_ends, ncols, col, nrows, kind, out_values, out_status);
  TDP_LAUNCH_CHECK("csv_numeric_kernel");
  return TDP_OK;
}

int tdp_csv_string_column(const uint8_t* bytes, const int64_t* field_ends, int32_t ncols,
                          int32_t col, int64_t nrows, int64_t* out_offsets, uint8_t* out_bytes,
                          void* ws, size_t ws_bytes, void* stream) {
  TDP_REQUIRE(ncols >= 1 && col >= 0 && col < ncols && nrows >= 0 && out_offsets != nullptr,
              "bad csv string arguments");
  cudaStream_t st = as_stream(stream);
  if (out_bytes == nullptr) {  // phase 1: offsets [nrows + 1] (the total last)
    TDP_REQUIRE(ws_bytes >= tdp_csv_string_workspace(nrows), "csv string workspace too small");
    if (nrows == 0) {
      TDP_CUDA_TRY(cudaMemsetAsync(out_offsets, 0, 8, st));
      return TDP_OK;
    }
    i64* lens = reinterpret_cast<i64*>(ws);
    void* sws = reinterpret_cast<unsigned char*>(ws) + (((size_t)nrows * 8 + 255) & ~(size_t)255);
    csv_str_len_kernel<<<(unsigned)stream_grid(nrows, 256, 16), 256, 0, st>>>(
        bytes, field_ends, ncols, col, nrows, lens);
    TDP_LAUNCH_CHECK("csv_str_len_kernel");
    return exclusive_scan_i64(lens, out_offsets, nrows, out_offsets + nrows, sws,
                              exclusive_scan_workspace(nrows) + 512, st);
  }
  if (nrows == 0) return TDP_OK;  // phase 2: the unescaped bytes at the offsets
  csv_str_copy_kernel<<<(unsigned)stream_grid(nrows, 256, 16), 256, 0, st>>>(
      bytes, field_ends, ncols, col, nrows, out_offsets, out_bytes);
  TDP_LAUNCH_CHECK("csv_str_copy_kernel");
  return TDP_OK;
}

}  // extern "C"
