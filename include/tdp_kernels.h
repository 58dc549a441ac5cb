/*
 * tdp_kernels.h — C ABI of the B200 (sm_100a) tensor-query hot path.
 *
 * This is the drop-in boundary for the relational operators of the reference
 * `tensorquery` package (TDP, arXiv 2211.02753).  Every function here replaces
 * one numpy primitive chain of /root/reference/pkg/src/tensorquery (abbreviated
 * tq/ below); the comment above each declaration cites the reference
 * interface it stands in for.  The Python host layer
 * (paper_2211_02753_b200/kernels.py) keeps the reference's operator
 * signatures and calls these entry points through ctypes.
 *
 * Conventions
 *  - Plain C types only: device pointers are `void*` / `const void*` owned by
 *    the caller (PyTorch allocates them); sizes are int64_t; streams are
 *    passed as `void*` (a cudaStream_t).
 *  - Every entry point returns an int status: TDP_OK (0) or a negative code.
 *    `tdp_last_error()` returns the thread-local message of the last failure.
 *  - Preconditions the reference checks in Python (KernelError / EncodingError
 *    classes) are checked by the host layer BEFORE launching; this layer
 *    returns TDP_EINVAL for malformed descriptors.
 *  - Variable-size results (selected row counts, group counts, join sizes) are
 *    written to caller-provided DEVICE int64 cells; the caller syncs lazily.
 *  - Workspace is caller-provided; `*_workspace()` functions size it.
 *  - All kernels are asynchronous on the given stream.
 */
#ifndef TDP_KERNELS_H
#define TDP_KERNELS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------------ */
/* status codes                                                              */
/* ------------------------------------------------------------------------ */
#define TDP_OK 0
#define TDP_EINVAL -1   /* malformed argument / descriptor                    */
#define TDP_ECUDA -2    /* CUDA runtime or launch failure                      */
#define TDP_ENOMEM -3   /* workspace too small                                 */
#define TDP_ENOTSUP -4  /* shape the kernel family does not cover              */
#define TDP_EJIT -5     /* runtime specialisation (NVRTC) failed               */

/* ------------------------------------------------------------------------ */
/* column descriptor                                                         */
/* ------------------------------------------------------------------------ */
/* Element types.  The reference stores int64 / float64 / float32 / bool
 * (tq/tensor.py:17-18); dictionary codes are int64 (tq/encodings.py:88).  */
enum tdp_dtype {
  TDP_I64 = 0,
  TDP_F64 = 1,
  TDP_F32 = 2,
  TDP_BOOL = 3, /* one byte per value, 0/1 */
  TDP_I32 = 4,
  /* compact storage widths: a narrow stored column whose
   * logical value is int64 (or float64 through TDP_CMP_DEC / a program
   * CAST + DIV); values are widened on load, never written              */
  TDP_I8 = 5,
  TDP_I16 = 6,
  TDP_U8 = 7
};

/* A column: `rows` values of `width` elements each, row-major, contiguous.
 * Scalar columns have width 1; PE matrices [n, k] have width k.            */
typedef struct tdp_column {
  const void* data;
  int32_t dtype;
  int32_t reserved;
  int64_t rows;
  int64_t width;
} tdp_column;

/* ------------------------------------------------------------------------ */
/* predicates (tq/kernels.py:54-84 comparison_mask)                          */
/* ------------------------------------------------------------------------ */
enum tdp_cmp_op { TDP_EQ = 0, TDP_NE = 1, TDP_LT = 2, TDP_GT = 3, TDP_LE = 4, TDP_GE = 5 };

/* How the column value and literal are compared.  The host layer resolves
 * numpy-2 (NEP 50) promotion once per predicate:
 *   TDP_CMP_I64  int64(x)  <op> lit_i
 *   TDP_CMP_F64  double(x) <op> lit_f
 *   TDP_CMP_F32  float(x)  <op> (float)lit_f  (lit_f holds an exact float32)
 *   TDP_CMP_NONE row never matches (absent dictionary literal, :74-76)
 *   TDP_CMP_ALL  row always matches (out-of-range int literal)
 *   TDP_CMP_DEC  double(x) / double(lit_i) <op> lit_f: a float64 column kept
 *                as scaled integers (x = value * lit_i exactly), compared
 *                after the same correctly rounded division that decodes it *   TDP_CMP_BITMAP  semi-join membership: x = int64(col) - lit_i, row
 *                   matches iff 0 <= x < (int64)lit_f and bit x is set in
 *                   the uint32-word bitmap passed as column `reserved`
 *                   (op ignored; built by tdp_join_dense_bitmap)
 */
enum tdp_cmp_type {
  TDP_CMP_I64 = 0,
  TDP_CMP_F64 = 1,
  TDP_CMP_F32 = 2,
  TDP_CMP_NONE = 3,
  TDP_CMP_ALL = 4,
  TDP_CMP_DEC = 5,
  TDP_CMP_BITMAP = 6
};

typedef struct tdp_predicate {
  int32_t column; /* index into the column array                        */
  int32_t op;     /* tdp_cmp_op                                         */
  int32_t cmp;    /* tdp_cmp_type                                       */
  int32_t reserved;
  int64_t lit_i;
  double lit_f;
} tdp_predicate;

/* ------------------------------------------------------------------------ */
/* library                                                                   */
/* ------------------------------------------------------------------------ */
const char* tdp_last_error(void);
const char* tdp_version(void);
/* Number of SMs of the current device (grid sizing); <0 on error. */
int tdp_device_sm_count(void);
/* Total kernels launched by this library in this process (benchmark
 * accounting of "our" launches). */
uint64_t tdp_launch_count(void);
/* Account `n` kernels of this library replayed inside a CUDA graph (a graph
 * captured from library launches relaunches them without calling in). */
void tdp_count_graph_launches(uint64_t n);
/* Replay bookkeeping without torch's stream objects (replay.py: a replayed
 * plan's host path is on the critical path of small queries):
 * stream_wait_event = cudaStreamWaitEvent; replay_done = count the replayed
 * graph's launches, then cudaEventRecord(event, stream).                   */
int tdp_stream_wait_event(void* stream, void* event);
int tdp_replay_done(void* event, void* stream, uint64_t graph_launches);
/* Read and clear the CUDA runtime error state of this library (after an
 * aborted graph capture); returns the cudaError_t that was pending.        */
int tdp_clear_error(void);
/* Replay guard (no reference counterpart: the reference re-plans every run).
 * Enqueue a check that the `n` (<= 16) integers at device `got` (element size
 * 4 or 8) equal `expected` (host array): a CUDA graph captured from a plan
 * sized by host reads of those integers traps on a mismatch instead of
 * overrunning buffers.                                                     */
/* Replay log of host decisions the library takes from device data (the
 * radix sort's skipped digit passes; thread-local).  mode 1 records them,
 * mode 2 (inside a CUDA-graph capture) replays `values` instead of
 * synchronising, each checked on the device; mode 0 is off.  end() copies a
 * recorded log to `out` (capacity `cap`, >= size()) and turns logging off. */
int tdp_replay_log_begin(int32_t mode, const int64_t* values, int64_t n);
int64_t tdp_replay_log_size(void);
int tdp_replay_log_end(int64_t* out, int64_t cap);
int tdp_expect_values(const void* got, int32_t esize, int32_t n, const int64_t* expected,
                      void* stream);
/* Benchmark timer: while enabled, CUDA events are recorded on the launch
 * stream immediately around every launch of the selected kernels (after all
 * host-side preparation): on = 1 the fused scan (tdp_scan_agg), on = 2 the
 * join probe passes (dense / hash / sorted count kernels), 0 off.  read()
 * waits for the recorded events, returns the summed milliseconds and the
 * launch count, and clears them.                                           */
int tdp_kernel_timer_enable(int32_t on);
int tdp_kernel_timer_read(double* total_ms, int64_t* launches);

/* ------------------------------------------------------------------------ */
/* filter / compaction / row movement                                        */
/* ------------------------------------------------------------------------ */

/* Conjunctive predicate mask, one byte per row (replaces the
 * `mask &= comparison_mask(...)` loop, tq/kernels.py:93-95).               */
int tdp_filter_mask(const tdp_column* cols, int32_t ncols, const tdp_predicate* preds,
                    int32_t npreds, int64_t n, uint8_t* out_mask, void* stream);

/* Workspace bytes for tdp_filter_select over n rows. */
size_t tdp_filter_workspace(int64_t n);

/* Fused predicate evaluation + order-preserving stream compaction: writes the
 * ascending indices of surviving rows and their count (device int64).
 * Replaces comparison_mask chain + np.nonzero (tq/kernels.py:87-96).       */
int tdp_filter_select(const tdp_column* cols, int32_t ncols, const tdp_predicate* preds,
                      int32_t npreds, int64_t n, int64_t* out_indices, int64_t* out_count,
                      void* ws, size_t ws_bytes, void* stream);

/* Row gather of several columns by one index vector in one launch:
 * dst[c][j, :] = src[c][idx[j], :].  Replaces take_rows (tq/kernels.py:44-51)
 * / gather forward (tq/tensor.py:597-607).                                 */
int tdp_gather_rows(const tdp_column* src, int32_t ncols, const int64_t* indices, int64_t m,
                    void* const* dst, void* stream);
/* The same with two index vectors of m rows in one launch: columns
 * [0, nfirst) are gathered at indices, the rest at indices2 -- both sides of
 * a join's output (probe rows, build rows) at once.                        */
int tdp_gather_rows2(const tdp_column* src, int32_t ncols, int32_t nfirst, const int64_t* indices,
                     const int64_t* indices2, int64_t m, void* const* dst, void* stream);

/* grad_in[idx[j], :] += grad_out[j, :] (float32/float64).  Replaces the
 * np.add.at VJP of gather (tq/tensor.py:609-612).  grad_in must be zeroed. */
int tdp_scatter_add_rows(const void* grad_out, int32_t dtype, int64_t width,
                         const int64_t* indices, int64_t m, void* grad_in, void* stream);

/* ------------------------------------------------------------------------ */
/* fused scan -> filter -> expression -> dense grouped aggregate              */
/* ------------------------------------------------------------------------ */
/* Expression program: SSA, instruction i defines value i.  Types follow the
 * numpy promotion the host layer resolved (tq/tensor.py:330-412 ops).       */
enum tdp_opcode {
  TDP_OP_LOAD = 0,   /* a = column index; value = column[row] as `dtype`   */
  TDP_OP_CONST = 1,  /* imm_i / imm_f                                       */
  TDP_OP_CAST = 2,   /* a -> dtype                                          */
  TDP_OP_ADD = 3,
  TDP_OP_SUB = 4,
  TDP_OP_MUL = 5,
  TDP_OP_DIV = 6,    /* float true divide                                   */
  TDP_OP_NEG = 7,
  TDP_OP_SQUARE = 8,
  TDP_OP_LOG = 9,
  TDP_OP_EXP = 10,
  TDP_OP_RELU = 11,
  TDP_OP_DECIMAL = 12 /* a (int64) / imm_f, correctly rounded without a
                       * divide: q = a*inv, q += fma(-q, imm_f, a)*inv with
                       * inv = bits(imm_i) = RN(1/imm_f); compact.py checks
                       * at ingestion that it equals the stored float64  */
};

typedef struct tdp_instr {
  int32_t op;    /* tdp_opcode                                             */
  int32_t dtype; /* result type: TDP_I64 / TDP_F64 / TDP_F32                */
  int32_t a;     /* operand value index (or column index for LOAD)          */
  int32_t b;     /* second operand value index                              */
  int64_t imm_i;
  double imm_f;
} tdp_instr;

/* Group key: program value `value` (int64) mapped to a dense digit
 * (v - lo) in [0, span).  slot = mixed radix over keys in GROUP BY order,
 * so ascending slot == ascending lexicographic key (np.unique order,
 * tq/kernels.py:128-136).                                                   */
typedef struct tdp_key {
  int32_t value;
  int32_t reserved;
  int64_t lo;
  int64_t span;
} tdp_key;

enum tdp_agg_kind { TDP_AGG_COUNT = 0, TDP_AGG_SUM_F64 = 1, TDP_AGG_SUM_I64 = 2 };
/* OR-ed into a SUM kind passed to a group-by *emit* call (hash / bitmap
 * group-by): that aggregate is emitted as the float64 mean
 * double(sum) / double(count) -- tq/kernels.py:160-161
 * `sums.astype(np.float64) / counts`, IEEE division -- instead of the sum.  */
#define TDP_AGG_AVG_BIT 0x100

typedef struct tdp_agg {
  int32_t kind;  /* tdp_agg_kind                                           */
  int32_t value; /* program value index (ignored for COUNT)                 */
} tdp_agg;

size_t tdp_scan_aggregate_workspace(int64_t n, int64_t slots, int32_t naggs);

/* One pass over n base rows: rows passing every predicate are grouped by the
 * keys and aggregated.  out_counts[slot] (int64) and out_sums[a][slot]
 * (8 bytes: double for SUM_F64, int64 for SUM_I64, count for COUNT) over all
 * prod(span) slots.  Replaces FilterOp -> TvfOp (elementwise UDF) ->
 * GroupAggExactOp / _global_aggregate (tq/compiler.py:146-215,
 * tq/kernels.py:108-167).  Specialised per program with NVRTC (sm_100a),
 * cached in-process.                                                        */
int tdp_scan_aggregate(const tdp_column* cols, int32_t ncols, int64_t n,
                       const tdp_predicate* preds, int32_t npreds, const tdp_instr* prog,
                       int32_t nprog, const tdp_key* keys, int32_t nkeys, const tdp_agg* aggs,
                       int32_t naggs, int64_t* out_counts, void* out_sums, void* ws,
                       size_t ws_bytes, void* stream);

/* tdp_scan_aggregate followed by tdp_groupby_finalize in one call: for
 * small group spaces the partial-row reduction and the finalisation run as
 * one single-CTA launch after the scan.  out_counts / out_sums receive the
 * raw per-slot results as in tdp_scan_aggregate; the finalisation outputs
 * are those of tdp_groupby_finalize (slots = prod(key spans)).             */
int tdp_scan_aggregate_grouped(const tdp_column* cols, int32_t ncols, int64_t n,
                               const tdp_predicate* preds, int32_t npreds, const tdp_instr* prog,
                               int32_t nprog, const tdp_key* keys, int32_t nkeys,
                               const tdp_agg* aggs, int32_t naggs, int64_t* out_counts,
                               void* out_sums, void* ws, size_t ws_bytes, uint64_t avg_mask,
                               int64_t* out_keys, int64_t* out_group_counts, void* out_aggs,
                               int64_t* out_groups, void* stream);

/* Same front half, but writes the selected rows' program values
 * (outputs[j] = value outs[j]) compacted in row order: the materialised
 * form of a lazily filtered, elementwise-UDF column.                       */
int tdp_scan_project(const tdp_column* cols, int32_t ncols, int64_t n,
                     const tdp_predicate* preds, int32_t npreds, const tdp_instr* prog,
                     int32_t nprog, const int32_t* outs, int32_t nouts, void* const* out_ptrs,
                     int64_t* out_count, void* ws, size_t ws_bytes, void* stream);

/* Diagnostic: emit (and, when `compile` != 0, NVRTC-compile for sm_100a) the
 * specialised pipeline source for a descriptor set without launching it.
 * Needs no GPU.  Returns the source length (>= 0) or an error code; the text
 * is copied (NUL-terminated, truncated to cap) into out_src when non-NULL.
 * For a projection pass keys/aggs are empty and outs lists the values.     */
int tdp_pipeline_codegen(const tdp_column* cols, int32_t ncols, int64_t n,
                         const tdp_predicate* preds, int32_t npreds, const tdp_instr* prog,
                         int32_t nprog, const tdp_key* keys, int32_t nkeys, const tdp_agg* aggs,
                         int32_t naggs, const int32_t* outs, int32_t nouts, int32_t compile,
                         char* out_src, size_t cap);

/* Compact occupied slots (count > 0) in ascending slot order: writes key
 * values (per key, int64), counts, and per aggregate either the sum or, when
 * avg_mask bit a is set, float64(sum)/count (tq/kernels.py:154-166).
 * out_groups receives the number of occupied groups (device int64).       */
int tdp_groupby_finalize(const int64_t* counts, const void* sums, int64_t slots,
                         const tdp_key* keys, int32_t nkeys, const tdp_agg* aggs, int32_t naggs,
                         uint64_t avg_mask, int64_t* out_keys, int64_t* out_counts,
                         void* out_aggs, int64_t* out_groups, void* stream);

/* Min / max of int64 key columns over rows passing the predicates
 * (dense-path planning for plain integer keys).  out_minmax[2*j] = min,
 * out_minmax[2*j+1] = max; empty selection leaves INT64_MAX / INT64_MIN. */
int tdp_scan_minmax(const tdp_column* cols, int32_t ncols, int64_t n,
                    const tdp_predicate* preds, int32_t npreds, const int32_t* key_cols,
                    int32_t nkeys, int64_t* out_minmax, void* stream);
/* tdp_scan_minmax plus, for one key and no predicates, out_runs (device
 * int64[2]): [0] = 1 if the key column is not non-decreasing, [1] = 1 if a
 * run of equal keys is longer than 32 rows -- both 0: the sorted-runs
 * group-by below applies.  Read with the range in one host read.           */
int tdp_scan_minmax_runs(const tdp_column* cols, int32_t ncols, int64_t n,
                         const tdp_predicate* preds, int32_t npreds, const int32_t* key_cols,
                         int32_t nkeys, int64_t* out_minmax, int64_t* out_runs, void* stream);
/* Sorted-runs group-by (groupby_exact, tq/kernels.py:108-167, for one int64
 * key that tdp_scan_minmax_runs found non-decreasing with runs <= 32 rows):
 * the groups are the runs.  prepare: out_ngroups (device) = m; emit (m from
 * the host): out_keys[m] ascending, out_counts[m], out_sums[naggs][m] as
 * tdp_groupby_hash_emit (TDP_AGG_AVG_BIT honoured); every sum adds its run's
 * rows in row order (np.add.at's order: float sums bit-identical).         */
size_t tdp_groupby_runs_workspace(int64_t n);
int tdp_groupby_runs_prepare(const int64_t* keys, int64_t n, int64_t* out_ngroups, void* ws,
                             size_t ws_bytes, void* stream);
int tdp_groupby_runs_emit(const int64_t* keys, int64_t n, const tdp_column* vals,
                          const int32_t* agg_kinds, int32_t naggs, int64_t m, int64_t* out_keys,
                          int64_t* out_counts, void* out_sums, void* ws, size_t ws_bytes,
                          void* stream);

/* ------------------------------------------------------------------------ */
/* sort-based group-by (general integer keys)                                */
/* ------------------------------------------------------------------------ */
size_t tdp_sort_workspace(int64_t n);

/* Stable argsort with numpy semantics (tq/kernels.py:256-264):
 * descending = stable ascending sort of the negated key (ties keep input
 * order; -INT64_MIN wraps), NaN last in both directions, -0.0 == 0.0.
 * key: TDP_I64 / TDP_F64 / TDP_F32 / TDP_I32 scalar column.               */
int tdp_sort_order(const tdp_column* key, int32_t descending, int64_t n, int64_t* out_order,
                   void* ws, size_t ws_bytes, void* stream);
/* The first k entries of tdp_sort_order's stable order (ORDER BY ... LIMIT k,
 * tq/kernels.py:267-273 sort_limit), 1 <= k <= 1024, without sorting all n:
 * per-CTA bitonic sorts of 2048 (key image, row) pairs keep their k smallest,
 * repeated on the survivors.  Writes min(k, n) row indices.                */
size_t tdp_topk_workspace(int64_t n, int64_t k);
int tdp_topk_order(const tdp_column* key, int32_t descending, int64_t n, int64_t k,
                   int64_t* out_order, void* ws, size_t ws_bytes, void* stream);

/* np.unique(key, return_inverse=True) for an int64 column
 * (tq/kernels.py:128): out_uniques[0:u) ascending, out_inverse[i] = rank of
 * key[i], out_nunique = u (device).                                        */
int tdp_unique_inverse(const int64_t* key, int64_t n, int64_t* out_uniques,
                       int64_t* out_inverse, int64_t* out_nunique, void* ws, size_t ws_bytes,
                       void* stream);

/* Grouped aggregation over dense codes in [0, slots): counts (int64) and per
 * aggregate 8-byte sums in the value column's accumulator type (float64 for
 * float input, int64 wrap-around for int input; np.bincount / np.add.at,
 * tq/kernels.py:138-153).  vals[a] may be NULL for COUNT.  Float sums are
 * accumulated in 256-bit fixed point (order-independent, bitwise repeatable)
 * in the caller's workspace of tdp_groupby_codes_workspace(slots, naggs)
 * bytes.                                                                    */
size_t tdp_groupby_codes_workspace(int64_t slots, int32_t naggs);
int tdp_groupby_codes(const int64_t* codes, int64_t n, int64_t slots, const tdp_column* vals,
                      const int32_t* agg_kinds, int32_t naggs, int64_t* out_counts,
                      void* out_sums, void* ws, size_t ws_bytes, void* stream);

/* Hash group-by over one int64 key (groupby_exact general path, tq/kernels.py
 * :108-167, for key ranges too wide for dense slots).  prepare: one pass
 * hashes every key into an open-addressing table and accumulates counts and
 * sums with warp-combined global atomics, then compacts the occupied slots;
 * out_ngroups (device int64) = distinct keys m.  emit (same workspace, m from
 * the host): stable radix sort of the m distinct keys, then out_keys[m],
 * out_counts[m] and out_sums[naggs][m] in ascending key order (8-byte values
 * as tdp_groupby_codes: double / int64 sums, the count for COUNT).        */
size_t tdp_groupby_hash_workspace(int64_t n, int32_t naggs);
int tdp_groupby_hash_prepare(const int64_t* keys, int64_t n, const tdp_column* vals,
                             const int32_t* agg_kinds, int32_t naggs, int64_t* out_ngroups,
                             void* ws, size_t ws_bytes, void* stream);
int tdp_groupby_hash_emit(int64_t n, const int32_t* agg_kinds, int32_t naggs, int64_t m,
                          int64_t* out_keys, int64_t* out_counts, void* out_sums, void* ws,
                          size_t ws_bytes, void* stream);
/* prepare_ex: prepare, plus the distinct keys' range: out_info (device
 * int64[3]) = {m, min key image, max key image} (images: key ^ INT64_MIN,
 * order-preserving).  emit_ranked: emit with the keys ordered by a bitmap
 * over [min_key, min_key + key_range) (ranks by popcount prefix) instead of
 * a radix sort -- for ranges up to a few dozen bits per distinct key; its
 * extra workspace is tdp_groupby_hash_rank_workspace(key_range).          */
int tdp_groupby_hash_prepare_ex(const int64_t* keys, int64_t n, const tdp_column* vals,
                                const int32_t* agg_kinds, int32_t naggs, int64_t* out_info,
                                void* ws, size_t ws_bytes, void* stream);
size_t tdp_groupby_hash_rank_workspace(int64_t key_range);
int tdp_groupby_hash_emit_ranked(int64_t n, const int32_t* agg_kinds, int32_t naggs, int64_t m,
                                 int64_t min_key, int64_t key_range, int64_t* out_keys,
                                 int64_t* out_counts, void* out_sums, void* ws, size_t ws_bytes,
                                 void* rank_ws, size_t rank_ws_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* equi-join (builder-defined; the reference has none)       */
/* ------------------------------------------------------------------------ */
size_t tdp_join_workspace(int64_t n_build, int64_t n_probe);

/* Inner equi-join on int64 keys, two calls sharing one workspace.
 * prepare: stable radix sort of the build keys, open-addressing hash table
 * over the distinct build keys (key -> run in sorted order), one hash probe
 * per probe row, per-tile match counts and their scan; writes the number of
 * result pairs to out_count (device int64).  emit: re-probes and writes the
 * pairs, ordered by probe row and, within a probe row, by ascending build row.
 * The workspace must not be touched between the two calls.                */
int tdp_join_prepare(const int64_t* build_keys, int64_t n_build, const int64_t* probe_keys,
                     int64_t n_probe, int64_t* out_count, void* ws, size_t ws_bytes,
                     void* stream);
/* Same as tdp_join_prepare for a filtered probe relation: probe row i of the
 * base key column takes part iff every predicate holds on the base columns
 * (tdp_filter_select semantics), evaluated inside the probe pass; the probe
 * indices tdp_join_emit then writes are base row ids.  Replaces filter_exact
 * (tq/kernels.py:87-97) + take_rows of the key column ahead of a join.     */
int tdp_join_prepare_filtered(const int64_t* build_keys, int64_t n_build,
                              const int64_t* probe_keys, int64_t n_probe,
                              const tdp_column* cols, int32_t ncols, const tdp_predicate* preds,
                              int32_t npreds, int64_t* out_count, void* ws, size_t ws_bytes,
                              void* stream);
/* Synchronisation-free two-phase prepare, both sides optionally filtered.
 * mode 0 (optimistic): the (filtered) build rows are hashed in input order
 *   as unique keys -- the primary-key side of a PK-FK join, no sort;
 *   out_info[0] = result pairs, out_info[1] != 0 when a build key repeats, in
 *   which case out_info[0] is invalid and the call must be repeated with
 *   mode 1.  Build rows failing the build predicates do not take part; the
 *   build indices tdp_join_emit writes are then base row ids.
 * mode 1 (runs): stable sort of the build keys, one entry per run of equal
 *   keys (build predicates not allowed: compact the build side first).
 * Probe predicates as in tdp_join_prepare_filtered.  out_info: device int64[2]. */
int tdp_join_prepare_ex(const int64_t* build_keys, int64_t n_build, const tdp_column* bcols,
                        int32_t nbcols, const tdp_predicate* bpreds, int32_t nbpreds,
                        const int64_t* probe_keys, int64_t n_probe, const tdp_column* pcols,
                        int32_t npcols, const tdp_predicate* ppreds, int32_t nppreds,
                        int32_t mode, int64_t* out_info, void* ws, size_t ws_bytes,
                        void* stream);
int tdp_join_emit(const int64_t* probe_keys, int64_t n_build, int64_t n_probe,
                  int64_t* out_probe_idx, int64_t* out_build_idx, void* ws, size_t ws_bytes,
                  void* stream);

/* Differentiable ORDER BY [LIMIT k] of trainable queries (
 * the reference rejects Sort/Limit when trainable, tq/compiler.py:464-475):
 * NeuralSort rows P[k][n] of float64 scores s (descending), temperature tau
 *   P[r, i] = softmax_i(((n + 1 - 2 (r + 1)) s_i - sum_j |s_i - s_j|) / tau).
 * fwd workspace: n doubles.  bwd: dP (overwritten with the softmax VJP),
 * out_ds = dL/ds; workspace 2 n doubles.                                    */
int tdp_softsort_fwd(const double* s, int64_t n, int32_t k, double tau, double* out_P,
                     double* ws, void* stream);
int tdp_softsort_bwd(const double* s, int64_t n, int32_t k, double tau, const double* P,
                     double* dP_inout, double* out_ds, double* ws, void* stream);

/* Device dictionary encoding (tq/encodings.py:127-133 dict_encode): a
 * 64-bit hash per string of a UTF-8 byte buffer (offsets int64 [n + 1]);
 * after tdp_unique_inverse of the hashes, tdp_string_groups writes each hash
 * group's first string (out_first int64 [m]) and sets *out_flag when a
 * string differs byte-wise from its group's first one (a hash collision: the
 * caller encodes on the host instead).  Codes = the groups' sorted ranks,
 * gathered by the inverse.                                                  */
int tdp_string_hash(const uint8_t* bytes, const int64_t* offsets, int64_t n, int64_t* out_hash,
                    void* stream);
int tdp_string_groups(const uint8_t* bytes, const int64_t* offsets, int64_t n,
                      const int64_t* inverse, int64_t m, int64_t* out_first, int32_t* out_flag,
                      void* stream);

/* Device CSV ingestion (tq/storage.py:190-249 read_csv /
 * register_csv: excel-dialect csv.reader + int() / float() / dict_encode).
 * The file's UTF-8 bytes (ending in a record terminator) are tokenised on
 * the device.  tdp_csv_index: out_counts[0] = fields, [1] = records (header
 * included), [2] = quote characters (device int64; odd = an unterminated
 * quoted field).  tdp_csv_fields: the byte position of every field end
 * (int64 [fields]) and each record's last field index (int64 [records]);
 * out_flags[0] != 0 reports what the device path does not model (a quote
 * inside an unquoted field or after a closing quote, an empty line,
 * malformed UTF-8), out_flags[1] the first record whose field count is not
 * ncols (INT32_MAX if none) -- the caller then uses the host reader, which
 * raises the reference's errors.  tdp_csv_parse_column: data rows' cells of
 * column col as int64 (kind 0, Python int()) or float64 (kind 1, Python
 * float(), exact on the device only on Clinger's fast path); out_status per
 * row: 0 ok, 1 the host converts this cell, 2 invalid.
 * tdp_csv_string_column: with out_bytes NULL the unescaped cell offsets
 * (int64 [nrows + 1], total last), then the bytes themselves -- the input of
 * tdp_string_hash / tdp_string_groups (dict_encode).                       */
size_t tdp_csv_workspace(int64_t nbytes);
size_t tdp_csv_string_workspace(int64_t nrows);
int tdp_csv_index(const uint8_t* bytes, int64_t nbytes, int64_t* out_counts, void* ws,
                  size_t ws_bytes, void* stream);
int tdp_csv_fields(const uint8_t* bytes, int64_t nbytes, int32_t ncols, int64_t nrecords,
                   int64_t* out_field_ends, int64_t* out_record_ends, int32_t* out_flags,
                   void* ws, size_t ws_bytes, void* stream);
int tdp_csv_parse_column(const uint8_t* bytes, const int64_t* field_ends, int32_t ncols,
                         int32_t col, int64_t nrows, int32_t kind, void* out_values,
                         uint8_t* out_status, void* stream);
int tdp_csv_string_column(const uint8_t* bytes, const int64_t* field_ends, int32_t ncols,
                          int32_t col, int64_t nrows, int64_t* out_offsets, uint8_t* out_bytes,
                          void* ws, size_t ws_bytes, void* stream);

/* Bitmap group-by over one int64 key whose values lie in [lo, lo+key_range)
 * (the scan's min/max), the range at most ~1024 values per row: the rank of
 * a key among the set bits of a key_range-bit map is its group id in
 * ascending key order, so rows accumulate straight into dense cells (float
 * SUMs in fixed point: bitwise repeatable).  prepare: out_ngroups (device) =
 * distinct keys m; emit (m from the host): out_keys[m] ascending,
 * out_counts[m], out_sums[naggs][m] as tdp_groupby_hash_emit.  Same contract
 * as the hash group-by (groupby_exact, tq/kernels.py:108-167).  From 2^22
 * rows on (and <= 4096 partitions of groups) the rows are first scattered
 * into partitions whose cells fit shared memory and aggregated there (every
 * row added exactly; repeatable bit for bit); the workspace then also holds
 * the partitioned rows
 * (2 + 4 + 8 x naggs bytes per row).  TDP_GROUPBY_PARTITION=0 disables it. */
size_t tdp_groupby_bitmap_workspace(int64_t n, int64_t key_range, int32_t naggs);
int tdp_groupby_bitmap_prepare(const int64_t* keys, int64_t n, int64_t lo, int64_t key_range,
                               const tdp_column* vals, const int32_t* agg_kinds, int32_t naggs,
                               int64_t* out_ngroups, void* ws, size_t ws_bytes, void* stream);
int tdp_groupby_bitmap_emit(int64_t n, int64_t lo, int64_t key_range, const int32_t* agg_kinds,
                            int32_t naggs, int64_t m, int64_t* out_keys, int64_t* out_counts,
                            void* out_sums, void* ws, size_t ws_bytes, void* stream);

/* Dense-range equi-join: the same contract as tdp_join_prepare_ex (mode 0) /
 * tdp_join_emit when every build key lies in [lo, lo + key_range) (a column
 * statistic) and the keys are unique: a bitmap of key_range bits replaces the
 * hash table and Bloom filter (one bit test per probe row, exact), build rows
 * are found by the key's rank among the set bits.  out_info[1] != 0 reports a
 * repeated build key or a key outside the range (the pair count is then not
 * valid: use the hash join).  need_rows = 0 skips the build-row index (a
 * semi-join: out_build_idx is not written).  Replaces the same
 * filter_exact -> take_rows -> join composition.           */
size_t tdp_join_dense_workspace(int64_t key_range, int64_t n_build, int64_t n_probe);
int tdp_join_dense_prepare(const int64_t* build_keys, int64_t n_build, const tdp_column* bcols,
                           int32_t nbcols, const tdp_predicate* bpreds, int32_t nbpreds,
                           const int64_t* probe_keys, int64_t n_probe, const tdp_column* pcols,
                           int32_t npcols, const tdp_predicate* ppreds, int32_t nppreds,
                           int64_t lo, int64_t key_range, int32_t need_rows, int64_t* out_info,
                           void* ws, size_t ws_bytes, void* stream);
/* Semi-join bitmap: bit (key - lo) of out_bits (ceil(key_range/32) uint32
 * words, cleared here) for every build row passing the build predicates;
 * out_flags[0] = a key repeats, [1] = a key outside [lo, lo + key_range)
 * (int32 each).  The bitmap is the operand of a TDP_CMP_BITMAP predicate:
 * a probe relation filtered by it is the left semi-join (inner join whose
 * right side contributes no columns, unique right keys) without pairs.      */
int tdp_join_dense_bitmap(const int64_t* build_keys, int64_t n_build, const tdp_column* bcols,
                          int32_t nbcols, const tdp_predicate* bpreds, int32_t nbpreds, int64_t lo,
                          int64_t key_range, uint32_t* out_bits, int32_t* out_flags, void* stream);
int tdp_join_dense_emit(const int64_t* probe_keys, int64_t n_build, int64_t n_probe, int64_t lo,
                        int64_t key_range, int32_t need_rows, int64_t* out_probe_idx,
                        int64_t* out_build_idx, void* ws, size_t ws_bytes, void* stream);

/* Sort / searchsorted equi-join (north_star's "radix sort + searchsorted
 * probing"): stable LSD radix sort of the build key images
 * with their row ids, then each probe row passing the probe predicates
 * searches the sorted keys (a <= 4096-fence top level in shared memory, then
 * the fence interval in global memory).  Same result contract as
 * tdp_join_prepare_ex / tdp_join_emit: *out_count (device int64) pairs,
 * ordered by probe row then ascending build row; any keys (repeats on both
 * sides, INT64 extremes).  The planner prefers the dense-range / hash joins
 * (one lookup per probe row, measured faster: DESIGN.md §3.3); this form is
 * selected with TDP_JOIN_ALGO=sort / kernels.JOIN_ALGORITHM.                */
size_t tdp_join_sorted_workspace(int64_t n_build, int64_t n_probe);
int tdp_join_sorted_prepare(const int64_t* build_keys, int64_t n_build, const int64_t* probe_keys,
                            int64_t n_probe, const tdp_column* pcols, int32_t npcols,
                            const tdp_predicate* ppreds, int32_t nppreds, int64_t* out_count,
                            void* ws, size_t ws_bytes, void* stream);
int tdp_join_sorted_emit(const int64_t* probe_keys, int64_t n_build, int64_t n_probe,
                         int64_t* out_probe_idx, int64_t* out_build_idx, void* ws,
                         size_t ws_bytes, void* stream);

/* One-pass LLP step (tq/kernels.py:190-229 soft_groupby over
 * pe_encode(Linear(X)), its tape backward tq/tensor.py:474, :364-365,
 * :515-527): for k = 2 classes and one one-hot bag key, the forward writes
 * the count grid AND the per-bag statistics stats[b] = (Q_b, S_b[0..d)) with
 * Q_b = sum P0 P1, S_b = sum P0 P1 x over the bag's rows; the backward forms
 * dW = sum_b (G[b,0] - G[b,1]) S_b [1, -1], db likewise from Q_b, without
 * reading X.  Rows are visited in bag order through perm (int32 stable
 * permutation) and offs (int64 [bags + 1] bag offsets).  float32 X, d = 32
 * or 64; grid cell of (bag b, class c) = b * bag_stride + c * dense_stride. */
size_t tdp_llp_onepass_workspace(int32_t bags, int32_t d);
int tdp_llp_onepass_fwd(const float* X, int64_t n, int32_t d, const float* W, const float* bias,
                        const int32_t* perm, const int64_t* offs, int32_t bags, int64_t bag_stride,
                        int64_t dense_stride, double* out_grid, double* out_stats, void* ws,
                        size_t ws_bytes, void* stream);
int tdp_llp_onepass_bwd(const double* stats, int32_t bags, int32_t d, const double* grad_grid,
                        int64_t bag_stride, int64_t dense_stride, float* dW, float* db,
                        void* stream);

/* ------------------------------------------------------------------------ */
/* probability encodings and soft (differentiable) group-by                 */
/* ------------------------------------------------------------------------ */

/* Row softmax with max subtraction (tq/tensor.py:515-521 via pe_encode,
 * tq/encodings.py:143-151).  float32 / float64, [n, k].                    */
int tdp_softmax_fwd(const void* logits, int32_t dtype, int64_t n, int64_t k, void* probs,
                    void* stream);
/* VJP: grad_logits = P * (g - sum(g * P)) (tq/tensor.py:523-525).          */
int tdp_softmax_bwd(const void* probs, const void* grad_probs, int32_t dtype, int64_t n,
                    int64_t k, void* grad_logits, void* stream);

/* PE invariant check (tq/encodings.py:101-107): out_flags[0] |= 1 when an
 * entry is outside [-tol, 1+tol], |= 2 when a row sum differs from 1 by
 * more than tol.  out_flags is a device int32 the caller zeroes.           */
int tdp_pe_validate(const void* probs, int32_t dtype, int64_t n, int64_t k, double tol,
                    int32_t* out_flags, void* stream);

/* Row argmax, first maximum wins (np.argmax, tq/encodings.py:161).         */
int tdp_pe_argmax(const void* probs, int32_t dtype, int64_t n, int64_t k, int64_t* out_codes,
                  void* stream);

/* Range check of int64 codes: out_flags |= 1 if any code < 0 or >= k
 * (tq/encodings.py:180-181, tq/kernels.py:244-245).                        */
int tdp_codes_check(const int64_t* codes, int64_t n, int64_t k, int32_t* out_flags,
                    void* stream);

/* A soft group-by key: a dense PE matrix [n, k] (float32/float64) or a
 * compact one-hot column given as int64 codes (one_hot_pe,
 * tq/encodings.py:175-183, never materialised).                            */
enum tdp_soft_kind { TDP_SOFT_DENSE = 0, TDP_SOFT_ONEHOT = 1 };
typedef struct tdp_soft_key {
  const void* data;
  int32_t kind;
  int32_t dtype; /* of dense probabilities                                  */
  int64_t k;
} tdp_soft_key;

/* grid[c1..cm] = sum_i w_i * prod_j P_j[i, c_j]   (w_i = 1 when values is
 * NULL), accumulated in float64, row-major over the keys
 * (tq/kernels.py:190-229 _joint_probabilities + reduce_sum).               */
int tdp_soft_groupby_fwd(const tdp_soft_key* keys, int32_t nkeys, int64_t n, const void* values,
                         int32_t values_dtype, double* out_grid, void* stream);

/* VJP of the above for upstream grid gradient G (float64, prod k):
 *   dP_j[i, c] = sum_{cells with c_j = c} G[cell] * w_i * prod_{l != j} P_l[i, c_l]
 *   dw_i       = sum_cells G[cell] * prod_l P_l[i, c_l]
 * grad_keys[j] is NULL for one-hot keys or keys needing no gradient;
 * grad_values may be NULL.  Outputs are written (not accumulated) in the
 * key / value dtype (tq/tensor.py:364-365, :474, :544 VJP chain).         */
int tdp_soft_groupby_bwd(const tdp_soft_key* keys, int32_t nkeys, int64_t n, const void* values,
                         int32_t values_dtype, const double* grad_grid, void* const* grad_keys,
                         void* grad_values, void* stream);

/* ------------------------------------------------------------------------ */
/* skinny dense layers of models embedded in trainable queries              */
/* ------------------------------------------------------------------------ */
/* Y[n,k] = X[n,d] W[d,k] (+ bias[k]); 1 <= d <= 256, 1 <= k <= 8, float32 /
 * float64, float64 accumulation.  Replaces matmul (tq/tensor.py:437-447) for
 * the tall-skinny products of Linear (tq/models.py:26-27).                 */
int tdp_linear_fwd(const void* X, int32_t dtype, int64_t n, int32_t d, int32_t k, const void* W,
                   const void* bias, void* Y, void* stream);
size_t tdp_linear_wgrad_workspace(int64_t n, int32_t d, int32_t k);
/* dW = X^T G, db = column sums of G (db may be NULL): the matmul VJP w.r.t.
 * the weight (tq/tensor.py:452) and of the bias add (:337-338).          */
int tdp_linear_wgrad(const void* X, const void* G, int32_t dtype, int64_t n, int32_t d, int32_t k,
                     void* dW, void* db, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* fused soft count over a linear classifier head (the LLP query)           */
/* ------------------------------------------------------------------------ */
/* Soft group-by COUNT (tdp_soft_groupby_fwd) whose key `dense_key` is the PE
 * column P = softmax(X W + bias), X [n, d], W [d, k], computed on the fly:
 * replaces Linear.__call__ (tq/models.py:26-27) -> pe_encode
 * (tq/encodings.py:143-151) -> soft_groupby count (tq/kernels.py:190-229)
 * for one pass over X.  All other keys are one-hot code columns.
 * keys[dense_key].data is ignored; keys[dense_key].k must equal k.
 * Supported shapes: tdp_soft_linear_supported() (d = 32 or 64 float32,
 * d = 32 float64, X 16-byte aligned, n >= 1024, k <= 8, <= 8192 cells);
 * otherwise TDP_ENOTSUP and the caller composes the unfused kernels.       */
int tdp_soft_linear_supported(int32_t dtype, int64_t n, int32_t d, int32_t k, int64_t cells,
                              const void* X);
int tdp_soft_linear_count_fwd(const void* X, int32_t dtype, int64_t n, int32_t d, int32_t k,
                              const void* W, const void* bias, const tdp_soft_key* keys,
                              int32_t nkeys, int32_t dense_key, double* out_grid, void* stream);
/* The exact swap of the same query (CompiledQuery.swap_to_exact inserts
 * pe_decode, tq/compiler.py:125-136, :378-381): exact COUNT grouped by the
 * one-hot codes and argmax(softmax(X W + bias)) (tq/encodings.py:154-165:
 * first maximum, NaN wins) in one pass over X; out_counts is the dense
 * int64 count grid over the cells (row-major in key order).              */
int tdp_linear_argmax_count(const void* X, int32_t dtype, int64_t n, int32_t d, int32_t k,
                            const void* W, const void* bias, const tdp_soft_key* keys,
                            int32_t nkeys, int32_t dense_key, int64_t* out_counts, void* stream);
size_t tdp_soft_linear_count_bwd_workspace(int64_t n, int32_t d, int32_t k);
/* VJP of the above w.r.t. W and bias for the upstream grid gradient G
 * (float64): the softmax VJP (tq/tensor.py:515-527) of dP[i,c] = G[cell(i,c)]
 * followed by the matmul / bias-add VJPs (tq/tensor.py:452, :337-338), with
 * P recomputed from X.  dW [d, k], db [k] (may be NULL) in X's dtype.      */
int tdp_soft_linear_count_bwd(const void* X, int32_t dtype, int64_t n, int32_t d, int32_t k,
                              const void* W, const void* bias, const tdp_soft_key* keys,
                              int32_t nkeys, int32_t dense_key, const double* grad_grid, void* dW,
                              void* db, void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TDP_KERNELS_H */
