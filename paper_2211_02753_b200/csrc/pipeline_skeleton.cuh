// Kernel skeleton of the fused scan -> filter -> expression -> aggregate
// pipeline.  This text is compiled at run time by NVRTC for sm_100a after the
// query-specific part (TdpRow, tdp_load / tdp_load_smem / tdp_issue_tile,
// tdp_eval, tdp_project), emitted by pipeline.cu from the tdp_instr program, is
// prepended.  It is embedded in libtdp_kernels.so as a string.
//
// tdp_scan_agg (main path): bulk-async-copy pipeline.
//   * one producer warp streams every column of a tile of TDP_PTILE rows from
//     HBM into a TDP_STAGES-deep shared-memory ring with
//     cp.async.bulk.shared::cluster.global (the TMA engine), completion
//     tracked by mbarrier transaction counts;
//   * TDP_CONS_WARPS consumer warps evaluate predicates, the expression program
//     and the slot of each row from shared memory and accumulate;
//   * loads in flight no longer occupy registers, so the depth of the memory
//     pipeline (TDP_STAGES x stage bytes per SM) is independent of the
//     accumulator footprint.
//   Full tiles go through the ring; the < TDP_PTILE-row tail is read directly.
// tdp_scan_agg_ldg: register-staged 8-byte loads (columns not 16-byte aligned,
//   or too few rows to fill the ring).
//
// Accumulation:
//   TDP_REGACC=1  slots*(1+NF+NI) <= 64: each thread keeps every group's
//                 accumulators in registers (predicated adds, no atomics); the
//                 CTA reduces in a fixed order and writes one partial row; the
//                 host-side reduction over CTAs is fixed-order too, so results
//                 are bitwise deterministic run to run.
//   TDP_REGACC=0  atomics straight into zeroed global accumulators.

#define TDP_NFA (TDP_NF > 0 ? TDP_NF : 1)
#define TDP_NIA (TDP_NI > 0 ? TDP_NI : 1)

template <class T>
__device__ __forceinline__ T tdp_warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// TDP_ACCMODE 0: registers, 1: per-thread columns in shared memory, 2: global atomics
#define TDP_REGACC (TDP_ACCMODE == 0)
#define TDP_SMEMACC (TDP_ACCMODE == 1)
// TDP_CELLS, TDP_ACC_THREADS (shared-memory accumulator columns, one per
// thread) are defined by the generated prefix

struct TdpAcc {
#if TDP_REGACC
  i64 cnt[TDP_G];
  double af[TDP_G][TDP_NFA];
  i64 ai[TDP_G][TDP_NIA];
#endif
#if TDP_SMEMACC
  // cell-major columns: a thread touches only its own column, so updates need
  // no atomics and consecutive threads hit consecutive words (conflict-free).
  // Layout and per-row updates are generated (tdp_smem_add / tdp_smem_flush):
  // the row count and bounded integer sums share packed 64-bit words.
  u64* sm;
  u64* mine;  // sm + this thread's column
  int col;
#endif
  __device__ __forceinline__ void zero(u64* smem_acc) {
#if TDP_REGACC
#pragma unroll
    for (int s = 0; s < TDP_G; ++s) {
      cnt[s] = 0;
#pragma unroll
      for (int a = 0; a < TDP_NFA; ++a) af[s][a] = 0.0;
#pragma unroll
      for (int a = 0; a < TDP_NIA; ++a) ai[s][a] = 0;
    }
#endif
#if TDP_SMEMACC
    sm = smem_acc;
    col = threadIdx.x;
    mine = sm + col;
    if (col < TDP_ACC_THREADS)
      for (int c = 0; c < TDP_SM_ROWS; ++c) sm[c * TDP_ACC_THREADS + col] = 0;
#endif
  }
  __device__ __forceinline__ void add(const TdpParams& P, bool keep, int slot, const double* f,
                                      const i64* q) {
#if TDP_REGACC
#pragma unroll
    for (int s = 0; s < TDP_G; ++s) {
      const bool hit = keep && (slot == s);
      cnt[s] += hit ? 1 : 0;
#pragma unroll
      for (int a = 0; a < TDP_NF; ++a) af[s][a] += hit ? f[a] : 0.0;
#pragma unroll
      for (int a = 0; a < TDP_NI; ++a) ai[s][a] = (i64)((u64)ai[s][a] + (hit ? (u64)q[a] : 0ull));
    }
#elif TDP_SMEMACC
    tdp_smem_add(mine, keep ? slot : TDP_G, f, q, P);  // branch-free: rejects -> slot G
#else
    if (keep) {
      atomicAdd(reinterpret_cast<u64*>(P.acc) + slot, 1ull);
#pragma unroll
      for (int a = 0; a < TDP_NF; ++a)
        atomicAdd(reinterpret_cast<double*>(P.acc) + (i64)TDP_G * (1 + a) + slot, f[a]);
#pragma unroll
      for (int a = 0; a < TDP_NI; ++a)
        atomicAdd(reinterpret_cast<u64*>(P.acc) + (i64)TDP_G * (1 + TDP_NF + a) + slot, (u64)q[a]);
    }
#endif
  }
  __device__ __forceinline__ void row(const TdpParams& P, const TdpRow& r, bool valid) {
    int slot = 0;
    double f[TDP_NFA];
    i64 q[TDP_NIA];
    const bool keep = tdp_eval(r, P, slot, f, q) && valid;
    add(P, keep, slot, f, q);
  }
  // CTA reduction in a fixed order (warp shuffle tree, then warps in order)
  // and one partial row per CTA.  Every thread of the CTA must call it.
  template <int NWARPS>
  __device__ __forceinline__ void flush(const TdpParams& P) {
#if TDP_REGACC
    __shared__ u64 red[NWARPS][TDP_CELLS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int s = 0; s < TDP_G; ++s) {
      const i64 c = tdp_warp_sum(cnt[s]);
      if (lane == 0) red[warp][s] = (u64)c;
#pragma unroll
      for (int a = 0; a < TDP_NF; ++a) {
        const double v = tdp_warp_sum(af[s][a]);
        if (lane == 0) red[warp][TDP_G * (1 + a) + s] = (u64)__double_as_longlong(v);
      }
#pragma unroll
      for (int a = 0; a < TDP_NI; ++a) {
        const u64 v = tdp_warp_sum((u64)ai[s][a]);
        if (lane == 0) red[warp][TDP_G * (1 + TDP_NF + a) + s] = v;
      }
    }
    __syncthreads();
    // partial rows are stored cell-major (acc[cell * gridDim.x + cta]) so the
    // reduction over CTAs reads each cell contiguously
    u64* out = reinterpret_cast<u64*>(P.acc) + blockIdx.x;
    for (int c = threadIdx.x; c < TDP_CELLS; c += blockDim.x) {
      if (c >= TDP_G && c < TDP_G * (1 + TDP_NF)) {
        double v = 0.0;
        for (int w = 0; w < NWARPS; ++w) v += __longlong_as_double((i64)red[w][c]);
        out[(i64)c * gridDim.x] = (u64)__double_as_longlong(v);
      } else {
        u64 v = 0;
        for (int w = 0; w < NWARPS; ++w) v += red[w][c];
        out[(i64)c * gridDim.x] = v;
      }
    }
#elif TDP_SMEMACC
    __syncthreads();
    tdp_smem_flush(sm, P);
#endif
  }
};

#if TDP_SMEMACC
#define TDP_ACC_SMEM_BYTES (TDP_SM_ROWS * TDP_ACC_THREADS * 8)
#else
#define TDP_ACC_SMEM_BYTES 0
#endif

// ---------------------------------------------------------------------------
// register-staged path
// ---------------------------------------------------------------------------
extern "C" __global__ void __launch_bounds__(TDP_THREADS)
    tdp_scan_agg_ldg(const __grid_constant__ TdpParams P) {
  extern __shared__ __align__(128) unsigned char tdp_dyn[];
  const i64 tile = (i64)TDP_THREADS * TDP_U;
  const i64 step = (i64)gridDim.x * tile;
  TdpAcc acc;
  acc.zero(reinterpret_cast<u64*>(tdp_dyn));
  for (i64 base = (i64)blockIdx.x * tile; base < P.n; base += step) {
    TdpRow r[TDP_U];
#pragma unroll
    for (int u = 0; u < TDP_U; ++u) {
      const i64 i = base + (i64)u * TDP_THREADS + threadIdx.x;
      if (i < P.n) tdp_load(r[u], P, i);
      else tdp_zero(r[u]);
    }
#pragma unroll
    for (int u = 0; u < TDP_U; ++u)
      acc.row(P, r[u], base + (i64)u * TDP_THREADS + threadIdx.x < P.n);
  }
  acc.flush<TDP_THREADS / 32>(P);
}

// ---------------------------------------------------------------------------
// bulk-copy pipeline path
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned tdp_smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void tdp_mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void tdp_mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tdp_mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tdp_mbar_wait(unsigned bar, unsigned parity) {
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
// global -> shared bulk copy on the TMA engine, completion counted on `bar`
__device__ __forceinline__ void tdp_bulk_load(unsigned dst, const void* src, unsigned bytes,
                                              unsigned bar, u64 policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}

#define TDP_PTHREADS ((TDP_CONS_WARPS + 1) * 32)

extern "C" __global__ void __launch_bounds__(TDP_PTHREADS)
    tdp_scan_agg(const __grid_constant__ TdpParams P) {
  extern __shared__ __align__(128) unsigned char tdp_ring[];
  __shared__ __align__(8) u64 full_bar[TDP_STAGES];
  __shared__ __align__(8) u64 empty_bar[TDP_STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 ntiles = P.n / TDP_PTILE;
  if (threadIdx.x == 0) {
    for (int s = 0; s < TDP_STAGES; ++s) {
      tdp_mbar_init(tdp_smem_addr(&full_bar[s]), 1);
      tdp_mbar_init(tdp_smem_addr(&empty_bar[s]), TDP_CONS_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  TdpAcc acc;
  acc.zero(reinterpret_cast<u64*>(tdp_ring + (size_t)TDP_STAGES * TDP_STAGE_BYTES));
  if (warp == TDP_CONS_WARPS) {
    // ---- producer: one elected lane streams tiles into the ring ----------
    if (lane == 0) {
      u64 policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      int s = 0;
      unsigned eph = 0;
      for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
        tdp_mbar_wait(tdp_smem_addr(&empty_bar[s]), eph ^ 1u);
        const unsigned bar = tdp_smem_addr(&full_bar[s]);
        tdp_mbar_expect_tx(bar, TDP_STAGE_BYTES);
        tdp_issue_tile(P, tdp_smem_addr(tdp_ring + (size_t)s * TDP_STAGE_BYTES),
                       t * (i64)TDP_PTILE, bar, policy);
        if (++s == TDP_STAGES) {
          s = 0;
          eph ^= 1u;
        }
      }
    }
  } else {
    // ---- consumers ---------------------------------------------------------
    int s = 0;
    unsigned fph = 0;
    for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
      tdp_mbar_wait(tdp_smem_addr(&full_bar[s]), fph);
      const unsigned char* sb = tdp_ring + (size_t)s * TDP_STAGE_BYTES;
#if TDP_VEC_RING
      TdpRow r[TDP_PU];
      tdp_load_smem_pu(r, sb, warp * 32 + lane);
#pragma unroll
      for (int u = 0; u < TDP_PU; ++u) acc.row(P, r[u], true);
#else
#pragma unroll
      for (int u = 0; u < TDP_PU; ++u) {
        TdpRow r;
        tdp_load_smem(r, sb, (u * TDP_CONS_WARPS + warp) * 32 + lane);
        acc.row(P, r, true);
      }
#endif
      __syncwarp();
      if (lane == 0) tdp_mbar_arrive(tdp_smem_addr(&empty_bar[s]));
      if (++s == TDP_STAGES) {
        s = 0;
        fph ^= 1u;
      }
    }
    // tail rows (fewer than one tile) straight from global memory
    const int ctid = warp * 32 + lane;
    for (i64 i = ntiles * (i64)TDP_PTILE + (i64)blockIdx.x * (TDP_CONS_WARPS * 32) + ctid; i < P.n;
         i += (i64)gridDim.x * (TDP_CONS_WARPS * 32)) {
      TdpRow r;
      tdp_load(r, P, i);
      acc.row(P, r, true);
    }
  }
  acc.flush<TDP_CONS_WARPS + 1>(P);
}

// Materialise the selected rows' output values, compacted in row order.
// With predicates: the CTA owns one filter tile (TDP_FTILE rows) whose ballot
// words and output offset were produced by the AOT filter pass.
extern "C" __global__ void __launch_bounds__(256)
    tdp_scan_project(const __grid_constant__ TdpParams P) {
  if (P.bits == nullptr) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < P.n;
         i += (i64)gridDim.x * blockDim.x) {
      TdpRow r;
      tdp_load(r, P, i);
      tdp_project(r, P, i);
    }
    return;
  }
  __shared__ int word_prefix[TDP_FWORDS];
  __shared__ int warp_tot[TDP_FWORDS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 tile = blockIdx.x;
  unsigned myword = 0;
  int pc = 0, incl = 0;
  if (threadIdx.x < TDP_FWORDS) {
    myword = P.bits[tile * TDP_FWORDS + threadIdx.x];
    pc = __popc(myword);
    incl = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
  }
  __syncthreads();
  if (threadIdx.x < TDP_FWORDS) {
    int add = 0;
    for (int k = 0; k < warp; ++k) add += warp_tot[k];
    word_prefix[threadIdx.x] = add + incl - pc;
  }
  __syncthreads();
  const i64 obase = P.tile_off[tile];
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  for (int w = warp; w < TDP_FWORDS; w += 8) {
    const unsigned word = P.bits[tile * TDP_FWORDS + w];
    if (((word >> lane) & 1u) == 0u) continue;
    const i64 i = tile * (i64)TDP_FTILE + (i64)w * 32 + lane;
    TdpRow r;
    tdp_load(r, P, i);
    tdp_project(r, P, obase + word_prefix[w] + __popc(word & lt));
  }
}
