// Kernel skeleton of the fused scan -> filter -> expression -> aggregate
// pipeline.  This text is compiled at run time by NVRTC for sm_100a after the
// query-specific part (TdpRow / tdp_load / tdp_eval / tdp_store, emitted by
// pipeline.cu from the tdp_instr program) is prepended.  It is embedded in
// libtdp_kernels.so as a string (see pipeline.cu, TDP_SKELETON).
//
// Row mapping: a CTA of TDP_THREADS threads consumes TDP_THREADS*TDP_U rows
// per step; row (base + u*TDP_THREADS + tid) so every load instruction of a
// warp covers 32 consecutive rows (256 contiguous bytes for 8-byte columns).
// All TDP_U rows' columns are loaded before any is evaluated to keep
// TDP_U * (#columns) independent loads in flight per thread.
//
// Accumulation modes:
//   TDP_REGACC=1  slots*(1+NF+NI) <= 64: every thread keeps all groups'
//                 accumulators in registers (predicated adds, no atomics),
//                 CTA tree-reduces and writes one partial row; a fixed-order
//                 reduction over CTAs makes the result deterministic.
//   TDP_REGACC=0  atomics straight into zeroed global accumulators.

#define TDP_CELLS (TDP_G * (1 + TDP_NF + TDP_NI))
#define TDP_NFA (TDP_NF > 0 ? TDP_NF : 1)
#define TDP_NIA (TDP_NI > 0 ? TDP_NI : 1)

template <class T>
__device__ __forceinline__ T tdp_warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

extern "C" __global__ void __launch_bounds__(TDP_THREADS)
    tdp_scan_agg(const __grid_constant__ TdpParams P) {
  const i64 tile = (i64)TDP_THREADS * TDP_U;
  const i64 step = (i64)gridDim.x * tile;
#if TDP_REGACC
  i64 cnt[TDP_G];
  double af[TDP_G][TDP_NFA];
  i64 ai[TDP_G][TDP_NIA];
#pragma unroll
  for (int s = 0; s < TDP_G; ++s) {
    cnt[s] = 0;
#pragma unroll
    for (int a = 0; a < TDP_NFA; ++a) af[s][a] = 0.0;
#pragma unroll
    for (int a = 0; a < TDP_NIA; ++a) ai[s][a] = 0;
  }
#endif
  for (i64 base = (i64)blockIdx.x * tile; base < P.n; base += step) {
    TdpRow r[TDP_U];
#pragma unroll
    for (int u = 0; u < TDP_U; ++u) {
      const i64 i = base + (i64)u * TDP_THREADS + threadIdx.x;
      if (i < P.n) tdp_load(r[u], P, i);
      else tdp_zero(r[u]);
    }
#pragma unroll
    for (int u = 0; u < TDP_U; ++u) {
      const i64 i = base + (i64)u * TDP_THREADS + threadIdx.x;
      int slot = 0;
      double f[TDP_NFA];
      i64 q[TDP_NIA];
      const bool keep = tdp_eval(r[u], P, slot, f, q) && (i < P.n);
#if TDP_REGACC
#pragma unroll
      for (int s = 0; s < TDP_G; ++s) {
        const bool hit = keep && (slot == s);
        cnt[s] += hit ? 1 : 0;
#pragma unroll
        for (int a = 0; a < TDP_NF; ++a) af[s][a] += hit ? f[a] : 0.0;
#pragma unroll
        for (int a = 0; a < TDP_NI; ++a)
          ai[s][a] = (i64)((u64)ai[s][a] + (hit ? (u64)q[a] : 0ull));
      }
#else
      if (keep) {
        atomicAdd(reinterpret_cast<u64*>(P.acc) + slot, 1ull);
#pragma unroll
        for (int a = 0; a < TDP_NF; ++a)
          atomicAdd(reinterpret_cast<double*>(P.acc) + (i64)TDP_G * (1 + a) + slot, f[a]);
#pragma unroll
        for (int a = 0; a < TDP_NI; ++a)
          atomicAdd(reinterpret_cast<u64*>(P.acc) + (i64)TDP_G * (1 + TDP_NF + a) + slot,
                    (u64)q[a]);
      }
#endif
    }
  }
#if TDP_REGACC
  // CTA reduction in a fixed order: warp shuffle tree, then warps 0..W-1.
  __shared__ u64 red[TDP_THREADS / 32][TDP_CELLS];
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
      const i64 v = (i64)tdp_warp_sum((u64)ai[s][a]);
      if (lane == 0) red[warp][TDP_G * (1 + TDP_NF + a) + s] = (u64)v;
    }
  }
  __syncthreads();
  u64* out = reinterpret_cast<u64*>(P.acc) + (i64)blockIdx.x * TDP_CELLS;
  for (int c = threadIdx.x; c < TDP_CELLS; c += TDP_THREADS) {
    const bool is_f = c >= TDP_G && c < TDP_G * (1 + TDP_NF);
    if (is_f) {
      double v = 0.0;
      for (int w = 0; w < TDP_THREADS / 32; ++w) v += __longlong_as_double((i64)red[w][c]);
      out[c] = (u64)__double_as_longlong(v);
    } else {
      u64 v = 0;
      for (int w = 0; w < TDP_THREADS / 32; ++w) v += red[w][c];
      out[c] = v;
    }
  }
#endif
}

// Materialise the selected rows' output values, compacted in row order.
// With predicates: the CTA owns one filter tile (TDP_FTILE rows) whose ballot
// words and output offset were produced by the AOT filter pass.
extern "C" __global__ void __launch_bounds__(256) tdp_scan_project(const __grid_constant__ TdpParams P) {
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
