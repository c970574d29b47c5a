// K9: building blocks of the pressure solve and the per-step reductions (K12).
//
// Reference: pressure_solve (pkg/src/hybridnodes/solver.py:283-314) runs scipy's
// bicgstab on the bordered Poisson matrix with the complete SuperLU factorisation as
// preconditioner (solver.py:213-214).  Per warm step that is 2 A-matvecs and 1
// preconditioner application = permute, unit-lower solve, upper solve, permute.
// SuperLU convention: Pr A Pc = L U, so x = Pc U^-1 L^-1 Pr b:
//     y[perm_r[i]] = b[i];  z = L^-1 y;  w = U^-1 z;  x[i] = w[perm_c[i]].
//
// Triangular solves are sync-free: one warp per row, rows claimed in dependency order
// through an atomic ticket (so every row a warp waits on is owned by a running warp),
// each dependency read with an L1-bypassing load and spun on until it differs from a
// sentinel bit pattern written before the solve.  The value doubles as its own ready
// flag (64-bit stores are single-copy atomic), so no fences or counters are needed per
// edge.  The per-row sum uses a fixed lane assignment and a fixed shuffle tree: results
// are bitwise reproducible run to run.
//
// Reductions (dot, norm, max|.|, sums) use a fixed two-level tree (fixed grid of
// partials, then one block) -> deterministic.
#include "pressure.cuh"

namespace hn {

constexpr unsigned long long kSentinel = 0xFFFFFFFFFFFFFFFFull;  // negative NaN, all payload bits set

__device__ __forceinline__ double ld_acquire_dbl(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return __longlong_as_double(static_cast<long long>(v));
}
__device__ __forceinline__ void st_release_dbl(double* p, double x) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" :: "l"(p), "l"(__double_as_longlong(x)) : "memory");
}
__device__ __forceinline__ bool is_sentinel(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x)) == kSentinel;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Dependencies are spun on with exponential __nanosleep backoff so idle warps do not
// saturate L2 with polling loads.
__device__ __forceinline__ double wait_value(const double* p) {
  double v = ld_acquire_dbl(p);
  unsigned ns = 32;
  while (is_sentinel(v)) {
    __nanosleep(ns);
    ns = ns < 256 ? 2 * ns : 256;
    v = ld_acquire_dbl(p);
  }
  return v;
}

constexpr int kTaskChunk = 256;  // row entries a warp requests before it waits on any of them
constexpr int kPerLane = kTaskChunk / 32;

// ---- supernodal sync-free triangular solve --------------------------------------------
// Rows are grouped into blocks [r0, r0+w) whose in-block triangle is dense (SuperLU
// supernodes, w <= 256).  One CTA per block: (1) every row's outside part is pulled (warp
// per row, load-first + spin, one global hop per block; heavy blocks get helper tasks on
// other SMs), (2) the dense in-block triangle is solved in 32-column tiles: the warp owning
// the tile's rows solves it with shuffles, then every thread applies it to its own row.
// Row layout in the strict CSR (sorted columns):
//   lower: [outside cols < r0 | inside cols r0..i-1]   (inside count = i - r0)
//   upper: [inside cols i+1..r1-1 | outside cols >= r1] (inside count = r1-1-i)
// The dense triangle is read from a packed copy (hn_host_pack_panels): per 32-column tile
// one panel, column-major over the rows the tile touches, so a warp's load of one column
// is 32 consecutive doubles and the next panel arrives by ONE bulk async copy (TMA engine,
// cp.async.bulk + mbarrier) while the current tile is solved.  The CSR copy of the same
// entries is what the outside sums read; the panels are only the dense part.
constexpr int kSnThreads = 256;
constexpr int kSnWarps = kSnThreads / 32;
constexpr int kSnMaxW = kSnThreads;  // block width cap (one row per thread)
constexpr int kSnMaxPairs = 512;     // (row, 256-entry chunk) pairs of one task's outside phase

// Panel tt of a packed block of width w, in processing order (lower: tiles left to right,
// upper: right to left).  Panel rows: lower [t0, w), upper [0, t0 + tw); stored column-
// major with a row stride rp (rows rounded up to even: 16-byte aligned panels), always 32
// columns (the last tile's missing columns are zero).  Entry (row, t0 + k) lives at
// panel[k * rp + row - rbase]; entries on or across the diagonal are zero.
__host__ __device__ __forceinline__ void panel_geom(bool lower, int w, int tt, int& t0, int& tw, int& rbase,
                                                    int& rows, int& rp) {
  const int ntiles = (w + 31) / 32;
  t0 = lower ? 32 * tt : 32 * (ntiles - 1 - tt);
  tw = w - t0 < 32 ? w - t0 : 32;
  rbase = lower ? t0 : 0;
  rows = lower ? w - t0 : t0 + tw;
  rp = (rows + 1) & ~1;
}

// The panel sequence of a block task whose adjacent predecessor block P (the rw rows just
// before it in processing order: lower [r0 - rw, r0), upper [r0 + w, r0 + w + rw)) couples
// densely into every row: first ceil(rw / 32) "rectangle" panels -- P's columns in P's own
// tile order, all w rows, column-major -- then the triangle panels of panel_geom.  The
// rectangle tiles are applied as P's tiles are solved (the task polls their x values), so
// the hop from P to this block no longer waits for helper sums over P's columns.
__host__ __device__ __forceinline__ void seq_geom(bool lower, int w, int rw, int pi, bool& rect, int& t0, int& tw,
                                                  int& rbase, int& rows, int& rp) {
  const int nrect = (rw + 31) / 32;
  rect = pi < nrect;
  if (rect) {
    t0 = lower ? 32 * pi : 32 * (nrect - 1 - pi);  // column offset inside P
    tw = rw - t0 < 32 ? rw - t0 : 32;
    rbase = 0;
    rows = w;
    rp = (w + 1) & ~1;
  } else {
    panel_geom(lower, w, pi - nrect, t0, tw, rbase, rows, rp);
  }
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one thread: arm the barrier with the byte count, then the bulk copy completes it
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void l2_prefetch(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ double row_outside_sum(const int* __restrict__ cols, const double* __restrict__ vals,
                                                  int64_t e0, int len, const double* x, int lane) {
  double sum = 0.0;
  for (int base = 0; base < len; base += kTaskChunk) {
    int c[kPerLane];
    double v[kPerLane], xv[kPerLane];
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) {
      const int e = base + lane + 32 * k;
      c[k] = e < len ? __ldg(cols + e0 + e) : -1;
      v[k] = e < len ? __ldg(vals + e0 + e) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) xv[k] = c[k] >= 0 ? ld_acquire_dbl(x + c[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) {
      if (c[k] >= 0 && is_sentinel(xv[k])) xv[k] = wait_value(x + c[k]);
      sum = fma(v[k], xv[k], sum);
    }
  }
  return warp_sum(sum);
}

// The 32-row diagonal tile of a block by one warp: lane = row - t0, yv = its right-hand
// side with every earlier tile applied, lv[k] = its entry in column t0 + k (zero on and
// across the diagonal).  Forward (lower, unit diagonal) or backward (upper) substitution
// through the shuffle network; returns the lane's solution.
template <bool LOWER>
__device__ __forceinline__ double tile_substitute(const double (&lv)[32], double yv, double dg, int lane, int tw) {
  const double rdg = 1.0 / dg;  // off the dependency chain (x * (1/d): <= 1 ulp from x / d)
  if (LOWER) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double xk = __shfl_sync(0xffffffffu, yv, k);
      if (lane > k) yv = fma(-lv[k], xk, yv);
    }
  } else {
#pragma unroll
    for (int k = 31; k >= 0; --k) {
      if (lane == k && lane < tw) yv = yv * rdg;
      const double xk = __shfl_sync(0xffffffffu, yv, k);
      if (lane < k) yv = fma(-lv[k], xk, yv);
    }
  }
  return yv;
}

// Small block (w <= 32) solved by one warp: lane r owns row r0+r -- its outside part by a
// serial loop with 8 loads in flight (the planner only batches blocks whose rows are
// short), then the dense triangle with shuffles.  No shared memory, no CTA barrier.
template <bool LOWER>
__device__ __forceinline__ void warp_small_block(const int64_t* __restrict__ rowptr, const int* __restrict__ cols,
                                                 const double* __restrict__ vals, const double* __restrict__ diag,
                                                 const double* __restrict__ b, double* x, int r0, int w, int lane) {
  double yv = 0.0, dg = 1.0;
  double lv[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) lv[k] = 0.0;
  if (lane < w) {
    const int i = r0 + lane;
    const int64_t a = __ldg(rowptr + i), z = __ldg(rowptr + i + 1);
    const int inside = LOWER ? lane : (w - 1 - lane);
    const int64_t e0 = LOWER ? a : a + inside;
    const int64_t e1 = e0 + (z - a) - inside;
    double s = 0.0;
    for (int64_t e = e0; e < e1; e += 8) {
      int c[8];
      double v[8], xv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        c[k] = e + k < e1 ? __ldg(cols + e + k) : -1;
        v[k] = e + k < e1 ? __ldg(vals + e + k) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) xv[k] = c[k] >= 0 ? ld_acquire_dbl(x + c[k]) : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (c[k] >= 0 && is_sentinel(xv[k])) xv[k] = wait_value(x + c[k]);
        s = fma(v[k], xv[k], s);
      }
    }
    yv = __ldg(b + i) - s;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (LOWER) {
        if (k < lane) lv[k] = __ldg(vals + (z - lane) + k);           // col r0 + k
      } else {
        if (k > lane && k < w) lv[k] = __ldg(vals + a + (k - lane - 1));  // col r0 + k
      }
    }
    if (!LOWER) dg = __ldg(diag + i);
  }
  yv = tile_substitute<LOWER>(lv, yv, dg, lane, w);
  if (lane < w) st_release_dbl(x + r0 + lane, yv);
}

#ifdef HN_TRACE
// dev builds only (libhn_trace.so): per-task timeline [start, outside-done, end] ns + SM id
__device__ unsigned long long* g_sn_trace = nullptr;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
#define SN_TRACE(slot, value)                               \
  do {                                                      \
    if (g_sn_trace) g_sn_trace[4 * t + (slot)] = (value);   \
  } while (0)
#else
#define SN_TRACE(slot, value) \
  do {                        \
  } while (0)
#endif

// Task kinds: 0 = whole block (outside + dense), 1 = helper (outside sums of rows
// [rb, rb+rc) of a heavy block -> ysum, sentinel-flagged), 2 = dense part of a heavy block
// whose outside sums come from its helpers (scheduled right before it), 3 = batch of up to
// kSnWarps independent small blocks of one level, warp k solving member rb+k (member
// entries live past the task list in the same arrays).  blk_off[t] = offset of task t's
// packed panels (kinds 0 and 2).
template <bool LOWER>
__global__ void __launch_bounds__(kSnThreads, 2) sptrsv_super_kernel(
    const int* __restrict__ blk_kind, const int* __restrict__ blk_r0, const int* __restrict__ blk_w,
    const int* __restrict__ blk_rb, const int* __restrict__ blk_rc, const int64_t* __restrict__ blk_off,
    const int* __restrict__ blk_rw, int64_t nblk, const int64_t* __restrict__ rowptr, const int* __restrict__ cols, const double* __restrict__ vals,
    const double* __restrict__ diag, const double* __restrict__ packed, int inv, const double* __restrict__ b,
    double* x, double* ysum, unsigned long long* ticket, const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double ys[kSnMaxW];
  __shared__ double s_xr[32];                          // a rectangle tile's x values
  __shared__ int s_cnt[kSnMaxW], s_off[kSnMaxW + 1];  // outside phase: chunks per row, their offsets
  __shared__ long long s_e0[kSnMaxW];                  // ... first outside entry of each row
  __shared__ int s_len[kSnMaxW];                       // ... and the number of outside entries
  __shared__ short s_prow[kSnMaxPairs];                // pair -> row
  __shared__ double s_part[kSnMaxPairs];               // pair partial sums
  __shared__ unsigned long long tk;
  __shared__ alignas(8) unsigned long long mbar;
  extern __shared__ __align__(128) double sn_nbuf[];  // the next panel: [32][rp] (bulk copy)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) mbar_init(&mbar);
  __syncthreads();
  unsigned phase = 0;
  while (true) {
    if (tid == 0) tk = atomicAdd(ticket, 1ull);
    __syncthreads();
    const unsigned long long t = tk;
    __syncthreads();
    if (t >= static_cast<unsigned long long>(nblk)) return;
#ifdef HN_TRACE
    if (tid == 0) {
      SN_TRACE(0, gtime());
      SN_TRACE(3, smid());
    }
#endif
    const int kind = __ldg(blk_kind + t);
    if (kind == 3) {
      const int mb = __ldg(blk_rb + t), mc = __ldg(blk_rc + t);
      if (warp < mc)
        warp_small_block<LOWER>(rowptr, cols, vals, diag, b, x, __ldg(blk_r0 + mb + warp), __ldg(blk_w + mb + warp),
                                lane);
#ifdef HN_TRACE
      __syncthreads();
      if (tid == 0) SN_TRACE(2, gtime());
#endif
      continue;
    }
    const int r0 = __ldg(blk_r0 + t), w = __ldg(blk_w + t);
    const int rw = blk_rw ? __ldg(blk_rw + t) : 0;  // dense predecessor columns (rectangle panels)
    const double* P = kind == 1 ? nullptr : packed + __ldg(blk_off + t);
    const int npanels = (rw + 31) / 32 + (w + 31) / 32;
    if (tid == 0 && P && npanels > 1) {  // the whole packed block towards L2 while the outside sums run
      bool rect;
      int t0, tw, rbase, rows, rp;
      unsigned bytes = 0;
      for (int pi = 0; pi < npanels; ++pi) {
        seq_geom(LOWER, w, rw, pi, rect, t0, tw, rbase, rows, rp);
        bytes += 32u * rp * 8u;
      }
      l2_prefetch(P, bytes);
    }
    if (kind == 2) {
      for (int rr = tid; rr < w; rr += kSnThreads) ys[rr] = wait_value(ysum + r0 + rr);
    } else {
      // (1) outside contributions of rows [rb, re): every row is cut into 256-entry chunks
      // and the (row, chunk) pairs are spread over the 8 warps, so a long row costs
      // ceil(chunks / 8) dependent memory round trips instead of one per chunk; the chunk
      // partials are then added per row in chunk order (deterministic)
      const int rb = kind == 1 ? __ldg(blk_rb + t) : 0;
      const int nr = (kind == 1 ? __ldg(blk_rc + t) : w);
      for (int q = tid; q < nr; q += kSnThreads) {
        const int rr = rb + q, i = r0 + rr;
        const int64_t a = __ldg(rowptr + i);
        const int inside = LOWER ? rr : (w - 1 - rr);
        const int len = static_cast<int>(__ldg(rowptr + i + 1) - a) - inside - rw;
        s_cnt[q] = len > 0 ? (len + kTaskChunk - 1) / kTaskChunk : 1;
        // the row's outside entries minus the rectangle's: [s_e0, s_e0 + s_len)
        s_e0[q] = LOWER ? a : a + inside + rw;
        s_len[q] = len;
      }
      __syncthreads();
      if (warp == 0) {  // exclusive scan of the chunk counts (nr <= 256: 8 per lane)
        int v[8], tot = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int q = lane * 8 + k;
          v[k] = q < nr ? s_cnt[q] : 0;
          tot += v[k];
        }
        int inc = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        int run = inc - tot;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int q = lane * 8 + k;
          if (q < nr) s_off[q] = run;
          run += v[k];
        }
        if (lane == 31) s_off[nr] = inc;
      }
      __syncthreads();
      const int npairs = s_off[nr];  // the planner keeps this <= kSnMaxPairs
      for (int q = tid; q < nr; q += kSnThreads)
        for (int p = s_off[q]; p < s_off[q + 1]; ++p) s_prow[p] = static_cast<short>(q);
      __syncthreads();
      for (int p = warp; p < npairs; p += kSnWarps) {
        const int q = s_prow[p];
        const int c0 = (p - s_off[q]) * kTaskChunk;
        const int clen = s_len[q] - c0 < kTaskChunk ? s_len[q] - c0 : kTaskChunk;
        const double sp = clen > 0 ? row_outside_sum(cols, vals, s_e0[q] + c0, clen, x, lane) : 0.0;
        if (lane == 0) s_part[p] = sp;
      }
      __syncthreads();
      for (int q = tid; q < nr; q += kSnThreads) {
        double sum = 0.0;
        for (int p = s_off[q]; p < s_off[q + 1]; ++p) sum += s_part[p];
        const int rr = rb + q, i = r0 + rr;
        if (kind == 1) st_release_dbl(ysum + i, __ldg(b + i) - sum);
        else ys[rr] = __ldg(b + i) - sum;
      }
      if (kind == 1) {
#ifdef HN_TRACE
        __syncthreads();
        if (tid == 0) SN_TRACE(2, gtime());
#endif
        continue;
      }
    }
    if (tid >= w) ys[tid] = 0.0;  // the last tile's missing columns multiply zeros, never stale values
    __syncthreads();
#ifdef HN_TRACE
    if (tid == 0) SN_TRACE(1, gtime());
#endif
    // (2) dense in-block triangle from the packed panels; thread tid owns block row tid
#ifdef HN_TRACE
    unsigned long long wait_ns = 0;
#endif
    const bool has = tid < w;
    const int i = r0 + tid;
    const double dg = (!LOWER && has) ? __ldg(diag + i) : 1.0;
    const int pbase = LOWER ? r0 - rw : r0 + w;  // first row of the rectangle's predecessor
    bool rect;
    int t0, tw, rbase, rows, rp;
    seq_geom(LOWER, w, rw, 0, rect, t0, tw, rbase, rows, rp);
    const double* panel = P;
    double cur[32];
    double acc = 0.0;  // inv == 2: this row of x = B^-1 y, summed panel by panel
    {
      const int rr = tid - rbase;
      const bool in = has && rr >= 0 && rr < rows;
#pragma unroll
      for (int k = 0; k < 32; ++k) cur[k] = in ? __ldg(panel + k * rp + rr) : 0.0;
    }
    for (int pi = 0; pi < npanels; ++pi) {
      const bool more = pi + 1 < npanels;
      bool nrect;
      int n0, nw, nbase, nrows, nrp;
      seq_geom(LOWER, w, rw, more ? pi + 1 : pi, nrect, n0, nw, nbase, nrows, nrp);
      if (more && tid == 0) {  // the next panel as 4 bulk copies of 8 columns (one mbarrier phase)
        const unsigned part = 8u * nrp * 8u;
        mbar_expect(&mbar, 4u * part);
#pragma unroll
        for (int k = 0; k < 4; ++k) bulk_copy(sn_nbuf + k * 8 * nrp, panel + 32 * rp + k * 8 * nrp, part, &mbar);
      }
      if (rect) {  // predecessor columns [pbase + t0, + tw): wait for their x, apply to every row
        if (warp == 0) s_xr[lane] = lane < tw ? wait_value(x + pbase + t0 + lane) : 0.0;
        __syncthreads();
        if (has) {
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
          for (int k = 0; k < 32; k += 4) {
            a0 = fma(cur[k], s_xr[k], a0);
            a1 = fma(cur[k + 1], s_xr[k + 1], a1);
            a2 = fma(cur[k + 2], s_xr[k + 2], a2);
            a3 = fma(cur[k + 3], s_xr[k + 3], a3);
          }
          ys[tid] -= (a0 + a1) + (a2 + a3);
        }
      } else if (inv == 2) {
        // whole-block inverse: the panels hold B^-1 (B = the block's triangle with its diagonal),
        // so every panel is an independent slice of x = B^-1 y -- no tile-to-tile chain, no
        // barrier besides the panel hand-over.  ys keeps y (the rectangle panels came first).
        if (has) {
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
          for (int k = 0; k < 32; k += 4) {
            a0 = fma(cur[k], ys[t0 + k], a0);
            a1 = fma(cur[k + 1], ys[t0 + k + 1], a1);
            a2 = fma(cur[k + 2], ys[t0 + k + 2], a2);
            a3 = fma(cur[k + 3], ys[t0 + k + 3], a3);
          }
          acc += (a0 + a1) + (a2 + a3);
        }
      } else {
        if (warp == t0 / 32 && inv) {  // x = T^-1 y: 32 independent products, no chain
          // y of the tile's rows straight from shared memory (broadcast reads; columns past tw
          // are zero in the panel and ys beyond w is zeroed above): no 32-shuffle sequence
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
          for (int k = 0; k < 32; k += 4) {
            a0 = fma(cur[k], ys[t0 + k], a0);
            a1 = fma(cur[k + 1], ys[t0 + k + 1], a1);
            a2 = fma(cur[k + 2], ys[t0 + k + 2], a2);
            a3 = fma(cur[k + 3], ys[t0 + k + 3], a3);
          }
          __syncwarp();  // every lane has read the tile's y before any lane overwrites its entry
          if (lane < tw) {
            ys[tid] = (a0 + a1) + (a2 + a3);
            st_release_dbl(x + i, ys[tid]);
          }
        } else if (warp == t0 / 32) {  // the diagonal tile's rows: lane = row - t0
          const double yv = tile_substitute<LOWER>(cur, lane < tw ? ys[tid] : 0.0, dg, lane, tw);
          if (lane < tw) {
            ys[tid] = yv;
            st_release_dbl(x + i, yv);
          }
        }
        __syncthreads();
        if (has && (LOWER ? tid >= t0 + tw : tid < t0)) {  // apply the solved tile to my row
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
          for (int k = 0; k < 32; k += 4) {
            a0 = fma(cur[k], ys[t0 + k], a0);
            a1 = fma(cur[k + 1], ys[t0 + k + 1], a1);
            a2 = fma(cur[k + 2], ys[t0 + k + 2], a2);
            a3 = fma(cur[k + 3], ys[t0 + k + 3], a3);
          }
          ys[tid] -= (a0 + a1) + (a2 + a3);
        }
      }
      if (more) {
#ifdef HN_TRACE
        const unsigned long long tw0 = gtime();
        mbar_wait(&mbar, phase);
        if (tid == 0) wait_ns += gtime() - tw0;
#else
        mbar_wait(&mbar, phase);
#endif
        phase ^= 1u;
        const int rr = tid - nbase;
        const bool in = has && rr >= 0 && rr < nrows;
#pragma unroll
        for (int k = 0; k < 32; ++k) cur[k] = in ? sn_nbuf[k * nrp + rr] : 0.0;
        panel += 32 * rp;
        rect = nrect;
        t0 = n0;
        tw = nw;
        rbase = nbase;
        rows = nrows;
        rp = nrp;
      }
      __syncthreads();
    }
    if (inv == 2 && has) st_release_dbl(x + i, acc);
#ifdef HN_TRACE
    if (tid == 0) {
      SN_TRACE(2, gtime());
      SN_TRACE(3, wait_ns);  // dense tasks: ns spent waiting for panel copies (instead of the SM id)
    }
#endif
  }
}

__global__ void permute_in_kernel(const int* __restrict__ perm_r, const double* __restrict__ b, int64_t n,
                                  double* __restrict__ y) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[perm_r[i]] = b[i];
}
__global__ void permute_out_kernel(const int* __restrict__ perm_c, const double* __restrict__ w, int64_t n,
                                   double* __restrict__ x) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = w[perm_c[i]];
}

// ---- deterministic reductions ----
constexpr int kRedBlocks = 296;
constexpr int kRedThreads = 256;

enum RedOp : int { kDot = 0, kMaxAbs = 1, kSumAbs = 2, kSum = 3, kMaxAbsIdx = 4 };

template <int OP>
__device__ __forceinline__ double red_elem(const double* a, const double* b, const int* idx, int64_t i) {
  const int64_t j = idx ? idx[i] : i;
  if (OP == kDot) return a[j] * b[j];
  if (OP == kMaxAbs || OP == kSumAbs) return fabs(a[j]);
  return a[j];
}

template <int OP>
__device__ __forceinline__ double red_combine(double x, double y) {
  return (OP == kMaxAbs) ? fmax(x, y) : x + y;
}

template <int OP>
__device__ double block_reduce(double v, double* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = red_combine<OP>(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < (blockDim.x >> 5) ? sm[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = red_combine<OP>(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  __syncthreads();
  return v;
}

template <int OP>
__global__ void __launch_bounds__(kRedThreads) reduce_partials_kernel(const double* __restrict__ a,
                                                                      const double* __restrict__ b,
                                                                      const int* __restrict__ idx, int64_t n,
                                                                      double* __restrict__ partials) {
  __shared__ double sm[32];
  double v = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v = red_combine<OP>(v, red_elem<OP>(a, b, idx, i));
  v = block_reduce<OP>(v, sm);
  if (threadIdx.x == 0) partials[blockIdx.x] = v;
}

template <int OP>
__global__ void __launch_bounds__(kRedThreads) reduce_final_kernel(const double* __restrict__ partials, int np,
                                                                   double* __restrict__ out) {
  __shared__ double sm[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) v = red_combine<OP>(v, partials[i]);
  v = block_reduce<OP>(v, sm);
  if (threadIdx.x == 0) *out = v;
}

// BiCGStab vector updates, numpy operation order (scipy _isolve/iterative.py bicgstab):
//   p -= omega*v; p *= beta; p += r          (kind 0)
//   r -= alpha*v                              (kind 1, r = r - alpha*v)
//   x += alpha*phat                           (kind 2)
__global__ void bicg_p_update_kernel(double* __restrict__ p, const double* __restrict__ v,
                                     const double* __restrict__ r, double omega, double beta, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = __dadd_rn(__dmul_rn(__dsub_rn(p[i], __dmul_rn(omega, v[i])), beta), r[i]);
}
__global__ void axpy_kernel(double* __restrict__ y, const double* __restrict__ x, double alpha, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __dadd_rn(y[i], __dmul_rn(alpha, x[i]));
}

}  // namespace hn

using namespace hn;

#ifdef HN_TRACE
// Dev builds only (libhn_trace.so, tools/trace_sptrsv.py): per-task timeline of the
// supernodal solves, trace = 4 x ntasks u64 per launch (NULL = off).
HN_EXPORT int hn_debug_sptrsv_trace(unsigned long long* trace) {
  return cudaMemcpyToSymbol(g_sn_trace, &trace, sizeof(trace)) == cudaSuccess ? 0 : -1;
}
#endif

namespace hn {

__global__ void sptrsv_reset_kernel(double* __restrict__ x, double* __restrict__ ysum, int64_t n,
                                    unsigned long long* __restrict__ ticket, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    x[i] = __longlong_as_double(static_cast<long long>(kSentinel));
    ysum[i] = __longlong_as_double(static_cast<long long>(kSentinel));
  }
  if (i == 0) *ticket = 0ull;
}

constexpr int kNbuf = 32 * kSnMaxW * static_cast<int>(sizeof(double));  // one panel (dynamic smem)

// ---- dense groups ---------------------------------------------------------------------
// The top of the elimination tree -- the separators' (nearly) dense supernodes -- is a chain
// of 256-wide pieces that can only run one after the other: at config 3 the block levels >= 40
// of L (56 of its 96 levels, 26 K rows in 24 contiguous row runs) cost ~10 us each on a
// single CTA while the other 295 wait.  Those rows leave the task list (their rows are empty
// in the task kernel's matrix: x = b, overwritten here).  Each run G = [a, b) is solved through
// the explicit inverse of its triangle, formed once at setup:
//     x_G = inv(T_GG) * (b_G - C_G x),   C_G = G's rows restricted to the columns outside G
// = one CSR product and one dense triangular product, each a single launch over every SM for
// all runs of one phase (runs of a phase do not depend on each other; a run's phase = 1 + the
// highest phase among the runs it reads).  Lower: after the task kernel, phases ascending
// (C_G = columns < a: leaves and earlier runs, all final).  Upper: before the task kernel,
// phases ascending from the root run (C_G = columns >= b); the other rows then read these
// columns as ordinary, already final, dependencies.  The runs are closed under the solves'
// dependencies (no other row of L reads them; they read no other row of U).
// One CTA per row, fixed column striding and a fixed reduction tree: deterministic.
constexpr int kGroupThreads = 256;

__device__ __forceinline__ double group_block_sum(double v, double* s_red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  double tot = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < kGroupThreads / 32; ++k) tot += s_red[k];
  }
  return tot;  // valid on thread 0
}

// y[row] = b[row] - sum_e vals[e] * x[cols[e]] over the row's entries outside its run
__global__ void __launch_bounds__(kGroupThreads) group_coupling_kernel(
    const int* __restrict__ g_row, const int64_t* __restrict__ rowptr, const int* __restrict__ cols,
    const double* __restrict__ vals, int64_t q0, const double* __restrict__ b, const double* __restrict__ x,
    double* __restrict__ y, const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double s_red[kGroupThreads / 32];
  const int64_t q = q0 + blockIdx.x;
  const int64_t e0 = __ldg(rowptr + q), e1 = __ldg(rowptr + q + 1);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += 4 * kGroupThreads) {
    const int64_t ea = e + kGroupThreads, eb = e + 2 * kGroupThreads, ec = e + 3 * kGroupThreads;
    const int c0 = __ldg(cols + e);
    const int c1 = ea < e1 ? __ldg(cols + ea) : -1;
    const int c2 = eb < e1 ? __ldg(cols + eb) : -1;
    const int c3 = ec < e1 ? __ldg(cols + ec) : -1;
    const double v0 = __ldg(vals + e);
    const double v1 = c1 >= 0 ? __ldg(vals + ea) : 0.0;
    const double v2 = c2 >= 0 ? __ldg(vals + eb) : 0.0;
    const double v3 = c3 >= 0 ? __ldg(vals + ec) : 0.0;
    a0 = fma(v0, x[c0], a0);
    a1 = fma(v1, c1 >= 0 ? x[c1] : 0.0, a1);
    a2 = fma(v2, c2 >= 0 ? x[c2] : 0.0, a2);
    a3 = fma(v3, c3 >= 0 ? x[c3] : 0.0, a3);
  }
  const double tot = group_block_sum((a0 + a1) + (a2 + a3), s_red);
  if (threadIdx.x == 0) {
    const int row = __ldg(g_row + q);
    y[row] = __ldg(b + row) - tot;
  }
}

// x[row] = sum_c inv[off + c] * y[ystart + c], c < cnt (the row's part of its run's inverse);
// echo (upper): the rhs entry takes the solution too, so the task kernel's trivial row
// (x = b / 1) reproduces it
__global__ void __launch_bounds__(kGroupThreads) group_gemv_kernel(
    const int* __restrict__ g_row, const int64_t* __restrict__ g_off, const int* __restrict__ g_cnt,
    const int* __restrict__ g_ystart, const double* __restrict__ inv, int64_t q0, const double* __restrict__ y,
    double* __restrict__ x, double* __restrict__ echo, const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double s_red[kGroupThreads / 32];
  const int64_t q = q0 + blockIdx.x;
  const double* row = inv + __ldg(g_off + q);
  const int cnt = __ldg(g_cnt + q);
  const double* yv = y + __ldg(g_ystart + q);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  for (int c = threadIdx.x; c < cnt; c += 4 * kGroupThreads) {
    const int ca = c + kGroupThreads, cb = c + 2 * kGroupThreads, cc = c + 3 * kGroupThreads;
    const double m0 = __ldg(row + c);
    const double m1 = ca < cnt ? __ldg(row + ca) : 0.0;
    const double m2 = cb < cnt ? __ldg(row + cb) : 0.0;
    const double m3 = cc < cnt ? __ldg(row + cc) : 0.0;
    a0 = fma(m0, yv[c], a0);
    a1 = fma(m1, ca < cnt ? yv[ca] : 0.0, a1);
    a2 = fma(m2, cb < cnt ? yv[cb] : 0.0, a2);
    a3 = fma(m3, cc < cnt ? yv[cc] : 0.0, a3);
  }
  const double tot = group_block_sum((a0 + a1) + (a2 + a3), s_red);
  if (threadIdx.x == 0) {
    const int r = __ldg(g_row + q);
    x[r] = tot;
    if (echo) echo[r] = tot;
  }
}

cudaError_t sptrsv_prepare() {
  // per-device function attributes: set on every call (cheap), so any device a process
  // drives gets the opt-in; never called inside a stream capture
  cudaError_t e = cudaFuncSetAttribute(sptrsv_super_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kNbuf);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(sptrsv_super_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kNbuf);
}

static void group_phases(const hn_tri_plan& p, double* b, double* x, const int* skip, cudaStream_t s) {
  // y lives in the plan's own scratch (g_y), never in ysum: there a non-sentinel value means
  // "the helpers' sum is ready", and an upper block may end in a group row (an empty row joins
  // the supernode of the rows before it), whose dense task would take the groups' y for it
  for (int ph = 0; ph < p.n_phases; ++ph) {
    const int64_t q0 = p.phase_ptr[ph], rows = p.phase_ptr[ph + 1] - q0;
    if (rows <= 0) continue;
    group_coupling_kernel<<<static_cast<unsigned>(rows), kGroupThreads, 0, s>>>(p.g_row, p.g_cpl_rowptr, p.g_cpl_cols,
                                                                                p.g_cpl_vals, q0, b, x, p.g_y, skip);
    group_gemv_kernel<<<static_cast<unsigned>(rows), kGroupThreads, 0, s>>>(p.g_row, p.g_inv_off, p.g_cnt, p.g_ystart,
                                                                            p.g_inv, q0, p.g_y, x,
                                                                            p.lower ? nullptr : b, skip);
  }
}

cudaError_t sptrsv_enqueue(const hn_tri_plan& p, double* b, double* x, double* ysum, int64_t n,
                           unsigned long long* ticket, int ctas_per_sm, const int* skip, cudaStream_t s) {
  const bool groups = p.g_inv != nullptr && p.g_y != nullptr && p.n_phases > 0;
  if ((p.ntasks == 0 && !groups) || n == 0) return cudaSuccess;
  sptrsv_reset_kernel<<<ceil_div(n, 256), 256, 0, s>>>(x, ysum, n, ticket, skip);
  if (!p.lower && groups) group_phases(p, b, x, skip, s);  // upper: the top of the tree first
  const int blocks = sm_count() * (ctas_per_sm > 0 ? ctas_per_sm : 2);
  if (p.ntasks > 0) {
    if (p.lower)
      sptrsv_super_kernel<true><<<blocks, kSnThreads, kNbuf, s>>>(p.kind, p.r0, p.w, p.rb, p.rc, p.off, p.rw,
                                                                  p.ntasks, p.rowptr, p.cols, p.vals, p.diag,
                                                                  p.packed, p.inv, b, x, ysum, ticket, skip);
    else
      sptrsv_super_kernel<false><<<blocks, kSnThreads, kNbuf, s>>>(p.kind, p.r0, p.w, p.rb, p.rc, p.off, p.rw,
                                                                   p.ntasks, p.rowptr, p.cols, p.vals, p.diag,
                                                                   p.packed, p.inv, b, x, ysum, ticket, skip);
  }
  if (p.lower && groups) group_phases(p, b, x, skip, s);  // lower: the top of the tree last
  return cudaGetLastError();
}

}  // namespace hn

using namespace hn;

// Supernodal solve over planned tasks (processing order), see sptrsv_super_kernel.
// x and ysum are reset to the sentinel here; ctas_per_sm persistent CTAs per SM.
HN_EXPORT int hn_sptrsv_super(int lower, const int* blk_kind, const int* blk_r0, const int* blk_w, const int* blk_rb,
                              const int* blk_rc, const int64_t* blk_off, const int* blk_rw, int64_t nblk,
                              const int64_t* rowptr,
                              const int* cols, const double* vals, const double* diag, const double* packed,
                              int inv, const double* b, double* x, double* ysum, int64_t n,
                              unsigned long long* ticket, int ctas_per_sm, void* stream) {
  if (nblk == 0) return 0;
  HN_TRY(sptrsv_prepare());
  const hn_tri_plan p{lower, inv, nblk, blk_kind, blk_r0, blk_w, blk_rb, blk_rc, blk_off, blk_rw, rowptr, cols, vals,
                      diag, packed, 0, {0}, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  HN_TRY(sptrsv_enqueue(p, const_cast<double*>(b), x, ysum, n, ticket, ctas_per_sm, nullptr, as_stream(stream)));
  return 0;
}

// The same solve from a plan struct, dense groups included.  An upper plan with groups
// overwrites the groups' entries of b with their solution (see group_gemv_kernel).
HN_EXPORT int hn_sptrsv_plan(const hn_tri_plan* plan, double* b, double* x, double* ysum, int64_t n,
                             unsigned long long* ticket, int ctas_per_sm, void* stream) {
  if (!plan) return 1;
  if (plan->n_phases < 0 || plan->n_phases > 16) return 2;
  HN_TRY(sptrsv_prepare());
  HN_TRY(sptrsv_enqueue(*plan, b, x, ysum, n, ticket, ctas_per_sm, nullptr, as_stream(stream)));
  return 0;
}

// Host helper (setup): the packed dense triangles sptrsv_super_kernel reads (see
// panel_geom), for every task of kind 0 or 2 (blk_off[t] = its offset in doubles; -1 for
// other kinds).  packed == NULL: offsets only.  Returns the total size in doubles.
HN_EXPORT int64_t hn_host_pack_panels(const int64_t* rowptr_host, const int* cols_host, const double* vals_host,
                                      const double* diag_host, int lower, int inverse, int64_t ntasks,
                                      const int* kind_host, const int* r0_host, const int* w_host,
                                      const int* rw_host, int64_t* off_host, double* packed_host) {
  int64_t total = 0;
  for (int64_t t = 0; t < ntasks; ++t) {
    const int w = w_host[t];
    const int rw = rw_host ? rw_host[t] : 0;
    if ((kind_host[t] != 0 && kind_host[t] != 2) || w < 1 || w > kSnMaxW || rw < 0 || rw > kSnMaxW) {
      off_host[t] = -1;
      continue;
    }
    off_host[t] = total;
    const int64_t r0 = r0_host[t];
    const int64_t pr0 = lower ? r0 - rw : r0 + w;  // the rectangle's predecessor rows
    const int npanels = (rw + 31) / 32 + (w + 31) / 32;
    // inverse == 2: X = B^-1 of the whole block triangle B (unit / U's diagonal included), by
    // substitution on the identity; the triangle panels then hold X instead of B
    static thread_local double* Bm = nullptr;
    static thread_local double* Xm = nullptr;
    if (inverse == 2 && packed_host) {
      if (!Bm) {
        Bm = new double[kSnMaxW * kSnMaxW];
        Xm = new double[kSnMaxW * kSnMaxW];
      }
      for (int row = 0; row < w; ++row) {
        const int64_t i = r0 + row;
        const int64_t a = rowptr_host[i], z = rowptr_host[i + 1];
        for (int c = 0; c < w; ++c) Bm[row * w + c] = 0.0;
        Bm[row * w + row] = lower ? 1.0 : diag_host[i];
        for (int c = (lower ? 0 : row + 1); c < (lower ? row : w); ++c) {
          const int64_t e = lower ? (z - row) + c : a + (c - row - 1);
          if (e < a || e >= z || cols_host[e] != r0 + c) return -1;  // not dense
          Bm[row * w + c] = vals_host[e];
        }
      }
      for (int j = 0; j < w; ++j) {
        if (lower) {
          for (int l = 0; l < w; ++l) {
            if (l < j) { Xm[l * w + j] = 0.0; continue; }
            double v = l == j ? 1.0 : 0.0;
            for (int k = j; k < l; ++k) v -= Bm[l * w + k] * Xm[k * w + j];
            Xm[l * w + j] = v;
          }
        } else {
          for (int l = w - 1; l >= 0; --l) {
            if (l > j) { Xm[l * w + j] = 0.0; continue; }
            double v = l == j ? 1.0 : 0.0;
            for (int k = l + 1; k <= j; ++k) v -= Bm[l * w + k] * Xm[k * w + j];
            Xm[l * w + j] = v / Bm[l * w + l];
          }
        }
      }
    }
    for (int pi = 0; pi < npanels; ++pi) {
      bool rect;
      int t0, tw, rbase, rows, rp;
      seq_geom(lower != 0, w, rw, pi, rect, t0, tw, rbase, rows, rp);
      if (packed_host) {
        double* pn = packed_host + total;
        for (int64_t q = 0; q < 32LL * rp; ++q) pn[q] = 0.0;
        for (int rr = 0; rr < rows; ++rr) {
          const int row = rbase + rr;
          const int64_t i = r0 + row;
          const int64_t a = rowptr_host[i], z = rowptr_host[i + 1];
          const int inside = lower ? row : w - 1 - row;
          for (int k = 0; k < tw; ++k) {
            const int c = t0 + k;
            int64_t e;
            int64_t want;
            if (rect) {  // predecessor column pr0 + c: the last rw outside entries (lower) / the first (upper)
              e = lower ? (z - inside - rw) + c : a + inside + c;
              want = pr0 + c;
            } else if (inverse == 2) {
              if (lower ? c <= row : c >= row) pn[static_cast<int64_t>(k) * rp + rr] = Xm[row * w + c];
              continue;
            } else {
              if (!(lower ? c < row : c > row)) continue;
              e = lower ? (z - row) + c : a + (c - row - 1);
              want = r0 + c;
            }
            if (e < a || e >= z || cols_host[e] != want) return -1;  // not dense
            pn[static_cast<int64_t>(k) * rp + rr] = vals_host[e];
          }
        }
        if (inverse == 1 && !rect) {  // the diagonal tile's rows hold T^-1 (substitution on the identity)
          double T[32][32], X[32][32];
          const int d0 = t0 - rbase;  // first diagonal-tile row inside the panel
          for (int l = 0; l < tw; ++l)
            for (int k = 0; k < tw; ++k)
              T[l][k] = l == k ? (lower ? 1.0 : diag_host[r0 + t0 + l])
                               : pn[static_cast<int64_t>(k) * rp + d0 + l];
          for (int j = 0; j < tw; ++j) {
            if (lower) {
              for (int l = 0; l < tw; ++l) {
                double v = l == j ? 1.0 : 0.0;
                for (int k = 0; k < l; ++k) v -= T[l][k] * X[k][j];
                X[l][j] = v;
              }
            } else {
              for (int l = tw - 1; l >= 0; --l) {
                double v = l == j ? 1.0 : 0.0;
                for (int k = l + 1; k < tw; ++k) v -= T[l][k] * X[k][j];
                X[l][j] = v / T[l][l];
              }
            }
          }
          for (int l = 0; l < tw; ++l)
            for (int k = 0; k < tw; ++k) pn[static_cast<int64_t>(k) * rp + d0 + l] = X[l][k];
        }
      }
      total += 32LL * rp;
    }
  }
  return total;
}

// Host helper (setup): split the rows of a strict triangular CSR (sorted columns) into
// blocks whose in-block triangle is dense, at most `cap` rows (<= 4096).  Writes blocks in
// row order (r0 ascending) and returns their number.
HN_EXPORT int64_t hn_host_supernodes(const int64_t* rowptr_host, const int* cols_host, int64_t n, int lower,
                                     int cap, int* blk_r0_host, int* blk_w_host) {
  if (cap <= 0 || cap > kSnMaxW) cap = kSnMaxW;
  int64_t nb = 0;
  if (lower) {
    int64_t r0 = 0;
    for (int64_t i = 1; i <= n; ++i) {
      bool join = false;
      if (i < n && i - r0 < cap) {
        const int64_t cnt = i - r0, a = rowptr_host[i], z = rowptr_host[i + 1];
        join = (z - a >= cnt) && cols_host[z - cnt] == r0 && cols_host[z - 1] == i - 1;
      }
      if (!join) {
        blk_r0_host[nb] = static_cast<int>(r0);
        blk_w_host[nb] = static_cast<int>(i - r0);
        ++nb;
        r0 = i;
      }
    }
  } else {
    int64_t r1 = n;  // current block [i+1, r1)
    for (int64_t i = n - 2; i >= -1; --i) {
      bool join = false;
      if (i >= 0 && r1 - 1 - i < cap) {
        const int64_t cnt = r1 - 1 - i, a = rowptr_host[i], z = rowptr_host[i + 1];
        join = (z - a >= cnt) && cols_host[a] == i + 1 && cols_host[a + cnt - 1] == r1 - 1;
      }
      if (!join) {
        blk_r0_host[nb] = static_cast<int>(i + 1);
        blk_w_host[nb] = static_cast<int>(r1 - (i + 1));
        ++nb;
        r1 = i + 1;
      }
    }
    // row order ascending
    for (int64_t k = 0; k < nb / 2; ++k) {
      int t0 = blk_r0_host[k]; blk_r0_host[k] = blk_r0_host[nb - 1 - k]; blk_r0_host[nb - 1 - k] = t0;
      int t1 = blk_w_host[k]; blk_w_host[k] = blk_w_host[nb - 1 - k]; blk_w_host[nb - 1 - k] = t1;
    }
  }
  return nb;
}

// Host helper (setup): dependency level of each block (blocks in row order).
HN_EXPORT int hn_host_block_levels(const int64_t* rowptr_host, const int* cols_host, int64_t n, int lower,
                                   int64_t nblk, const int* blk_r0_host, const int* blk_w_host, int* levels_host) {
  int* owner = new int[n];
  for (int64_t k = 0; k < nblk; ++k)
    for (int r = 0; r < blk_w_host[k]; ++r) owner[blk_r0_host[k] + r] = static_cast<int>(k);
  for (int64_t q = 0; q < nblk; ++q) {
    const int64_t k = lower ? q : nblk - 1 - q;
    const int r0 = blk_r0_host[k], r1 = r0 + blk_w_host[k];
    int lev = 0;
    for (int i = r0; i < r1; ++i)
      for (int64_t e = rowptr_host[i]; e < rowptr_host[i + 1]; ++e) {
        const int c = cols_host[e];
        if (c >= r0 && c < r1) continue;
        const int l = levels_host[owner[c]] + 1;
        lev = l > lev ? l : lev;
      }
    levels_host[k] = lev;
  }
  delete[] owner;
  return 0;
}

HN_EXPORT int hn_permute(int direction, const int* perm, const double* in, int64_t n, double* out, void* stream) {
  if (n == 0) return 0;
  const int th = 256;
  if (direction == 0) permute_in_kernel<<<ceil_div(n, th), th, 0, as_stream(stream)>>>(perm, in, n, out);
  else permute_out_kernel<<<ceil_div(n, th), th, 0, as_stream(stream)>>>(perm, in, n, out);
  HN_CHECK_LAUNCH();
  return 0;
}

// op: 0 dot(a,b), 1 max|a|, 2 sum|a|, 3 sum(a); idx (optional) gathers a[idx[i]], b[idx[i]].
// scratch: >= 296 doubles; result written to out[0] (device).
HN_EXPORT int hn_reduce(int op, const double* a, const double* b, const int* idx, int64_t n, double* scratch,
                        double* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  const int blocks = static_cast<int>(n > 0 ? (ceil_div(n, kRedThreads) < kRedBlocks ? ceil_div(n, kRedThreads) : kRedBlocks) : 1);
  switch (op) {
    case kDot:
      reduce_partials_kernel<kDot><<<blocks, kRedThreads, 0, s>>>(a, b, idx, n, scratch);
      reduce_final_kernel<kDot><<<1, kRedThreads, 0, s>>>(scratch, blocks, out);
      break;
    case kMaxAbs:
      reduce_partials_kernel<kMaxAbs><<<blocks, kRedThreads, 0, s>>>(a, b, idx, n, scratch);
      reduce_final_kernel<kMaxAbs><<<1, kRedThreads, 0, s>>>(scratch, blocks, out);
      break;
    case kSumAbs:
      reduce_partials_kernel<kSumAbs><<<blocks, kRedThreads, 0, s>>>(a, b, idx, n, scratch);
      reduce_final_kernel<kSumAbs><<<1, kRedThreads, 0, s>>>(scratch, blocks, out);
      break;
    case kSum:
      reduce_partials_kernel<kSum><<<blocks, kRedThreads, 0, s>>>(a, b, idx, n, scratch);
      reduce_final_kernel<kSum><<<1, kRedThreads, 0, s>>>(scratch, blocks, out);
      break;
    default:
      return 1;
  }
  HN_CHECK_LAUNCH();
  return 0;
}

// kind 0: p = ((p - omega*v) * beta) + r ; kind 1: y += alpha * x
HN_EXPORT int hn_bicg_update(int kind, double* y, const double* x, const double* r, double alpha, double beta,
                             int64_t n, void* stream) {
  if (n == 0) return 0;
  const int th = 256;
  cudaStream_t s = as_stream(stream);
  if (kind == 0) bicg_p_update_kernel<<<ceil_div(n, th), th, 0, s>>>(y, x, r, alpha, beta, n);
  else axpy_kernel<<<ceil_div(n, th), th, 0, s>>>(y, x, alpha, n);
  HN_CHECK_LAUNCH();
  return 0;
}
