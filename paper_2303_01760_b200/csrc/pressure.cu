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
#include "hn_common.cuh"

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

// LOWER=true: rows 0..n-1, x_i = b_i - sum_j L_ij x_j (unit diagonal not stored)
// LOWER=false: rows n-1..0, x_i = (b_i - sum_j U_ij x_j) / diag_i
template <bool LOWER>
__global__ void __launch_bounds__(256) sptrsv_kernel(const int64_t* __restrict__ rowptr, const int* __restrict__ cols,
                                                     const double* __restrict__ vals, const double* __restrict__ diag,
                                                     const double* __restrict__ b, double* x, int64_t n,
                                                     unsigned long long* ticket) {
  const int lane = threadIdx.x & 31;
  while (true) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= static_cast<unsigned long long>(n)) return;
    const int64_t row = LOWER ? static_cast<int64_t>(t) : n - 1 - static_cast<int64_t>(t);
    const int64_t e0 = __ldg(rowptr + row), e1 = __ldg(rowptr + row + 1);
    double sum = 0.0;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const int c = __ldg(cols + e);
      const double v = __ldg(vals + e);
      double xc = ld_acquire_dbl(x + c);
      while (is_sentinel(xc)) xc = ld_acquire_dbl(x + c);
      sum = fma(v, xc, sum);
    }
    sum = warp_sum(sum);
    if (lane == 0) {
      double r = __ldg(b + row) - sum;
      if (!LOWER) r = r / __ldg(diag + row);
      st_release_dbl(x + row, r);
    }
  }
}

// Scheduled variant: tasks in dependency-level order; a row longer than the chunk size is
// split into partial-sum tasks (np = -1, written to partial[part]) followed by a final
// task (np = number of partials) that adds them in fixed order -> deterministic.
// Waiting uses exponential __nanosleep backoff so idle warps do not saturate L2.
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

constexpr int kTaskChunk = 256;           // nnz per task (host planner uses the same)
constexpr int kPerLane = kTaskChunk / 32;

template <bool DIV>
__global__ void __launch_bounds__(256) sptrsv_tasks_kernel(
    const int* __restrict__ task_row, const int64_t* __restrict__ task_beg, const int* __restrict__ task_len,
    const int* __restrict__ task_part, const int* __restrict__ task_np, int64_t ntasks, const int* __restrict__ cols,
    const double* __restrict__ vals, const double* __restrict__ diag, const double* __restrict__ b, double* x,
    double* partial, unsigned long long* ticket) {
  const int lane = threadIdx.x & 31;
  while (true) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= static_cast<unsigned long long>(ntasks)) return;
    const int row = __ldg(task_row + t);
    const int64_t e0 = __ldg(task_beg + t);
    const int len = __ldg(task_len + t);
    // all of the lane's operands are requested before anything waits: one L2 round trip
    // per task instead of one per element; then spin only on values not yet produced
    int c[kPerLane];
    double v[kPerLane], xv[kPerLane];
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) {
      const int e = lane + 32 * k;
      c[k] = e < len ? __ldg(cols + e0 + e) : -1;
      v[k] = e < len ? __ldg(vals + e0 + e) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) xv[k] = c[k] >= 0 ? ld_acquire_dbl(x + c[k]) : 0.0;
    double sum = 0.0;
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) {
      if (c[k] >= 0 && is_sentinel(xv[k])) xv[k] = wait_value(x + c[k]);
      sum = fma(v[k], xv[k], sum);
    }
    sum = warp_sum(sum);
    if (lane == 0) {
      const int np = __ldg(task_np + t);
      const int part = __ldg(task_part + t);
      if (np < 0) {
        st_release_dbl(partial + part, sum);
      } else {
        double tot = 0.0;
        for (int k = 0; k < np; ++k) tot += wait_value(partial + part + k);
        tot += sum;
        double r = __ldg(b + row) - tot;
        if (DIV) r = r / __ldg(diag + row);
        st_release_dbl(x + row, r);
      }
    }
  }
}

// ---- supernodal variant -------------------------------------------------------------
// Rows are grouped into blocks [r0, r0+w) whose in-block triangle is dense (SuperLU
// supernodes).  One CTA per block: (1) every row's outside part is pulled (warp per row,
// load-first + spin, one global hop per block), (2) the dense in-block triangle is solved
// in 32-column tiles: one warp solves the diagonal tile with shuffles, then all warps
// apply the tile to the remaining rows.  Row layout in the strict CSR (sorted columns):
//   lower: [outside cols < r0 | inside cols r0..i-1]   (inside count = i - r0)
//   upper: [inside cols i+1..r1-1 | outside cols >= r1] (inside count = r1-1-i)
constexpr int kSnThreads = 256;
constexpr int kSnWarps = kSnThreads / 32;
constexpr int kSnMaxW = 4096;

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

// Small block (w <= 32) solved by one warp: lane r owns row r0+r -- its outside part by a
// serial loop with 8 loads in flight (the planner only batches blocks whose rows are
// short), then the dense triangle with shuffles.  No shared memory, no CTA barrier.
template <bool LOWER>
__device__ __forceinline__ void warp_small_block(const int64_t* __restrict__ rowptr, const int* __restrict__ cols,
                                                 const double* __restrict__ vals, const double* __restrict__ diag,
                                                 const double* __restrict__ tinv, const double* __restrict__ b,
                                                 double* x, int r0, int w, int lane) {
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
      if (tinv) {
        if (k < w) lv[k] = __ldg(tinv + static_cast<int64_t>(i) * 32 + k);  // row of the tile inverse
      } else if (LOWER) {
        if (k < lane) lv[k] = __ldg(vals + (z - lane) + k);           // col r0 + k
      } else {
        if (k > lane && k < w) lv[k] = __ldg(vals + a + (k - lane - 1));  // col r0 + k
      }
    }
    if (!LOWER) dg = __ldg(diag + i);
  }
  if (tinv) {  // x = T^-1 y: 32 independent products, no dependency chain through the shuffles
    double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
    for (int k = 0; k < 32; k += 2) {
      acc0 = fma(lv[k], __shfl_sync(0xffffffffu, yv, k), acc0);
      acc1 = fma(lv[k + 1], __shfl_sync(0xffffffffu, yv, k + 1), acc1);
    }
    if (lane < w) st_release_dbl(x + r0 + lane, acc0 + acc1);
    return;
  }
  const double rdg = 1.0 / dg;  // off the dependency chain below (x * (1/d): <= 1 ulp from x / d)
  if (LOWER) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double xk = __shfl_sync(0xffffffffu, yv, k);
      if (lane > k) yv = fma(-lv[k], xk, yv);
    }
  } else {
#pragma unroll
    for (int k = 31; k >= 0; --k) {
      if (lane == k && lane < w) yv = yv * rdg;
      const double xk = __shfl_sync(0xffffffffu, yv, k);
      if (lane < k) yv = fma(-lv[k], xk, yv);
    }
  }
  if (lane < w) st_release_dbl(x + r0 + lane, yv);
}

// Task kinds: 0 = whole block (outside + dense), 1 = helper (outside sums of rows
// [rb, rb+rc) of a heavy block -> ysum, sentinel-flagged), 2 = dense part of a heavy block
// whose outside sums come from its helpers (scheduled right before it), 3 = batch of up to
// kSnWarps independent small blocks of one level, warp k solving member rb+k (member
// entries live past the task list in the same arrays).
// optional per-task timeline (hn_debug_sptrsv_trace): [start, outside-done, end] ns + SM id
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

template <bool LOWER>
__global__ void __launch_bounds__(kSnThreads) sptrsv_super_kernel(
    const int* __restrict__ blk_kind, const int* __restrict__ blk_r0, const int* __restrict__ blk_w,
    const int* __restrict__ blk_rb, const int* __restrict__ blk_rc, int64_t nblk, const int64_t* __restrict__ rowptr,
    const int* __restrict__ cols, const double* __restrict__ vals, const double* __restrict__ diag,
    const double* __restrict__ tinv, const double* __restrict__ b, double* x, double* ysum,
    unsigned long long* ticket) {
  __shared__ double ys[kSnMaxW];
  __shared__ unsigned long long tk;
  extern __shared__ double sn_nbuf[];  // [32][kSnThreads]: the next tile's entries (cp.async)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  while (true) {
    if (tid == 0) tk = atomicAdd(ticket, 1ull);
    __syncthreads();
    const unsigned long long t = tk;
    __syncthreads();
    if (t >= static_cast<unsigned long long>(nblk)) return;
    unsigned long long* tr = g_sn_trace;
    if (tr && tid == 0) {
      tr[4 * t] = gtime();
      tr[4 * t + 3] = smid();
    }
    const int kind = __ldg(blk_kind + t);
    if (kind == 3) {
      const int mb = __ldg(blk_rb + t), mc = __ldg(blk_rc + t);
      if (warp < mc)
        warp_small_block<LOWER>(rowptr, cols, vals, diag, tinv, b, x, __ldg(blk_r0 + mb + warp), __ldg(blk_w + mb + warp),
                                lane);
      if (tr) {
        __syncthreads();
        if (tid == 0) tr[4 * t + 2] = gtime();
      }
      continue;
    }
    const int r0 = __ldg(blk_r0 + t), w = __ldg(blk_w + t);
    if (kind == 2) {
      for (int rr = tid; rr < w; rr += kSnThreads) ys[rr] = wait_value(ysum + r0 + rr);
    } else {
      // (1) outside contributions, warp per row
      const int rb = kind == 1 ? __ldg(blk_rb + t) : 0;
      const int re = kind == 1 ? rb + __ldg(blk_rc + t) : w;
      for (int rr = rb + warp; rr < re; rr += kSnWarps) {
        const int i = r0 + rr;
        const int64_t a = __ldg(rowptr + i), z = __ldg(rowptr + i + 1);
        const int inside = LOWER ? rr : (w - 1 - rr);
        const int64_t e0 = LOWER ? a : a + inside;
        const int len = static_cast<int>(z - a) - inside;
        const double s = row_outside_sum(cols, vals, e0, len, x, lane);
        if (lane == 0) {
          if (kind == 1) st_release_dbl(ysum + i, __ldg(b + i) - s);
          else ys[rr] = __ldg(b + i) - s;
        }
      }
      if (kind == 1) {
        if (tr) {
          __syncthreads();
          if (tid == 0) tr[4 * t + 2] = gtime();
        }
        continue;
      }
    }
    __syncthreads();
    if (tr && tid == 0) tr[4 * t + 1] = gtime();
    // (2) dense in-block triangle, 32-column tiles
    const int ntiles = (w + 31) / 32;
    if (w <= kSnThreads) {
      // thread tid owns block row tid: it loads its 32 entries of the next tile while the
      // current tile is solved (the diagonal tile by the warp that owns its rows, lane =
      // row - t0), so the apply of a tile never waits on memory; same arithmetic and order
      const bool has = tid < w;
      const int i = r0 + tid;
      const int64_t ra = has ? __ldg(rowptr + i) : 0, rz = has ? __ldg(rowptr + i + 1) : 0;
      auto tile_t0 = [&](int tt) { return LOWER ? 32 * tt : 32 * (ntiles - 1 - tt); };
      auto load_tile = [&](int t0, double* v) {
        const int tw = min(32, w - t0);
        const bool own = tinv && has && tid >= t0 && tid < t0 + tw;  // my diagonal tile: its inverse
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int c = t0 + k;
          const bool ok = has && k < tw && (LOWER ? c < tid : c > tid);
          v[k] = own ? (k < tw ? __ldg(tinv + static_cast<int64_t>(i) * 32 + k) : 0.0)
                     : (ok ? __ldg(vals + (LOWER ? (rz - tid) + c : ra + (c - tid - 1))) : 0.0);
        }
      };
      // the next tile goes to shared memory by cp.async (thread tid only touches column tid,
      // so no barrier guards it): no registers held for it across the tile
      auto prefetch_tile = [&](int t0) {
        const int tw = min(32, w - t0);
        const bool own = tinv && has && tid >= t0 && tid < t0 + tw;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int c = t0 + k;
          const bool ok = has && k < tw && (LOWER ? c < tid : c > tid);
          double* dst = sn_nbuf + k * kSnThreads + tid;
          const double* src = own ? (k < tw ? tinv + static_cast<int64_t>(i) * 32 + k : nullptr)
                                  : (ok ? vals + (LOWER ? (rz - tid) + c : ra + (c - tid - 1)) : nullptr);
          if (src) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<unsigned>(
                             __cvta_generic_to_shared(dst))), "l"(src) : "memory");
          } else {
            *dst = 0.0;
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      double cur[32];
      load_tile(tile_t0(0), cur);
      for (int tt = 0; tt < ntiles; ++tt) {
        const int t0 = tile_t0(tt);
        const int tw = min(32, w - t0);
        if (tt + 1 < ntiles) prefetch_tile(tile_t0(tt + 1));
        if (warp == t0 / 32 && tinv) {  // x = T^-1 y, no dependency chain
          const double yv = lane < tw ? ys[tid] : 0.0;
          double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
          for (int k = 0; k < 32; k += 2) {
            acc0 = fma(cur[k], __shfl_sync(0xffffffffu, yv, k), acc0);
            acc1 = fma(cur[k + 1], __shfl_sync(0xffffffffu, yv, k + 1), acc1);
          }
          if (lane < tw) {
            ys[tid] = acc0 + acc1;
            st_release_dbl(x + i, acc0 + acc1);
          }
        } else if (warp == t0 / 32) {  // the diagonal tile's rows: lane = row - t0
          double yv = lane < tw ? ys[tid] : 0.0;
          const double dg = (!LOWER && lane < tw) ? __ldg(diag + i) : 1.0;
          const double rdg = 1.0 / dg;
          if (LOWER) {
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              const double xk = __shfl_sync(0xffffffffu, yv, k);
              if (lane > k) yv = fma(-cur[k], xk, yv);
            }
          } else {
#pragma unroll
            for (int k = 31; k >= 0; --k) {
              if (lane == k && lane < tw) yv = yv * rdg;
              const double xk = __shfl_sync(0xffffffffu, yv, k);
              if (lane < k) yv = fma(-cur[k], xk, yv);
            }
          }
          if (lane < tw) {
            ys[tid] = yv;
            st_release_dbl(x + i, yv);
          }
        }
        __syncthreads();
        if (has && (LOWER ? tid >= t0 + tw : tid < t0)) {  // apply the solved tile to my row
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (k < tw) acc = fma(cur[k], ys[t0 + k], acc);
          ys[tid] -= acc;
        }
        __syncthreads();
        if (tt + 1 < ntiles) {
          asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
          for (int k = 0; k < 32; ++k) cur[k] = sn_nbuf[k * kSnThreads + tid];
        }
      }
      if (tr && tid == 0) tr[4 * t + 2] = gtime();
      continue;
    }
    for (int tt = 0; tt < ntiles; ++tt) {
      const int t0 = LOWER ? 32 * tt : 32 * (ntiles - 1 - tt);  // first block row of the tile
      const int tw = min(32, w - t0);
      if (warp == (tt % kSnWarps)) {
        const int rr = t0 + lane;
        double yv = lane < tw ? ys[rr] : 0.0;
        const int i = r0 + rr;
        // this lane's row entries inside the diagonal tile
        double lv[32];
        if (lane < tw) {
          const int64_t a = __ldg(rowptr + i), z = __ldg(rowptr + i + 1);
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            double val = 0.0;
            if (LOWER) {
              if (k < lane) val = __ldg(vals + (z - rr) + t0 + k);           // col r0 + t0 + k
            } else {
              if (k > lane && k < tw) val = __ldg(vals + a + (t0 + k - rr - 1));  // col r0 + t0 + k
            }
            lv[k] = val;
          }
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) lv[k] = 0.0;
        }
        const double dg = (!LOWER && lane < tw) ? __ldg(diag + i) : 1.0;
        const double rdg = 1.0 / dg;
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
        if (lane < tw) {
          ys[rr] = yv;
          st_release_dbl(x + i, yv);
        }
      }
      __syncthreads();
      // apply the solved tile to the rows not yet solved
      const int lo = LOWER ? t0 + tw : 0;
      const int hi = LOWER ? w : t0;
      for (int rr = lo + tid; rr < hi; rr += kSnThreads) {
        const int i = r0 + rr;
        double acc = 0.0;
        if (LOWER) {
          const double* rowv = vals + (__ldg(rowptr + i + 1) - rr) + t0;  // cols r0+t0 ..
          for (int k = 0; k < tw; ++k) acc = fma(__ldg(rowv + k), ys[t0 + k], acc);
        } else {
          const double* rowv = vals + __ldg(rowptr + i) + (t0 - rr - 1);     // col r0+t0+k at +k
          for (int k = 0; k < tw; ++k) acc = fma(__ldg(rowv + k), ys[t0 + k], acc);
        }
        ys[rr] -= acc;
      }
      __syncthreads();
    }
    if (tr && tid == 0) tr[4 * t + 2] = gtime();
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

HN_EXPORT int hn_sptrsv(int lower, const int64_t* rowptr, const int* cols, const double* vals, const double* diag,
                        const double* b, double* x, int64_t n, unsigned long long* ticket, void* stream) {
  if (n == 0) return 0;
  cudaStream_t s = as_stream(stream);
  HN_TRY(cudaMemsetAsync(x, 0xFF, sizeof(double) * n, s));
  HN_TRY(cudaMemsetAsync(ticket, 0, sizeof(unsigned long long), s));
  const int blocks = sm_count() * 4;  // 8 warps per block -> 32 resident rows per SM
  if (lower) sptrsv_kernel<true><<<blocks, 256, 0, s>>>(rowptr, cols, vals, diag, b, x, n, ticket);
  else sptrsv_kernel<false><<<blocks, 256, 0, s>>>(rowptr, cols, vals, diag, b, x, n, ticket);
  HN_CHECK_LAUNCH();
  return 0;
}

// Scheduled sync-free solve (see sptrsv_tasks_kernel).  divide != 0: x_row /= diag[row].
// x (n) and partial (npartial) are reset to the sentinel here; warps_per_sm resident warps.
HN_EXPORT int hn_sptrsv_tasks(int divide, const int* task_row, const int64_t* task_beg, const int* task_len,
                              const int* task_part, const int* task_np, int64_t ntasks, const int* cols,
                              const double* vals, const double* diag, const double* b, double* x, int64_t n,
                              double* partial, int64_t npartial, unsigned long long* ticket, int warps_per_sm,
                              void* stream) {
  if (ntasks == 0) return 0;
  cudaStream_t s = as_stream(stream);
  HN_TRY(cudaMemsetAsync(x, 0xFF, sizeof(double) * n, s));
  if (npartial > 0) HN_TRY(cudaMemsetAsync(partial, 0xFF, sizeof(double) * npartial, s));
  HN_TRY(cudaMemsetAsync(ticket, 0, sizeof(unsigned long long), s));
  const int wps = warps_per_sm > 0 ? warps_per_sm : 16;
  const int blocks = sm_count() * ((wps + 7) / 8);
  if (divide)
    sptrsv_tasks_kernel<true><<<blocks, 256, 0, s>>>(task_row, task_beg, task_len, task_part, task_np, ntasks, cols,
                                                     vals, diag, b, x, partial, ticket);
  else
    sptrsv_tasks_kernel<false><<<blocks, 256, 0, s>>>(task_row, task_beg, task_len, task_part, task_np, ntasks, cols,
                                                      vals, diag, b, x, partial, ticket);
  HN_CHECK_LAUNCH();
  return 0;
}

// Debug timeline for hn_sptrsv_super: trace = 4 x ntasks u64 per launch (NULL = off).
HN_EXPORT int hn_debug_sptrsv_trace(unsigned long long* trace) {
  return cudaMemcpyToSymbol(g_sn_trace, &trace, sizeof(trace)) == cudaSuccess ? 0 : -1;
}

// Supernodal solve over planned blocks (processing order), see sptrsv_super_kernel.
HN_EXPORT int hn_sptrsv_super_inv(int lower, const int* blk_kind, const int* blk_r0, const int* blk_w,
                                  const int* blk_rb, const int* blk_rc, int64_t nblk, const int64_t* rowptr,
                                  const int* cols, const double* vals, const double* diag, const double* tinv,
                                  const double* b, double* x, double* ysum, int64_t n, unsigned long long* ticket,
                                  int ctas_per_sm, void* stream);

HN_EXPORT int hn_sptrsv_super(int lower, const int* blk_kind, const int* blk_r0, const int* blk_w, const int* blk_rb,
                              const int* blk_rc, int64_t nblk, const int64_t* rowptr, const int* cols,
                              const double* vals, const double* diag, const double* b, double* x, double* ysum,
                              int64_t n, unsigned long long* ticket, int ctas_per_sm, void* stream) {
  return hn_sptrsv_super_inv(lower, blk_kind, blk_r0, blk_w, blk_rb, blk_rc, nblk, rowptr, cols, vals, diag, nullptr,
                             b, x, ysum, n, ticket, ctas_per_sm, stream);
}

// As hn_sptrsv_super; tinv (n x 32, or NULL) holds, for every row, its row of the inverse of
// its 32-row diagonal tile (hn_host_tile_inverse): the in-tile triangle is then one
// matrix-vector product instead of a 32-step substitution chain.
HN_EXPORT int hn_sptrsv_super_inv(int lower, const int* blk_kind, const int* blk_r0, const int* blk_w,
                                  const int* blk_rb, const int* blk_rc, int64_t nblk, const int64_t* rowptr,
                                  const int* cols, const double* vals, const double* diag, const double* tinv,
                                  const double* b, double* x, double* ysum, int64_t n, unsigned long long* ticket,
                                  int ctas_per_sm, void* stream) {
  if (nblk == 0) return 0;
  cudaStream_t s = as_stream(stream);
  HN_TRY(cudaMemsetAsync(x, 0xFF, sizeof(double) * n, s));
  HN_TRY(cudaMemsetAsync(ysum, 0xFF, sizeof(double) * n, s));
  HN_TRY(cudaMemsetAsync(ticket, 0, sizeof(unsigned long long), s));
  const int blocks = sm_count() * (ctas_per_sm > 0 ? ctas_per_sm : 2);
  constexpr int kNbuf = 32 * kSnThreads * static_cast<int>(sizeof(double));  // next-tile buffer
  // per-device function attribute: set on every call (cheap), so any device a process drives
  // gets the opt-in
  HN_TRY(cudaFuncSetAttribute(sptrsv_super_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kNbuf));
  HN_TRY(cudaFuncSetAttribute(sptrsv_super_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kNbuf));
  if (lower)
    sptrsv_super_kernel<true><<<blocks, kSnThreads, kNbuf, s>>>(blk_kind, blk_r0, blk_w, blk_rb, blk_rc, nblk, rowptr, cols,
                                                            vals, diag, tinv, b, x, ysum, ticket);
  else
    sptrsv_super_kernel<false><<<blocks, kSnThreads, kNbuf, s>>>(blk_kind, blk_r0, blk_w, blk_rb, blk_rc, nblk, rowptr,
                                                             cols, vals, diag, tinv, b, x, ysum, ticket);
  HN_CHECK_LAUNCH();
  return 0;
}

// Host helper (setup): inverses of the 32-row diagonal tiles of every block [r0, r0+w)
// (tiles start at r0, r0+32, ..; the last one may be narrower), as hn_sptrsv_super_inv
// reads them: tinv[i*32 + k] = row (i - tile start) of T^-1, column k.  T = I + the strict
// lower in-tile entries (lower) or diag + the strict upper in-tile entries (upper); the
// inverse by substitution on the identity columns.  tinv must hold n*32 doubles.
HN_EXPORT int hn_host_tile_inverse(const int64_t* rowptr, const int* cols, const double* vals, const double* diag,
                                   int64_t n, int lower, int64_t nb, const int* r0, const int* w, double* tinv) {
  for (int64_t q = 0; q < n * 32; ++q) tinv[q] = 0.0;
  double T[32][32], X[32][32];
  for (int64_t blk = 0; blk < nb; ++blk) {
    for (int t0 = 0; t0 < w[blk]; t0 += 32) {
      const int tw = w[blk] - t0 < 32 ? w[blk] - t0 : 32;
      const int64_t base = static_cast<int64_t>(r0[blk]) + t0;
      for (int l = 0; l < tw; ++l)
        for (int k = 0; k < tw; ++k) T[l][k] = 0.0;
      for (int l = 0; l < tw; ++l) {
        const int64_t i = base + l;
        T[l][l] = lower ? 1.0 : diag[i];
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
          const int64_t c = cols[e];
          if (c >= base && c < base + tw && (lower ? c < i : c > i)) T[l][c - base] = vals[e];
        }
      }
      for (int j = 0; j < tw; ++j) {  // column j of X = T^-1
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
        for (int k = 0; k < tw; ++k) tinv[(base + l) * 32 + k] = X[l][k];
    }
  }
  return 0;
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

// Host helper (setup): dependency level of every row of a triangular CSR, sweeping rows in
// increasing (lower != 0) or decreasing order.  Host pointers.
HN_EXPORT int hn_host_levels(const int64_t* rowptr_host, const int* cols_host, int64_t n, int lower,
                             int* levels_host) {
  for (int64_t k = 0; k < n; ++k) {
    const int64_t i = lower ? k : n - 1 - k;
    int lev = 0;
    for (int64_t e = rowptr_host[i]; e < rowptr_host[i + 1]; ++e) {
      const int l = levels_host[cols_host[e]] + 1;
      lev = l > lev ? l : lev;
    }
    levels_host[i] = lev;
  }
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
