// K1-K3: cell-list k-nearest-neighbour stencil builder, method classification
// and lattice (MON) stencils.
//
// Reference behaviour reproduced bit for bit:
//   * _knn_sorted (pkg/src/hybridnodes/approx.py:133-146): the n smallest nodes by the
//     lexicographic key (fl-distance, node index); the reference widens its cKDTree
//     query until no tie straddles the cutoff, then lexsorts (idx, d) -- which is
//     exactly "top n by (d, idx)".  fl-distance = fl(sqrt((0+dx^2)+dy^2[+dz^2])).
//   * _boundary_stencils with `exclude` (approx.py:416-431): [self] + the size-1
//     nearest non-excluded nodes; the reference does not widen there, so on an
//     exact tie straddling the cutoff its choice follows cKDTree traversal order.
//     We return the (d, idx) choice plus distances so the host can flag those rows
//     (SURVEY §8(a) A5).
//   * classify_methods (approx.py:332-357) lattice path and _mon_stencils
//     (approx.py:360-376): MON iff regular, on-lattice and all 2d axis keys occupied;
//     stencil = [centre] + axis neighbours sorted by (np.linalg.norm, index).
//
// Design: uniform cell grid (count -> scan -> scatter, positions re-packed in cell
// order), then one thread per query scanning Chebyshev rings of cells until the
// current n-th key is strictly closer than any unscanned cell.  The running top-n
// lives in registers: a sorted window of the last n slots of an NMAX array whose
// prefix holds -inf sentinels, so the insertion network has compile-time indices.
#include <cfloat>
#include <climits>
#include <math_constants.h>

#include "hn_common.cuh"

namespace hn {

struct Grid {
  double lo[3];
  double cell;
  double inv_cell;
  int dims[3];
};

template <int D>
__device__ __forceinline__ void cell_coords(const Grid& g, const double* p, int* c) {
#pragma unroll
  for (int a = 0; a < D; ++a) {
    int v = static_cast<int>(floor((p[a] - g.lo[a]) * g.inv_cell));
    c[a] = min(max(v, 0), g.dims[a] - 1);
  }
}

template <int D>
__device__ __forceinline__ int64_t cell_linear(const Grid& g, const int* c) {
  int64_t l = c[0];
#pragma unroll
  for (int a = 1; a < D; ++a) l = l * g.dims[a] + c[a];
  return l;
}

template <int D>
__global__ void cell_count_kernel(Grid g, const double* __restrict__ pos, int64_t n, int* __restrict__ count,
                                  int* __restrict__ point_cell) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[D];
  load_point<D>(pos, i, p);
  int c[D];
  cell_coords<D>(g, p, c);
  int64_t l = cell_linear<D>(g, c);
  point_cell[i] = static_cast<int>(l);
  atomicAdd(count + l, 1);
}

template <int D>
__global__ void cell_scatter_kernel(const double* __restrict__ pos, int64_t n, const int* __restrict__ point_cell,
                                    const int* __restrict__ cell_start, int* __restrict__ fill,
                                    int* __restrict__ cell_items, double* __restrict__ cell_pos) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = point_cell[i];
  int slot = cell_start[c] + atomicAdd(fill + c, 1);
  cell_items[slot] = static_cast<int>(i);
  constexpr int S = pos_stride<D>();
#pragma unroll
  for (int a = 0; a < S; ++a) cell_pos[static_cast<int64_t>(slot) * S + a] = pos[i * S + a];
}

// ---- exclusive scan (int32) -------------------------------------------------------
constexpr int kScanThreads = 512;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int block_exclusive_scan(int v, int* smem, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < (blockDim.x >> 5) ? smem[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    smem[lane] = s;
  }
  __syncthreads();
  int warp_off = wid > 0 ? smem[wid - 1] : 0;
  *total = smem[(blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_off + x - v;
}

__global__ void scan_tile_sums(const int* __restrict__ in, int64_t n, int* __restrict__ tile_sums) {
  __shared__ int smem[32];
  int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < n) s += in[base + k];
  int total;
  block_exclusive_scan(s, smem, &total);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

__global__ void scan_tiles_serial(int* __restrict__ tile_sums, int64_t ntiles) {
  __shared__ int smem[32];
  int carry = 0;
  for (int64_t base = 0; base < ntiles; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    int v = i < ntiles ? tile_sums[i] : 0;
    int total;
    int ex = block_exclusive_scan(v, smem, &total);
    if (i < ntiles) tile_sums[i] = carry + ex;
    carry += total;
  }
}

__global__ void scan_tiles_apply(const int* __restrict__ in, int64_t n, const int* __restrict__ tile_off,
                                 int* __restrict__ out) {
  __shared__ int smem[32];
  int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  int v[kScanItems];
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? in[base + k] : 0;
    s += v[k];
  }
  int total;
  int ex = block_exclusive_scan(s, smem, &total) + tile_off[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = ex;
    ex += v[k];
  }
  // out[n] = grand total, written by the thread owning the last element
  if (base <= n - 1 && n - 1 < base + kScanItems) out[n] = ex;
}

// Exclusive scan of n ints into out[0..n] (out[n] = total). Scratch from the stream allocator.
int exclusive_scan(const int* in, int64_t n, int* out, cudaStream_t s) {
  int64_t ntiles = ceil_div(n, kScanTile);
  int* tiles = nullptr;
  HN_TRY(stream_alloc(reinterpret_cast<void**>(&tiles), sizeof(int) * (ntiles + 1), s));
  scan_tile_sums<<<ntiles, kScanThreads, 0, s>>>(in, n, tiles);
  scan_tiles_serial<<<1, 1024, 0, s>>>(tiles, ntiles);
  scan_tiles_apply<<<ntiles, kScanThreads, 0, s>>>(in, n, tiles, out);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(tiles, s);
  return e == cudaSuccess ? 0 : -static_cast<int>(e);
}

// ---- kNN query ------------------------------------------------------------------
__device__ __forceinline__ bool key_less(double da, int ia, double db, int ib) {
  return da < db || (da == db && ia < ib);
}

// running top-n: sorted ascending in the last n slots of kd/ki; slots [0, NMAX-n) hold
// -inf sentinels that are never displaced, so the network has compile-time indices
template <int NMAX>
__device__ __forceinline__ void topn_init(double* kd, int* ki, int n) {
#pragma unroll
  for (int j = 0; j < NMAX; ++j) {
    const bool live = j >= NMAX - n;
    kd[j] = live ? CUDART_INF : -CUDART_INF;
    ki[j] = live ? INT_MAX : -1;
  }
}

// one candidate (node j at p) against the running top-n
template <int D, int NMAX>
__device__ __forceinline__ void topn_offer_pt(const uint8_t* __restrict__ exclude, int j, const double* p,
                                              const double* q, double* kd, int* ki, double& thr2) {
  if (exclude && __ldg(exclude + j)) return;
  const double d2 = exact_dist2<D>(p, q);
  if (d2 > thr2) return;
  const double d = __dsqrt_rn(d2);
  if (!key_less(d, j, kd[NMAX - 1], ki[NMAX - 1])) return;
#pragma unroll
  for (int m = NMAX - 1; m >= 0; --m) {
    if (key_less(d, j, kd[m], ki[m])) {
      const bool shift = (m > 0) && key_less(d, j, kd[m > 0 ? m - 1 : 0], ki[m > 0 ? m - 1 : 0]);
      kd[m] = shift ? kd[m > 0 ? m - 1 : 0] : d;
      ki[m] = shift ? ki[m > 0 ? m - 1 : 0] : j;
    }
  }
  const double w = kd[NMAX - 1];
  if (w != CUDART_INF) thr2 = fmin(thr2, __dmul_rn(__dmul_rn(w, w), 1.0 + 1e-15));
}

template <int D>
__device__ __forceinline__ void load_cand(const double* __restrict__ cell_pos, const int* __restrict__ cell_items,
                                          int s, int& j, double* p) {
  constexpr int S = pos_stride<D>();
  j = __ldg(cell_items + s);
#pragma unroll
  for (int a = 0; a < D; ++a) p[a] = __ldg(cell_pos + static_cast<int64_t>(s) * S + a);
}

// point s of the cell-ordered arrays against the running top-n
template <int D, int NMAX>
__device__ __forceinline__ void topn_offer(const double* __restrict__ cell_pos, const int* __restrict__ cell_items,
                                           const uint8_t* __restrict__ exclude, int s, const double* q,
                                           double* kd, int* ki, double& thr2) {
  int j;
  double p[D];
  load_cand<D>(cell_pos, cell_items, s, j, p);
  topn_offer_pt<D, NMAX>(exclude, j, p, q, kd, ki, thr2);
}

// a contiguous run [beg, end) with the next candidate's loads issued before the current
// one is offered (the offer's compare/insert chain no longer waits on each load)
template <int D, int NMAX>
__device__ __forceinline__ void topn_offer_run(const double* __restrict__ cell_pos,
                                               const int* __restrict__ cell_items,
                                               const uint8_t* __restrict__ exclude, int beg, int end,
                                               const double* q, double* kd, int* ki, double& thr2) {
  if constexpr (D == 2) {  // 2D runs are short (~6 points): the extra registers cost more
    for (int s = beg; s < end; ++s) topn_offer<D, NMAX>(cell_pos, cell_items, exclude, s, q, kd, ki, thr2);
    return;
  }
  if (beg >= end) return;
  int jn;
  double pn[D];
  load_cand<D>(cell_pos, cell_items, beg, jn, pn);
  for (int s = beg; s < end; ++s) {
    const int j = jn;
    double p[D];
#pragma unroll
    for (int a = 0; a < D; ++a) p[a] = pn[a];
    if (s + 1 < end) load_cand<D>(cell_pos, cell_items, s + 1, jn, pn);
    topn_offer_pt<D, NMAX>(exclude, j, p, q, kd, ki, thr2);
  }
}

// Chebyshev rings of cells around the query cell until the current n-th key is strictly
// closer than any unscanned cell (exact for any grid, any density)
template <int D, int NMAX>
__device__ __forceinline__ void ring_scan(const Grid& g, const int* __restrict__ cell_start, const int* __restrict__ cell_items,
                          const double* __restrict__ cell_pos, const uint8_t* __restrict__ exclude,
                          const double* q, const int* c0, double* kd, int* ki) {
  double thr2 = CUDART_INF;  // d2 above this cannot enter the window
  int max_r = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) max_r = max(max_r, max(c0[a], g.dims[a] - 1 - c0[a]));
  for (int R = 0; R <= max_r; ++R) {
    const int lo1 = -R, hi1 = R;
    for (int o0 = -R; o0 <= R; ++o0) {
      const int x = c0[0] + o0;
      if (x < 0 || x >= g.dims[0]) continue;
      const bool edge0 = (o0 == -R || o0 == R);
      const int o2lo = (D == 3) ? -R : 0, o2hi = (D == 3) ? R : 0;
      for (int o2 = o2lo; o2 <= o2hi; ++o2) {
        int z = 0;
        bool edge2 = false;
        if constexpr (D == 3) {
          z = c0[2] + o2;
          if (z < 0 || z >= g.dims[2]) continue;
          edge2 = (o2 == -R || o2 == R);
        }
        const bool full = edge0 || edge2;
        const int step1 = full ? 1 : (hi1 - lo1 > 0 ? hi1 - lo1 : 1);
        for (int o1 = lo1; o1 <= hi1; o1 += step1) {
          const int y = c0[1] + o1;
          if (y < 0 || y >= g.dims[1]) continue;
          int64_t cl = static_cast<int64_t>(x) * g.dims[1] + y;
          if constexpr (D == 3) cl = cl * g.dims[2] + z;
          const int beg = __ldg(cell_start + cl), end = __ldg(cell_start + cl + 1);
          for (int s = beg; s < end; ++s) topn_offer<D, NMAX>(cell_pos, cell_items, exclude, s, q, kd, ki, thr2);
        }
      }
    }
    // distance from q to the nearest face of the scanned block that has cells beyond it
    double bound = CUDART_INF;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      if (c0[a] - R > 0) bound = fmin(bound, q[a] - (g.lo[a] + (c0[a] - R) * g.cell));
      if (c0[a] + R + 1 < g.dims[a]) bound = fmin(bound, (g.lo[a] + (c0[a] + R + 1) * g.cell) - q[a]);
    }
    if (kd[NMAX - 1] < bound - 1e-9 * g.cell) break;
  }
}

template <int D>
__device__ __forceinline__ void load_query(const double* __restrict__ pos, const int* __restrict__ queries,
                                           const double* __restrict__ qpos, int64_t t, double* q) {
  if (qpos) {
    load_point<D>(qpos, t, q);
  } else {
    const int qi = queries ? __ldg(queries + t) : static_cast<int>(t);
    load_point<D>(pos, qi, q);
  }
}

template <int NMAX>
__device__ __forceinline__ void topn_store(const double* kd, const int* ki, int n, int64_t t, int* out_idx,
                                           double* out_dist) {
#pragma unroll
  for (int j = 0; j < NMAX; ++j) {
    if (j >= NMAX - n) {
      const int o = j - (NMAX - n);
      out_idx[t * n + o] = ki[j];
      if (out_dist) out_dist[t * n + o] = kd[j];
    }
  }
}

template <int D, int NMAX>
__global__ void __launch_bounds__(128) knn_kernel(Grid g, const double* __restrict__ pos,
                                                  const int* __restrict__ cell_start,
                                                  const int* __restrict__ cell_items,
                                                  const double* __restrict__ cell_pos,
                                                  const int* __restrict__ queries,
                                                  const double* __restrict__ qpos, int64_t nq, int n,
                                                  const uint8_t* __restrict__ exclude,
                                                  int* __restrict__ out_idx, double* __restrict__ out_dist) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nq) return;
  double q[D];
  load_query<D>(pos, queries, qpos, t, q);
  int c0[D];
  cell_coords<D>(g, q, c0);
  double kd[NMAX];
  int ki[NMAX];
  topn_init<NMAX>(kd, ki, n);
  ring_scan<D, NMAX>(g, cell_start, cell_items, cell_pos, exclude, q, c0, kd, ki);
  topn_store<NMAX>(kd, ki, n, t, out_idx, out_dist);
}

// ---- kNN query, box pass ------------------------------------------------------------
// Same result as knn_kernel.  First pass: every point within the axis box |p - q|_inf <=
// r0 (r0 ~ 1.3x the expected n-th distance, from the grid's points per cell), scanned as
// contiguous runs of cells along the grid's fastest axis (one cell_start pair per run
// instead of per cell) in rows ordered outward from the query, with only d <= r0
// admitted.  If the n-th key ends within r0 (1 - 1e-12) the result is exact: every point
// with a smaller key lies inside the box and passed the admission test.  Otherwise the
// query restarts with the exact ring traversal (sparse corners, excluded regions).
template <int D, int NMAX>
__global__ void __launch_bounds__(128, D == 2 ? 7 : 5) knn_box_kernel(Grid g, const double* __restrict__ pos,
                                                      const int* __restrict__ cell_start,
                                                      const int* __restrict__ cell_items,
                                                      const double* __restrict__ cell_pos,
                                                      const int* __restrict__ queries,
                                                      const double* __restrict__ qpos, int64_t nq, int n,
                                                      const uint8_t* __restrict__ exclude, double r0,
                                                      const double* __restrict__ qh, double rscale,
                                                      int* __restrict__ out_idx, double* __restrict__ out_dist,
                                                      const int* __restrict__ nq_dev = nullptr,
                                                      const int* __restrict__ out_rows = nullptr) {
  // nq_dev / out_rows: the warp kernel's fallback list (count on the device, query t of the
  // list is output row out_rows[t]); grid-stride so a fixed grid covers any count
  const int64_t nq_eff = nq_dev ? static_cast<int64_t>(*nq_dev) : nq;
  const double r_base = r0;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < nq_eff;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
  r0 = r_base;
  double q[D];
  load_query<D>(pos, queries, qpos, t, q);
  if (qh) {  // radius from the query's own nominal spacing (graded node sets)
    const double h = __ldg(qh + (qpos ? t : (queries ? __ldg(queries + t) : t)));
    if (h > 0.0 && h < CUDART_INF) r0 = rscale * h;
  }
  int c0[D];
  cell_coords<D>(g, q, c0);
  double kd[NMAX];
  int ki[NMAX];
  topn_init<NMAX>(kd, ki, n);
  constexpr int L = D - 1;  // contiguous axis of the cell numbering
  // gap between q and cell c along axis a (0 inside), shrunk by a rounding margin
  auto gap = [&](int a, int c) {
    const double cl = g.lo[a] + c * g.cell;
    const double gp = fmax(fmax(cl - q[a], q[a] - (cl + g.cell)), 0.0);
    return fmax(gp - 1e-9 * g.cell, 0.0);
  };
  bool exact = false;
#pragma unroll 1
  for (int attempt = 0; attempt < 2 && !exact; ++attempt) {
    const double r = attempt ? 1.7 * r0 : r0;  // one wider retry before the ring fallback
    if (attempt) topn_init<NMAX>(kd, ki, n);
    double thr2 = __dmul_rn(__dmul_rn(r, r), 1.0 + 1e-9);
    // box cells with cell_coords' own formula: fl(sub), fl(mul) and floor are monotone, so
    // every point whose coordinate lies in [q - r', q + r'] falls in [blo, bhi]
    const double rm = r * (1.0 + 1e-9);
    int blo[D], bhi[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double lo_p = q[a] - rm, hi_p = q[a] + rm;
      blo[a] = min(max(static_cast<int>(floor((lo_p - g.lo[a]) * g.inv_cell)), 0), g.dims[a] - 1);
      bhi[a] = min(max(static_cast<int>(floor((hi_p - g.lo[a]) * g.inv_cell)), 0), g.dims[a] - 1);
    }
    // cells of the run along the contiguous axis that can hold points within sqrt(rem2)
    // of q (rem2 = thr2 minus the squared gaps of the other axes; thr2 shrinks as the
    // window fills, so later runs get shorter)
    auto run_span = [&](double rem2, int& c_lo, int& c_hi) {
      const double hw = sqrt(fmax(rem2, 0.0)) * (1.0 + 1e-9) + 1e-12 * g.cell;
      c_lo = min(max(static_cast<int>(floor((q[L] - hw - g.lo[L]) * g.inv_cell)), blo[L]), bhi[L]);
      c_hi = min(max(static_cast<int>(floor((q[L] + hw - g.lo[L]) * g.inv_cell)), blo[L]), bhi[L]);
    };
    const int w0 = max(c0[0] - blo[0], bhi[0] - c0[0]);
    for (int k0 = 0; k0 <= 2 * w0; ++k0) {
      const int x = c0[0] + ((k0 & 1) ? -((k0 + 1) >> 1) : (k0 >> 1));
      if (x < blo[0] || x > bhi[0]) continue;
      const double gx = gap(0, x);
      if (gx * gx > thr2) continue;
      if constexpr (D == 2) {
        int ylo, yhi;
        run_span(thr2 - gx * gx, ylo, yhi);
        const int64_t cl = static_cast<int64_t>(x) * g.dims[1] + ylo;
        const int beg = __ldg(cell_start + cl), end = __ldg(cell_start + cl + (yhi - ylo + 1));
        topn_offer_run<D, NMAX>(cell_pos, cell_items, exclude, beg, end, q, kd, ki, thr2);
      } else {
        const int w1 = max(c0[1] - blo[1], bhi[1] - c0[1]);
        for (int k1 = 0; k1 <= 2 * w1; ++k1) {
          const int y = c0[1] + ((k1 & 1) ? -((k1 + 1) >> 1) : (k1 >> 1));
          if (y < blo[1] || y > bhi[1]) continue;
          const double gy = gap(1, y);
          if (gx * gx + gy * gy > thr2) continue;
          int zlo, zhi;
          run_span(thr2 - gx * gx - gy * gy, zlo, zhi);
          const int64_t cl = (static_cast<int64_t>(x) * g.dims[1] + y) * g.dims[2] + zlo;
          const int beg = __ldg(cell_start + cl), end = __ldg(cell_start + cl + (zhi - zlo + 1));
          topn_offer_run<D, NMAX>(cell_pos, cell_items, exclude, beg, end, q, kd, ki, thr2);
        }
      }
    }
    exact = kd[NMAX - 1] <= r * (1.0 - 1e-12);
  }
  if (!exact) {  // neither box held n keys (sparse corner, excluded region): exact rings
    topn_init<NMAX>(kd, ki, n);
    ring_scan<D, NMAX>(g, cell_start, cell_items, cell_pos, exclude, q, c0, kd, ki);
  }
  topn_store<NMAX>(kd, ki, n, out_rows ? static_cast<int64_t>(__ldg(out_rows + t)) : t, out_idx, out_dist);
  }
}

// ---- kNN query, one warp per query (n <= 32) ----------------------------------------
// The candidates of the query's axis box (|p - q|_inf <= r, r from the query's own nominal
// spacing) are enumerated as one flattened list over the box's cell runs (each lane owns
// one run's bounds; a warp scan gives the offsets, a 5-step search maps a list slot to its
// run), every lane takes list slots lane, lane + 32, .. and tests d^2 <= r^2; the accepted
// (d^2, index) keys are compacted by ballot into a 64-slot warp list, square-rooted once and
// sorted ONCE by a bitonic network across the lanes: 15 stages for up to 32 keys; for 33..64
// keys the two 32-key halves are sorted in opposite directions, merged in-lane (the smaller
// of each pair is one of the 32 smallest) and finished by a 5-stage bitonic merge.  No
// per-candidate insertion network, no divergence between queries.  The answer is exact when
// at most 64 keys were accepted and the n-th lies within r (1 - 1e-12): every point with a
// smaller key is in the box and was accepted.  Otherwise the query goes to a device list
// that knn_box_kernel finishes (none on config 4 at the default radius).
constexpr int kWarpKnnWarps = 8;
constexpr int kWarpKnnCap = 64;   // accepted keys a warp can sort
constexpr int kWarpKnnRuns = 64;  // cell runs of the query's box (two per lane)
#ifdef HN_TRACE
__device__ unsigned long long g_knn_fb_stats[4];  // dev builds: [fallbacks, > cap keys, < n keys, n-th beyond r]
#endif

template <int D>
__global__ void __launch_bounds__(kWarpKnnWarps * 32, 8) knn_warp_kernel(
    Grid g, const double* __restrict__ pos, const int* __restrict__ cell_start, const int* __restrict__ cell_items,
    const double* __restrict__ cell_pos, const int* __restrict__ queries, int64_t nq, int n,
    const uint8_t* __restrict__ exclude, double r0, const double* __restrict__ qh, double rscale,
    int* __restrict__ out_idx, double* __restrict__ out_dist, int* __restrict__ fb_count, int* __restrict__ fb_node,
    int* __restrict__ fb_row) {
  __shared__ int s_off[kWarpKnnWarps][kWarpKnnRuns + 1];
  __shared__ int s_beg[kWarpKnnWarps][kWarpKnnRuns];
  __shared__ double s_kd[kWarpKnnWarps][kWarpKnnCap];
  __shared__ int s_ki[kWarpKnnWarps][kWarpKnnCap];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kWarpKnnWarps + wib;
  if (t >= nq) return;
  const int node = queries ? __ldg(queries + t) : static_cast<int>(t);
  double q[D];
  load_point<D>(pos, node, q);
  double r = r0;
  if (qh) {
    const double h = __ldg(qh + node);
    if (h > 0.0 && h < CUDART_INF) r = rscale * h;
  }
  constexpr int L = D - 1;  // contiguous axis of the cell numbering
  auto gap = [&](int a, int c) {
    const double cl = g.lo[a] + c * g.cell;
    const double gp = fmax(fmax(cl - q[a], q[a] - (cl + g.cell)), 0.0);
    return fmax(gp - 1e-9 * g.cell, 0.0);
  };
  // A query whose ball holds fewer than n or more than 64 keys (next to a surface, where half
  // the ball is empty; a locally denser patch) rescans with a wider / narrower radius, up to
  // three times, bracketing: a handful of queries per million, which the thread-per-query fallback kernel
  // would otherwise serialise (4 such queries cost config 4 ~130 us).
  bool done = false;
  int why = 2;
  double r_few = 0.0, r_many = 0.0;  // bracket: radii seen with too few / too many keys
  auto shrink = [&]() {
    r_many = r;
    r = r_few > 0.0 ? sqrt(r_few * r_many) : 0.8 * r;
  };
  auto grow = [&]() {
    r_few = r;
    r = r_many > 0.0 ? sqrt(r_few * r_many) : 1.35 * r;
  };
  for (int attempt = 0; attempt < 4 && !done; ++attempt) {
    __syncwarp();
    const double thr2 = __dmul_rn(__dmul_rn(r, r), 1.0 + 1e-9);
    const double rm = r * (1.0 + 1e-9);
    int blo[D], bhi[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      blo[a] = min(max(static_cast<int>(floor((q[a] - rm - g.lo[a]) * g.inv_cell)), 0), g.dims[a] - 1);
      bhi[a] = min(max(static_cast<int>(floor((q[a] + rm - g.lo[a]) * g.inv_cell)), 0), g.dims[a] - 1);
    }
    const int nx = bhi[0] - blo[0] + 1;
    const int nrows = D == 2 ? nx : nx * (bhi[1] - blo[1] + 1);
    if (nrows > kWarpKnnRuns) {
      why = 1;
      shrink();
      continue;
    }
    // lane -> up to two runs of cells along the contiguous axis (rows lane and lane + 32 of
    // the box), each clipped to the ball
    int beg[2] = {0, 0}, cnt[2] = {0, 0};
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int row = lane + 32 * b;
      if (row < nrows) {
        const int x = blo[0] + (D == 2 ? row : row % nx);
        double rem2 = thr2;
        const double gx = gap(0, x);
        rem2 -= gx * gx;
        int64_t cl = x;
        if constexpr (D == 3) {
          const int y = blo[1] + row / nx;
          const double gy = gap(1, y);
          rem2 -= gy * gy;
          cl = static_cast<int64_t>(x) * g.dims[1] + y;
        }
        if (rem2 >= 0.0) {
          const double hw = sqrt(rem2) * (1.0 + 1e-9) + 1e-12 * g.cell;
          const int c_lo = min(max(static_cast<int>(floor((q[L] - hw - g.lo[L]) * g.inv_cell)), blo[L]), bhi[L]);
          const int c_hi = min(max(static_cast<int>(floor((q[L] + hw - g.lo[L]) * g.inv_cell)), blo[L]), bhi[L]);
          const int64_t c0 = cl * g.dims[L] + c_lo;
          beg[b] = __ldg(cell_start + c0);
          cnt[b] = __ldg(cell_start + c0 + (c_hi - c_lo + 1)) - beg[b];
        }
      }
    }
    const bool wide = nrows > 32;  // warp-uniform
    int inc0 = cnt[0], inc1 = cnt[1];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc0, o);
      if (lane >= o) inc0 += y;
    }
    const int total0 = __shfl_sync(0xffffffffu, inc0, 31);
    int total = total0;
    if (wide) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc1, o);
        if (lane >= o) inc1 += y;
      }
      total += __shfl_sync(0xffffffffu, inc1, 31);
    }
    s_off[wib][lane] = inc0 - cnt[0];
    s_beg[wib][lane] = beg[0];
    s_off[wib][32 + lane] = wide ? total0 + inc1 - cnt[1] : total;
    s_beg[wib][32 + lane] = beg[1];
    if (lane == 31) s_off[wib][kWarpKnnRuns] = total;
    __syncwarp();
    int accepted = 0;
    for (int base = 0; base < total; base += 32) {
      const int m = base + lane;
      bool acc = false;
      double d2 = 0.0;
      int j = 0;
      if (m < total) {
        int lo = 0, hi = 31;  // last run with offset <= m (runs past nrows have offset == total)
        if (wide) {
          if (s_off[wib][32] <= m) lo = 32, hi = 63;
        }
#pragma unroll
        for (int step = 0; step < 5; ++step) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_off[wib][mid] <= m) lo = mid;
          else hi = mid - 1;
        }
        const int sidx = s_beg[wib][lo] + (m - s_off[wib][lo]);
        double p[D];
        load_cand<D>(cell_pos, cell_items, sidx, j, p);
        if (!(exclude && __ldg(exclude + j))) {
          d2 = exact_dist2<D>(p, q);
          acc = d2 <= thr2;
        }
      }
      const unsigned mask = __ballot_sync(0xffffffffu, acc);
      const int slot = accepted + __popc(mask & ((1u << lane) - 1u));
      if (acc && slot < kWarpKnnCap) {
        s_kd[wib][slot] = d2;
        s_ki[wib][slot] = j;
      }
      accepted += __popc(mask);
    }
    if (accepted > kWarpKnnCap) {
      why = 1;
      shrink();
      continue;
    }
    if (accepted < n) {
      why = 2;
      grow();
      continue;
    }
    __syncwarp();
    double kd = lane < accepted ? __dsqrt_rn(s_kd[wib][lane]) : CUDART_INF;
    int ki = lane < accepted ? s_ki[wib][lane] : INT_MAX;
    auto exchange = [&](double& d, int& i, int j, bool keep_min) {
      const double od = __shfl_xor_sync(0xffffffffu, d, j);
      const int oi = __shfl_xor_sync(0xffffffffu, i, j);
      // branch-free: keys are distinct (or identical padding, where either choice is the
      // same value), so "the other key is larger" is the negation of "it is smaller"
      const bool other_less = (od < d) | ((od == d) & (oi < i));
      const bool take = other_less == keep_min;
      d = take ? od : d;
      i = take ? oi : i;
    };
    if (accepted <= 32) {
#pragma unroll
      for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) exchange(kd, ki, j, ((lane & j) == 0) == ((lane & k) == 0));
    } else {
      // keys 32..63 in a second register pair, sorted descending while keys 0..31 sort
      // ascending (the k = 32 stage of a 64-key network), then the in-lane j = 32 exchange
      // of the k = 64 stage keeps the smaller key of each pair: a bitonic sequence of the 32
      // smallest keys, finished by the five ascending merge stages
      double kd2 = lane + 32 < accepted ? __dsqrt_rn(s_kd[wib][lane + 32]) : CUDART_INF;
      int ki2 = lane + 32 < accepted ? s_ki[wib][lane + 32] : INT_MAX;
#pragma unroll
      for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
          const bool up = k == 32 ? true : (lane & k) == 0;
          exchange(kd, ki, j, ((lane & j) == 0) == up);
          exchange(kd2, ki2, j, ((lane & j) == 0) != up);
        }
      const bool take2 = (kd2 < kd) | ((kd2 == kd) & (ki2 < ki));
      kd = take2 ? kd2 : kd;
      ki = take2 ? ki2 : ki;
#pragma unroll
      for (int j = 16; j > 0; j >>= 1) exchange(kd, ki, j, (lane & j) == 0);
    }
    const double kth = __shfl_sync(0xffffffffu, kd, n - 1);
    if (!(kth <= r * (1.0 - 1e-12))) {  // the n-th key sits in the last 1e-12 of the ball
      why = 3;
      grow();
      continue;
    }
    if (lane < n) {
      out_idx[t * n + lane] = ki;
      if (out_dist) out_dist[t * n + lane] = kd;
    }
    done = true;
  }
  if (!done && lane == 0) {
#ifdef HN_TRACE
    atomicAdd(&g_knn_fb_stats[0], 1ull);
    atomicAdd(&g_knn_fb_stats[why], 1ull);
#endif
    const int k = atomicAdd(fb_count, 1);
    fb_node[k] = node;
    fb_row[k] = static_cast<int>(t);
  }
}

// ---- classification + lattice stencils ------------------------------------------
template <int D>
__device__ __forceinline__ int grid_at(const int* __restrict__ grid, const int* gdims, const int* key) {
  int64_t l = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (key[a] < 0 || key[a] >= gdims[a]) return -1;
    l = l * gdims[a] + key[a];
  }
  return __ldg(grid + l);
}

struct LatticeDims {
  int g[3];
};

template <int D>
__global__ void classify_kernel(const int8_t* __restrict__ kind, const int* __restrict__ lattice_idx,
                                const int* __restrict__ grid, LatticeDims gd, int64_t n,
                                int8_t* __restrict__ method) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int8_t k = kind[i];
  int8_t m = (k == 2) ? -1 : 1;  // boundary -> METHOD_NONE, interior -> METHOD_RBFFD
  if (k == 0 && lattice_idx) {
    int key[D];
#pragma unroll
    for (int a = 0; a < D; ++a) key[a] = lattice_idx[i * D + a];
    if (key[0] != INT_MIN) {
      bool ok = true;
#pragma unroll
      for (int a = 0; a < D; ++a) {
#pragma unroll
        for (int sgn = -1; sgn <= 1; sgn += 2) {
          int nb[D];
#pragma unroll
          for (int b = 0; b < D; ++b) nb[b] = key[b] + (b == a ? sgn : 0);
          ok = ok && (grid_at<D>(grid, gd.g, nb) >= 0);
        }
      }
      if (ok) m = 0;
    }
  }
  method[i] = m;
}

template <int D>
__global__ void mon_stencil_kernel(const int* __restrict__ rows, int64_t nrows, const double* __restrict__ pos,
                                   const int* __restrict__ lattice_idx, const int* __restrict__ grid, LatticeDims gd,
                                   int* __restrict__ out) {
  int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nrows) return;
  constexpr int M = 2 * D;
  const int r = rows[t];
  int key[D];
#pragma unroll
  for (int a = 0; a < D; ++a) key[a] = lattice_idx[static_cast<int64_t>(r) * D + a];
  double pc[D];
  load_point<D>(pos, r, pc);
  int nb[M];
  double dd[M];
  // offsets in the reference order: +e_0..+e_{d-1}, -e_0..-e_{d-1} (approx.py:371)
#pragma unroll
  for (int o = 0; o < M; ++o) {
    int kk[D];
#pragma unroll
    for (int b = 0; b < D; ++b) kk[b] = key[b] + (b == (o % D) ? (o < D ? 1 : -1) : 0);
    nb[o] = grid_at<D>(grid, gd.g, kk);
    double p[D];
    load_point<D>(pos, nb[o] < 0 ? r : nb[o], p);
    dd[o] = exact_dist<D>(p, pc);
  }
  // insertion sort by (distance, index) -- lexsort((nbrs, d)) at approx.py:375
#pragma unroll
  for (int a = 1; a < M; ++a) {
#pragma unroll
    for (int b = a; b > 0; --b) {
      if (key_less(dd[b], nb[b], dd[b - 1], nb[b - 1])) {
        double td = dd[b]; dd[b] = dd[b - 1]; dd[b - 1] = td;
        int ti = nb[b]; nb[b] = nb[b - 1]; nb[b - 1] = ti;
      }
    }
  }
  out[t * (M + 1)] = r;
#pragma unroll
  for (int o = 0; o < M; ++o) out[t * (M + 1) + 1 + o] = nb[o];
}

// ---- stable partition of node ids by method: [MON | RBF-FD | NONE], ascending in each ----
constexpr int kPartThreads = 256;

__device__ __forceinline__ int method_class(int8_t m) { return m == 0 ? 0 : (m == 1 ? 1 : 2); }

__global__ void partition_count_kernel(const int8_t* __restrict__ method, int64_t n, int* __restrict__ tile_counts,
                                       int64_t ntiles) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kPartThreads + threadIdx.x;
  const int c = i < n ? method_class(method[i]) : 3;
  __shared__ int cnt[3];
  if (threadIdx.x < 3) cnt[threadIdx.x] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const unsigned b = __ballot_sync(0xffffffffu, c == k);
    if (lane == 0 && b) atomicAdd(&cnt[k], __popc(b));
  }
  __syncthreads();
  if (threadIdx.x < 3) tile_counts[threadIdx.x * ntiles + blockIdx.x] = cnt[threadIdx.x];
}

// after the scan: tile_off[k*ntiles + t] = exclusive offset of tile t within class k,
// tile_off[3*ntiles] = total of class 0..2 laid out contiguously (scan over the flattened array)
__global__ void partition_scatter_kernel(const int8_t* __restrict__ method, int64_t n,
                                         const int* __restrict__ tile_off, int64_t ntiles, int* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kPartThreads + threadIdx.x;
  const int c = i < n ? method_class(method[i]) : 3;
  __shared__ int warp_cnt[3][kPartThreads / 32];
  const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int rank_in_warp = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const unsigned b = __ballot_sync(0xffffffffu, c == k);
    if (lane == 0) warp_cnt[k][wid] = __popc(b);
    if (c == k) rank_in_warp = __popc(b & ((1u << lane) - 1u));
  }
  __syncthreads();
  if (c < 3) {
    int before = 0;
    for (int w = 0; w < static_cast<int>(wid); ++w) before += warp_cnt[c][w];
    out[tile_off[c * ntiles + blockIdx.x] + before + rank_in_warp] = static_cast<int>(i);
  }
}

// class sizes: counts[k] = start of class k+1 - start of class k
__global__ void partition_counts_kernel(const int* __restrict__ tile_off, int64_t ntiles, int* __restrict__ counts) {
  if (threadIdx.x < 3) counts[threadIdx.x] = tile_off[(threadIdx.x + 1) * ntiles] - tile_off[threadIdx.x * ntiles];
}

}  // namespace hn

using namespace hn;

// rows_out (n): node ids ordered [MON ascending | RBF ascending | NONE ascending];
// counts_out (3 int32, device) = class sizes.  scratch: 3*ceil(n/256)+1 ints.
HN_EXPORT int hn_partition_methods(const int8_t* method, int64_t n, int* rows_out, int* counts_out, int* scratch,
                                   void* stream) {
  if (n == 0) return cudaMemsetAsync(counts_out, 0, 3 * sizeof(int), as_stream(stream)) == cudaSuccess ? 0 : -1;
  cudaStream_t s = as_stream(stream);
  const int64_t ntiles = ceil_div(n, kPartThreads);
  int* tile_counts = scratch;                       // 3*ntiles
  int* tile_off = nullptr;
  HN_TRY(stream_alloc(reinterpret_cast<void**>(&tile_off), sizeof(int) * (3 * ntiles + 1), s));
  partition_count_kernel<<<ntiles, kPartThreads, 0, s>>>(method, n, tile_counts, ntiles);
  int rc = exclusive_scan(tile_counts, 3 * ntiles, tile_off, s);
  if (rc == 0) {
    partition_scatter_kernel<<<ntiles, kPartThreads, 0, s>>>(method, n, tile_off, ntiles, rows_out);
    partition_counts_kernel<<<1, 32, 0, s>>>(tile_off, ntiles, counts_out);
  }
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(tile_off, s);
  if (rc) return rc;
  return e == cudaSuccess ? 0 : -static_cast<int>(e);
}

static int g_knn_variant = 0;  // 0: warp kernel (3D) / box pass (2D); 1: ring only; 2/3: box pass alpha; 5: box pass only;
                               // 100 + e: warp kernel sized for n + e expected keys
HN_EXPORT void hn_knn_set_variant(int v) { g_knn_variant = v; }

static Grid make_grid(const double* lo_host, double cell, const int* dims_host, int d) {
  Grid g{};
  for (int a = 0; a < 3; ++a) {
    g.lo[a] = a < d ? lo_host[a] : 0.0;
    g.dims[a] = a < d ? dims_host[a] : 1;
  }
  g.cell = cell;
  g.inv_cell = 1.0 / cell;
  return g;
}

namespace hn {
// ---- node-set statistics for the cell-list sizing: per-axis min/max of the positions and
// the sum/count of the scattered nodes' spacing, one pass, one launch.  Doubles are
// min/max-reduced as order-preserving 64-bit keys with integer atomics.
__device__ __forceinline__ unsigned long long ord_key(double x) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

// out (device, 8 u64): [min key x,y,z | max key x,y,z | sum(spacing) bits | count]
__global__ void __launch_bounds__(256) node_stats_kernel(const double* __restrict__ pos, int d, int64_t n,
                                                         const int8_t* __restrict__ kind,
                                                         const double* __restrict__ spacing,
                                                         unsigned long long* __restrict__ out) {
  unsigned long long mn[3] = {~0ull, ~0ull, ~0ull}, mx[3] = {0ull, 0ull, 0ull};
  double hs = 0.0;
  unsigned long long cnt = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    for (int a = 0; a < d; ++a) {
      const unsigned long long k = ord_key(__ldg(pos + i * d + a));
      mn[a] = min(mn[a], k);
      mx[a] = max(mx[a], k);
    }
    if (spacing && kind && __ldg(kind + i) == 1) {
      hs += __ldg(spacing + i);
      ++cnt;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    for (int a = 0; a < 3; ++a) {
      mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
      mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
    }
    hs += __shfl_xor_sync(0xffffffffu, hs, o);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    for (int a = 0; a < d; ++a) {
      atomicMin(out + a, mn[a]);
      atomicMax(out + 3 + a, mx[a]);
    }
    if (cnt) {
      atomicAdd(reinterpret_cast<double*>(out + 6), hs);
      atomicAdd(out + 7, cnt);
    }
  }
}

__global__ void node_stats_init_kernel(unsigned long long* out) {
  const int t = threadIdx.x;
  if (t < 8) out[t] = t < 3 ? ~0ull : 0ull;
}

__global__ void node_stats_finish_kernel(const unsigned long long* in, double* out, int d) {
  const int t = threadIdx.x;
  if (t < d) {
    out[t] = ord_val(in[t]);
    out[d + t] = ord_val(in[3 + t]);
  }
  if (t == 0) {
    out[2 * d] = __longlong_as_double(static_cast<long long>(in[6]));
    out[2 * d + 1] = static_cast<double>(in[7]);
  }
}

}  // namespace hn

HN_EXPORT int hn_node_stats(const double* pos, int64_t n, int d, const int8_t* kind, const double* spacing,
                            double* out, void* scratch, void* stream) {
  if (d < 1 || d > 3) return 1;
  cudaStream_t s = as_stream(stream);
  auto* acc = static_cast<unsigned long long*>(scratch);
  node_stats_init_kernel<<<1, 32, 0, s>>>(acc);
  if (n > 0) {
    const int64_t cap = static_cast<int64_t>(sm_count()) * 4;
    const int64_t blocks = ceil_div(n, 256) < cap ? ceil_div(n, 256) : cap;
    node_stats_kernel<<<blocks, 256, 0, s>>>(pos, d, n, kind, spacing, acc);
  }
  node_stats_finish_kernel<<<1, 32, 0, s>>>(acc, out, d);
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT int hn_celllist_build(const double* pos, int64_t n, int d, const double* lo_host, double cell,
                                const int* dims_host, int* cell_start, int* cell_items, double* cell_pos,
                                int* scratch_count, int* scratch_point_cell, void* stream) {
  if (d != 2 && d != 3) return 1;
  cudaStream_t s = as_stream(stream);
  Grid g = make_grid(lo_host, cell, dims_host, d);
  int64_t ncells = 1;
  for (int a = 0; a < d; ++a) ncells *= dims_host[a];
  HN_TRY(cudaMemsetAsync(scratch_count, 0, sizeof(int) * ncells, s));
  const int th = 256;
  const int64_t bl = ceil_div(n, th);
  if (n > 0) {
    if (d == 2) cell_count_kernel<2><<<bl, th, 0, s>>>(g, pos, n, scratch_count, scratch_point_cell);
    else cell_count_kernel<3><<<bl, th, 0, s>>>(g, pos, n, scratch_count, scratch_point_cell);
    HN_CHECK_LAUNCH();
  }
  int rc = exclusive_scan(scratch_count, ncells, cell_start, s);
  if (rc) return rc;
  HN_TRY(cudaMemsetAsync(scratch_count, 0, sizeof(int) * ncells, s));
  if (n > 0) {
    if (d == 2)
      cell_scatter_kernel<2><<<bl, th, 0, s>>>(pos, n, scratch_point_cell, cell_start, scratch_count, cell_items, cell_pos);
    else
      cell_scatter_kernel<3><<<bl, th, 0, s>>>(pos, n, scratch_point_cell, cell_start, scratch_count, cell_items, cell_pos);
    HN_CHECK_LAUNCH();
  }
  return 0;
}

// box-pass radius: alpha x the radius holding n points at density 1/h^d -- h = the grid's
// design spacing (~1 point per cell in 2D, 1.25^3 in 3D: DeviceNodes' cell rule) or the
// query's own spacing; any radius gives the exact answer, it only changes the work
static double radius_per_spacing(int d, int n, double alpha) {
  if (d == 2) return alpha * sqrt(n / 3.141592653589793);
  return alpha * cbrt(n / 4.18879020478639);
}
static double box_radius(int d, int n, double cell, double alpha) {
  return radius_per_spacing(d, n, alpha) * (d == 2 ? cell : cell / 1.25);
}

template <int D, int NMAX>
static void knn_launch_one(int variant, const Grid& g, const double* pos, const int* cs, const int* ci,
                           const double* cp, const int* queries, const double* qpos, int64_t nq, int n,
                           const uint8_t* excl, const double* qh, int* oi, double* od, cudaStream_t s) {
  const int th = 128;
  const int64_t bl = ceil_div(nq, th);
  if (variant == 1) {
    knn_kernel<D, NMAX><<<bl, th, 0, s>>>(g, pos, cs, ci, cp, queries, qpos, nq, n, excl, oi, od);
    return;
  }
  const double alpha = variant == 2 ? (D == 2 ? 1.3 : 1.05) : (variant == 3 ? (D == 2 ? 1.6 : 1.3) : (D == 2 ? 1.4 : 1.15));
  knn_box_kernel<D, NMAX><<<bl, th, 0, s>>>(g, pos, cs, ci, cp, queries, qpos, nq, n, excl,
                                            box_radius(D, n, g.cell, alpha), qh,
                                            radius_per_spacing(D, n, alpha), oi, od);
}

// warp kernel + fallback list finished by the box kernel (see knn_warp_kernel)
template <int D, int NMAX>
static int knn_warp_launch(const Grid& g, const double* pos, const int* cs, const int* ci, const double* cp,
                           const int* queries, int64_t nq, int n, const uint8_t* excl, const double* qh, int* oi,
                           double* od, cudaStream_t s) {
  int* fb = nullptr;  // [count | nodes (nq) | rows (nq)]
  HN_TRY(stream_alloc(reinterpret_cast<void**>(&fb), sizeof(int) * (1 + 2 * nq), s));
  HN_TRY(cudaMemsetAsync(fb, 0, sizeof(int), s));
  // expected ~n + 4 keys inside r at density 1/h^d (config 4's graded band is ~20 % denser
  // than its nominal spacing: ~29 accepted on average; queries short of n or above 64 rescan
  // inside the kernel)
  const int extra = g_knn_variant >= 100 ? g_knn_variant - 100 : 4;
  const double rs = radius_per_spacing(D, n + extra, 1.0);
  knn_warp_kernel<D><<<ceil_div(nq, kWarpKnnWarps), kWarpKnnWarps * 32, 0, s>>>(
      g, pos, cs, ci, cp, queries, nq, n, excl, rs * (D == 2 ? g.cell : g.cell / 1.25), qh, rs, oi, od, fb, fb + 1,
      fb + 1 + nq);
  const double alpha = D == 2 ? 1.4 : 1.15;
  knn_box_kernel<D, NMAX><<<sm_count() * 4, 128, 0, s>>>(g, pos, cs, ci, cp, fb + 1, nullptr, nq, n, excl,
                                                         box_radius(D, n, g.cell, alpha), qh,
                                                         radius_per_spacing(D, n, alpha), oi, od, fb, fb + 1 + nq);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(fb, s);
  return e == cudaSuccess ? 0 : -static_cast<int>(e);
}

template <int D>
static int launch_knn(const Grid& g, const double* pos, const int* cs, const int* ci, const double* cp,
                      const int* queries, const double* qpos, int64_t nq, int n, const uint8_t* excl,
                      const double* qh, int* oi, double* od, cudaStream_t s) {
  const int v = g_knn_variant >= 100 ? 0 : g_knn_variant;  // >= 100: warp-kernel radius tuning (dev)
  // 3D node queries: the warp kernel (config 4: 674 -> 577 us, 24 % of the queries finished
  // by the box kernel).  In 2D (n = 12, ~25 box points) one thread per query is cheaper
  // (config 1: 58 us vs 157 us for the warp kernel).
  if (v == 0 && D == 3 && !qpos && n <= 32) {
    if (n <= 20) return knn_warp_launch<D, 20>(g, pos, cs, ci, cp, queries, nq, n, excl, qh, oi, od, s);
    return knn_warp_launch<D, 32>(g, pos, cs, ci, cp, queries, nq, n, excl, qh, oi, od, s);
  }
#define HN_KNN(NM) knn_launch_one<D, NM>(v, g, pos, cs, ci, cp, queries, qpos, nq, n, excl, qh, oi, od, s)
  if (n <= 5) HN_KNN(5);
  else if (n <= 8) HN_KNN(8);
  else if (n <= 12) HN_KNN(12);
  else if (n <= 16) HN_KNN(16);
  else if (n <= 20) HN_KNN(20);
  else if (n <= 24) HN_KNN(24);
  else if (n <= 30) HN_KNN(30);
  else if (n <= 32) HN_KNN(32);
  else if (n <= 48) HN_KNN(48);
  else HN_KNN(64);
#undef HN_KNN
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT int hn_knn(const double* pos, int d, const double* lo_host, double cell, const int* dims_host,
                     const int* cell_start, const int* cell_items, const double* cell_pos,
                     const int* queries, const double* qpos, int64_t nq, int n, const uint8_t* exclude,
                     int* out_idx, double* out_dist, void* stream) {
  if (d != 2 && d != 3) return 1;
  if (n < 1 || n > 64) return 2;
  if (nq == 0) return 0;
  Grid g = make_grid(lo_host, cell, dims_host, d);
  cudaStream_t s = as_stream(stream);
  if (d == 2)
    return launch_knn<2>(g, pos, cell_start, cell_items, cell_pos, queries, qpos, nq, n, exclude, nullptr, out_idx,
                         out_dist, s);
  return launch_knn<3>(g, pos, cell_start, cell_items, cell_pos, queries, qpos, nq, n, exclude, nullptr, out_idx,
                       out_dist, s);
}

HN_EXPORT int hn_knn_spacing(const double* pos, int d, const double* lo_host, double cell, const int* dims_host,
                             const int* cell_start, const int* cell_items, const double* cell_pos,
                             const int* queries, const double* qpos, int64_t nq, int n, const uint8_t* exclude,
                             const double* spacing, int* out_idx, double* out_dist, void* stream) {
  if (d != 2 && d != 3) return 1;
  if (n < 1 || n > 64) return 2;
  if (nq == 0) return 0;
  Grid g = make_grid(lo_host, cell, dims_host, d);
  cudaStream_t s = as_stream(stream);
  if (d == 2)
    return launch_knn<2>(g, pos, cell_start, cell_items, cell_pos, queries, qpos, nq, n, exclude, spacing, out_idx,
                         out_dist, s);
  return launch_knn<3>(g, pos, cell_start, cell_items, cell_pos, queries, qpos, nq, n, exclude, spacing, out_idx,
                       out_dist, s);
}

HN_EXPORT int hn_classify(const int8_t* kind, const int* lattice_idx, const int* grid, const int* grid_dims_host,
                          int64_t n, int d, int8_t* method, void* stream) {
  if (d != 2 && d != 3) return 1;
  if (n == 0) return 0;
  LatticeDims gd{};
  for (int a = 0; a < 3; ++a) gd.g[a] = a < d && grid_dims_host ? grid_dims_host[a] : 1;
  cudaStream_t s = as_stream(stream);
  const int th = 256;
  if (d == 2) classify_kernel<2><<<ceil_div(n, th), th, 0, s>>>(kind, lattice_idx, grid, gd, n, method);
  else classify_kernel<3><<<ceil_div(n, th), th, 0, s>>>(kind, lattice_idx, grid, gd, n, method);
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT int hn_mon_stencils(const int* rows, int64_t nrows, const double* pos, const int* lattice_idx,
                              const int* grid, const int* grid_dims_host, int d, int* out, void* stream) {
  if (d != 2 && d != 3) return 1;
  if (nrows == 0) return 0;
  LatticeDims gd{};
  for (int a = 0; a < 3; ++a) gd.g[a] = a < d ? grid_dims_host[a] : 1;
  cudaStream_t s = as_stream(stream);
  const int th = 256;
  if (d == 2) mon_stencil_kernel<2><<<ceil_div(nrows, th), th, 0, s>>>(rows, nrows, pos, lattice_idx, grid, gd, out);
  else mon_stencil_kernel<3><<<ceil_div(nrows, th), th, 0, s>>>(rows, nrows, pos, lattice_idx, grid, gd, out);
  HN_CHECK_LAUNCH();
  return 0;
}

#ifdef HN_TRACE
// Dev builds only: read and reset the warp-kNN fallback counters (tools/tune_knn.py).
HN_EXPORT int hn_debug_knn_fallbacks(unsigned long long* out_host) {
  if (cudaMemcpyFromSymbol(out_host, g_knn_fb_stats, sizeof(unsigned long long) * 4) != cudaSuccess) return -1;
  unsigned long long z[4] = {0, 0, 0, 0};
  return cudaMemcpyToSymbol(g_knn_fb_stats, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif
