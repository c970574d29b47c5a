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
  if (qpos) {
    load_point<D>(qpos, t, q);
  } else {
    const int qi = queries ? __ldg(queries + t) : static_cast<int>(t);
    load_point<D>(pos, qi, q);
  }
  int c0[D];
  cell_coords<D>(g, q, c0);

  // sorted ascending; slots [0, NMAX-n) hold -inf sentinels and are never displaced
  double kd[NMAX];
  int ki[NMAX];
#pragma unroll
  for (int j = 0; j < NMAX; ++j) {
    const bool live = j >= NMAX - n;
    kd[j] = live ? CUDART_INF : -CUDART_INF;
    ki[j] = live ? INT_MAX : -1;
  }
  double thr2 = CUDART_INF;  // d2 above this cannot enter the window
  constexpr int S = pos_stride<D>();

  int max_r = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) max_r = max(max_r, max(c0[a], g.dims[a] - 1 - c0[a]));

  for (int R = 0; R <= max_r; ++R) {
    // visit every cell with Chebyshev offset exactly R
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
          for (int s = beg; s < end; ++s) {
            const int j = __ldg(cell_items + s);
            if (exclude && __ldg(exclude + j)) continue;
            double p[D];
#pragma unroll
            for (int a = 0; a < D; ++a) p[a] = __ldg(cell_pos + static_cast<int64_t>(s) * S + a);
            const double d2 = exact_dist2<D>(p, q);
            if (d2 > thr2) continue;
            const double d = __dsqrt_rn(d2);
            if (!key_less(d, j, kd[NMAX - 1], ki[NMAX - 1])) continue;
#pragma unroll
            for (int m = NMAX - 1; m >= 0; --m) {
              if (key_less(d, j, kd[m], ki[m])) {
                const bool shift = (m > 0) && key_less(d, j, kd[m > 0 ? m - 1 : 0], ki[m > 0 ? m - 1 : 0]);
                kd[m] = shift ? kd[m > 0 ? m - 1 : 0] : d;
                ki[m] = shift ? ki[m > 0 ? m - 1 : 0] : j;
              }
            }
            const double w = kd[NMAX - 1];
            thr2 = (w == CUDART_INF) ? CUDART_INF : __dmul_rn(__dmul_rn(w, w), 1.0 + 1e-15);
          }
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
#pragma unroll
  for (int j = 0; j < NMAX; ++j) {
    if (j >= NMAX - n) {
      const int o = j - (NMAX - n);
      out_idx[t * n + o] = ki[j];
      if (out_dist) out_dist[t * n + o] = kd[j];
    }
  }
}

// ---- kNN query v2: batched ring traversal, integer keys ------------------------------
// Same result as knn_kernel (top n by (fl-distance, index)).  Each ring of cells is walked
// in batches of KB cells whose [start, end) ranges are loaded together; points are then
// taken slot-major across the batch so KB independent point loads are in flight.  The
// top-n network compares fl-distances as uint64 bit patterns (non-negative doubles order
// like their bits), keeping the FP64 pipe for the distance arithmetic only.
template <int D, int NMAX>
__global__ void __launch_bounds__(128) knn2_kernel(Grid g, const double* __restrict__ pos,
                                                   const int* __restrict__ cell_start,
                                                   const int* __restrict__ cell_items,
                                                   const double* __restrict__ cell_pos,
                                                   const int* __restrict__ queries,
                                                   const double* __restrict__ qpos, int64_t nq, int n,
                                                   const uint8_t* __restrict__ exclude,
                                                   int* __restrict__ out_idx, double* __restrict__ out_dist) {
  constexpr int KB = 8;
  constexpr int S = pos_stride<D>();
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nq) return;
  double q[D];
  if (qpos) {
    load_point<D>(qpos, t, q);
  } else {
    const int qi = queries ? __ldg(queries + t) : static_cast<int>(t);
    load_point<D>(pos, qi, q);
  }
  int c0[D];
  cell_coords<D>(g, q, c0);
  unsigned long long kd[NMAX];
  int ki[NMAX];
#pragma unroll
  for (int j = 0; j < NMAX; ++j) {
    const bool live = j >= NMAX - n;
    kd[j] = live ? ~0ull : 0ull;  // ~0 > any distance bits; 0 sentinel never displaced
    ki[j] = live ? INT_MAX : -1;
  }
  double thr2 = CUDART_INF;
  int max_r = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) max_r = max(max_r, max(c0[a], g.dims[a] - 1 - c0[a]));

  for (int R = 0; R <= max_r; ++R) {
    const int side = 2 * R + 1;
    int ncube = side * side;
    if constexpr (D == 3) ncube *= side;
    for (int base = 0; base < ncube; base += KB) {
      int cs[KB], ce[KB];
#pragma unroll
      for (int b = 0; b < KB; ++b) {
        int tt = base + b;
        int o[D];
        bool ok = tt < ncube;
#pragma unroll
        for (int a = D - 1; a >= 0; --a) {
          o[a] = tt % side - R;
          tt /= side;
        }
        int m = 0;
        int64_t cl = 0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          m = max(m, abs(o[a]));
          const int x = c0[a] + o[a];
          ok = ok && x >= 0 && x < g.dims[a];
          cl = cl * g.dims[a] + x;
        }
        ok = ok && m == R;
        cs[b] = ok ? __ldg(cell_start + cl) : 0;
        ce[b] = ok ? __ldg(cell_start + cl + 1) : 0;
      }
      for (int slot = 0;; ++slot) {
        bool any = false;
        int jj[KB];
        double pp[KB][D];
#pragma unroll
        for (int b = 0; b < KB; ++b) {
          const int s_ = cs[b] + slot;
          const bool live = s_ < ce[b];
          any = any || live;
          jj[b] = live ? __ldg(cell_items + s_) : -1;
#pragma unroll
          for (int a = 0; a < D; ++a) pp[b][a] = live ? __ldg(cell_pos + static_cast<int64_t>(s_) * S + a) : 0.0;
        }
        if (!any) break;
#pragma unroll
        for (int b = 0; b < KB; ++b) {
          const int j = jj[b];
          if (j < 0) continue;
          if (exclude && __ldg(exclude + j)) continue;
          const double d2 = exact_dist2<D>(pp[b], q);
          if (d2 > thr2) continue;
          const unsigned long long d = static_cast<unsigned long long>(__double_as_longlong(__dsqrt_rn(d2)));
          if (!(d < kd[NMAX - 1] || (d == kd[NMAX - 1] && j < ki[NMAX - 1]))) continue;
#pragma unroll
          for (int mm = NMAX - 1; mm >= 0; --mm) {
            const bool lt = d < kd[mm] || (d == kd[mm] && j < ki[mm]);
            if (lt) {
              const int pm = mm > 0 ? mm - 1 : 0;
              const bool shift = (mm > 0) && (d < kd[pm] || (d == kd[pm] && j < ki[pm]));
              kd[mm] = shift ? kd[pm] : d;
              ki[mm] = shift ? ki[pm] : j;
            }
          }
          const unsigned long long w = kd[NMAX - 1];
          if (w != ~0ull) {
            const double wd = __longlong_as_double(static_cast<long long>(w));
            thr2 = __dmul_rn(__dmul_rn(wd, wd), 1.0 + 1e-15);
          }
        }
      }
    }
    double bound = CUDART_INF;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      if (c0[a] - R > 0) bound = fmin(bound, q[a] - (g.lo[a] + (c0[a] - R) * g.cell));
      if (c0[a] + R + 1 < g.dims[a]) bound = fmin(bound, (g.lo[a] + (c0[a] + R + 1) * g.cell) - q[a]);
    }
    const unsigned long long w = kd[NMAX - 1];
    if (w != ~0ull && __longlong_as_double(static_cast<long long>(w)) < bound - 1e-9 * g.cell) break;
  }
#pragma unroll
  for (int j = 0; j < NMAX; ++j) {
    if (j >= NMAX - n) {
      const int o = j - (NMAX - n);
      out_idx[t * n + o] = ki[j];
      if (out_dist) out_dist[t * n + o] = __longlong_as_double(static_cast<long long>(kd[j]));
    }
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

static int g_knn_variant = 1;  // 1: per-cell traversal (knn, default), 0: batched rings (knn2)
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

template <int D>
static int launch_knn(const Grid& g, const double* pos, const int* cs, const int* ci, const double* cp,
                      const int* queries, const double* qpos, int64_t nq, int n, const uint8_t* excl, int* oi,
                      double* od, cudaStream_t s) {
  const int th = 128;
  const int64_t bl = ceil_div(nq, th);
  if (g_knn_variant == 0) {
    if (n <= 8) knn2_kernel<D, 8><<<bl, th, 0, s>>>(g, pos, cs, ci, cp, queries, qpos, nq, n, excl, oi, od);
    else if (n <= 16) knn2_kernel<D, 16><<<bl, th, 0, s>>>(g, pos, cs, ci, cp, queries, qpos, nq, n, excl, oi, od);
    else if (n <= 24) knn2_kernel<D, 24><<<bl, th, 0, s>>>(g, pos, cs, ci, cp, queries, qpos, nq, n, excl, oi, od);
    else if (n <= 32) knn2_kernel<D, 32><<<bl, th, 0, s>>>(g, pos, cs, ci, cp, queries, qpos, nq, n, excl, oi, od);
    else if (n <= 48) knn2_kernel<D, 48><<<bl, th, 0, s>>>(g, pos, cs, ci, cp, queries, qpos, nq, n, excl, oi, od);
    else knn2_kernel<D, 64><<<bl, th, 0, s>>>(g, pos, cs, ci, cp, queries, qpos, nq, n, excl, oi, od);
    HN_CHECK_LAUNCH();
    return 0;
  }
  if (n <= 8) knn_kernel<D, 8><<<bl, th, 0, s>>>(g, pos, cs, ci, cp, queries, qpos, nq, n, excl, oi, od);
  else if (n <= 16) knn_kernel<D, 16><<<bl, th, 0, s>>>(g, pos, cs, ci, cp, queries, qpos, nq, n, excl, oi, od);
  else if (n <= 24) knn_kernel<D, 24><<<bl, th, 0, s>>>(g, pos, cs, ci, cp, queries, qpos, nq, n, excl, oi, od);
  else if (n <= 32) knn_kernel<D, 32><<<bl, th, 0, s>>>(g, pos, cs, ci, cp, queries, qpos, nq, n, excl, oi, od);
  else if (n <= 48) knn_kernel<D, 48><<<bl, th, 0, s>>>(g, pos, cs, ci, cp, queries, qpos, nq, n, excl, oi, od);
  else knn_kernel<D, 64><<<bl, th, 0, s>>>(g, pos, cs, ci, cp, queries, qpos, nq, n, excl, oi, od);
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
  if (d == 2) return launch_knn<2>(g, pos, cell_start, cell_items, cell_pos, queries, qpos, nq, n, exclude, out_idx, out_dist, s);
  return launch_knn<3>(g, pos, cell_start, cell_items, cell_pos, queries, qpos, nq, n, exclude, out_idx, out_dist, s);
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
