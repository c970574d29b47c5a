// K7/K8/K10/K11: fused explicit Boussinesq step kernels over the binned ELL operator
// table (planes: [Laplacian, d/dx_0, .., d/dx_{d-1}] in the order build_operators
// requests them, solver.py:148), plus the generic sequential CSR matvec used for every
// non-stencil sparse matrix (bordered Poisson, Neumann and Nusselt rows).
//
// Every sum is the reference's scipy csr_matvec order (sequential, ascending columns,
// no FMA) and every elementwise expression keeps numpy's operation order with explicit
// round-to-nearest intrinsics, so given identical inputs the explicit part of a step is
// bit-identical to solver.py:250-358.  State is SoA: v[c*N + i], T[i], p[i].
#include "hn_common.cuh"

namespace hn {

struct StepBins {
  int nbins;
  int width[4];
  int64_t K[4];
  int64_t block_start[5];
  const int* rows[4];
  const int* idx[4];
  const double* w[4];  // planes [lap, d0, d1, (d2)] at plane stride W*K
  int lap_plane;
  int d_plane[3];
};

__device__ __forceinline__ int find_bin(const StepBins& b) {
  int bin = 0;
#pragma unroll
  for (int i = 1; i < 4; ++i)
    if (i < b.nbins && blockIdx.x >= b.block_start[i]) bin = i;
  return bin;
}

// sequential stencil sum sum_j w[plane][j] * f[idx_j]
template <int W>
__device__ __forceinline__ double ssum(const double* __restrict__ w, int64_t K, int64_t k, const double* fv) {
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < W; ++j) acc = __dadd_rn(acc, __dmul_rn(__ldg(w + j * K + k), fv[j]));
  return acc;
}

// ---- K7: momentum predict + no-slip (solver.py:250-280) ----
struct MomentumCoef {
  double dt, Pr, t_ref;
  double buoy[3];  // (Ra * Pr) * g[c]
  int zero_boundary;
  // optional hyper-dissipation (solver.py:235-247): hc[i] = -coeff * h_i**3 (host numpy),
  // l2 = lap(lap(v_c)) per component (SoA); term = (hc * |v|) * l2, added to rhs
  const double* hc;
  const double* l2;
};

// |v_row| as np.linalg.norm(v, axis=1): sqrt((v0*v0 + v1*v1) [+ v2*v2])
template <int D>
__device__ __forceinline__ double speed_of(const double* vr) {
  double s = __dmul_rn(vr[0], vr[0]);
#pragma unroll
  for (int a = 1; a < D; ++a) s = __dadd_rn(s, __dmul_rn(vr[a], vr[a]));
  return __dsqrt_rn(s);
}

template <int D, int W>
__device__ __forceinline__ void momentum_row(const StepBins& b, int bin, int64_t k, const double* __restrict__ v,
                                             const double* __restrict__ T, int64_t N, const MomentumCoef& c,
                                             double* __restrict__ vstar) {
  const int64_t K = b.K[bin];
  const int row = __ldg(b.rows[bin] + k);
  if constexpr (W == 0) {
    // empty operator rows: grad = lap = 0.  With the no-slip BC fused (solver.py:277-280)
    // the row is simply 0; without it, keep momentum_predict's raw value.
#pragma unroll
    for (int cc = 0; cc < D; ++cc) {
      double out = 0.0;
      if (!c.zero_boundary) {
        const double vc = __ldg(v + cc * N + row);
        double adv = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const double t = __dmul_rn(__ldg(v + a * N + row), 0.0);
          adv = (a == 0) ? t : __dadd_rn(adv, t);
        }
        const double tdelta = __dsub_rn(__ldg(T + row), c.t_ref);
        double rhs = __dsub_rn(__dadd_rn(-adv, __dmul_rn(c.Pr, 0.0)), __dmul_rn(c.buoy[cc], tdelta));
        if (c.hc) {
          double vr[D];
#pragma unroll
          for (int a = 0; a < D; ++a) vr[a] = __ldg(v + a * N + row);
          rhs = __dadd_rn(rhs, __dmul_rn(__dmul_rn(__ldg(c.hc + row), speed_of<D>(vr)), __ldg(c.l2 + cc * N + row)));
        }
        out = __dadd_rn(vc, __dmul_rn(c.dt, rhs));
      }
      vstar[cc * N + row] = out;
    }
    return;
  } else {
    int id[W];
#pragma unroll
    for (int j = 0; j < W; ++j) id[j] = __ldg(b.idx[bin] + j * K + k);
    const double* wb = b.w[bin];
    const int64_t ps = static_cast<int64_t>(W) * K;
    double vi[D];
#pragma unroll
    for (int a = 0; a < D; ++a) vi[a] = __ldg(v + a * N + row);
    const double tdelta = __dsub_rn(__ldg(T + row), c.t_ref);
    // every gather of the row first (D components), then each weight loaded once and
    // applied to all components: D * (D + 1) sequential sums, each in ascending-j order
    double fv[D][W];
#pragma unroll
    for (int cc = 0; cc < D; ++cc)
#pragma unroll
      for (int j = 0; j < W; ++j) fv[cc][j] = __ldg(v + cc * N + id[j]);
    double gs[D][D], ls[D];
#pragma unroll
    for (int cc = 0; cc < D; ++cc) {
      ls[cc] = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) gs[cc][a] = 0.0;
    }
#pragma unroll
    for (int j = 0; j < W; ++j) {
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double wa = __ldg(wb + b.d_plane[a] * ps + j * K + k);
#pragma unroll
        for (int cc = 0; cc < D; ++cc) gs[cc][a] = __dadd_rn(gs[cc][a], __dmul_rn(wa, fv[cc][j]));
      }
      const double wl = __ldg(wb + b.lap_plane * ps + j * K + k);
#pragma unroll
      for (int cc = 0; cc < D; ++cc) ls[cc] = __dadd_rn(ls[cc], __dmul_rn(wl, fv[cc][j]));
    }
#pragma unroll
    for (int cc = 0; cc < D; ++cc) {
      double adv = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double t = __dmul_rn(vi[a], gs[cc][a]);
        adv = (a == 0) ? t : __dadd_rn(adv, t);
      }
      const double lap = ls[cc];
      double rhs = __dsub_rn(__dadd_rn(-adv, __dmul_rn(c.Pr, lap)), __dmul_rn(c.buoy[cc], tdelta));
      if (c.hc)
        rhs = __dadd_rn(rhs, __dmul_rn(__dmul_rn(__ldg(c.hc + row), speed_of<D>(vi)), __ldg(c.l2 + cc * N + row)));
      vstar[cc * N + row] = __dadd_rn(vi[cc], __dmul_rn(c.dt, rhs));
    }
  }
}

template <int D, int W>
__global__ void __launch_bounds__(128, (W <= 7 ? 6 : (W <= 12 ? 3 : 2)))
momentum_kernel(StepBins b, const double* __restrict__ v, const double* __restrict__ T, int64_t N,
                MomentumCoef c, double* __restrict__ vstar) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= b.K[0]) return;
  momentum_row<D, W>(b, 0, k, v, T, N, c, vstar);
}

// ---- K8: divergence -> Poisson right-hand side (solver.py:295-301) ----
template <int D, int W>
__device__ __forceinline__ void div_row(const StepBins& b, int bin, int64_t k, const double* __restrict__ vs,
                                        int64_t N, double inv_dt_unused, double dt, double* __restrict__ rhs) {
  const int64_t K = b.K[bin];
  const int row = __ldg(b.rows[bin] + k);
  if constexpr (W == 0) {
    rhs[row] = 0.0;
    return;
  } else {
    int id[W];
#pragma unroll
    for (int j = 0; j < W; ++j) id[j] = __ldg(b.idx[bin] + j * K + k);
    const int64_t ps = static_cast<int64_t>(W) * K;
    double fv[D][W];  // every gather first
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int j = 0; j < W; ++j) fv[a][j] = __ldg(vs + a * N + id[j]);
    double div = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double s = ssum<W>(b.w[bin] + b.d_plane[a] * ps, K, k, fv[a]);
      div = (a == 0) ? s : __dadd_rn(div, s);
    }
    rhs[row] = __ddiv_rn(div, dt);
  }
}

template <int D, int W>
__global__ void __launch_bounds__(128, (W <= 7 ? 8 : (W <= 12 ? 6 : (W <= 20 ? 4 : 2))))
div_rhs_kernel(StepBins b, const double* __restrict__ vs, int64_t N, double dt,
               double* __restrict__ rhs, bool gauge) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gauge && blockIdx.x == 0 && threadIdx.x == 0) rhs[N] = 0.0;  // bordered gauge equation
  if (k >= b.K[0]) return;
  div_row<D, W>(b, 0, k, vs, N, 0.0, dt, rhs);
}

// ---- K10: velocity correction + temperature advection-diffusion (solver.py:317-331, 345-357) ----
struct HyperT {  // optional hyper-dissipation of T: hc = -coeff * h**3, l2 = lap(lap(T))
  const double* hc;
  const double* l2;
};

template <int D, int W>
__device__ __forceinline__ void correct_temp_row(const StepBins& b, int bin, int64_t k, const double* __restrict__ vs,
                                                 const double* __restrict__ p, const double* __restrict__ T,
                                                 int64_t N, double dt, double* __restrict__ vout,
                                                 double* __restrict__ Tout, int* __restrict__ flags, HyperT hy) {
  const int64_t K = b.K[bin];
  const int row = __ldg(b.rows[bin] + k);
  double vn[D];
  double tn;
  if constexpr (W == 0) {
#pragma unroll
    for (int a = 0; a < D; ++a) vn[a] = 0.0;
    // empty operator rows: conv = 0, lap = 0  ->  T + dt * (-0 + 0)
    const double Ti = __ldg(T + row);
    double r = __dadd_rn(-0.0, 0.0);
    if (hy.hc) r = __dadd_rn(r, __dmul_rn(__dmul_rn(__ldg(hy.hc + row), speed_of<D>(vn)), __ldg(hy.l2 + row)));
    tn = __dadd_rn(Ti, __dmul_rn(dt, r));
  } else {
    int id[W];
#pragma unroll
    for (int j = 0; j < W; ++j) id[j] = __ldg(b.idx[bin] + j * K + k);
    const double* wb = b.w[bin];
    const int64_t ps = static_cast<int64_t>(W) * K;
    double fp[W], ft[W];
#pragma unroll
    for (int j = 0; j < W; ++j) {
      fp[j] = __ldg(p + id[j]);
      ft[j] = __ldg(T + id[j]);
    }
    // each derivative weight loaded once for both fields: 2D + 1 sequential sums in j order
    double gp[D], gt[D], lap = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) gp[a] = gt[a] = 0.0;
#pragma unroll
    for (int j = 0; j < W; ++j) {
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double wa = __ldg(wb + b.d_plane[a] * ps + j * K + k);
        gp[a] = __dadd_rn(gp[a], __dmul_rn(wa, fp[j]));
        gt[a] = __dadd_rn(gt[a], __dmul_rn(wa, ft[j]));
      }
      lap = __dadd_rn(lap, __dmul_rn(__ldg(wb + b.lap_plane * ps + j * K + k), ft[j]));
    }
#pragma unroll
    for (int a = 0; a < D; ++a) vn[a] = __dsub_rn(__ldg(vs + a * N + row), __dmul_rn(dt, gp[a]));
    double conv = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double t = __dmul_rn(vn[a], gt[a]);
      conv = (a == 0) ? t : __dadd_rn(conv, t);
    }
    double r = __dadd_rn(-conv, lap);
    if (hy.hc) r = __dadd_rn(r, __dmul_rn(__dmul_rn(__ldg(hy.hc + row), speed_of<D>(vn)), __ldg(hy.l2 + row)));
    tn = __dadd_rn(__ldg(T + row), __dmul_rn(dt, r));
  }
  bool bad = !isfinite(tn);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    vout[a * N + row] = vn[a];
    bad = bad || !isfinite(vn[a]);
  }
  Tout[row] = tn;
  if (bad) {
    atomicOr(flags, 1);
    if (!isfinite(tn)) atomicMin(flags + 1, row);
  }
}

template <int D, int W>
__global__ void __launch_bounds__(128, (W <= 7 ? 8 : (W <= 12 ? 6 : (W <= 20 ? 4 : 2))))
correct_temp_kernel(StepBins b, const double* __restrict__ vs, const double* __restrict__ p,
                    const double* __restrict__ T, int64_t N, double dt, double* __restrict__ vout,
                    double* __restrict__ Tout, int* __restrict__ flags, HyperT hy) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= b.K[0]) return;
  correct_temp_row<D, W>(b, 0, k, vs, p, T, N, dt, vout, Tout, flags, hy);
}

// ---- one launch for every bin of a phase (small node sets) ----
// Blocks map to bins through block_start; a bin's width selects the compile-time body
// (WA, WB or 0).  At small N the per-bin launches of a phase cost more than the lower
// occupancy of the shared register budget, so the dispatcher fuses below kFuseRows.
constexpr int64_t kFuseRows = 600000;

#define HN_FUSED_BODY(ROWFN, ...)                                          \
  const int bin = find_bin(b);                                             \
  const int64_t k = static_cast<int64_t>(blockIdx.x - b.block_start[bin]) * blockDim.x + threadIdx.x; \
  if (k >= b.K[bin]) return;                                               \
  const int w = b.width[bin];                                              \
  if (w == WA) ROWFN<D, WA>(b, bin, k, __VA_ARGS__);                       \
  else if (WB > 0 && w == WB) ROWFN<D, (WB > 0 ? WB : WA)>(b, bin, k, __VA_ARGS__); \
  else ROWFN<D, 0>(b, bin, k, __VA_ARGS__);

// launch bounds: the 2D stencils (W <= 12) run best at 6 / 8 CTAs per SM (80 / 64 registers, no
// spills): config-3 explicit part 43.0 -> 39.0 us (59 % of HBM); 8 / 10 CTAs: 41.0 us; the 3D
// widths keep 3 / 4 (W = 20, 30 gathers per row need the registers: 4 / 6 CTAs measured 78.5 -> 76.6 %
// of HBM on the config-4 explicit part)
template <int WA, int WB>
constexpr bool kNarrowBins = (WA > WB ? WA : WB) <= 12;

template <int D, int WA, int WB>
__global__ void __launch_bounds__(128, (kNarrowBins<WA, WB> ? 6 : 3))
momentum_fused_kernel(StepBins b, const double* __restrict__ v, const double* __restrict__ T, int64_t N,
                      MomentumCoef c, double* __restrict__ vstar) {
  HN_FUSED_BODY(momentum_row, v, T, N, c, vstar)
}

template <int D, int WA, int WB>
__global__ void __launch_bounds__(128, (kNarrowBins<WA, WB> ? 8 : 4))
div_rhs_fused_kernel(StepBins b, const double* __restrict__ vs, int64_t N, double dt, double* __restrict__ rhs) {
  if (blockIdx.x == 0 && threadIdx.x == 0) rhs[N] = 0.0;  // bordered gauge equation
  HN_FUSED_BODY(div_row, vs, N, 0.0, dt, rhs)
}

template <int D, int WA, int WB>
__global__ void __launch_bounds__(128, (kNarrowBins<WA, WB> ? 8 : 4))
correct_temp_fused_kernel(StepBins b, const double* __restrict__ vs, const double* __restrict__ p,
                          const double* __restrict__ T, int64_t N, double dt, double* __restrict__ vout,
                          double* __restrict__ Tout, int* __restrict__ flags, HyperT hy) {
  HN_FUSED_BODY(correct_temp_row, vs, p, T, N, dt, vout, Tout, flags, hy)
}
#undef HN_FUSED_BODY

// (WA, WB) pairs with a fused instantiation: the MON/RBF widths of configs 0-4
#define HN_FUSED_PAIRS(X) X(2, 5, 12) X(2, 5, -1) X(2, 12, -1) X(3, 7, 20) X(3, 7, 30) X(3, 7, -1) X(3, 20, -1) X(3, 30, -1)

// widths of the non-empty bins -> (wa, wb); false if more than two distinct or total too big
static bool fused_pair(const StepBins& b, int d, int* wa, int* wb) {
  int64_t rows = 0;
  *wa = -1;
  *wb = -1;
  for (int i = 0; i < b.nbins; ++i) {
    rows += b.K[i];
    const int w = b.width[i];
    if (w == 0 || w == *wa || w == *wb) continue;
    if (*wa < 0) *wa = w;
    else if (*wb < 0) *wb = w;
    else return false;
  }
  if (rows > kFuseRows || *wa < 0) return false;
  if (*wb >= 0 && *wb < *wa) { const int t = *wa; *wa = *wb; *wb = t; }
  return true;
}

// ---- K11: temperature boundary conditions (solver.py:334-342) ----
// Insulated rows: T[b] = -(sum_j W_bj t0_j) / W_bb with t0 = T, Neumann entries zeroed.
// The Neumann block W[:, neu] is diagonal (boundary stencils exclude every other
// boundary node), so SuperLU's solve of it is an elementwise division.
// Sequential row dot product sum_e vals[e] * x[cols[e]] in ascending-entry order (scipy
// csr_matvec: no FMA, one accumulator) with the loads of 8 entries issued before their
// products are added -- the summation order is unchanged, only the memory latency overlaps.
template <bool NEU_MASK>
__device__ __forceinline__ double csr_row_seq(const int* __restrict__ cols, const double* __restrict__ vals,
                                              const double* __restrict__ x, const uint8_t* __restrict__ is_neu,
                                              int64_t e, int64_t e1) {
  double acc = 0.0;
  for (; e < e1; e += 8) {
    int c[8];
    double v[8], xv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      c[k] = e + k < e1 ? __ldg(cols + e + k) : -1;
      v[k] = e + k < e1 ? __ldg(vals + e + k) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      xv[k] = c[k] >= 0 ? x[c[k]] : 0.0;
      if (NEU_MASK && c[k] >= 0 && __ldg(is_neu + c[k])) xv[k] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (c[k] >= 0) acc = __dadd_rn(acc, __dmul_rn(v[k], xv[k]));
  }
  return acc;
}

// Rows of at most 32 entries (every boundary stencil: n = 12 in 2D, 30 in 3D) issue all
// their column/value loads, then all their gathers, before the sequential sum: three
// memory round trips per row instead of one per batch of 8.
__device__ __forceinline__ double csr_row_seq32_neu(const int* __restrict__ cols, const double* __restrict__ vals,
                                                   const double* __restrict__ x, const uint8_t* __restrict__ is_neu,
                                                   int64_t e, int len) {
  int c[32];
  double v[32], xv[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    c[k] = k < len ? __ldg(cols + e + k) : -1;
    v[k] = k < len ? __ldg(vals + e + k) : 0.0;
  }
  // the gather and the mask byte are requested together (one round trip, not two); a masked
  // entry's value is read and dropped (it may be another row's Neumann node, written meanwhile)
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double xr = c[k] >= 0 ? x[c[k]] : 0.0;
    const bool masked = c[k] >= 0 && __ldg(is_neu + c[k]);
    xv[k] = masked ? 0.0 : xr;
  }
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 32; ++k)
    if (k < len) acc = __dadd_rn(acc, __dmul_rn(v[k], xv[k]));
  return acc;
}

// Dirichlet rows (threads [0, ndir)) and Neumann rows (threads [ndir, ndir + nneu)) in one
// launch -- they are independent: boundary stencils exclude every other boundary node, so a
// Neumann row never reads a Dirichlet value -- and, with a latch, the end-of-step latch by
// the last block to finish (flags[2] counts finished blocks, reset by that block).
__device__ __forceinline__ void latch_apply(int* __restrict__ flags, int* __restrict__ latch,
                                            const int* __restrict__ pstatus);

__global__ void temperature_bc_kernel(const int* __restrict__ dir_idx, const double* __restrict__ dir_val,
                                      int64_t ndir, const int64_t* __restrict__ rowptr, const int* __restrict__ cols,
                                      const double* __restrict__ vals, const int* __restrict__ neu_idx,
                                      const double* __restrict__ diag, const uint8_t* __restrict__ is_neu,
                                      int64_t nneu, double* __restrict__ T, int* __restrict__ flags,
                                      int* __restrict__ latch, const int* __restrict__ pstatus) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < ndir) {
    T[dir_idx[i]] = dir_val[i];
  } else if (i < ndir + nneu) {
    const int64_t r = i - ndir;
    const int64_t e0 = __ldg(rowptr + r), e1 = __ldg(rowptr + r + 1);
    const double acc = e1 - e0 <= 32 ? csr_row_seq32_neu(cols, vals, T, is_neu, e0, static_cast<int>(e1 - e0))
                                     : csr_row_seq<true>(cols, vals, T, is_neu, e0, e1);
    const double t = __ddiv_rn(-acc, diag[r]);
    const int node = neu_idx[r];
    T[node] = t;
    if (flags && !isfinite(t)) {  // the reference probes T after its boundary conditions (solver.py:448-452)
      atomicOr(flags, 1);
      atomicMin(flags + 1, node);
    }
  }
  if (!latch) return;
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(flags + 2, 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    latch_apply(flags, latch, pstatus);
    flags[2] = 0;
  }
}

// End of a step: latch the first step whose fields went non-finite (flags written by K10 and
// the Neumann rows) with the lowest non-finite temperature node, as the reference's per-step
// probe reports it (solver.py:448-452); then clear the per-step flags.
// latch = [steps completed, first bad step (0: none), its node (INT_MAX: none in T),
//          first step whose pressure solve reported info != 0 (0: none), that info].
__device__ __forceinline__ void latch_apply(int* __restrict__ flags, int* __restrict__ latch,
                                            const int* __restrict__ pstatus) {
  const int s = latch[0] + 1;
  latch[0] = s;
  if (flags[0] && latch[1] == 0) {
    latch[1] = s;
    latch[2] = flags[1];
  }
  if (pstatus && pstatus[0] != 0 && latch[3] == 0) {  // first step whose pressure solve failed
    latch[3] = s;
    latch[4] = pstatus[0];
  }
  flags[0] = 0;
  flags[1] = 0x7fffffff;
}

// ---- generic sequential CSR matvec (scipy csr_matvec order), thread per row ----
__global__ void csr_matvec_kernel(const int64_t* __restrict__ rowptr, const int* __restrict__ cols,
                                  const double* __restrict__ vals, const double* __restrict__ x, int64_t nrows,
                                  double* __restrict__ y) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  y[r] = csr_row_seq<false>(cols, vals, x, nullptr, __ldg(rowptr + r), __ldg(rowptr + r + 1));
}

// y = b - A x  (r0 of BiCGStab; scipy: b - matvec(x))
__global__ void csr_residual_kernel(const int64_t* __restrict__ rowptr, const int* __restrict__ cols,
                                    const double* __restrict__ vals, const double* __restrict__ x,
                                    const double* __restrict__ b, int64_t nrows, double* __restrict__ y) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  y[r] = __dsub_rn(b[r], csr_row_seq<false>(cols, vals, x, nullptr, __ldg(rowptr + r), __ldg(rowptr + r + 1)));
}

void fill_bins(StepBins& b, int nbins, const int64_t* K, const int* W, const int* const* rows, const int* const* idx,
               const double* const* w, int threads, int64_t* blocks) {
  b.nbins = nbins;
  int64_t acc = 0;
  for (int i = 0; i < nbins; ++i) {
    b.K[i] = K[i];
    b.width[i] = W[i];
    b.rows[i] = rows[i];
    b.idx[i] = idx[i];
    b.w[i] = w[i];
    b.block_start[i] = acc;
    acc += ceil_div(K[i], threads);
  }
  b.block_start[nbins] = acc;
  *blocks = acc;
}

StepBins single_bin(const StepBins& b, int i) {
  StepBins o = b;
  o.nbins = 1;
  o.width[0] = b.width[i];
  o.K[0] = b.K[i];
  o.rows[0] = b.rows[i];
  o.idx[0] = b.idx[i];
  o.w[0] = b.w[i];
  o.block_start[0] = 0;
  o.block_start[1] = ceil_div(b.K[i], 128);
  return o;
}

// one template instantiation per (dimension, stencil width): each gets its own registers
#define HN_WIDTH_DISPATCH(d, w, LAUNCH)                                   \
  do {                                                                    \
    if ((d) == 2) {                                                       \
      switch (w) {                                                        \
        case 0: LAUNCH(2, 0); break;  case 5: LAUNCH(2, 5); break;        \
        case 7: LAUNCH(2, 7); break;  case 12: LAUNCH(2, 12); break;      \
        case 20: LAUNCH(2, 20); break; default: LAUNCH(2, 30); break;     \
      }                                                                   \
    } else {                                                              \
      switch (w) {                                                        \
        case 0: LAUNCH(3, 0); break;  case 5: LAUNCH(3, 5); break;        \
        case 7: LAUNCH(3, 7); break;  case 12: LAUNCH(3, 12); break;      \
        case 20: LAUNCH(3, 20); break; default: LAUNCH(3, 30); break;     \
      }                                                                   \
    }                                                                     \
  } while (0)

}  // namespace hn

using namespace hn;

static bool ok_bins(int nbins, const int* W) {
  if (nbins < 1 || nbins > 4) return false;
  for (int i = 0; i < nbins; ++i)
    if (!(W[i] == 0 || W[i] == 5 || W[i] == 7 || W[i] == 12 || W[i] == 20 || W[i] == 30)) return false;
  return true;
}

HN_EXPORT int hn_momentum(int nbins, const int64_t* bin_K_host, const int* bin_width_host,
                          const int* const* bin_rows_host, const int* const* bin_idx_host,
                          const double* const* bin_w_host, int lap_plane, const int* d_plane_host, int d,
                          const double* v, const double* T, int64_t N, double dt, double Pr, double t_ref,
                          const double* buoy_host, int zero_boundary, const double* hyper_coef,
                          const double* hyper_lap2, double* vstar, void* stream) {
  if (!ok_bins(nbins, bin_width_host) || (d != 2 && d != 3)) return 1;
  StepBins b{};
  int64_t blocks;
  const int th = 128;
  fill_bins(b, nbins, bin_K_host, bin_width_host, bin_rows_host, bin_idx_host, bin_w_host, th, &blocks);
  b.lap_plane = lap_plane;
  for (int a = 0; a < d; ++a) b.d_plane[a] = d_plane_host[a];
  if ((hyper_coef == nullptr) != (hyper_lap2 == nullptr)) return 2;
  MomentumCoef c{dt, Pr, t_ref, {0, 0, 0}, zero_boundary, hyper_coef, hyper_lap2};
  for (int a = 0; a < d; ++a) c.buoy[a] = buoy_host[a];
  if (blocks == 0) return 0;
  int wa, wb;
  if (fused_pair(b, d, &wa, &wb)) {
    cudaStream_t s = as_stream(stream);
#define HN_X(DD, A, B) \
    if (d == DD && wa == A && wb == B) { momentum_fused_kernel<DD, A, B><<<blocks, th, 0, s>>>(b, v, T, N, c, vstar); HN_CHECK_LAUNCH(); return 0; }
    HN_FUSED_PAIRS(HN_X)
#undef HN_X
  }
  // bins are independent row sets: their kernels run concurrently (fork/join)
  launch_forked(as_stream(stream), nbins, [&](int i, cudaStream_t s) {
    StepBins one = single_bin(b, i);
    const int64_t bl = ceil_div(one.K[0], th);
    if (bl == 0) return;
#define HN_MOM(DD, WW) momentum_kernel<DD, WW><<<bl, th, 0, s>>>(one, v, T, N, c, vstar)
    HN_WIDTH_DISPATCH(d, one.width[0], HN_MOM);
#undef HN_MOM
  });
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT int hn_div_rhs(int nbins, const int64_t* bin_K_host, const int* bin_width_host,
                         const int* const* bin_rows_host, const int* const* bin_idx_host,
                         const double* const* bin_w_host, const int* d_plane_host, int d, const double* vstar,
                         int64_t N, double dt, double* rhs, void* stream) {
  if (!ok_bins(nbins, bin_width_host) || (d != 2 && d != 3)) return 1;
  StepBins b{};
  int64_t blocks;
  const int th = 128;
  fill_bins(b, nbins, bin_K_host, bin_width_host, bin_rows_host, bin_idx_host, bin_w_host, th, &blocks);
  for (int a = 0; a < d; ++a) b.d_plane[a] = d_plane_host[a];
  if (blocks == 0) return 0;
  int wa, wb;
  if (fused_pair(b, d, &wa, &wb)) {
    cudaStream_t s = as_stream(stream);
#define HN_X(DD, A, B) \
    if (d == DD && wa == A && wb == B) { div_rhs_fused_kernel<DD, A, B><<<blocks, th, 0, s>>>(b, vstar, N, dt, rhs); HN_CHECK_LAUNCH(); return 0; }
    HN_FUSED_PAIRS(HN_X)
#undef HN_X
  }
  launch_forked(as_stream(stream), nbins, [&](int i, cudaStream_t s) {
    StepBins one = single_bin(b, i);
    const int64_t bl = ceil_div(one.K[0], th);
    if (bl == 0) return;
#define HN_DIV(DD, WW) div_rhs_kernel<DD, WW><<<bl, th, 0, s>>>(one, vstar, N, dt, rhs, i == 0)
    HN_WIDTH_DISPATCH(d, one.width[0], HN_DIV);
#undef HN_DIV
  });
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT int hn_correct_temperature(int nbins, const int64_t* bin_K_host, const int* bin_width_host,
                                     const int* const* bin_rows_host, const int* const* bin_idx_host,
                                     const double* const* bin_w_host, int lap_plane, const int* d_plane_host, int d,
                                     const double* vstar, const double* p, const double* T, int64_t N, double dt,
                                     double* vout, double* Tout, int* flags, const double* hyper_coef,
                                     const double* hyper_lap2, void* stream) {
  if (!ok_bins(nbins, bin_width_host) || (d != 2 && d != 3)) return 1;
  if ((hyper_coef == nullptr) != (hyper_lap2 == nullptr)) return 2;
  const HyperT hy{hyper_coef, hyper_lap2};
  StepBins b{};
  int64_t blocks;
  const int th = 128;
  fill_bins(b, nbins, bin_K_host, bin_width_host, bin_rows_host, bin_idx_host, bin_w_host, th, &blocks);
  b.lap_plane = lap_plane;
  for (int a = 0; a < d; ++a) b.d_plane[a] = d_plane_host[a];
  if (blocks == 0) return 0;
  int wa, wb;
  if (fused_pair(b, d, &wa, &wb)) {
    cudaStream_t s = as_stream(stream);
#define HN_X(DD, A, B) \
    if (d == DD && wa == A && wb == B) { correct_temp_fused_kernel<DD, A, B><<<blocks, th, 0, s>>>(b, vstar, p, T, N, dt, vout, Tout, flags, hy); HN_CHECK_LAUNCH(); return 0; }
    HN_FUSED_PAIRS(HN_X)
#undef HN_X
  }
  launch_forked(as_stream(stream), nbins, [&](int i, cudaStream_t s) {
    StepBins one = single_bin(b, i);
    const int64_t bl = ceil_div(one.K[0], th);
    if (bl == 0) return;
#define HN_COR(DD, WW) correct_temp_kernel<DD, WW><<<bl, th, 0, s>>>(one, vstar, p, T, N, dt, vout, Tout, flags, hy)
    HN_WIDTH_DISPATCH(d, one.width[0], HN_COR);
#undef HN_COR
  });
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT int hn_temperature_bc(const int* dir_idx, const double* dir_val, int64_t ndir, const int64_t* neu_rowptr,
                                const int* neu_cols, const double* neu_vals, const int* neu_idx,
                                const double* neu_diag, const uint8_t* is_neu, int64_t nneu, double* T,
                                int* flags, int* latch, const int* pstatus, void* stream) {
  if (latch && !flags) return 1;
  const int64_t n = ndir + nneu;
  if (n == 0 && !latch) return 0;
  const int th = 128;
  temperature_bc_kernel<<<n > 0 ? ceil_div(n, th) : 1, th, 0, as_stream(stream)>>>(
      dir_idx, dir_val, ndir, neu_rowptr, neu_cols, neu_vals, neu_idx, neu_diag, is_neu, nneu, T, flags, latch,
      pstatus);
  HN_CHECK_LAUNCH();
  return 0;
}


HN_EXPORT int hn_csr_matvec(const int64_t* rowptr, const int* cols, const double* vals, const double* x,
                            int64_t nrows, double* y, void* stream) {
  if (nrows == 0) return 0;
  const int th = 128;
  csr_matvec_kernel<<<ceil_div(nrows, th), th, 0, as_stream(stream)>>>(rowptr, cols, vals, x, nrows, y);
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT int hn_csr_residual(const int64_t* rowptr, const int* cols, const double* vals, const double* x,
                              const double* b, int64_t nrows, double* y, void* stream) {
  if (nrows == 0) return 0;
  const int th = 128;
  csr_residual_kernel<<<ceil_div(nrows, th), th, 0, as_stream(stream)>>>(rowptr, cols, vals, x, b, nrows, y);
  HN_CHECK_LAUNCH();
  return 0;
}
