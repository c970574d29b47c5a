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
};

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
        const double rhs = __dsub_rn(__dadd_rn(-adv, __dmul_rn(c.Pr, 0.0)), __dmul_rn(c.buoy[cc], tdelta));
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
#pragma unroll
    for (int cc = 0; cc < D; ++cc) {
      double fv[W];
#pragma unroll
      for (int j = 0; j < W; ++j) fv[j] = __ldg(v + cc * N + id[j]);
      double adv = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double g = ssum<W>(wb + b.d_plane[a] * ps, K, k, fv);
        const double t = __dmul_rn(vi[a], g);
        adv = (a == 0) ? t : __dadd_rn(adv, t);
      }
      const double lap = ssum<W>(wb + b.lap_plane * ps, K, k, fv);
      const double rhs = __dsub_rn(__dadd_rn(-adv, __dmul_rn(c.Pr, lap)), __dmul_rn(c.buoy[cc], tdelta));
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
    double div = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double fv[W];
#pragma unroll
      for (int j = 0; j < W; ++j) fv[j] = __ldg(vs + a * N + id[j]);
      const double s = ssum<W>(b.w[bin] + b.d_plane[a] * ps, K, k, fv);
      div = (a == 0) ? s : __dadd_rn(div, s);
    }
    rhs[row] = __ddiv_rn(div, dt);
  }
}

template <int D, int W>
__global__ void __launch_bounds__(128, (W <= 7 ? 8 : (W <= 12 ? 6 : (W <= 20 ? 4 : 2))))
div_rhs_kernel(StepBins b, const double* __restrict__ vs, int64_t N, double dt,
               double* __restrict__ rhs) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (blockIdx.x == 0 && threadIdx.x == 0) rhs[N] = 0.0;  // bordered gauge equation
  if (k >= b.K[0]) return;
  div_row<D, W>(b, 0, k, vs, N, 0.0, dt, rhs);
}

// ---- K10: velocity correction + temperature advection-diffusion (solver.py:317-331, 345-357) ----
template <int D, int W>
__device__ __forceinline__ void correct_temp_row(const StepBins& b, int bin, int64_t k, const double* __restrict__ vs,
                                                 const double* __restrict__ p, const double* __restrict__ T,
                                                 int64_t N, double dt, double* __restrict__ vout,
                                                 double* __restrict__ Tout, int* __restrict__ flags) {
  const int64_t K = b.K[bin];
  const int row = __ldg(b.rows[bin] + k);
  double vn[D];
  double tn;
  if constexpr (W == 0) {
#pragma unroll
    for (int a = 0; a < D; ++a) vn[a] = 0.0;
    // empty operator rows: conv = 0, lap = 0  ->  T + dt * (-0 + 0)
    const double Ti = __ldg(T + row);
    tn = __dadd_rn(Ti, __dmul_rn(dt, __dadd_rn(-0.0, 0.0)));
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
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double gp = ssum<W>(wb + b.d_plane[a] * ps, K, k, fp);
      vn[a] = __dsub_rn(__ldg(vs + a * N + row), __dmul_rn(dt, gp));
    }
    double conv = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double gt = ssum<W>(wb + b.d_plane[a] * ps, K, k, ft);
      const double t = __dmul_rn(vn[a], gt);
      conv = (a == 0) ? t : __dadd_rn(conv, t);
    }
    const double lap = ssum<W>(wb + b.lap_plane * ps, K, k, ft);
    tn = __dadd_rn(__ldg(T + row), __dmul_rn(dt, __dadd_rn(-conv, lap)));
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
                    double* __restrict__ Tout, int* __restrict__ flags) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= b.K[0]) return;
  correct_temp_row<D, W>(b, 0, k, vs, p, T, N, dt, vout, Tout, flags);
}

// ---- K11: temperature boundary conditions (solver.py:334-342) ----
__global__ void dirichlet_kernel(const int* __restrict__ idx, const double* __restrict__ val, int64_t n,
                                 double* __restrict__ T) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) T[idx[i]] = val[i];
}

// Insulated rows: T[b] = -(sum_j W_bj t0_j) / W_bb with t0 = T, Neumann entries zeroed.
// The Neumann block W[:, neu] is diagonal (boundary stencils exclude every other
// boundary node), so SuperLU's solve of it is an elementwise division.
__global__ void neumann_kernel(const int64_t* __restrict__ rowptr, const int* __restrict__ cols,
                               const double* __restrict__ vals, const int* __restrict__ neu_idx,
                               const double* __restrict__ diag, const uint8_t* __restrict__ is_neu, int64_t nrows,
                               double* __restrict__ T) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  double acc = 0.0;
  for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
    const int c = cols[e];
    const double t0 = is_neu[c] ? 0.0 : T[c];
    acc = __dadd_rn(acc, __dmul_rn(vals[e], t0));
  }
  T[neu_idx[r]] = __ddiv_rn(-acc, diag[r]);
}

// ---- generic sequential CSR matvec (scipy csr_matvec order), thread per row ----
__global__ void csr_matvec_kernel(const int64_t* __restrict__ rowptr, const int* __restrict__ cols,
                                  const double* __restrict__ vals, const double* __restrict__ x, int64_t nrows,
                                  double* __restrict__ y) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  double acc = 0.0;
  const int64_t e1 = __ldg(rowptr + r + 1);
  for (int64_t e = __ldg(rowptr + r); e < e1; ++e) acc = __dadd_rn(acc, __dmul_rn(__ldg(vals + e), __ldg(x + __ldg(cols + e))));
  y[r] = acc;
}

// y = b - A x  (r0 of BiCGStab; scipy: b - matvec(x))
__global__ void csr_residual_kernel(const int64_t* __restrict__ rowptr, const int* __restrict__ cols,
                                    const double* __restrict__ vals, const double* __restrict__ x,
                                    const double* __restrict__ b, int64_t nrows, double* __restrict__ y) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  double acc = 0.0;
  const int64_t e1 = __ldg(rowptr + r + 1);
  for (int64_t e = __ldg(rowptr + r); e < e1; ++e) acc = __dadd_rn(acc, __dmul_rn(__ldg(vals + e), __ldg(x + __ldg(cols + e))));
  y[r] = __dsub_rn(b[r], acc);
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
                          const double* buoy_host, int zero_boundary, double* vstar, void* stream) {
  if (!ok_bins(nbins, bin_width_host) || (d != 2 && d != 3)) return 1;
  StepBins b{};
  int64_t blocks;
  const int th = 128;
  fill_bins(b, nbins, bin_K_host, bin_width_host, bin_rows_host, bin_idx_host, bin_w_host, th, &blocks);
  b.lap_plane = lap_plane;
  for (int a = 0; a < d; ++a) b.d_plane[a] = d_plane_host[a];
  MomentumCoef c{dt, Pr, t_ref, {0, 0, 0}, zero_boundary};
  for (int a = 0; a < d; ++a) c.buoy[a] = buoy_host[a];
  if (blocks == 0) return 0;
  cudaStream_t s = as_stream(stream);
  for (int i = 0; i < nbins; ++i) {
    StepBins one = single_bin(b, i);
    const int64_t bl = ceil_div(one.K[0], th);
    if (bl == 0) continue;
#define HN_MOM(DD, WW) momentum_kernel<DD, WW><<<bl, th, 0, s>>>(one, v, T, N, c, vstar)
    HN_WIDTH_DISPATCH(d, one.width[0], HN_MOM);
#undef HN_MOM
  }
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
  cudaStream_t s = as_stream(stream);
  for (int i = 0; i < nbins; ++i) {
    StepBins one = single_bin(b, i);
    const int64_t bl = ceil_div(one.K[0], th);
    if (bl == 0) continue;
#define HN_DIV(DD, WW) div_rhs_kernel<DD, WW><<<bl, th, 0, s>>>(one, vstar, N, dt, rhs)
    HN_WIDTH_DISPATCH(d, one.width[0], HN_DIV);
#undef HN_DIV
  }
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT int hn_correct_temperature(int nbins, const int64_t* bin_K_host, const int* bin_width_host,
                                     const int* const* bin_rows_host, const int* const* bin_idx_host,
                                     const double* const* bin_w_host, int lap_plane, const int* d_plane_host, int d,
                                     const double* vstar, const double* p, const double* T, int64_t N, double dt,
                                     double* vout, double* Tout, int* flags, void* stream) {
  if (!ok_bins(nbins, bin_width_host) || (d != 2 && d != 3)) return 1;
  StepBins b{};
  int64_t blocks;
  const int th = 128;
  fill_bins(b, nbins, bin_K_host, bin_width_host, bin_rows_host, bin_idx_host, bin_w_host, th, &blocks);
  b.lap_plane = lap_plane;
  for (int a = 0; a < d; ++a) b.d_plane[a] = d_plane_host[a];
  if (blocks == 0) return 0;
  cudaStream_t s = as_stream(stream);
  for (int i = 0; i < nbins; ++i) {
    StepBins one = single_bin(b, i);
    const int64_t bl = ceil_div(one.K[0], th);
    if (bl == 0) continue;
#define HN_COR(DD, WW) correct_temp_kernel<DD, WW><<<bl, th, 0, s>>>(one, vstar, p, T, N, dt, vout, Tout, flags)
    HN_WIDTH_DISPATCH(d, one.width[0], HN_COR);
#undef HN_COR
  }
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT int hn_temperature_bc(const int* dir_idx, const double* dir_val, int64_t ndir, const int64_t* neu_rowptr,
                                const int* neu_cols, const double* neu_vals, const int* neu_idx,
                                const double* neu_diag, const uint8_t* is_neu, int64_t nneu, double* T,
                                void* stream) {
  cudaStream_t s = as_stream(stream);
  const int th = 256;
  if (ndir > 0) {
    dirichlet_kernel<<<ceil_div(ndir, th), th, 0, s>>>(dir_idx, dir_val, ndir, T);
    HN_CHECK_LAUNCH();
  }
  if (nneu > 0) {
    neumann_kernel<<<ceil_div(nneu, th), th, 0, s>>>(neu_rowptr, neu_cols, neu_vals, neu_idx, neu_diag, is_neu, nneu, T);
    HN_CHECK_LAUNCH();
  }
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
