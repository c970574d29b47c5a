// K13: 2-norm condition numbers of the local weight systems (the weights diagnostic).
//
// Reference: _batched_mon_weights / _batched_rbf_weights with with_kappa=True
// (pkg/src/hybridnodes/approx.py:229-233, 285-289) take np.linalg.svd of every local
// system and report s_max / s_min (inf when s_min == 0), on the stencil's local coordinates
// (rel = pts - centre, divided by the largest |rel|, approx.py:245-250).
//
// One warp per system, rows in registers (lane l owns rows l and l + 32):
//   RBF-FD: the saddle matrix [[A P], [P^T 0]] is symmetric, so its singular values are the
//           |eigenvalues|: kappa = max|lambda| / min|lambda|;
//   MON:    the monomial matrix M is not; its singular values are the square roots of the
//           eigenvalues of M M^T: kappa = sqrt(lambda_max / lambda_min).
// The symmetric matrix is reduced to tridiagonal form by Householder reflections (backward
// stable, like LAPACK's reduction), then the few eigenvalues kappa needs -- the extreme
// ones and, for the indefinite saddle matrix, the two bracketing 0 -- are found by Sturm-
// sequence multisection: each round, the 32 lanes count eigenvalues below 32 points of the
// current interval at once (33x narrower per round).  Accuracy: eigenvalues to ~eps ||S||
// absolute, as the SVD's singular values, so kappa agrees to ~kappa * eps relative.
#include <math_constants.h>

#include "hn_common.cuh"

namespace hn {
namespace {

constexpr int kKapWarps = 4;

template <int D>
__device__ __forceinline__ double mono(int m, const double* y) {
  // [1, x_a.., then degree-2 products in lexicographic order] (approx.py:69-78)
  if (m == 0) return 1.0;
  if (m <= D) return y[m - 1];
  int k = m - 1 - D;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = a; b < D; ++b) {
      if (k == 0) return y[a] * y[b];
      --k;
    }
  return 0.0;
}

// number of eigenvalues of the tridiagonal (d, e) below x (LAPACK dstebz-style pivmin guard)
template <int NS>
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, double x, double pivmin) {
  int c = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  c += q < 0.0;
#pragma unroll 4
  for (int i = 1; i < NS; ++i) {
    q = (d[i] - x) - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    c += q < 0.0;
  }
  return c;
}

// the k-th smallest eigenvalue (0-based), every lane of the warp cooperating
template <int NS>
__device__ double kth_eigenvalue(const double* d, const double* e2, int k, double lo, double hi, double pivmin,
                                 int lane) {
  for (int round = 0; round < 14; ++round) {
    const double width = hi - lo;
    if (!(width > 2.2e-16 * fmax(fabs(lo), fabs(hi))) || !(width > pivmin)) break;
    const double xl = lo + width * (lane + 1) / 33.0;
    const bool above = sturm_count<NS>(d, e2, xl, pivmin) > k;  // eigenvalue k lies below xl
    const unsigned m = __ballot_sync(0xffffffffu, above);
    const int first = m ? __ffs(m) - 1 : 32;  // first point with more than k eigenvalues below
    const double nlo = first == 0 ? lo : lo + width * first / 33.0;
    const double nhi = first == 32 ? hi : lo + width * (first + 1) / 33.0;
    lo = nlo;
    hi = nhi;
  }
  return 0.5 * (lo + hi);
}

template <int D, int NST, bool MON>
__global__ void __launch_bounds__(kKapWarps * 32) kappa_kernel(const double* __restrict__ pos, int ps,
                                                               const int* __restrict__ idx, int64_t rs, int64_t cs,
                                                               const int* __restrict__ centers, int64_t K,
                                                               double* __restrict__ out) {
  constexpr int NQ = D == 2 ? 6 : 10;
  constexpr int NS = MON ? NST : NST + NQ;  // system size
  constexpr int RPL = (NS + 31) / 32;       // rows per lane
  static_assert(NS <= 64, "two rows per lane at most");
  __shared__ double sy[kKapWarps][NST][D];
  __shared__ double sd[kKapWarps][NS], se2[kKapWarps][NS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t k = static_cast<int64_t>(blockIdx.x) * kKapWarps + warp;
  if (k >= K) return;
  // local coordinates: shift to the centre, divide by the largest distance (approx.py:245-250)
  double yl[D], r2 = 0.0;
  if (lane < NST) {
    const int c = centers ? __ldg(centers + k) : __ldg(idx + k * rs);
    const int j = __ldg(idx + k * rs + lane * cs);
#pragma unroll
    for (int a = 0; a < D; ++a) {
      yl[a] = __ldg(pos + static_cast<int64_t>(j) * ps + a) - __ldg(pos + static_cast<int64_t>(c) * ps + a);
      r2 += yl[a] * yl[a];
    }
  }
  double scale = lane < NST ? sqrt(r2) : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
  if (lane < NST)
#pragma unroll
    for (int a = 0; a < D; ++a) sy[warp][lane][a] = yl[a] / scale;
  __syncwarp();

  // ---- the symmetric matrix S, rows in registers ----
  double S[RPL][NS];
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = lane + 32 * r;
#pragma unroll
    for (int j = 0; j < NS; ++j) S[r][j] = 0.0;
    if (i >= NS) continue;
    if constexpr (MON) {  // S = M M^T, M[row][node]: 1, y_a, y_a^2 (approx.py:158-170)
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < NST; ++c) {
          const double* y = sy[warp][c];
          auto mrow = [&](int row) {
            if (row == 0) return 1.0;
            if (row <= D) return y[row - 1];
            return y[row - 1 - D] * y[row - 1 - D];
          };
          s = fma(mrow(i), mrow(j), s);
        }
        S[r][j] = s;
      }
    } else {
      double yi[D];
      if (i < NST) {
#pragma unroll
        for (int a = 0; a < D; ++a) yi[a] = sy[warp][i][a];
      }
#pragma unroll
      for (int j = 0; j < NST; ++j) {
        const double* yj = sy[warp][j];
        if (i < NST) {
          double q = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) q += (yi[a] - yj[a]) * (yi[a] - yj[a]);
          const double rr = sqrt(q);
          S[r][j] = rr * rr * rr;
        } else {
          S[r][j] = mono<D>(i - NST, yj);
        }
      }
#pragma unroll
      for (int m = 0; m < NQ; ++m) S[r][NST + m] = i < NST ? mono<D>(m, yi) : 0.0;
    }
  }

  // ---- Householder tridiagonalisation: S <- H S H, column by column ----
  auto shfl_row = [&](double (&Sr)[RPL][NS], int row, int col) {  // S[row][col] from its owner lane
    double v = 0.0;
#pragma unroll
    for (int r = 0; r < RPL; ++r) v = (row >> 5) == r ? Sr[r][col] : v;
    return __shfl_sync(0xffffffffu, v, row & 31);
  };
#pragma unroll
  for (int c = 0; c < NS - 2; ++c) {
    // v = x - alpha e_1 over rows c+1.., x = column c below the diagonal
    double vr[RPL], xnorm2 = 0.0;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      vr[r] = (i > c && i < NS) ? S[r][c] : 0.0;
      xnorm2 += vr[r] * vr[r];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xnorm2 += __shfl_xor_sync(0xffffffffu, xnorm2, o);
    const double x0 = shfl_row(S, c + 1, c);
    const double alpha = x0 >= 0.0 ? -sqrt(xnorm2) : sqrt(xnorm2);
    const double vnorm2 = xnorm2 - x0 * x0 + (x0 - alpha) * (x0 - alpha);
    if (!(vnorm2 > 0.0)) continue;  // column already reduced
#pragma unroll
    for (int r = 0; r < RPL; ++r)
      if (lane + 32 * r == c + 1) vr[r] = x0 - alpha;
    const double beta = 2.0 / vnorm2;
    // p = beta S v;  K = beta/2 p.v;  w = p - K v  (v_j broadcast from its owner lane)
    auto vbc = [&](int j) {
      double v = 0.0;
#pragma unroll
      for (int r = 0; r < RPL; ++r) v = (j >> 5) == r ? vr[r] : v;
      return __shfl_sync(0xffffffffu, v, j & 31);
    };
    double pr[RPL], pv = 0.0;
#pragma unroll
    for (int r = 0; r < RPL; ++r) pr[r] = 0.0;
#pragma unroll
    for (int j = c + 1; j < NS; ++j) {
      const double v = vbc(j);
#pragma unroll
      for (int r = 0; r < RPL; ++r) pr[r] = fma(S[r][j], v, pr[r]);
    }
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      pr[r] *= beta;
      pv += (lane + 32 * r < NS) ? pr[r] * vr[r] : 0.0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
    const double Kc = 0.5 * beta * pv;
    double wr[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) wr[r] = pr[r] - Kc * vr[r];
#pragma unroll
    for (int j = c; j < NS; ++j) {
      double w = 0.0;
#pragma unroll
      for (int r = 0; r < RPL; ++r) w = (j >> 5) == r ? wr[r] : w;
      const double wj = __shfl_sync(0xffffffffu, w, j & 31);
      const double vj = j > c ? vbc(j) : 0.0;
#pragma unroll
      for (int r = 0; r < RPL; ++r) S[r][j] = S[r][j] - vr[r] * wj - wr[r] * vj;
    }
  }
  // ---- the tridiagonal (d, e^2) to shared memory ----
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = lane + 32 * r;
    if (i < NS) {
      double di = 0.0, ei = 0.0;
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        di = j == i ? S[r][j] : di;
        ei = j == i + 1 ? S[r][j] : ei;
      }
      sd[warp][i] = di;
      se2[warp][i] = ei * ei;
    }
  }
  __syncwarp();
  const double* d = sd[warp];
  const double* e2 = se2[warp];
  // Gershgorin interval and the pivot guard
  double lo = 1e300, hi = -1e300, tn = 0.0;
  for (int i = 0; i < NS; ++i) {
    const double off = (i > 0 ? sqrt(e2[i - 1]) : 0.0) + (i + 1 < NS ? sqrt(e2[i]) : 0.0);
    lo = fmin(lo, d[i] - off);
    hi = fmax(hi, d[i] + off);
    tn = fmax(tn, fabs(d[i]) + off);
  }
  const double pivmin = fmax(1e-300, 2.2e-16 * 2.2e-16 * tn * tn / fmax(tn, 1e-300));
  lo -= 4.4e-16 * tn + pivmin;
  hi += 4.4e-16 * tn + pivmin;
  double kappa;
  if constexpr (MON) {  // eigenvalues of M M^T = singular values squared
    const double lmax = kth_eigenvalue<NS>(d, e2, NS - 1, lo, hi, pivmin, lane);
    const double lmin = kth_eigenvalue<NS>(d, e2, 0, lo, hi, pivmin, lane);
    kappa = lmin > 0.0 ? sqrt(lmax / lmin) : CUDART_INF;
  } else {
    const double l0 = kth_eigenvalue<NS>(d, e2, 0, lo, hi, pivmin, lane);
    const double ln = kth_eigenvalue<NS>(d, e2, NS - 1, lo, hi, pivmin, lane);
    const int nneg = sturm_count<NS>(d, e2, 0.0, pivmin);
    double amin = CUDART_INF;
    if (nneg > 0) amin = fmin(amin, fabs(kth_eigenvalue<NS>(d, e2, nneg - 1, lo, fmin(hi, 0.0), pivmin, lane)));
    if (nneg < NS) amin = fmin(amin, fabs(kth_eigenvalue<NS>(d, e2, nneg, fmax(lo, 0.0), hi, pivmin, lane)));
    const double amax = fmax(fabs(l0), fabs(ln));
    kappa = amin > 0.0 ? amax / amin : CUDART_INF;
  }
  if (lane == 0) out[k] = kappa;
}

template <int D, int NST, bool MON>
cudaError_t launch_kappa(const double* pos, int ps, const int* idx, int64_t rs, int64_t cs, const int* centers,
                         int64_t K, double* out, cudaStream_t s) {
  kappa_kernel<D, NST, MON><<<ceil_div(K, kKapWarps), kKapWarps * 32, 0, s>>>(pos, ps, idx, rs, cs, centers, K, out);
  return cudaGetLastError();
}

}  // namespace
}  // namespace hn

using namespace hn;

// kappa (2-norm condition number) of K local systems.  pos: node coordinates with row stride
// ps (>= d) fp64; stencil node j of system k at idx[k * rs + j * cs] (row-major: rs = n,
// cs = 1; an ELL bin: rs = 1, cs = K); centers (may be NULL: node 0 of each stencil) the
// centre node ids; out K fp64.  mon != 0: the monomial system (n = 2d+1); else the RBF-FD
// saddle system (n + q).  Returns 2 for an unsupported (d, n).
HN_EXPORT int hn_condition_numbers(const double* pos, int ps, int d, const int* idx, int64_t rs, int64_t cs,
                                   const int* centers, int64_t K, int n, int mon, double* out, void* stream) {
  if (K == 0) return 0;
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaErrorInvalidValue;
#define HN_KAP(DD, NN, MM) e = launch_kappa<DD, NN, MM>(pos, ps, idx, rs, cs, centers, K, out, s)
  if (d == 2 && mon && n == 5) HN_KAP(2, 5, true);
  else if (d == 3 && mon && n == 7) HN_KAP(3, 7, true);
  else if (d == 2 && !mon && n == 12) HN_KAP(2, 12, false);
  else if (d == 3 && !mon && n == 20) HN_KAP(3, 20, false);
  else if (d == 3 && !mon && n == 30) HN_KAP(3, 30, false);
  else return 2;
#undef HN_KAP
  return e == cudaSuccess ? 0 : -static_cast<int>(e);
}
