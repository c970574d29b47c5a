// K9 driver: the pressure Poisson solve of one time step as ONE device-driven graph.
//
// Reference: pressure_solve (pkg/src/hybridnodes/solver.py:283-314) calls
//   scipy.sparse.linalg.bicgstab(A, rhs, x0, M=LU.solve, rtol=tol, atol=0, maxiter)
// with the complete SuperLU factorisation as preconditioner (solver.py:213-214).  This file
// runs scipy's BiCGStab (scipy 1.18, _isolve/iterative.py: same recurrences, breakdown
// tests rhotol = omegatol = eps^2, stopping rule ||r|| < max(0, rtol ||b||), numpy operation
// order in every vector update) with every scalar on the device: dot products are fixed-
// grid partial sums (deterministic) reduced by one-block control kernels that also take the
// branch decisions.  The iteration is the body of a CUDA-graph WHILE node whose condition
// the last control kernel sets, so a solve needs no host round trip at all; once a branch
// finishes the loop (converged, breakdown, maxiter) the remaining kernels of that body pass
// return at once (they test the device `done` word).  One body pass = 2 preconditioner
// applications (permute, supernodal L, supernodal U, permute) + 2 A-matvecs; with the
// complete LU the loop normally exits at the first half-step check.
//
// Status (device int[2]): [info, iterations] with scipy's info convention (0 converged,
// maxiter = not converged, -10 / -11 breakdowns).  The caller decides what a failure means
// (the reference retries with lgmres, solver.py:306-312).
#include <cstdlib>

#include "pressure.cuh"

namespace hn {
namespace {

constexpr int kParts = 296;   // fixed partial-sum grid: 2 blocks per SM, results independent of timing
constexpr int kThr = 256;
constexpr double kRhoTol = 4.930380657631324e-32;  // eps^2 (scipy rhotol = omegatol)

enum Scalar { kBnrm = 0, kAtol, kRho, kRhoPrev, kAlpha, kOmega, kBeta, kNumScalars = 8 };
enum State { kDone = 0, kInfo, kIter, kHalf, kSpecial, kUseRes, kNumState = 8 };  // kSpecial: 1 non-finite b, 2 b == 0

__device__ __forceinline__ double block_sum(double v, double* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < (kThr >> 5) ? sm[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  __syncthreads();
  return v;  // valid in thread 0
}

__device__ __forceinline__ double block_max(double v, double* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < (kThr >> 5) ? sm[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  __syncthreads();
  return v;
}

// scipy csr_matvec order: one row, entries in storage order, sequential adds
__device__ __forceinline__ double row_dot(const int64_t* __restrict__ rowptr, const int* __restrict__ cols,
                                          const double* __restrict__ vals, const double* __restrict__ x, int64_t r) {
  const int64_t e1 = __ldg(rowptr + r + 1);
  double acc = 0.0;
  for (int64_t e = __ldg(rowptr + r); e < e1; e += 8) {
    int c[8];
    double v[8], xv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      c[k] = e + k < e1 ? __ldg(cols + e + k) : -1;
      v[k] = e + k < e1 ? __ldg(vals + e + k) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) xv[k] = c[k] >= 0 ? x[c[k]] : 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (c[k] >= 0) acc = __dadd_rn(acc, __dmul_rn(v[k], xv[k]));
  }
  return acc;
}

#define GRID_LOOP(i, n) \
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x; i < (n); i += static_cast<int64_t>(kParts) * kThr)

// ---- set-up kernels (no done test: they run first) -----------------------------------
__global__ void init_state_kernel(int* __restrict__ st) {
  if (threadIdx.x < kNumState) st[threadIdx.x] = 0;
}

// partials of b.b
__global__ void __launch_bounds__(kThr) bnorm_partial_kernel(const double* __restrict__ b, int64_t n,
                                                             double* __restrict__ part) {
  __shared__ double sm[32];
  double s = 0.0;
  GRID_LOOP(i, n) s += b[i] * b[i];
  s = block_sum(s, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// x = x0 (x0 != x) or 0 (x0 == NULL); partial max|x| for the r0 choice
__global__ void __launch_bounds__(kThr) init_x_kernel(const double* __restrict__ x0, double* __restrict__ x, int64_t n,
                                                      double* __restrict__ part, const int* __restrict__ st) {
  __shared__ double sm[32];
  if (st[kDone]) return;
  double m = 0.0;
  GRID_LOOP(i, n) {
    const double v = x0 ? x0[i] : 0.0;
    if (x0 != x) x[i] = v;
    m = fmax(m, fabs(v));
  }
  m = block_max(m, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = m;
}

// r = b - A x if any x != 0 else b (scipy: r = b - A@x if x.any() else b.copy()); rt = r;
// partials of r.r (the loop-top norm) and rt.r (= r.r here)
__global__ void __launch_bounds__(kThr) init_r_kernel(const int64_t* __restrict__ rowptr, const int* __restrict__ cols,
                                                      const double* __restrict__ vals, const double* __restrict__ x,
                                                      const double* __restrict__ b, int64_t n, double* __restrict__ r,
                                                      double* __restrict__ rt, double* __restrict__ part,
                                                      const int* __restrict__ st) {
  __shared__ double sm[32];
  if (st[kDone]) return;
  const bool res = st[kUseRes] != 0;
  double s = 0.0;
  GRID_LOOP(i, n) {
    const double v = res ? __dsub_rn(b[i], row_dot(rowptr, cols, vals, x, i)) : b[i];
    r[i] = v;
    rt[i] = v;
    s += v * v;
  }
  s = block_sum(s, sm);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    part[kParts + blockIdx.x] = s;
  }
}

// ---- loop kernels (return at once when done) -----------------------------------------
// p = r (first pass) or p = ((p - omega v) * beta) + r
__global__ void __launch_bounds__(kThr) p_update_kernel(double* __restrict__ p, const double* __restrict__ v,
                                                        const double* __restrict__ r, int64_t n,
                                                        const double* __restrict__ sc, const int* __restrict__ st) {
  if (st[kDone]) return;
  const bool first = st[kIter] == 0;
  const double omega = sc[kOmega], beta = sc[kBeta];
  GRID_LOOP(i, n) p[i] = first ? r[i] : __dadd_rn(__dmul_rn(__dsub_rn(p[i], __dmul_rn(omega, v[i])), beta), r[i]);
}

__global__ void permute_in_skip_kernel(const int* __restrict__ perm_r, const double* __restrict__ b, int64_t n,
                                       double* __restrict__ y, const int* __restrict__ st) {
  if (st[kDone]) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[perm_r[i]] = b[i];
}
__global__ void permute_out_skip_kernel(const int* __restrict__ perm_c, const double* __restrict__ w, int64_t n,
                                        double* __restrict__ x, const int* __restrict__ st) {
  if (st[kDone]) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = w[perm_c[i]];
}

// y = A x with partials of a1.y (and a2.y when a2 != NULL)
__global__ void __launch_bounds__(kThr) matvec_dot_kernel(const int64_t* __restrict__ rowptr,
                                                          const int* __restrict__ cols, const double* __restrict__ vals,
                                                          const double* __restrict__ x, int64_t n,
                                                          double* __restrict__ y, const double* __restrict__ a1,
                                                          const double* __restrict__ a2, double* __restrict__ part,
                                                          const int* __restrict__ st) {
  __shared__ double sm[32];
  if (st[kDone]) return;
  double s1 = 0.0, s2 = 0.0;
  // a2 may be y itself (t.t of the omega step): the product then uses the value just formed --
  // reading it back through the restrict-qualified a2 may be scheduled before the store to y
  // and return the previous contents of the buffer
  const bool a2_is_y = a2 == y;
  GRID_LOOP(i, n) {
    const double v = row_dot(rowptr, cols, vals, x, i);
    y[i] = v;
    s1 += a1[i] * v;
    if (a2) s2 += (a2_is_y ? v : a2[i]) * v;
  }
  s1 = block_sum(s1, sm);
  if (a2) s2 = block_sum(s2, sm);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s1;
    part[kParts + blockIdx.x] = s2;
  }
}

// s = r - alpha v (in place in r); partials of s.s
__global__ void __launch_bounds__(kThr) s_update_kernel(double* __restrict__ r, const double* __restrict__ v, int64_t n,
                                                        const double* __restrict__ sc, double* __restrict__ part,
                                                        const int* __restrict__ st) {
  __shared__ double sm[32];
  if (st[kDone]) return;
  const double alpha = sc[kAlpha];
  double s = 0.0;
  GRID_LOOP(i, n) {
    const double v2 = __dsub_rn(r[i], __dmul_rn(alpha, v[i]));
    r[i] = v2;
    s += v2 * v2;
  }
  s = block_sum(s, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// converged at the half step: x += alpha phat
__global__ void half_x_kernel(double* __restrict__ x, const double* __restrict__ phat, int64_t n,
                              const double* __restrict__ sc, const int* __restrict__ st) {
  if (!st[kHalf]) return;
  const double alpha = sc[kAlpha];
  GRID_LOOP(i, n) x[i] = __dadd_rn(x[i], __dmul_rn(alpha, phat[i]));
}

// x += alpha phat; x += omega shat; r = s - omega t; partials of r.r and rt.r for the next top
__global__ void __launch_bounds__(kThr) xr_update_kernel(double* __restrict__ x, const double* __restrict__ phat,
                                                         const double* __restrict__ shat, double* __restrict__ r,
                                                         const double* __restrict__ t, const double* __restrict__ rt,
                                                         int64_t n, const double* __restrict__ sc,
                                                         double* __restrict__ part, const int* __restrict__ st) {
  __shared__ double sm[32];
  if (st[kDone]) return;
  const double alpha = sc[kAlpha], omega = sc[kOmega];
  double s1 = 0.0, s2 = 0.0;
  GRID_LOOP(i, n) {
    x[i] = __dadd_rn(__dadd_rn(x[i], __dmul_rn(alpha, phat[i])), __dmul_rn(omega, shat[i]));
    const double v = __dsub_rn(r[i], __dmul_rn(omega, t[i]));
    r[i] = v;
    s1 += v * v;
    s2 += rt[i] * v;
  }
  s1 = block_sum(s1, sm);
  s2 = block_sum(s2, sm);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s1;
    part[kParts + blockIdx.x] = s2;
  }
}

// ---- control kernels: one block reduces the partials and takes scipy's branches ----------
enum Ctrl { kCtrlBnorm = 0, kCtrlUseRes, kCtrlTop, kCtrlAlpha, kCtrlHalf, kCtrlOmega };

template <int C>
__global__ void __launch_bounds__(kThr) ctrl_kernel(const double* __restrict__ part, double* __restrict__ sc,
                                                    int* __restrict__ st, double rtol) {
  __shared__ double sm[32];
  if (C != kCtrlBnorm && st[kDone]) return;
  double a = 0.0, b = 0.0;
  for (int k = threadIdx.x; k < kParts; k += kThr) {
    if (C == kCtrlUseRes) a = fmax(a, part[k]);
    else a += part[k];
    if (C == kCtrlTop || C == kCtrlOmega) b += part[kParts + k];
  }
  if (C == kCtrlUseRes) a = block_max(a, sm);
  else a = block_sum(a, sm);
  if (C == kCtrlTop || C == kCtrlOmega) b = block_sum(b, sm);
  if (threadIdx.x != 0) return;
  if (C == kCtrlBnorm) {
    const double bnrm2 = sqrt(a);
    sc[kBnrm] = bnrm2;
    sc[kAtol] = fmax(0.0, rtol * bnrm2);
    if (!isfinite(bnrm2)) {  // non-finite rhs: fields went non-finite earlier; the step latch reports it
      st[kSpecial] = 1;
      st[kDone] = 1;
    } else if (bnrm2 == 0.0) {
      st[kSpecial] = 2;
      st[kDone] = 1;
    }
  } else if (C == kCtrlUseRes) {
    st[kUseRes] = a > 0.0;
  } else if (C == kCtrlTop) {
    if (sqrt(a) < sc[kAtol]) {
      st[kDone] = 1;  // info 0
      return;
    }
    const double rho = b;
    if (fabs(rho) < kRhoTol) {
      st[kDone] = 1;
      st[kInfo] = -10;
      return;
    }
    if (st[kIter] > 0) {
      const double omega = sc[kOmega];
      if (fabs(omega) < kRhoTol) {
        st[kDone] = 1;
        st[kInfo] = -11;
        return;
      }
      sc[kBeta] = (rho / sc[kRhoPrev]) * (sc[kAlpha] / omega);
    }
    sc[kRho] = rho;
  } else if (C == kCtrlAlpha) {
    if (a == 0.0) {
      st[kDone] = 1;
      st[kInfo] = -11;
      return;
    }
    sc[kAlpha] = sc[kRho] / a;
  } else if (C == kCtrlHalf) {
    if (sqrt(a) < sc[kAtol]) {
      st[kHalf] = 1;
      st[kDone] = 1;
    }
  } else if (C == kCtrlOmega) {
    sc[kOmega] = a / b;
  }
}

// end of one loop pass: iteration count, maxiter, the WHILE condition (GRAPH = false: the
// dev-only eager mode, a fixed number of passes enqueued on the stream for profilers)
template <bool GRAPH>
__global__ void end_pass_kernel(double* __restrict__ sc, int* __restrict__ st, int maxiter,
                                cudaGraphConditionalHandle cond) {
  if (threadIdx.x != 0) return;
  if (!st[kDone]) {
    sc[kRhoPrev] = sc[kRho];
    const int it = st[kIter] + 1;
    st[kIter] = it;
    if (it >= maxiter) {
      st[kDone] = 1;
      st[kInfo] = maxiter;
    }
  }
  if constexpr (GRAPH) cudaGraphSetConditional(cond, st[kDone] ? 0u : 1u);
}

// the IF condition around a pass's second half: it runs only while the solve is not done
// (the complete-LU preconditioner converges at the first half-step check of nearly every step)
__global__ void second_half_cond_kernel(const int* __restrict__ st, cudaGraphConditionalHandle cond) {
  if (threadIdx.x == 0) cudaGraphSetConditional(cond, st[kDone] ? 0u : 1u);
}

// after the loop: special right-hand sides, status out
__global__ void finish_kernel(double* __restrict__ x, const double* __restrict__ b, int64_t n,
                              const int* __restrict__ st, int* __restrict__ status) {
  const int special = st[kSpecial];
  if (special) {
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    GRID_LOOP(i, n) x[i] = special == 1 ? nan : b[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && status) {
    status[0] = st[kDone] ? st[kInfo] : -99;  // -99: the eager dev mode ran out of passes
    status[1] = st[kIter];  // completed passes (a solve that stops at the first half-step: 0)
  }
}

}  // namespace

struct PressureSolver {
  int64_t n = 0;
  const int64_t* a_rowptr = nullptr;
  const int* a_cols = nullptr;
  const double* a_vals = nullptr;
  hn_tri_plan tl{}, tu{};
  const int* perm_r = nullptr;
  const int* perm_c = nullptr;
  int ctas = 2;
  double *y = nullptr, *z = nullptr, *w = nullptr, *ysum = nullptr;
  unsigned long long* ticket = nullptr;
  double *r = nullptr, *rt = nullptr, *p = nullptr, *phat = nullptr, *v = nullptr, *shat = nullptr, *t = nullptr;
  double *part = nullptr, *sc = nullptr;
  int* st = nullptr;
  cudaStream_t cap = nullptr;   // private capture stream for the loop body
  cudaStream_t cap2 = nullptr;  // ... and for the IF body inside it (a pass's second half)
  // cached standalone graph (calls outside a stream capture)
  cudaGraphExec_t exec = nullptr;
  const double* kb = nullptr;
  const double* kx0 = nullptr;
  double* kx = nullptr;
  int* kstatus = nullptr;
  double krtol = -1.0;
  int kmaxiter = -1;
};

namespace {

cudaError_t precond(PressureSolver& S, const double* in, double* out, cudaStream_t s) {
  const int64_t n = S.n;
  permute_in_skip_kernel<<<ceil_div(n, 256), 256, 0, s>>>(S.perm_r, in, n, S.y, S.st);
  cudaError_t e = sptrsv_enqueue(S.tl, S.y, S.z, S.ysum, n, S.ticket, S.ctas, S.st, s);
  if (e != cudaSuccess) return e;
  e = sptrsv_enqueue(S.tu, S.z, S.w, S.ysum, n, S.ticket, S.ctas, S.st, s);
  if (e != cudaSuccess) return e;
  permute_out_skip_kernel<<<ceil_div(n, 256), 256, 0, s>>>(S.perm_c, S.w, n, out, S.st);
  return cudaGetLastError();
}

template <bool GRAPH>
cudaError_t enqueue_pass(PressureSolver& S, double* x, double rtol, int maxiter, cudaGraphConditionalHandle cond,
                         cudaStream_t c);

// Enqueue one solve on s, which must be capturing: set-up nodes, the WHILE node whose body
// is one BiCGStab pass (captured on the private stream into the node's body graph), finish.
void enqueue_init(PressureSolver& S, const double* b, const double* x0, double* x, double rtol, cudaStream_t s) {
  const int64_t n = S.n;
  init_state_kernel<<<1, 32, 0, s>>>(S.st);
  bnorm_partial_kernel<<<kParts, kThr, 0, s>>>(b, n, S.part);
  ctrl_kernel<kCtrlBnorm><<<1, kThr, 0, s>>>(S.part, S.sc, S.st, rtol);
  init_x_kernel<<<kParts, kThr, 0, s>>>(x0, x, n, S.part, S.st);
  if (x0) ctrl_kernel<kCtrlUseRes><<<1, kThr, 0, s>>>(S.part, S.sc, S.st, rtol);
  init_r_kernel<<<kParts, kThr, 0, s>>>(S.a_rowptr, S.a_cols, S.a_vals, x, b, n, S.r, S.rt, S.part, S.st);
}

// Dev-only eager mode (HN_PRESSURE_EAGER=k in the environment): the set-up kernels, k
// passes and the finish kernel enqueued directly on the stream (no graph), so profilers
// that do not descend into conditional graph nodes see every kernel.  A solve that needs
// more than k passes reports info = -99.
cudaError_t enqueue_eager(PressureSolver& S, const double* b, const double* x0, double* x, double rtol, int maxiter,
                          int* status, int passes, cudaStream_t s) {
  enqueue_init(S, b, x0, x, rtol, s);
  for (int k = 0; k < passes; ++k) {
    cudaError_t e = enqueue_pass<false>(S, x, rtol, maxiter, cudaGraphConditionalHandle{}, s);
    if (e != cudaSuccess) return e;
  }
  finish_kernel<<<kParts, kThr, 0, s>>>(x, b, S.n, S.st, status);
  return cudaGetLastError();
}

cudaError_t enqueue_captured(PressureSolver& S, const double* b, const double* x0, double* x, double rtol,
                             int maxiter, int* status, cudaStream_t s) {
  const int64_t n = S.n;
  enqueue_init(S, b, x0, x, rtol, s);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;

  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  if ((e = cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &ndeps)) != cudaSuccess) return e;
  if (cs != cudaStreamCaptureStatusActive) return cudaErrorStreamCaptureInvalidated;
  cudaGraphConditionalHandle cond;
  if ((e = cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault)) != cudaSuccess) return e;
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = cond;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t loop;
  if ((e = cudaGraphAddNode(&loop, g, deps, ndeps, &np)) != cudaSuccess) return e;
  cudaGraph_t body = np.conditional.phGraph_out[0];

  cudaStream_t c = S.cap;
  if ((e = cudaStreamBeginCaptureToGraph(c, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)) != cudaSuccess)
    return e;
  e = enqueue_pass<true>(S, x, rtol, maxiter, cond, c);
  cudaError_t e2 = cudaStreamEndCapture(c, &body);
  if (e != cudaSuccess) return e;
  if (e2 != cudaSuccess) return e2;
  if ((e = cudaStreamUpdateCaptureDependencies(s, &loop, 1, cudaStreamSetCaptureDependencies)) != cudaSuccess)
    return e;
  finish_kernel<<<kParts, kThr, 0, s>>>(x, b, n, S.st, status);
  return cudaGetLastError();
}

// one BiCGStab pass (the WHILE body)
template <bool GRAPH>
cudaError_t enqueue_pass(PressureSolver& S, double* x, double rtol, int maxiter, cudaGraphConditionalHandle cond,
                         cudaStream_t c) {
  const int64_t n = S.n;
  cudaError_t e;
  ctrl_kernel<kCtrlTop><<<1, kThr, 0, c>>>(S.part, S.sc, S.st, rtol);
  p_update_kernel<<<kParts, kThr, 0, c>>>(S.p, S.v, S.r, n, S.sc, S.st);
  e = precond(S, S.p, S.phat, c);
  matvec_dot_kernel<<<kParts, kThr, 0, c>>>(S.a_rowptr, S.a_cols, S.a_vals, S.phat, n, S.v, S.rt, nullptr, S.part,
                                            S.st);
  ctrl_kernel<kCtrlAlpha><<<1, kThr, 0, c>>>(S.part, S.sc, S.st, rtol);
  s_update_kernel<<<kParts, kThr, 0, c>>>(S.r, S.v, n, S.sc, S.part, S.st);
  ctrl_kernel<kCtrlHalf><<<1, kThr, 0, c>>>(S.part, S.sc, S.st, rtol);
  half_x_kernel<<<kParts, kThr, 0, c>>>(x, S.phat, n, S.sc, S.st);
  if (e != cudaSuccess) return e;
  auto second_half = [&](cudaStream_t q) {
    cudaError_t e2 = precond(S, S.r, S.shat, q);
    matvec_dot_kernel<<<kParts, kThr, 0, q>>>(S.a_rowptr, S.a_cols, S.a_vals, S.shat, n, S.t, S.r, S.t, S.part, S.st);
    ctrl_kernel<kCtrlOmega><<<1, kThr, 0, q>>>(S.part, S.sc, S.st, rtol);
    xr_update_kernel<<<kParts, kThr, 0, q>>>(x, S.phat, S.shat, S.r, S.t, S.rt, n, S.sc, S.part, S.st);
    return e2;
  };
  if constexpr (GRAPH) {
    // the second half as the body of an IF node (nested in the WHILE body): when the half-step
    // check converged -- nearly every step -- its ~27 kernels are not launched at all instead
    // of launching and returning
    cudaStreamCaptureStatus cs;
    cudaGraph_t g;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    if ((e = cudaStreamGetCaptureInfo(c, &cs, nullptr, &g, &deps, &ndeps)) != cudaSuccess) return e;
    if (cs != cudaStreamCaptureStatusActive) return cudaErrorStreamCaptureInvalidated;
    cudaGraphConditionalHandle cond2;
    if ((e = cudaGraphConditionalHandleCreate(&cond2, g, 0, 0)) != cudaSuccess) return e;
    second_half_cond_kernel<<<1, 32, 0, c>>>(S.st, cond2);
    if ((e = cudaStreamGetCaptureInfo(c, &cs, nullptr, &g, &deps, &ndeps)) != cudaSuccess) return e;
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond2;
    np.conditional.type = cudaGraphCondTypeIf;
    np.conditional.size = 1;
    cudaGraphNode_t ifnode;
    if ((e = cudaGraphAddNode(&ifnode, g, deps, ndeps, &np)) != cudaSuccess) return e;
    cudaGraph_t ifbody = np.conditional.phGraph_out[0];
    if ((e = cudaStreamBeginCaptureToGraph(S.cap2, ifbody, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)) !=
        cudaSuccess)
      return e;
    e = second_half(S.cap2);
    cudaError_t e3 = cudaStreamEndCapture(S.cap2, &ifbody);
    if (e != cudaSuccess) return e;
    if (e3 != cudaSuccess) return e3;
    if ((e = cudaStreamUpdateCaptureDependencies(c, &ifnode, 1, cudaStreamSetCaptureDependencies)) != cudaSuccess)
      return e;
  } else {
    e = second_half(c);
    if (e != cudaSuccess) return e;
  }
  end_pass_kernel<GRAPH><<<1, 32, 0, c>>>(S.sc, S.st, maxiter, cond);
  return cudaGetLastError();
}

template <class T>
cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * (count ? count : 1));
}

}  // namespace
}  // namespace hn

using namespace hn;

HN_EXPORT int hn_pressure_setup(int64_t n, const int64_t* a_rowptr, const int* a_cols, const double* a_vals,
                                const hn_tri_plan* lower, const hn_tri_plan* upper, const int* perm_r,
                                const int* perm_c, int ctas_per_sm, int64_t* handle_out) {
  if (!lower || !upper || !handle_out || n <= 0) return 1;
  HN_TRY(sptrsv_prepare());
  (void)sm_count();  // cached before any capture
  PressureSolver* S = new PressureSolver();
  S->n = n;
  S->a_rowptr = a_rowptr;
  S->a_cols = a_cols;
  S->a_vals = a_vals;
  S->tl = *lower;
  S->tu = *upper;
  S->perm_r = perm_r;
  S->perm_c = perm_c;
  S->ctas = ctas_per_sm > 0 ? ctas_per_sm : 2;
  cudaError_t e = cudaSuccess;
  for (double** q : {&S->y, &S->z, &S->w, &S->ysum, &S->r, &S->rt, &S->p, &S->phat, &S->v, &S->shat, &S->t})
    if (e == cudaSuccess) e = dalloc(q, static_cast<size_t>(n));
  if (e == cudaSuccess) e = dalloc(&S->part, 2 * kParts);
  if (e == cudaSuccess) e = dalloc(&S->sc, kNumScalars);
  if (e == cudaSuccess) e = dalloc(&S->st, kNumState);
  if (e == cudaSuccess) e = dalloc(&S->ticket, 1);
  if (e == cudaSuccess) e = cudaMemset(S->p, 0, sizeof(double) * n);
  if (e == cudaSuccess) e = cudaMemset(S->v, 0, sizeof(double) * n);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&S->cap, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&S->cap2, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    *handle_out = reinterpret_cast<int64_t>(S);
    return -static_cast<int>(e);
  }
  *handle_out = reinterpret_cast<int64_t>(S);
  return 0;
}

// One pressure solve (see the file comment).  x0: warm start (NULL = zero; x0 == x = start
// from x's current contents).  status: device int[2] = [info, iterations] (may be NULL).
// Inside a stream capture the solve becomes nodes of the caller's graph; otherwise a graph
// cached per (b, x0, x, status, rtol, maxiter) is launched on the stream.
HN_EXPORT int hn_pressure_solve(int64_t handle, const double* b, const double* x0, double* x, double rtol,
                                int maxiter, int* status, void* stream) {
  PressureSolver* S = reinterpret_cast<PressureSolver*>(handle);
  if (!S || !b || !x || maxiter < 1) return 1;
  cudaStream_t s = as_stream(stream);
  cudaStreamCaptureStatus cs;
  HN_TRY(cudaStreamIsCapturing(s, &cs));
  if (cs == cudaStreamCaptureStatusActive) {
    HN_TRY(enqueue_captured(*S, b, x0, x, rtol, maxiter, status, s));
    return 0;
  }
  if (const char* ev = getenv("HN_PRESSURE_EAGER")) {
    const int passes = atoi(ev) > 0 ? atoi(ev) : 1;
    HN_TRY(enqueue_eager(*S, b, x0, x, rtol, maxiter, status, passes, s));
    return 0;
  }
  const bool hit = S->exec && S->kb == b && S->kx0 == x0 && S->kx == x && S->kstatus == status && S->krtol == rtol &&
                   S->kmaxiter == maxiter;
  if (!hit) {
    if (S->exec) {
      cudaGraphExecDestroy(S->exec);
      S->exec = nullptr;
    }
    cudaStream_t own;
    HN_TRY(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamBeginCapture(own, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      cudaError_t e1 = enqueue_captured(*S, b, x0, x, rtol, maxiter, status, own);
      e = cudaStreamEndCapture(own, &g);
      if (e1 != cudaSuccess) e = e1;
    }
    if (e == cudaSuccess) e = cudaGraphInstantiate(&S->exec, g, 0);
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(own);
    if (e != cudaSuccess) {
      S->exec = nullptr;
      return -static_cast<int>(e);
    }
    S->kb = b;
    S->kx0 = x0;
    S->kx = x;
    S->kstatus = status;
    S->krtol = rtol;
    S->kmaxiter = maxiter;
  }
  HN_TRY(cudaGraphLaunch(S->exec, s));
  return 0;
}

HN_EXPORT int hn_pressure_free(int64_t handle) {
  PressureSolver* S = reinterpret_cast<PressureSolver*>(handle);
  if (!S) return 0;
  if (S->exec) cudaGraphExecDestroy(S->exec);
  for (void* q : {static_cast<void*>(S->y), static_cast<void*>(S->z), static_cast<void*>(S->w),
                  static_cast<void*>(S->ysum), static_cast<void*>(S->r), static_cast<void*>(S->rt),
                  static_cast<void*>(S->p), static_cast<void*>(S->phat), static_cast<void*>(S->v),
                  static_cast<void*>(S->shat), static_cast<void*>(S->t), static_cast<void*>(S->part),
                  static_cast<void*>(S->sc), static_cast<void*>(S->st), static_cast<void*>(S->ticket)})
    if (q) cudaFree(q);
  if (S->cap) cudaStreamDestroy(S->cap);
  if (S->cap2) cudaStreamDestroy(S->cap2);
  delete S;
  return 0;
}
