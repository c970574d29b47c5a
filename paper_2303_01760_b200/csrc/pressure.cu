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
