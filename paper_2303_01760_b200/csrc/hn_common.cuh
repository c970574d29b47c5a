// Shared helpers for the hybridnodes sm_100a kernels (libhn.so).
//
// Conventions (see include/hn.h):
//   * every entry point returns int: 0 = ok, < 0 = -(cudaError_t), > 0 = domain count
//     (e.g. number of singular systems);
//   * all array arguments are DEVICE pointers unless the name ends in `_host`;
//   * every launch goes on the caller's stream (`void* stream`, 0 = legacy default);
//   * fp64 arithmetic that must be bit-identical to the CPU reference uses the
//     explicit round-to-nearest intrinsics (__dmul_rn / __dadd_rn / __dsqrt_rn), which
//     ptxas never contracts into DFMA.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define HN_EXPORT extern "C" __attribute__((visibility("default")))

#define HN_CHECK_LAUNCH()                                   \
  do {                                                      \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) return -static_cast<int>(_e);    \
  } while (0)

#define HN_TRY(expr)                                        \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return -static_cast<int>(_e);    \
  } while (0)

namespace hn {

constexpr int kWarp = 32;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Stream-ordered scratch from the device's default pool.  The pool's release threshold is
// raised once per device so freed scratch stays cached: with the default threshold 0 every
// synchronize hands it back to the driver and the next cudaMallocAsync costs ~100-250 us.
inline cudaError_t stream_alloc(void** p, size_t bytes, cudaStream_t s) {
  static bool kept[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < 64 && !kept[dev]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    kept[dev] = true;
  }
  return cudaMallocAsync(p, bytes, s);
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Number of SMs on the current device (cached per process).
int sm_count();

// Fork/join of independent launches: launch i > 0 goes to a side stream that waits for
// everything already queued on s; s waits for every side before anything later runs.
// Capturable into CUDA graphs (event record/wait become graph edges).
struct ForkJoin {
  static constexpr int kSides = 3;
  cudaStream_t side[kSides];
  cudaEvent_t done[kSides];
  cudaEvent_t start;
};
ForkJoin& fork_join();

template <typename F>
inline void launch_forked(cudaStream_t s, int n, F&& launch) {
  if (n <= 1) {
    if (n == 1) launch(0, s);
    return;
  }
  ForkJoin& fj = fork_join();
  const int sides = n - 1 < ForkJoin::kSides ? n - 1 : ForkJoin::kSides;
  cudaEventRecord(fj.start, s);
  for (int k = 0; k < sides; ++k) cudaStreamWaitEvent(fj.side[k], fj.start, 0);
  for (int i = 0; i < n; ++i) launch(i, i == 0 ? s : fj.side[(i - 1) % sides]);
  for (int k = 0; k < sides; ++k) {
    cudaEventRecord(fj.done[k], fj.side[k]);
    cudaStreamWaitEvent(s, fj.done[k], 0);
  }
}

// fl(sqrt(((0 + dx*dx) + dy*dy) [+ dz*dz])) -- the distance scipy's cKDTree and
// np.linalg.norm return for these inputs; no FMA contraction.
template <int D>
__device__ __forceinline__ double exact_dist(const double* a, const double* b) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double t = __dsub_rn(a[k], b[k]);
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  return __dsqrt_rn(s);
}

template <int D>
__device__ __forceinline__ double exact_dist2(const double* a, const double* b) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double t = __dsub_rn(a[k], b[k]);
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  return s;
}

// Load point i from a padded AoS position array (stride = 2 in 2D, 4 in 3D).
template <int D>
__device__ __forceinline__ void load_point(const double* __restrict__ pos, int64_t i, double* p) {
  if constexpr (D == 2) {
    double2 v = __ldg(reinterpret_cast<const double2*>(pos) + i);
    p[0] = v.x;
    p[1] = v.y;
  } else {
    const double4* q = reinterpret_cast<const double4*>(pos) + i;
    double2 v0 = __ldg(reinterpret_cast<const double2*>(q));
    double2 v1 = __ldg(reinterpret_cast<const double2*>(q) + 1);
    p[0] = v0.x;
    p[1] = v0.y;
    p[2] = v1.x;
  }
}

template <int D>
constexpr int pos_stride() { return D == 2 ? 2 : 4; }

// Operator codes shared by the weight kernels (include/hn.h HN_OP_*).
enum OpKind : int { kOpLaplacian = 0, kOpPartial = 1, kOpNormal = 2 };

}  // namespace hn
