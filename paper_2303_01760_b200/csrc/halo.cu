// Halo plumbing of the row-sharded explicit step: pack the field values a
// peer needs into one send buffer, scatter received values into the halo tail of the local
// SoA arrays, and renumber stencil column ids from node ids to a rank's local numbering
// (owned rows first, then halo nodes grouped by owner).  The exchange itself is NCCL
// (torch.distributed) on the same stream; these kernels are HBM-bound gathers of a few
// hundred KB per step.
#include "hn_common.cuh"
#include "hn.h"

namespace hn {
namespace {

constexpr int kThr = 256;

__global__ void __launch_bounds__(kThr) halo_gather_kernel(const double* __restrict__ src,
                                                           const int64_t* __restrict__ map, int64_t n,
                                                           double* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThr;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x; i < n; i += stride)
    out[i] = __ldg(src + __ldg(map + i));
}

__global__ void __launch_bounds__(kThr) halo_scatter_kernel(const double* __restrict__ in,
                                                            const int64_t* __restrict__ map, int64_t n,
                                                            double* __restrict__ dst) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThr;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x; i < n; i += stride)
    dst[__ldg(map + i)] = __ldg(in + i);
}

__global__ void __launch_bounds__(kThr) remap_kernel(const int* __restrict__ in, const int* __restrict__ map,
                                                     int64_t n, int* __restrict__ out, int* __restrict__ bad) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThr;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x; i < n; i += stride) {
    const int v = __ldg(map + __ldg(in + i));
    out[i] = v;
    if (v < 0) atomicAdd(bad, 1);
  }
}

inline int grid_for(int64_t n) {
  const int64_t want = ceil_div(n, kThr);
  const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
  return static_cast<int>(want < cap ? want : cap);
}

}  // namespace
}  // namespace hn

HN_EXPORT int hn_halo_gather(const double* src, const int64_t* map, int64_t n, double* out, void* stream) {
  if (n == 0) return 0;
  hn::halo_gather_kernel<<<hn::grid_for(n), hn::kThr, 0, hn::as_stream(stream)>>>(src, map, n, out);
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT int hn_halo_scatter(const double* in, const int64_t* map, int64_t n, double* dst, void* stream) {
  if (n == 0) return 0;
  hn::halo_scatter_kernel<<<hn::grid_for(n), hn::kThr, 0, hn::as_stream(stream)>>>(in, map, n, dst);
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT int hn_remap_indices(const int* in, const int* map, int64_t n, int* out, int* bad, void* stream) {
  if (n == 0) return 0;
  hn::remap_kernel<<<hn::grid_for(n), hn::kThr, 0, hn::as_stream(stream)>>>(in, map, n, out, bad);
  HN_CHECK_LAUNCH();
  return 0;
}
