// Library identity and the fp64 peak probe used for the weight-solver roofline.
#include "hn_common.cuh"

namespace hn {

int sm_count() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

// Side streams for fork/join launches (per device, created on first use; non-blocking so
// they never serialise against the legacy default stream) and their join events.
ForkJoin& fork_join() {
  static ForkJoin fj[16];
  static bool made[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  dev = dev < 16 ? dev : 15;
  if (!made[dev]) {
    for (int i = 0; i < ForkJoin::kSides; ++i) {
      cudaStreamCreateWithFlags(&fj[dev].side[i], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&fj[dev].done[i], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&fj[dev].start, cudaEventDisableTiming);
    made[dev] = true;
  }
  return fj[dev];
}

// 16 independent DFMA chains per thread keep the FP64 pipe saturated; the result is
// folded into a checksum so nothing is dead code.
__global__ void __launch_bounds__(256) dfma_probe_kernel(double* out, int iters) {
  double a[16];
  const double x = 1.0 + 1e-9 * threadIdx.x, y = 0.999999;
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 1e-3 * (i + 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], y, x);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;  // never true; keeps the chains live
}

// FP64 tensor-core probe: 4 independent m8n8k4 DMMA accumulators per warp.
__global__ void __launch_bounds__(256) dmma_probe_kernel(double* out, int iters) {
  const double a = 1.0 + 1e-9 * threadIdx.x, b = 0.999;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = 1e-3 * i; c[i][1] = 2e-3 * i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

}  // namespace hn

HN_EXPORT int hn_version(void) { return 1; }

// flops per launch = blocks * 8 warps * iters * 4 * (8*8*4*2)
HN_EXPORT int hn_bench_dmma(double* out, int blocks, int iters, void* stream) {
  hn::dmma_probe_kernel<<<blocks, 256, 0, hn::as_stream(stream)>>>(out, iters);
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT int hn_bench_dfma(double* out, int blocks, int iters, void* stream) {
  hn::dfma_probe_kernel<<<blocks, 256, 0, hn::as_stream(stream)>>>(out, iters);
  HN_CHECK_LAUNCH();
  return 0;
}
