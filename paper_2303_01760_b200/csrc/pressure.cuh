// Internal (C++) interface between the supernodal triangular solves (pressure.cu) and the
// device-driven BiCGStab (bicgstab.cu).  Not part of the C ABI.
#pragma once
#include "hn_common.cuh"
#include "hn.h"

namespace hn {

// One supernodal triangular solve: reset of x / ysum / ticket, then the persistent task
// kernel.  skip (device int, may be NULL): when *skip != 0 both kernels return at once
// (a converged Krylov loop inside a CUDA graph).  An upper plan with dense groups overwrites the
// groups' entries of b with their solution.
cudaError_t sptrsv_enqueue(const hn_tri_plan& p, double* b, double* x, double* ysum, int64_t n,
                           unsigned long long* ticket, int ctas_per_sm, const int* skip, cudaStream_t s);

// The dynamic shared-memory opt-in of the trisolve kernels on the current device (outside
// any stream capture).
cudaError_t sptrsv_prepare();

}  // namespace hn
