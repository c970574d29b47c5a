// K6: fused multi-operator application over binned ELL stencil slabs.
//
// Replaces scipy's csr_matvec behind SparseOperator.apply / apply / divergence
// (reference: pkg/src/hybridnodes/operators.py:51-54, :80-90).  The reference
// matvec accumulates every row sequentially in ascending column order starting
// from 0.0 with separate multiply and add, and the weight tables are
// stored ascending by node index (approx.py:407-410), so this kernel reproduces
// it bit for bit: acc = 0.0; acc = acc (+) (w (*) f[j]) with __dmul_rn/__dadd_rn.
//
// Layout (one "bin" per stencil width; MON and RBF rows never share a warp):
//   rows[k]                       node id of the k-th row of the bin (int32)
//   idx[j*K + k]                  j-th stencil node of row k, ascending (int32)
//   w[(op*W + j)*K + k]           weight of operator op (fp64)
// so a warp of 32 consecutive rows reads every (op, j) column with one
// coalesced 256 B transaction, and the gathered field f (8 N bytes) stays in L2.
#include "hn_common.cuh"

namespace hn {

struct ApplyBins {
  int nbins;
  int nops;
  int width[4];
  int64_t K[4];
  int64_t block_start[5];
  const int* rows[4];
  const int* idx[4];
  const double* w[4];
  int op_sel[4];          // which weight planes of the bins to apply
  int64_t out_stride;     // distance between output planes (elements)
};

template <int W, int NOPS>
__device__ __forceinline__ void apply_rows(const ApplyBins& b, int bin, int64_t k,
                                           const double* __restrict__ f,
                                           double* __restrict__ out) {
  const int64_t K = b.K[bin];
  const int* __restrict__ idx = b.idx[bin];
  const double* __restrict__ w = b.w[bin];
  const int row = __ldg(b.rows[bin] + k);
  double fv[W > 0 ? W : 1];
#pragma unroll
  for (int j = 0; j < W; ++j) fv[j] = __ldg(f + __ldg(idx + j * K + k));
#pragma unroll
  for (int o = 0; o < NOPS; ++o) {
    const double* __restrict__ wo = w + static_cast<int64_t>(b.op_sel[o]) * W * K;
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < W; ++j) acc = __dadd_rn(acc, __dmul_rn(__ldg(wo + j * K + k), fv[j]));
    out[o * b.out_stride + row] = acc;
  }
}

template <int NOPS>
__global__ void __launch_bounds__(256) apply_ell_kernel(ApplyBins b, const double* __restrict__ f,
                                                        double* __restrict__ out) {
  int bin = 0;
#pragma unroll
  for (int i = 1; i < 4; ++i)
    if (i < b.nbins && blockIdx.x >= b.block_start[i]) bin = i;
  const int64_t k = (static_cast<int64_t>(blockIdx.x) - b.block_start[bin]) * blockDim.x + threadIdx.x;
  if (k >= b.K[bin]) return;
  switch (b.width[bin]) {
    case 0: apply_rows<0, NOPS>(b, bin, k, f, out); break;
    case 5: apply_rows<5, NOPS>(b, bin, k, f, out); break;
    case 7: apply_rows<7, NOPS>(b, bin, k, f, out); break;
    case 12: apply_rows<12, NOPS>(b, bin, k, f, out); break;
    case 20: apply_rows<20, NOPS>(b, bin, k, f, out); break;
    case 30: apply_rows<30, NOPS>(b, bin, k, f, out); break;
    default: break;
  }
}

int g_apply_threads = 128;  // tuning knob (hn_apply_set_threads); results identical

bool supported_width(int w) { return w == 0 || w == 5 || w == 7 || w == 12 || w == 20 || w == 30; }

// ELL bins -> the reference's WeightTable layout (approx.py:311-323): indices (N, n_max)
// int64 -1 padded, sizes (N,) int64, weights (nops, N, n_max) fp64 zero padded.
struct TableBins {
  int nbins;
  int width[4];
  int64_t K[4];
  int64_t block_start[5];
  const int* rows[4];
  const int* idx[4];
  const double* w[4];
};

__global__ void ell_to_table_kernel(TableBins b, int nops, int n_max, int64_t N, int64_t* __restrict__ idx_out,
                                    int64_t* __restrict__ sizes_out, double* __restrict__ w_out) {
  int bin = 0;
#pragma unroll
  for (int i = 1; i < 4; ++i)
    if (i < b.nbins && blockIdx.x >= b.block_start[i]) bin = i;
  const int64_t k = (static_cast<int64_t>(blockIdx.x) - b.block_start[bin]) * blockDim.x + threadIdx.x;
  if (k >= b.K[bin]) return;
  const int64_t K = b.K[bin];
  const int W = b.width[bin];
  const int64_t row = __ldg(b.rows[bin] + k);
  sizes_out[row] = W;
  for (int j = 0; j < n_max; ++j) idx_out[row * n_max + j] = j < W ? __ldg(b.idx[bin] + j * K + k) : -1;
  for (int o = 0; o < nops; ++o)
    for (int j = 0; j < n_max; ++j)
      w_out[(o * N + row) * n_max + j] = j < W ? __ldg(b.w[bin] + (static_cast<int64_t>(o) * W + j) * K + k) : 0.0;
}

}  // namespace hn

using namespace hn;

HN_EXPORT int hn_ell_to_table(int nbins, const int64_t* bin_K_host, const int* bin_width_host,
                              const int* const* bin_rows_host, const int* const* bin_idx_host,
                              const double* const* bin_w_host, int nops, int n_max, int64_t N, int64_t* idx_out,
                              int64_t* sizes_out, double* w_out, void* stream) {
  if (nbins < 1 || nbins > 4) return 1;
  TableBins b{};
  b.nbins = nbins;
  const int threads = 128;
  int64_t blocks = 0;
  for (int i = 0; i < nbins; ++i) {
    if (bin_width_host[i] > n_max) return 2;
    b.width[i] = bin_width_host[i];
    b.K[i] = bin_K_host[i];
    b.rows[i] = bin_rows_host[i];
    b.idx[i] = bin_idx_host[i];
    b.w[i] = bin_w_host[i];
    b.block_start[i] = blocks;
    blocks += ceil_div(b.K[i], threads);
  }
  b.block_start[nbins] = blocks;
  if (blocks == 0) return 0;
  ell_to_table_kernel<<<blocks, threads, 0, as_stream(stream)>>>(b, nops, n_max, N, idx_out, sizes_out, w_out);
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT void hn_apply_set_threads(int t) { g_apply_threads = (t == 64 || t == 128 || t == 256) ? t : 128; }

HN_EXPORT int hn_apply_ell(int nbins, const int64_t* bin_K_host, const int* bin_width_host,
                           const int* const* bin_rows_host, const int* const* bin_idx_host,
                           const double* const* bin_w_host, int nops, const int* op_sel_host,
                           const double* field, double* out, int64_t out_stride, void* stream) {
  if (nbins < 1 || nbins > 4 || nops < 1 || nops > 4) return 1;
  ApplyBins b{};
  b.nbins = nbins;
  b.nops = nops;
  b.out_stride = out_stride;
  const int threads = g_apply_threads;
  int64_t blocks = 0;
  for (int i = 0; i < nbins; ++i) {
    if (!supported_width(bin_width_host[i])) return 2;
    b.width[i] = bin_width_host[i];
    b.K[i] = bin_K_host[i];
    b.rows[i] = bin_rows_host[i];
    b.idx[i] = bin_idx_host[i];
    b.w[i] = bin_w_host[i];
    b.block_start[i] = blocks;
    blocks += ceil_div(b.K[i], threads);
  }
  b.block_start[nbins] = blocks;
  for (int o = 0; o < nops; ++o) b.op_sel[o] = op_sel_host[o];
  if (blocks == 0) return 0;
  cudaStream_t s = as_stream(stream);
  switch (nops) {
    case 1: apply_ell_kernel<1><<<blocks, threads, 0, s>>>(b, field, out); break;
    case 2: apply_ell_kernel<2><<<blocks, threads, 0, s>>>(b, field, out); break;
    case 3: apply_ell_kernel<3><<<blocks, threads, 0, s>>>(b, field, out); break;
    default: apply_ell_kernel<4><<<blocks, threads, 0, s>>>(b, field, out); break;
  }
  HN_CHECK_LAUNCH();
  return 0;
}
