// compute_weights' device sequence as one native call (the public API's hot path):
//   classify -> stable partition [MON | RBF | NONE] -> (class sizes) -> MON stencils + solves
//   -> kNN + RBF-FD solves -> WeightTable layout -> async copy-back into pinned host memory.
// Python calls it once per compute_weights; each stage is the same library entry point the
// step-by-step path uses (approx.py:379-413 is the reference orchestration), so results are
// identical -- this only removes ~0.4 ms of per-stage host work from the call.
//
// Buffers are caller-owned (device unless noted).  Bins are written with stride = their
// row count K into capacity buffers: mon_idx (>= (2d+1) K_mon), mon_w (>= nops (2d+1) K_mon),
// rbf_idx (>= n_rbf K_rbf), rbf_w (>= nops n_rbf K_rbf).
#include "hn_common.cuh"

extern "C" {
int hn_classify(const int8_t* kind, const int* lattice_idx, const int* grid, const int* grid_dims_host, int64_t n,
                int d, int8_t* method, void* stream);
int hn_partition_methods(const int8_t* method, int64_t n, int* rows_out, int* counts_out, int* scratch,
                         void* stream);
int hn_mon_stencils(const int* rows, int64_t nrows, const double* pos, const int* lattice_idx, const int* grid,
                    const int* grid_dims_host, int d, int* out, void* stream);
int hn_weights_mon(const double* pos, int d, const int* stencils, int64_t K, int nops, const int* op_kind_host,
                   const int* op_axis_host, const double* op_normal_host, int* out_idx, double* out_w, int* info,
                   void* stream);
int hn_knn_spacing(const double* pos, int d, const double* lo_host, double cell, const int* dims_host,
                   const int* cell_start, const int* cell_items, const double* cell_pos, const int* queries,
                   const double* qpos, int64_t nq, int n, const uint8_t* exclude, const double* spacing,
                   int* out_idx, double* out_dist, void* stream);
int hn_knn(const double* pos, int d, const double* lo_host, double cell, const int* dims_host,
           const int* cell_start, const int* cell_items, const double* cell_pos, const int* queries,
           const double* qpos, int64_t nq, int n, const uint8_t* exclude, int* out_idx, double* out_dist,
           void* stream);
int hn_weights_rbf(const double* pos, int d, const int* stencils, int64_t K, int n, int nops,
                   const int* op_kind_host, const int* op_axis_host, const double* op_normal_host,
                   const double* row_normals, double* workspace, int* out_idx, double* out_w, int* info,
                   void* stream);
int hn_weights_rbf_is_tuned(int d, int n, int nops);
int hn_ell_to_table(int nbins, const int64_t* bin_K_host, const int* bin_width_host, const int* const* bin_rows_host,
                    const int* const* bin_idx_host, const double* const* bin_w_host, int nops, int n_max, int64_t N,
                    int64_t* idx_out, int64_t* sizes_out, double* w_out, void* stream);
}

namespace hn {
// singular-flag summary of a bin: out = [count of nonzero info, first flagged row]
__global__ void info_summary_kernel(const int* __restrict__ info, int64_t K, int* __restrict__ out) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < K;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (info[k]) {
      atomicAdd(out, 1);
      atomicMin(out + 1, static_cast<int>(k));
    }
  }
}
}  // namespace hn

#define HN_RC(expr)              \
  do {                           \
    const int _rc = (expr);      \
    if (_rc != 0) return _rc;    \
  } while (0)

HN_EXPORT int hn_weights_pipeline(
    const double* pos, int d, int64_t n, const int8_t* kind, const int* lattice_idx, const int* lattice_grid,
    const int* grid_dims_host, const double* lo_host, double cell, const int* dims_host, const int* cell_start,
    const int* cell_items, const double* cell_pos, const double* spacing, int nops, const int* op_kind_host,
    const int* op_axis_host, const double* op_normal_host, int n_rbf, int64_t k_mon_host, int64_t k_rbf_host, int8_t* method,
    int* rows, int* counts, int* part_scratch, int* mon_st, int* mon_idx, double* mon_w, int* mon_info,
    int* rbf_st, int* rbf_idx, double* rbf_w, int* rbf_info, int64_t* tab_idx, int64_t* tab_sizes,
    double* tab_w, int64_t* h_idx, int64_t* h_sizes, double* h_w, int8_t* h_method, int64_t* counts_host,
    int* summary, int* h_summary, int chunks, const int64_t* cut_host, void* stream) {
  if (d != 2 && d != 3) return 1;
  if (n_rbf < 1 || n_rbf > 64 || hn_weights_rbf_is_tuned(d, n_rbf, nops) != 0) return 2;
  cudaStream_t s = hn::as_stream(stream);
  const int nmon = 2 * d + 1;
  HN_RC(hn_classify(kind, lattice_grid ? lattice_idx : nullptr, lattice_grid, grid_dims_host, n, d, method,
                    stream));
  HN_RC(hn_partition_methods(method, n, rows, counts, part_scratch, stream));
  int64_t k_mon, k_rbf, k_none;
  if (k_rbf_host >= 0) {  // class sizes known to the caller (no regular node, or a frozen
    k_mon = k_mon_host;    // replay): no read-back, the call is capturable in a CUDA graph
    k_rbf = k_rbf_host;
    k_none = n - k_mon - k_rbf;
  } else {
    int c3[3];
    HN_TRY(cudaMemcpyAsync(c3, counts, sizeof(c3), cudaMemcpyDeviceToHost, s));
    HN_TRY(cudaStreamSynchronize(s));
    k_mon = c3[0];
    k_rbf = c3[1];
    k_none = c3[2];
  }
  counts_host[0] = k_mon;
  counts_host[1] = k_rbf;
  counts_host[2] = k_none;
  if (k_rbf && n_rbf > n) return 3;
  if (k_mon) {
    if (lattice_grid) {
      HN_RC(hn_mon_stencils(rows, k_mon, pos, lattice_idx, lattice_grid, grid_dims_host, d, mon_st, stream));
    } else {
      HN_RC(hn_knn(pos, d, lo_host, cell, dims_host, cell_start, cell_items, cell_pos, rows, nullptr, k_mon, nmon,
                   nullptr, mon_st, nullptr, stream));
    }
    HN_RC(hn_weights_mon(pos, d, mon_st, k_mon, nops, op_kind_host, op_axis_host, op_normal_host, mon_idx, mon_w,
                         mon_info, stream));
  }
  // WeightTable layout: every row belongs to exactly one bin (MON | RBF chunk c | NONE).
  // MON and empty rows go first, then each RBF chunk (rows ascending by node id) is solved,
  // laid out and copied back on a side stream while the next chunk computes.
  int nb = 0;
  int64_t bK[3];
  int bW[3];
  const int* bR[3];
  const int* bI[3];
  const double* bWt[3];
  auto add = [&](int64_t K, int W, const int* r, const int* i, const double* w) {
    if (K <= 0) return;
    bK[nb] = K;
    bW[nb] = W;
    bR[nb] = r;
    bI[nb] = i;
    bWt[nb] = w;
    ++nb;
  };
  add(k_mon, nmon, rows, mon_idx, mon_w);
  add(k_none, 0, rows + k_mon + k_rbf, mon_idx, mon_w);
  if (tab_idx) {  // NULL: the caller keeps the ELL bins (operator assembly, device-resident runs)
    HN_TRY(cudaMemsetAsync(tab_sizes, 0, sizeof(int64_t) * n, s));
    if (nb) HN_RC(hn_ell_to_table(nb, bK, bW, bR, bI, bWt, nops, n_rbf, n, tab_idx, tab_sizes, tab_w, stream));
  } else if (h_idx) {
    return 4;  // a host copy needs the table
  }
  if (chunks < 1 || k_rbf == 0 || !h_idx) chunks = 1;
  if (chunks > k_rbf && k_rbf > 0) chunks = static_cast<int>(k_rbf);
  if (chunks > 64) chunks = 64;
  int64_t bounds[65], cut[65];  // chunk c = RBF rows [bounds[c], bounds[c+1]); its table rows [cut[c], cut[c+1])
  for (int c = 0; c <= chunks; ++c) bounds[c] = k_rbf * c / chunks;
  cut[0] = 0;
  cut[chunks] = n;
  if (chunks > 1 && h_idx) {
    if (cut_host) {
      for (int c = 1; c < chunks; ++c) cut[c] = cut_host[c - 1];
    } else {  // node id of each chunk's first row (rows are ascending within the RBF segment)
      int ids[64];
      for (int c = 1; c < chunks; ++c)
        HN_TRY(cudaMemcpyAsync(ids + c, rows + k_mon + bounds[c], sizeof(int), cudaMemcpyDeviceToHost, s));
      HN_TRY(cudaStreamSynchronize(s));
      for (int c = 1; c < chunks; ++c) cut[c] = ids[c];
    }
  }
  hn::ForkJoin& fj = hn::fork_join();
  cudaStream_t cs = fj.side[0];
  for (int c = 0; c < chunks; ++c) {
    const int64_t k0 = bounds[c], kc = bounds[c + 1] - bounds[c];
    if (kc > 0) {
      int* st_c = rbf_st + static_cast<int64_t>(n_rbf) * k0;
      int* idx_c = rbf_idx + static_cast<int64_t>(n_rbf) * k0;
      double* w_c = rbf_w + static_cast<int64_t>(nops) * n_rbf * k0;
      const int* rows_c = rows + k_mon + k0;
      HN_RC(hn_knn_spacing(pos, d, lo_host, cell, dims_host, cell_start, cell_items, cell_pos, rows_c, nullptr, kc,
                           n_rbf, nullptr, spacing, st_c, nullptr, stream));
      HN_RC(hn_weights_rbf(pos, d, st_c, kc, n_rbf, nops, op_kind_host, op_axis_host, op_normal_host, nullptr,
                           nullptr, idx_c, w_c, rbf_info + k0, stream));
      const int64_t K1[1] = {kc};
      const int W1[1] = {n_rbf};
      const int* R1[1] = {rows_c};
      const int* I1[1] = {idx_c};
      const double* Wt1[1] = {w_c};
      if (tab_idx) HN_RC(hn_ell_to_table(1, K1, W1, R1, I1, Wt1, nops, n_rbf, n, tab_idx, tab_sizes, tab_w, stream));
    }
    if (h_idx && cut[c + 1] > cut[c]) {  // this chunk's slice of the host table, on the side stream
      const int64_t lo = cut[c], m = cut[c + 1] - cut[c];
      HN_TRY(cudaEventRecord(fj.start, s));
      HN_TRY(cudaStreamWaitEvent(cs, fj.start, 0));
      HN_TRY(cudaMemcpyAsync(h_idx + lo * n_rbf, tab_idx + lo * n_rbf, sizeof(int64_t) * m * n_rbf,
                             cudaMemcpyDeviceToHost, cs));
      HN_TRY(cudaMemcpyAsync(h_sizes + lo, tab_sizes + lo, sizeof(int64_t) * m, cudaMemcpyDeviceToHost, cs));
      for (int o = 0; o < nops; ++o)
        HN_TRY(cudaMemcpyAsync(h_w + (o * n + lo) * n_rbf, tab_w + (o * n + lo) * n_rbf,
                               sizeof(double) * m * n_rbf, cudaMemcpyDeviceToHost, cs));
    }
  }
  if (h_idx) {
    HN_TRY(cudaMemcpyAsync(h_method, method, n, cudaMemcpyDeviceToHost, cs));
    HN_TRY(cudaEventRecord(fj.done[0], cs));
    HN_TRY(cudaStreamWaitEvent(s, fj.done[0], 0));
  }
  // singular flags of both bins in 4 ints: [MON count, MON first, RBF count, RBF first]
  // (summary == NULL: the caller inspects mon_info / rbf_info itself)
  if (!summary) return 0;
  HN_TRY(cudaMemsetAsync(summary, 0, 4 * sizeof(int), s));
  HN_TRY(cudaMemsetAsync(summary + 1, 0x7f, sizeof(int), s));
  HN_TRY(cudaMemsetAsync(summary + 3, 0x7f, sizeof(int), s));
  const int sb = hn::sm_count() * 2;
  if (k_mon) hn::info_summary_kernel<<<sb, 256, 0, s>>>(mon_info, k_mon, summary);
  if (k_rbf) hn::info_summary_kernel<<<sb, 256, 0, s>>>(rbf_info, k_rbf, summary + 2);
  HN_TRY(cudaGetLastError());
  if (h_summary) HN_TRY(cudaMemcpyAsync(h_summary, summary, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
  return 0;
}
