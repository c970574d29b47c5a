/* hn.h -- C ABI of libhn.so, the sm_100a hot path of the hybrid scattered-regular
 * RBF-FD method (arXiv 2303.01760), drop-in beneath the reference package
 * `hybridnodes` (pkg/src/hybridnodes).
 *
 * The reference is pure Python over numpy/scipy; its "FFI" for this path is the set of
 * third-party native calls it makes (scipy cKDTree, LAPACK dgesv via np.linalg.solve,
 * scipy csr_matvec, SuperLU + bicgstab).  Each entry point below replaces one of them
 * and cites the reference call site.  Python binds this header with ctypes
 * (paper_2303_01760_b200/_lib.py); INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - plain C types only; every array is a DEVICE pointer unless its name ends in
 *     `_host` (small parameter arrays read on the host during the call);
 *   - every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy stream);
 *   - return 0 on success, a negative value = -(cudaError_t) on a CUDA failure, a
 *     positive value for an argument error (documented per call); numerical failures
 *     (singular systems, non-finite fields) are reported through device `info` arrays;
 *   - the library never frees caller memory; scratch is caller-provided or taken from
 *     the stream-ordered allocator and released before the call returns;
 *   - index arrays are int32 (N < 2^31 nodes); fields and weights are fp64.
 */
#ifndef HN_H_
#define HN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* operator kinds (approx.py:35-52: Laplacian / Partial / NormalDerivative) */
#define HN_OP_LAPLACIAN 0
#define HN_OP_PARTIAL 1
#define HN_OP_NORMAL 2

/* ---------------------------------------------------------------- stencils (K1-K3) */

/* Uniform cell list over positions (N x stride fp64 AoS, stride 2 in 2D / 4 in 3D).
 * cell_start: ncells+1, cell_items: N, cell_pos: N*stride, scratch_count: ncells,
 * scratch_point_cell: N, with ncells = prod(dims_host[0..d)).
 * Replaces: cKDTree(nodeset.positions)  approx.py:386, solver.py:144. */
/* Node-set statistics for the cell-list sizing, one pass: out (device, 2d+2 fp64) =
 * [min x_a (d) | max x_a (d) | sum of spacing over kind == 1 | count of kind == 1].
 * pos: N x d fp64 (unpadded); kind / spacing may be NULL; scratch: 8 u64 (device).
 * Replaces: the np.min/np.max bounding box and mean spacing the host would compute. */
int hn_node_stats(const double* pos, int64_t n, int d, const int8_t* kind, const double* spacing, double* out,
                  void* scratch, void* stream);

int hn_celllist_build(const double* pos, int64_t n, int d, const double* lo_host, double cell,
                      const int* dims_host, int* cell_start, int* cell_items, double* cell_pos,
                      int* scratch_count, int* scratch_point_cell, void* stream);

/* n nearest nodes of each query by the key (fl-distance, node index); queries are node
 * ids (queries, NULL = 0..nq-1) or, when qpos != NULL, points (nq x stride fp64).
 * out_idx (nq x n) ascending by key, out_dist optional.
 * exclude (N bytes, nonzero = skip) or NULL.  1 <= n <= 64.
 * Replaces: _knn_sorted approx.py:133-146 (cKDTree.query + tie widening + lexsort) and
 * the sub-tree query of _boundary_stencils approx.py:425-431. */
int hn_knn(const double* pos, int d, const double* lo_host, double cell, const int* dims_host,
           const int* cell_start, const int* cell_items, const double* cell_pos,
           const int* queries, const double* qpos, int64_t nq, int n, const uint8_t* exclude,
           int* out_idx, double* out_dist, void* stream);

/* hn_knn with a per-node nominal spacing (N fp64, indexed like the queries: node id, or
 * query number when qpos != NULL): the box pass sizes each query's first search radius
 * from its own spacing, which keeps graded node sets on the fast path.  Same results.
 * Replaces: the same reference calls as hn_knn (nodeset.spacing, nodegen.py:90-179). */
int hn_knn_spacing(const double* pos, int d, const double* lo_host, double cell, const int* dims_host,
                   const int* cell_start, const int* cell_items, const double* cell_pos,
                   const int* queries, const double* qpos, int64_t nq, int n, const uint8_t* exclude,
                   const double* spacing, int* out_idx, double* out_dist, void* stream);

/* kNN kernel variant (tuning knob, identical results): 0 default (3D: warp-per-query kernel +
 * box-pass fallback list; 2D: box pass + exact ring fallback), 1 ring traversal only, 2/3 box
 * pass with a smaller/larger first radius, 5 box pass only. */
void hn_knn_set_variant(int v);

/* compute_weights' whole device sequence in one call: classify -> partition [MON | RBF |
 * NONE] -> (class sizes: k_mon_host / k_rbf_host when the caller knows them, k_rbf_host >= 0
 * -- no regular node, or a frozen replay; the call is then capturable in a CUDA graph --
 * else one read-back) -> MON stencils + solves -> kNN (spacing-sized, on the given grid) +
 * RBF-FD solves -> WeightTable layout (tab_*, skipped when tab_idx is NULL: the caller keeps
 * the ELL bins) -> async copy into pinned host memory (h_*, skipped when h_idx is NULL).  Bins are written with stride K into capacity buffers;
 * counts_host (host, 3) receives (K_mon, K_rbf, K_none); summary (device, 4 int, may be
 * NULL: no summary) and its copy h_summary (pinned, may be NULL) = [MON singular count, first
 * MON row, RBF count, first RBF row].  chunks > 1 splits the RBF rows into node-ordered chunks whose table
 * slices are copied back on a side stream while the next chunk computes; cut_host (host,
 * chunks-1 node ids where chunks 1.. start) or NULL (read back).  Returns without synchronising
 * (unless sizes were read back); info arrays flag singular stencils as in hn_weights_*.
 * Requires a tuned RBF size (hn_weights_rbf_is_tuned == 0).
 * Replaces: compute_weights approx.py:379-413 (orchestration of the calls above). */
int hn_weights_pipeline(const double* pos, int d, int64_t n, const int8_t* kind, const int* lattice_idx,
                        const int* lattice_grid, const int* grid_dims_host, const double* lo_host, double cell,
                        const int* dims_host, const int* cell_start, const int* cell_items, const double* cell_pos,
                        const double* spacing, int nops, const int* op_kind_host, const int* op_axis_host,
                        const double* op_normal_host, int n_rbf, int64_t k_mon_host, int64_t k_rbf_host, int8_t* method, int* rows,
                        int* counts, int* part_scratch, int* mon_st, int* mon_idx, double* mon_w, int* mon_info,
                        int* rbf_st, int* rbf_idx, double* rbf_w, int* rbf_info, int64_t* tab_idx,
                        int64_t* tab_sizes, double* tab_w, int64_t* h_idx, int64_t* h_sizes, double* h_w,
                        int8_t* h_method, int64_t* counts_host, int* summary, int* h_summary, int chunks,
                        const int64_t* cut_host, void* stream);

/* method per node: -1 boundary, 0 MON, 1 RBF-FD.  lattice_idx (N x d int32, INT32_MIN =
 * off-lattice) and grid (prod(grid_dims) int32, -1 vacant) may be NULL (no lattice).
 * Replaces: classify_methods approx.py:332-351. */
int hn_classify(const int8_t* kind, const int* lattice_idx, const int* grid,
                const int* grid_dims_host, int64_t n, int d, int8_t* method, void* stream);

/* MON stencils [row, axis neighbours sorted by (distance, index)] -> out (nrows x (2d+1)).
 * Replaces: _mon_stencils approx.py:360-376. */
int hn_mon_stencils(const int* rows, int64_t nrows, const double* pos, const int* lattice_idx,
                    const int* grid, const int* grid_dims_host, int d, int* out, void* stream);

/* Stable partition of node ids by method: rows_out = [MON asc | RBF-FD asc | NONE asc],
 * counts_out (3 int32, device) = class sizes; scratch >= 3*ceil(n/256) ints. */
int hn_partition_methods(const int8_t* method, int64_t n, int* rows_out, int* counts_out, int* scratch,
                         void* stream);

/* ----------------------------------------------------------------- weights (K4-K5) */

/* Outputs go straight into an ELL slab of K rows: out_idx[j*K + k] (ascending node ids),
 * out_w[(op*n + j)*K + k]; info[k] = 0 or (first zero-pivot step + 1).
 * op_kind_host/op_axis_host: nops entries; op_normal_host: nops x d (NormalDerivative). */

/* MON (2d+1)^2 collocation solves.  Replaces: _batched_mon_weights approx.py:212-234. */
int hn_weights_mon(const double* pos, int d, const int* stencils, int64_t K, int nops,
                   const int* op_kind_host, const int* op_axis_host, const double* op_normal_host,
                   int* out_idx, double* out_w, int* info, void* stream);

/* RBF-FD PHS r^3 + degree-2 saddle solves ((n+q)^2, q = 6 / 10).  row_normals (K x d) or
 * NULL: when given, every op must be HN_OP_NORMAL and uses its row's normal (the
 * `normals` variant, approx.py:260-270).  Tuned warp-cooperative kernels exist for
 * (d,n) = (2,12), (3,20), (3,30) and 1..4 ops (hn_weights_rbf_is_tuned): a static
 * null-space elimination order (pivoted LU of P, then a fixed Gauss-Jordan order whose last
 * phase pivots on the SPD Schur complement) with the partial-pivoting kernel re-solving any
 * stencil whose static pivots fall below their floors -- so the exact-zero-pivot semantics
 * of dgesv (info[k] != 0) are kept.  Other sizes use a generic thread-per-stencil kernel
 * that needs `workspace` of hn_weights_rbf_workspace(d, n, nops, K) doubles (returns 3 if
 * workspace is NULL then).  Replaces: _batched_rbf_weights approx.py:237-290. */
int hn_weights_rbf(const double* pos, int d, const int* stencils, int64_t K, int n, int nops,
                   const int* op_kind_host, const int* op_axis_host, const double* op_normal_host,
                   const double* row_normals, double* workspace, int* out_idx, double* out_w,
                   int* info, void* stream);
int hn_weights_rbf_is_tuned(int d, int n, int nops);
/* Kernel variant (0 = default).  100 = partial-pivoting kernel for every stencil, 101 = static
 * kernel with every stencil flagged (exercises the fallback), 10..19 = launch shapes (tuning).
 * Every variant matches dgesv to ~1e-13; a tuning/testing knob, not a numerics switch. */
void hn_weights_rbf_set_variant(int v);
int64_t hn_weights_rbf_workspace(int d, int n, int nops, int64_t K);

/* --------------------------------------------------------------- application (K6) */

/* Threads per block of hn_apply_ell (64, 128 or 256; tuning knob, identical results). */
void hn_apply_set_threads(int threads);

/* out[o*out_stride + rows_b[k]] = sum_j w_b[(op_sel[o]*W_b + j)*K_b + k] * field[idx_b[j*K_b + k]]
 * over up to 4 bins b (widths 0,5,7,12,20,30; width 0 writes zeros), 1..4 ops.
 * Bit-identical to scipy csr_matvec (sequential, ascending columns, no FMA).
 * Replaces: SparseOperator.apply / apply / divergence operators.py:51-54,80-90. */
int hn_apply_ell(int nbins, const int64_t* bin_K_host, const int* bin_width_host,
                 const int* const* bin_rows_host, const int* const* bin_idx_host,
                 const double* const* bin_w_host, int nops, const int* op_sel_host,
                 const double* field, double* out, int64_t out_stride, void* stream);

/* ELL bins -> the reference WeightTable layout (approx.py:311-323): idx_out (N x n_max)
 * int64 -1 padded, sizes_out (N) int64, w_out (nops x N x n_max) fp64 zero padded; every
 * node must belong to one bin. */
int hn_ell_to_table(int nbins, const int64_t* bin_K_host, const int* bin_width_host,
                    const int* const* bin_rows_host, const int* const* bin_idx_host,
                    const double* const* bin_w_host, int nops, int n_max, int64_t N, int64_t* idx_out,
                    int64_t* sizes_out, double* w_out, void* stream);

/* ------------------------------------------------------ explicit step (K7, K8, K10, K11) */

/* Bins as in hn_apply_ell over the interior operator table; planes lap_plane and
 * d_plane_host[0..d) select the Laplacian and d/dx_a weight planes.  State is SoA:
 * v[c*N + i]. */

/* Optional hyper-dissipation (PhysicsParams.dissipation != 0, solver.py:235-247): hyper_coef
 * (N fp64) = -coeff * spacing**3 as numpy computes it, hyper_lap2 = lap(lap(field)) (d x N
 * for hn_momentum, N for hn_correct_temperature); the term (hyper_coef * |v|) * hyper_lap2
 * is added to the right-hand side.  Both NULL = off. */
/* v* = v + dt*(-(v.grad)v + Pr lap v - buoy_c (T - t_ref)); buoy_host[c] = (Ra*Pr)*g[c].
 * zero_boundary != 0 fuses apply_velocity_bc (v* = 0 on the width-0 bin rows).
 * Replaces: momentum_predict + apply_velocity_bc solver.py:250-280. */
int hn_momentum(int nbins, const int64_t* bin_K_host, const int* bin_width_host,
                const int* const* bin_rows_host, const int* const* bin_idx_host,
                const double* const* bin_w_host, int lap_plane, const int* d_plane_host, int d,
                const double* v, const double* T, int64_t N, double dt, double Pr, double t_ref,
                const double* buoy_host, int zero_boundary, const double* hyper_coef,
                const double* hyper_lap2, double* vstar, void* stream);

/* rhs[0..N) = (sum_a D_a v*_a)/dt on interior rows, 0 on boundary rows; rhs[N] = 0.
 * Replaces: solver.py:295-301. */
int hn_div_rhs(int nbins, const int64_t* bin_K_host, const int* bin_width_host,
               const int* const* bin_rows_host, const int* const* bin_idx_host,
               const double* const* bin_w_host, const int* d_plane_host, int d, const double* vstar,
               int64_t N, double dt, double* rhs, void* stream);

/* v = v* - dt grad p (0 on boundary); T' = T + dt(-v.grad T + lap T) with the corrected v.
 * flags[0] |= 1 on any non-finite output, flags[1] = min non-finite T node (init INT_MAX).
 * Replaces: velocity_correct + temperature_step solver.py:317-331, 345-357. */
int hn_correct_temperature(int nbins, const int64_t* bin_K_host, const int* bin_width_host,
                           const int* const* bin_rows_host, const int* const* bin_idx_host,
                           const double* const* bin_w_host, int lap_plane, const int* d_plane_host, int d,
                           const double* vstar, const double* p, const double* T, int64_t N, double dt,
                           double* vout, double* Tout, int* flags, const double* hyper_coef,
                           const double* hyper_lap2, void* stream);

/* T[dir_idx] = dir_val; T[neu_idx[r]] = -(W_r . t0) / neu_diag[r], t0 = T with Neumann
 * entries zeroed (is_neu mask); one launch.  flags (nullable, the K10 words + a block
 * counter, int[3]): a non-finite Neumann value sets flags[0] and lowers flags[1] to its
 * node.  latch (nullable): the last block to finish also applies hn_step_latch (then flags
 * is required).  Replaces: apply_temperature_bc solver.py:334-342 (+ the per-step probe). */
int hn_temperature_bc(const int* dir_idx, const double* dir_val, int64_t ndir, const int64_t* neu_rowptr,
                      const int* neu_cols, const double* neu_vals, const int* neu_idx,
                      const double* neu_diag, const uint8_t* is_neu, int64_t nneu, double* T,
                      int* flags, int* latch, const int* pstatus, void* stream);

/* (The end-of-step latch of the finite probe rides on hn_temperature_bc: latch = [steps done,
 * first non-finite step (0 = none), lowest non-finite temperature node of that step (INT_MAX =
 * none), first step whose pressure solve reported info != 0, that info]; flags cleared.  Lets
 * the host read the probe every nu_stride steps and still report the reference's step and
 * node.  Replaces: the per-step probe of run() solver.py:448-452.) */

/* y = A x / y = b - A x for a CSR matrix (int64 rowptr), scipy csr_matvec order. */
int hn_csr_matvec(const int64_t* rowptr, const int* cols, const double* vals, const double* x,
                  int64_t nrows, double* y, void* stream);
int hn_csr_residual(const int64_t* rowptr, const int* cols, const double* vals, const double* x,
                    const double* b, int64_t nrows, double* y, void* stream);

/* ---------------------------------------------------------------- pressure (K9, K12) */

/* Supernodal sync-free triangular solve over tasks in dependency-level order (one
 * preconditioner application = permute, this for L, this for U, permute).
 * Replaces: SuperLU lu.solve inside the bicgstab preconditioner, solver.py:213-214,304-305.
 * A block [r0, r0+w) (w <= 256) has a dense in-block triangle.  kind 0: one CTA pulls the
 * block's outside part (one global hop) and solves the dense triangle in 32-column tiles
 * read from `packed` (hn_host_pack_panels; next panel by bulk async copy); kind 1: helper
 * computing the outside sums of block rows [rb, rb+rc) into ysum (heavy blocks); kind 2:
 * dense part of a heavy block, fed by its helpers (scheduled just before it); kind 3: up to
 * 8 small blocks (w <= 32) of one level, one warp each (members listed after the tasks).
 * inv: 1 = the packed diagonal tiles are inverses (x = T^-1 y per tile instead of substitution),
 * 2 = the packed triangle is the whole block's inverse (x = B^-1 y, no tile-to-tile chain).
 * blk_rw (may be NULL): per task, the width of the dense rectangle coupling the block to its
 * adjacent predecessor (lower: the rw rows before r0, upper: after r0 + w); those columns are
 * left out of the off-block sums and applied from packed rectangle panels as the
 * predecessor's tiles are solved.
 * lower: unit diagonal; upper: divides by diag.  Strict CSR, sorted columns.  x and ysum
 * (n each) are reset inside.  Deterministic. */
/* One triangular factor's supernodal task list (all device pointers; see hn_sptrsv_super). */
typedef struct hn_tri_plan {
  int lower;             /* 1: unit-lower L, 0: upper U (divides by diag) */
  int inv;               /* 0 substitution, 1 diagonal-tile inverses, 2 whole-block inverses */
  int64_t ntasks;
  const int* kind;
  const int* r0;
  const int* w;
  const int* rb;
  const int* rc;
  const int64_t* off;
  const int* rw;         /* per task: width of the dense rectangle to the adjacent predecessor block (may be NULL) */
  const int64_t* rowptr; /* strict triangle, CSR, sorted columns */
  const int* cols;
  const double* vals;
  const double* diag;    /* U only */
  const double* packed;
  /* Dense groups (optional, g_inv != NULL): row runs at the top of the elimination tree that
   * leave the task list (their rows are empty in rowptr/cols/vals; for U their diag entries
   * are 1) and are solved as x_G = inv(T_GG) (b_G - C_G x), phase by phase (<= 16 phases; the
   * runs of one phase are independent): rows [phase_ptr[p], phase_ptr[p+1]) of the arrays
   * below.  g_row: row id; g_cpl_*: CSR of C_G (the row's entries outside its run: columns
   * before it for L, after it for U) over the same row order; x[row] = sum_{c < g_cnt}
   * g_inv[g_inv_off + c] * y[g_ystart + c], the row's slice of its run's inverse triangle
   * (row-packed).  L: after the tasks; U: before them, and b's group entries are overwritten
   * with the solution. */
  int n_phases;
  int64_t phase_ptr[17];
  const int* g_row;
  const int64_t* g_cpl_rowptr;
  const int* g_cpl_cols;
  const double* g_cpl_vals;
  const int64_t* g_inv_off;
  const int* g_cnt;
  const int* g_ystart;
  const double* g_inv;
  double* g_y;           /* scratch, n fp64, owned by the plan's creator (y of the group rows) */
} hn_tri_plan;

int hn_sptrsv_super(int lower, const int* blk_kind, const int* blk_r0, const int* blk_w, const int* blk_rb,
                    const int* blk_rc, const int64_t* blk_off, const int* blk_rw, int64_t nblk, const int64_t* rowptr,
                    const int* cols, const double* vals, const double* diag, const double* packed, int inv,
                    const double* b, double* x, double* ysum, int64_t n, unsigned long long* ticket,
                    int ctas_per_sm, void* stream);

/* hn_sptrsv_super from a plan struct, dense groups included (an upper plan with groups
 * overwrites the groups' entries of b). */
int hn_sptrsv_plan(const hn_tri_plan* plan, double* b, double* x, double* ysum, int64_t n,
                   unsigned long long* ticket, int ctas_per_sm, void* stream);

/* Setup helpers on HOST arrays: dense-triangle row blocks (returns the count; blocks in row
 * order, w <= cap <= 256), their dependency levels, and the packed dense triangles of the
 * tasks of kind 0/2 (panels of 32 columns, column-major; off[t] in doubles, -1 for other
 * kinds; packed == NULL computes offsets only; returns the total, -1 if a block's in-block
 * triangle or rectangle is not dense; rw_host may be NULL).  Rectangle panels (rw_host[t] > 0)
 * come first: the predecessor's columns in its tile order, all w rows.  inverse = 1: every
 * diagonal tile's rows hold that tile's inverse; inverse = 2: the triangle panels hold the
 * inverse of the block's whole triangle (diagonal included), the block is then x = B^-1 y panel
 * by panel (diag_host = U's diagonal for upper); hn_sptrsv_super must be called with inv =
 * the same value. */
int64_t hn_host_supernodes(const int64_t* rowptr_host, const int* cols_host, int64_t n, int lower, int cap,
                           int* blk_r0_host, int* blk_w_host);
int hn_host_block_levels(const int64_t* rowptr_host, const int* cols_host, int64_t n, int lower, int64_t nblk,
                         const int* blk_r0_host, const int* blk_w_host, int* levels_host);
int64_t hn_host_pack_panels(const int64_t* rowptr_host, const int* cols_host, const double* vals_host,
                            const double* diag_host, int lower, int inverse, int64_t ntasks, const int* kind_host,
                            const int* r0_host, const int* w_host, const int* rw_host, int64_t* off_host,
                            double* packed_host);

/* Device-driven pressure solve (K9 driver, csrc/bicgstab.cu).
 * Replaces: pressure_solve's bicgstab call with the LU preconditioner, solver.py:304-305
 * (scipy BiCGStab, rtol, atol = 0, maxiter), every scalar on the device; the loop is a
 * CUDA-graph WHILE node, so no host round trip happens per solve.  setup: A = the bordered
 * Poisson matrix (CSR, n rows), the L and U task lists (hn_tri_plan), SuperLU's perm_r /
 * perm_c; all device pointers, kept (not copied) -> *handle_out.  solve: x0 NULL = zero
 * start, x0 == x = start from x's contents; status (device int[2], may be NULL) = [scipy
 * info, completed passes].  Inside a stream capture the solve is added to the caller's
 * graph; otherwise a cached graph is launched on the stream. */
int hn_pressure_setup(int64_t n, const int64_t* a_rowptr, const int* a_cols, const double* a_vals,
                      const hn_tri_plan* lower, const hn_tri_plan* upper, const int* perm_r, const int* perm_c,
                      int ctas_per_sm, int64_t* handle_out);
int hn_pressure_solve(int64_t handle, const double* b, const double* x0, double* x, double rtol, int maxiter,
                      int* status, void* stream);
int hn_pressure_free(int64_t handle);

/* Condition numbers (2-norm, s_max / s_min as numpy's SVD; inf when singular) of K local
 * weight systems, one warp each: the RBF-FD saddle matrix is symmetric (|eigenvalues|), the
 * MON matrix via M M^T; Householder tridiagonalisation + Sturm multisection.  pos: node
 * coordinates, row stride ps; stencil node j of system k at idx[k*rs + j*cs]; centers (may be
 * NULL: node 0) the centre ids; out K fp64.  Supported: MON n = 2d+1, RBF-FD (d, n) in
 * {(2,12), (3,20), (3,30)} (else returns 2).
 * Replaces: the with_kappa SVDs of approx.py:229-233, 285-289. */
int hn_condition_numbers(const double* pos, int ps, int d, const int* idx, int64_t rs, int64_t cs,
                         const int* centers, int64_t K, int n, int mon, double* out, void* stream);

/* ------------------------------------------------------ row-sharded explicit step (§8(e), F4) */

/* One rank's view of the step: its owned rows first, then the halo nodes its stencils reach
 * (grouped by owner).  The reference loop body (solver.py:439-452) has no distributed form;
 * these three calls are the device side of the 1-hop halo exchange SURVEY §8(e) specifies
 * (the transfer itself is NCCL send/recv on the same stream).
 * hn_halo_gather: out[i] = src[map[i]] (pack a send buffer, or take the local part of a
 * replicated vector).  hn_halo_scatter: dst[map[i]] = in[i] (received values into the halo
 * tail; a rank's rows into a replicated vector).  hn_remap_indices: out[i] = map[in[i]]
 * (stencil column ids to local numbering); *bad counts entries that map to < 0. */
int hn_halo_gather(const double* src, const int64_t* map, int64_t n, double* out, void* stream);
int hn_halo_scatter(const double* in, const int64_t* map, int64_t n, double* dst, void* stream);
int hn_remap_indices(const int* in, const int* map, int64_t n, int* out, int* bad, void* stream);

/* direction 0: out[perm[i]] = in[i]; direction 1: out[i] = in[perm[i]]. */
int hn_permute(int direction, const int* perm, const double* in, int64_t n, double* out, void* stream);

/* Deterministic reduction into out[0]: op 0 dot(a,b), 1 max|a|, 2 sum|a|, 3 sum a; idx
 * optional gather; scratch >= 296 doubles. */
int hn_reduce(int op, const double* a, const double* b, const int* idx, int64_t n, double* scratch,
              double* out, void* stream);

/* BiCGStab updates in numpy operation order: kind 0 y = ((y - alpha*x)*beta) + r;
 * kind 1 y = y + alpha*x. */
int hn_bicg_update(int kind, double* y, const double* x, const double* r, double alpha, double beta,
                   int64_t n, void* stream);

/* ------------------------------------------------------- node-set generation (K12) */

/* Domain + spacing + scattered-region description shared by the node-generation calls
 * (passed by pointer, read on the host; the arrays it points to are device memory).
 * Box: [lo, hi]; obstacles: kind 0 circle/sphere (par = centre[d], radius), 1 star
 * (cx, cy, mean radius, amplitude, lobes, phase), 2 ellipse (cx, cy, a, b, cos angle,
 * sin angle); curves (kinds 1, 2) carry a 1024-point parameter table (curve_t) and its
 * points (curve_tab + 2048*j for obstacle j).
 * Spacing (SpacingFunction nodegen.py:33-60): graded = 0 -> h_r everywhere, else
 * h_s + (h_r - h_s)*clip(obstacle_distance/width, 0, 1).
 * Region (_scattered_region nodegen.py:384-433): 0 none, 1 everywhere, 2 dvd quarters
 * (rc = box centre), 3 axis split (axis, p[axis] < rt[0]; near: < rt[1]), 4 obstacle
 * layer (obstacle_distance < rt[0]; near: < rt[1]); quarters' near test: seam < rt[1]. */
typedef struct hn_geom {
  int dim;
  int n_obs;
  double lo[3], hi[3];
  int graded;
  double h_r, h_s, width;
  const int* obs_kind;
  const double* obs_par; /* n_obs x 8 */
  const double* curve_t; /* 1024 */
  const double* curve_tab; /* n_obs x 1024 x 2 */
  int region;
  int axis;
  double rc[2];
  double rt[2];
} hn_geom;

/* Point queries (pts: n x dim fp64, unpadded): mode 0 signed distance to the fluid
 * region, 1 obstacle distance (+inf without obstacles), 2 target spacing, 3 box signed
 * distance, 4 region predicate (0/1), 5 near-region predicate (0/1).
 * Replaces: DomainSpec.signed_distance / obstacle_distance / box_signed_distance
 * geometry.py:279-312, SpacingFunction.__call__ nodegen.py:53-60, the region predicates
 * nodegen.py:384-433. */
int hn_geom_eval(const hn_geom* g, const double* pts, int64_t n, int mode, double* out, void* stream);

/* Interior lattice: every key k (1 <= k_a < cells_a) at lo + k*step, kept when
 * signed_distance <= thr and, with drop_region, outside the scattered region; when
 * carve > 0 also obstacle_distance >= carve.  Writes the kept nodes in C (ij) order:
 * out_pos (K x dim), out_key (K x dim int64); *out_count_host = K (synchronises).
 * out_* must hold prod(cells-1) rows.
 * Replaces: regular_fill nodegen.py:196-216, carve_transition :219-227, the region cut
 * of hybrid_discretize :457-461. */
int hn_lattice_fill(const hn_geom* g, const int64_t* cells_host, const double* step_host, double thr,
                    int drop_region, double carve, double* out_pos, int64_t* out_key, int64_t* out_count_host,
                    void* stream);

/* One advancing-front wave, part 1: the candidates of k parents (parent ids `front`, or
 * front_lo + 0..k-1 when front is NULL) from the caller's random draws rnd (k x (d+1) x d
 * standard normals) and u (k x (3d+1) uniforms): 2d axis + d+1 random unit directions in
 * argsort(u) order, radius by the 3-step spacing fixed point; ok = inside the domain by
 * half a spacing (and in the region when use_region).  cand ((3d+1)k x d), hcand, ok.
 * Replaces: _wave_candidates nodegen.py:270-294 and the ok mask of scattered_fill :346-349. */
int hn_front_candidates(const hn_geom* g, const double* pts, const double* hs, const int64_t* front,
                        int64_t front_lo, int64_t k, const double* rnd, const double* u, int use_region,
                        double* cand, double* hcand, uint8_t* ok, void* stream);

/* Part 2: first-fit acceptance of the m candidates in order, exactly as the sequential
 * loop of scattered_fill nodegen.py:350-374 (reject when any node -- existing or accepted
 * earlier in this wave -- lies closer than 0.995*h_c, or a regular seed closer than seam;
 * seam <= 0: no seam rule), decided in parallel (pre-test against the existing nodes, then
 * an in-order sync-free resolution of the in-wave conflicts).  Accepted candidates are
 * appended in order at pts[count..], hs[count..]; *new_count_host receives the new count
 * (synchronises).  Needs capacity >= count + m.  cell >= every acceptance radius.
 * seed_regular: n_seeds bytes (NULL = none regular). */
int hn_front_accept(int d, double* pts, double* hs, int64_t count, int64_t capacity, const uint8_t* seed_regular,
                    int64_t n_seeds, const double* cand, const double* hcand, const uint8_t* ok, int64_t m,
                    double seam, const double* lo_host, const double* hi_host, double cell,
                    int64_t* new_count_host, void* stream);

/* Lattice index map (hybrid_discretize nodegen.py:503-516): grid ((cells_a+1) per axis,
 * int64) = -1, then grid[key_i] = i for the n_reg regular nodes (keys: n_reg x d), then
 * every boundary node (positions bpos, n_b x d; node id = b0 + i) whose position lies on
 * a lattice point within tol takes a vacant key (lowest id first) and gets its key in
 * out_bkey (n_b x d int64; LATTICE_NONE = INT64_MIN otherwise). */
int hn_lattice_map(int d, const int64_t* cells_host, const double* origin_host, const double* step_host,
                   double tol, const int64_t* keys, int64_t n_reg, const double* bpos, int64_t n_b, int64_t b0,
                   int64_t* grid, int64_t* out_bkey, void* stream);

/* Pairs i < j closer than 0.5*min(h_i, h_j) - 1e-12 (pts n x d, h n); cell >= 0.5*max h
 * and the points inside [lo, hi] (a window of 3^d cells is then exact); synchronises.
 * Replaces: NodeSet.min_distance_violations nodegen.py:139-148 (cKDTree.query_pairs). */
int hn_close_pairs(int d, const double* pts, const double* h, int64_t n, const double* lo_host,
                   const double* hi_host, double cell, int64_t* out_count_host, void* stream);

/* ----------------------------------------------------------- diagnostics / peaks */

/* DFMA throughput probe: `blocks` x 256 threads, `iters` x 16 independent DFMA chains
 * per thread; out[0] receives a checksum.  Used by bench.py for the fp64 peak. */
int hn_bench_dfma(double* out, int blocks, int iters, void* stream);
/* FP64 tensor-core (DMMA m8n8k4) probe: blocks x 8 warps x iters x 4 MMAs of 512 flop. */
int hn_bench_dmma(double* out, int blocks, int iters, void* stream);

int hn_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HN_H_ */
