// K4/K5: batched per-stencil fp64 weight solves.
//
// Reference: _batched_mon_weights (pkg/src/hybridnodes/approx.py:212-234) and
// _batched_rbf_weights (approx.py:237-290), both ending in np.linalg.solve (LAPACK
// dgesv, LU with partial pivoting).  For every stencil (centre first):
//     rel = pts - pts[0];  scale = max_j ||rel_j||;  y = rel / scale
//   MON:  M[b][j] = basis_b(y_j), basis = [1, y_a.., y_a^2..]          (2d+1)^2
//   RBF:  [[A P],[P^T 0]], A_ij = |y_i - y_j|^3, P_jm = monomial_m(y_j)  (n+q)^2
//   RHS:  operator applied to each basis function at the centre (approx.py:81-97,
//         169-179, 199-209); weights = solution[:n] / scale^order.
// Output rows are stored ascending by node index (approx.py:407-410), directly into
// the device ELL slab of the bin: idx[j*K + k], w[(op*n + j)*K + k].
//
// MON: one thread per stencil, matrix in registers, LU with partial pivoting.
// RBF: LPS lanes per stencil, RPL matrix rows per lane held in registers
//      (row i lives in lane i % LPS, slot i / LPS), 32/LPS stencils per warp.
//      Gauss-Jordan with implicit partial pivoting: every step picks the largest
//      |a_ik| among not-yet-pivoted rows (segmented shuffle argmax on a packed
//      key), the owner lane stages the pivot row in shared memory, and every lane
//      updates all of its rows with DFMA.  Gauss-Jordan instead of LU+back
//      substitution: in this layout lanes whose rows are already eliminated would
//      idle anyway, and it removes the sequential, latency-bound back-solve.
//      Exact zero pivot => SingularSystemError (info = step + 1), as dgesv does.
#include <cfloat>
#include <climits>

#include "hn_common.cuh"

namespace hn {

struct OpSpec {
  int nops;
  int kind[4];        // OpKind
  int axis[4];        // Partial axis
  int order[4];       // scale exponent
  double normal[4][3];
};

// predicated select that NVVM cannot turn back into dynamic (local-memory) indexing
__device__ __forceinline__ double selp(bool c, double a, double b) {
  double r;
  asm("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\tselp.f64 %0, %1, %2, p;\n\t}"
      : "=d"(r) : "d"(a), "d"(b), "r"(static_cast<int>(c)));
  return r;
}

template <int D>
__device__ __forceinline__ double pick_axis(const double* y, int axis) {
  double v = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) v = (a == axis) ? y[a] : v;
  return v;
}

template <int D>
constexpr int poly_count() { return D == 2 ? 6 : 10; }

// exponent table of _monomial_exponents (approx.py:69-78): [1, x_a.., then
// combinations_with_replacement of degree 2 in lexicographic order]
template <int D>
__device__ __forceinline__ void mono_exp(int m, int* e) {
  // 2-bit exponents packed per monomial index (no local-memory table lookups)
  if constexpr (D == 2) {
    // e0: 0 1 0 2 1 0   e1: 0 0 1 0 1 2
    constexpr unsigned E0 = (1u << 2) | (2u << 6) | (1u << 8);
    constexpr unsigned E1 = (1u << 4) | (1u << 8) | (2u << 10);
    e[0] = (E0 >> (2 * m)) & 3u;
    e[1] = (E1 >> (2 * m)) & 3u;
  } else {
    // e0: 0 1 0 0 2 1 1 0 0 0   e1: 0 0 1 0 0 1 0 2 1 0   e2: 0 0 0 1 0 0 1 0 1 2
    constexpr unsigned E0 = (1u << 2) | (2u << 8) | (1u << 10) | (1u << 12);
    constexpr unsigned E1 = (1u << 4) | (1u << 10) | (2u << 14) | (1u << 16);
    constexpr unsigned E2 = (1u << 6) | (1u << 12) | (1u << 16) | (2u << 18);
    e[0] = (E0 >> (2 * m)) & 3u;
    e[1] = (E1 >> (2 * m)) & 3u;
    e[2] = (E2 >> (2 * m)) & 3u;
  }
}

// monomial value with the reference's evaluation order: ((1 * y0^e0) * y1^e1) * y2^e2,
// factors with e = 0 skipped, y^2 = y*y  (approx.py:189-196)
template <int D>
__device__ __forceinline__ double mono_val(int m, const double* y) {
  int e[D];
  mono_exp<D>(m, e);
  double v = 1.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (e[a] == 1) v = __dmul_rn(v, y[a]);
    else if (e[a] == 2) v = __dmul_rn(v, __dmul_rn(y[a], y[a]));
  }
  return v;
}

// (op p_m)(0) -- approx.py:81-97
template <int D>
__device__ __forceinline__ double poly_rhs(const OpSpec& ops, int o, int m, bool use_rn, const double* rn) {
  int e[D];
  mono_exp<D>(m, e);
  int deg = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) deg += e[a];
  const int kind = ops.kind[o];
  if (kind == kOpLaplacian) {
    double r = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a)
      if (e[a] == 2 && deg == 2) r += 2.0;
    return r;
  }
  if (deg != 1) return 0.0;
  int ax = 0;
#pragma unroll
  for (int a = 0; a < D; ++a)
    if (e[a] == 1) ax = a;
  if (kind == kOpPartial) return ax == ops.axis[o] ? 1.0 : 0.0;
  double v = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) v = (a == ax) ? (use_rn ? rn[a] : ops.normal[o][a]) : v;
  return v;
}

// (op phi(. - y_j))(0) with phi = r^3 -- approx.py:199-209 (normals variant :260-270)
template <int D>
__device__ __forceinline__ double phs_rhs(const OpSpec& ops, int o, const double* y, double r,
                                          bool use_rn, const double* rn) {
  const int kind = ops.kind[o];
  if (kind == kOpLaplacian) return 3.0 * (D + 1) * r;
  if (kind == kOpPartial) return -3.0 * r * pick_axis<D>(y, ops.axis[o]);
  double dot = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) dot = fma(y[a], use_rn ? rn[a] : ops.normal[o][a], dot);
  return -3.0 * r * dot;
}

// same value as mono_val but branch-free for a per-lane (runtime) monomial index
template <int D>
__device__ __forceinline__ double mono_val_sel(int m, const double* y) {
  int e[D];
  mono_exp<D>(m, e);
  double v = 1.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double f = e[a] == 2 ? y[a] * y[a] : (e[a] == 1 ? y[a] : 1.0);
    v = v * f;
  }
  return v;
}

// sqrt via MUFU rsqrt seed + two Newton steps (~1 ulp, no slow-path call); 0 -> 0
__device__ __forceinline__ double fast_sqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return x > 0.0 ? x * y : 0.0;
}

template <int D>
__device__ __forceinline__ double norm_fast(const double* y) {
  double s = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) s = fma(y[a], y[a], s);
  return fast_sqrt(s);
}

template <int D>
__device__ __forceinline__ double norm_rn(const double* y) {
  double s = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) s = __dadd_rn(s, __dmul_rn(y[a], y[a]));
  return __dsqrt_rn(s);
}

// reciprocal: MUFU seed + two Newton steps (~1 ulp; pivots are O(1) after scaling)
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  return y;
}

// ============================ MON (thread per stencil) ============================
// Fast path for a lattice MON stencil [centre, the 2d axis neighbours]: with the columns in
// canonical order (centre, -x, +x, -y, +y, ...) every such system has one structure whose
// partial-pivoting choices are known -- column 0 -> row 0 (basis 1), column -a -> row 1+a
// (y_a, pivot -1), column +a -> row 1+D+a (y_a^2, pivot 2) -- so it is eliminated in that
// static order: no pivot search, no row swaps (their selects were 3/4 of the general
// path's instructions), reciprocal multiplies.  Returns false (nothing written) for any
// other stencil or any pivot below 1/4 of its column; the caller then runs the general
// partial-pivoting path.  Weights agree with dgesv's to rounding (kappa ~ 10).
template <int D, int NOPS>
__device__ __forceinline__ bool mon_static(const double* __restrict__ pos, const int* sid, const double* c,
                                           int64_t K, int64_t k, const OpSpec& ops, int* __restrict__ out_idx,
                                           double* __restrict__ out_w) {
  constexpr int N = 2 * D + 1;
  constexpr int NC = N + NOPS;
  // slots and scale from the stencil-order offsets (sign/axis are scale-invariant)
  int cn[N];
#pragma unroll
  for (int s = 0; s < N; ++s) cn[s] = -1;
  cn[0] = sid[0];
  double scale = 0.0;
  bool ok = true;
  unsigned used = 1u;
#pragma unroll
  for (int j = 1; j < N; ++j) {
    double p[D], yj[D];
    load_point<D>(pos, sid[j], p);
#pragma unroll
    for (int a = 0; a < D; ++a) yj[a] = __dsub_rn(p[a], c[a]);
    scale = fmax(scale, norm_rn<D>(yj));
    int ax = 0;
    double best = fabs(yj[0]);
    int nz = best != 0.0;
#pragma unroll
    for (int a = 1; a < D; ++a) {
      nz += fabs(yj[a]) != 0.0;
      const bool g = fabs(yj[a]) > best;
      best = g ? fabs(yj[a]) : best;
      ax = g ? a : ax;
    }
    const int sl = 1 + 2 * ax + (pick_axis<D>(yj, ax) > 0.0 ? 1 : 0);
    ok = ok && nz == 1 && !(used & (1u << sl));
    used |= 1u << sl;
#pragma unroll
    for (int s = 1; s < N; ++s) cn[s] = (s == sl) ? sid[j] : cn[s];
  }
  if (!ok) return false;
  // In canonical order the system is block-structured with exact zeros (a neighbour along
  // axis a has y_b = 0 exactly for b != a, the centre has y = 0): row 0 (basis 1) couples
  // every column, and axis a only couples rows (y_a, y_a^2) with columns (-a, +a).  The
  // static elimination (pivot rows 0, 1+a, 1+D+a) therefore reduces to one 2x2 solve per
  // axis plus the row-0 back substitution -- the same operations the dense static
  // elimination performs on its nonzeros, in the same order.
  double x[N][NOPS];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double pm[D], pp[D];
    load_point<D>(pos, cn[1 + 2 * a], pm);
    load_point<D>(pos, cn[2 + 2 * a], pp);
    const double u = __ddiv_rn(__dsub_rn(pick_axis<D>(pm, a), c[a]), scale);  // y_a at -a (pivot)
    const double v = __ddiv_rn(__dsub_rn(pick_axis<D>(pp, a), c[a]), scale);  // y_a at +a
    const double su = __dmul_rn(u, u), sv = __dmul_rn(v, v);
    if (!(fabs(u) >= 0.25 * fmax(fabs(u), fabs(su)) && u != 0.0)) return false;
    const double inv_u = fast_rcp(u);
    const double l = su * inv_u;
    const double p2 = fma(-l, v, sv);
    if (p2 == 0.0) return false;
    const double inv_p = fast_rcp(p2);
#pragma unroll
    for (int o = 0; o < NOPS; ++o) {
      const int kind = ops.kind[o];
      const double lin = kind == kOpPartial ? ((a == ops.axis[o]) ? 1.0 : 0.0)
                                            : (kind == kOpNormal ? ops.normal[o][a] : 0.0);
      const double sq = kind == kOpLaplacian ? 2.0 : 0.0;
      const double xp = fma(-l, lin, sq) * inv_p;
      x[2 + 2 * a][o] = xp;
      x[1 + 2 * a][o] = fma(-v, xp, lin) * inv_u;
    }
  }
#pragma unroll
  for (int o = 0; o < NOPS; ++o) {
    double acc = 0.0;
#pragma unroll
    for (int s2 = 1; s2 < N; ++s2) acc = fma(-1.0, x[s2][o], acc);
    x[0][o] = acc;
  }
  const double r1 = 1.0 / scale, r2 = 1.0 / __dmul_rn(scale, scale);
#pragma unroll
  for (int s = 0; s < N; ++s) {
    int rank = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) rank += (sid[i] < cn[s]);  // lattice stencils have distinct ids
    out_idx[rank * K + k] = cn[s];
#pragma unroll
    for (int o = 0; o < NOPS; ++o)
      out_w[(static_cast<int64_t>(o) * N + rank) * K + k] = x[s][o] * (ops.order[o] == 2 ? r2 : r1);
  }
  return true;
}

// Fast kernel: canonical lattice stencils (mon_static); any other row is flagged
// (flag[k] = 1) for mon_general_kernel, which runs the general partial-pivoting path.
// Two kernels, so the general path's register budget does not set the fast path's
// occupancy (a called device function would).
template <int D, int NOPS>
__global__ void __launch_bounds__(128) mon_weights_kernel(const double* __restrict__ pos,
                                                          const int* __restrict__ stencils, int64_t K,
                                                          OpSpec ops, int* __restrict__ out_idx,
                                                          double* __restrict__ out_w, int* __restrict__ info,
                                                          int* __restrict__ flag) {
  constexpr int N = 2 * D + 1;
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= K) return;
  int sid[N];
#pragma unroll
  for (int j = 0; j < N; ++j) sid[j] = __ldg(stencils + k * N + j);
  double c[D];
  load_point<D>(pos, sid[0], c);
  const bool done = mon_static<D, NOPS>(pos, sid, c, K, k, ops, out_idx, out_w);
  flag[k] = done ? 0 : 1;
  if (done && info) info[k] = 0;
}

template <int D, int NOPS>
__device__ __forceinline__ void mon_general(const double* __restrict__ pos, const int* __restrict__ stencils,
                                            int64_t K, int64_t k, const OpSpec& ops, int* __restrict__ out_idx,
                                            double* __restrict__ out_w, int* __restrict__ info);

template <int D, int NOPS>
__global__ void __launch_bounds__(128) mon_general_kernel(const double* __restrict__ pos,
                                                          const int* __restrict__ stencils, int64_t K,
                                                          OpSpec ops, int* __restrict__ out_idx,
                                                          double* __restrict__ out_w, int* __restrict__ info,
                                                          const int* __restrict__ flag) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= K || !flag[k]) return;
  mon_general<D, NOPS>(pos, stencils, K, k, ops, out_idx, out_w, info);
}

template <int D, int NOPS>
__device__ __forceinline__ void mon_general(const double* __restrict__ pos, const int* __restrict__ stencils,
                                            int64_t K, int64_t k, const OpSpec& ops, int* __restrict__ out_idx,
                                            double* __restrict__ out_w, int* __restrict__ info) {
  constexpr int N = 2 * D + 1;
  constexpr int NC = N + NOPS;
  int sid[N];
#pragma unroll
  for (int j = 0; j < N; ++j) sid[j] = __ldg(stencils + k * N + j);
  double c[D];
  load_point<D>(pos, sid[0], c);
  double y[N][D];
  double scale = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double p[D];
    load_point<D>(pos, sid[j], p);
#pragma unroll
    for (int a = 0; a < D; ++a) y[j][a] = __dsub_rn(p[a], c[a]);
    scale = fmax(scale, norm_rn<D>(y[j]));
  }
#pragma unroll
  for (int j = 0; j < N; ++j)
#pragma unroll
    for (int a = 0; a < D; ++a) y[j][a] = __ddiv_rn(y[j][a], scale);

  // M[b][j] = basis_b(y_j): rows = [1, y_a (a<D), y_a^2 (a<D)]  (approx.py:158-166)
  double m[N][NC];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    m[0][j] = 1.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      m[1 + a][j] = y[j][a];
      m[1 + D + a][j] = __dmul_rn(y[j][a], y[j][a]);
    }
  }
  // RHS (approx.py:169-179), branch-free so the matrix stays in registers
#pragma unroll
  for (int o = 0; o < NOPS; ++o) {
    const int kind = ops.kind[o];
    m[0][N + o] = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double lin = kind == kOpPartial ? ((a == ops.axis[o]) ? 1.0 : 0.0)
                                            : (kind == kOpNormal ? ops.normal[o][a] : 0.0);
      m[1 + a][N + o] = lin;
      m[1 + D + a][N + o] = kind == kOpLaplacian ? 2.0 : 0.0;
    }
  }
  // LU with partial pivoting (first maximal |pivot|, as idamax), physical row swaps.
  // Loops keep constant trip counts (guards instead of triangular bounds) so NVVM
  // unrolls them before scalar replacement and the matrix never leaves registers.
  int sing = 0;
#pragma unroll
  for (int kk = 0; kk < N; ++kk) {
    int p = kk;
    double best = fabs(m[kk][kk]);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (i > kk) {
        const double v = fabs(m[i][kk]);
        const bool g = v > best;
        best = g ? v : best;
        p = g ? i : p;
      }
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (i > kk) {
        const bool sw = (p == i);
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          if (j >= kk) {
            const double t = m[i][j];
            m[i][j] = selp(sw, m[kk][j], t);
            m[kk][j] = selp(sw, t, m[kk][j]);
          }
        }
      }
    }
    const double piv = m[kk][kk];
    if (piv == 0.0 && sing == 0) sing = kk + 1;
    const double inv = 1.0 / piv;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (i > kk) {
        const double l = m[i][kk] * inv;
#pragma unroll
        for (int j = 0; j < NC; ++j)
          if (j > kk) m[i][j] = fma(-l, m[kk][j], m[i][j]);
      }
    }
  }
  // back substitution for every RHS, in place in the RHS columns
#pragma unroll
  for (int o = 0; o < NOPS; ++o) {
#pragma unroll
    for (int i = N - 1; i >= 0; --i) {
      double s = m[i][N + o];
#pragma unroll
      for (int j = 0; j < N; ++j)
        if (j > i) s = fma(-m[i][j], m[j][N + o], s);
      m[i][N + o] = s / m[i][i];
    }
  }
  if (info) info[k] = sing;
  // ascending-index storage order: rank of every stencil node
  const double s2 = __dmul_rn(scale, scale);
#pragma unroll
  for (int j = 0; j < N; ++j) {
    int rank = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) rank += (sid[i] < sid[j]) || (sid[i] == sid[j] && i < j);
    out_idx[rank * K + k] = sid[j];
#pragma unroll
    for (int o = 0; o < NOPS; ++o) {
      const double den = ops.order[o] == 2 ? s2 : scale;
      out_w[(static_cast<int64_t>(o) * N + rank) * K + k] = __ddiv_rn(m[j][N + o], den);
    }
  }
}

// ===================== RBF-FD (LPS lanes per stencil, rows in registers) ===================
template <int D, int NST, int NOPS>
struct __align__(16) RbfSmem {  // 16 B: every system's prow takes v2.f64 stores
  static constexpr int NQ = poly_count<D>();
  static constexpr int NS = NST + NQ;
  static constexpr int NC = NS + NOPS;
  static constexpr int NCP = (NC + 1) & ~1;  // even length keeps every pair 16 B aligned
  double prow[2][NCP + 2];                      // double-buffered pivot row (16 B aligned pairs)
  double inv_hist[NS + (NS & 1)];               // 1/pivot of every step
  double y[NST][D];
  double w[NST][NOPS];
  int sid[NST];
};

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// predicated shared stores (no branch, no reconvergence bookkeeping)
__device__ __forceinline__ void st_pred2(bool p, unsigned addr, double x, double y) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t@q st.shared.v2.f64 [%1], {%2, %3};\n\t}"
               :: "r"(static_cast<int>(p)), "r"(addr), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void st_pred1(bool p, unsigned addr, double x) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t@q st.shared.f64 [%1], %2;\n\t}"
               :: "r"(static_cast<int>(p)), "r"(addr), "d"(x) : "memory");
}

// r^3 from r^2: MUFU rsqrt seed + two Newton steps (~1 ulp), exact 0 at r^2 = 0 (the
// clamp keeps rsqrt finite there: r = 1e-300 * 1e150, and d2 * r = 0 with no select)
__device__ __forceinline__ double cube_from_sq(double d2) {
  const double q = fmax(d2, 1e-300);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
  const double h = 0.5 * q;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return d2 * (q * y);
}

template <int D, int NST, int NOPS, int LPS, int RPL, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) rbf_weights_kernel(
    const double* __restrict__ pos, const int* __restrict__ stencils, int64_t K, OpSpec ops,
    const double* __restrict__ row_normals, int* __restrict__ out_idx, double* __restrict__ out_w,
    int* __restrict__ info) {
  constexpr int NQ = poly_count<D>();
  constexpr int NS = NST + NQ;
  constexpr int NC = NS + NOPS;
  constexpr int SPW = 32 / LPS;
  static_assert(LPS * RPL >= NS, "rows do not fit");
  static_assert(NS <= 63, "packed pivot key holds 6 row bits");
  using Sm = RbfSmem<D, NST, NOPS>;
  __shared__ __align__(16) Sm smem_all[WARPS * SPW];

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int sys_w = lane / LPS;                 // system slot within the warp
  const int s = lane - sys_w * LPS;             // lane within the system segment
  const bool lane_live = sys_w < SPW;
  const int seg_base = sys_w * LPS;
  const int64_t k_raw = (static_cast<int64_t>(blockIdx.x) * WARPS + warp) * SPW + (lane_live ? sys_w : 0);
  const bool sys_live = lane_live && k_raw < K;
  const int64_t k = k_raw < K ? k_raw : K - 1;  // idle segments recompute the last stencil
  Sm& sm = smem_all[warp * SPW + (lane_live ? sys_w : 0)];
  // butterfly partner in segment-relative numbering; out-of-segment partners read
  // themselves, which leaves segment lane 0 holding the full reduction
  auto seg_src = [&](int off) {
    const int t = s ^ off;
    return (lane_live && t < LPS) ? seg_base + t : lane;
  };

  const bool use_rn = row_normals != nullptr;
  double rn[D];
#pragma unroll
  for (int a = 0; a < D; ++a) rn[a] = use_rn ? __ldg(row_normals + k * D + a) : 0.0;

  // ---- gather, shift to the centre, scale by the stencil radius (approx.py:245-250) ----
  double c[D];
  load_point<D>(pos, __ldg(stencils + k * NST), c);
  double myy[RPL][D];
  double scale = 0.0;
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int j = s + r * LPS;
#pragma unroll
    for (int a = 0; a < D; ++a) myy[r][a] = 0.0;
    if (j < NST) {
      const int id = __ldg(stencils + k * NST + j);
      if (lane_live) sm.sid[j] = id;
      double p[D];
      load_point<D>(pos, id, p);
#pragma unroll
      for (int a = 0; a < D; ++a) myy[r][a] = __dsub_rn(p[a], c[a]);
      scale = fmax(scale, norm_rn<D>(myy[r]));
    }
  }
#pragma unroll
  for (int off = 1; off < LPS; off <<= 1) scale = fmax(scale, __shfl_sync(0xffffffffu, scale, seg_src(off)));
  scale = __shfl_sync(0xffffffffu, scale, lane_live ? seg_base : lane);
  const double s1 = 1.0 / scale;
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int j = s + r * LPS;
    if (j < NST) {
#pragma unroll
      for (int a = 0; a < D; ++a) {
        // exact division as the reference (approx.py:250): local coordinates are bitwise
        // identical, and exact-arithmetic singular stencils still hit an exact zero pivot
        myy[r][a] = __ddiv_rn(myy[r][a], scale);
        if (lane_live) sm.y[j][a] = myy[r][a];
      }
    }
  }
  __syncwarp();

  // ---- assemble my rows of [[A P],[P^T 0]] | RHS (approx.py:254-277) ----
  double a[RPL][NC];
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = s + r * LPS;
    if (i < NST) {
#pragma unroll
      for (int j = 0; j < NST; ++j) {
        double d2 = 0.0;
#pragma unroll
        for (int q = 0; q < D; ++q) {
          const double t = myy[r][q] - sm.y[j][q];
          d2 = fma(t, t, d2);
        }
        a[r][j] = cube_from_sq(d2);
      }
#pragma unroll
      for (int m = 0; m < NQ; ++m) a[r][NST + m] = mono_val<D>(m, myy[r]);
      const double r0 = norm_rn<D>(myy[r]);
#pragma unroll
      for (int o = 0; o < NOPS; ++o) a[r][NS + o] = phs_rhs<D>(ops, o, myy[r], r0, use_rn, rn);
    } else if (i < NS) {
      const int m = i - NST;
#pragma unroll
      for (int j = 0; j < NST; ++j) {
        double yj[D];
#pragma unroll
        for (int q = 0; q < D; ++q) yj[q] = sm.y[j][q];
        a[r][j] = mono_val_sel<D>(m, yj);
      }
#pragma unroll
      for (int mm = 0; mm < NQ; ++mm) a[r][NST + mm] = 0.0;
#pragma unroll
      for (int o = 0; o < NOPS; ++o) a[r][NS + o] = poly_rhs<D>(ops, o, m, use_rn, rn);
    } else {
#pragma unroll
      for (int j = 0; j < NC; ++j) a[r][j] = 0.0;
    }
  }

  // ---- Gauss-Jordan with implicit partial pivoting, branch-free, software-pipelined ----
  // tag[r] = 63 - row id identifies the (lane, slot) of every row; padding rows start done.
  // Step kk: select + stage pivot row kk, update column kk+1 first, start the pivot
  // search of step kk+1 (shuffle chain + speculative reciprocal), then the bulk update
  // runs while that search is in flight.
  // vm[r] = 0x7fffffc0 | tag while row r is live, 0 once it has pivoted: the search key of
  // a row is then one LOP3, (hi(a) | 63) & vm = (|a| top bits | tag) or 0 (no predicates)
  unsigned vm[RPL];
  int pcol[RPL];
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = s + r * LPS;
    vm[r] = (!lane_live || i >= NS) ? 0u : (0x7fffffc0u | static_cast<unsigned>(63 - i));
    pcol[r] = -1;
  }
  const unsigned pbase0 = smem_addr(&sm.prow[0][0]);
  const unsigned pbase1 = smem_addr(&sm.prow[1][0]);
  const unsigned hist = smem_addr(&sm.inv_hist[0]);

  unsigned key = 0;
  auto search = [&](int col) {  // local key of column col, then the segmented max
    key = 0;
#pragma unroll
    for (int r = 0; r < RPL; ++r)
      key = max(key, (static_cast<unsigned>(__double2hiint(a[r][col])) | 63u) & vm[r]);
#pragma unroll
    for (int off = 1; off < LPS; off <<= 1) key = max(key, __shfl_sync(0xffffffffu, key, seg_src(off)));
    key = __shfl_sync(0xffffffffu, key, lane_live ? seg_base : lane);
  };
  search(0);

#pragma unroll
  for (int kk = 0; kk < NS; ++kk) {
    const int buf = kk & 1;
    const unsigned pbase = buf ? pbase1 : pbase0;
    const unsigned ptag = key & 63u;
    bool isp[RPL];
    bool own_any = false;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      // live ptags are >= 46, so a pivoted (vm = 0) row never matches; idle lanes (which
      // alias segment 0's shared slot) see ptag = 0 and must be excluded explicitly
      isp[r] = ((vm[r] & 63u) == ptag) && lane_live;
      own_any = own_any || isp[r];
    }
    // owner stages the pivot row, columns kk..NC-1 (prow[kk] = the pivot)
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      int j = kk;
      if (j & 1) {
        st_pred1(isp[r], pbase + 8u * j, a[r][j]);
        ++j;
      }
#pragma unroll
      for (int jj = 0; jj < NC; jj += 2) {
        if (jj >= j) {
          if (jj + 1 < NC) st_pred2(isp[r], pbase + 8u * jj, a[r][jj], a[r][jj + 1]);
          else st_pred1(isp[r], pbase + 8u * jj, a[r][jj]);
        }
      }
    }
    __syncwarp();
    const double* prow = sm.prow[buf];
    const double inv = fast_rcp(prow[kk]);  // every lane: 1/pivot (NaN for a zero pivot)
    st_pred1(own_any, hist + 8u * kk, inv);
    double l[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      pcol[r] = isp[r] ? kk : pcol[r];
      vm[r] = isp[r] ? 0u : vm[r];
      l[r] = a[r][kk] * (isp[r] ? 0.0 : inv);
    }
    if (kk + 1 < NS) {
#pragma unroll
      for (int r = 0; r < RPL; ++r) a[r][kk + 1] = fma(-l[r], prow[kk + 1], a[r][kk + 1]);
      search(kk + 1);
    }
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
#pragma unroll
      for (int j = 0; j < NC; ++j)
        if (j > kk + 1 || (j == kk + 1 && kk + 1 >= NS)) a[r][j] = fma(-l[r], prow[j], a[r][j]);
    }
  }

  // ---- solution x_{pcol} = rhs / pivot; stage the n weights (approx.py:282) ----
  // a zero pivot leaves a non-finite reciprocal in the history: dgesv's singular case
  __syncwarp();
  int sing = 0;
  if (s == 0) {
#pragma unroll
    for (int kk = NS - 1; kk >= 0; --kk)
      if (!isfinite(sm.inv_hist[kk])) sing = kk + 1;
  }
  const double s2 = s1 * s1;
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    if (lane_live && pcol[r] >= 0 && pcol[r] < NST) {
      const double pi = sm.inv_hist[pcol[r]];
#pragma unroll
      for (int o = 0; o < NOPS; ++o) sm.w[pcol[r]][o] = a[r][NS + o] * pi;
    }
  }
  int sflag = sing;
#pragma unroll
  for (int off = 1; off < LPS; off <<= 1) {
    const int o = __shfl_sync(0xffffffffu, sflag, seg_src(off));
    sflag = (sflag == 0) ? o : sflag;
  }
  sflag = __shfl_sync(0xffffffffu, sflag, lane_live ? seg_base : lane);
  __syncwarp();
  if (!sys_live) return;
  if (info && s == 0) info[k] = sflag;
  // ---- epilogue: ascending node-index order, un-scale (approx.py:283-284, 407-410) ----
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int j = s + r * LPS;
    if (j < NST) {
      const int id = sm.sid[j];
      int rank = 0;
#pragma unroll
      for (int i = 0; i < NST; ++i) {
        const int o = sm.sid[i];
        rank += (o < id) || (o == id && i < j);
      }
      out_idx[static_cast<int64_t>(rank) * K + k] = id;
#pragma unroll
      for (int o = 0; o < NOPS; ++o) {
        const double f = ops.order[o] == 2 ? s2 : s1;
        out_w[(static_cast<int64_t>(o) * NST + rank) * K + k] = sm.w[j][o] * f;
      }
    }
  }
}

// ===================== generic fallback (any n, any op count): thread per stencil ==========
// Used for stencil sizes without a tuned instantiation (per-stencil API calls in tests).
// Matrix lives in a caller-provided global workspace; LU with partial pivoting + row swaps.
template <int D>
__global__ void rbf_weights_generic_kernel(const double* __restrict__ pos, const int* __restrict__ stencils,
                                           int64_t K, int nst, OpSpec ops, const double* __restrict__ row_normals,
                                           double* __restrict__ work, int* __restrict__ out_idx,
                                           double* __restrict__ out_w, int* __restrict__ info) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= K) return;
  constexpr int NQ = poly_count<D>();
  const int ns = nst + NQ, nops = ops.nops, nc = ns + nops;
  double* A = work + k * static_cast<int64_t>(ns) * nc;  // row-major ns x nc
  double* Y = work + K * static_cast<int64_t>(ns) * nc + k * static_cast<int64_t>(nst) * D;
  const int* sid = stencils + k * nst;
  const bool use_rn = row_normals != nullptr;
  double rn[D];
  for (int a = 0; a < D; ++a) rn[a] = use_rn ? row_normals[k * D + a] : 0.0;
  double c[D];
  load_point<D>(pos, sid[0], c);
  double scale = 0.0;
  for (int j = 0; j < nst; ++j) {
    double p[D];
    load_point<D>(pos, sid[j], p);
    for (int a = 0; a < D; ++a) Y[j * D + a] = __dsub_rn(p[a], c[a]);
    scale = fmax(scale, norm_rn<D>(Y + j * D));
  }
  for (int j = 0; j < nst * D; ++j) Y[j] = __ddiv_rn(Y[j], scale);
  for (int i = 0; i < nst; ++i) {
    for (int j = 0; j < nst; ++j) {
      double d2 = 0.0;
      for (int q = 0; q < D; ++q) {
        double t = Y[i * D + q] - Y[j * D + q];
        d2 = fma(t, t, d2);
      }
      double rr = sqrt(d2);
      A[i * nc + j] = rr * rr * rr;
    }
    for (int m = 0; m < NQ; ++m) A[i * nc + nst + m] = mono_val<D>(m, Y + i * D);
    double r0 = norm_rn<D>(Y + i * D);
    for (int o = 0; o < nops; ++o) A[i * nc + ns + o] = phs_rhs<D>(ops, o, Y + i * D, r0, use_rn, rn);
  }
  for (int m = 0; m < NQ; ++m) {
    const int i = nst + m;
    for (int j = 0; j < nst; ++j) A[i * nc + j] = mono_val<D>(m, Y + j * D);
    for (int j = nst; j < ns; ++j) A[i * nc + j] = 0.0;
    for (int o = 0; o < nops; ++o) A[i * nc + ns + o] = poly_rhs<D>(ops, o, m, use_rn, rn);
  }
  int sing = 0;
  for (int kk = 0; kk < ns; ++kk) {
    int p = kk;
    double best = fabs(A[kk * nc + kk]);
    for (int i = kk + 1; i < ns; ++i) {
      double v = fabs(A[i * nc + kk]);
      if (v > best) { best = v; p = i; }
    }
    if (p != kk)
      for (int j = 0; j < nc; ++j) {
        double t = A[kk * nc + j];
        A[kk * nc + j] = A[p * nc + j];
        A[p * nc + j] = t;
      }
    const double piv = A[kk * nc + kk];
    if (piv == 0.0 && sing == 0) sing = kk + 1;
    const double inv = 1.0 / piv;
    for (int i = kk + 1; i < ns; ++i) {
      const double l = A[i * nc + kk] * inv;
      for (int j = kk + 1; j < nc; ++j) A[i * nc + j] = fma(-l, A[kk * nc + j], A[i * nc + j]);
    }
  }
  for (int o = 0; o < nops; ++o)
    for (int i = ns - 1; i >= 0; --i) {
      double s = A[i * nc + ns + o];
      for (int j = i + 1; j < ns; ++j) s = fma(-A[i * nc + j], A[j * nc + ns + o], s);
      A[i * nc + ns + o] = s / A[i * nc + i];
    }
  if (info) info[k] = sing;
  const double s1 = 1.0 / scale, s2 = s1 * s1;
  for (int j = 0; j < nst; ++j) {
    int rank = 0;
    for (int i = 0; i < nst; ++i) rank += (sid[i] < sid[j]) || (sid[i] == sid[j] && i < j);
    out_idx[static_cast<int64_t>(rank) * K + k] = sid[j];
    for (int o = 0; o < nops; ++o)
      out_w[(static_cast<int64_t>(o) * nst + rank) * K + k] = A[j * nc + ns + o] * (ops.order[o] == 2 ? s2 : s1);
  }
}

}  // namespace hn

using namespace hn;

static bool make_ops(int nops, const int* kind, const int* axis, const double* normal, int d, OpSpec* o) {
  if (nops < 1 || nops > 4) return false;
  *o = OpSpec{};
  o->nops = nops;
  for (int i = 0; i < nops; ++i) {
    o->kind[i] = kind[i];
    o->axis[i] = axis ? axis[i] : 0;
    o->order[i] = kind[i] == kOpLaplacian ? 2 : 1;
    for (int a = 0; a < d; ++a) o->normal[i][a] = normal ? normal[i * d + a] : 0.0;
  }
  return true;
}

HN_EXPORT int hn_weights_mon(const double* pos, int d, const int* stencils, int64_t K, int nops,
                             const int* op_kind_host, const int* op_axis_host, const double* op_normal_host,
                             int* out_idx, double* out_w, int* info, void* stream) {
  OpSpec ops;
  if (d != 2 && d != 3) return 1;
  if (!make_ops(nops, op_kind_host, op_axis_host, op_normal_host, d, &ops)) return 2;
  if (K == 0) return 0;
  cudaStream_t s = as_stream(stream);
  const int th = 128;
  const int64_t bl = ceil_div(K, th);
  int* flag = nullptr;
  HN_TRY(stream_alloc(reinterpret_cast<void**>(&flag), sizeof(int) * K, s));
#define HN_MON(DD, NO)                                                                                  \
  do {                                                                                                  \
    mon_weights_kernel<DD, NO><<<bl, th, 0, s>>>(pos, stencils, K, ops, out_idx, out_w, info, flag);    \
    mon_general_kernel<DD, NO><<<bl, th, 0, s>>>(pos, stencils, K, ops, out_idx, out_w, info, flag);    \
  } while (0)
  if (d == 2) {
    switch (nops) { case 1: HN_MON(2, 1); break; case 2: HN_MON(2, 2); break; case 3: HN_MON(2, 3); break; default: HN_MON(2, 4); }
  } else {
    switch (nops) { case 1: HN_MON(3, 1); break; case 2: HN_MON(3, 2); break; case 3: HN_MON(3, 3); break; default: HN_MON(3, 4); }
  }
#undef HN_MON
  cudaFreeAsync(flag, s);
  HN_CHECK_LAUNCH();
  return 0;
}

template <int D, int NST, int NOPS, int LPS, int RPL, int WARPS, int MINB>
static void launch_rbf_v(const double* pos, const int* st, int64_t K, const OpSpec& ops, const double* rn, int* oi,
                         double* ow, int* info, cudaStream_t s) {
  constexpr int SPW = 32 / LPS;
  const int64_t per_block = static_cast<int64_t>(WARPS) * SPW;
  rbf_weights_kernel<D, NST, NOPS, LPS, RPL, WARPS, MINB><<<ceil_div(K, per_block), WARPS * 32, 0, s>>>(
      pos, st, K, ops, rn, oi, ow, info);
}

// launch-shape variant for the 2D n=12 kernel (tuning experiments; 0 = default)
static int g_rbf_variant = 0;
HN_EXPORT void hn_weights_rbf_set_variant(int v) { g_rbf_variant = v; }

template <int D, int NST, int NOPS, int LPS, int RPL>
static void launch_rbf(const double* pos, const int* st, int64_t K, const OpSpec& ops, const double* rn, int* oi,
                       double* ow, int* info, cudaStream_t s) {
  if constexpr (D == 2 && NST == 12) {
    switch (g_rbf_variant) {
      case 1: launch_rbf_v<2, 12, NOPS, 6, 3, 4, 1>(pos, st, K, ops, rn, oi, ow, info, s); return;
      case 2: launch_rbf_v<2, 12, NOPS, 9, 2, 4, 1>(pos, st, K, ops, rn, oi, ow, info, s); return;
      case 3: launch_rbf_v<2, 12, NOPS, 9, 2, 4, 4>(pos, st, K, ops, rn, oi, ow, info, s); return;
      case 4: launch_rbf_v<2, 12, NOPS, 6, 3, 2, 5>(pos, st, K, ops, rn, oi, ow, info, s); return;
      case 5: launch_rbf_v<2, 12, NOPS, 6, 3, 1, 12>(pos, st, K, ops, rn, oi, ow, info, s); return;
      default: launch_rbf_v<2, 12, NOPS, 6, 3, 4, 3>(pos, st, K, ops, rn, oi, ow, info, s); return;
    }
  }
  launch_rbf_v<D, NST, NOPS, LPS, RPL, 4, 1>(pos, st, K, ops, rn, oi, ow, info, s);
}

// Workspace (doubles) the generic path needs for K stencils of size n: K*(ns*nc + n*d).
HN_EXPORT int64_t hn_weights_rbf_workspace(int d, int n, int nops, int64_t K) {
  const int ns = n + (d == 2 ? 6 : 10);
  return K * (static_cast<int64_t>(ns) * (ns + nops) + static_cast<int64_t>(n) * d);
}

// Returns 0 when a tuned kernel exists for (d, n, nops), 1 when the generic path (and its workspace) is needed.
HN_EXPORT int hn_weights_rbf_is_tuned(int d, int n, int nops) {
  if (nops < 1 || nops > 4) return 1;
  if (d == 2 && n == 12) return 0;
  if (d == 3 && (n == 20 || n == 30)) return 0;
  return 1;
}

HN_EXPORT int hn_weights_rbf(const double* pos, int d, const int* stencils, int64_t K, int n, int nops,
                             const int* op_kind_host, const int* op_axis_host, const double* op_normal_host,
                             const double* row_normals, double* workspace, int* out_idx, double* out_w, int* info,
                             void* stream) {
  OpSpec ops;
  if (d != 2 && d != 3) return 1;
  if (!make_ops(nops, op_kind_host, op_axis_host, op_normal_host, d, &ops)) return 2;
  if (K == 0) return 0;
  cudaStream_t s = as_stream(stream);
  if (hn_weights_rbf_is_tuned(d, n, nops) == 0) {
    if (d == 2) {
      switch (nops) {
        case 1: launch_rbf<2, 12, 1, 6, 3>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s); break;
        case 2: launch_rbf<2, 12, 2, 6, 3>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s); break;
        case 3: launch_rbf<2, 12, 3, 6, 3>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s); break;
        default: launch_rbf<2, 12, 4, 6, 3>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s); break;
      }
    } else if (n == 20) {
      switch (nops) {
        case 1: launch_rbf<3, 20, 1, 15, 2>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s); break;
        case 2: launch_rbf<3, 20, 2, 15, 2>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s); break;
        case 3: launch_rbf<3, 20, 3, 15, 2>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s); break;
        default: launch_rbf<3, 20, 4, 15, 2>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s); break;
      }
    } else {
      switch (nops) {
        case 1: launch_rbf<3, 30, 1, 20, 2>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s); break;
        case 2: launch_rbf<3, 30, 2, 20, 2>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s); break;
        case 3: launch_rbf<3, 30, 3, 20, 2>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s); break;
        default: launch_rbf<3, 30, 4, 20, 2>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s); break;
      }
    }
  } else {
    if (!workspace) return 3;
    const int th = 64;
    if (d == 2)
      rbf_weights_generic_kernel<2><<<ceil_div(K, th), th, 0, s>>>(pos, stencils, K, n, ops, row_normals, workspace,
                                                                   out_idx, out_w, info);
    else
      rbf_weights_generic_kernel<3><<<ceil_div(K, th), th, 0, s>>>(pos, stencils, K, n, ops, row_normals, workspace,
                                                                   out_idx, out_w, info);
  }
  HN_CHECK_LAUNCH();
  return 0;
}
