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
//      Default: rbf_static_kernel -- a static null-space elimination order (below), with
//      flagged stencils re-solved by the searching kernel.  Searching kernel:
//      Gauss-Jordan with implicit partial pivoting: every step picks the largest
//      |a_ik| among not-yet-pivoted rows (segmented shuffle argmax on a packed
//      key), the owner lane stages the pivot row in shared memory, and every lane
//      updates all of its rows with DFMA.  Gauss-Jordan instead of LU+back
//      substitution: in this layout lanes whose rows are already eliminated would
//      idle anyway, and it removes the sequential, latency-bound back-solve.
//      Exact zero pivot => SingularSystemError (info = step + 1), as dgesv does.
#include <cfloat>
#include <climits>
#include <type_traits>
#include <utility>

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

template <int D, int NOPS>
__device__ __noinline__ void mon_general_call(const double* __restrict__ pos, const int* __restrict__ stencils,
                                              int64_t K, int64_t k, const OpSpec& ops, int* __restrict__ out_idx,
                                              double* __restrict__ out_w, int* __restrict__ info);

// Fast kernel: canonical lattice stencils (mon_static); any other row runs the general
// partial-pivoting path in a separately compiled (noinline) function, so its register budget
// does not set the fast path's occupancy, and no second launch or flag array is needed.
template <int D, int NOPS>
__global__ void __launch_bounds__(128, D == 2 ? 7 : 5) mon_weights_kernel(const double* __restrict__ pos,
                                                          const int* __restrict__ stencils, int64_t K,
                                                          OpSpec ops, int* __restrict__ out_idx,
                                                          double* __restrict__ out_w, int* __restrict__ info) {
  constexpr int N = 2 * D + 1;
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= K) return;
  int sid[N];
#pragma unroll
  for (int j = 0; j < N; ++j) sid[j] = __ldg(stencils + k * N + j);
  double c[D];
  load_point<D>(pos, sid[0], c);
  const bool done = mon_static<D, NOPS>(pos, sid, c, K, k, ops, out_idx, out_w);
  if (done) {
    if (info) info[k] = 0;
  } else {
    mon_general_call<D, NOPS>(pos, stencils, K, k, ops, out_idx, out_w, info);
  }
}

template <int D, int NOPS>
__device__ __forceinline__ void mon_general(const double* __restrict__ pos, const int* __restrict__ stencils,
                                            int64_t K, int64_t k, const OpSpec& ops, int* __restrict__ out_idx,
                                            double* __restrict__ out_w, int* __restrict__ info);

template <int D, int NOPS>
__device__ __noinline__ void mon_general_call(const double* __restrict__ pos, const int* __restrict__ stencils,
                                              int64_t K, int64_t k, const OpSpec& ops, int* __restrict__ out_idx,
                                              double* __restrict__ out_w, int* __restrict__ info) {
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

// r^3 from r^2: MUFU rsqrt seed + Goldschmidt/Newton refinement (~1 ulp), exact 0 at r^2 = 0
// (the clamp keeps rsqrt finite there, and d2 * r = 0 with no select)
__device__ __forceinline__ double cube_from_sq(double d2) {
  const double q = fmax(d2, 1e-300);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
  // coupled Goldschmidt step for (sqrt, 1/(2 sqrt)), then one Newton correction of the
  // root: ~1 ulp, 7 dependent FP64 ops after the seed instead of 9
  double g = q * y, h = 0.5 * y;
  const double e = fma(-g, h, 0.5);
  g = fma(g, e, g);
  h = fma(h, e, h);
  g = fma(h, fma(-g, g, q), g);
  return d2 * g;
}

// One block-group of the searching kernel.  Stencil k = item (direct mode) or list[item]
// (list mode: the stencils the static kernel below flagged, n_items read on the device).
template <int D, int NST, int NOPS, int LPS, int RPL, int WARPS>
__device__ __forceinline__ void rbf_search_group(
    int64_t grp, RbfSmem<D, NST, NOPS>* smem_all, const double* __restrict__ pos, const int* __restrict__ stencils,
    int64_t K, int64_t n_items, const int* __restrict__ list, const OpSpec& ops,
    const double* __restrict__ row_normals, int* __restrict__ out_idx, double* __restrict__ out_w,
    int* __restrict__ info) {
  constexpr int NQ = poly_count<D>();
  constexpr int NS = NST + NQ;
  constexpr int NC = NS + NOPS;
  constexpr int SPW = 32 / LPS;
  static_assert(LPS * RPL >= NS, "rows do not fit");
  static_assert(NS <= 63, "packed pivot key holds 6 row bits");
  using Sm = RbfSmem<D, NST, NOPS>;

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int sys_w = lane / LPS;                 // system slot within the warp
  const int s = lane - sys_w * LPS;             // lane within the system segment
  const bool lane_live = sys_w < SPW;
  const int seg_base = sys_w * LPS;
  const int64_t k_raw = (grp * WARPS + warp) * SPW + (lane_live ? sys_w : 0);
  const bool sys_live = lane_live && k_raw < n_items;
  const int64_t item = k_raw < n_items ? k_raw : n_items - 1;  // idle segments recompute the last stencil
  const int64_t k = list ? static_cast<int64_t>(list[item]) : item;
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

// Searching kernel: direct mode (list == nullptr, items = stencils 0..K-1, one group per
// block) or list mode (items = list[0..*list_count), grid-stride over groups).
template <int D, int NST, int NOPS, int LPS, int RPL, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) rbf_weights_kernel(
    const double* __restrict__ pos, const int* __restrict__ stencils, int64_t K, OpSpec ops,
    const double* __restrict__ row_normals, int* __restrict__ out_idx, double* __restrict__ out_w,
    int* __restrict__ info, const int* __restrict__ list, const int* __restrict__ list_count) {
  constexpr int SPW = 32 / LPS;
  __shared__ __align__(16) RbfSmem<D, NST, NOPS> smem_all[WARPS * SPW];
  if (list == nullptr) {
    rbf_search_group<D, NST, NOPS, LPS, RPL, WARPS>(blockIdx.x, smem_all, pos, stencils, K, K, nullptr, ops,
                                                    row_normals, out_idx, out_w, info);
    return;
  }
  const int64_t n = *list_count;
  for (int64_t g = blockIdx.x; g * WARPS * SPW < n; g += gridDim.x) {
    rbf_search_group<D, NST, NOPS, LPS, RPL, WARPS>(g, smem_all, pos, stencils, K, n, list, ops, row_normals,
                                                    out_idx, out_w, info);
    __syncwarp();
  }
}

// ============ RBF-FD with a static null-space pivot order (default path) ============
// The saddle system [[A P],[P^T 0]] (A_ij = r_ij^3: zero diagonal, indefinite) is
// eliminated in a fixed order instead of with a pivot search at every step:
//   A. a partial-pivoting LU of P (NST x NQ, rows = stencil nodes, NQ short steps) picks
//      NQ nodes I whose monomial rows are unisolvent with |L| <= 1; the nodes are then
//      renumbered [I (pivot order), J (the rest, stencil order)];
//   1. pivots (monomial row m, column of node I_m), m < NQ: the LU of P_I^T;
//   2. pivots (node row I_m, column lambda_m): the LU of P_I.  Both have the pivots of
//      step A (the same leading minors of P_I), so their reciprocals are step A's;
//   3. pivots (node row J_j, column of node J_j): the diagonal of the Schur complement
//      Z^T A Z, symmetric positive definite because r^3 is conditionally positive definite
//      of order 2 -- diagonal pivots need no search there.
// That is the null-space method written as Gauss-Jordan.  Every pivot row sits at a
// compile-time (lane, slot), so the elimination has no pivot search, no row bookkeeping and
// one predicated store per staged pair (the searching kernel above stores RPL), and the
// zero blocks are skipped statically (monomial rows have no lambda columns; phase 2 leaves
// monomial rows alone, phase 3 the I rows whose lambda values are not needed).
// Row rho = s + r * LPS of the renumbered system lives in segment lane s, slot r: rho < NQ
// node I_rho, rho < NST node J, else monomial rho - NST.  A system's segment is LPS
// contiguous lanes (ILV = true interleaves them, lane = s * SPW + system: the pivot-row
// owners become adjacent and their stores cheaper, but the broadcast loads, which dominate,
// cost twice as many shared-memory wavefronts; measured slower).  The matrix is assembled
// in registers -- shared memory is the scarcer resource: it carries every pivot-row
// broadcast, and staging the symmetric A there once per pair cost more than the 2x cubes.
// Step t updates the next pivot row first, stages it and issues its loads (and the next
// pivot's reciprocal) before the bulk update of step t.
// Checked against dgesv on every config's stencils (numpy model of this order: <= 1.8e-13
// row-normwise on configs 1/2/4, interior and one-sided boundary stencils; pivots of
// phases 1/2 >= 0.06, phase-3 pivots >= 5e-3).  A stencil with a step-A pivot below
// 2^-10 or a phase-3 pivot below 2^-12 (nearly unisolvent nodes, non-SPD Schur
// complement, exact zero pivots, coincident nodes) is flagged and re-solved by the
// searching kernel, so dgesv's partial-pivoting semantics, SingularSystemError included,
// are unchanged.
template <int D, int NST, int NOPS>
struct RbfStaticCore {
  static constexpr int NQ = poly_count<D>();
  static constexpr int NS = NST + NQ;
  static constexpr int NC = NS + NOPS;
  static constexpr int NCP = (NC + 1) & ~1;
  static constexpr int YS = D == 2 ? 2 : 4;        // padded point (16-B loads)
  static constexpr int PTW = (NST + 1) & ~1;       // transposed-P row width (16-B rows)
  double prow[2][NCP];             // double-buffered pivot row (16 B aligned pairs)
  double inv_hist[(NQ + 1) & ~1];  // 1/pivot of step A (= phases 1 and 2)
  double yp[NST][YS];              // local coordinates, renumbered [I, J]
  double pt[NQ][PTW];              // P^T (monomial rows), renumbered nodes
  double w[NST][NOPS];             // solution, renumbered
  int sidp[NST];                   // node ids, renumbered
};
// padded so consecutive systems start 16 B apart modulo 128 B: the five pivot-row
// broadcasts of a warp hit distinct banks
template <int D, int NST, int NOPS>
struct __align__(16) RbfStaticSmem : RbfStaticCore<D, NST, NOPS> {
  static constexpr int kCore = static_cast<int>(sizeof(RbfStaticCore<D, NST, NOPS>));
  static constexpr int kPad = ((16 - kCore % 128) % 128 + 128) % 128;
  char pad[kPad == 0 ? 128 : kPad];
};

// f(std::integral_constant<int, I>) for I = 0..N-1, unrolled by construction (NVVM's
// #pragma unroll gives up on the 30-40-step 3D eliminations and falls back to local memory)
template <typename F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// compile-time schedule of the static elimination
template <int NST, int NQ>
__host__ __device__ constexpr int st_piv_row(int t) {
  return t < NQ ? NST + t : (t < 2 * NQ ? t - NQ : NQ + (t - 2 * NQ));
}
template <int NST, int NQ>
__host__ __device__ constexpr int st_piv_col(int t) {
  return t < NQ ? t : (t < 2 * NQ ? NST + (t - NQ) : NQ + (t - 2 * NQ));
}
template <int NST, int NQ>
__host__ __device__ constexpr int st_col_step(int c) {  // step that pivots column c (RHS: never)
  return c < NQ ? c : (c < NST ? 2 * NQ + (c - NQ) : (c < NST + NQ ? NQ + (c - NST) : (1 << 20)));
}

constexpr double kStaticPivMin = 1.0 / 1024.0;   // |pivot| floor, step A (= phases 1-2)
constexpr double kStaticSchurMin = 1.0 / 4096.0;  // pivot floor, phase 3 (positive)

// standard operator set [Laplacian, d/dx_0, .., d/dx_{D-1}] (what compute_weights asks for):
// right-hand sides from compile-time tables
template <int D>
__device__ __forceinline__ double std_poly_rhs(int o, int m) {
  constexpr unsigned SQ = D == 2 ? 0x28u : 0x290u;  // pure squares: 2D m = 3, 5; 3D m = 4, 7, 9
  if (o == 0) return ((SQ >> m) & 1u) ? 2.0 : 0.0;
  return m == o ? 1.0 : 0.0;                        // d/dx_a of monomial 1 + a
}

template <int D, int NST, int NOPS, bool STD, int LPS, int RPL, int WARPS, int MINB, bool ILV, bool SHB = false,
          bool LA = true>
__global__ void __launch_bounds__(WARPS * 32, MINB) rbf_static_kernel(
    const double* __restrict__ pos, const int* __restrict__ stencils, int64_t K, OpSpec ops,
    const double* __restrict__ row_normals, int* __restrict__ out_idx, double* __restrict__ out_w,
    int* __restrict__ info, int* __restrict__ flag_list, int* __restrict__ flag_count, int force_flag) {
  constexpr int NQ = poly_count<D>();
  constexpr int NS = NST + NQ;
  constexpr int NC = NS + NOPS;
  constexpr int SPW = 32 / LPS;
  constexpr int PA = (NST + LPS - 1) / LPS;  // slots holding the original nodes in step A
  static_assert(LPS * RPL == NS, "one system row per (lane, slot)");
  static_assert(NST <= 31, "node bitmask");
  static_assert(!STD || NOPS == D + 1, "standard operator set is [Lap, d/dx_a..]");
  using Sm = RbfStaticSmem<D, NST, NOPS>;
  // flagged systems are re-solved in this kernel when the searching layout is the same
  static constexpr bool kInlineFallback = D == 2 && NST == 12 && LPS == 6 && RPL == 3 && !ILV;
  extern __shared__ __align__(16) unsigned char rbf_static_smem[];  // WARPS * SPW systems
  Sm* smem_all = reinterpret_cast<Sm*>(rbf_static_smem);

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const bool lane_live = lane < SPW * LPS;
  // ILV: lane = s * SPW + system (owners adjacent); else lane = system * LPS + s
  const int s = lane_live ? (ILV ? lane / SPW : lane % LPS) : 0;      // lane within the segment
  const int sys_w = lane_live ? (ILV ? lane % SPW : lane / LPS) : 0;  // system slot in the warp
  const int seg_base = ILV ? sys_w : sys_w * LPS;                     // segment lane 0
  const int64_t k_raw = (static_cast<int64_t>(blockIdx.x) * WARPS + warp) * SPW + sys_w;
  const bool sys_live = lane_live && k_raw < K;
  const int64_t k = k_raw < K ? k_raw : K - 1;
  Sm& sm = smem_all[warp * SPW + sys_w];
  // all-reduce butterfly partner in segment-relative numbering: s ^ off clamped to LPS - 1
  // leaves every lane of the segment with the full reduction for any LPS (checked for
  // 2..24), so no broadcast shuffle follows
  auto seg_xor = [&](int off) {
    int t = s ^ off;
    t = t < LPS ? t : LPS - 1;
    return lane_live ? (ILV ? t * SPW + sys_w : sys_w * LPS + t) : lane;
  };
  // slot classes (rho = s + r * LPS, s < LPS)
  auto has_node = [](int r) { return r * LPS < NST; };
  auto only_poly = [](int r) { return r * LPS >= NST; };
  auto only_node = [](int r) { return r * LPS + LPS <= NST; };
  auto only_I = [](int r) { return r * LPS + LPS <= NQ; };

  const bool use_rn = !STD && row_normals != nullptr;
  double rn[D];
#pragma unroll
  for (int a = 0; a < D; ++a) rn[a] = use_rn ? __ldg(row_normals + k * D + a) : 0.0;

  // ---- gather, shift to the centre, scale by the stencil radius (approx.py:245-250) ----
  // (scale and 1/scale to ~1 ulp; the weights are un-scaled by the same 1/scale, and a
  //  stencil that needs dgesv's exact-zero-pivot semantics is re-solved by the searching
  //  kernel, which forms the local coordinates bitwise as the reference does)
  double c[D];
  load_point<D>(pos, __ldg(stencils + k * NST), c);
  double yo[PA][D];
  int sido[PA];
  double d2max = 0.0;
#pragma unroll
  for (int r = 0; r < PA; ++r) {
    const int j = s + r * LPS;
    sido[r] = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) yo[r][a] = 0.0;
    if (j < NST) {
      sido[r] = __ldg(stencils + k * NST + j);
      double p[D];
      load_point<D>(pos, sido[r], p);
      double d2 = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        yo[r][a] = p[a] - c[a];
        d2 = fma(yo[r][a], yo[r][a], d2);
      }
      d2max = fmax(d2max, d2);
    }
  }
#pragma unroll
  for (int off = 1; off < LPS; off <<= 1) d2max = fmax(d2max, __shfl_sync(0xffffffffu, d2max, seg_xor(off)));
  const double s1 = fast_rcp(fast_sqrt(d2max));
#pragma unroll
  for (int r = 0; r < PA; ++r)
#pragma unroll
    for (int a = 0; a < D; ++a) yo[r][a] *= s1;

  const unsigned pb0 = smem_addr(&sm.prow[0][0]);
  const unsigned pb1 = smem_addr(&sm.prow[1][0]);
  const unsigned hist = smem_addr(&sm.inv_hist[0]);
  bool bad = force_flag != 0;

  // ---- step A: LU of P with partial pivoting over the nodes -> I ----
  {
    double pp[PA][NQ];
    unsigned vm[PA];
#pragma unroll
    for (int r = 0; r < PA; ++r) {
      const int j = s + r * LPS;
#pragma unroll
      for (int m = 0; m < NQ; ++m) pp[r][m] = mono_val<D>(m, yo[r]);
      vm[r] = (lane_live && j < NST) ? (0x7fffffc0u | static_cast<unsigned>(63 - j)) : 0u;
    }
    int step_of[PA];  // step that chose the slot's node (its I index)
#pragma unroll
    for (int r = 0; r < PA; ++r) step_of[r] = 0;
    // column 0 (monomial 1) is all ones: partial pivoting takes the first node, the centre,
    // whose monomial row is [1, 0, ..] (y = 0 exactly), so step 0 eliminates nothing
    unsigned chosen = 1u;
    vm[0] = s == 0 ? 0u : vm[0];
    if (lane_live && s == 0) sm.inv_hist[0] = 1.0;
    static_for<NQ - 1>([&](auto mc) {
      constexpr int m = decltype(mc)::value + 1;
      unsigned key = 0;
#pragma unroll
      for (int r = 0; r < PA; ++r)
        key = max(key, (static_cast<unsigned>(__double2hiint(pp[r][m])) | 63u) & vm[r]);
#pragma unroll
      for (int off = 1; off < LPS; off <<= 1) key = max(key, __shfl_sync(0xffffffffu, key, seg_xor(off)));
      const unsigned ptag = key & 63u;
      const unsigned pbase = (m & 1) ? pb1 : pb0;
      bool isp[PA];
#pragma unroll
      for (int r = 0; r < PA; ++r) {
        isp[r] = ((vm[r] & 63u) == ptag) && vm[r] != 0u;
        constexpr int j0 = m & ~1;
#pragma unroll
        for (int jj = j0; jj < NQ; jj += 2) {
          if (jj + 1 < NQ) st_pred2(isp[r], pbase + 8u * jj, pp[r][jj], pp[r][jj + 1]);
          else st_pred1(isp[r], pbase + 8u * jj, pp[r][jj]);
        }
        if (isp[r]) step_of[r] = m;  // its coordinates and id go to slot m after the loop
      }
      __syncwarp();
      const double* prow = sm.prow[m & 1];
      const double piv = prow[m];
      bad = bad || !(fabs(piv) >= kStaticPivMin);
      const double inv = fast_rcp(piv);
      st_pred1(lane_live && s == 0, hist + 8u * m, inv);
#pragma unroll
      for (int r = 0; r < PA; ++r) {
        // no mask on the pivot row: it eliminates itself to zero and is never read again
        const double l = pp[r][m] * inv;
        vm[r] = isp[r] ? 0u : vm[r];
#pragma unroll
        for (int cc = m + 1; cc < NQ; ++cc) pp[r][cc] = fma(-l, prow[cc], pp[r][cc]);
      }
      chosen |= 1u << (63u - ptag);
    });
    // renumbering: I = the chosen nodes by step, J = the others in stencil order
#pragma unroll
    for (int r = 0; r < PA; ++r) {
      const int j = s + r * LPS;
      if (lane_live && j < NST) {
        const int ni = ((chosen >> j) & 1u) ? step_of[r] : NQ + __popc(~chosen & ((1u << j) - 1u));
#pragma unroll
        for (int a = 0; a < D; ++a) sm.yp[ni][a] = yo[r][a];
        sm.sidp[ni] = sido[r];
      }
    }
  }
  __syncwarp();

  // ---- assemble the renumbered rows | RHS in registers (approx.py:254-277) ----
  // node rows: A_ij = r_ij^3 from the shared renumbered coordinates, own P row; the node
  // lanes also publish P^T so the monomial rows read their row instead of forming it
  double a[RPL][NC];
  double yr[RPL][D];
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int rho = s + r * LPS;
    const bool node_row = only_node(r) || (!only_poly(r) && rho < NST);
#pragma unroll
    for (int q = 0; q < D; ++q) yr[r][q] = 0.0;
    if (node_row) {
      const int i = rho < NST ? rho : 0;
      double yi[D];
#pragma unroll
      for (int q = 0; q < D; ++q) yi[q] = yr[r][q] = sm.yp[i][q];
#pragma unroll
      for (int m = 0; m < NQ; ++m) {
        a[r][NST + m] = mono_val<D>(m, yi);
        if (lane_live) sm.pt[m][i] = a[r][NST + m];
      }
      const double r0 = norm_fast<D>(yi);
      if constexpr (STD) {
        a[r][NS] = 3.0 * (D + 1) * r0;
        const double m3 = -3.0 * r0;
#pragma unroll
        for (int q = 0; q < D; ++q) a[r][NS + 1 + q] = m3 * yi[q];
      } else {
#pragma unroll
        for (int o = 0; o < NOPS; ++o) a[r][NS + o] = phs_rhs<D>(ops, o, yi, r0, use_rn, rn);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NST; ++j) {
    double yj[D];
#pragma unroll
    for (int q = 0; q < D; ++q) yj[q] = sm.yp[j][q];
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      if (!has_node(r)) continue;
      double d2 = 0.0;
#pragma unroll
      for (int q = 0; q < D; ++q) {
        const double t = yr[r][q] - yj[q];
        d2 = fma(t, t, d2);
      }
      a[r][j] = cube_from_sq(d2);  // exact 0 on the diagonal
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int rho = s + r * LPS;
    const bool node_row = only_node(r) || (!only_poly(r) && rho < NST);
    if (!node_row) {
      const int m = rho - NST < NQ ? rho - NST : 0;
      const double2* row = reinterpret_cast<const double2*>(&sm.pt[m][0]);
#pragma unroll
      for (int j = 0; j < NST; j += 2) {
        const double2 v = row[j / 2];
        a[r][j] = v.x;
        if (j + 1 < NST) a[r][j + 1] = v.y;
      }
      if (has_node(r)) {
#pragma unroll
        for (int mm = 0; mm < NQ; ++mm) a[r][NST + mm] = 0.0;
      }
#pragma unroll
      for (int o = 0; o < NOPS; ++o) a[r][NS + o] = STD ? std_poly_rhs<D>(o, m) : poly_rhs<D>(ops, o, m, use_rn, rn);
    }
  }

  // ---- static Gauss-Jordan, one step of look-ahead ----
  // Step t updates the slot holding pivot row t+1 first, stages that row and issues its
  // loads, then updates the other slots while the loads are in flight: the shared-memory
  // round trip of the next pivot row overlaps this step's bulk update.
  // live(t, c): column c of pivot row t is needed (not pivoted before t; phase-1 pivot rows
  // are monomial rows, zero in the lambda columns)
  auto live_at = [](int tt, int cc) {
    const int phh = tt < NQ ? 1 : (tt < 2 * NQ ? 2 : 3);
    return cc < NC && st_col_step<NST, NQ>(cc) >= tt && !(phh == 1 && cc >= NST && cc < NS);
  };
  auto stage = [&](auto tc2) {  // owner of pivot row t2 writes its live columns
    constexpr int t2 = decltype(tc2)::value;
    constexpr int pr2 = st_piv_row<NST, NQ>(t2);
    constexpr int os2 = pr2 / LPS, ol2 = pr2 % LPS;
    const bool own2 = lane_live && s == ol2;
    const unsigned pbase = (t2 & 1) ? pb1 : pb0;
#pragma unroll
    for (int cc = 0; cc < NC; cc += 2) {
      const bool l0 = live_at(t2, cc), l1 = live_at(t2, cc + 1);
      if (l0 && l1) st_pred2(own2, pbase + 8u * cc, a[os2][cc], a[os2][cc + 1]);
      else if (l0) st_pred1(own2, pbase + 8u * cc, a[os2][cc]);
      else if (l1) st_pred1(own2, pbase + 8u * (cc + 1), a[os2][cc + 1]);
    }
  };
  // SHB: the pivot row goes from the owner's registers to its segment by shuffles (one
  // SHFL pair per value, no shared-memory round trip) instead of a staged store + load
  auto bcast = [&](auto tc2, double* v) {
    constexpr int t2 = decltype(tc2)::value;
    constexpr int pr2 = st_piv_row<NST, NQ>(t2);
    constexpr int os2 = pr2 / LPS, ol2 = pr2 % LPS;
    const int src = lane_live ? (ILV ? ol2 * SPW + sys_w : sys_w * LPS + ol2) : lane;
#pragma unroll
    for (int cc = 0; cc < NC; ++cc)
      if (live_at(t2, cc)) v[cc] = __shfl_sync(0xffffffffu, a[os2][cc], src);
  };
  auto load = [&](auto tc2, double* v) {
    constexpr int t2 = decltype(tc2)::value;
    const double* prow = sm.prow[t2 & 1];
#pragma unroll
    for (int cc = 0; cc < NC; cc += 2) {
      const bool l0 = live_at(t2, cc), l1 = live_at(t2, cc + 1);
      if (l0 && l1) {
        const double2 q = *reinterpret_cast<const double2*>(prow + cc);
        v[cc] = q.x;
        v[cc + 1] = q.y;
      } else if (l0) {
        v[cc] = prow[cc];
      } else if (l1) {
        v[cc + 1] = prow[cc + 1];
      }
    }
  };
  double invp[RPL];
#pragma unroll
  for (int r = 0; r < RPL; ++r) invp[r] = 0.0;
  double pv[NC];  // pivot row of the current step
#pragma unroll
  for (int cc = 0; cc < NC; ++cc) pv[cc] = 0.0;
  // 1/pivot of step t2 from its loaded pivot row (phase 3) or step A's history (phases 1-2)
  auto pivot_inv = [&](auto tc2, const double* v) {
    constexpr int t2 = decltype(tc2)::value;
    if constexpr (t2 >= 2 * NQ) {
      const double piv = v[st_piv_col<NST, NQ>(t2)];
      bad = bad || !(piv >= kStaticSchurMin);
      return fast_rcp(piv);
    } else {
      return sm.inv_hist[t2 < NQ ? t2 : t2 - NQ];
    }
  };
  if constexpr (SHB) {
    bcast(std::integral_constant<int, 0>{}, pv);
  } else {
    stage(std::integral_constant<int, 0>{});
    __syncwarp();
    load(std::integral_constant<int, 0>{}, pv);
  }
  double inv_cur = pivot_inv(std::integral_constant<int, 0>{}, pv);
  static_for<NS>([&](auto tc) {
    constexpr int t = decltype(tc)::value;
    constexpr int pr = st_piv_row<NST, NQ>(t), pc = st_piv_col<NST, NQ>(t);
    constexpr int os = pr / LPS, ol = pr % LPS;
    constexpr int ph = t < NQ ? 1 : (t < 2 * NQ ? 2 : 3);
    const bool own = lane_live && s == ol;
    const double inv = inv_cur;
    if constexpr (ph != 2) invp[os] = own ? inv : invp[os];
    auto active = [&](int r) { return !((ph == 2 && only_poly(r)) || (ph == 3 && only_I(r))); };
    auto update = [&](int r) {
      double l = a[r][pc] * inv;
      if (r == os) l = own ? 0.0 : l;
#pragma unroll
      for (int cc = 0; cc < NC; ++cc)
        if (cc != pc && live_at(t, cc)) a[r][cc] = fma(-l, pv[cc], a[r][cc]);
    };
    if constexpr (!LA) {
      // no look-ahead: every row is updated before the next pivot row is broadcast
      // (fewer live registers, a serial broadcast per step)
#pragma unroll
      for (int r = 0; r < RPL; ++r)
        if (active(r)) update(r);
      if constexpr (t + 1 < NS) {
        if constexpr (SHB) {
          bcast(std::integral_constant<int, t + 1>{}, pv);
        } else {
          stage(std::integral_constant<int, t + 1>{});
          __syncwarp();
          load(std::integral_constant<int, t + 1>{}, pv);
        }
        inv_cur = pivot_inv(std::integral_constant<int, t + 1>{}, pv);
      }
    } else if constexpr (t + 1 < NS) {
      constexpr int os_next = st_piv_row<NST, NQ>(t + 1) / LPS;
      if (active(os_next)) update(os_next);
      double pn[NC];
      if constexpr (SHB) {
        bcast(std::integral_constant<int, t + 1>{}, pn);
      } else {
        stage(std::integral_constant<int, t + 1>{});
        __syncwarp();
        load(std::integral_constant<int, t + 1>{}, pn);
      }
      inv_cur = pivot_inv(std::integral_constant<int, t + 1>{}, pn);
#pragma unroll
      for (int r = 0; r < RPL; ++r)
        if (r != os_next && active(r)) update(r);
#pragma unroll
      for (int cc = 0; cc < NC; ++cc)
        if (live_at(t + 1, cc)) pv[cc] = pn[cc];
    } else {
#pragma unroll
      for (int r = 0; r < RPL; ++r)
        if (active(r)) update(r);
    }
  });

  // ---- solution: J rows give w_J, monomial row m gives w_{I_m} (approx.py:282) ----
  double* w = &sm.w[0][0];
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    if (only_I(r)) continue;
    const int rho = s + r * LPS;
    if (lane_live && rho >= NQ) {
      const int node = rho < NST ? rho : (rho - NST < NQ ? rho - NST : 0);
#pragma unroll
      for (int o = 0; o < NOPS; ++o) w[node * NOPS + o] = a[r][NS + o] * invp[r];
    }
  }
  __syncwarp();
  if constexpr (kInlineFallback) {
    // same lane layout as the searching kernel: a warp with a flagged system re-solves its
    // whole group with partial pivoting, in its own part of shared memory (no second launch)
    if (__any_sync(0xffffffffu, sys_live && bad)) {
      using SmS = RbfSmem<D, NST, NOPS>;
      static_assert(sizeof(SmS) <= sizeof(Sm), "searching layout must fit the warp's shared memory");
      SmS* mine = reinterpret_cast<SmS*>(smem_all + warp * SPW);
      rbf_search_group<D, NST, NOPS, LPS, RPL, WARPS>(blockIdx.x, mine - warp * SPW, pos, stencils, K, K, nullptr,
                                                      ops, row_normals, out_idx, out_w, info);
      return;
    }
  }
  if (!sys_live) return;
  if (bad) {
    if (s == 0) flag_list[atomicAdd(flag_count, 1)] = static_cast<int>(k);
    return;
  }
  if (info && s == 0) info[k] = 0;
  // ---- epilogue: ascending node-index order, un-scale (approx.py:283-284, 407-410) ----
  // (node ids of an unflagged stencil are distinct: a repeated node makes two equal rows)
  const double s2 = s1 * s1;
#pragma unroll
  for (int r = 0; r < PA; ++r) {
    const int j = s + r * LPS;
    if (j < NST) {
      const int id = sm.sidp[j];
      int rank = 0;
#pragma unroll
      for (int i = 0; i < NST; ++i) rank += sm.sidp[i] < id;
      out_idx[static_cast<int64_t>(rank) * K + k] = id;
#pragma unroll
      for (int o = 0; o < NOPS; ++o) {
        const double f = (STD ? o == 0 : ops.order[o] == 2) ? s2 : s1;
        out_w[(static_cast<int64_t>(o) * NST + rank) * K + k] = w[j * NOPS + o] * f;
      }
    }
  }
}

// ===================== null-space kernel (default for the tuned 3D sizes) ======================
// The same static null-space elimination order as rbf_static_kernel (step A: partial-
// pivoting LU of P picks the unisolvent nodes I, nodes renumbered [I, J]), but the saddle
// system is reduced algebraically instead of by a Gauss-Jordan sweep over all n+q rows:
//   P^T w = c          ->  w_I = g - M^T w_J,      M = P_J P_I^-1 = L_J L_I^-1,  g = P_I^-T c
//   A w + P lambda = f ->  S w_J = h - B_I g,      B = A_J: - M A_I:,   h = f_J - M f_I,
//                          S = B_J - B_I M^T       (= Z^T A Z, SPD for r^3 on a unisolvent set)
// where step A's LU of P (Pi P = L U, L = [L_I; L_J]) gives M without another elimination:
// (1) every lane keeps its rows' step-A multipliers; M's rows by a back substitution with
// L_I, g = L_I^-T U^-T c by two tiny substitutions, (2) B and h from the I rows of A (staged
// in shared memory; A is symmetric, so a J row's I part is read from there too), (3) S and
// its right-hand side, (4) a (n - q)-step Gauss-Jordan of [S | rhs] (diagonal pivots, S is
// SPD), (5) w_I.  One segment of q lanes per system: lane s owns node row I_s and the J rows
// s, s + q, .. (n - q = q or 2q).  Stencils with a small pivot are flagged for the searching
// kernel as in the sweep.
template <int D, int NST, int NOPS>
struct RbfNsCore {
  static constexpr int NQ = poly_count<D>();
  static constexpr int NJ = NST - NQ;
  static constexpr int YS = D == 2 ? 2 : 4;
  static constexpr int NQP = (NQ + 1) & ~1;
  static constexpr int NLU = NQ * NQP + NJ * NQ + NQ * NQP;  // u, lj, li
  static constexpr int NAI = NQ * NST;                       // ai, later w and w_J
  double inv_hist[NQP];        // step A 1/pivots
  double yp[NST][YS];          // local coordinates, renumbered [I, J]
  static constexpr int NOP2 = (NOPS + 1) & ~1;
  double fi[NQ][NOP2];         // f rows of the I nodes (16-B rows)
  double mt[NQ][NJ];           // M^T
  double g[NQ][NOP2];          // P_I^-T c
  // step A's U rows | L_J rows | L_I rows, then (aliased) the I rows of A, then w and w_J
  double work[NLU > NAI ? NLU : NAI];
  int sidp[NST];               // node ids, renumbered
};
template <int D, int NST, int NOPS>
struct __align__(16) RbfNsSmem : RbfNsCore<D, NST, NOPS> {
  static constexpr int kCore = static_cast<int>(sizeof(RbfNsCore<D, NST, NOPS>));
  static constexpr int kPad = ((16 - kCore % 128) % 128 + 128) % 128;
  char pad[kPad == 0 ? 128 : kPad];
};

template <int D, int NST, int NOPS, bool STD, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) rbf_ns_kernel(
    const double* __restrict__ pos, const int* __restrict__ stencils, int64_t K, OpSpec ops,
    const double* __restrict__ row_normals, int* __restrict__ out_idx, double* __restrict__ out_w,
    int* __restrict__ info, int* __restrict__ flag_list, int* __restrict__ flag_count, int force_flag) {
  constexpr int NQ = poly_count<D>();
  constexpr int NJ = NST - NQ;
  constexpr int LPS = NQ;              // lanes per system
  constexpr int JPL = NJ / LPS;        // J rows per lane
  constexpr int SPW = 32 / LPS;
  constexpr int PA = (NST + LPS - 1) / LPS;  // step-A slots
  constexpr int NQP = (NQ + 1) & ~1;
  static_assert(NJ % LPS == 0, "J rows spread evenly over the segment");
  static_assert(NJ % 2 == 0 && NST % 2 == 0, "16-B shared-memory rows");
  static_assert(NST <= 31, "node bitmask");
  static_assert(NQ * NST >= NST * NOPS + NJ * NOPS, "w and w_J alias the I rows of A");
  using Sm = RbfNsSmem<D, NST, NOPS>;
  extern __shared__ __align__(16) unsigned char rbf_ns_smem[];
  Sm* smem_all = reinterpret_cast<Sm*>(rbf_ns_smem);

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const bool lane_live = lane < SPW * LPS;
  const int s = lane_live ? lane % LPS : 0;
  const int sys_w = lane_live ? lane / LPS : 0;
  const int64_t k_raw = (static_cast<int64_t>(blockIdx.x) * WARPS + warp) * SPW + sys_w;
  const bool sys_live = lane_live && k_raw < K;
  const int64_t k = k_raw < K ? k_raw : K - 1;
  Sm& sm = smem_all[warp * SPW + sys_w];
  double* su = sm.work;                  // U[NQ][NQP]
  double* slj = su + NQ * NQP;           // L_J[NJ][NQ]
  double* sli = slj + NJ * NQ;           // L_I[NQ][NQP]
  double* sai = sm.work;                 // A_I[NQ][NST]   (after (1))
  double* wsm = sm.work;                 // w[NST][NOPS]   (after (3))
  double* wjs = wsm + NST * NOPS;        // w_J[NJ][NOPS]
  auto seg_lane = [&](int t) { return lane_live ? sys_w * LPS + t : lane; };
  auto seg_xor = [&](int off) {
    int t = s ^ off;
    t = t < LPS ? t : LPS - 1;
    return seg_lane(t);
  };

  const bool use_rn = !STD && row_normals != nullptr;
  double rn[D];
#pragma unroll
  for (int a = 0; a < D; ++a) rn[a] = use_rn ? __ldg(row_normals + k * D + a) : 0.0;

  // ---- gather, shift to the centre, scale by the stencil radius (approx.py:245-250) ----
  double c[D];
  load_point<D>(pos, __ldg(stencils + k * NST), c);
  double yo[PA][D];
  int sido[PA];
  double d2max = 0.0;
#pragma unroll
  for (int r = 0; r < PA; ++r) {
    const int j = s + r * LPS;
    sido[r] = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) yo[r][a] = 0.0;
    if (j < NST) {
      sido[r] = __ldg(stencils + k * NST + j);
      double p[D];
      load_point<D>(pos, sido[r], p);
      double d2 = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        yo[r][a] = p[a] - c[a];
        d2 = fma(yo[r][a], yo[r][a], d2);
      }
      d2max = fmax(d2max, d2);
    }
  }
#pragma unroll
  for (int off = 1; off < LPS; off <<= 1) d2max = fmax(d2max, __shfl_sync(0xffffffffu, d2max, seg_xor(off)));
  const double s1 = fast_rcp(fast_sqrt(d2max));
#pragma unroll
  for (int r = 0; r < PA; ++r)
#pragma unroll
    for (int a = 0; a < D; ++a) yo[r][a] *= s1;

  const unsigned ub = smem_addr(su);
  const unsigned hist = smem_addr(&sm.inv_hist[0]);
  bool bad = force_flag != 0;

  // ---- step A: LU of P with partial pivoting over the nodes -> I; U rows to shared memory,
  // every row's multipliers kept (L) ----
  {
    double pp[PA][NQ], lm[PA][NQ];
    unsigned vm[PA];
    int step_of[PA];  // step that chose the slot's node (I index), -1: a J node
#pragma unroll
    for (int r = 0; r < PA; ++r) {
      const int j = s + r * LPS;
#pragma unroll
      for (int m = 0; m < NQ; ++m) {
        pp[r][m] = mono_val<D>(m, yo[r]);
        lm[r][m] = 0.0;
      }
      lm[r][0] = 1.0;  // column 0 is all ones: every row's step-0 multiplier is 1
      vm[r] = (lane_live && j < NST) ? (0x7fffffc0u | static_cast<unsigned>(63 - j)) : 0u;
      step_of[r] = -1;
    }
    unsigned chosen = 1u;
    vm[0] = s == 0 ? 0u : vm[0];
    if (s == 0) step_of[0] = 0;
    if (lane_live && s == 0) {
#pragma unroll
      for (int a = 0; a < D; ++a) sm.yp[0][a] = yo[0][a];
      sm.sidp[0] = sido[0];
      sm.inv_hist[0] = 1.0;
#pragma unroll
      for (int m = 0; m < NQ; ++m) su[m] = pp[0][m];  // the centre's row: [1, 0, ..] (y = 0)
    }
    static_for<NQ - 1>([&](auto mc) {
      constexpr int m = decltype(mc)::value + 1;
      unsigned key = 0;
#pragma unroll
      for (int r = 0; r < PA; ++r)
        key = max(key, (static_cast<unsigned>(__double2hiint(pp[r][m])) | 63u) & vm[r]);
#pragma unroll
      for (int off = 1; off < LPS; off <<= 1) key = max(key, __shfl_sync(0xffffffffu, key, seg_xor(off)));
      const unsigned ptag = key & 63u;
      const unsigned pbase = ub + 8u * m * NQP;
      bool isp[PA];
#pragma unroll
      for (int r = 0; r < PA; ++r) {
        isp[r] = ((vm[r] & 63u) == ptag) && vm[r] != 0u;
        constexpr int j0 = m & ~1;
#pragma unroll
        for (int jj = j0; jj < NQ; jj += 2) {
          if (jj + 1 < NQ) st_pred2(isp[r], pbase + 8u * jj, pp[r][jj], pp[r][jj + 1]);
          else st_pred1(isp[r], pbase + 8u * jj, pp[r][jj]);
        }
        if (isp[r]) step_of[r] = m;  // its coordinates and id go to slot m after the loop
      }
      __syncwarp();
      const double* prow = su + m * NQP;
      const double piv = prow[m];
      bad = bad || !(fabs(piv) >= kStaticPivMin);
      const double inv = fast_rcp(piv);
      st_pred1(lane_live && s == 0, hist + 8u * m, inv);
#pragma unroll
      for (int r = 0; r < PA; ++r) {
        // no masks: a row pivoted at step i only keeps its multipliers m < i (L_I is unit lower),
        // and its pp entries are never read again (vm = 0 keeps it out of every later search),
        // so eliminating it like any other row is harmless and saves the selects
        const double l = pp[r][m] * inv;
        lm[r][m] = l;
        vm[r] = isp[r] ? 0u : vm[r];
#pragma unroll
        for (int cc = m + 1; cc < NQ; ++cc) pp[r][cc] = fma(-l, prow[cc], pp[r][cc]);
      }
      chosen |= 1u << (63u - ptag);
    });
    // renumbered coordinates and ids of J; multiplier rows by renumbered index
#pragma unroll
    for (int r = 0; r < PA; ++r) {
      const int j = s + r * LPS;
      if (!(lane_live && j < NST)) continue;
      if (!((chosen >> j) & 1u)) {
        const int jr = __popc(~chosen & ((1u << j) - 1u));
#pragma unroll
        for (int a = 0; a < D; ++a) sm.yp[NQ + jr][a] = yo[r][a];
        sm.sidp[NQ + jr] = sido[r];
#pragma unroll
        for (int m = 0; m < NQ; ++m) slj[jr * NQ + m] = lm[r][m];
      } else {
        const int i = step_of[r];
#pragma unroll
        for (int a = 0; a < D; ++a) sm.yp[i][a] = yo[r][a];
        sm.sidp[i] = sido[r];
#pragma unroll
        for (int m = 0; m < NQ; ++m) sli[i * NQP + m] = m < i ? lm[r][m] : (m == i ? 1.0 : 0.0);
      }
    }
  }
  __syncwarp();

  // ---- (1) M rows (J rows of mine) by back substitution with L_I; g = L_I^-T U^-T c ----
  // (right-looking: a finished unknown updates every pending one at once, so the dependent
  // chain is q FMAs deep instead of q(q-1)/2)
  double mj[JPL][NQ];
#pragma unroll
  for (int r = 0; r < JPL; ++r) {
    const int jr = s + r * LPS;
#pragma unroll
    for (int i = 0; i < NQ; i += 2) {
      const double2 lv = *reinterpret_cast<const double2*>(slj + jr * NQ + i);
      mj[r][i] = lv.x;
      if (i + 1 < NQ) mj[r][i + 1] = lv.y;
    }
#pragma unroll
    for (int i = NQ - 1; i > 0; --i)
#pragma unroll
      for (int i2 = 0; i2 < i; ++i2) mj[r][i2] = fma(-mj[r][i], sli[i * NQP + i2], mj[r][i2]);
#pragma unroll
    for (int i = 0; i < NQ; ++i)
      if (lane_live) sm.mt[i][jr] = mj[r][i];
  }
  if (s < NOPS) {  // lane s: column o = s of g, U^T z = c forward then L_I^T g = z backward
    double z[NQ];
#pragma unroll
    for (int m = 0; m < NQ; ++m) {
      double cv = 0.0;
#pragma unroll
      for (int o = 0; o < NOPS; ++o)
        if (o == s) cv = STD ? std_poly_rhs<D>(o, m) : poly_rhs<D>(ops, o, m, use_rn, rn);
      z[m] = cv;
    }
#pragma unroll
    for (int m = 0; m < NQ; ++m) {  // right-looking: z[m] final, update the pending ones
      z[m] *= sm.inv_hist[m];
#pragma unroll
      for (int m2 = m + 1; m2 < NQ; ++m2) z[m2] = fma(-su[m * NQP + m2], z[m], z[m2]);
    }
#pragma unroll
    for (int i = NQ - 1; i > 0; --i)
#pragma unroll
      for (int m = 0; m < i; ++m) z[m] = fma(-sli[i * NQP + m], z[i], z[m]);
#pragma unroll
    for (int m = 0; m < NQ; ++m)
      if (lane_live) sm.g[m][s] = z[m];
  }
  __syncwarp();  // U and L are dead: the I rows of A take their place

  // ---- the I row of A and f (node I_s) -> shared memory ----
  {
    double yI[D];
#pragma unroll
    for (int a = 0; a < D; ++a) yI[a] = sm.yp[s][a];
    const double rI = norm_fast<D>(yI);
#pragma unroll
    for (int o = 0; o < NOPS; ++o) {
      double f;
      if constexpr (STD) f = o == 0 ? 3.0 * (D + 1) * rI : -3.0 * rI * yI[o - 1];
      else f = phs_rhs<D>(ops, o, yI, rI, use_rn, rn);
      if (lane_live) sm.fi[s][o] = f;
    }
#pragma unroll
    for (int cc = 0; cc < NST; cc += 2) {
      double v[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        v[h] = 0.0;
        if (cc + h < NST) {
          double d2 = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const double t = yI[a] - sm.yp[cc + h][a];
            d2 = fma(t, t, d2);
          }
          v[h] = cube_from_sq(d2);
        }
      }
      if (cc + 1 < NST) st_pred2(lane_live, smem_addr(sai + s * NST + cc), v[0], v[1]);
      else st_pred1(lane_live, smem_addr(sai + s * NST + cc), v[0]);
    }
  }
  __syncwarp();

  // ---- (2)-(3) B row, h, then S row and its right-hand side, for each of my J rows ----
  double S[JPL][NJ], R[JPL][NOPS];
#pragma unroll
  for (int r = 0; r < JPL; ++r) {
    const int jr = s + r * LPS;  // J index
    double yJ[D];
#pragma unroll
    for (int a = 0; a < D; ++a) yJ[a] = sm.yp[NQ + jr][a];
    double b[NST], h[NOPS];
    const double rJ = norm_fast<D>(yJ);
#pragma unroll
    for (int o = 0; o < NOPS; ++o) {
      if constexpr (STD) h[o] = o == 0 ? 3.0 * (D + 1) * rJ : -3.0 * rJ * yJ[o - 1];
      else h[o] = phs_rhs<D>(ops, o, yJ, rJ, use_rn, rn);
    }
#pragma unroll
    for (int i = 0; i < NQ; ++i) b[i] = sai[i * NST + NQ + jr];  // A symmetric: A[J][I_i] = A[I_i][J]
#pragma unroll
    for (int cc = NQ; cc < NST; ++cc) {
      double d2 = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double t = yJ[a] - sm.yp[cc][a];
        d2 = fma(t, t, d2);
      }
      b[cc] = cube_from_sq(d2);
    }
    // B row = A_J row - sum_i M[j][i] A_I row i;  h = f_J - sum_i M[j][i] f_I row i
#pragma unroll
    for (int i = 0; i < NQ; ++i) {
      const double mji = mj[r][i];
#pragma unroll
      for (int cc = 0; cc < NST; cc += 2) {
        if (cc + 1 < NST) {
          const double2 av = *reinterpret_cast<const double2*>(sai + i * NST + cc);
          b[cc] = fma(-mji, av.x, b[cc]);
          b[cc + 1] = fma(-mji, av.y, b[cc + 1]);
        } else {
          b[cc] = fma(-mji, sai[i * NST + cc], b[cc]);
        }
      }
#pragma unroll
      for (int o = 0; o < NOPS; o += 2) {
        if (o + 1 < NOPS) {
          const double2 fv = *reinterpret_cast<const double2*>(&sm.fi[i][o]);
          h[o] = fma(-mji, fv.x, h[o]);
          h[o + 1] = fma(-mji, fv.y, h[o + 1]);
        } else {
          h[o] = fma(-mji, sm.fi[i][o], h[o]);
        }
      }
    }
    // S row = B_J - B_I M^T;  rhs = h - B_I g
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) S[r][jj] = b[NQ + jj];
#pragma unroll
    for (int o = 0; o < NOPS; ++o) R[r][o] = h[o];
#pragma unroll
    for (int i = 0; i < NQ; ++i) {
      const double bi = b[i];
#pragma unroll
      for (int jj = 0; jj < NJ; jj += 2) {
        const double2 mv = *reinterpret_cast<const double2*>(&sm.mt[i][jj]);
        S[r][jj] = fma(-bi, mv.x, S[r][jj]);
        S[r][jj + 1] = fma(-bi, mv.y, S[r][jj + 1]);
      }
#pragma unroll
      for (int o = 0; o < NOPS; o += 2) {
        if (o + 1 < NOPS) {
          const double2 gv = *reinterpret_cast<const double2*>(&sm.g[i][o]);
          R[r][o] = fma(-bi, gv.x, R[r][o]);
          R[r][o + 1] = fma(-bi, gv.y, R[r][o + 1]);
        } else {
          R[r][o] = fma(-bi, sm.g[i][o], R[r][o]);
        }
      }
    }
  }
  __syncwarp();  // the I rows of A are dead from here on: w / w_J take their place

  // ---- (4) Gauss-Jordan on [S | rhs], diagonal pivots (S is SPD) ----
  static_for<NJ>([&](auto kc) {
    constexpr int kk = decltype(kc)::value;
    constexpr int ko = kk % LPS, kr = kk / LPS;  // owner lane and slot of pivot row kk
    const int src = seg_lane(ko);
    const double piv = __shfl_sync(0xffffffffu, S[kr][kk], src);
    bad = bad || !(piv >= kStaticSchurMin);
    const double inv = fast_rcp(piv);
    double pr[NJ + NOPS];
#pragma unroll
    for (int cc = kk + 1; cc < NJ; ++cc) pr[cc] = __shfl_sync(0xffffffffu, S[kr][cc], src);
#pragma unroll
    for (int o = 0; o < NOPS; ++o) pr[NJ + o] = __shfl_sync(0xffffffffu, R[kr][o], src);
#pragma unroll
    for (int r = 0; r < JPL; ++r) {
      const bool mine = (r == kr) && (s == ko);
      const double l = mine ? 0.0 : S[r][kk] * inv;
#pragma unroll
      for (int cc = kk + 1; cc < NJ; ++cc) S[r][cc] = fma(-l, pr[cc], S[r][cc]);
#pragma unroll
      for (int o = 0; o < NOPS; ++o) R[r][o] = fma(-l, pr[NJ + o], R[r][o]);
    }
  });
#pragma unroll
  for (int r = 0; r < JPL; ++r) {
    const int jr = s + r * LPS;
    double dg = 0.0;
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) dg = jj == jr ? S[r][jj] : dg;
    const double inv = fast_rcp(dg);
#pragma unroll
    for (int o = 0; o < NOPS; ++o) {
      const double wv = R[r][o] * inv;
      if (lane_live) {
        wjs[jr * NOPS + o] = wv;
        wsm[(NQ + jr) * NOPS + o] = wv;
      }
    }
  }
  __syncwarp();

  // ---- (5) w_I = g - M^T w_J ----
#pragma unroll
  for (int o = 0; o < NOPS; ++o) {
    double v = sm.g[s][o];
#pragma unroll
    for (int j = 0; j < NJ; ++j) v = fma(-sm.mt[s][j], wjs[j * NOPS + o], v);
    if (lane_live) wsm[s * NOPS + o] = v;
  }
  __syncwarp();

  if (!sys_live) return;
  if (bad) {
    if (s == 0) flag_list[atomicAdd(flag_count, 1)] = static_cast<int>(k);
    return;
  }
  if (info && s == 0) info[k] = 0;
  // ---- epilogue: ascending node-index order, un-scale (approx.py:283-284, 407-410) ----
  const double s2 = s1 * s1;
#pragma unroll
  for (int r = 0; r < PA; ++r) {
    const int j = s + r * LPS;
    if (j < NST) {
      const int id = sm.sidp[j];
      int rank = 0;
#pragma unroll
      for (int i = 0; i < NST; ++i) rank += sm.sidp[i] < id;
      out_idx[static_cast<int64_t>(rank) * K + k] = id;
#pragma unroll
      for (int o = 0; o < NOPS; ++o) {
        const double f = (STD ? o == 0 : ops.order[o] == 2) ? s2 : s1;
        out_w[(static_cast<int64_t>(o) * NST + rank) * K + k] = wsm[j * NOPS + o] * f;
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

#define HN_MON(DD, NO)                                                                                  \
  do {                                                                                                  \
    mon_weights_kernel<DD, NO><<<bl, th, 0, s>>>(pos, stencils, K, ops, out_idx, out_w, info);          \
  } while (0)
  if (d == 2) {
    switch (nops) { case 1: HN_MON(2, 1); break; case 2: HN_MON(2, 2); break; case 3: HN_MON(2, 3); break; default: HN_MON(2, 4); }
  } else {
    switch (nops) { case 1: HN_MON(3, 1); break; case 2: HN_MON(3, 2); break; case 3: HN_MON(3, 3); break; default: HN_MON(3, 4); }
  }
#undef HN_MON
  HN_CHECK_LAUNCH();
  return 0;
}

template <int D, int NST, int NOPS, int LPS, int RPL, int WARPS, int MINB>
static void launch_rbf_v(const double* pos, const int* st, int64_t K, const OpSpec& ops, const double* rn, int* oi,
                         double* ow, int* info, cudaStream_t s) {
  constexpr int SPW = 32 / LPS;
  const int64_t per_block = static_cast<int64_t>(WARPS) * SPW;
  rbf_weights_kernel<D, NST, NOPS, LPS, RPL, WARPS, MINB><<<ceil_div(K, per_block), WARPS * 32, 0, s>>>(
      pos, st, K, ops, rn, oi, ow, info, nullptr, nullptr);
}

// Static-order kernel, then the searching kernel over the stencils it flagged (list mode,
// grid-stride: an empty list costs one short launch).
template <int D, int NST, int NOPS, int LPS, int RPL, int WARPS, int MINB, int FLPS, int FRPL, bool ILV = false,
          bool SHB = false, bool LA = true>
static cudaError_t launch_rbf_static(const double* pos, const int* st, int64_t K, const OpSpec& ops,
                                     const double* rn, int* oi, double* ow, int* info, cudaStream_t s, int force) {
  // the standard operator set [Lap, d/dx_0, ..] gets compile-time right-hand sides
  bool std_ops = rn == nullptr && NOPS == D + 1 && ops.kind[0] == kOpLaplacian;
  for (int o = 1; o < NOPS && std_ops; ++o) std_ops = ops.kind[o] == kOpPartial && ops.axis[o] == o - 1;
  // same lane layout as the searching kernel: flagged systems are re-solved in the kernel
  constexpr bool inline_fb = D == 2 && NST == 12 && LPS == 6 && RPL == 3 && !ILV;
  int* buf = nullptr;  // [count, list...] of flagged stencils (second launch)
  if (!inline_fb) {
    cudaError_t e = stream_alloc(reinterpret_cast<void**>(&buf), sizeof(int) * (K + 1), s);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(buf, 0, sizeof(int), s);
  }
  constexpr int SPW = 32 / LPS;
  const int64_t grid = ceil_div(K, static_cast<int64_t>(WARPS) * SPW);
  const size_t smem = sizeof(RbfStaticSmem<D, NST, NOPS>) * WARPS * SPW;
  auto go = [&](auto kc) {
    constexpr auto kern = decltype(kc)::value;
    // dynamic smem may exceed 48 KB; function attributes are per device, so set every call (cheap)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<grid, WARPS * 32, smem, s>>>(pos, st, K, ops, rn, oi, ow, info, buf ? buf + 1 : nullptr, buf, force);
  };
  using KT = decltype(&rbf_static_kernel<D, NST, NOPS, false, LPS, RPL, WARPS, MINB, ILV, SHB, LA>);
  if constexpr (NOPS == D + 1) {
    if (std_ops) go(std::integral_constant<KT, &rbf_static_kernel<D, NST, NOPS, true, LPS, RPL, WARPS, MINB, ILV, SHB, LA>>{});
    else go(std::integral_constant<KT, &rbf_static_kernel<D, NST, NOPS, false, LPS, RPL, WARPS, MINB, ILV, SHB, LA>>{});
  } else {
    go(std::integral_constant<KT, &rbf_static_kernel<D, NST, NOPS, false, LPS, RPL, WARPS, MINB, ILV, SHB, LA>>{});
  }
  if constexpr (inline_fb) return cudaGetLastError();
  constexpr int FSPW = 32 / FLPS;
  const int64_t groups = ceil_div(K, static_cast<int64_t>(4) * FSPW);
  const int64_t cap = static_cast<int64_t>(sm_count()) * 2;
  rbf_weights_kernel<D, NST, NOPS, FLPS, FRPL, 4, 1><<<static_cast<int>(groups < cap ? groups : cap), 128, 0, s>>>(
      pos, st, K, ops, rn, oi, ow, info, buf + 1, buf);
  return cudaFreeAsync(buf, s);
}

// Null-space kernel, then the searching kernel over the stencils it flagged (list mode).
template <int D, int NST, int NOPS, int WARPS, int MINB, int FLPS, int FRPL>
static cudaError_t launch_rbf_ns(const double* pos, const int* st, int64_t K, const OpSpec& ops, const double* rn,
                                 int* oi, double* ow, int* info, cudaStream_t s, int force) {
  bool std_ops = rn == nullptr && NOPS == D + 1 && ops.kind[0] == kOpLaplacian;
  for (int o = 1; o < NOPS && std_ops; ++o) std_ops = ops.kind[o] == kOpPartial && ops.axis[o] == o - 1;
  int* buf = nullptr;  // [count, list...] of flagged stencils
  cudaError_t e = stream_alloc(reinterpret_cast<void**>(&buf), sizeof(int) * (K + 1), s);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(buf, 0, sizeof(int), s);
  constexpr int SPW = 32 / poly_count<D>();
  const int64_t grid = ceil_div(K, static_cast<int64_t>(WARPS) * SPW);
  const size_t smem = sizeof(RbfNsSmem<D, NST, NOPS>) * WARPS * SPW;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<grid, WARPS * 32, smem, s>>>(pos, st, K, ops, rn, oi, ow, info, buf + 1, buf, force);
  };
  if constexpr (NOPS == D + 1) {
    if (std_ops) go(rbf_ns_kernel<D, NST, NOPS, true, WARPS, MINB>);
    else go(rbf_ns_kernel<D, NST, NOPS, false, WARPS, MINB>);
  } else {
    go(rbf_ns_kernel<D, NST, NOPS, false, WARPS, MINB>);
  }
  constexpr int FSPW = 32 / FLPS;
  const int64_t groups = ceil_div(K, static_cast<int64_t>(4) * FSPW);
  const int64_t cap = static_cast<int64_t>(sm_count()) * 2;
  rbf_weights_kernel<D, NST, NOPS, FLPS, FRPL, 4, 1><<<static_cast<int>(groups < cap ? groups : cap), 128, 0, s>>>(
      pos, st, K, ops, rn, oi, ow, info, buf + 1, buf);
  return cudaFreeAsync(buf, s);
}

// Kernel choice (tests; 0 = default: null-space kernel + flagged fallback): 100 = searching
// kernel for every stencil; 101 = default kernel with every stencil flagged (exercises the
// fallback); 102 = the Gauss-Jordan sweep kernel (rbf_static_kernel) in 3D; 103 = the
// null-space kernel in 2D.  The launch shapes tried while tuning are
// recorded in DESIGN.md section 4.
static int g_rbf_variant = 0;
HN_EXPORT void hn_weights_rbf_set_variant(int v) { g_rbf_variant = v; }

template <int D, int NST, int NOPS>
static cudaError_t launch_rbf(const double* pos, const int* st, int64_t K, const OpSpec& ops, const double* rn,
                              int* oi, double* ow, int* info, cudaStream_t s) {
  const int v = g_rbf_variant;
  const int force = v == 101 ? 1 : 0;
  if constexpr (D == 2) {
    if (v == 100) {
      launch_rbf_v<2, 12, NOPS, 6, 3, 4, 3>(pos, st, K, ops, rn, oi, ow, info, s);
      return cudaSuccess;
    }
    // 2D: the Gauss-Jordan sweep with pivot rows broadcast by shuffles (config 1: 86 us; the
    // null-space kernel, variant 103, is 6 % slower at this size: 6 lanes per system)
    if (v == 103) return launch_rbf_ns<2, 12, NOPS, 4, 4, 6, 3>(pos, st, K, ops, rn, oi, ow, info, s, 0);
    return launch_rbf_static<2, 12, NOPS, 6, 3, 4, 4, 6, 3, false, true>(pos, st, K, ops, rn, oi, ow, info, s, force);
  } else if constexpr (NST == 20) {
    if (v == 100) {
      launch_rbf_v<3, 20, NOPS, 15, 2, 4, 1>(pos, st, K, ops, rn, oi, ow, info, s);
      return cudaSuccess;
    }
    // 3D: no look-ahead (the 34/40-wide pivot row would be a second live register row;
    // measured 2.3% (n=20) and 4.5% (n=30) faster than staging the next row early)
    if (v == 102)
      return launch_rbf_static<3, 20, NOPS, 10, 3, 4, 2, 15, 2, false, false, false>(pos, st, K, ops, rn, oi, ow, info, s, 0);
    return launch_rbf_ns<3, 20, NOPS, 4, 4, 15, 2>(pos, st, K, ops, rn, oi, ow, info, s, force);
  } else {
    if (v == 100) {
      launch_rbf_v<3, 30, NOPS, 20, 2, 4, 1>(pos, st, K, ops, rn, oi, ow, info, s);
      return cudaSuccess;
    }
    if (v == 102)
      return launch_rbf_static<3, 30, NOPS, 20, 2, 4, 1, 20, 2, false, false, false>(pos, st, K, ops, rn, oi, ow, info, s, 0);
    return launch_rbf_ns<3, 30, NOPS, 4, 2, 20, 2>(pos, st, K, ops, rn, oi, ow, info, s, force);
  }
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
        case 1: HN_TRY((launch_rbf<2, 12, 1>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s))); break;
        case 2: HN_TRY((launch_rbf<2, 12, 2>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s))); break;
        case 3: HN_TRY((launch_rbf<2, 12, 3>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s))); break;
        default: HN_TRY((launch_rbf<2, 12, 4>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s))); break;
      }
    } else if (n == 20) {
      switch (nops) {
        case 1: HN_TRY((launch_rbf<3, 20, 1>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s))); break;
        case 2: HN_TRY((launch_rbf<3, 20, 2>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s))); break;
        case 3: HN_TRY((launch_rbf<3, 20, 3>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s))); break;
        default: HN_TRY((launch_rbf<3, 20, 4>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s))); break;
      }
    } else {
      switch (nops) {
        case 1: HN_TRY((launch_rbf<3, 30, 1>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s))); break;
        case 2: HN_TRY((launch_rbf<3, 30, 2>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s))); break;
        case 3: HN_TRY((launch_rbf<3, 30, 3>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s))); break;
        default: HN_TRY((launch_rbf<3, 30, 4>(pos, stencils, K, ops, row_normals, out_idx, out_w, info, s))); break;
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
