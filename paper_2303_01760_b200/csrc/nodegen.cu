// K12: node-set generation on the device.
//
// Reference: pkg/src/hybridnodes/nodegen.py -- regular_fill :196-216, carve_transition
// :219-227, _wave_candidates :270-294, scattered_fill :297-381 (advancing front),
// hybrid_discretize :436-518 (region cut + lattice map); geometry.py -- box / circle /
// star / ellipse signed distances :37-199, DomainSpec :253-312.
//
// The reference's advancing front is a Python loop over candidates: a candidate is accepted
// when no node accepted before it (seed, earlier wave, or earlier in this wave) lies closer
// than 0.995 of its target spacing.  Here one wave is three parallel steps:
//   1. candidates of all parents at once (one thread per candidate; the random draws are
//      the caller's -- numpy's Generator stream, so the directions are the reference's);
//   2. a pre-test of every candidate against the nodes that existed before the wave
//      (uniform grid of cell >= every acceptance radius: a 3^d window is exact);
//   3. the in-wave conflicts (candidate j rejected by an ACCEPTED earlier candidate i with
//      |c_i - c_j| < 0.995 h_j) resolved in candidate order by a sync-free pass: CTAs take
//      tickets in order, wait only on decisions of earlier CTAs, and decide their own
//      128 candidates sequentially from conflict bit masks -- the same accept set as the
//      sequential loop (lexicographically-first greedy), in any schedule.
// Box / circle / sphere geometry uses only correctly rounded + - * / sqrt in numpy's
// operation order (no contraction), so those node sets are bit-identical to the
// reference's.  Star / ellipse distances go through sin/cos/atan2 (device libm, not the
// host's), so their node sets agree to rounding.
#include <algorithm>
#include <cmath>

#include <cub/cub.cuh>

#include "hn.h"
#include "hn_common.cuh"

namespace hn {
namespace {

constexpr int kTable = 1024;           // _CURVE_TABLE geometry.py:21
constexpr double kAccept = 0.995;      // _ACCEPT nodegen.py:31
constexpr int kThr = 256;
constexpr int kResolve = 128;          // candidates decided per CTA in the in-wave pass

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

// ---------------------------------------------------------------- geometry (device)
// DomainSpec.box_signed_distance geometry.py:279-287
template <int D>
__device__ double box_sd(const hn_geom& g, const double* p) {
  double s = 0.0, mx = -INFINITY;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double c = mul(add(g.lo[a], g.hi[a]), 0.5), half = mul(sub(g.hi[a], g.lo[a]), 0.5);
    const double q = sub(fabs(sub(p[a], c)), half);
    const double m = q > 0.0 ? q : 0.0;
    s = add(s, mul(m, m));
    mx = q > mx ? q : mx;
  }
  return add(__dsqrt_rn(s), mx < 0.0 ? mx : 0.0);
}

// Circle.signed_distance geometry.py:53-54 (circle in 2D, sphere in 3D)
template <int D>
__device__ double circle_sd(const double* par, const double* p) {
  double s = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double t = sub(p[a], par[a]);
    s = add(s, mul(t, t));
  }
  return sub(__dsqrt_rn(s), par[D]);
}

// Star (geometry.py:148-197): r(t) = mean + amp cos(lobes t + phase)
struct StarEval {
  double cx, cy, mean, amp, lobes, phase;
  __device__ double radius(double t) const { return add(mean, mul(amp, cos(add(mul(lobes, t), phase)))); }
  __device__ void point(double t, double* o) const {
    const double r = radius(t);
    o[0] = add(cx, mul(r, cos(t)));
    o[1] = add(cy, mul(r, sin(t)));
  }
  __device__ void vel_acc(double t, double* v, double* ac) const {
    const double c = cos(t), s = sin(t), arg = add(mul(lobes, t), phase);
    const double r = radius(t);
    const double rp = mul(mul(-amp, lobes), sin(arg));
    const double rpp = mul(mul(-amp, mul(lobes, lobes)), cos(arg));
    v[0] = add(mul(rp, c), mul(r, -s));
    v[1] = add(mul(rp, s), mul(r, c));
    const double k = sub(rpp, r), rp2 = mul(2.0, rp);
    ac[0] = add(mul(k, c), mul(rp2, -s));
    ac[1] = add(mul(k, s), mul(rp2, c));
  }
  __device__ bool inside(const double* p) const {
    const double rx = sub(p[0], cx), ry = sub(p[1], cy);
    return __dsqrt_rn(add(mul(rx, rx), mul(ry, ry))) < radius(atan2(ry, rx));
  }
};

// Ellipse (geometry.py:104-145): point = centre + [a cos t, b sin t] R^T, R = [[c,-s],[s,c]]
struct EllipseEval {
  double cx, cy, a, b, c, s;
  __device__ void rot(double w0, double w1, double* o) const {
    o[0] = add(mul(w0, c), mul(w1, -s));
    o[1] = add(mul(w0, s), mul(w1, c));
  }
  __device__ void point(double t, double* o) const {
    rot(mul(a, cos(t)), mul(b, sin(t)), o);
    o[0] = add(cx, o[0]);
    o[1] = add(cy, o[1]);
  }
  __device__ void vel_acc(double t, double* v, double* ac) const {
    const double ct = cos(t), st = sin(t);
    rot(mul(-a, st), mul(b, ct), v);
    rot(mul(-a, ct), mul(-b, st), ac);
  }
  __device__ bool inside(const double* p) const {
    const double r0 = sub(p[0], cx), r1 = sub(p[1], cy);
    const double z0 = add(mul(r0, c), mul(r1, s)), z1 = add(mul(r0, -s), mul(r1, c));
    const double u = dvd(z0, a), w = dvd(z1, b);
    return add(mul(u, u), mul(w, w)) < 1.0;
  }
};

// _ClosedCurve.signed_distance geometry.py:73-92: nearest table point (the reference's
// cKDTree query), three Newton starts one table step apart, 6 clipped Newton steps each.
template <class C>
__device__ double curve_sd(const C& cv, const double* t_tab, const double* tab, const double* p) {
  double best = INFINITY;
  int bi = 0;
  for (int k = 0; k < kTable; ++k) {
    const double dx = sub(p[0], __ldg(tab + 2 * k)), dy = sub(p[1], __ldg(tab + 2 * k + 1));
    const double d2 = add(mul(dx, dx), mul(dy, dy));
    if (d2 < best) {
      best = d2;
      bi = k;
    }
  }
  const double step = 6.283185307179586 / kTable;
  double dmin = INFINITY;
#pragma unroll 1
  for (int st = -1; st <= 1; ++st) {
    double t = add(__ldg(t_tab + bi), st * step);
    for (int it = 0; it < 6; ++it) {
      double gm[2], v[2], ac[2];
      cv.point(t, gm);
      cv.vel_acc(t, v, ac);
      const double d0 = sub(p[0], gm[0]), d1 = sub(p[1], gm[1]);
      const double gg = add(mul(d0, v[0]), mul(d1, v[1]));
      const double gp = add(-add(mul(v[0], v[0]), mul(v[1], v[1])), add(mul(d0, ac[0]), mul(d1, ac[1])));
      double dt = dvd(gg, fabs(gp) > 1e-300 ? gp : 1.0);
      dt = fmin(fmax(dt, -2.0 * step), 2.0 * step);
      t = sub(t, dt);
    }
    double gm[2];
    cv.point(t, gm);
    const double e0 = sub(p[0], gm[0]), e1 = sub(p[1], gm[1]);
    const double d = __dsqrt_rn(add(mul(e0, e0), mul(e1, e1)));
    dmin = d < dmin ? d : dmin;
  }
  return cv.inside(p) ? -dmin : dmin;
}

// DomainSpec.obstacle_distance geometry.py:289-296 (+inf without obstacles)
template <int D>
__device__ double obstacle_distance(const hn_geom& g, const double* p) {
  double best = INFINITY;
  for (int j = 0; j < g.n_obs; ++j) {
    const double* par = g.obs_par + 8 * j;
    const int kind = __ldg(g.obs_kind + j);
    double d;
    if (kind == 0) {
      double pr[D + 1];
#pragma unroll
      for (int a = 0; a <= D; ++a) pr[a] = __ldg(par + a);
      d = circle_sd<D>(pr, p);
    } else if constexpr (D == 2) {
      if (kind == 1) {
        StarEval s{__ldg(par), __ldg(par + 1), __ldg(par + 2), __ldg(par + 3), __ldg(par + 4), __ldg(par + 5)};
        d = curve_sd(s, g.curve_t, g.curve_tab + 2 * kTable * j, p);
      } else {
        EllipseEval e{__ldg(par), __ldg(par + 1), __ldg(par + 2), __ldg(par + 3), __ldg(par + 4), __ldg(par + 5)};
        d = curve_sd(e, g.curve_t, g.curve_tab + 2 * kTable * j, p);
      }
    } else {
      d = NAN;
    }
    best = d < best ? d : best;
  }
  return best;
}

// DomainSpec.signed_distance geometry.py:298-303
template <int D>
__device__ double signed_distance(const hn_geom& g, const double* p) {
  double sd = box_sd<D>(g, p);
  if (g.n_obs) {
    const double o = -obstacle_distance<D>(g, p);
    sd = o > sd ? o : sd;
  }
  return sd;
}

// SpacingFunction.__call__ nodegen.py:53-60
template <int D>
__device__ double spacing(const hn_geom& g, const double* p) {
  if (!g.graded) return g.h_r;
  double t = dvd(obstacle_distance<D>(g, p), g.width);
  t = fmin(fmax(t, 0.0), 1.0);
  return add(g.h_s, mul(sub(g.h_r, g.h_s), t));
}

// _scattered_region nodegen.py:384-433; near = the dilated predicate used for the queue
template <int D>
__device__ bool in_region(const hn_geom& g, const double* p, bool near) {
  switch (g.region) {
    case 1:
      return true;
    case 2: {
      const bool q = (p[0] < g.rc[0]) == (p[1] < g.rc[1]);
      if (!near) return q;
      const double seam = fmin(fabs(sub(p[0], g.rc[0])), fabs(sub(p[1], g.rc[1])));
      return q || seam < g.rt[1];
    }
    case 3:
      return p[g.axis] < (near ? g.rt[1] : g.rt[0]);
    case 4:
      return obstacle_distance<D>(g, p) < (near ? g.rt[1] : g.rt[0]);
    default:
      return false;
  }
}

template <int D>
__device__ __forceinline__ void ld(const double* __restrict__ a, int64_t i, double* p) {
#pragma unroll
  for (int k = 0; k < D; ++k) p[k] = a[i * D + k];
}

// ---------------------------------------------------------------- kernels
template <int D>
__global__ void __launch_bounds__(kThr) geom_eval_kernel(hn_geom g, const double* __restrict__ pts, int64_t n,
                                                         int mode, double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (i >= n) return;
  double p[D];
  ld<D>(pts, i, p);
  double v;
  switch (mode) {
    case 0: v = signed_distance<D>(g, p); break;
    case 1: v = obstacle_distance<D>(g, p); break;
    case 2: v = spacing<D>(g, p); break;
    case 3: v = box_sd<D>(g, p); break;
    case 4: v = in_region<D>(g, p, false) ? 1.0 : 0.0; break;
    default: v = in_region<D>(g, p, true) ? 1.0 : 0.0; break;
  }
  out[i] = v;
}

struct LatticeDims {
  int64_t n[3];     // keys 1..cells_a-1 -> n_a = cells_a - 1
  double step[3];
};

// regular_fill's meshgrid(indexing="ij").ravel() order: the last axis fastest
template <int D>
__device__ __forceinline__ void lattice_key(const LatticeDims& L, int64_t id, int64_t* key) {
#pragma unroll
  for (int a = D - 1; a >= 0; --a) {
    key[a] = id % L.n[a] + 1;
    id /= L.n[a];
  }
}

template <int D>
__global__ void __launch_bounds__(kThr) lattice_flag_kernel(hn_geom g, LatticeDims L, int64_t total, double thr,
                                                            int drop_region, double carve,
                                                            uint8_t* __restrict__ keep) {
  const int64_t id = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (id >= total) return;
  int64_t key[D];
  lattice_key<D>(L, id, key);
  double p[D];
#pragma unroll
  for (int a = 0; a < D; ++a) p[a] = add(g.lo[a], mul(static_cast<double>(key[a]), L.step[a]));
  bool k = signed_distance<D>(g, p) <= thr;
  if (k && drop_region) k = !in_region<D>(g, p, false);
  if (k && carve > 0.0) k = obstacle_distance<D>(g, p) >= carve;
  keep[id] = k;
}

template <int D>
__global__ void __launch_bounds__(kThr) lattice_gather_kernel(hn_geom g, LatticeDims L,
                                                              const int64_t* __restrict__ ids,
                                                              const int64_t* __restrict__ count,
                                                              double* __restrict__ pos, int64_t* __restrict__ keys) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (i >= *count) return;
  int64_t key[D];
  lattice_key<D>(L, ids[i], key);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    pos[i * D + a] = add(g.lo[a], mul(static_cast<double>(key[a]), L.step[a]));
    keys[i * D + a] = key[a];
  }
}

// _wave_candidates nodegen.py:270-294 + the ok mask of scattered_fill :346-349.
// One thread per (parent, direction m); the direction's slot is its rank in u.
template <int D>
__global__ void __launch_bounds__(kThr) candidates_kernel(hn_geom g, const double* __restrict__ pts,
                                                          const double* __restrict__ hs,
                                                          const int64_t* __restrict__ front, int64_t front_lo,
                                                          int64_t k, const double* __restrict__ rnd,
                                                          const double* __restrict__ u, int use_region,
                                                          double* __restrict__ cand, double* __restrict__ hcand,
                                                          uint8_t* __restrict__ ok) {
  constexpr int kDir = 3 * D + 1;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (t >= k * kDir) return;
  const int64_t q = t / kDir;
  const int m = static_cast<int>(t % kDir);
  double dir[D];
  if (m < 2 * D) {
#pragma unroll
    for (int a = 0; a < D; ++a) dir[a] = (a == m % D) ? (m < D ? 1.0 : -1.0) : (m < D ? 0.0 : -0.0);
  } else {
    const double* v = rnd + (q * (D + 1) + (m - 2 * D)) * D;
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) s = add(s, mul(v[a], v[a]));
    double nrm = __dsqrt_rn(s);
    if (nrm < 1e-12) nrm = 1.0;
#pragma unroll
    for (int a = 0; a < D; ++a) dir[a] = dvd(v[a], nrm);
  }
  const double* uq = u + q * kDir;
  const double um = uq[m];
  int rank = 0;
#pragma unroll
  for (int j = 0; j < kDir; ++j) rank += (uq[j] < um) || (uq[j] == um && j < m);
  const int64_t parent = front ? front[q] : front_lo + q;
  double base[D], c[D];
  ld<D>(pts, parent, base);
  double r = hs[parent];
#pragma unroll
  for (int a = 0; a < D; ++a) c[a] = add(base[a], mul(r, dir[a]));
  for (int it = 0; it < 3; ++it) {
    r = spacing<D>(g, c);
#pragma unroll
    for (int a = 0; a < D; ++a) c[a] = add(base[a], mul(r, dir[a]));
  }
  const double h = spacing<D>(g, c);
  bool good = signed_distance<D>(g, c) <= mul(-0.5, h);
  if (good && use_region) good = in_region<D>(g, c, false);
  const int64_t s = q * kDir + rank;
#pragma unroll
  for (int a = 0; a < D; ++a) cand[s * D + a] = c[a];
  hcand[s] = h;
  ok[s] = good;
}

// ---- uniform grid (CSR by cell) over a point set
struct Grid {
  double lo[3], inv;   // cell index = floor((x - lo) * inv) -- monotone, so a 3^d window covers
  int dims[3];         // every point within one cell edge
  int64_t ncells;
};

template <int D>
__device__ __forceinline__ int64_t cell_of(const Grid& G, const double* p, int* c) {
  int64_t lin = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double f = floor((p[a] - G.lo[a]) * G.inv);
    int ci = f < 0.0 ? 0 : (f >= G.dims[a] ? G.dims[a] - 1 : static_cast<int>(f));
    c[a] = ci;
    lin = lin * G.dims[a] + ci;
  }
  return lin;
}

template <int D>
__global__ void __launch_bounds__(kThr) grid_count_kernel(Grid G, const double* __restrict__ pts,
                                                          const int64_t* __restrict__ sel, int64_t n,
                                                          int* __restrict__ cnt, int* __restrict__ cell) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (i >= n) return;
  double p[D];
  ld<D>(pts, sel ? sel[i] : i, p);
  int c[D];
  const int64_t lin = cell_of<D>(G, p, c);
  cell[i] = static_cast<int>(lin);
  atomicAdd(cnt + lin, 1);
}

__global__ void __launch_bounds__(kThr) grid_fill_kernel(const int* __restrict__ cell, int64_t n,
                                                         int* __restrict__ cursor, int* __restrict__ items) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (i >= n) return;
  items[atomicAdd(cursor + cell[i], 1)] = static_cast<int>(i);
}

// Pre-test against the nodes that existed before the wave (scattered_fill :355-366).
template <int D>
__global__ void __launch_bounds__(kThr) pretest_kernel(Grid G, const int* __restrict__ start,
                                                       const int* __restrict__ items, const double* __restrict__ pts,
                                                       const uint8_t* __restrict__ seed_regular, int64_t n_seeds,
                                                       double seam, const double* __restrict__ cand,
                                                       const double* __restrict__ hcand,
                                                       const uint8_t* __restrict__ ok, int64_t m,
                                                       uint8_t* __restrict__ pass) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (j >= m) return;
  if (!ok[j]) {
    pass[j] = 0;
    return;
  }
  double c[D];
  ld<D>(cand, j, c);
  const double lim = mul(kAccept, hcand[j]);
  int cc[D];
  cell_of<D>(G, c, cc);
  bool good = true;
  int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
#pragma unroll
  for (int a = 0; a < D; ++a) {
    lo[a] = cc[a] > 0 ? cc[a] - 1 : 0;
    hi[a] = cc[a] + 1 < G.dims[a] ? cc[a] + 1 : G.dims[a] - 1;
  }
  for (int x = lo[0]; x <= hi[0] && good; ++x)
    for (int y = lo[1]; y <= hi[1] && good; ++y)
      for (int z = (D == 3 ? lo[2] : 0); z <= (D == 3 ? hi[2] : 0) && good; ++z) {
        const int64_t lin = D == 3 ? (static_cast<int64_t>(x) * G.dims[1] + y) * G.dims[2] + z
                                   : static_cast<int64_t>(x) * G.dims[1] + y;
        for (int e = start[lin]; e < start[lin + 1]; ++e) {
          const int i = items[e];
          double p[D];
          ld<D>(pts, i, p);
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const double t = sub(p[a], c[a]);
            s = add(s, mul(t, t));
          }
          const double d = __dsqrt_rn(s);
          if (d < lim || (seam > 0.0 && i < n_seeds && seed_regular && seed_regular[i] && d < seam)) {
            good = false;
            break;
          }
        }
      }
  pass[j] = good;
}

// In-wave conflicts, decided in candidate order (see the file comment).  P: positions of
// the pre-tested candidates in candidate order; the grid indexes positions into P.
template <int D>
__global__ void __launch_bounds__(kResolve) resolve_kernel(Grid G, const int* __restrict__ start,
                                                           const int* __restrict__ items,
                                                           const int64_t* __restrict__ P, int64_t np,
                                                           const double* __restrict__ cand,
                                                           const double* __restrict__ hcand,
                                                           int* __restrict__ state, int* __restrict__ ticket) {
  __shared__ int blk_s;
  __shared__ uint32_t mask_s[kResolve][kResolve / 32];
  __shared__ uint8_t ext_s[kResolve];
  __shared__ uint8_t acc_s[kResolve];
  if (threadIdx.x == 0) blk_s = atomicAdd(ticket, 1);
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blk_s) * kResolve;
  const int64_t j = base + threadIdx.x;
  uint32_t mask[kResolve / 32] = {};
  bool ext = false;
  if (j < np) {
    double c[D];
    ld<D>(cand, P[j], c);
    const double lim = mul(kAccept, hcand[P[j]]);
    int cc[D];
    cell_of<D>(G, c, cc);
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < D; ++a) {
      lo[a] = cc[a] > 0 ? cc[a] - 1 : 0;
      hi[a] = cc[a] + 1 < G.dims[a] ? cc[a] + 1 : G.dims[a] - 1;
    }
    for (int x = lo[0]; x <= hi[0] && !ext; ++x)
      for (int y = lo[1]; y <= hi[1] && !ext; ++y)
        for (int z = (D == 3 ? lo[2] : 0); z <= (D == 3 ? hi[2] : 0) && !ext; ++z) {
          const int64_t lin = D == 3 ? (static_cast<int64_t>(x) * G.dims[1] + y) * G.dims[2] + z
                                     : static_cast<int64_t>(x) * G.dims[1] + y;
          for (int e = start[lin]; e < start[lin + 1]; ++e) {
            const int64_t i = items[e];
            if (i >= j) continue;
            double p[D];
            ld<D>(cand, P[i], p);
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) {
              const double t = sub(p[a], c[a]);
              s = add(s, mul(t, t));
            }
            if (!(__dsqrt_rn(s) < lim)) continue;
            if (i >= base) {
              const int b = static_cast<int>(i - base);
              mask[b >> 5] |= 1u << (b & 31);
            } else {
              int st;
              while ((st = *reinterpret_cast<volatile int*>(state + i)) == 0) __nanosleep(64);
              if (st == 1) {
                ext = true;
                break;
              }
            }
          }
        }
  }
#pragma unroll
  for (int w = 0; w < kResolve / 32; ++w) mask_s[threadIdx.x][w] = mask[w];
  ext_s[threadIdx.x] = ext || j >= np;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t acc[kResolve / 32] = {};
    for (int b = 0; b < kResolve; ++b) {
      bool good = !ext_s[b];
#pragma unroll
      for (int w = 0; w < kResolve / 32; ++w) good = good && !(mask_s[b][w] & acc[w]);
      if (good) acc[b >> 5] |= 1u << (b & 31);
      acc_s[b] = good;
    }
  }
  __syncthreads();
  if (j < np) {
    __threadfence();
    atomicExch(state + j, acc_s[threadIdx.x] ? 1 : 2);
  }
}

__global__ void __launch_bounds__(kThr) flag_accepted_kernel(const int* __restrict__ state, int64_t np,
                                                             uint8_t* __restrict__ flag) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (i < np) flag[i] = state[i] == 1;
}

template <int D>
__global__ void __launch_bounds__(kThr) append_kernel(const int64_t* __restrict__ P, const int64_t* __restrict__ A,
                                                      const int64_t* __restrict__ na, const double* __restrict__ cand,
                                                      const double* __restrict__ hcand, int64_t count,
                                                      double* __restrict__ pts, double* __restrict__ hs) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (r >= *na) return;
  const int64_t s = P[A[r]];
#pragma unroll
  for (int a = 0; a < D; ++a) pts[(count + r) * D + a] = cand[s * D + a];
  hs[count + r] = hcand[s];
}

// lattice map (hybrid_discretize nodegen.py:503-516)
template <int D>
__device__ __forceinline__ int64_t grid_lin(const int64_t* cells1, const int64_t* key) {
  int64_t lin = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) lin = lin * cells1[a] + key[a];
  return lin;
}

struct MapDims {
  int64_t cells1[3];  // cells_a + 1
  double origin[3], step[3];
};

template <int D>
__global__ void __launch_bounds__(kThr) map_regular_kernel(MapDims M, const int64_t* __restrict__ keys, int64_t n,
                                                           int64_t* __restrict__ grid) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (i < n) grid[grid_lin<D>(M.cells1, keys + i * D)] = i;
}

template <int D>
__device__ bool on_lattice(const MapDims& M, const double* p, double tol, int64_t* key) {
  bool on = true;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double f = dvd(sub(p[a], M.origin[a]), M.step[a]);
    const double r = rint(f);  // np.round: half to even
    key[a] = static_cast<int64_t>(r);
    on = on && mul(fabs(sub(f, r)), M.step[a]) < tol;
    on = on && key[a] >= 0 && key[a] < M.cells1[a];
  }
  return on;
}

template <int D>
__global__ void __launch_bounds__(kThr) map_boundary_kernel(MapDims M, double tol, const double* __restrict__ bpos,
                                                            int64_t nb, int64_t b0, int64_t n_reg,
                                                            unsigned long long* __restrict__ grid) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (i >= nb) return;
  double p[D];
  ld<D>(bpos, i, p);
  int64_t key[D];
  if (!on_lattice<D>(M, p, tol, key)) return;
  // vacant keys hold INT64_MAX here; regular ids (< n_reg <= b0) are never displaced
  atomicMin(grid + grid_lin<D>(M.cells1, key), static_cast<unsigned long long>(b0 + i));
  (void)n_reg;
}

template <int D>
__global__ void __launch_bounds__(kThr) map_finish_kernel(MapDims M, double tol, const double* __restrict__ bpos,
                                                          int64_t nb, int64_t b0, const int64_t* __restrict__ grid,
                                                          int64_t* __restrict__ out_bkey) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (i >= nb) return;
  double p[D];
  ld<D>(bpos, i, p);
  int64_t key[D];
  const bool won = on_lattice<D>(M, p, tol, key) && grid[grid_lin<D>(M.cells1, key)] == b0 + i;
#pragma unroll
  for (int a = 0; a < D; ++a) out_bkey[i * D + a] = won ? key[a] : INT64_MIN;
}

__global__ void __launch_bounds__(kThr) fill_i64_kernel(int64_t* __restrict__ a, int64_t n, int64_t v) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (i < n) a[i] = v;
}

__global__ void __launch_bounds__(kThr) vacant_kernel(int64_t* __restrict__ a, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (i < n && a[i] == INT64_MAX) a[i] = -1;
}

inline unsigned blocks(int64_t n, int t = kThr) { return static_cast<unsigned>(ceil_div(n > 0 ? n : 1, t)); }

// Scratch kept for the life of one call (released on every return path).
struct Scratch {
  cudaStream_t s;
  static constexpr int kMax = 32;
  void* p[kMax] = {};
  int n = 0;
  explicit Scratch(cudaStream_t st) : s(st) {}
  template <class T>
  cudaError_t get(T** out, size_t count) {
    void* q = nullptr;
    if (n == kMax) return cudaErrorMemoryAllocation;
    cudaError_t e = stream_alloc(&q, sizeof(T) * (count ? count : 1), s);
    if (e == cudaSuccess) p[n++] = q;
    *out = static_cast<T*>(q);
    return e;
  }
  ~Scratch() {
    for (int i = 0; i < n; ++i) cudaFreeAsync(p[i], s);
  }
};

// Build the CSR grid of n points (pts[sel[i]] or pts[i]); start (ncells+1), items (n).
template <int D>
cudaError_t build_grid(const Grid& G, const double* pts, const int64_t* sel, int64_t n, Scratch& S, int** start,
                       int** items, cudaStream_t s) {
  int *cnt, *cell, *cursor;
  cudaError_t e;
  if ((e = S.get(&cnt, G.ncells + 1)) != cudaSuccess) return e;
  if ((e = S.get(start, G.ncells + 1)) != cudaSuccess) return e;
  if ((e = S.get(&cursor, G.ncells + 1)) != cudaSuccess) return e;
  if ((e = S.get(&cell, n)) != cudaSuccess) return e;
  if ((e = S.get(items, n)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(cnt, 0, sizeof(int) * (G.ncells + 1), s)) != cudaSuccess) return e;
  if (n) grid_count_kernel<D><<<blocks(n), kThr, 0, s>>>(G, pts, sel, n, cnt, cell);
  size_t tmp = 0;
  if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, *start, G.ncells + 1, s)) != cudaSuccess) return e;
  void* t;
  if ((e = S.get(reinterpret_cast<char**>(&t), tmp)) != cudaSuccess) return e;
  if ((e = cub::DeviceScan::ExclusiveSum(t, tmp, cnt, *start, G.ncells + 1, s)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(cursor, *start, sizeof(int) * (G.ncells + 1), cudaMemcpyDeviceToDevice, s)) !=
      cudaSuccess)
    return e;
  if (n) grid_fill_kernel<<<blocks(n), kThr, 0, s>>>(cell, n, cursor, *items);
  return cudaGetLastError();
}

// Order-preserving selection of the flagged indices 0..n-1 into out; *count on the device.
cudaError_t select_flagged(const uint8_t* flags, int64_t n, int64_t* out, int64_t* count, Scratch& S,
                           cudaStream_t s) {
  cub::CountingInputIterator<int64_t> it(0);
  size_t tmp = 0;
  cudaError_t e = cub::DeviceSelect::Flagged(nullptr, tmp, it, flags, out, count, n, s);
  if (e != cudaSuccess) return e;
  char* t;
  if ((e = S.get(&t, tmp)) != cudaSuccess) return e;
  return cub::DeviceSelect::Flagged(t, tmp, it, flags, out, count, n, s);
}

template <int D>
int front_accept(double* pts, double* hs, int64_t count, int64_t capacity, const uint8_t* seed_regular,
                 int64_t n_seeds, const double* cand, const double* hcand, const uint8_t* ok, int64_t m, double seam,
                 const double* lo, const double* hi, double cell, int64_t* new_count, cudaStream_t s) {
  if (count + m > capacity) return 3;
  Grid G{};
  G.inv = 1.0 / cell;
  G.ncells = 1;
  for (int a = 0; a < D; ++a) {
    G.lo[a] = lo[a];
    const double ext = (hi[a] - lo[a]) / cell;
    G.dims[a] = static_cast<int>(std::max(1.0, std::floor(ext) + 1.0));
    G.ncells *= G.dims[a];
  }
  if (G.ncells > (int64_t{1} << 30)) return 4;
  Scratch S(s);
  int *start, *items;
  HN_TRY(build_grid<D>(G, pts, nullptr, count, S, &start, &items, s));
  uint8_t* pass;
  int64_t *P, *np_d;
  HN_TRY(S.get(&pass, m));
  HN_TRY(S.get(&P, m));
  HN_TRY(S.get(&np_d, 2));
  if (m) pretest_kernel<D><<<blocks(m), kThr, 0, s>>>(G, start, items, pts, seed_regular, n_seeds, seam, cand, hcand,
                                                       ok, m, pass);
  HN_CHECK_LAUNCH();
  HN_TRY(select_flagged(pass, m, P, np_d, S, s));
  int64_t np = 0;
  HN_TRY(cudaMemcpyAsync(&np, np_d, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  HN_TRY(cudaStreamSynchronize(s));
  if (np == 0) {
    *new_count = count;
    return 0;
  }
  int *cstart, *citems, *state, *ticket;
  // grid over the surviving candidates (positions into P)
  {
    int *cnt, *cellv, *cursor;
    HN_TRY(S.get(&cnt, G.ncells + 1));
    HN_TRY(S.get(&cstart, G.ncells + 1));
    HN_TRY(S.get(&cursor, G.ncells + 1));
    HN_TRY(S.get(&cellv, np));
    HN_TRY(S.get(&citems, np));
    HN_TRY(cudaMemsetAsync(cnt, 0, sizeof(int) * (G.ncells + 1), s));
    grid_count_kernel<D><<<blocks(np), kThr, 0, s>>>(G, cand, P, np, cnt, cellv);
    size_t tmp = 0;
    HN_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, cstart, G.ncells + 1, s));
    char* t;
    HN_TRY(S.get(&t, tmp));
    HN_TRY(cub::DeviceScan::ExclusiveSum(t, tmp, cnt, cstart, G.ncells + 1, s));
    HN_TRY(cudaMemcpyAsync(cursor, cstart, sizeof(int) * (G.ncells + 1), cudaMemcpyDeviceToDevice, s));
    grid_fill_kernel<<<blocks(np), kThr, 0, s>>>(cellv, np, cursor, citems);
    HN_CHECK_LAUNCH();
  }
  HN_TRY(S.get(&state, np));
  HN_TRY(S.get(&ticket, 1));
  HN_TRY(cudaMemsetAsync(state, 0, sizeof(int) * np, s));
  HN_TRY(cudaMemsetAsync(ticket, 0, sizeof(int), s));
  resolve_kernel<D><<<blocks(np, kResolve), kResolve, 0, s>>>(G, cstart, citems, P, np, cand, hcand, state, ticket);
  HN_CHECK_LAUNCH();
  uint8_t* acc;
  int64_t *A, *na_d;
  HN_TRY(S.get(&acc, np));
  HN_TRY(S.get(&A, np));
  HN_TRY(S.get(&na_d, 2));
  flag_accepted_kernel<<<blocks(np), kThr, 0, s>>>(state, np, acc);
  HN_CHECK_LAUNCH();
  HN_TRY(select_flagged(acc, np, A, na_d, S, s));
  append_kernel<D><<<blocks(np), kThr, 0, s>>>(P, A, na_d, cand, hcand, count, pts, hs);
  HN_CHECK_LAUNCH();
  int64_t na = 0;
  HN_TRY(cudaMemcpyAsync(&na, na_d, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  HN_TRY(cudaStreamSynchronize(s));
  *new_count = count + na;
  return 0;
}

bool geom_ok(const hn_geom* g) {
  return g && (g->dim == 2 || g->dim == 3) && g->n_obs >= 0 && (g->n_obs == 0 || (g->obs_kind && g->obs_par));
}

}  // namespace
}  // namespace hn

using namespace hn;

HN_EXPORT int hn_geom_eval(const hn_geom* g, const double* pts, int64_t n, int mode, double* out, void* stream) {
  if (!geom_ok(g) || mode < 0 || mode > 5) return 1;
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  if (g->dim == 2)
    geom_eval_kernel<2><<<blocks(n), kThr, 0, s>>>(*g, pts, n, mode, out);
  else
    geom_eval_kernel<3><<<blocks(n), kThr, 0, s>>>(*g, pts, n, mode, out);
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT int hn_lattice_fill(const hn_geom* g, const int64_t* cells_host, const double* step_host, double thr,
                              int drop_region, double carve, double* out_pos, int64_t* out_key,
                              int64_t* out_count_host, void* stream) {
  if (!geom_ok(g) || !cells_host || !step_host || !out_count_host) return 1;
  cudaStream_t s = as_stream(stream);
  const int D = g->dim;
  LatticeDims L{};
  int64_t total = 1;
  for (int a = 0; a < D; ++a) {
    L.n[a] = cells_host[a] - 1;
    L.step[a] = step_host[a];
    total *= L.n[a] > 0 ? L.n[a] : 0;
  }
  *out_count_host = 0;
  if (total <= 0) return 0;
  Scratch S(s);
  uint8_t* keep;
  int64_t *ids, *cnt;
  HN_TRY(S.get(&keep, total));
  HN_TRY(S.get(&ids, total));
  HN_TRY(S.get(&cnt, 2));
  if (D == 2)
    lattice_flag_kernel<2><<<blocks(total), kThr, 0, s>>>(*g, L, total, thr, drop_region, carve, keep);
  else
    lattice_flag_kernel<3><<<blocks(total), kThr, 0, s>>>(*g, L, total, thr, drop_region, carve, keep);
  HN_CHECK_LAUNCH();
  HN_TRY(select_flagged(keep, total, ids, cnt, S, s));
  if (D == 2)
    lattice_gather_kernel<2><<<blocks(total), kThr, 0, s>>>(*g, L, ids, cnt, out_pos, out_key);
  else
    lattice_gather_kernel<3><<<blocks(total), kThr, 0, s>>>(*g, L, ids, cnt, out_pos, out_key);
  HN_CHECK_LAUNCH();
  HN_TRY(cudaMemcpyAsync(out_count_host, cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  HN_TRY(cudaStreamSynchronize(s));
  return 0;
}

HN_EXPORT int hn_front_candidates(const hn_geom* g, const double* pts, const double* hs, const int64_t* front,
                                  int64_t front_lo, int64_t k, const double* rnd, const double* u, int use_region,
                                  double* cand, double* hcand, uint8_t* ok, void* stream) {
  if (!geom_ok(g) || k < 0) return 1;
  if (k == 0) return 0;
  cudaStream_t s = as_stream(stream);
  const int64_t m = k * (3 * g->dim + 1);
  if (g->dim == 2)
    candidates_kernel<2><<<blocks(m), kThr, 0, s>>>(*g, pts, hs, front, front_lo, k, rnd, u, use_region, cand, hcand,
                                                     ok);
  else
    candidates_kernel<3><<<blocks(m), kThr, 0, s>>>(*g, pts, hs, front, front_lo, k, rnd, u, use_region, cand, hcand,
                                                     ok);
  HN_CHECK_LAUNCH();
  return 0;
}

HN_EXPORT int hn_front_accept(int d, double* pts, double* hs, int64_t count, int64_t capacity,
                              const uint8_t* seed_regular, int64_t n_seeds, const double* cand, const double* hcand,
                              const uint8_t* ok, int64_t m, double seam, const double* lo_host, const double* hi_host,
                              double cell, int64_t* new_count_host, void* stream) {
  if ((d != 2 && d != 3) || !lo_host || !hi_host || !new_count_host || !(cell > 0.0) || m < 0 || count < 0) return 1;
  cudaStream_t s = as_stream(stream);
  return d == 2 ? front_accept<2>(pts, hs, count, capacity, seed_regular, n_seeds, cand, hcand, ok, m, seam, lo_host,
                                  hi_host, cell, new_count_host, s)
                : front_accept<3>(pts, hs, count, capacity, seed_regular, n_seeds, cand, hcand, ok, m, seam, lo_host,
                                  hi_host, cell, new_count_host, s);
}

HN_EXPORT int hn_lattice_map(int d, const int64_t* cells_host, const double* origin_host, const double* step_host,
                             double tol, const int64_t* keys, int64_t n_reg, const double* bpos, int64_t n_b,
                             int64_t b0, int64_t* grid, int64_t* out_bkey, void* stream) {
  if ((d != 2 && d != 3) || !cells_host || !origin_host || !step_host || !grid) return 1;
  cudaStream_t s = as_stream(stream);
  MapDims M{};
  int64_t total = 1;
  for (int a = 0; a < d; ++a) {
    M.cells1[a] = cells_host[a] + 1;
    M.origin[a] = origin_host[a];
    M.step[a] = step_host[a];
    total *= M.cells1[a];
  }
  fill_i64_kernel<<<blocks(total), kThr, 0, s>>>(grid, total, INT64_MAX);
  if (n_reg > 0) {
    if (d == 2)
      map_regular_kernel<2><<<blocks(n_reg), kThr, 0, s>>>(M, keys, n_reg, grid);
    else
      map_regular_kernel<3><<<blocks(n_reg), kThr, 0, s>>>(M, keys, n_reg, grid);
  }
  if (n_b > 0) {
    auto* ug = reinterpret_cast<unsigned long long*>(grid);
    if (d == 2) {
      map_boundary_kernel<2><<<blocks(n_b), kThr, 0, s>>>(M, tol, bpos, n_b, b0, n_reg, ug);
      map_finish_kernel<2><<<blocks(n_b), kThr, 0, s>>>(M, tol, bpos, n_b, b0, grid, out_bkey);
    } else {
      map_boundary_kernel<3><<<blocks(n_b), kThr, 0, s>>>(M, tol, bpos, n_b, b0, n_reg, ug);
      map_finish_kernel<3><<<blocks(n_b), kThr, 0, s>>>(M, tol, bpos, n_b, b0, grid, out_bkey);
    }
  }
  vacant_kernel<<<blocks(total), kThr, 0, s>>>(grid, total);
  HN_CHECK_LAUNCH();
  return 0;
}

// NodeSet.min_distance_violations nodegen.py:139-148: pairs i < j with
// |x_i - x_j| < 0.5 min(h_i, h_j) - 1e-12 (cell >= 0.5 max h: a 3^d window is exact).
namespace hn {
namespace {
template <int D>
__global__ void __launch_bounds__(kThr) close_pairs_kernel(Grid G, const int* __restrict__ start,
                                                           const int* __restrict__ items,
                                                           const double* __restrict__ pts,
                                                           const double* __restrict__ h, int64_t n,
                                                           unsigned long long* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kThr + threadIdx.x;
  if (i >= n) return;
  double c[D];
  ld<D>(pts, i, c);
  const double hi_ = h[i];
  int cc[D];
  cell_of<D>(G, c, cc);
  int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
#pragma unroll
  for (int a = 0; a < D; ++a) {
    lo[a] = cc[a] > 0 ? cc[a] - 1 : 0;
    hi[a] = cc[a] + 1 < G.dims[a] ? cc[a] + 1 : G.dims[a] - 1;
  }
  unsigned long long bad = 0;
  for (int x = lo[0]; x <= hi[0]; ++x)
    for (int y = lo[1]; y <= hi[1]; ++y)
      for (int z = (D == 3 ? lo[2] : 0); z <= (D == 3 ? hi[2] : 0); ++z) {
        const int64_t lin = D == 3 ? (static_cast<int64_t>(x) * G.dims[1] + y) * G.dims[2] + z
                                   : static_cast<int64_t>(x) * G.dims[1] + y;
        for (int e = start[lin]; e < start[lin + 1]; ++e) {
          const int64_t j = items[e];
          if (j <= i) continue;
          double p[D];
          ld<D>(pts, j, p);
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const double t = sub(c[a], p[a]);
            s = add(s, mul(t, t));
          }
          const double hj = h[j];
          bad += __dsqrt_rn(s) < sub(mul(0.5, hi_ < hj ? hi_ : hj), 1e-12);
        }
      }
  if (bad) atomicAdd(out, bad);
}

template <int D>
int close_pairs(const double* pts, const double* h, int64_t n, const double* lo, const double* hi, double cell,
                int64_t* out, cudaStream_t s) {
  Grid G{};
  G.inv = 1.0 / cell;
  G.ncells = 1;
  for (int a = 0; a < D; ++a) {
    G.lo[a] = lo[a];
    G.dims[a] = static_cast<int>(std::max(1.0, std::min(std::floor((hi[a] - lo[a]) / cell) + 1.0, 4096.0)));
    G.ncells *= G.dims[a];
  }
  if (G.dims[0] >= 4096 || G.dims[1] >= 4096 || (D == 3 && G.dims[2] >= 4096) || G.ncells > (int64_t{1} << 30))
    return 4;
  Scratch S(s);
  int *start, *items;
  HN_TRY(build_grid<D>(G, pts, nullptr, n, S, &start, &items, s));
  unsigned long long* cnt;
  HN_TRY(S.get(&cnt, 1));
  HN_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
  close_pairs_kernel<D><<<blocks(n), kThr, 0, s>>>(G, start, items, pts, h, n, cnt);
  HN_CHECK_LAUNCH();
  unsigned long long v = 0;
  HN_TRY(cudaMemcpyAsync(&v, cnt, sizeof(v), cudaMemcpyDeviceToHost, s));
  HN_TRY(cudaStreamSynchronize(s));
  *out = static_cast<int64_t>(v);
  return 0;
}
}  // namespace
}  // namespace hn

HN_EXPORT int hn_close_pairs(int d, const double* pts, const double* h, int64_t n, const double* lo_host,
                             const double* hi_host, double cell, int64_t* out_count_host, void* stream) {
  if ((d != 2 && d != 3) || !lo_host || !hi_host || !out_count_host || !(cell > 0.0) || n < 0) return 1;
  *out_count_host = 0;
  if (n < 2) return 0;
  cudaStream_t s = as_stream(stream);
  return d == 2 ? close_pairs<2>(pts, h, n, lo_host, hi_host, cell, out_count_host, s)
                : close_pairs<3>(pts, h, n, lo_host, hi_host, cell, out_count_host, s);
}
