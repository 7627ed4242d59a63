// narrow.cu — the narrow phase: elementary DCD / CCD
// feature tests on the broad phase's candidate triangle pairs, merged and
// deduplicated like sync_shared_cells.
//
// Reference: narrow_phase_pair (proj/src/collision.cpp:214-309), the
// elementary tests and the cubic solver (proj/src/collision_geom.cpp:
// 35-317), sort_dedup / sync_shared_cells (collision.cpp:313-325,380-389),
// collide (:391-417). Every expression keeps the reference's association
// (Vec3 algebra of oracle/shim/Eigen/Dense: strict left-to-right 3-term
// reductions) and the library is built with -fmad=false; the operations are
// IEEE +, -, *, /, sqrt, so hits are bitwise the reference's.
//
// Device pipeline: build_grid -> candidate walk (pairs written) -> one
// thread per candidate pair runs the 6 vertex-face and 9 edge-edge tests
// and appends hits (key = kind<<62 | a<<31 | b, 8 doubles) -> CUB radix sort
// by key -> keep the first of equal keys (duplicates come from different
// triangle pairs sharing a feature pair and are identical).
#include <cub/cub.cuh>

#include <algorithm>
#include <unordered_map>
#include <vector>

#include "ctx.cuh"
#include "elements.cuh"

namespace weft_gpu {
namespace {

constexpr double kBaryEps = 1e-8;        // collision_geom.cpp:9
constexpr double kRootClampEps = 1e-12;  // collision_geom.cpp:10

__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }  // std::min
__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }  // std::max
__device__ __forceinline__ double dclamp(double v, double lo, double hi) {            // std::clamp
  return v < lo ? lo : (hi < v ? hi : v);
}
__device__ __forceinline__ V3 neg(V3 a) { return V3{-a.x, -a.y, -a.z}; }
__device__ __forceinline__ double sqn(V3 a) { return dot(a, a); }
__device__ __forceinline__ V3 lerp3(V3 a, V3 b, double t) { return add(a, scl(t, sub(b, a))); }
__device__ __forceinline__ V3 ldx(const double* __restrict__ x, int v) {
  return V3{x[3 * v], x[3 * v + 1], x[3 * v + 2]};
}

// Eigen's unitOrthogonal for 3-vectors, as oracle/shim/Eigen/Dense.
__device__ __forceinline__ V3 unit_orthogonal(V3 s) {
  const double prec = 1e-12;
  if (!(fabs(s.x) <= fabs(s.z) * prec) || !(fabs(s.y) <= fabs(s.z) * prec)) {
    const double invnm = 1.0 / sqrt(s.x * s.x + s.y * s.y);
    return V3{-s.y * invnm, s.x * invnm, 0.0};
  }
  const double invnm = 1.0 / sqrt(s.y * s.y + s.z * s.z);
  return V3{0.0, -s.z * invnm, s.y * invnm};
}

struct Hit {
  double s;  // gap (DCD) or toi (CCD)
  V3 n;
  double w[4];
};

__device__ __forceinline__ double poly_eval(double c3, double c2, double c1, double c0, double t) {
  return ((c3 * t + c2) * t + c1) * t + c0;
}

// bisect_root (collision_geom.cpp:17-31).
__device__ double bisect_root(double c3, double c2, double c1, double c0, double lo, double hi) {
  double flo = poly_eval(c3, c2, c1, c0, lo);
  for (int it = 0; it < 90; ++it) {
    const double mid = 0.5 * (lo + hi);
    const double fm = poly_eval(c3, c2, c1, c0, mid);
    if (fm == 0.0) return mid;
    if ((flo < 0.0) == (fm < 0.0)) {
      lo = mid;
      flo = fm;
    } else {
      hi = mid;
    }
  }
  return 0.5 * (lo + hi);
}

// cubic_roots_in_unit_interval (collision_geom.cpp:35-88). -1 = identically zero.
__device__ int cubic_roots(double c3, double c2, double c1, double c0, double roots[3]) {
  const double scale = dmax(dmax(dmax(fabs(c3), fabs(c2)), fabs(c1)), fabs(c0));
  if (scale == 0.0) return -1;
  c3 = c3 / scale;
  c2 = c2 / scale;
  c1 = c1 / scale;
  c0 = c0 / scale;
  double bp[4] = {0.0, 1.0, 0.0, 0.0};
  int nbp = 2;
  const double qa = 3.0 * c3, qb = 2.0 * c2, qc = c1;
  if (fabs(qa) > 1e-14) {
    const double disc = qb * qb - 4.0 * qa * qc;
    if (disc > 0.0) {
      const double sq = sqrt(disc);
      const double q = -0.5 * (qb + (qb >= 0.0 ? sq : -sq));
      const double t0 = q / qa, t1 = qc / q;
      if (t0 > 0.0 && t0 < 1.0) bp[nbp++] = t0;
      if (t1 > 0.0 && t1 < 1.0) bp[nbp++] = t1;
    }
  } else if (fabs(qb) > 1e-14) {
    const double t = -qc / qb;
    if (t > 0.0 && t < 1.0) bp[nbp++] = t;
  }
  for (int i = 1; i < nbp; ++i)  // std::sort of <= 4 breakpoints
    for (int j = i; j > 0 && bp[j] < bp[j - 1]; --j) {
      const double t = bp[j];
      bp[j] = bp[j - 1];
      bp[j - 1] = t;
    }
  int count = 0;
  for (int k = 0; k + 1 < nbp; ++k) {
    const double lo = bp[k], hi = bp[k + 1];
    if (hi - lo < 1e-15) continue;
    const double flo = poly_eval(c3, c2, c1, c0, lo);
    const double fhi = poly_eval(c3, c2, c1, c0, hi);
    double root = -1.0;
    if (flo == 0.0) {
      root = lo;
    } else if ((flo < 0.0) != (fhi <= 0.0)) {
      root = bisect_root(c3, c2, c1, c0, lo, hi);
    } else if (fhi == 0.0 && k + 2 == nbp) {
      root = hi;
    }
    if (root >= -kRootClampEps && root <= 1.0 + kRootClampEps) {
      root = dmin(1.0, dmax(0.0, root));
      if (count == 0 || fabs(roots[count - 1] - root) > 1e-14) roots[count++] = root;
    }
  }
  return count;
}

// dcd_vertex_face (collision_geom.cpp:90-162): closest point on the
// triangle (Ericson), hit iff the distance is < h.
__device__ bool dcd_vf(V3 v, V3 a, V3 b, V3 c, double h, Hit& hit) {
  const V3 ab = sub(b, a), ac = sub(c, a), av = sub(v, a);
  const double d1 = dot(ab, av), d2 = dot(ac, av);
  V3 cp;
  double b0, b1, b2;
  if (d1 <= 0.0 && d2 <= 0.0) {
    cp = a;
    b0 = 1;
    b1 = 0;
    b2 = 0;
  } else {
    const V3 bv = sub(v, b);
    const double d3 = dot(ab, bv), d4 = dot(ac, bv);
    if (d3 >= 0.0 && d4 <= d3) {
      cp = b;
      b0 = 0;
      b1 = 1;
      b2 = 0;
    } else {
      const double vc = d1 * d4 - d3 * d2;
      if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
        const double w = d1 / (d1 - d3);
        cp = add(a, scl(w, ab));
        b0 = 1 - w;
        b1 = w;
        b2 = 0;
      } else {
        const V3 cv = sub(v, c);
        const double d5 = dot(ab, cv), d6 = dot(ac, cv);
        if (d6 >= 0.0 && d5 <= d6) {
          cp = c;
          b0 = 0;
          b1 = 0;
          b2 = 1;
        } else {
          const double vb = d5 * d2 - d1 * d6;
          if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
            const double w = d2 / (d2 - d6);
            cp = add(a, scl(w, ac));
            b0 = 1 - w;
            b1 = 0;
            b2 = w;
          } else {
            const double va = d3 * d6 - d5 * d4;
            if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
              const double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
              cp = add(b, scl(w, sub(c, b)));
              b0 = 0;
              b1 = 1 - w;
              b2 = w;
            } else {
              const double denom = 1.0 / ((va + vb) + vc);
              const double wb = vb * denom, wc = vc * denom;
              cp = add(add(a, scl(wb, ab)), scl(wc, ac));
              b0 = (1.0 - wb) - wc;
              b1 = wb;
              b2 = wc;
            }
          }
        }
      }
    }
  }
  const V3 diff = sub(v, cp);
  const double dist = norm(diff);
  if (!(dist < h)) return false;  // dist >= h (NaN never hits either way)
  hit.s = dist;
  if (dist > 1e-12) {
    hit.n = divs(diff, dist);
  } else {
    const V3 n = cross(ab, ac);
    const double len = norm(n);
    if (len > 1e-16) {
      hit.n = divs(n, len);
    } else {
      const V3 d = sqn(ab) > sqn(ac) ? ab : ac;
      hit.n = unit_orthogonal(d);
    }
  }
  hit.w[0] = 1.0;
  hit.w[1] = b0;
  hit.w[2] = b1;
  hit.w[3] = b2;
  return true;
}

// dcd_edge_edge (collision_geom.cpp:164-213).
__device__ bool dcd_ee(V3 p1, V3 p2, V3 q1, V3 q2, double h, Hit& hit) {
  const V3 d1 = sub(p2, p1), d2 = sub(q2, q1), r = sub(p1, q1);
  const double a = sqn(d1), e = sqn(d2), f = dot(d2, r);
  double s = 0.0, t = 0.0;
  if (a <= 1e-18 && e <= 1e-18) {
  } else if (a <= 1e-18) {
    t = dclamp(f / e, 0.0, 1.0);
  } else {
    const double c = dot(d1, r);
    if (e <= 1e-18) {
      s = dclamp(-c / a, 0.0, 1.0);
    } else {
      const double b = dot(d1, d2);
      const double denom = a * e - b * b;
      s = denom > 1e-18 ? dclamp((b * f - c * e) / denom, 0.0, 1.0) : 0.0;
      t = (b * s + f) / e;
      if (t < 0.0) {
        t = 0.0;
        s = dclamp(-c / a, 0.0, 1.0);
      } else if (t > 1.0) {
        t = 1.0;
        s = dclamp((b - c) / a, 0.0, 1.0);
      }
    }
  }
  const V3 cp = add(p1, scl(s, d1));
  const V3 cq = add(q1, scl(t, d2));
  const V3 diff = sub(cp, cq);
  const double dist = norm(diff);
  if (!(dist < h)) return false;
  hit.s = dist;
  if (dist > 1e-12) {
    hit.n = divs(diff, dist);
  } else {
    const V3 n = cross(d1, d2);
    const double len = norm(n);
    if (len > 1e-16) {
      hit.n = divs(n, len);
    } else {
      const V3 d = sqn(d1) > sqn(d2) ? d1 : d2;
      hit.n = sqn(d) > 1e-18 ? unit_orthogonal(d) : V3{1, 0, 0};
    }
  }
  hit.w[0] = 1.0 - s;
  hit.w[1] = s;
  hit.w[2] = 1.0 - t;
  hit.w[3] = t;
  return true;
}

// triple_product_cubic (collision_geom.cpp:219-227).
__device__ __forceinline__ void triple_cubic(V3 u0, V3 du, V3 v0, V3 dv, V3 w0, V3 dw, double& c3, double& c2,
                                             double& c1, double& c0) {
  c0 = dot(cross(u0, v0), w0);
  c1 = (dot(cross(du, v0), w0) + dot(cross(u0, dv), w0)) + dot(cross(u0, v0), dw);
  c2 = (dot(cross(du, dv), w0) + dot(cross(du, v0), dw)) + dot(cross(u0, dv), dw);
  c3 = dot(cross(du, dv), dw);
}

// ccd_vertex_face (collision_geom.cpp:231-272).
__device__ bool ccd_vf(V3 v0, V3 v1, V3 a0, V3 a1, V3 b0, V3 b1, V3 c0v, V3 c1v, Hit& out) {
  const V3 u0 = sub(b0, a0), du = sub(sub(b1, a1), u0);
  const V3 w0 = sub(c0v, a0), dw = sub(sub(c1v, a1), w0);
  const V3 q0 = sub(v0, a0), dq = sub(sub(v1, a1), q0);
  double c3, c2, c1, c0;
  triple_cubic(u0, du, w0, dw, q0, dq, c3, c2, c1, c0);
  double roots[3];
  int count = cubic_roots(c3, c2, c1, c0, roots);
  if (count < 0) {
    roots[0] = 0.0;
    roots[1] = 0.5;
    roots[2] = 1.0;
    count = 3;
  }
  for (int k = 0; k < count; ++k) {
    const double t = roots[k];
    const V3 v = lerp3(v0, v1, t), a = lerp3(a0, a1, t), b = lerp3(b0, b1, t), c = lerp3(c0v, c1v, t);
    Hit hit;
    if (!dcd_vf(v, a, b, c, 1e100, hit)) continue;
    const double scale = dmax(dmax(norm(sub(b, a)), norm(sub(c, a))), 1e-12);
    if (hit.s > 1e-9 * scale) continue;
    V3 n = cross(sub(b, a), sub(c, a));
    const double len = norm(n);
    n = len > 1e-16 ? divs(n, len) : hit.n;
    const V3 cp0 = add(add(scl(hit.w[1], a0), scl(hit.w[2], b0)), scl(hit.w[3], c0v));
    if (dot(n, sub(v0, cp0)) < 0.0) n = neg(n);
    out.s = t;
    out.n = n;
    for (int q = 0; q < 4; ++q) out.w[q] = hit.w[q];
    return true;
  }
  return false;
}

// ccd_edge_edge (collision_geom.cpp:274-317).
__device__ bool ccd_ee(V3 p10, V3 p11, V3 p20, V3 p21, V3 q10, V3 q11, V3 q20, V3 q21, Hit& out) {
  const V3 u0 = sub(p20, p10), du = sub(sub(p21, p11), u0);
  const V3 v0 = sub(q20, q10), dv = sub(sub(q21, q11), v0);
  const V3 w0 = sub(q10, p10), dw = sub(sub(q11, p11), w0);
  double c3, c2, c1, c0;
  triple_cubic(u0, du, v0, dv, w0, dw, c3, c2, c1, c0);
  double roots[3];
  int count = cubic_roots(c3, c2, c1, c0, roots);
  if (count < 0) {
    roots[0] = 0.0;
    roots[1] = 0.5;
    roots[2] = 1.0;
    count = 3;
  }
  for (int k = 0; k < count; ++k) {
    const double t = roots[k];
    const V3 p1 = lerp3(p10, p11, t), p2 = lerp3(p20, p21, t);
    const V3 q1 = lerp3(q10, q11, t), q2 = lerp3(q20, q21, t);
    Hit hit;
    if (!dcd_ee(p1, p2, q1, q2, 1e100, hit)) continue;
    const double scale = dmax(dmax(norm(sub(p2, p1)), norm(sub(q2, q1))), 1e-12);
    if (hit.s > 1e-9 * scale) continue;
    const double s = hit.w[1], u = hit.w[3];
    if (s < -kBaryEps || s > 1.0 + kBaryEps || u < -kBaryEps || u > 1.0 + kBaryEps) continue;
    V3 n = cross(sub(p2, p1), sub(q2, q1));
    const double len = norm(n);
    if (len < 1e-16) n = hit.n;
    else n = divs(n, len);
    const V3 cp0 = add(scl(1.0 - s, p10), scl(s, p20));
    const V3 cq0 = add(scl(1.0 - u, q10), scl(u, q20));
    if (dot(n, sub(cp0, cq0)) < 0.0) n = neg(n);
    out.s = t;
    out.n = n;
    for (int q = 0; q < 4; ++q) out.w[q] = hit.w[q];
    return true;
  }
  return false;
}

struct NarrowArgs {
  int64_t npairs;
  const int2* __restrict__ pairs;
  const int32_t* __restrict__ tris;       // 3 per triangle
  const int32_t* __restrict__ tri_edges;  // 3 per triangle
  const int2* __restrict__ edges;
  const uint8_t* __restrict__ movable;
  const double* __restrict__ x0;
  const double* __restrict__ x1;
  bool ccd;
  double thickness;
  unsigned long long* __restrict__ keys;  // kind << 62 | a << 31 | b
  double* __restrict__ vals;              // 8 per hit
  unsigned long long* __restrict__ count;
  unsigned long long cap;
  const float4* __restrict__ tbox;  // per triangle: (lo xyz, -) (hi xyz, -), rounded outward
  const double* __restrict__ vbox;  // per vertex: lo xyz, hi xyz over begin (and end) positions (exact)
  const double* __restrict__ dbox;  // per triangle: the same over its 3 vertices (exact)
  // two-pass narrow phase: features that survive their box test, as
  // {kind, a, b, v0} {v1, v2, v3, 0} (a, b = the hit key's ids; v = the
  // feature's vertices), claimed from *feat_count; entries at or beyond
  // feat_cap are dropped and the host re-runs with the exact count
  int4* __restrict__ feats;
  unsigned long long* __restrict__ feat_count;
  unsigned long long feat_cap;
};

// Per-triangle box over the 3 vertices (begin and, for CCD, end positions),
// rounded outward to float: a conservative stand-in for the exact box in the
// whole-pair rejection of k_narrow (lo rounds down, hi rounds up, and
// hi + margin rounds monotonically, so "apart" on the float boxes implies
// apart on the exact ones).
__global__ void k_tri_fbox(int ntris, const int32_t* __restrict__ tris, const double* __restrict__ x0,
                           const double* __restrict__ x1, bool ccd, float4* __restrict__ out,
                           double* __restrict__ dbox) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntris) return;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int k = 0; k < 3; ++k) {
    const int v = tris[3 * t + k];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double p0 = x0[3 * v + a];
      lo[a] = dmin(lo[a], p0);
      hi[a] = dmax(hi[a], p0);
      if (ccd) {
        const double p1 = x1[3 * v + a];
        lo[a] = dmin(lo[a], p1);
        hi[a] = dmax(hi[a], p1);
      }
    }
  }
  out[2 * t] = make_float4(__double2float_rd(lo[0]), __double2float_rd(lo[1]), __double2float_rd(lo[2]), 0.f);
  out[2 * t + 1] = make_float4(__double2float_ru(hi[0]), __double2float_ru(hi[1]), __double2float_ru(hi[2]), 0.f);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    dbox[6 * t + a] = lo[a];
    dbox[6 * t + 3 + a] = hi[a];
  }
}

// Per-vertex box over its begin (and, for CCD, end) position, with the
// sentinels of the reference's feature_apart (collision.cpp:226-254, running
// std::min / std::max from +-1e300): dmin / dmax ignore a NaN second operand
// and never return one here, so combining these boxes (and the triangle
// boxes of k_tri_fbox) gives exactly the lo / hi that running min / max over
// the feature's positions gives, for any input.
__global__ void k_vert_box(int nverts, const double* __restrict__ x0, const double* __restrict__ x1, bool ccd,
                           double* __restrict__ vbox) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nverts) return;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double lo = dmin(1e300, x0[3 * v + a]), hi = dmax(-1e300, x0[3 * v + a]);
    if (ccd) {
      lo = dmin(lo, x1[3 * v + a]);
      hi = dmax(hi, x1[3 * v + a]);
    }
    vbox[6 * v + a] = lo;
    vbox[6 * v + 3 + a] = hi;
  }
}

// feature_apart (collision.cpp:226-254) on precomputed exact boxes: box a =
// the min / max of the boxes at pa[0..NA), box b likewise; apart when some
// axis separates them by more than the margin.
template <int NA, int NB>
__device__ __forceinline__ bool boxes_apart_d(const double* const (&pa)[NA], const double* const (&pb)[NB],
                                              double margin) {
#pragma unroll
  for (int axis = 0; axis < 3; ++axis) {
    double lo_a = __ldg(pa[0] + axis), hi_a = __ldg(pa[0] + 3 + axis);
#pragma unroll
    for (int k = 1; k < NA; ++k) {
      lo_a = dmin(lo_a, __ldg(pa[k] + axis));
      hi_a = dmax(hi_a, __ldg(pa[k] + 3 + axis));
    }
    double lo_b = __ldg(pb[0] + axis), hi_b = __ldg(pb[0] + 3 + axis);
#pragma unroll
    for (int k = 1; k < NB; ++k) {
      lo_b = dmin(lo_b, __ldg(pb[k] + axis));
      hi_b = dmax(hi_b, __ldg(pb[k] + 3 + axis));
    }
    if (lo_a > hi_b + margin || lo_b > hi_a + margin) return true;
  }
  return false;
}

__device__ __forceinline__ void emit(const NarrowArgs& g, int kind, int a, int b, const Hit& h) {
  const unsigned long long slot = atomicAdd(g.count, 1ull);
  if (slot >= g.cap) return;  // host re-runs with the exact capacity
  g.keys[slot] = (static_cast<unsigned long long>(kind) << 62) | (static_cast<unsigned long long>(a) << 31) |
                 static_cast<unsigned long long>(b);
  double* o = g.vals + 8 * slot;
  o[0] = h.s;
  o[1] = h.n.x;
  o[2] = h.n.y;
  o[3] = h.n.z;
  o[4] = h.w[0];
  o[5] = h.w[1];
  o[6] = h.w[2];
  o[7] = h.w[3];
}

// narrow_phase_pair (collision.cpp:214-309), one thread per candidate pair.
// Compiled once per mode (kCcd): the DCD instance carries none of the
// cubic-solver registers (150 -> fewer registers, higher occupancy).
template <bool kCcd>
__global__ void __launch_bounds__(128) k_narrow(NarrowArgs g) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= g.npairs) return;
  const int2 pr = g.pairs[i];
  const int t1 = pr.x, t2 = pr.y;
  const double margin0 = kCcd ? 1e-9 : g.thickness;
  {  // whole-pair rejection on the conservative float boxes (k_tri_fbox)
    const float4 la = __ldg(g.tbox + 2 * t1), ha = __ldg(g.tbox + 2 * t1 + 1);
    const float4 lb = __ldg(g.tbox + 2 * t2), hb = __ldg(g.tbox + 2 * t2 + 1);
    if ((double)la.x > (double)hb.x + margin0 || (double)lb.x > (double)ha.x + margin0 ||
        (double)la.y > (double)hb.y + margin0 || (double)lb.y > (double)ha.y + margin0 ||
        (double)la.z > (double)hb.z + margin0 || (double)lb.z > (double)ha.z + margin0)
      return;
  }
  const int tri1[3] = {g.tris[3 * t1], g.tris[3 * t1 + 1], g.tris[3 * t1 + 2]};
  const int tri2[3] = {g.tris[3 * t2], g.tris[3 * t2 + 1], g.tris[3 * t2 + 2]};
  const double margin = kCcd ? 1e-9 : g.thickness;
  // Whole-pair rejection: every feature of a triangle has a box inside the
  // triangle's box (min / max are exact and x + margin rounds monotonically),
  // so triangle boxes apart by more than the margin imply that all 15
  // feature_apart tests below reject — same hits, far less work.
  {
    const double* const ta[1] = {g.dbox + 6 * (size_t)t1};
    const double* const tb[1] = {g.dbox + 6 * (size_t)t2};
    if (boxes_apart_d(ta, tb, margin)) return;
  }
  // vertex-face, both directions; shared vertices are exempt
  for (int dir = 0; dir < 2; ++dir) {
    const int* vt = dir == 0 ? tri1 : tri2;
    const int* ft = dir == 0 ? tri2 : tri1;
    const int face_id = dir == 0 ? t2 : t1;
    for (int k = 0; k < 3; ++k) {
      const int v = vt[k];
      if (ft[0] == v || ft[1] == v || ft[2] == v) continue;
      if (!g.movable[v] && !g.movable[ft[0]] && !g.movable[ft[1]] && !g.movable[ft[2]]) continue;
      const double* const fa[1] = {g.vbox + 6 * (size_t)v};
      const double* const fb[1] = {g.dbox + 6 * (size_t)face_id};
      if (boxes_apart_d(fa, fb, margin)) continue;
      Hit h;
      bool hit;
      if (!kCcd) {
        hit = dcd_vf(ldx(g.x0, v), ldx(g.x0, ft[0]), ldx(g.x0, ft[1]), ldx(g.x0, ft[2]), g.thickness, h);
      } else {
        hit = ccd_vf(ldx(g.x0, v), ldx(g.x1, v), ldx(g.x0, ft[0]), ldx(g.x1, ft[0]), ldx(g.x0, ft[1]),
                     ldx(g.x1, ft[1]), ldx(g.x0, ft[2]), ldx(g.x1, ft[2]), h);
      }
      if (hit) emit(g, 0, v, face_id, h);
    }
  }
  // edge-edge in canonical (min id, max id) orientation
  for (int ka = 0; ka < 3; ++ka) {
    const int ea = g.tri_edges[3 * t1 + ka];
    for (int kb = 0; kb < 3; ++kb) {
      const int eb = g.tri_edges[3 * t2 + kb];
      if (ea == eb) continue;
      const int lo = ea < eb ? ea : eb, hi = ea < eb ? eb : ea;
      const int2 e1 = g.edges[lo], e2 = g.edges[hi];
      if (e1.x == e2.x || e1.x == e2.y || e1.y == e2.x || e1.y == e2.y) continue;
      if (!g.movable[e1.x] && !g.movable[e1.y] && !g.movable[e2.x] && !g.movable[e2.y]) continue;
      const double* const fa[2] = {g.vbox + 6 * (size_t)e1.x, g.vbox + 6 * (size_t)e1.y};
      const double* const fb[2] = {g.vbox + 6 * (size_t)e2.x, g.vbox + 6 * (size_t)e2.y};
      if (boxes_apart_d(fa, fb, margin)) continue;
      Hit h;
      bool hit;
      if (!kCcd) {
        hit = dcd_ee(ldx(g.x0, e1.x), ldx(g.x0, e1.y), ldx(g.x0, e2.x), ldx(g.x0, e2.y), g.thickness, h);
      } else {
        hit = ccd_ee(ldx(g.x0, e1.x), ldx(g.x1, e1.x), ldx(g.x0, e1.y), ldx(g.x1, e1.y), ldx(g.x0, e2.x),
                     ldx(g.x1, e2.x), ldx(g.x0, e2.y), ldx(g.x1, e2.y), h);
      }
      if (hit) emit(g, 1, lo, hi, h);
    }
  }
}

// Two-pass narrow phase, pass 1: the box tests of k_narrow, one thread per
// candidate pair, every survivor compacted by ballot into the warp's
// shared-memory buffer (flushed with one atomic claim). The elementary tests
// then run densely in pass 2 (k_narrow_solve): at config D ~0.5 features
// per pair reach the CCD cubic solve and ~1.9 the DCD distance tests, which
// left most lanes of a fused warp (k_narrow, WEFT_NARROW_TWO=0) idle.
#ifndef WEFT_FEAT_BUF
#define WEFT_FEAT_BUF 64  // 8 KB per CTA: occupancy over fewer atomics (256: 11.0, 128: 10.4, 64: 10.1 ms broad + narrow)
#endif
constexpr int kFeatBuf = WEFT_FEAT_BUF;  // records per warp
constexpr int kFeatWarps = 4;
__device__ __forceinline__ void feat_flush(const NarrowArgs& g, int4* buf, int& bn, int lane) {
  __syncwarp();
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(g.feat_count, static_cast<unsigned long long>(bn));
  base = __shfl_sync(0xffffffffu, base, 0);
  for (int k = lane; k < 2 * bn; k += 32)
    if (base + (k >> 1) < g.feat_cap) g.feats[2 * base + k] = buf[k];
  __syncwarp();
  bn = 0;
}

template <bool kCcd>
__global__ void __launch_bounds__(kFeatWarps * 32) k_narrow_feats(NarrowArgs g) {
  __shared__ int4 sm_buf[kFeatWarps][2 * kFeatBuf];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int4* buf = sm_buf[warp];
  int bn = 0;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool alive = i < g.npairs;
  int t1 = 0, t2 = 0;
  if (alive) {
    const int2 pr = g.pairs[i];
    t1 = pr.x;
    t2 = pr.y;
  }
  const double margin = kCcd ? 1e-9 : g.thickness;
  if (alive) {  // the whole-pair rejections of k_narrow (float, then exact boxes)
    const float4 la = __ldg(g.tbox + 2 * t1), ha = __ldg(g.tbox + 2 * t1 + 1);
    const float4 lb = __ldg(g.tbox + 2 * t2), hb = __ldg(g.tbox + 2 * t2 + 1);
    if ((double)la.x > (double)hb.x + margin || (double)lb.x > (double)ha.x + margin ||
        (double)la.y > (double)hb.y + margin || (double)lb.y > (double)ha.y + margin ||
        (double)la.z > (double)hb.z + margin || (double)lb.z > (double)ha.z + margin)
      alive = false;
  }
  if (alive) {
    const double* const ta[1] = {g.dbox + 6 * (size_t)t1};
    const double* const tb[1] = {g.dbox + 6 * (size_t)t2};
    if (boxes_apart_d(ta, tb, margin)) alive = false;
  }
  int tri1[3] = {0, 0, 0}, tri2[3] = {0, 0, 0};
  if (alive) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      tri1[k] = g.tris[3 * t1 + k];
      tri2[k] = g.tris[3 * t2 + k];
    }
  }
  auto push = [&](bool keep, int4 r0, int4 r1) {
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const int at = bn + __popc(m & ((1u << lane) - 1u));
      buf[2 * at] = r0;
      buf[2 * at + 1] = r1;
    }
    bn += __popc(m);
    if (bn > kFeatBuf - 32) feat_flush(g, buf, bn, lane);
  };
  // vertex-face, both directions (k_narrow's order and skips)
  for (int dir = 0; dir < 2; ++dir) {
    for (int k = 0; k < 3; ++k) {
      bool keep = false;
      int v = 0, f0 = 0, f1 = 0, f2 = 0, face_id = 0;
      if (alive) {
        const int* vt = dir == 0 ? tri1 : tri2;
        const int* ft = dir == 0 ? tri2 : tri1;
        face_id = dir == 0 ? t2 : t1;
        v = vt[k];
        f0 = ft[0];
        f1 = ft[1];
        f2 = ft[2];
        keep = !(f0 == v || f1 == v || f2 == v) && (g.movable[v] || g.movable[f0] || g.movable[f1] || g.movable[f2]);
        if (keep) {
          const double* const fa[1] = {g.vbox + 6 * (size_t)v};
          const double* const fb[1] = {g.dbox + 6 * (size_t)face_id};
          keep = !boxes_apart_d(fa, fb, margin);
        }
      }
      push(keep, make_int4(0, v, face_id, v), make_int4(f0, f1, f2, 0));
    }
  }
  // edge-edge in canonical (min id, max id) orientation
  for (int ka = 0; ka < 3; ++ka) {
    for (int kb = 0; kb < 3; ++kb) {
      bool keep = false;
      int lo = 0, hi = 0;
      int2 e1 = make_int2(0, 0), e2 = make_int2(0, 0);
      if (alive) {
        const int ea = g.tri_edges[3 * t1 + ka], eb = g.tri_edges[3 * t2 + kb];
        if (ea != eb) {
          lo = ea < eb ? ea : eb;
          hi = ea < eb ? eb : ea;
          e1 = g.edges[lo];
          e2 = g.edges[hi];
          keep = !(e1.x == e2.x || e1.x == e2.y || e1.y == e2.x || e1.y == e2.y) &&
                 (g.movable[e1.x] || g.movable[e1.y] || g.movable[e2.x] || g.movable[e2.y]);
          if (keep) {
            const double* const fa[2] = {g.vbox + 6 * (size_t)e1.x, g.vbox + 6 * (size_t)e1.y};
            const double* const fb[2] = {g.vbox + 6 * (size_t)e2.x, g.vbox + 6 * (size_t)e2.y};
            keep = !boxes_apart_d(fa, fb, margin);
          }
        }
      }
      push(keep, make_int4(1, lo, hi, e1.x), make_int4(e1.y, e2.x, e2.y, 0));
    }
  }
  if (bn) feat_flush(g, buf, bn, lane);
}

// Pass 2: one thread per surviving feature, the elementary test of k_narrow.
template <bool kCcd>
__global__ void __launch_bounds__(128) k_narrow_solve(NarrowArgs g, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int4 r0 = g.feats[2 * i], r1 = g.feats[2 * i + 1];
  const int kind = r0.x;
  Hit h;
  bool hit;
  if (kind == 0) {
    const int v = r0.w, f0 = r1.x, f1 = r1.y, f2 = r1.z;
    if (!kCcd) {
      hit = dcd_vf(ldx(g.x0, v), ldx(g.x0, f0), ldx(g.x0, f1), ldx(g.x0, f2), g.thickness, h);
    } else {
      hit = ccd_vf(ldx(g.x0, v), ldx(g.x1, v), ldx(g.x0, f0), ldx(g.x1, f0), ldx(g.x0, f1), ldx(g.x1, f1),
                   ldx(g.x0, f2), ldx(g.x1, f2), h);
    }
  } else {
    const int a0 = r0.w, a1 = r1.x, b0 = r1.y, b1 = r1.z;
    if (!kCcd) {
      hit = dcd_ee(ldx(g.x0, a0), ldx(g.x0, a1), ldx(g.x0, b0), ldx(g.x0, b1), g.thickness, h);
    } else {
      hit = ccd_ee(ldx(g.x0, a0), ldx(g.x1, a0), ldx(g.x0, a1), ldx(g.x1, a1), ldx(g.x0, b0), ldx(g.x1, b0),
                   ldx(g.x0, b1), ldx(g.x1, b1), h);
    }
  }
  if (hit) emit(g, kind, r0.y, r0.z, h);
}

__global__ void k_iota(int64_t n, int64_t* __restrict__ v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

// sort_dedup (collision.cpp:313-325): keep the first of each run of equal keys.
__global__ void k_unique_flags(int64_t n, const unsigned long long* __restrict__ keys, int64_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void k_compact_hits(int64_t n, const unsigned long long* __restrict__ keys,
                               const int64_t* __restrict__ idx, const int64_t* __restrict__ pos,
                               const double* __restrict__ vals, unsigned long long* __restrict__ out_keys,
                               double* __restrict__ out_vals) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (!(i == 0 || keys[i] != keys[i - 1])) return;
  const int64_t o = pos[i];
  out_keys[o] = keys[i];
#pragma unroll
  for (int q = 0; q < 8; ++q) out_vals[8 * o + q] = vals[8 * idx[i] + q];
}

// ---- proximities_to_elements (response.cpp:43-106) ------------------------
struct ContactArgs {
  int64_t n;
  const unsigned long long* __restrict__ keys;
  const double* __restrict__ vals;
  const int32_t* __restrict__ tris;
  const int2* __restrict__ edges;
  const uint8_t* __restrict__ movable;
  const double* __restrict__ mass;
  const double* __restrict__ x;
  const double* __restrict__ v;
  double dt;
  ContactParamsDev kp;
  int* __restrict__ active;  // per vertex
  int64_t* __restrict__ flag;  // per proximity (then exclusive positions)
  // element records (after the static list)
  int64_t n_static, static_pay, static_res;
  int4* __restrict__ est;
  int2* __restrict__ einfo;
  double* __restrict__ edamp;
  double* __restrict__ epay;
  int32_t* __restrict__ eres_off;
};

// participants (response.cpp:21-39): four (vertex, signed weight) pairs.
__device__ __forceinline__ void participants(const ContactArgs& g, int64_t i, int vtx[4], double w[4]) {
  const unsigned long long k = g.keys[i];
  const int kind = static_cast<int>(k >> 62);
  const int a = static_cast<int>((k >> 31) & 0x7FFFFFFFull), b = static_cast<int>(k & 0x7FFFFFFFull);
  const double* hw = g.vals + 8 * i + 4;
  if (kind == 0) {
    vtx[0] = a;
    w[0] = 1.0;
    for (int q = 0; q < 3; ++q) {
      vtx[q + 1] = g.tris[3 * b + q];
      w[q + 1] = -hw[q + 1];
    }
  } else {
    const int2 e1 = g.edges[a], e2 = g.edges[b];
    vtx[0] = e1.x;
    w[0] = hw[0];
    vtx[1] = e1.y;
    w[1] = hw[1];
    vtx[2] = e2.x;
    w[2] = -hw[2];
    vtx[3] = e2.y;
    w[3] = -hw[3];
  }
}

__global__ void k_contact_active(ContactArgs g) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  if (g.vals[8 * i] >= g.kp.thickness) return;
  int vtx[4];
  double w[4];
  participants(g, i, vtx, w);
  for (int q = 0; q < 4; ++q)
    if (g.movable[vtx[q]]) atomicAdd(g.active + vtx[q], 1);
}

// kEmit false: flag[i] = 1 iff proximity i becomes an element; true: write
// it at n_static + flag[i] (flag scanned to positions).
template <bool kEmit>
__global__ void k_contact_elems(ContactArgs g) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  const double gap = g.vals[8 * i];
  if (gap >= g.kp.thickness) {
    if (!kEmit) g.flag[i] = 0;
    return;
  }
  int vtx[4];
  double w[4];
  participants(g, i, vtx, w);
  const V3 nrm = v3(g.vals[8 * i + 1], g.vals[8 * i + 2], g.vals[8 * i + 3]);
  int count = 0, overlap = 1;
  int st[4] = {-1, -1, -1, -1};
  double cw[4] = {0.0, 0.0, 0.0, 0.0};
  V3 rel_vel = v3(0.0, 0.0, 0.0), rel_bias = v3(0.0, 0.0, 0.0);
  double inv_mass = 0.0, bias = 0.0;
  for (int q = 0; q < 4; ++q) {
    const V3 vq = ldx(g.v, vtx[q]);
    rel_vel = add(rel_vel, scl(w[q], vq));
    if (g.movable[vtx[q]]) {
      st[count] = vtx[q];
      cw[count] = w[q];
      inv_mass = inv_mass + (w[q] * w[q]) / g.mass[vtx[q]];
      const int ac = g.active[vtx[q]];
      overlap = overlap < ac ? ac : overlap;  // std::max
      ++count;
    } else {
      bias = bias + w[q] * dot(nrm, ldx(g.x, vtx[q]));
      rel_bias = add(rel_bias, scl(w[q], vq));
    }
  }
  const bool live = count > 0 && !(inv_mass <= 0.0);
  if (!kEmit) {
    g.flag[i] = live ? 1 : 0;
    return;
  }
  if (!live) return;
  const double stiffness = g.kp.stiffness_scale / (((inv_mass * g.dt) * g.dt) * static_cast<double>(overlap));
  const double pen = g.kp.thickness - gap;
  const double frozen = stiffness * (0.0 < pen ? pen : 0.0);
  double tdamp = 0.0;
  if (g.kp.friction > 0.0) {
    const V3 vt = sub(rel_vel, scl(dot(nrm, rel_vel), nrm));
    const double vn = norm(vt);
    tdamp = (g.kp.friction * frozen) / (vn < 0.05 ? 0.05 : vn);
  }
  const int64_t k = g.flag[i];
  const int64_t e = g.n_static + k;
  const int64_t pay = g.static_pay + static_cast<int64_t>(kContactPay) * k;
  g.est[e] = make_int4(st[0], st[1], st[2], st[3]);
  g.einfo[e] = make_int2(WEFT_CONTACT | (count << 8), static_cast<int>(pay));
  g.edamp[e] = g.kp.damping;
  g.eres_off[e] = static_cast<int32_t>(g.static_res + static_cast<int64_t>(kContactRes) * k);
  double* d = g.epay + pay;  // ContactData layout of weft_element.data (weft_gpu.h)
  d[0] = nrm.x;
  d[1] = nrm.y;
  d[2] = nrm.z;
  for (int q = 0; q < 4; ++q) d[3 + q] = cw[q];
  d[7] = bias;
  d[8] = g.kp.thickness;
  d[9] = stiffness;
  d[10] = g.kp.friction;
  d[11] = tdamp;
  d[12] = frozen;
  d[13] = rel_bias.x;
  d[14] = rel_bias.y;
  d[15] = rel_bias.z;
}

}  // namespace

int64_t contacts_from_proximities(Ctx& c, const double* x, const double* v, double dt, const ContactParamsDev& kp) {
  cudaStream_t s = c.stream;
  const int64_t n = c.n_contacts_found;
  if (c.static_res + static_cast<int64_t>(kContactRes) * n > INT32_MAX)
    throw Error(WEFT_ERR_DIMENSION, "contact element results exceed 2^31 doubles");
  c.contact_active.resize(static_cast<size_t>(c.soup_verts) + 1);
  c.contact_active.zero(s);
  c.contact_flag.resize(static_cast<size_t>(n) + 1);
  ContactArgs g{n,  c.contact_keys.data(), c.contact_vals.data(), c.tris.data(), c.soup_edges.data(),
                c.soup_movable.data(), c.mass.data(), x, v, dt, kp, c.contact_active.data(), c.contact_flag.data(),
                c.n_static, c.static_pay, c.static_res, nullptr, nullptr, nullptr, nullptr, nullptr};
  int64_t count = 0;
  if (n) {
    k_contact_active<<<div_up(n, 256), 256, 0, ls(c)>>>(g);
    k_contact_elems<false><<<div_up(n, 256), 256, 0, ls(c)>>>(g);
    WG_CUDA(cudaMemsetAsync(c.contact_flag.data() + n, 0, sizeof(int64_t), s));
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, c.contact_flag.data(), c.contact_flag.data(), n + 1, s);
    void* t = scratch(c, tmp);
    WG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, c.contact_flag.data(), c.contact_flag.data(), n + 1, s));
    WG_CUDA(cudaMemcpyAsync(&count, c.contact_flag.data() + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    reserve_contacts(c, count);
    g.est = c.est.data();
    g.einfo = c.einfo.data();
    g.edamp = c.edamp.data();
    g.epay = c.epay.data();
    g.eres_off = c.eres_off.data();
    k_contact_elems<true><<<div_up(n, 256), 256, 0, ls(c)>>>(g);
    WG_CUDA(cudaGetLastError());
  } else {
    reserve_contacts(c, 0);
  }
  finish_contacts(c, count);
  return count;
}

// CollisionSoup::build (collision.cpp:95-116): unique sorted edges with ids in
// order of first appearance (triangle order, k = 0, 1, 2), per-triangle edge
// ids. Host, once per soup.
void build_soup_edges(Ctx& c, const std::vector<int32_t>& tris) {
  const size_t T = tris.size() / 3;
  std::unordered_map<uint64_t, int32_t> ids;
  ids.reserve(3 * T);
  std::vector<int2> edges;
  std::vector<int32_t> te(3 * T);
  for (size_t t = 0; t < T; ++t)
    for (int k = 0; k < 3; ++k) {
      int a = tris[3 * t + k], b = tris[3 * t + (k + 1) % 3];
      if (a > b) std::swap(a, b);
      const uint64_t key = (static_cast<uint64_t>(static_cast<uint32_t>(a)) << 32) | static_cast<uint32_t>(b);
      auto it = ids.find(key);
      if (it == ids.end()) {
        it = ids.emplace(key, static_cast<int32_t>(edges.size())).first;
        edges.push_back(make_int2(a, b));
      }
      te[3 * t + k] = it->second;
    }
  c.soup_edges.upload(edges.data(), edges.size(), c.stream);
  c.soup_tri_edges.upload(te.data(), te.size(), c.stream);
  std::vector<uint8_t> mv(static_cast<size_t>(c.soup_verts), 1);
  c.soup_movable.upload(mv.data(), mv.size(), c.stream);
  WG_CUDA(cudaStreamSynchronize(c.stream));
}

void set_soup_movable(Ctx& c, const uint8_t* movable) {
  std::vector<uint8_t> mv(static_cast<size_t>(c.soup_verts), 1);
  if (movable && c.soup_verts)
    WG_CUDA(cudaMemcpy(mv.data(), movable, mv.size(), cudaMemcpyDefault));
  for (auto& m : mv) m = m ? 1 : 0;
  c.soup_movable.upload(mv.data(), mv.size(), c.stream);
  WG_CUDA(cudaStreamSynchronize(c.stream));
}

// collide (collision.cpp:391-417) for this rank's pair range on the current
// grid: narrow phase of every candidate pair, sorted and deduplicated.
int64_t narrow_phase(Ctx& c, const double* x0, const double* x1, int mode, double thickness, int64_t begin,
                     int64_t end) {
  cudaStream_t s = c.stream;
  const bool ccd = mode == WEFT_CONTINUOUS;
  // conservative float triangle boxes: the walk emits only the candidate
  // pairs they do not separate by the margin (most do not reach a feature
  // test: ~92 % of config-D DCD candidates), k_narrow tests the rest
  c.zn_tbox.resize(2 * static_cast<size_t>(c.soup_tris) + 2);
  c.zn_dbox.resize(6 * static_cast<size_t>(c.soup_tris) + 6);
  c.zn_vbox.resize(6 * static_cast<size_t>(c.soup_verts) + 6);
  if (c.soup_tris)
    k_tri_fbox<<<div_up(c.soup_tris, 256), 256, 0, ls(c)>>>(c.soup_tris, c.tris.data(), x0, ccd ? x1 : x0, ccd,
                                                            c.zn_tbox.data(), c.zn_dbox.data());
  if (c.soup_verts)
    k_vert_box<<<div_up(c.soup_verts, 256), 256, 0, ls(c)>>>(c.soup_verts, x0, ccd ? x1 : x0, ccd,
                                                             c.zn_vbox.data());
  int64_t all = 0;
  const int64_t npairs = candidates(c, begin, end, nullptr, /*count_only=*/false, c.zn_tbox.data(),
                                    ccd ? 1e-9 : thickness, &all);
  NarrowArgs g{npairs,
               reinterpret_cast<const int2*>(c.cand_pairs.data()),
               c.tris.data(),
               c.soup_tri_edges.data(),
               c.soup_edges.data(),
               c.soup_movable.data(),
               x0,
               ccd ? x1 : x0,
               ccd,
               thickness,
               nullptr,
               nullptr,
               nullptr,
               0,
               nullptr};
  g.tbox = c.zn_tbox.data();
  g.vbox = c.zn_vbox.data();
  g.dbox = c.zn_dbox.data();
  c.hit_count.resize(1);
  unsigned long long nh = 0;
  // two-pass (features, then their elementary tests) per mode; WEFT_NARROW_TWO
  // = 0 / 1 / 2 / 3: fused for both / CCD only / DCD only / both two-pass
  static const int two_env = std::getenv("WEFT_NARROW_TWO") ? std::atoi(std::getenv("WEFT_NARROW_TWO")) : 3;
  const bool two_pass = ccd ? (two_env & 1) != 0 : (two_env & 2) != 0;
  int64_t nfeat = 0;
  static const int64_t fcap_env = std::getenv("WEFT_NARROW_FCAP") ? std::atoll(std::getenv("WEFT_NARROW_FCAP")) : 0;
  int64_t fcap = fcap_env > 0 ? fcap_env
                              : std::max<int64_t>((static_cast<int64_t>(c.zn_feats.cap) - 2) / 2, int64_t{1} << 20);
  c.zn_feat_count.resize(1);
  if (npairs) {
    size_t cap = std::max<size_t>(c.hit_keys.cap, static_cast<size_t>(1) << 20);
    for (int attempt = 0; attempt < 2; ++attempt) {
      c.hit_keys.resize(cap);
      c.hit_vals.resize(8 * cap);
      g.keys = c.hit_keys.data();
      g.vals = c.hit_vals.data();
      g.count = c.hit_count.data();
      g.cap = cap;
      WG_CUDA(cudaMemsetAsync(c.hit_count.data(), 0, sizeof(unsigned long long), s));
      if (two_pass) {
        for (int fa = 0; fa < 2; ++fa) {  // features pass (exact count on overflow, once)
          c.zn_feats.resize(2 * static_cast<size_t>(fcap) + 2);
          g.feats = reinterpret_cast<int4*>(c.zn_feats.data());
          g.feat_count = c.zn_feat_count.data();
          g.feat_cap = static_cast<unsigned long long>(fcap);
          WG_CUDA(cudaMemsetAsync(c.zn_feat_count.data(), 0, sizeof(unsigned long long), s));
          if (ccd) k_narrow_feats<true><<<div_up(npairs, kFeatWarps * 32), kFeatWarps * 32, 0, ls(c)>>>(g);
          else k_narrow_feats<false><<<div_up(npairs, kFeatWarps * 32), kFeatWarps * 32, 0, ls(c)>>>(g);
          WG_CUDA(cudaGetLastError());
          unsigned long long nf = 0;
          read_small(c, s, {c.zn_feat_count.data(), &nf, sizeof(nf)});
          nfeat = static_cast<int64_t>(nf);
          if (nfeat <= fcap) break;
          fcap = nfeat;
        }
        if (nfeat) {
          if (ccd) k_narrow_solve<true><<<div_up(nfeat, 128), 128, 0, ls(c)>>>(g, nfeat);
          else k_narrow_solve<false><<<div_up(nfeat, 128), 128, 0, ls(c)>>>(g, nfeat);
        }
      } else if (ccd) {
        k_narrow<true><<<div_up(npairs, 128), 128, 0, ls(c)>>>(g);
      } else {
        k_narrow<false><<<div_up(npairs, 128), 128, 0, ls(c)>>>(g);
      }
      WG_CUDA(cudaGetLastError());
      WG_CUDA(cudaMemcpyAsync(&nh, c.hit_count.data(), sizeof(nh), cudaMemcpyDeviceToHost, s));
      WG_CUDA(cudaStreamSynchronize(s));
      if (nh <= cap) break;
      cap = static_cast<size_t>(nh);  // exact capacity, run once more
    }
  }
  c.narrow_pairs = all;  // every candidate pair of the range (the reference's count)
  c.narrow_raw_hits = static_cast<int64_t>(nh);
  return dedup_hits(c, static_cast<int64_t>(nh));
}

// sort_dedup (collision.cpp:313-325): radix sort by key, the first of every
// equal-key run kept (duplicates — one feature pair reached from several
// triangle pairs — carry identical values).
int64_t dedup_hits(Ctx& c, int64_t n) {
  cudaStream_t s = c.stream;
  c.hit_keys_sorted.resize(static_cast<size_t>(n) + 1);
  c.hit_idx.resize(static_cast<size_t>(n) + 1);
  c.hit_idx_sorted.resize(static_cast<size_t>(n) + 1);
  c.hit_flag.resize(static_cast<size_t>(n) + 1);
  int64_t nu = 0;
  if (n) {
    k_iota<<<div_up(n, 256), 256, 0, ls(c)>>>(n, c.hit_idx.data());
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, c.hit_keys.data(), c.hit_keys_sorted.data(), c.hit_idx.data(),
                                    c.hit_idx_sorted.data(), n, 0, 63, s);
    size_t tmp2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp2, c.hit_flag.data(), c.hit_flag.data(), n + 1, s);
    void* t = scratch(c, std::max(tmp, tmp2));
    WG_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, c.hit_keys.data(), c.hit_keys_sorted.data(), c.hit_idx.data(),
                                            c.hit_idx_sorted.data(), n, 0, 63, s));
    k_unique_flags<<<div_up(n, 256), 256, 0, ls(c)>>>(n, c.hit_keys_sorted.data(), c.hit_flag.data());
    WG_CUDA(cudaMemsetAsync(c.hit_flag.data() + n, 0, sizeof(int64_t), s));
    WG_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp2, c.hit_flag.data(), c.hit_flag.data(), n + 1, s));
    WG_CUDA(cudaMemcpyAsync(&nu, c.hit_flag.data() + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    c.contact_keys.resize(static_cast<size_t>(nu) + 1);
    c.contact_vals.resize(8 * static_cast<size_t>(nu) + 8);
    k_compact_hits<<<div_up(n, 256), 256, 0, ls(c)>>>(n, c.hit_keys_sorted.data(), c.hit_idx_sorted.data(),
                                                      c.hit_flag.data(), c.hit_vals.data(), c.contact_keys.data(),
                                                      c.contact_vals.data());
    WG_CUDA(cudaGetLastError());
    WG_CUDA(cudaStreamSynchronize(s));
  }
  c.n_contacts_found = nu;
  return nu;
}

int64_t collide(Ctx& c, const double* x0, const double* x1, int mode, double thickness, double cell_scale) {
  build_grid(c, x0, x1, mode, thickness, cell_scale);
  // a rank of a group walks its split_workload share (collision.cpp:402)
  const int64_t total = c.grid_total, base = total / c.world, extra = total % c.world;
  const int64_t b = c.rank * base + std::min<int64_t>(c.rank, extra);
  const int64_t e = b + base + (c.rank < extra ? 1 : 0);
  const int64_t n = narrow_phase(c, x0, x1, mode, thickness, b, e);
  return c.world > 1 ? merge_hits(c) : n;
}

void download_contacts(Ctx& c, int32_t* kab, double* vals) {
  const int64_t n = c.n_contacts_found;
  if (n <= 0) return;
  cudaStream_t s = c.stream;
  std::vector<unsigned long long> keys(static_cast<size_t>(n));
  WG_CUDA(cudaMemcpyAsync(keys.data(), c.contact_keys.data(), 8 * n, cudaMemcpyDeviceToHost, s));
  if (vals) WG_CUDA(cudaMemcpyAsync(vals, c.contact_vals.data(), 64 * n, cudaMemcpyDefault, s));
  WG_CUDA(cudaStreamSynchronize(s));
  if (kab)
    for (int64_t i = 0; i < n; ++i) {
      const unsigned long long k = keys[static_cast<size_t>(i)];
      kab[3 * i] = static_cast<int32_t>(k >> 62);
      kab[3 * i + 1] = static_cast<int32_t>((k >> 31) & 0x7FFFFFFFull);
      kab[3 * i + 2] = static_cast<int32_t>(k & 0x7FFFFFFFull);
    }
}

}  // namespace weft_gpu
