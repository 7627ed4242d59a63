// elements.cuh — per-element force / Jacobian kernels for one stencil row.
//
// Device restatement of proj/src/elements.cpp (element_force :320-340,
// element_jacobian :342-361, element_friction_force :363-382,
// element_velocity_damping :389-403) evaluated only for the stencil row `a`
// the calling thread owns. Every expression keeps the reference's
// association (the reference compiled against oracle/shim/Eigen/Dense:
// strict left-to-right 3-term reductions, scalar chains evaluated before the
// vector product) and the library is built with -fmad=false, so the
// assembled matrix is bitwise equal to the CPU reference. The only
// non-bitwise quantity is the hinge angle: glibc's atan2 is not correctly
// rounded (about 1 draw in 10^3 lands 1 ulp off), so no device atan2 can
// reproduce it everywhere; cr::atan2 (cr_atan2.cuh) is correctly rounded,
// which agrees with glibc on all but ~1e-5 of near-flat hinges (CUDA's
// 2-ulp atan2 disagreed far more often). The angle enters the right-hand
// side and the Exact-mode bend Hessian scale.
#pragma once

#include "common.cuh"
#include "cr_atan2.cuh"

namespace weft_gpu {

struct V3 {
  double x, y, z;
};

__device__ __forceinline__ V3 v3(double a, double b, double c) { return V3{a, b, c}; }
__device__ __forceinline__ V3 ld3(const double* __restrict__ p, int i) {
  return V3{__ldg(p + 3 * i), __ldg(p + 3 * i + 1), __ldg(p + 3 * i + 2)};
}
__device__ __forceinline__ V3 add(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 sub(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 scl(double s, V3 a) { return V3{s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ V3 divs(V3 a, double s) { return V3{a.x / s, a.y / s, a.z / s}; }
__device__ __forceinline__ double dot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__device__ __forceinline__ V3 cross(V3 a, V3 b) {
  return V3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double norm(V3 a) { return sqrt(dot(a, a)); }
__device__ __forceinline__ double comp(V3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

constexpr double kDeg = 1e-24;  // kDegenerateNormal2, elements.cpp:9

// ---------------------------------------------------------------- stretch
// stretch_state (elements.cpp:133-141)
struct StretchSt {
  V3 wu, wv;
  double wu_len, wv_len;
  bool ok;
};

__device__ __forceinline__ StretchSt stretch_state(const double* d, V3 x0, V3 x1, V3 x2) {
  StretchSt s;
  s.wu = add(add(scl(d[0], x0), scl(d[1], x1)), scl(d[2], x2));
  s.wv = add(add(scl(d[3], x0), scl(d[4], x1)), scl(d[5], x2));
  s.wu_len = norm(s.wu);
  s.wv_len = norm(s.wv);
  s.ok = s.wu_len > 1e-12 && s.wv_len > 1e-12;
  return s;
}

// stretch_force row a (elements.cpp:161-181).
__device__ __forceinline__ void stretch_force_row(const double* d, V3 x0, V3 x1, V3 x2, int i, double f[3]) {
  f[0] = f[1] = f[2] = 0.0;
  const StretchSt st = stretch_state(d, x0, x1, x2);
  if (!st.ok) return;
  const V3 wu_hat = divs(st.wu, st.wu_len), wv_hat = divs(st.wv, st.wv_len);
  const double a = d[6];
  const double cu = a * (st.wu_len - 1.0), cv = a * (st.wv_len - 1.0), cs = a * dot(st.wu, st.wv);
  const V3 gu = scl(a * d[i], wu_hat);
  const V3 gv = scl(a * d[3 + i], wv_hat);
  const V3 gs = scl(a, add(scl(d[i], st.wv), scl(d[3 + i], st.wu)));
  const double su = -(d[7] * cu), sv = d[8] * cv, ss = d[9] * cs;
  f[0] = 0.0 + ((su * gu.x - sv * gv.x) - ss * gs.x);
  f[1] = 0.0 + ((su * gu.y - sv * gv.y) - ss * gs.y);
  f[2] = 0.0 + ((su * gu.z - sv * gv.z) - ss * gs.z);
}

// stretch_jacobian blocks (i, j), j = 0..2 (elements.cpp:183-230), streamed
// to emit(j, block) one block at a time (keeps the 3x3 block in registers).
template <class F>
__device__ __forceinline__ void stretch_jac_row(const double* d, V3 x0, V3 x1, V3 x2, int i, bool exact, F&& emit) {
  const StretchSt st = stretch_state(d, x0, x1, x2);
  double J[9];
  if (!st.ok) {
#pragma unroll
    for (int q = 0; q < 9; ++q) J[q] = 0.0;
    for (int j = 0; j < 3; ++j) emit(j, J);
    return;
  }
  const V3 wu_hat = divs(st.wu, st.wu_len), wv_hat = divs(st.wv, st.wv_len);
  const double a = d[6];
  const double cu = a * (st.wu_len - 1.0), cv = a * (st.wv_len - 1.0), cs = a * dot(st.wu, st.wv);
  const bool keep_u2 = exact || cu >= 0.0, keep_v2 = exact || cv >= 0.0, keep_s2 = exact;
  const double ui = d[i], vi = d[3 + i];
  const V3 gui = scl(a * ui, wu_hat), gvi = scl(a * vi, wv_hat);
  const V3 gsi = scl(a, add(scl(ui, st.wv), scl(vi, st.wu)));
  for (int j = 0; j < 3; ++j) {
    const double uj = d[j], vj = d[3 + j];
    const V3 guj = scl(a * uj, wu_hat), gvj = scl(a * vj, wv_hat);
    const V3 gsj = scl(a, add(scl(uj, st.wv), scl(vj, st.wu)));
    const double su2 = (d[7] * cu) * (((a * ui) * uj) / st.wu_len);
    const double sv2 = (d[8] * cv) * (((a * vi) * vj) / st.wv_len);
    const double ss2 = (d[9] * cs) * (a * (ui * vj + vi * uj));
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double id = r == c ? 1.0 : 0.0;
        double m = 0.0;
        m = m - d[7] * (comp(gui, r) * comp(guj, c));
        m = m - d[8] * (comp(gvi, r) * comp(gvj, c));
        m = m - d[9] * (comp(gsi, r) * comp(gsj, c));
        if (keep_u2) m = m - su2 * (id - comp(wu_hat, r) * comp(wu_hat, c));
        if (keep_v2) m = m - sv2 * (id - comp(wv_hat, r) * comp(wv_hat, c));
        if (keep_s2) m = m - ss2 * id;
        J[r * 3 + c] = 0.0 + m;
      }
    emit(j, J);
  }
}

// ---------------------------------------------------------------- bend
// dihedral_gradient_t<double> (elements.cpp:66-90)
__device__ __forceinline__ void dihedral_gradient(V3 x0, V3 x1, V3 x2, V3 x3, V3 g[4]) {
  const V3 e = sub(x1, x0);
  const V3 na = cross(e, sub(x2, x0));
  const V3 nb = cross(sub(x3, x0), e);
  const double na2 = dot(na, na), nb2 = dot(nb, nb);
  const double elen = sqrt(dot(e, e));
  g[0] = g[1] = g[2] = g[3] = v3(0.0, 0.0, 0.0);
  if (na2 < kDeg || nb2 < kDeg || elen < 1e-12) return;
  const double sa = -elen / na2, sb = -elen / nb2;
  g[2] = v3(na.x * sa, na.y * sa, na.z * sa);
  g[3] = v3(nb.x * sb, nb.y * sb, nb.z * sb);
  const double ca0 = dot(sub(x1, x2), e) / (elen * na2);
  const double cb0 = dot(sub(x1, x3), e) / (elen * nb2);
  const double ca1 = dot(sub(x2, x0), e) / (elen * na2);
  const double cb1 = dot(sub(x3, x0), e) / (elen * nb2);
  g[0] = v3(na.x * ca0 + nb.x * cb0, na.y * ca0 + nb.y * cb0, na.z * ca0 + nb.z * cb0);
  g[1] = v3(na.x * ca1 + nb.x * cb1, na.y * ca1 + nb.y * cb1, na.z * ca1 + nb.z * cb1);
}

// dihedral_angle (elements.cpp:94-104)
__device__ __forceinline__ double dihedral_angle(V3 x0, V3 x1, V3 x2, V3 x3) {
  const V3 e = sub(x1, x0);
  const V3 na = cross(e, sub(x2, x0));
  const V3 nb = cross(sub(x3, x0), e);
  const double elen = norm(e);
  if (dot(na, na) < kDeg || dot(nb, nb) < kDeg || elen < 1e-12) return 0.0;
  const double s = dot(cross(na, nb), e) / elen;
  const double c = dot(na, nb);
  return cr::atan2(s, c);
}

// Forward-mode dual (elements.cpp:13-30)
struct Dual {
  double v, d;
};
__device__ __forceinline__ Dual operator+(Dual a, Dual b) { return Dual{a.v + b.v, a.d + b.d}; }
__device__ __forceinline__ Dual operator-(Dual a, Dual b) { return Dual{a.v - b.v, a.d - b.d}; }
__device__ __forceinline__ Dual operator*(Dual a, Dual b) { return Dual{a.v * b.v, a.d * b.v + a.v * b.d}; }
__device__ __forceinline__ Dual operator/(Dual a, Dual b) {
  return Dual{a.v / b.v, (a.d * b.v - a.v * b.d) / (b.v * b.v)};
}
__device__ __forceinline__ Dual operator-(Dual a) { return Dual{-a.v, -a.d}; }
__device__ __forceinline__ Dual dsqrt(Dual a) {
  const double s = sqrt(a.v);
  return Dual{s, a.d / (2.0 * s)};
}

// dihedral_gradient_t<Dual>: derivative of the gradient along coordinate j.
// Returns the 12 derivative components (gradient index i = 3*vertex+comp).
static __device__ __noinline__ void dihedral_gradient_dual(const double xs[12], int j, double out[12]) {
  Dual x[4][3];
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int c = 0; c < 3; ++c) x[v][c] = Dual{xs[3 * v + c], (3 * v + c == j) ? 1.0 : 0.0};
  Dual e[3], t[3], na[3], nb[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) e[c] = x[1][c] - x[0][c];
#pragma unroll
  for (int c = 0; c < 3; ++c) t[c] = x[2][c] - x[0][c];
  na[0] = e[1] * t[2] - e[2] * t[1];
  na[1] = e[2] * t[0] - e[0] * t[2];
  na[2] = e[0] * t[1] - e[1] * t[0];
#pragma unroll
  for (int c = 0; c < 3; ++c) t[c] = x[3][c] - x[0][c];
  nb[0] = t[1] * e[2] - t[2] * e[1];
  nb[1] = t[2] * e[0] - t[0] * e[2];
  nb[2] = t[0] * e[1] - t[1] * e[0];
  const Dual na2 = (na[0] * na[0] + na[1] * na[1]) + na[2] * na[2];
  const Dual nb2 = (nb[0] * nb[0] + nb[1] * nb[1]) + nb[2] * nb[2];
  const Dual elen = dsqrt((e[0] * e[0] + e[1] * e[1]) + e[2] * e[2]);
#pragma unroll
  for (int i = 0; i < 12; ++i) out[i] = 0.0;
  if (na2.v < kDeg || nb2.v < kDeg || elen.v < 1e-12) return;
  const Dual sa = (-elen) / na2, sb = (-elen) / nb2;
  Dual d12[3], d13[3], d20[3], d30[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    d12[c] = x[1][c] - x[2][c];
    d13[c] = x[1][c] - x[3][c];
    d20[c] = x[2][c] - x[0][c];
    d30[c] = x[3][c] - x[0][c];
  }
  const Dual ca0 = ((d12[0] * e[0] + d12[1] * e[1]) + d12[2] * e[2]) / (elen * na2);
  const Dual cb0 = ((d13[0] * e[0] + d13[1] * e[1]) + d13[2] * e[2]) / (elen * nb2);
  const Dual ca1 = ((d20[0] * e[0] + d20[1] * e[1]) + d20[2] * e[2]) / (elen * na2);
  const Dual cb1 = ((d30[0] * e[0] + d30[1] * e[1]) + d30[2] * e[2]) / (elen * nb2);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    out[c] = (na[c] * ca0 + nb[c] * cb0).d;
    out[3 + c] = (na[c] * ca1 + nb[c] * cb1).d;
    out[6 + c] = (na[c] * sa).d;
    out[9 + c] = (nb[c] * sb).d;
  }
}

// Exact-mode bend blocks (a, b): -k g_a g_b^T - (k dtheta) H_ab with the
// symmetrized dual Hessian (elements.cpp:131-159, 244-267).
static __device__ __noinline__ void bend_jac_exact_row(const double* d, V3 x0, V3 x1, V3 x2, V3 x3, int a,
                                                double (*J)[9]) {
  V3 g[4];
  dihedral_gradient(x0, x1, x2, x3, g);
  const double dtheta = dihedral_angle(x0, x1, x2, x3) - d[0];
  const double xs[12] = {x0.x, x0.y, x0.z, x1.x, x1.y, x1.z, x2.x, x2.y, x2.z, x3.x, x3.y, x3.z};
  // H[i][j] = dg_i/dx_j. Needed: rows 3a..3a+2 (all columns) and columns
  // 3a..3a+2 (all rows). Column j comes from sweep j.
  double Hrow[3][12];  // H[3a+r][j]
  double Hcol[12][3];  // H[i][3a+r]
  double col[12];
  for (int j = 0; j < 12; ++j) {
    dihedral_gradient_dual(xs, j, col);
#pragma unroll
    for (int r = 0; r < 3; ++r) Hrow[r][j] = col[3 * a + r];
    if (j / 3 == a)
      for (int i = 0; i < 12; ++i) Hcol[i][j - 3 * a] = col[i];
  }
  const double nk = -d[1];
  const double kd = d[1] * dtheta;
  const V3 ga = g[a];
#pragma unroll
  for (int b = 0; b < 4; ++b)
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double h = 0.5 * (Hrow[r][3 * b + c] + Hcol[3 * b + c][r]);
        double m = nk * (comp(ga, r) * comp(g[b], c));
        m = m - kd * h;
        J[b][r * 3 + c] = 0.0 + m;
      }
}

// ---------------------------------------------------------------- evaluate
// One element instance, stencil row a. Returns f = element_force(x_adv).f[a]
// + element_friction_force(v).f[a] (assembly.hpp:185) and streams the row's
// Jacobian blocks J_ab (x_cur) with the velocity-damping blocks D_ab (or
// nullptr when the element has none) to emit(b, J, D, add) in ascending b;
// add = false marks a block whose matrix contribution is exactly -0.
// Payload layout per kind: include/weft_gpu.h.
template <bool exact, class F>
__device__ __forceinline__ void eval_row(int kind, int ss, const int st[4], const double* __restrict__ d, int a,
                                         const double* __restrict__ xc, const double* __restrict__ xa,
                                         const double* __restrict__ vel, double f[3], F&& emit) {
  f[0] = f[1] = f[2] = 0.0;
  double fr[3] = {0.0, 0.0, 0.0};
  switch (kind) {
    case WEFT_STRETCH: {
      stretch_force_row(d, ld3(xa, st[0]), ld3(xa, st[1]), ld3(xa, st[2]), a, f);
      stretch_jac_row(d, ld3(xc, st[0]), ld3(xc, st[1]), ld3(xc, st[2]), a, exact,
                      [&](int b, const double* J) { emit(b, J, nullptr, true); });
      break;
    }
    case WEFT_BEND: {
      {  // bend_force (elements.cpp:232-242) at x_adv
        const V3 p0 = ld3(xa, st[0]), p1 = ld3(xa, st[1]), p2 = ld3(xa, st[2]), p3 = ld3(xa, st[3]);
        const double theta = dihedral_angle(p0, p1, p2, p3);
        V3 g[4];
        dihedral_gradient(p0, p1, p2, p3, g);
        const double coeff = -d[1] * (theta - d[0]);
        const V3 ga = g[a];
        f[0] = 0.0 + coeff * ga.x;
        f[1] = 0.0 + coeff * ga.y;
        f[2] = 0.0 + coeff * ga.z;
      }
      const V3 p0 = ld3(xc, st[0]), p1 = ld3(xc, st[1]), p2 = ld3(xc, st[2]), p3 = ld3(xc, st[3]);
      if constexpr (exact) {
        double J[4][9];
        bend_jac_exact_row(d, p0, p1, p2, p3, a, J);
        for (int b = 0; b < 4; ++b) emit(b, J[b], nullptr, true);
      } else {  // bend_jacobian SpdProjected (elements.cpp:244-267)
        V3 g[4];
        dihedral_gradient(p0, p1, p2, p3, g);
        const double nk = -d[1];
        const V3 ga = g[a];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          double J[9];
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) J[r * 3 + c] = 0.0 + nk * (comp(ga, r) * comp(g[b], c));
          emit(b, J, nullptr, true);
        }
      }
      break;
    }
    case WEFT_SPRING: {
      {  // spring_force (elements.cpp:269-279)
        const V3 dd = sub(ld3(xa, st[1]), ld3(xa, st[0]));
        const double len = norm(dd);
        if (len >= 1e-12) {
          const V3 dir = divs(dd, len);
          const V3 fa = scl(d[1] * (len - d[0]), dir);
          if (a == 0) {
            f[0] = 0.0 + fa.x;
            f[1] = 0.0 + fa.y;
            f[2] = 0.0 + fa.z;
          } else {
            f[0] = 0.0 - fa.x;
            f[1] = 0.0 - fa.y;
            f[2] = 0.0 - fa.z;
          }
        }
      }
      {  // spring_jacobian (elements.cpp:281-293): blocks (a,0), (a,1)
        const V3 dd = sub(ld3(xc, st[1]), ld3(xc, st[0]));
        const double len = norm(dd);
        double K[9];
        if (len >= 1e-12) {
          const V3 dir = divs(dd, len);
          double lateral = 1.0 - d[0] / len;
          if (!exact) lateral = lateral > 0.0 ? lateral : 0.0;
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const double oo = comp(dir, r) * comp(dir, c);
              K[r * 3 + c] = d[1] * (oo + lateral * ((r == c ? 1.0 : 0.0) - oo));
            }
        } else {
#pragma unroll
          for (int q = 0; q < 9; ++q) K[q] = 0.0;  // blocks stay zero
        }
        double J[9];
        const bool live = len >= 1e-12;
#pragma unroll
        for (int b = 0; b < 2; ++b) {
#pragma unroll
          for (int q = 0; q < 9; ++q) J[q] = !live ? 0.0 : (b == a ? 0.0 - K[q] : 0.0 + K[q]);
          emit(b, J, nullptr, true);
        }
      }
      break;
    }
    case WEFT_EXTERNAL: {  // constant force; drag friction + damping (elements.cpp:335-337, 364-368, 390-393)
      f[0] = d[0];
      f[1] = d[1];
      f[2] = d[2];
      if (d[3] > 0.0) {
        const V3 v = ld3(vel, st[0]);
        fr[0] = -d[3] * v.x;
        fr[1] = -d[3] * v.y;
        fr[2] = -d[3] * v.z;
        double J[9], D[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            J[r * 3 + c] = 0.0;
            D[r * 3 + c] = 0.0 + d[3] * (r == c ? 1.0 : 0.0);
          }
        emit(0, J, D, true);
      } else {
        // (-scale) * 0 = -0 never changes a sum: only the damping product
        // J v (exactly 0 or -0) is needed.
        double J[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) J[q] = 0.0;
        emit(0, J, nullptr, false);
      }
      break;
    }
    case WEFT_CONTACT: {
      const V3 n = v3(d[0], d[1], d[2]);
      {  // contact_force (elements.cpp:295-303) at x_adv
        double gap = d[7];
        for (int i = 0; i < ss; ++i) gap = gap + d[3 + i] * dot(n, ld3(xa, st[i]));
        if (gap < d[8]) {
          const double mag = d[9] * (d[8] - gap);
          const double s = mag * d[3 + a];
          f[0] = 0.0 + s * n.x;
          f[1] = 0.0 + s * n.y;
          f[2] = 0.0 + s * n.z;
        }
      }
      const bool damped = d[11] > 0.0;
      if (damped) {  // friction (elements.cpp:370-381)
        V3 rel = v3(d[13], d[14], d[15]);
        for (int i = 0; i < ss; ++i) rel = add(rel, scl(d[3 + i], ld3(vel, st[i])));
        const double rn = dot(n, rel);
        const V3 tang = sub(rel, scl(rn, n));
        const V3 frv = scl(-d[11], tang);
        fr[0] = d[3 + a] * frv.x;
        fr[1] = d[3 + a] * frv.y;
        fr[2] = d[3 + a] * frv.z;
      }
      double gap = d[7];  // contact_jacobian (elements.cpp:305-316) at x_cur
      for (int i = 0; i < ss; ++i) gap = gap + d[3 + i] * dot(n, ld3(xc, st[i]));
      const bool active = gap < d[8];
      for (int j = 0; j < ss; ++j) {
        double J[9], D[9];
        const double k = (d[9] * d[3 + a]) * d[3 + j];
        const double kd = (d[11] * d[3 + a]) * d[3 + j];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double nn = comp(n, r) * comp(n, c);
            J[r * 3 + c] = active ? 0.0 - k * nn : 0.0;
            D[r * 3 + c] = 0.0 + kd * ((r == c ? 1.0 : 0.0) - nn);
          }
        emit(j, J, damped ? D : nullptr, true);
      }
      break;
    }
    default:
      break;
  }
  f[0] = f[0] + fr[0];
  f[1] = f[1] + fr[1];
  f[2] = f[2] + fr[2];
}

}  // namespace weft_gpu
