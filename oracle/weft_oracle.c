/*
 * weft_oracle.c — CPU restatement of the reference hot path (TEST
 * INFRASTRUCTURE ONLY; see weft_oracle.h). Compile with -ffp-contract=off.
 * Each block cites the reference file:line it restates; the arithmetic is
 * written in the exact association of the reference built against
 * oracle/shim/Eigen/Dense.
 */
#include "weft_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================
 * Partitions and work queues
 * ====================================================================== */

/* make_partitions: proj/src/exec.cpp:10-23 */
void orc_make_partitions(int32_t p, int32_t n, int32_t* begin, int32_t* end) {
  const int32_t base = p / n, extra = p % n;
  int32_t cursor = 0;
  for (int32_t d = 0; d < n; ++d) {
    const int32_t size = base + (d < extra ? 1 : 0);
    begin[d] = cursor;
    end[d] = cursor + size;
    cursor += size;
  }
}

/* PartitionMap::owner: proj/include/weft/assembly.hpp:27-31 */
int32_t orc_owner(int32_t p, int32_t n, int32_t v) {
  const int32_t base = p / n, extra = p % n;
  const int32_t split = extra * (base + 1);
  if (v < split) return v / (base + 1);
  return extra + (v - split) / (base > 1 ? base : 1);
}

/* generate_range: proj/src/topology.cpp:34-56 */
static void gen_range(int32_t lo, int32_t hi, int32_t n, int32_t* peer, int32_t* vec, int32_t* len) {
  const int32_t size = hi - lo;
  if (size == 1) return;
  const int32_t half = size / 2, mid = lo + half;
  gen_range(lo, mid, n, peer, vec, len);
  gen_range(mid, hi, n, peer, vec, len);
  const int32_t child_len = len[lo];
  const int32_t stride = n - 1;
  for (int32_t i = lo; i < mid; ++i) {
    peer[i * stride + len[i]] = i + half;
    vec[i * stride + len[i]] = i + half;
    len[i] += 1;
  }
  for (int32_t j = mid; j < hi; ++j) {
    peer[j * stride + len[j]] = j - half;
    vec[j * stride + len[j]] = j - half;
    len[j] += 1;
  }
  for (int32_t i = lo; i < hi; ++i) {
    const int32_t offset = i < mid ? half : -half;
    for (int32_t k = 0; k < child_len; ++k) {
      peer[i * stride + len[i]] = peer[i * stride + k];
      vec[i * stride + len[i]] = vec[i * stride + k] + offset;
      len[i] += 1;
    }
  }
}

/* generate_work_queues: proj/src/topology.cpp:79-89 */
int32_t orc_work_queues(int32_t n, int32_t* peer, int32_t* vec) {
  if (n < 1 || (n & (n - 1)) != 0) return -1;
  int32_t* len = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  gen_range(0, n, n, peer, vec, len);
  free(len);
  return 0;
}

/* ======================================================================
 * SpMV
 * ====================================================================== */

/* One sub-block partial of row `row` restricted to columns in [cb, ce):
 * BellMatrix::multiply_into's inner loop, proj/src/bell.cpp:87-106 (slots in
 * ascending column order, fresh accumulators per sub-block). */
static void row_partial(const int64_t* row_ptr, const int32_t* cols, const double* vals, int32_t row,
                        int32_t cb, int32_t ce, const double* x, double acc[3]) {
  double a0 = 0, a1 = 0, a2 = 0;
  for (int64_t k = row_ptr[row]; k < row_ptr[row + 1]; ++k) {
    const int32_t c = cols[k];
    if (c < cb || c >= ce) continue;
    const double* v = vals + 9 * k;
    const double x0 = x[3 * c], x1 = x[3 * c + 1], x2 = x[3 * c + 2];
    a0 += v[0] * x0 + v[1] * x1 + v[2] * x2;
    a1 += v[3] * x0 + v[4] * x1 + v[5] * x2;
    a2 += v[6] * x0 + v[7] * x1 + v[8] * x2;
  }
  acc[0] = a0;
  acc[1] = a1;
  acc[2] = a2;
}

/* spmv_partitioned_serial: proj/src/oracle/sparse_oracle.hpp:12-42 — per
 * device the diagonal sub-block product (multiply_into) then the queued
 * sub-blocks in queue order (multiply_accumulate, bell.cpp:108-129). */
void orc_spmv(int32_t rows, const int64_t* row_ptr, const int32_t* cols, const double* vals, int32_t n,
              const double* x, double* y) {
  int32_t* pb = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* pe = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* peer = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n * (n > 1 ? n - 1 : 1)));
  int32_t* vec = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n * (n > 1 ? n - 1 : 1)));
  orc_make_partitions(rows, n, pb, pe);
  if (n > 1) orc_work_queues(n, peer, vec);
  for (int32_t d = 0; d < n; ++d) {
    for (int32_t row = pb[d]; row < pe[d]; ++row) {
      double acc[3];
      row_partial(row_ptr, cols, vals, row, pb[d], pe[d], x, acc);
      y[3 * row] = acc[0];
      y[3 * row + 1] = acc[1];
      y[3 * row + 2] = acc[2];
      for (int32_t k = 0; k < n - 1; ++k) {
        const int32_t q = vec[d * (n - 1) + k];
        row_partial(row_ptr, cols, vals, row, pb[q], pe[q], x, acc);
        y[3 * row] += acc[0];
        y[3 * row + 1] += acc[1];
        y[3 * row + 2] += acc[2];
      }
    }
  }
  free(pb);
  free(pe);
  free(peer);
  free(vec);
}

/* ======================================================================
 * PCG: proj/include/weft/solver.hpp:36-178
 * ====================================================================== */

/* Eigen 3x3 inverse by cofactors as in oracle/shim/Eigen/Dense
 * (Matrix::inverse), used at solver.hpp:62. m, out row-major. */
static void inv3(const double* m, double* out) {
#define M(i, j) m[(i) * 3 + (j)]
#define COF(i, j)                                                                                   \
  (M(((i) + 1) % 3, ((j) + 1) % 3) * M(((i) + 2) % 3, ((j) + 2) % 3) -                              \
   M(((i) + 1) % 3, ((j) + 2) % 3) * M(((i) + 2) % 3, ((j) + 1) % 3))
  const double c00 = COF(0, 0), c10 = COF(1, 0), c20 = COF(2, 0);
  const double det = (c00 * M(0, 0) + c10 * M(1, 0)) + c20 * M(2, 0);
  const double invdet = 1.0 / det;
  out[0] = c00 * invdet;
  out[1] = c10 * invdet;
  out[2] = c20 * invdet;
  out[3] = COF(0, 1) * invdet;
  out[4] = COF(1, 1) * invdet;
  out[5] = COF(2, 1) * invdet;
  out[6] = COF(0, 2) * invdet;
  out[7] = COF(1, 2) * invdet;
  out[8] = COF(2, 2) * invdet;
#undef COF
#undef M
}

/* dot + Engine::all_reduce_sum: solver.hpp:91-100, exec.cpp:170-174 */
static double pdot(const double* u, const double* v, int32_t n, const int32_t* pb, const int32_t* pe) {
  double sum = 0.0;
  for (int32_t d = 0; d < n; ++d) {
    double acc = 0.0;
    for (int64_t i = 3 * (int64_t)pb[d]; i < 3 * (int64_t)pe[d]; ++i) acc += u[i] * v[i];
    sum += acc;
  }
  return sum;
}

int32_t orc_pcg(int32_t rows, const int64_t* row_ptr, const int32_t* cols, const double* vals, int32_t n,
                const double* b, double* x, const weft_pcg_config* cfg, weft_pcg_report* rep, char* err) {
  const int64_t len = 3 * (int64_t)rows;
  int32_t* pb = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* pe = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  orc_make_partitions(rows, n, pb, pe);
  double* r = (double*)calloc((size_t)len + 1, sizeof(double));
  double* z = (double*)calloc((size_t)len + 1, sizeof(double));
  double* p = (double*)calloc((size_t)len + 1, sizeof(double));
  double* q = (double*)calloc((size_t)len + 1, sizeof(double));
  double* dinv = (double*)calloc(9 * (size_t)rows + 1, sizeof(double));
  int32_t status = 0;
  const int bj = cfg->preconditioner == WEFT_PRECOND_BLOCK_JACOBI;

  /* block-Jacobi inverse of the diagonal blocks: solver.hpp:49-65 */
  if (bj) {
    for (int32_t row = 0; row < rows; ++row) {
      double m[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
      for (int64_t k = row_ptr[row]; k < row_ptr[row + 1]; ++k) {
        if (cols[k] == row) {
          memcpy(m, vals + 9 * k, sizeof(m));
          break;
        }
      }
      inv3(m, dinv + 9 * (size_t)row);
    }
  }
  /* apply_precond: solver.hpp:67-89 */
#define PRECOND(in, out)                                                         \
  do {                                                                           \
    if (!bj) {                                                                   \
      memcpy(out, in, sizeof(double) * (size_t)len);                             \
    } else {                                                                     \
      for (int32_t row_ = 0; row_ < rows; ++row_) {                              \
        const double* mi = dinv + 9 * (size_t)row_;                              \
        for (int i_ = 0; i_ < 3; ++i_) {                                         \
          double acc_ = 0.0;                                                     \
          for (int j_ = 0; j_ < 3; ++j_) acc_ += mi[i_ * 3 + j_] * in[3 * row_ + j_]; \
          out[3 * row_ + i_] = acc_;                                             \
        }                                                                        \
      }                                                                          \
    }                                                                            \
  } while (0)

  const double b_norm = sqrt(pdot(b, b, n, pb, pe));
  for (int64_t i = 0; i < len; ++i) x[i] = 0.0;
  rep->iterations = 0;
  rep->converged = 0;
  rep->rel_residual = 0.0;
  if (b_norm == 0.0) {
    rep->converged = 1;
    goto done;
  }
  memcpy(r, b, sizeof(double) * (size_t)len);
  PRECOND(r, z);
  memcpy(p, z, sizeof(double) * (size_t)len);
  double rho = pdot(r, z, n, pb, pe);
  const double tol = cfg->rel_tolerance * b_norm;
  double r_norm = b_norm;
  for (int32_t it = 1; it <= cfg->max_iterations; ++it) {
    orc_spmv(rows, row_ptr, cols, vals, n, p, q);
    const double pq = pdot(p, q, n, pb, pe);
    if (!isfinite(pq)) {
      snprintf(err, 256, "pcg: non-finite curvature at iteration %d", it);
      status = 2;
      goto done;
    }
    if (pq <= 0.0) {
      snprintf(err, 256, "pcg: non-positive curvature at iteration %d (matrix not SPD)", it);
      status = 2;
      goto done;
    }
    const double alpha = rho / pq;
    for (int64_t i = 0; i < len; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * q[i];
    }
    r_norm = sqrt(pdot(r, r, n, pb, pe));
    if (!isfinite(r_norm)) {
      snprintf(err, 256, "pcg: divergence (non-finite residual) at iteration %d", it);
      status = 2;
      goto done;
    }
    rep->iterations = it;
    if (rep->residual_history) rep->residual_history[it - 1] = r_norm / b_norm;
    PRECOND(r, z);
    const double rho_next = pdot(r, z, n, pb, pe);
    if (rep->precond_norm_history) rep->precond_norm_history[it - 1] = sqrt(rho_next > 0.0 ? rho_next : 0.0);
    if (r_norm <= tol) {
      rep->converged = 1;
      break;
    }
    const double beta = rho_next / rho;
    rho = rho_next;
    for (int64_t i = 0; i < len; ++i) p[i] = z[i] + beta * p[i];
  }
  rep->rel_residual = r_norm / b_norm;
#undef PRECOND
done:
  free(pb);
  free(pe);
  free(r);
  free(z);
  free(p);
  free(q);
  free(dinv);
  return status;
}

/* ======================================================================
 * Elements: proj/src/elements.cpp
 * ====================================================================== */

typedef struct {
  double v[3];
} v3;

static inline v3 mk(double a, double b, double c) {
  v3 r = {{a, b, c}};
  return r;
}
static inline v3 ld3(const double* x, int32_t i) { return mk(x[3 * i], x[3 * i + 1], x[3 * i + 2]); }
static inline v3 add3(v3 a, v3 b) { return mk(a.v[0] + b.v[0], a.v[1] + b.v[1], a.v[2] + b.v[2]); }
static inline v3 sub3(v3 a, v3 b) { return mk(a.v[0] - b.v[0], a.v[1] - b.v[1], a.v[2] - b.v[2]); }
static inline v3 scl3(double s, v3 a) { return mk(s * a.v[0], s * a.v[1], s * a.v[2]); }
static inline double dot3(v3 a, v3 b) { return a.v[0] * b.v[0] + a.v[1] * b.v[1] + a.v[2] * b.v[2]; }
static inline v3 cross3(v3 a, v3 b) {
  return mk(a.v[1] * b.v[2] - a.v[2] * b.v[1], a.v[2] * b.v[0] - a.v[0] * b.v[2],
            a.v[0] * b.v[1] - a.v[1] * b.v[0]);
}
static inline double norm3(v3 a) { return sqrt(dot3(a, a)); }
static inline v3 div3(v3 a, double s) { return mk(a.v[0] / s, a.v[1] / s, a.v[2] / s); }

#define KDEG 1e-24 /* kDegenerateNormal2, elements.cpp:9 */

/* Forward-mode dual number: elements.cpp:13-30 */
typedef struct {
  double v, d;
} dual;
static inline dual dadd(dual a, dual b) { return (dual){a.v + b.v, a.d + b.d}; }
static inline dual dsub(dual a, dual b) { return (dual){a.v - b.v, a.d - b.d}; }
static inline dual dmul(dual a, dual b) { return (dual){a.v * b.v, a.d * b.v + a.v * b.d}; }
static inline dual ddiv(dual a, dual b) { return (dual){a.v / b.v, (a.d * b.v - a.v * b.d) / (b.v * b.v)}; }
static inline dual dneg(dual a) { return (dual){-a.v, -a.d}; }
static inline dual dsq(dual a) {
  const double s = sqrt(a.v);
  return (dual){s, a.d / (2.0 * s)};
}

/* dihedral_gradient_t<double>: elements.cpp:66-90 */
static void dihedral_gradient(const v3 x[4], v3 g[4]) {
  const v3 e = sub3(x[1], x[0]);
  const v3 na = cross3(e, sub3(x[2], x[0]));
  const v3 nb = cross3(sub3(x[3], x[0]), e);
  const double na2 = dot3(na, na), nb2 = dot3(nb, nb);
  const double elen = sqrt(dot3(e, e));
  for (int i = 0; i < 4; ++i) g[i] = mk(0, 0, 0);
  if (na2 < KDEG || nb2 < KDEG || elen < 1e-12) return;
  const double sa = -elen / na2, sb = -elen / nb2;
  g[2] = mk(na.v[0] * sa, na.v[1] * sa, na.v[2] * sa);
  g[3] = mk(nb.v[0] * sb, nb.v[1] * sb, nb.v[2] * sb);
  const double ca0 = dot3(sub3(x[1], x[2]), e) / (elen * na2);
  const double cb0 = dot3(sub3(x[1], x[3]), e) / (elen * nb2);
  const double ca1 = dot3(sub3(x[2], x[0]), e) / (elen * na2);
  const double cb1 = dot3(sub3(x[3], x[0]), e) / (elen * nb2);
  for (int c = 0; c < 3; ++c) {
    g[0].v[c] = na.v[c] * ca0 + nb.v[c] * cb0;
    g[1].v[c] = na.v[c] * ca1 + nb.v[c] * cb1;
  }
}

/* dihedral_gradient_t<Dual>: same formula over duals (elements.cpp:66-90) */
static void dihedral_gradient_dual(const dual x[4][3], dual g[4][3]) {
  dual e[3], t[3], na[3], nb[3];
  for (int c = 0; c < 3; ++c) e[c] = dsub(x[1][c], x[0][c]);
  for (int c = 0; c < 3; ++c) t[c] = dsub(x[2][c], x[0][c]);
  na[0] = dsub(dmul(e[1], t[2]), dmul(e[2], t[1]));
  na[1] = dsub(dmul(e[2], t[0]), dmul(e[0], t[2]));
  na[2] = dsub(dmul(e[0], t[1]), dmul(e[1], t[0]));
  for (int c = 0; c < 3; ++c) t[c] = dsub(x[3][c], x[0][c]);
  nb[0] = dsub(dmul(t[1], e[2]), dmul(t[2], e[1]));
  nb[1] = dsub(dmul(t[2], e[0]), dmul(t[0], e[2]));
  nb[2] = dsub(dmul(t[0], e[1]), dmul(t[1], e[0]));
  const dual na2 = dadd(dadd(dmul(na[0], na[0]), dmul(na[1], na[1])), dmul(na[2], na[2]));
  const dual nb2 = dadd(dadd(dmul(nb[0], nb[0]), dmul(nb[1], nb[1])), dmul(nb[2], nb[2]));
  const dual elen = dsq(dadd(dadd(dmul(e[0], e[0]), dmul(e[1], e[1])), dmul(e[2], e[2])));
  for (int i = 0; i < 4; ++i)
    for (int c = 0; c < 3; ++c) g[i][c] = (dual){0.0, 0.0};
  if (na2.v < KDEG || nb2.v < KDEG || elen.v < 1e-12) return;
  const dual sa = ddiv(dneg(elen), na2), sb = ddiv(dneg(elen), nb2);
  for (int c = 0; c < 3; ++c) {
    g[2][c] = dmul(na[c], sa);
    g[3][c] = dmul(nb[c], sb);
  }
  dual d12[3], d13[3], d20[3], d30[3];
  for (int c = 0; c < 3; ++c) {
    d12[c] = dsub(x[1][c], x[2][c]);
    d13[c] = dsub(x[1][c], x[3][c]);
    d20[c] = dsub(x[2][c], x[0][c]);
    d30[c] = dsub(x[3][c], x[0][c]);
  }
#define DDOT(a, b) dadd(dadd(dmul(a[0], b[0]), dmul(a[1], b[1])), dmul(a[2], b[2]))
  const dual ca0 = ddiv(DDOT(d12, e), dmul(elen, na2));
  const dual cb0 = ddiv(DDOT(d13, e), dmul(elen, nb2));
  const dual ca1 = ddiv(DDOT(d20, e), dmul(elen, na2));
  const dual cb1 = ddiv(DDOT(d30, e), dmul(elen, nb2));
#undef DDOT
  for (int c = 0; c < 3; ++c) {
    g[0][c] = dadd(dmul(na[c], ca0), dmul(nb[c], cb0));
    g[1][c] = dadd(dmul(na[c], ca1), dmul(nb[c], cb1));
  }
}

/* dihedral_angle: elements.cpp:94-104 */
double orc_dihedral_angle(const double* x0, const double* x1, const double* x2, const double* x3) {
  const v3 p0 = mk(x0[0], x0[1], x0[2]), p1 = mk(x1[0], x1[1], x1[2]);
  const v3 p2 = mk(x2[0], x2[1], x2[2]), p3 = mk(x3[0], x3[1], x3[2]);
  const v3 e = sub3(p1, p0);
  const v3 na = cross3(e, sub3(p2, p0));
  const v3 nb = cross3(sub3(p3, p0), e);
  const double elen = norm3(e);
  if (dot3(na, na) < KDEG || dot3(nb, nb) < KDEG || elen < 1e-12) return 0.0;
  const double s = dot3(cross3(na, nb), e) / elen;
  const double c = dot3(na, nb);
  return atan2(s, c);
}

/* dihedral_hessian: elements.cpp:131-159 (12 dual sweeps, symmetrized) */
static void dihedral_hessian(const v3 x[4], double* h /* 144, block (a,b) at (a*4+b)*9 */) {
  double hess[12][12];
  for (int j = 0; j < 12; ++j) {
    dual xd[4][3];
    for (int v = 0; v < 4; ++v)
      for (int c = 0; c < 3; ++c) xd[v][c] = (dual){x[v].v[c], (3 * v + c == j) ? 1.0 : 0.0};
    dual gd[4][3];
    dihedral_gradient_dual(xd, gd);
    for (int i = 0; i < 12; ++i) hess[i][j] = gd[i / 3][i % 3].d;
  }
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b)
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
          h[(a * 4 + b) * 9 + r * 3 + c] = 0.5 * (hess[3 * a + r][3 * b + c] + hess[3 * b + c][3 * a + r]);
}

/* stretch_state: elements.cpp:133-141 */
typedef struct {
  v3 wu, wv;
  double wu_len, wv_len;
  int ok;
} stretch_st;
static stretch_st stretch_state(const double* d, v3 x0, v3 x1, v3 x2) {
  stretch_st st;
  st.wu = add3(add3(scl3(d[0], x0), scl3(d[1], x1)), scl3(d[2], x2));
  st.wv = add3(add3(scl3(d[3], x0), scl3(d[4], x1)), scl3(d[5], x2));
  st.wu_len = norm3(st.wu);
  st.wv_len = norm3(st.wv);
  st.ok = st.wu_len > 1e-12 && st.wv_len > 1e-12;
  return st;
}

#define F(i, c) force[(i) * 3 + (c)]
#define J(a, b, r, c) jac[((a) * 4 + (b)) * 9 + (r) * 3 + (c)]

/* element_force: elements.cpp:320-340 (kernels :161-181, :232-242,
 * :269-279, :295-303). force[] must be zeroed (ElementForces ctor). */
void orc_element_force(const weft_element* e, const double* x, double* force) {
  const double* d = e->data;
  const int32_t* s = e->stencil;
  for (int i = 0; i < 12; ++i) force[i] = 0.0;
  switch (e->kind) {
    case WEFT_STRETCH: { /* stretch_force :161-181 */
      const stretch_st st = stretch_state(d, ld3(x, s[0]), ld3(x, s[1]), ld3(x, s[2]));
      if (!st.ok) return;
      const v3 wu_hat = div3(st.wu, st.wu_len), wv_hat = div3(st.wv, st.wv_len);
      const double a = d[6];
      const double cu = a * (st.wu_len - 1.0), cv = a * (st.wv_len - 1.0), cs = a * dot3(st.wu, st.wv);
      for (int i = 0; i < 3; ++i) {
        const v3 gu = scl3(a * d[i], wu_hat);
        const v3 gv = scl3(a * d[3 + i], wv_hat);
        const v3 gs = scl3(a, add3(scl3(d[i], st.wv), scl3(d[3 + i], st.wu)));
        const double su = -(d[7] * cu), sv = d[8] * cv, ss = d[9] * cs;
        for (int c = 0; c < 3; ++c) F(i, c) = F(i, c) + ((su * gu.v[c] - sv * gv.v[c]) - ss * gs.v[c]);
      }
      return;
    }
    case WEFT_BEND: { /* bend_force :232-242 */
      v3 xs[4] = {ld3(x, s[0]), ld3(x, s[1]), ld3(x, s[2]), ld3(x, s[3])};
      const double theta = orc_dihedral_angle(xs[0].v, xs[1].v, xs[2].v, xs[3].v);
      v3 g[4];
      dihedral_gradient(xs, g);
      const double coeff = -d[1] * (theta - d[0]);
      for (int i = 0; i < 4; ++i)
        for (int c = 0; c < 3; ++c) F(i, c) = F(i, c) + coeff * g[i].v[c];
      return;
    }
    case WEFT_SPRING: { /* spring_force :269-279 */
      const v3 dd = sub3(ld3(x, s[1]), ld3(x, s[0]));
      const double len = norm3(dd);
      if (len < 1e-12) return;
      const v3 dir = div3(dd, len);
      const v3 fa = scl3(d[1] * (len - d[0]), dir);
      for (int c = 0; c < 3; ++c) {
        F(0, c) = F(0, c) + fa.v[c];
        F(1, c) = F(1, c) - fa.v[c];
      }
      return;
    }
    case WEFT_EXTERNAL: /* :335-337 (assignment, not accumulation) */
      for (int c = 0; c < 3; ++c) F(0, c) = d[c];
      return;
    case WEFT_CONTACT: { /* contact_force :295-303 */
      const v3 nrm = mk(d[0], d[1], d[2]);
      double gap = d[7];
      for (int i = 0; i < e->stencil_size; ++i) gap += d[3 + i] * dot3(nrm, ld3(x, s[i]));
      if (gap >= d[8]) return;
      const double mag = d[9] * (d[8] - gap);
      for (int i = 0; i < e->stencil_size; ++i)
        for (int c = 0; c < 3; ++c) F(i, c) = F(i, c) + (mag * d[3 + i]) * nrm.v[c];
      return;
    }
  }
}

/* element_jacobian: elements.cpp:342-361. jac[] zeroed (ElementJacobian). */
void orc_element_jacobian(const weft_element* e, const double* x, int32_t mode, double* jac) {
  const double* d = e->data;
  const int32_t* s = e->stencil;
  for (int i = 0; i < 144; ++i) jac[i] = 0.0;
  const int exact = mode == WEFT_JAC_EXACT;
  switch (e->kind) {
    case WEFT_STRETCH: { /* stretch_jacobian :183-230 */
      const stretch_st st = stretch_state(d, ld3(x, s[0]), ld3(x, s[1]), ld3(x, s[2]));
      if (!st.ok) return;
      const v3 wu_hat = div3(st.wu, st.wu_len), wv_hat = div3(st.wv, st.wv_len);
      const double a = d[6];
      const double cu = a * (st.wu_len - 1.0), cv = a * (st.wv_len - 1.0), cs = a * dot3(st.wu, st.wv);
      double pu[9], pv[9];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          const double id = r == c ? 1.0 : 0.0;
          pu[r * 3 + c] = id - wu_hat.v[r] * wu_hat.v[c];
          pv[r * 3 + c] = id - wv_hat.v[r] * wv_hat.v[c];
        }
      const int keep_u2 = exact || cu >= 0.0, keep_v2 = exact || cv >= 0.0, keep_s2 = exact;
      for (int i = 0; i < 3; ++i) {
        const double ui = d[i], vi = d[3 + i];
        const v3 gui = scl3(a * ui, wu_hat), gvi = scl3(a * vi, wv_hat);
        const v3 gsi = scl3(a, add3(scl3(ui, st.wv), scl3(vi, st.wu)));
        for (int j = 0; j < 3; ++j) {
          const double uj = d[j], vj = d[3 + j];
          const v3 guj = scl3(a * uj, wu_hat), gvj = scl3(a * vj, wv_hat);
          const v3 gsj = scl3(a, add3(scl3(uj, st.wv), scl3(vj, st.wu)));
          const double su2 = (d[7] * cu) * (((a * ui) * uj) / st.wu_len);
          const double sv2 = (d[8] * cv) * (((a * vi) * vj) / st.wv_len);
          const double ss2 = (d[9] * cs) * (a * (ui * vj + vi * uj));
          for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
              double m = 0.0;
              m = m - d[7] * (gui.v[r] * guj.v[c]);
              m = m - d[8] * (gvi.v[r] * gvj.v[c]);
              m = m - d[9] * (gsi.v[r] * gsj.v[c]);
              if (keep_u2) m = m - su2 * pu[r * 3 + c];
              if (keep_v2) m = m - sv2 * pv[r * 3 + c];
              if (keep_s2) m = m - ss2 * (r == c ? 1.0 : 0.0);
              J(i, j, r, c) = J(i, j, r, c) + m;
            }
        }
      }
      return;
    }
    case WEFT_BEND: { /* bend_jacobian :244-267 */
      v3 xs[4] = {ld3(x, s[0]), ld3(x, s[1]), ld3(x, s[2]), ld3(x, s[3])};
      v3 g[4];
      dihedral_gradient(xs, g);
      double hess[144];
      double dtheta = 0.0;
      if (exact) {
        dtheta = orc_dihedral_angle(xs[0].v, xs[1].v, xs[2].v, xs[3].v) - d[0];
        dihedral_hessian(xs, hess);
      }
      const double nk = -d[1];
      for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j)
          for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
              double m = nk * (g[i].v[r] * g[j].v[c]);
              if (exact) m = m - (d[1] * dtheta) * hess[(i * 4 + j) * 9 + r * 3 + c];
              J(i, j, r, c) = J(i, j, r, c) + m;
            }
      return;
    }
    case WEFT_SPRING: { /* spring_jacobian :281-293 */
      const v3 dd = sub3(ld3(x, s[1]), ld3(x, s[0]));
      const double len = norm3(dd);
      if (len < 1e-12) return;
      const v3 dir = div3(dd, len);
      double lateral = 1.0 - d[0] / len;
      if (!exact) lateral = lateral > 0.0 ? lateral : 0.0; /* std::max(0.0, lateral) */
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          const double oo = dir.v[r] * dir.v[c];
          const double k = d[1] * (oo + lateral * ((r == c ? 1.0 : 0.0) - oo));
          J(0, 0, r, c) = J(0, 0, r, c) - k;
          J(1, 1, r, c) = J(1, 1, r, c) - k;
          J(0, 1, r, c) = J(0, 1, r, c) + k;
          J(1, 0, r, c) = J(1, 0, r, c) + k;
        }
      return;
    }
    case WEFT_EXTERNAL:
      return;
    case WEFT_CONTACT: { /* contact_jacobian :305-316 */
      const v3 nrm = mk(d[0], d[1], d[2]);
      double gap = d[7];
      for (int i = 0; i < e->stencil_size; ++i) gap += d[3 + i] * dot3(nrm, ld3(x, s[i]));
      if (gap >= d[8]) return;
      for (int i = 0; i < e->stencil_size; ++i)
        for (int j = 0; j < e->stencil_size; ++j) {
          const double k = (d[9] * d[3 + i]) * d[3 + j];
          for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) J(i, j, r, c) = J(i, j, r, c) - k * (nrm.v[r] * nrm.v[c]);
        }
      return;
    }
  }
}

/* element_friction_force: elements.cpp:363-382 */
void orc_element_friction(const weft_element* e, const double* vel, double* force) {
  const double* d = e->data;
  for (int i = 0; i < 12; ++i) force[i] = 0.0;
  if (e->kind == WEFT_EXTERNAL) {
    if (d[3] > 0.0) {
      const v3 v = ld3(vel, e->stencil[0]);
      for (int c = 0; c < 3; ++c) F(0, c) = -d[3] * v.v[c];
    }
    return;
  }
  if (e->kind != WEFT_CONTACT) return;
  if (d[11] <= 0.0) return;
  v3 rel = mk(d[13], d[14], d[15]);
  for (int i = 0; i < e->stencil_size; ++i) rel = add3(rel, scl3(d[3 + i], ld3(vel, e->stencil[i])));
  const v3 nrm = mk(d[0], d[1], d[2]);
  const double rn = dot3(nrm, rel);
  const v3 tang = sub3(rel, scl3(rn, nrm));
  const v3 fr = scl3(-d[11], tang);
  for (int i = 0; i < e->stencil_size; ++i)
    for (int c = 0; c < 3; ++c) F(i, c) = d[3 + i] * fr.v[c];
}

/* element_has_velocity_damping: elements.cpp:384-387 */
int32_t orc_element_has_damping(const weft_element* e) {
  if (e->kind == WEFT_EXTERNAL) return e->data[3] > 0.0;
  return e->kind == WEFT_CONTACT && e->data[11] > 0.0;
}

/* element_velocity_damping: elements.cpp:389-403 (adds into jac) */
void orc_element_velocity_damping(const weft_element* e, double* jac) {
  if (!orc_element_has_damping(e)) return;
  const double* d = e->data;
  if (e->kind == WEFT_EXTERNAL) {
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) J(0, 0, r, c) = J(0, 0, r, c) + d[3] * (r == c ? 1.0 : 0.0);
    return;
  }
  for (int i = 0; i < e->stencil_size; ++i)
    for (int j = 0; j < e->stencil_size; ++j) {
      const double k = (d[11] * d[3 + i]) * d[3 + j];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
          J(i, j, r, c) = J(i, j, r, c) + k * ((r == c ? 1.0 : 0.0) - d[r] * d[c]);
    }
}
#undef F
#undef J

/* ======================================================================
 * Assembly: fill_matrix (assembly.hpp:74-220) restated globally
 * ====================================================================== */

static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

int32_t orc_fill_matrix(int32_t p, int64_t n_elem, const weft_element* elems, const double* x_cur,
                        const double* x_adv, const double* vel, const double* mass, const uint8_t* pinned,
                        double dt, int32_t mode, orc_system* out, char* err) {
  memset(out, 0, sizeof(*out));
  if (dt <= 0.0) { /* assembly.hpp:81 */
    snprintf(err, 256, "fill_matrix: dt must be positive");
    return 1;
  }
  /* distribute_elements stencil check: assembly.cpp:18-22 */
  for (int64_t id = 0; id < n_elem; ++id) {
    for (int a = 0; a < elems[id].stencil_size; ++a) {
      const int32_t v = elems[id].stencil[a];
      if (v < 0 || v >= p) {
        snprintf(err, 256, "element %lld: stencil vertex %d outside all partitions", (long long)id, v);
        return 1;
      }
    }
  }
  /* (1)-(3) pattern: diagonal + non-pinned stencil pairs, sorted unique
   * (assembly.hpp:93-134). */
  int64_t* cap = (int64_t*)calloc((size_t)p + 1, sizeof(int64_t));
  for (int32_t r = 0; r < p; ++r) cap[r + 1] = 1;
  for (int64_t id = 0; id < n_elem; ++id) {
    const weft_element* e = &elems[id];
    for (int a = 0; a < e->stencil_size; ++a) cap[e->stencil[a] + 1] += e->stencil_size;
  }
  for (int32_t r = 0; r < p; ++r) cap[r + 1] += cap[r];
  int32_t* raw = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap[p] + 1));
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(p + 1));
  for (int32_t r = 0; r < p; ++r) {
    cur[r] = cap[r];
    raw[cur[r]++] = r;
  }
  for (int64_t id = 0; id < n_elem; ++id) {
    const weft_element* e = &elems[id];
    for (int a = 0; a < e->stencil_size; ++a) {
      const int32_t rv = e->stencil[a];
      if (pinned[rv]) continue;
      for (int b = 0; b < e->stencil_size; ++b) {
        const int32_t cv = e->stencil[b];
        if (pinned[cv]) continue;
        raw[cur[rv]++] = cv;
      }
    }
  }
  out->rows = p;
  out->row_ptr = (int64_t*)calloc((size_t)p + 1, sizeof(int64_t));
  for (int32_t r = 0; r < p; ++r) {
    int32_t* first = raw + cap[r];
    const int64_t cnt = cur[r] - cap[r];
    qsort(first, (size_t)cnt, sizeof(int32_t), cmp_i32);
    int64_t u = 0;
    for (int64_t k = 0; k < cnt; ++k)
      if (k == 0 || first[k] != first[u - 1]) first[u++] = first[k];
    cur[r] = u;
    out->row_ptr[r + 1] = out->row_ptr[r] + u;
  }
  out->nnzb = out->row_ptr[p];
  out->cols = (int32_t*)malloc(sizeof(int32_t) * (size_t)(out->nnzb + 1));
  out->vals = (double*)calloc(9 * (size_t)out->nnzb + 1, sizeof(double));
  out->rhs = (double*)calloc(3 * (size_t)p + 1, sizeof(double));
  for (int32_t r = 0; r < p; ++r) memcpy(out->cols + out->row_ptr[r], raw + cap[r], sizeof(int32_t) * (size_t)cur[r]);
  free(raw);
  free(cur);
  free(cap);

  /* slot lookup: find_slot (bell.cpp:78-85) on the sorted row */
#define SLOT(row, col)                                                               \
  ({                                                                                 \
    int64_t s_ = -1;                                                                 \
    for (int64_t k_ = out->row_ptr[row]; k_ < out->row_ptr[(row) + 1]; ++k_)         \
      if (out->cols[k_] == (col)) {                                                  \
        s_ = k_;                                                                     \
        break;                                                                       \
      }                                                                              \
    s_;                                                                              \
  })

  /* (5) mass diagonal: assembly.hpp:155-166 */
  for (int32_t r = 0; r < p; ++r) {
    const int pin = pinned[r] != 0;
    if (!pin && mass[r] <= 0.0) {
      snprintf(err, 256, "fill_matrix: vertex %d has non-positive mass", r);
      orc_free_system(out);
      return 1;
    }
    const double m = pin ? 1.0 : mass[r];
    const int64_t k = SLOT(r, r);
    for (int c = 0; c < 3; ++c) out->vals[9 * k + c * 3 + c] += m;
  }
  /* (5) element values in ascending element order: assembly.hpp:168-216 */
  double force[12], jac[144], fric[12], vd[144];
  for (int64_t id = 0; id < n_elem; ++id) {
    const weft_element* e = &elems[id];
    orc_element_force(e, x_adv, force);
    orc_element_jacobian(e, x_cur, mode, jac);
    orc_element_friction(e, vel, fric);
    const double scale = dt * dt + e->damping * dt;
    const int damped = orc_element_has_damping(e);
    if (damped) {
      for (int i = 0; i < 144; ++i) vd[i] = 0.0;
      orc_element_velocity_damping(e, vd);
    }
    for (int a = 0; a < e->stencil_size; ++a) {
      const int32_t row = e->stencil[a];
      if (pinned[row]) continue;
      double f[3];
      for (int c = 0; c < 3; ++c) f[c] = force[a * 3 + c] + fric[a * 3 + c];
      if (e->damping > 0.0) {
        for (int b = 0; b < e->stencil_size; ++b) {
          const double* m = jac + (a * 4 + b) * 9;
          const v3 vb = ld3(vel, e->stencil[b]);
          for (int c = 0; c < 3; ++c) {
            const double mv = m[c * 3 + 0] * vb.v[0] + m[c * 3 + 1] * vb.v[1] + m[c * 3 + 2] * vb.v[2];
            f[c] = f[c] + e->damping * mv;
          }
        }
      }
      for (int c = 0; c < 3; ++c) out->rhs[3 * row + c] += dt * f[c];
      for (int b = 0; b < e->stencil_size; ++b) {
        const int32_t col = e->stencil[b];
        if (pinned[col]) continue;
        const int64_t k = SLOT(row, col);
        const double* m = jac + (a * 4 + b) * 9;
        for (int i = 0; i < 9; ++i) {
          double cval = -scale * m[i];
          if (damped) cval = cval + dt * vd[(a * 4 + b) * 9 + i];
          out->vals[9 * k + i] += cval;
        }
      }
    }
  }
#undef SLOT
  return 0;
}

void orc_free_system(orc_system* s) {
  free(s->row_ptr);
  free(s->cols);
  free(s->vals);
  free(s->rhs);
  memset(s, 0, sizeof(*s));
}

/* ======================================================================
 * Broad phase: collision.cpp:16-25, 77-192, 205-210, 329-378
 * ====================================================================== */

#define LAT_BIAS ((int64_t)1 << 20)

/* clamp_lattice: collision.cpp:16-19 (x86-64 cvttsd2si semantics for
 * out-of-range conversions: INT64_MIN, then clamped). */
static int64_t clamp_lattice(double v) {
  const double f = floor(v);
  int64_t i;
  if (!(f >= -9223372036854775808.0 && f < 9223372036854775808.0)) i = INT64_MIN;
  else i = (int64_t)f;
  if (i < -LAT_BIAS + 1) i = -LAT_BIAS + 1;
  if (i > LAT_BIAS - 1) i = LAT_BIAS - 1;
  return i;
}

/* pack_cell: collision.cpp:21-25 */
static uint64_t pack_cell(int64_t ix, int64_t iy, int64_t iz) {
  return ((uint64_t)(ix + LAT_BIAS) << 42) | ((uint64_t)(iy + LAT_BIAS) << 21) | (uint64_t)(iz + LAT_BIAS);
}

typedef struct {
  uint64_t key;
  int32_t tri;
  int64_t order;
} cell_entry;

static int cmp_entry(const void* a, const void* b) {
  const cell_entry* x = (const cell_entry*)a;
  const cell_entry* y = (const cell_entry*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return (x->order > y->order) - (x->order < y->order);
}

void orc_build_grid(int32_t tri_count, const int32_t* tris, const double* x0, const double* x1, int32_t mode,
                    double thickness, double cell_scale, orc_grid* out) {
  memset(out, 0, sizeof(*out));
  out->tri_count = tri_count;
  const int ccd = mode == WEFT_CONTINUOUS;
  const double inflate = ccd ? 1e-9 : 0.5 * thickness; /* :122 */
  double* lo = (double*)malloc(sizeof(double) * 3 * (size_t)(tri_count + 1));
  double* hi = (double*)malloc(sizeof(double) * 3 * (size_t)(tri_count + 1));
  /* triangle_query_box :77-91 and the serial diagonal sum :124-133 */
  double diag_sum = 0.0;
  for (int32_t t = 0; t < tri_count; ++t) {
    double l[3] = {1e300, 1e300, 1e300}, h[3] = {-1e300, -1e300, -1e300};
    for (int k = 0; k < 3; ++k) {
      const int32_t v = tris[3 * t + k];
      for (int c = 0; c < 3; ++c) {
        const double p0 = x0[3 * v + c];
        l[c] = p0 < l[c] ? p0 : l[c];
        h[c] = h[c] < p0 ? p0 : h[c];
        if (ccd) {
          const double p1 = x1[3 * v + c];
          l[c] = p1 < l[c] ? p1 : l[c];
          h[c] = h[c] < p1 ? p1 : h[c];
        }
      }
    }
    for (int c = 0; c < 3; ++c) {
      l[c] = l[c] - inflate;
      h[c] = h[c] + inflate;
      lo[3 * t + c] = l[c];
      hi[3 * t + c] = h[c];
    }
    const double dx = h[0] - l[0], dy = h[1] - l[1], dz = h[2] - l[2];
    diag_sum += sqrt(dx * dx + dy * dy + dz * dz);
  }
  const double mean_diag = tri_count > 0 ? diag_sum / tri_count : 1.0;
  double cell = cell_scale * mean_diag;
  if (!(cell >= 1e-9)) cell = cell < 1e-9 ? 1e-9 : cell; /* std::max(cell, 1e-9) */
  out->cell_size = cell;
  /* lattice boxes + cell memberships :139-163 */
  out->tri_boxes = (int64_t*)malloc(sizeof(int64_t) * 6 * (size_t)(tri_count + 1));
  int64_t n_entries = 0;
  for (int32_t t = 0; t < tri_count; ++t) {
    int64_t* lat = out->tri_boxes + 6 * (size_t)t;
    for (int c = 0; c < 3; ++c) {
      lat[c] = clamp_lattice(lo[3 * t + c] / cell);
      lat[c + 3] = clamp_lattice(hi[3 * t + c] / cell);
    }
    n_entries += (lat[3] - lat[0] + 1) * (lat[4] - lat[1] + 1) * (lat[5] - lat[2] + 1);
  }
  cell_entry* ent = (cell_entry*)malloc(sizeof(cell_entry) * (size_t)(n_entries + 1));
  int64_t k = 0;
  for (int32_t t = 0; t < tri_count; ++t) {
    const int64_t* lat = out->tri_boxes + 6 * (size_t)t;
    for (int64_t ix = lat[0]; ix <= lat[3]; ++ix)
      for (int64_t iy = lat[1]; iy <= lat[4]; ++iy)
        for (int64_t iz = lat[2]; iz <= lat[5]; ++iz) {
          ent[k].key = pack_cell(ix, iy, iz);
          ent[k].tri = t;
          ent[k].order = k;
          ++k;
        }
  }
  qsort(ent, (size_t)n_entries, sizeof(cell_entry), cmp_entry);
  int64_t cells = 0;
  for (int64_t i = 0; i < n_entries; ++i)
    if (i == 0 || ent[i].key != ent[i - 1].key) ++cells;
  out->cells = cells;
  out->cell_keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(cells + 1));
  out->cell_offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cells + 1));
  out->cell_tris = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_entries + 1));
  out->prefix = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cells + 1));
  int64_t c = -1;
  for (int64_t i = 0; i < n_entries; ++i) {
    if (i == 0 || ent[i].key != ent[i - 1].key) {
      ++c;
      out->cell_keys[c] = ent[i].key;
      out->cell_offsets[c] = i;
    }
    out->cell_tris[i] = ent[i].tri;
  }
  out->cell_offsets[cells] = n_entries;
  /* WorkloadTable :165-177 */
  out->prefix[0] = 0;
  for (int64_t i = 0; i < cells; ++i) {
    const int64_t cnt = out->cell_offsets[i + 1] - out->cell_offsets[i];
    out->prefix[i + 1] = out->prefix[i] + cnt * (cnt - 1) / 2;
  }
  out->total = out->prefix[cells];
  free(ent);
  free(lo);
  free(hi);
}

/* narrow_phase_range walk (collision.cpp:329-378) with the min-common-cell
 * rule (:205-210, :366-369); emits the candidate pairs instead of running
 * the (out-of-scope) elementary tests. */
int64_t orc_candidates(const orc_grid* g, int64_t begin, int64_t end, int32_t* pairs) {
  if (begin >= end) return 0;
  /* upper_bound(prefix, begin) - 1 */
  int64_t lo = 0, hi = g->cells + 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (g->prefix[mid] <= begin) lo = mid + 1;
    else hi = mid;
  }
  int64_t cell = lo - 1;
  int64_t local = begin - g->prefix[cell];
  int32_t s = (int32_t)(g->cell_offsets[cell + 1] - g->cell_offsets[cell]);
  int32_t i = 0;
  int64_t remaining = local;
  while (remaining >= s - 1 - i) {
    remaining -= s - 1 - i;
    ++i;
  }
  int32_t j = i + 1 + (int32_t)remaining;
  int64_t count = 0;
  for (int64_t gi = begin; gi < end; ++gi) {
    while (gi >= g->prefix[cell + 1]) {
      ++cell;
      i = 0;
      j = 1;
    }
    const int32_t* tris = g->cell_tris + g->cell_offsets[cell];
    const int32_t size = (int32_t)(g->cell_offsets[cell + 1] - g->cell_offsets[cell]);
    const int32_t t1 = tris[i], t2 = tris[j];
    const int64_t* a = g->tri_boxes + 6 * (size_t)t1;
    const int64_t* b = g->tri_boxes + 6 * (size_t)t2;
    const uint64_t key = pack_cell(a[0] > b[0] ? a[0] : b[0], a[1] > b[1] ? a[1] : b[1], a[2] > b[2] ? a[2] : b[2]);
    if (key == g->cell_keys[cell]) {
      if (pairs) {
        pairs[2 * count] = t1;
        pairs[2 * count + 1] = t2;
      }
      ++count;
    }
    if (++j >= size) {
      ++i;
      j = i + 1;
    }
  }
  return count;
}

void orc_free_grid(orc_grid* g) {
  free(g->tri_boxes);
  free(g->cell_keys);
  free(g->cell_offsets);
  free(g->cell_tris);
  free(g->prefix);
  memset(g, 0, sizeof(*g));
}

/* ======================================================================
 * oracle::Rng = std::mt19937_64 + top-53-bit uniform (oracle.hpp:19-43)
 * ====================================================================== */

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i) r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

uint64_t orc_rng_raw(orc_rng* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

double orc_rng_uniform(orc_rng* r, double lo, double hi) {
  const double u = (double)(orc_rng_raw(r) >> 11) * 0x1.0p-53;
  return lo + (hi - lo) * u;
}

int32_t orc_rng_uniform_int(orc_rng* r, int32_t lo, int32_t hi) {
  return lo + (int32_t)(orc_rng_raw(r) % (uint64_t)(hi - lo + 1));
}
