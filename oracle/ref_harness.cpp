// ref_harness.cpp — C-ABI over the UNMODIFIED reference engine (TEST
// INFRASTRUCTURE). Compiled with the reference sources into
// oracle/_ref/libweft_ref.so by `make -C oracle ref`; loaded via ctypes by
// tests/ (parity checks and golden-fixture generation) and by bench.py's
// reference arm. It only marshals flat arrays into the reference's own types
// and calls the reference's public functions; no algorithm lives here except
// the candidate-pair walk, which replays narrow_phase_range's loop
// (proj/src/collision.cpp:329-378) over the reference's own HashGrid because
// the reference does not expose candidates separately.
#include <chrono>
#include <cstring>
#include <algorithm>
#include <memory>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "oracle/physics_oracle.hpp"
#include "oracle/sparse_oracle.hpp"
#include "oracle/collision_oracle.hpp"
#include "weft/assembly.hpp"
#include "weft/collision.hpp"
#include "weft/mesh.hpp"
#include "weft/physics.hpp"
#include "weft/response.hpp"
#include "weft/solver.hpp"
#include "weft/scene.hpp"
#include "weft/driver.hpp"

#include "../include/weft_gpu.h"

using namespace weft;

namespace {

thread_local std::string g_err;

AssemblyElement to_element(const weft_element& f) {
  AssemblyElement e;
  e.kind = static_cast<ElementKind>(f.kind);
  e.stencil_size = f.stencil_size;
  for (int i = 0; i < 4; ++i) e.stencil[static_cast<std::size_t>(i)] = f.stencil[i];
  e.damping = f.damping;
  const double* d = f.data;
  switch (e.kind) {
    case ElementKind::Stretch: {
      StretchData s;
      s.pwu = {d[0], d[1], d[2]};
      s.pwv = {d[3], d[4], d[5]};
      s.area = d[6];
      s.k_warp = d[7];
      s.k_weft = d[8];
      s.k_shear = d[9];
      e.data = s;
      break;
    }
    case ElementKind::Bend:
      e.data = BendData{d[0], d[1]};
      break;
    case ElementKind::Spring:
      e.data = SpringData{d[0], d[1]};
      break;
    case ElementKind::External:
      e.data = ExternalData{Vec3(d[0], d[1], d[2]), d[3]};
      break;
    case ElementKind::Contact: {
      ContactData c;
      c.normal = Vec3(d[0], d[1], d[2]);
      c.w = {d[3], d[4], d[5], d[6]};
      c.bias = d[7];
      c.activation = d[8];
      c.stiffness = d[9];
      c.friction = d[10];
      c.tangential_damping = d[11];
      c.frozen_normal_force = d[12];
      c.rel_vel_bias = Vec3(d[13], d[14], d[15]);
      e.data = c;
      break;
    }
  }
  return e;
}

weft_element from_element(const AssemblyElement& e) {
  weft_element f{};
  f.kind = static_cast<int32_t>(e.kind);
  f.stencil_size = e.stencil_size;
  for (int i = 0; i < 4; ++i) f.stencil[i] = e.stencil[static_cast<std::size_t>(i)];
  f.damping = e.damping;
  double* d = f.data;
  switch (e.kind) {
    case ElementKind::Stretch: {
      const auto& s = std::get<StretchData>(e.data);
      for (int i = 0; i < 3; ++i) {
        d[i] = s.pwu[static_cast<std::size_t>(i)];
        d[3 + i] = s.pwv[static_cast<std::size_t>(i)];
      }
      d[6] = s.area;
      d[7] = s.k_warp;
      d[8] = s.k_weft;
      d[9] = s.k_shear;
      break;
    }
    case ElementKind::Bend: {
      const auto& b = std::get<BendData>(e.data);
      d[0] = b.rest_angle;
      d[1] = b.stiffness;
      break;
    }
    case ElementKind::Spring: {
      const auto& s = std::get<SpringData>(e.data);
      d[0] = s.rest_length;
      d[1] = s.stiffness;
      break;
    }
    case ElementKind::External: {
      const auto& x = std::get<ExternalData>(e.data);
      for (int i = 0; i < 3; ++i) d[i] = x.force[i];
      d[3] = x.drag;
      break;
    }
    case ElementKind::Contact: {
      const auto& c = std::get<ContactData>(e.data);
      for (int i = 0; i < 3; ++i) d[i] = c.normal[i];
      for (int i = 0; i < 4; ++i) d[3 + i] = c.w[static_cast<std::size_t>(i)];
      d[7] = c.bias;
      d[8] = c.activation;
      d[9] = c.stiffness;
      d[10] = c.friction;
      d[11] = c.tangential_damping;
      d[12] = c.frozen_normal_force;
      for (int i = 0; i < 3; ++i) d[13 + i] = c.rel_vel_bias[i];
      break;
    }
  }
  return f;
}

std::vector<Vec3> to_vec3(const double* x, int count) {
  std::vector<Vec3> out(static_cast<std::size_t>(count));
  for (int i = 0; i < count; ++i) out[static_cast<std::size_t>(i)] = Vec3(x[3 * i], x[3 * i + 1], x[3 * i + 2]);
  return out;
}

struct Csr {
  int rows = 0;
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> cols;
  std::vector<double> vals;
  std::vector<double> rhs;
};

template <class Real = double>
Csr from_bell(const BellMatrix<Real>& a) {
  Csr c;
  c.rows = a.block_rows();
  c.row_ptr.assign(static_cast<std::size_t>(c.rows) + 1, 0);
  for (int r = 0; r < c.rows; ++r) {
    for (int s = 0; s < a.ell_width(); ++s) {
      const int32_t col = a.col_at(r, s);
      if (col == BellMatrix<Real>::kNoBlock) break;
      c.cols.push_back(col);
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) c.vals.push_back(a.value_at(r, s, i, j));
    }
    c.row_ptr[static_cast<std::size_t>(r) + 1] = static_cast<int64_t>(c.cols.size());
  }
  return c;
}

template <class Real = double>
BellMatrix<Real> to_bell(int rows, const int64_t* row_ptr, const int32_t* cols, const Real* vals) {
  std::vector<BlockEntry<Real>> entries;
  for (int r = 0; r < rows; ++r) {
    for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
      BlockEntry<Real> e;
      e.row = r;
      e.col = cols[k];
      for (int i = 0; i < 9; ++i) e.m[static_cast<std::size_t>(i)] = vals[9 * k + i];
      entries.push_back(e);
    }
  }
  return BellMatrix<Real>::from_entries(rows, entries);
}

ValidatedSchedule schedule_for(int n) {
  return n == 1 ? ValidatedSchedule() : ValidatedSchedule(generate_work_queues(FatTree::make(n)), n);
}

int set_error(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const SolverError*>(&e)) return WEFT_ERR_SOLVER;
  if (dynamic_cast<const DimensionError*>(&e)) return WEFT_ERR_DIMENSION;
  if (dynamic_cast<const ExecError*>(&e)) return WEFT_ERR_EXEC;
  if (dynamic_cast<const TopologyError*>(&e)) return WEFT_ERR_TOPOLOGY;
  if (dynamic_cast<const ScheduleError*>(&e)) return WEFT_ERR_SCHEDULE;
  if (dynamic_cast<const ZoneFailure*>(&e)) return WEFT_ERR_ZONE;
  return WEFT_ERR_INVALID;
}

struct MeshHandle {
  ClothMesh mesh;
};

struct GridHandle {
  GridBuildResult built;
  std::vector<int64_t> offsets;
  std::vector<int32_t> flat;
};

}  // namespace

namespace {
// Candidate pairs of [begin, end): the loop of narrow_phase_range
// (collision.cpp:340-376) with narrow_phase_pair replaced by emission.
int64_t ref_grid_candidates_impl(const GridBuildResult& built, int64_t begin, int64_t end, int32_t* pairs = nullptr) {
  const auto& grid = built.grid;
  const auto& table = built.table;
  if (begin >= end) return 0;
  std::size_t cell = static_cast<std::size_t>(
      std::upper_bound(table.prefix.begin(), table.prefix.end(), begin) - table.prefix.begin() - 1);
  const std::int64_t local = begin - table.prefix[cell];
  int i = 0, j = 0;
  {
    const int s = static_cast<int>(grid.cell_tris[cell].size());
    std::int64_t remaining = local;
    while (remaining >= s - 1 - i) {
      remaining -= s - 1 - i;
      ++i;
    }
    j = i + 1 + static_cast<int>(remaining);
  }
  int64_t count = 0;
  for (std::int64_t gi = begin; gi < end; ++gi) {
    while (gi >= table.prefix[cell + 1]) {
      ++cell;
      i = 0;
      j = 1;
    }
    const auto& tl = grid.cell_tris[cell];
    const int t1 = tl[static_cast<std::size_t>(i)];
    const int t2 = tl[static_cast<std::size_t>(j)];
    const auto& a = grid.tri_boxes[static_cast<std::size_t>(t1)];
    const auto& b = grid.tri_boxes[static_cast<std::size_t>(t2)];
    constexpr std::int64_t bias = 1 << 20;
    const std::uint64_t key = (static_cast<std::uint64_t>(std::max(a[0], b[0]) + bias) << 42) |
                              (static_cast<std::uint64_t>(std::max(a[1], b[1]) + bias) << 21) |
                              static_cast<std::uint64_t>(std::max(a[2], b[2]) + bias);
    if (key == grid.cell_keys[cell]) {
      if (pairs) {
        pairs[2 * count] = t1;
        pairs[2 * count + 1] = t2;
      }
      ++count;
    }
    if (++j >= static_cast<int>(tl.size())) {
      ++i;
      j = i + 1;
    }
  }
  return count;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- systems
}  // extern "C"
template <class Real>
void* ref_fill_matrix_t(int32_t p, int32_t n, int64_t n_elem, const weft_element* elems, const double* x_cur,
                        const double* x_adv, const double* vel, const double* mass, const uint8_t* pinned,
                        double dt, int32_t mode, int32_t* status) {
  try {
    std::vector<AssemblyElement> elements;
    elements.reserve(static_cast<std::size_t>(n_elem));
    for (int64_t i = 0; i < n_elem; ++i) elements.push_back(to_element(elems[i]));
    const auto xc = to_vec3(x_cur, p), xa = to_vec3(x_adv, p), v = to_vec3(vel, p);
    std::vector<double> m(mass, mass + p);
    std::vector<uint8_t> pin(pinned, pinned + p);
    SystemInputs in;
    in.elements = elements;
    in.x_current = xc;
    in.x_advanced = xa;
    in.velocity = v;
    in.mass = m;
    in.pinned = pin;
    in.dt = dt;
    in.mode = mode == WEFT_JAC_EXACT ? JacobianMode::Exact : JacobianMode::SpdProjected;
    Engine engine(n);
    const auto parts = make_partitions(p, n);
    const auto dist = distribute_elements(elements, parts);
    const auto sys = fill_matrix<Real>(engine, dist, in, parts);
    auto* out = new Csr(from_bell<Real>(gather_matrix(sys.matrix)));  // float values exact in double
    const auto rg = sys.rhs.gather();
    out->rhs.assign(rg.begin(), rg.end());
    *status = 0;
    return out;
  } catch (const std::exception& e) {
    *status = set_error(e);
    return nullptr;
  }
}
extern "C" {
void* ref_fill_matrix(int32_t p, int32_t n, int64_t n_elem, const weft_element* elems, const double* x_cur,
                      const double* x_adv, const double* vel, const double* mass, const uint8_t* pinned,
                      double dt, int32_t mode, int32_t* status) {
  return ref_fill_matrix_t<double>(p, n, n_elem, elems, x_cur, x_adv, vel, mass, pinned, dt, mode, status);
}
// fill_matrix<float> (Precision::Single)
void* ref_fill_matrix_f32(int32_t p, int32_t n, int64_t n_elem, const weft_element* elems, const double* x_cur,
                          const double* x_adv, const double* vel, const double* mass, const uint8_t* pinned,
                          double dt, int32_t mode, int32_t* status) {
  return ref_fill_matrix_t<float>(p, n, n_elem, elems, x_cur, x_adv, vel, mass, pinned, dt, mode, status);
}

void ref_system_info(void* h, int32_t* rows, int64_t* nnzb) {
  auto* c = static_cast<Csr*>(h);
  *rows = c->rows;
  *nnzb = static_cast<int64_t>(c->cols.size());
}

void ref_system_copy(void* h, int64_t* row_ptr, int32_t* cols, double* vals, double* rhs) {
  auto* c = static_cast<Csr*>(h);
  if (row_ptr) std::memcpy(row_ptr, c->row_ptr.data(), c->row_ptr.size() * sizeof(int64_t));
  if (cols) std::memcpy(cols, c->cols.data(), c->cols.size() * sizeof(int32_t));
  if (vals) std::memcpy(vals, c->vals.data(), c->vals.size() * sizeof(double));
  if (rhs && !c->rhs.empty()) std::memcpy(rhs, c->rhs.data(), c->rhs.size() * sizeof(double));
}

void ref_system_free(void* h) { delete static_cast<Csr*>(h); }

// oracle::random_bell (src/oracle/sparse_oracle.cpp:7-23) as CSR.
void* ref_random_bell(uint64_t seed, int32_t rows, int32_t extra) {
  oracle::Rng rng(seed);
  return new Csr(from_bell(oracle::random_bell(rng, rows, extra)));
}

// ---------------------------------------------------------------- SpMV/PCG
}  // extern "C"
template <class Real>
int32_t ref_spmv_t(int32_t rows, const int64_t* row_ptr, const int32_t* cols, const Real* vals, int32_t n,
                   const Real* x, Real* y) {
  try {
    const auto global = to_bell<Real>(rows, row_ptr, cols, vals);
    const auto parts = make_partitions(rows, n);
    const auto split = partition_matrix(global, parts);
    Engine engine(n);
    const auto sched = schedule_for(n);
    DistVector<Real> xv(&engine, parts), yv(&engine, parts);
    for (int d = 0; d < n; ++d) {
      const auto& part = parts[static_cast<std::size_t>(d)];
      std::copy(x + 3 * part.begin, x + 3 * part.end, xv.local(d).begin());
    }
    SpmvWorkspace<Real> ws(n, split.padded_len);
    spmv_pipelined(engine, split, sched, xv, yv, ws);
    const auto yg = yv.gather();
    std::copy(yg.begin(), yg.end(), y);
    return 0;
  } catch (const std::exception& e) {
    return set_error(e);
  }
}

template <class Real>
int32_t ref_pcg_t(int32_t rows, const int64_t* row_ptr, const int32_t* cols, const Real* vals, int32_t n,
                  const Real* b, Real* x, const weft_pcg_config* cfg, weft_pcg_report* rep) {
  try {
    const auto global = to_bell<Real>(rows, row_ptr, cols, vals);
    const auto parts = make_partitions(rows, n);
    const auto split = partition_matrix(global, parts);
    Engine engine(n);
    const auto sched = schedule_for(n);
    DistVector<Real> bv(&engine, parts), xv(&engine, parts);
    for (int d = 0; d < n; ++d) {
      const auto& part = parts[static_cast<std::size_t>(d)];
      std::copy(b + 3 * part.begin, b + 3 * part.end, bv.local(d).begin());
    }
    PcgConfig config;
    config.rel_tolerance = cfg->rel_tolerance;
    config.max_iterations = cfg->max_iterations;
    config.preconditioner =
        cfg->preconditioner == WEFT_PRECOND_NONE ? Preconditioner::None : Preconditioner::BlockJacobi;
    const auto r = pcg_solve(engine, split, sched, bv, xv, config);
    const auto xg = xv.gather();
    std::copy(xg.begin(), xg.end(), x);
    rep->iterations = r.iterations;
    rep->converged = r.converged ? 1 : 0;
    rep->rel_residual = r.rel_residual;
    if (rep->residual_history)
      std::copy(r.residual_history.begin(), r.residual_history.end(), rep->residual_history);
    if (rep->precond_norm_history)
      std::copy(r.precond_norm_history.begin(), r.precond_norm_history.end(), rep->precond_norm_history);
    return 0;
  } catch (const std::exception& e) {
    return set_error(e);
  }
}

extern "C" {
int32_t ref_spmv(int32_t rows, const int64_t* row_ptr, const int32_t* cols, const double* vals, int32_t n,
                 const double* x, double* y) {
  return ref_spmv_t<double>(rows, row_ptr, cols, vals, n, x, y);
}
int32_t ref_pcg(int32_t rows, const int64_t* row_ptr, const int32_t* cols, const double* vals, int32_t n,
                const double* b, double* x, const weft_pcg_config* cfg, weft_pcg_report* rep) {
  return ref_pcg_t<double>(rows, row_ptr, cols, vals, n, b, x, cfg, rep);
}
// Precision::Single: spmv_pipelined<float>, pcg_solve<float>
int32_t ref_spmv_f32(int32_t rows, const int64_t* row_ptr, const int32_t* cols, const float* vals, int32_t n,
                     const float* x, float* y) {
  return ref_spmv_t<float>(rows, row_ptr, cols, vals, n, x, y);
}
int32_t ref_pcg_f32(int32_t rows, const int64_t* row_ptr, const int32_t* cols, const float* vals, int32_t n,
                    const float* b, float* x, const weft_pcg_config* cfg, weft_pcg_report* rep) {
  return ref_pcg_t<float>(rows, row_ptr, cols, vals, n, b, x, cfg, rep);
}

// ---------------------------------------------------------------- meshes
void* ref_grid_mesh(int32_t nx, int32_t ny, double w, double h, double ox, double oy, double oz, double density) {
  try {
    return new MeshHandle{make_grid_mesh(nx, ny, w, h, Vec3(ox, oy, oz), density)};
  } catch (const std::exception& e) {
    set_error(e);
    return nullptr;
  }
}

void* ref_build_mesh(int32_t nverts, const double* verts, int32_t ntris, const int32_t* tris, double density) {
  try {
    std::vector<std::array<int, 3>> t(static_cast<std::size_t>(ntris));
    for (int i = 0; i < ntris; ++i) t[static_cast<std::size_t>(i)] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
    return new MeshHandle{ClothMesh::build(to_vec3(verts, nverts), std::move(t), density)};
  } catch (const std::exception& e) {
    set_error(e);
    return nullptr;
  }
}

// oracle::random_cloth (src/oracle/physics_oracle.cpp:90-101).
void* ref_random_cloth(uint64_t seed, int32_t max_side) {
  oracle::Rng rng(seed);
  return new MeshHandle{oracle::random_cloth(rng, max_side)};
}

void ref_mesh_info(void* h, int32_t* verts, int32_t* tris, int32_t* hinges, int32_t* edges) {
  const auto& m = static_cast<MeshHandle*>(h)->mesh;
  *verts = m.vertex_count();
  *tris = m.triangle_count();
  *hinges = static_cast<int32_t>(m.hinges.size());
  *edges = static_cast<int32_t>(m.edges.size());
}

// rest (3/v), tris (3/t), tri_rest (7/t: pwu, pwv, area; degenerate flag
// in tri_degenerate), hinges (4 ints + rest_angle + stiffness_scale),
// vertex_area, vertex_mass. Any pointer may be NULL.
void ref_mesh_copy(void* h, double* rest, int32_t* tris, double* tri_rest, uint8_t* tri_degenerate,
                   int32_t* hinge_verts, double* hinge_data, double* vertex_area, double* vertex_mass) {
  const auto& m = static_cast<MeshHandle*>(h)->mesh;
  for (int v = 0; v < m.vertex_count() && rest; ++v)
    for (int c = 0; c < 3; ++c) rest[3 * v + c] = m.rest_positions[static_cast<std::size_t>(v)][c];
  for (int t = 0; t < m.triangle_count(); ++t) {
    const auto& tr = m.triangles[static_cast<std::size_t>(t)];
    const auto& r = m.tri_rest[static_cast<std::size_t>(t)];
    for (int c = 0; c < 3; ++c) {
      if (tris) tris[3 * t + c] = tr[static_cast<std::size_t>(c)];
      if (tri_rest) {
        tri_rest[7 * t + c] = r.pwu[static_cast<std::size_t>(c)];
        tri_rest[7 * t + 3 + c] = r.pwv[static_cast<std::size_t>(c)];
      }
    }
    if (tri_rest) tri_rest[7 * t + 6] = r.area;
    if (tri_degenerate) tri_degenerate[t] = r.degenerate ? 1 : 0;
  }
  for (std::size_t k = 0; k < m.hinges.size(); ++k) {
    for (int c = 0; c < 4; ++c)
      if (hinge_verts) hinge_verts[4 * k + static_cast<std::size_t>(c)] = m.hinges[k].verts[static_cast<std::size_t>(c)];
    if (hinge_data) {
      hinge_data[2 * k] = m.hinges[k].rest_angle;
      hinge_data[2 * k + 1] = m.hinges[k].stiffness_scale;
    }
  }
  for (int v = 0; v < m.vertex_count(); ++v) {
    if (vertex_area) vertex_area[v] = m.vertex_area[static_cast<std::size_t>(v)];
    if (vertex_mass) vertex_mass[v] = m.vertex_mass[static_cast<std::size_t>(v)];
  }
}

// build_elements (src/physics.cpp:5-63): writes up to `cap` records,
// returns the element count. material: stretch_warp, stretch_weft, shear,
// bend, density, damping, air_drag (physics.hpp:8-16).
int64_t ref_build_elements(void* h, const double* material, const double* gravity, const double* wind,
                           weft_element* out, int64_t cap) {
  const auto& m = static_cast<MeshHandle*>(h)->mesh;
  MaterialParams params;
  params.stretch_warp = material[0];
  params.stretch_weft = material[1];
  params.shear = material[2];
  params.bend = material[3];
  params.density = material[4];
  params.damping = material[5];
  params.air_drag = material[6];
  const auto elements = build_elements(m, params, Vec3(gravity[0], gravity[1], gravity[2]),
                                       Vec3(wind[0], wind[1], wind[2]));
  for (std::size_t i = 0; i < elements.size() && static_cast<int64_t>(i) < cap; ++i) out[i] = from_element(elements[i]);
  return static_cast<int64_t>(elements.size());
}

void ref_mesh_free(void* h) { delete static_cast<MeshHandle*>(h); }

// ---------------------------------------------------------------- elements
void ref_element_eval(const weft_element* fe, int32_t count_x, const double* x, const double* v, int32_t mode,
                      double* force, double* jac, double* fric, double* vdamp) {
  const auto e = to_element(*fe);
  const auto xs = to_vec3(x, count_x), vs = to_vec3(v, count_x);
  const auto f = element_force(e, xs);
  const auto j = element_jacobian(e, xs, mode == WEFT_JAC_EXACT ? JacobianMode::Exact : JacobianMode::SpdProjected);
  const auto fr = element_friction_force(e, vs);
  ElementJacobian vd;
  element_velocity_damping(e, vd);
  for (int a = 0; a < 4; ++a) {
    for (int c = 0; c < 3; ++c) {
      force[3 * a + c] = f.f[static_cast<std::size_t>(a)][c];
      fric[3 * a + c] = fr.f[static_cast<std::size_t>(a)][c];
    }
    for (int b = 0; b < 4; ++b)
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          jac[(a * 4 + b) * 9 + r * 3 + c] = j.block[static_cast<std::size_t>(a)][static_cast<std::size_t>(b)](r, c);
          vdamp[(a * 4 + b) * 9 + r * 3 + c] = vd.block[static_cast<std::size_t>(a)][static_cast<std::size_t>(b)](r, c);
        }
  }
}

// ---------------------------------------------------------------- broad phase
void* ref_build_grid(int32_t vertex_count, int32_t tri_count, const int32_t* tris, const double* x0,
                     const double* x1, int32_t mode, double thickness, double cell_scale) {
  std::vector<std::array<int, 3>> t(static_cast<std::size_t>(tri_count));
  for (int i = 0; i < tri_count; ++i) t[static_cast<std::size_t>(i)] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
  const auto soup = CollisionSoup::build(std::move(t), vertex_count,
                                         std::vector<std::uint8_t>(static_cast<std::size_t>(vertex_count), 1));
  const auto xb = to_vec3(x0, vertex_count);
  const auto xe = to_vec3(x1 ? x1 : x0, vertex_count);
  CollisionParams params;
  params.thickness = thickness;
  params.cell_scale = cell_scale;
  auto* g = new GridHandle{build_grid(soup, xb, xe, mode == WEFT_CONTINUOUS ? CollisionMode::Continuous
                                                                           : CollisionMode::Discrete,
                                      params), {}, {}};
  g->offsets.push_back(0);
  for (const auto& tl : g->built.grid.cell_tris) {
    g->flat.insert(g->flat.end(), tl.begin(), tl.end());
    g->offsets.push_back(static_cast<int64_t>(g->flat.size()));
  }
  return g;
}

void ref_grid_info(void* h, double* cell_size, int64_t* cells, int64_t* entries, int64_t* total) {
  const auto* g = static_cast<GridHandle*>(h);
  *cell_size = g->built.grid.cell_size;
  *cells = static_cast<int64_t>(g->built.grid.cell_keys.size());
  *entries = static_cast<int64_t>(g->flat.size());
  *total = g->built.table.total;
}

void ref_grid_copy(void* h, uint64_t* keys, int64_t* offsets, int32_t* cell_tris, int64_t* prefix, int64_t* boxes) {
  const auto* g = static_cast<GridHandle*>(h);
  const auto& gr = g->built.grid;
  if (keys) std::copy(gr.cell_keys.begin(), gr.cell_keys.end(), keys);
  if (offsets) std::copy(g->offsets.begin(), g->offsets.end(), offsets);
  if (cell_tris) std::copy(g->flat.begin(), g->flat.end(), cell_tris);
  if (prefix) std::copy(g->built.table.prefix.begin(), g->built.table.prefix.end(), prefix);
  if (boxes)
    for (std::size_t t = 0; t < gr.tri_boxes.size(); ++t)
      for (int c = 0; c < 6; ++c) boxes[6 * t + static_cast<std::size_t>(c)] = gr.tri_boxes[t][static_cast<std::size_t>(c)];
}

// split_workload (collision.cpp:181-192) over the reference grid's table.
void ref_grid_split(void* h, int32_t devices, int64_t* begin, int64_t* end) {
  const auto ranges = split_workload(static_cast<GridHandle*>(h)->built.table, devices);
  for (int d = 0; d < devices; ++d) {
    begin[d] = ranges[static_cast<std::size_t>(d)].begin;
    end[d] = ranges[static_cast<std::size_t>(d)].end;
  }
}

int64_t ref_grid_candidates(void* h, int64_t begin, int64_t end, int32_t* pairs) {
  return ref_grid_candidates_impl(static_cast<GridHandle*>(h)->built, begin, end, pairs);
}

void ref_grid_free(void* h) { delete static_cast<GridHandle*>(h); }

// collide (collision.cpp:391-417) with Engine(devices): broad phase, narrow
// phase over every device's pair range, sync_shared_cells. Returns the hit
// count; fills (kind, a, b) triples and (gap | toi, normal, weights) octets
// for up to `cap` hits. movable: NULL = all movable.
int64_t ref_collide(int32_t vertex_count, int32_t tri_count, const int32_t* tris, const uint8_t* movable,
                    const double* x0, const double* x1, int32_t mode, double thickness, double cell_scale,
                    int32_t devices, int64_t cap, int32_t* kab, double* vals) {
  try {
    std::vector<std::array<int, 3>> t(static_cast<std::size_t>(tri_count));
    for (int i = 0; i < tri_count; ++i) t[static_cast<std::size_t>(i)] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
    std::vector<std::uint8_t> mv(static_cast<std::size_t>(vertex_count), 1);
    if (movable) mv.assign(movable, movable + vertex_count);
    const auto soup = CollisionSoup::build(std::move(t), vertex_count, std::move(mv));
    const auto xb = to_vec3(x0, vertex_count);
    const auto xe = to_vec3(x1 ? x1 : x0, vertex_count);
    CollisionParams params;
    params.thickness = thickness;
    params.cell_scale = cell_scale;
    Engine engine(devices);
    const bool ccd = mode == WEFT_CONTINUOUS;
    const auto r = collide(engine, soup, xb, xe, ccd ? CollisionMode::Continuous : CollisionMode::Discrete, params);
    auto emit = [&](const auto& items, auto scalar) -> int64_t {
      const int64_t n = static_cast<int64_t>(items.size());
      for (int64_t i = 0; i < std::min(n, cap); ++i) {
        const auto& h = items[static_cast<std::size_t>(i)];
        if (kab) {
          kab[3 * i] = static_cast<int32_t>(h.kind);
          kab[3 * i + 1] = h.a;
          kab[3 * i + 2] = h.b;
        }
        if (vals) {
          double* o = vals + 8 * i;
          o[0] = scalar(h);
          for (int c = 0; c < 3; ++c) o[1 + c] = h.normal[c];
          for (int c = 0; c < 4; ++c) o[4 + c] = h.weights[static_cast<std::size_t>(c)];
        }
      }
      return n;
    };
    if (ccd) return emit(r.impacts, [](const Impact& h) { return h.toi; });
    return emit(r.proximities, [](const Proximity& h) { return h.gap; });
  } catch (const std::exception& e) {
    set_error(e);
    return -1;
  }
}

// oracle::random_two_cloth_scene (src/oracle/collision_oracle.cpp:110-138).
// Returns vertex count; fills tris (cap) / x_begin / x_end when non-NULL.
int32_t ref_two_cloth_scene(uint64_t seed, int32_t max_side, int32_t* tri_count, int32_t* tris, double* x0,
                            double* x1) {
  oracle::Rng rng(seed);
  const auto s = oracle::random_two_cloth_scene(rng, max_side);
  *tri_count = static_cast<int32_t>(s.soup.triangles.size());
  if (tris)
    for (std::size_t t = 0; t < s.soup.triangles.size(); ++t)
      for (int c = 0; c < 3; ++c) tris[3 * t + static_cast<std::size_t>(c)] = s.soup.triangles[t][static_cast<std::size_t>(c)];
  for (std::size_t v = 0; v < s.x_begin.size(); ++v)
    for (int c = 0; c < 3; ++c) {
      if (x0) x0[3 * v + static_cast<std::size_t>(c)] = s.x_begin[v][c];
      if (x1) x1[3 * v + static_cast<std::size_t>(c)] = s.x_end[v][c];
    }
  return s.soup.vertex_count;
}


static ZoneSolveParams zone_params_from(const double* zp) {
  ZoneSolveParams z;
  z.clearance = zp[0];
  z.initial_penalty = zp[1];
  z.inner_tolerance = zp[2];
  z.al_iterations = static_cast<int>(zp[3]);
  z.inner_iterations = static_cast<int>(zp[4]);
  z.outer_cap = static_cast<int>(zp[5]);
  z.retry_cap = static_cast<int>(zp[6]);
  z.max_correction_factor = zp[7];
  return z;
}

static CollisionSoup soup_from(int32_t vertex_count, int32_t tri_count, const int32_t* tris, const uint8_t* movable) {
  std::vector<std::array<int, 3>> t(static_cast<std::size_t>(tri_count));
  for (int i = 0; i < tri_count; ++i) t[static_cast<std::size_t>(i)] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
  std::vector<std::uint8_t> mv(static_cast<std::size_t>(vertex_count), 1);
  if (movable) mv.assign(movable, movable + vertex_count);
  return CollisionSoup::build(std::move(t), vertex_count, std::move(mv));
}

// build_zones (response.cpp:108-162) over (kind, a, b) triples. Fills
// impact_zone (n), vert_off (zones + 1, up to cap_off), verts (up to
// cap_verts); returns the zone count.
int32_t ref_build_zones(int32_t vertex_count, int32_t tri_count, const int32_t* tris, const uint8_t* movable, int64_t n,
                        const int32_t* kab, int32_t* impact_zone, int64_t cap_off, int32_t* vert_off,
                        int64_t cap_verts, int32_t* verts) {
  try {
    const auto soup = soup_from(vertex_count, tri_count, tris, movable);
    std::vector<Impact> imps(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      auto& h = imps[static_cast<std::size_t>(i)];
      h.kind = kab[3 * i] == 0 ? FeatureKind::VertexFace : FeatureKind::EdgeEdge;
      h.a = kab[3 * i + 1];
      h.b = kab[3 * i + 2];
    }
    const auto zones = build_zones(imps, soup);
    int64_t off = 0;
    for (std::size_t z = 0; z < zones.size(); ++z) {
      for (int i : zones[z].impacts) impact_zone[i] = static_cast<int32_t>(z);
      if (static_cast<int64_t>(z) < cap_off) vert_off[z] = static_cast<int32_t>(off);
      for (int v : zones[z].vertices) {
        if (off < cap_verts) verts[off] = v;
        ++off;
      }
    }
    if (static_cast<int64_t>(zones.size()) < cap_off) vert_off[zones.size()] = static_cast<int32_t>(off);
    return static_cast<int32_t>(zones.size());
  } catch (const std::exception& e) {
    set_error(e);
    return -1;
  }
}

// resolve_zones (response.cpp:338-400) with Engine(devices). x_cand is
// updated in place. zp: clearance, initial_penalty, inner_tolerance,
// al_iterations, inner_iterations, outer_cap, retry_cap,
// max_correction_factor. report: outer_iterations, zone_count,
// max_zone_vertices, impacts_resolved, first_round_impacts.
int32_t ref_resolve_zones(int32_t vertex_count, int32_t tri_count, const int32_t* tris, const uint8_t* movable,
                          const double* mass, const double* x_begin, double* x_cand, double thickness,
                          double cell_scale, int32_t devices, const double* zp, int64_t* report) {
  try {
    const auto soup = soup_from(vertex_count, tri_count, tris, movable);
    const auto xb = to_vec3(x_begin, vertex_count);
    auto xc = to_vec3(x_cand, vertex_count);
    const std::vector<double> m(mass, mass + vertex_count);
    CollisionParams cp;
    cp.thickness = thickness;
    cp.cell_scale = cell_scale;
    Engine engine(devices);
    int32_t status = 0;
    ZoneResolveReport r;
    try {
      r = resolve_zones(engine, soup, xb, xc, m, cp, zone_params_from(zp));
    } catch (const std::exception& e) {
      status = set_error(e);
    }
    for (int v = 0; v < vertex_count; ++v)
      for (int c = 0; c < 3; ++c) x_cand[3 * v + c] = xc[static_cast<std::size_t>(v)][c];
    report[0] = r.outer_iterations;
    report[1] = r.zone_count;
    report[2] = r.max_zone_vertices;
    report[3] = r.impacts_resolved;
    report[4] = r.first_round_impacts;
    return status;
  } catch (const std::exception& e) {
    return set_error(e);
  }
}

}  // extern "C"

// ---------------------------------------------------------------------------
// The reference arm of bench.py: the same hot-path step as weft_gpu_sim_step
// executed by the reference's own functions and Engine threads:
//   collide()'s broad-phase structure (replicated build_grid per device,
//   split_workload, per-device candidate walk; collision.cpp:391-417, with
//   narrow_phase_pair out of scope), step_system<double>, pcg_solve,
//   candidate update, CCD broad phase, commit (driver.cpp:96-215).
// ---------------------------------------------------------------------------
namespace {

struct RefSim {
  ClothMesh mesh;
  std::vector<uint8_t> pinned;
  MaterialParams material;
  CollisionSoup soup;
  SimState state;
  std::unique_ptr<Engine> engine;
  ValidatedSchedule sched;
};

int64_t ref_collide_candidates(RefSim& s, std::span<const Vec3> x0, std::span<const Vec3> x1, CollisionMode mode,
                               const CollisionParams& params, double* grid_ms) {
  const int n = s.engine->devices();
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<GridBuildResult> grids(static_cast<std::size_t>(n));
  s.engine->parallel([&](int d) { grids[static_cast<std::size_t>(d)] = build_grid(s.soup, x0, x1, mode, params); });
  const auto t1 = std::chrono::steady_clock::now();
  *grid_ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
  const auto ranges = split_workload(grids[0].table, n);
  std::vector<int64_t> counts(static_cast<std::size_t>(n), 0);
  s.engine->parallel([&](int d) {
    counts[static_cast<std::size_t>(d)] = ref_grid_candidates_impl(
        grids[static_cast<std::size_t>(d)], ranges[static_cast<std::size_t>(d)].begin, ranges[static_cast<std::size_t>(d)].end);
  });
  int64_t total = 0;
  for (auto c : counts) total += c;
  return total;
}

}  // namespace

extern "C" {

void* ref_sim_create(int32_t nverts, const double* verts, int32_t ntris, const int32_t* tris, const uint8_t* pinned,
                     double density, const double* material, int32_t devices) {
  try {
    auto* s = new RefSim();
    std::vector<std::array<int, 3>> t(static_cast<std::size_t>(ntris));
    for (int i = 0; i < ntris; ++i) t[static_cast<std::size_t>(i)] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
    s->mesh = ClothMesh::build(to_vec3(verts, nverts), t, density);
    s->pinned.assign(pinned, pinned + nverts);
    s->material.stretch_warp = material[0];
    s->material.stretch_weft = material[1];
    s->material.shear = material[2];
    s->material.bend = material[3];
    s->material.density = material[4];
    s->material.damping = material[5];
    s->material.air_drag = material[6];
    std::vector<std::uint8_t> movable(static_cast<std::size_t>(nverts));
    for (int v = 0; v < nverts; ++v) movable[static_cast<std::size_t>(v)] = pinned[v] ? 0 : 1;
    s->soup = CollisionSoup::build(std::move(t), nverts, std::move(movable));
    s->state = SimState::rest(s->mesh);
    s->engine = std::make_unique<Engine>(devices);
    s->sched = schedule_for(devices);
    return s;
  } catch (const std::exception& e) {
    set_error(e);
    return nullptr;
  }
}

void ref_sim_set_state(void* h, const double* x, const double* v) {
  auto* s = static_cast<RefSim*>(h);
  const int p = s->mesh.vertex_count();
  s->state.x = to_vec3(x, p);
  s->state.v = to_vec3(v, p);
}

void ref_sim_get_state(void* h, double* x, double* v) {
  auto* s = static_cast<RefSim*>(h);
  for (std::size_t i = 0; i < s->state.x.size(); ++i)
    for (int c = 0; c < 3; ++c) {
      if (x) x[3 * i + static_cast<std::size_t>(c)] = s->state.x[i][c];
      if (v) v[3 * i + static_cast<std::size_t>(c)] = s->state.v[i][c];
    }
}

// params: dt, thickness, cell_scale, pcg tol, pcg max its. out (8 doubles):
// pcg iterations, converged, residual, dcd candidates, ccd candidates,
// ms broad, ms assemble, ms solve.
int32_t ref_sim_step(void* h, const double* params, double* out) {
  auto* s = static_cast<RefSim*>(h);
  try {
    const double dt = params[0];
    CollisionParams cp;
    cp.thickness = params[1];
    cp.cell_scale = params[2];
    PcgConfig pc;
    pc.rel_tolerance = params[3];
    pc.max_iterations = static_cast<int>(params[4]);
    const int p = s->mesh.vertex_count();
    double broad_ms = 0.0;
    const auto tb0 = std::chrono::steady_clock::now();
    const int64_t dcd = ref_collide_candidates(*s, s->state.x, s->state.x, CollisionMode::Discrete, cp, &broad_ms);
    const auto tb1 = std::chrono::steady_clock::now();
    auto system = step_system<double>(*s->engine, s->mesh, s->state, s->material, s->pinned, {}, dt,
                                      Vec3(0, 0, -9.81), Vec3::Zero());
    const auto ta = std::chrono::steady_clock::now();
    DistVector<double> dv(s->engine.get(), system.matrix.partitions);
    const auto rep = pcg_solve(*s->engine, system.matrix, s->sched, system.rhs, dv, pc);
    const auto tsol = std::chrono::steady_clock::now();
    if (!rep.converged) throw SolverError("PCG did not converge (residual " + std::to_string(rep.rel_residual) + ")");
    const auto dvg = dv.gather();
    std::vector<Vec3> cand(static_cast<std::size_t>(p));
    for (int i = 0; i < p; ++i) {
      for (int c = 0; c < 3; ++c) s->state.v[static_cast<std::size_t>(i)][c] += dvg[static_cast<std::size_t>(3 * i + c)];
      cand[static_cast<std::size_t>(i)] = s->state.x[static_cast<std::size_t>(i)] + dt * s->state.v[static_cast<std::size_t>(i)];
    }
    const auto tc0 = std::chrono::steady_clock::now();
    const int64_t ccd = ref_collide_candidates(*s, s->state.x, cand, CollisionMode::Continuous, cp, &broad_ms);
    const auto tc1 = std::chrono::steady_clock::now();
    s->state.x = std::move(cand);
    s->state.time += dt;
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    out[0] = rep.iterations;
    out[1] = rep.converged ? 1 : 0;
    out[2] = rep.rel_residual;
    out[3] = static_cast<double>(dcd);
    out[4] = static_cast<double>(ccd);
    out[5] = ms(tb0, tb1) + ms(tc0, tc1);
    out[6] = ms(tb1, ta);
    out[7] = ms(ta, tsol);
    return 0;
  } catch (const std::exception& e) {
    return set_error(e);
  }
}

// Per-function CPU medians on the current state (SURVEY.md §8(d) "CPU
// timing"): fill_matrix<double> over step_system's inputs (assembly.hpp:74-220;
// build_elements / distribute_elements done once, outside the timing),
// spmv_pipelined on the assembled system (sparse.hpp:72-101, one global
// y = A x), build_grid in DCD mode on x (collision.cpp:118-179, one build;
// collide() replicates it per device). params: dt, thickness, cell_scale.
// out: median ms of fill_matrix, spmv_pipelined, build_grid.
int32_t ref_sim_time_functions(void* h, const double* params, int32_t reps, double* out) {
  auto* s = static_cast<RefSim*>(h);
  try {
    const double dt = params[0];
    CollisionParams cp;
    cp.thickness = params[1];
    cp.cell_scale = params[2];
    const int p = s->mesh.vertex_count();
    const int n = s->engine->devices();
    const auto elements = build_elements(s->mesh, s->material, Vec3(0, 0, -9.81), Vec3::Zero());
    std::vector<Vec3> adv(static_cast<std::size_t>(p));
    for (int i = 0; i < p; ++i)
      adv[static_cast<std::size_t>(i)] = s->state.x[static_cast<std::size_t>(i)] + dt * s->state.v[static_cast<std::size_t>(i)];
    const auto parts = make_partitions(p, n);
    const auto dist = distribute_elements(elements, parts);
    SystemInputs in;
    in.elements = elements;
    in.x_current = s->state.x;
    in.x_advanced = adv;
    in.velocity = s->state.v;
    in.mass = s->mesh.vertex_mass;
    in.pinned = s->pinned;
    in.dt = dt;
    in.mode = JacobianMode::SpdProjected;
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    auto median = [](std::vector<double> v) {
      std::sort(v.begin(), v.end());
      return v[v.size() / 2];
    };
    std::vector<double> tf, ts, tg;
    std::optional<AssembledSystem<double>> sys;
    for (int r = 0; r < std::max(reps, 1); ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      auto a = fill_matrix<double>(*s->engine, dist, in, parts);
      tf.push_back(ms(t0, std::chrono::steady_clock::now()));
      if (!sys) sys.emplace(std::move(a));
    }
    DistVector<double> x(s->engine.get(), sys->matrix.partitions), y(s->engine.get(), sys->matrix.partitions);
    x.fill(1.0);
    SpmvWorkspace<double> ws(n, sys->matrix.padded_len);
    for (int r = 0; r < std::max(reps, 1); ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      spmv_pipelined(*s->engine, sys->matrix, s->sched, x, y, ws);
      ts.push_back(ms(t0, std::chrono::steady_clock::now()));
    }
    for (int r = 0; r < std::max(reps, 1); ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      const auto g = build_grid(s->soup, s->state.x, s->state.x, CollisionMode::Discrete, cp);
      tg.push_back(ms(t0, std::chrono::steady_clock::now()));
    }
    out[0] = median(tf);
    out[1] = median(ts);
    out[2] = median(tg);
    return 0;
  } catch (const std::exception& e) {
    return set_error(e);
  }
}

// Simulator::step_impl (driver.cpp:96-215) without impact zones: DCD collide
// (broad + narrow phase), proximities_to_elements, step_system with the
// contacts, pcg_solve, candidate update, CCD collide (impacts counted, not
// resolved), commit. params: dt, thickness, cell_scale, pcg tol, pcg max
// its, contact stiffness_scale, friction, contact damping, zones flag, the 8
// zone params (ref_resolve_zones); with the flag set, resolve_zones and the
// commit's velocity correction run too (the full step_impl). out: pcg its,
// converged, residual, proximities, contacts, impacts (first CCD round),
// zone count, zone outer rounds.
int32_t ref_sim_step_contacts(void* h, const double* params, double* out) {
  auto* s = static_cast<RefSim*>(h);
  try {
    const double dt = params[0];
    CollisionParams cp;
    cp.thickness = params[1];
    cp.cell_scale = params[2];
    PcgConfig pc;
    pc.rel_tolerance = params[3];
    pc.max_iterations = static_cast<int>(params[4]);
    ContactParams kp;
    kp.thickness = params[1];
    kp.stiffness_scale = params[5];
    kp.friction = params[6];
    kp.damping = params[7];
    const int p = s->mesh.vertex_count();
    const auto dcd = collide(*s->engine, s->soup, s->state.x, s->state.x, CollisionMode::Discrete, cp);
    auto contacts = proximities_to_elements(dcd.proximities, s->soup, s->state.x, s->state.v, s->mesh.vertex_mass,
                                            dt, kp);
    const auto ncontacts = contacts.size();
    auto system = step_system<double>(*s->engine, s->mesh, s->state, s->material, s->pinned, std::move(contacts), dt,
                                      Vec3(0, 0, -9.81), Vec3::Zero());
    DistVector<double> dv(s->engine.get(), system.matrix.partitions);
    const auto rep = pcg_solve(*s->engine, system.matrix, s->sched, system.rhs, dv, pc);
    if (!rep.converged) throw SolverError("PCG did not converge (residual " + std::to_string(rep.rel_residual) + ")");
    const auto dvg = dv.gather();
    std::vector<Vec3> cand(static_cast<std::size_t>(p));
    for (int i = 0; i < p; ++i) {
      for (int c = 0; c < 3; ++c) s->state.v[static_cast<std::size_t>(i)][c] += dvg[static_cast<std::size_t>(3 * i + c)];
      cand[static_cast<std::size_t>(i)] = s->state.x[static_cast<std::size_t>(i)] + dt * s->state.v[static_cast<std::size_t>(i)];
    }
    const auto ccd = collide(*s->engine, s->soup, s->state.x, cand, CollisionMode::Continuous, cp);
    if (params[8] != 0.0) {
      // 5-7. resolve_zones + the commit's velocity correction (driver.cpp:181-204)
      const std::vector<Vec3> pre = cand;
      const auto zr = resolve_zones(*s->engine, s->soup, s->state.x, cand, s->mesh.vertex_mass, cp,
                                    zone_params_from(params + 9));
      for (int i = 0; i < p; ++i)
        if (cand[static_cast<std::size_t>(i)] != pre[static_cast<std::size_t>(i)])
          s->state.v[static_cast<std::size_t>(i)] += (cand[static_cast<std::size_t>(i)] - pre[static_cast<std::size_t>(i)]) / dt;
      out[6] = zr.zone_count;
      out[7] = zr.outer_iterations;
    }
    s->state.x = std::move(cand);
    s->state.time += dt;
    out[0] = rep.iterations;
    out[1] = rep.converged ? 1 : 0;
    out[2] = rep.rel_residual;
    out[3] = static_cast<double>(dcd.proximities.size());
    out[4] = static_cast<double>(ncontacts);
    out[5] = static_cast<double>(ccd.impacts.size());
    return 0;
  } catch (const std::exception& e) {
    return set_error(e);
  }
}

void ref_sim_free(void* h) { delete static_cast<RefSim*>(h); }

}  // extern "C"

// ---------------------------------------------------------------------------
// Scenes (scene.cpp) and the reference Simulator (driver.cpp): parity of the
// scene loader and of whole simulation runs.
// ---------------------------------------------------------------------------
namespace {
struct SceneHandle {
  Scene scene;
  std::unique_ptr<Simulator> sim;
  std::ostringstream log;  // the Simulator's EngineOptions::instrument stream
  bool instrument = false;
};
}  // namespace

extern "C" {

// load_scene (scene.cpp:167-178) from a file, or parse_scene from text when
// `is_text` (base_dir for relative OBJ paths).
void* ref_scene_load(const char* path_or_text, int32_t is_text, const char* base_dir) {
  try {
    auto* h = new SceneHandle();
    h->scene = is_text ? parse_scene(path_or_text, base_dir ? base_dir : ".") : load_scene(path_or_text);
    return h;
  } catch (const std::exception& e) {
    set_error(e);
    return nullptr;
  }
}

// counts: cloth verts, cloth tris, obstacles, then per obstacle (verts, tris, keyframes) up to cap_obs
void ref_scene_info(void* hp, int32_t* counts, int32_t cap_obs) {
  const auto& sc = static_cast<SceneHandle*>(hp)->scene;
  counts[0] = sc.cloth.vertex_count();
  counts[1] = static_cast<int32_t>(sc.cloth.triangles.size());
  counts[2] = static_cast<int32_t>(sc.obstacles.size());
  for (int o = 0; o < std::min<int>(cap_obs, static_cast<int>(sc.obstacles.size())); ++o) {
    counts[3 + 3 * o] = static_cast<int32_t>(sc.obstacles[static_cast<std::size_t>(o)].shape.vertices.size());
    counts[4 + 3 * o] = static_cast<int32_t>(sc.obstacles[static_cast<std::size_t>(o)].shape.triangles.size());
    counts[5 + 3 * o] = static_cast<int32_t>(sc.obstacles[static_cast<std::size_t>(o)].keyframes.size());
  }
}

// config doubles: dt, frames, devices, gravity xyz, wind xyz, seed, material (7: warp, weft, shear, bend,
// density, damping, air_drag), thickness, cell_scale, stiffness_scale, friction, clearance_fraction,
// contact damping, pcg tol, pcg max its, preconditioner, zone outer_cap, zone initial_penalty, precision
void ref_scene_config(void* hp, double* cfg) {
  const auto& c = static_cast<SceneHandle*>(hp)->scene.config;
  double v[] = {c.dt, (double)c.frames, (double)c.devices, c.gravity.x(), c.gravity.y(), c.gravity.z(), c.wind.x(),
                c.wind.y(), c.wind.z(), (double)c.seed, c.material.stretch_warp, c.material.stretch_weft,
                c.material.shear, c.material.bend, c.material.density, c.material.damping, c.material.air_drag,
                c.collision.thickness, c.collision.cell_scale, c.contact.stiffness_scale, c.contact.friction,
                c.contact.clearance_fraction, c.contact.damping, c.solver.rel_tolerance,
                (double)c.solver.max_iterations, c.solver.preconditioner == Preconditioner::BlockJacobi ? 1.0 : 0.0,
                (double)c.zones.outer_cap, c.zones.initial_penalty,
                c.precision == Precision::Double ? 1.0 : 0.0};
  std::memcpy(cfg, v, sizeof(v));
}

// cloth rest positions (3 per vertex), triangles, pinned flags; obstacle o's shape
void ref_scene_cloth(void* hp, double* verts, int32_t* tris, uint8_t* pinned) {
  const auto& sc = static_cast<SceneHandle*>(hp)->scene;
  for (std::size_t i = 0; i < sc.cloth.rest_positions.size(); ++i)
    for (int c = 0; c < 3; ++c) verts[3 * i + static_cast<std::size_t>(c)] = sc.cloth.rest_positions[i][c];
  for (std::size_t t = 0; t < sc.cloth.triangles.size(); ++t)
    for (int c = 0; c < 3; ++c) tris[3 * t + static_cast<std::size_t>(c)] = sc.cloth.triangles[t][static_cast<std::size_t>(c)];
  std::memcpy(pinned, sc.pinned.data(), sc.pinned.size());
}

// obstacle o: its vertex positions at time t (Obstacle::positions_at), triangles
void ref_scene_obstacle(void* hp, int32_t o, double t, double* verts, int32_t* tris) {
  const auto& ob = static_cast<SceneHandle*>(hp)->scene.obstacles[static_cast<std::size_t>(o)];
  const auto pos = ob.positions_at(t);
  for (std::size_t i = 0; i < pos.size(); ++i)
    for (int c = 0; c < 3; ++c) verts[3 * i + static_cast<std::size_t>(c)] = pos[i][c];
  if (tris)
    for (std::size_t k = 0; k < ob.shape.triangles.size(); ++k)
      for (int c = 0; c < 3; ++c) tris[3 * k + static_cast<std::size_t>(c)] = ob.shape.triangles[k][static_cast<std::size_t>(c)];
}

// Simulator(scene) with `devices` engine devices (<= 0: the scene's), then step():
// out = frame, time, pcg its, pcg residual, proximities, contacts, impacts, zones, zone_outer, committed.
int32_t ref_scene_step(void* hp, int32_t devices, double* out) {
  auto* h = static_cast<SceneHandle*>(hp);
  try {
    if (!h->sim) {
      SimConfig cfg = h->scene.config;
      if (devices > 0) cfg.devices = devices;
      h->sim = std::make_unique<Simulator>(h->scene.cloth, h->scene.pinned, h->scene.obstacles, cfg,
                                           h->instrument ? &h->log : nullptr);
    }
    const auto r = h->sim->step();
    const double v[] = {(double)r.frame, r.time, (double)r.pcg_iterations, r.pcg_residual, (double)r.proximities,
                        (double)r.contacts, (double)r.impacts, (double)r.zone_count, (double)r.zone_outer,
                        r.committed ? 1.0 : 0.0};
    std::memcpy(out, v, sizeof(v));
    return 0;
  } catch (const std::exception& e) {
    return set_error(e);
  }
}

void ref_scene_state(void* hp, double* x, double* v) {
  auto* h = static_cast<SceneHandle*>(hp);
  const auto& st = h->sim->state();
  for (std::size_t i = 0; i < st.x.size(); ++i)
    for (int c = 0; c < 3; ++c) {
      if (x) x[3 * i + static_cast<std::size_t>(c)] = st.x[i][c];
      if (v) v[3 * i + static_cast<std::size_t>(c)] = st.v[i][c];
    }
}

// save_obj (mesh.cpp:320-332) of the cloth at its current state into buf; returns the length
int64_t ref_scene_save_obj(void* hp, char* buf, int64_t cap) {
  auto* h = static_cast<SceneHandle*>(hp);
  std::ostringstream os;
  save_obj(os, h->sim ? h->sim->state().x : h->scene.cloth.rest_positions, h->scene.cloth.triangles);
  const std::string str = os.str();
  if (buf) std::memcpy(buf, str.data(), std::min<int64_t>(cap, static_cast<int64_t>(str.size())));
  return static_cast<int64_t>(str.size());
}

void ref_scene_free(void* hp) { delete static_cast<SceneHandle*>(hp); }

// Instrument the Simulator created by the next ref_scene_step; take_log
// returns the lines written so far (size query with buf = NULL) and clears.
void ref_scene_instrument(void* hp) { static_cast<SceneHandle*>(hp)->instrument = true; }
int64_t ref_scene_take_log(void* hp, char* buf, int64_t cap) {
  auto* h = static_cast<SceneHandle*>(hp);
  const std::string s = h->log.str();
  if (!buf || cap < static_cast<int64_t>(s.size()) + 1) return static_cast<int64_t>(s.size());
  std::memcpy(buf, s.data(), s.size());
  buf[s.size()] = '\0';
  h->log.str("");
  return static_cast<int64_t>(s.size());
}

}  // extern "C"
