// weft_dropin.hpp — drop-in replacements for the reference's hot-path entry
// points with the reference's own C++ signatures, implemented over the C-ABI
// of libweft_gpu.so (include/weft_gpu.h). A maintainer of the reference
// switches a call site from weft::fill_matrix(...) to weft::gpu::fill_matrix(...)
// (same arguments, same return types, same exception classes); see
// INTEGRATION.md.
//
// Header-only; include after the reference headers (proj/include) and link
// against libweft_gpu.so. Only Real = double is supported on the GPU path
// (the reference default, driver.hpp:35); float throws.
#pragma once

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "weft/assembly.hpp"
#include "weft/collision.hpp"
#include "weft/response.hpp"
#include "weft/solver.hpp"
#include "weft/sparse.hpp"
#include "weft_gpu.h"

namespace weft::gpu {

// Rethrows a C-ABI status as the reference's exception class.
inline void check(weft_status s) {
  if (s == WEFT_OK) return;
  const std::string msg = weft_gpu_last_error();
  switch (s) {
    case WEFT_ERR_DIMENSION: throw DimensionError(msg);
    case WEFT_ERR_SOLVER: throw SolverError(msg);
    case WEFT_ERR_EXEC: throw ExecError(msg);
    case WEFT_ERR_TOPOLOGY: throw TopologyError(msg);
    case WEFT_ERR_SCHEDULE: throw ScheduleError(msg);
    case WEFT_ERR_ZONE: throw ZoneFailure(msg);
    default: throw Error(msg);
  }
}

// One GPU context per (partition count, CUDA device): the partition count is
// the only property of a reference Engine the GPU path depends on (the
// SpMV / dot-product orders are the Engine(n) orders). Each context carries
// its own mutex, held by a Lease for the whole drop-in call, so two threads
// driving different Engines with the same device count serialise on the
// shared device state instead of racing on it. The reference's public API
// is single-threaded per Engine (exec.hpp:83-85); this only makes the shared
// cache safe.
class Context {
 public:
  explicit Context(int partitions, int cuda_device = 0) {
    weft_gpu_options o{cuda_device, partitions, 0, partitions};
    check(weft_gpu_create(&o, &ctx_));
  }
  ~Context() { weft_gpu_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  weft_gpu_ctx* get() const { return ctx_; }
  std::mutex& mutex() { return mu_; }

  // Static inputs last uploaded (fill_matrix / step_system): the device
  // keeps the static element list, its row-incidence tables and pattern
  // resident, so a caller stepping the same mesh only uploads what changed.
  std::vector<double> mass;
  std::vector<uint8_t> pinned;
  std::vector<weft_element> static_elems;
  bool vertices_set = false, elements_set = false;
  // step_system's build_elements cache key (mesh identity + material)
  const void* mesh_key = nullptr;
  std::vector<double> elem_params;

 private:
  weft_gpu_ctx* ctx_ = nullptr;
  std::mutex mu_;
};

struct Lease {
  Context& c;
  std::unique_lock<std::mutex> lock;
  weft_gpu_ctx* get() const { return c.get(); }
};

inline Lease acquire(int partitions, int cuda_device = 0) {
  // Intentionally leaked: contexts must not be torn down during static
  // destruction, after the CUDA runtime itself may already be gone.
  static std::mutex mu;
  static auto* ctxs = new std::map<std::pair<int, int>, std::unique_ptr<Context>>();
  Context* c = nullptr;
  {
    std::lock_guard lock(mu);
    auto& slot = (*ctxs)[{partitions, cuda_device}];
    if (!slot) slot = std::make_unique<Context>(partitions, cuda_device);
    c = slot.get();
  }
  return Lease{*c, std::unique_lock<std::mutex>(c->mutex())};
}

inline Lease acquire(const Engine& engine) { return acquire(engine.devices()); }

inline weft_element to_flat(const AssemblyElement& e) {
  weft_element f;
  std::memset(&f, 0, sizeof(f));  // padding too: the static-list cache compares records bytewise
  f.kind = static_cast<int32_t>(e.kind);
  f.stencil_size = e.stencil_size;
  for (int i = 0; i < 4; ++i) f.stencil[i] = e.stencil[static_cast<std::size_t>(i)];
  f.damping = e.damping;
  double* d = f.data;
  std::visit(
      [&](const auto& v) {
        using T = std::decay_t<decltype(v)>;
        if constexpr (std::is_same_v<T, StretchData>) {
          for (int i = 0; i < 3; ++i) {
            d[i] = v.pwu[static_cast<std::size_t>(i)];
            d[3 + i] = v.pwv[static_cast<std::size_t>(i)];
          }
          d[6] = v.area;
          d[7] = v.k_warp;
          d[8] = v.k_weft;
          d[9] = v.k_shear;
        } else if constexpr (std::is_same_v<T, BendData>) {
          d[0] = v.rest_angle;
          d[1] = v.stiffness;
        } else if constexpr (std::is_same_v<T, SpringData>) {
          d[0] = v.rest_length;
          d[1] = v.stiffness;
        } else if constexpr (std::is_same_v<T, ExternalData>) {
          for (int i = 0; i < 3; ++i) d[i] = v.force[i];
          d[3] = v.drag;
        } else {
          for (int i = 0; i < 3; ++i) d[i] = v.normal[i];
          for (int i = 0; i < 4; ++i) d[3 + i] = v.w[static_cast<std::size_t>(i)];
          d[7] = v.bias;
          d[8] = v.activation;
          d[9] = v.stiffness;
          d[10] = v.friction;
          d[11] = v.tangential_damping;
          d[12] = v.frozen_normal_force;
          for (int i = 0; i < 3; ++i) d[13 + i] = v.rel_vel_bias[i];
        }
      },
      e.data);
  return f;
}

inline std::vector<double> flat3(std::span<const Vec3> v) {
  std::vector<double> out(3 * v.size());
  for (std::size_t i = 0; i < v.size(); ++i)
    for (int c = 0; c < 3; ++c) out[3 * i + static_cast<std::size_t>(c)] = v[i][c];
  return out;
}

// Global block CSR -> the reference's partitioned BELL type
// (partition_matrix(from_entries(...)), sparse.hpp:103-147).
template <class Real>
PartitionedMatrix<Real> to_partitioned(int rows, const std::vector<int64_t>& rp, const std::vector<int32_t>& cols,
                                       const std::vector<Real>& vals, const std::vector<DevicePartition>& parts) {
  std::vector<BlockEntry<Real>> entries;
  entries.reserve(cols.size());
  for (int r = 0; r < rows; ++r)
    for (int64_t k = rp[static_cast<std::size_t>(r)]; k < rp[static_cast<std::size_t>(r) + 1]; ++k) {
      BlockEntry<Real> e;
      e.row = r;
      e.col = cols[static_cast<std::size_t>(k)];
      std::memcpy(e.m.data(), &vals[static_cast<std::size_t>(9 * k)], sizeof(Real) * 9);
      entries.push_back(e);
    }
  return partition_matrix(BellMatrix<Real>::from_entries(rows, entries), parts);
}

// Real-dispatched C-ABI calls (Precision::Single: the _f32 entry points).
inline weft_status set_matrix_r(weft_gpu_ctx* c, int32_t rows, const int64_t* rp, const int32_t* cols,
                                const double* vals) {
  return weft_gpu_set_matrix(c, rows, rp, cols, vals);
}
inline weft_status set_matrix_r(weft_gpu_ctx* c, int32_t rows, const int64_t* rp, const int32_t* cols,
                                const float* vals) {
  return weft_gpu_set_matrix_f32(c, rows, rp, cols, vals);
}
inline weft_status spmv_r(weft_gpu_ctx* c, const double* x, double* y) { return weft_gpu_spmv(c, x, y); }
inline weft_status spmv_r(weft_gpu_ctx* c, const float* x, float* y) { return weft_gpu_spmv_f32(c, x, y); }

template <class Real>
void upload_partitioned(Context& cx, const PartitionedMatrix<Real>& a) {
  weft_gpu_ctx* ctx = cx.get();
  cx.vertices_set = cx.elements_set = false;  // set_matrix replaces the assembled system
  const auto g = gather_matrix(a);
  std::vector<int64_t> rp(static_cast<std::size_t>(g.block_rows()) + 1, 0);
  std::vector<int32_t> cols;
  std::vector<Real> vals;
  for (int r = 0; r < g.block_rows(); ++r) {
    for (int s = 0; s < g.ell_width(); ++s) {
      const int32_t c = g.col_at(r, s);
      if (c == BellMatrix<Real>::kNoBlock) break;
      cols.push_back(c);
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) vals.push_back(g.value_at(r, s, i, j));
    }
    rp[static_cast<std::size_t>(r) + 1] = static_cast<int64_t>(cols.size());
  }
  check(set_matrix_r(ctx, g.block_rows(), rp.data(), cols.data(), vals.data()));
}

// Uploads the vertex data and the static element list only when they differ
// from what the context already holds (the device keeps the static list's
// row-incidence tables and pattern resident); `contacts` go up every call
// as the per-step contact list (assembly order: static list, then contacts).
inline void sync_inputs(Context& cx, int p, std::span<const double> mass, std::span<const uint8_t> pinned,
                        const std::vector<weft_element>& static_elems, const std::vector<weft_element>& contacts) {
  weft_gpu_ctx* ctx = cx.get();
  const bool same_v = cx.vertices_set && static_cast<int>(cx.mass.size()) == p &&
                      mass.size() == static_cast<std::size_t>(p) && pinned.size() == static_cast<std::size_t>(p) &&
                      std::equal(mass.begin(), mass.end(), cx.mass.begin()) &&
                      std::equal(pinned.begin(), pinned.end(), cx.pinned.begin());
  if (!same_v) {
    if (mass.size() != static_cast<std::size_t>(p) || pinned.size() != static_cast<std::size_t>(p))
      throw DimensionError("fill_matrix: mass/pinned size mismatch");
    cx.vertices_set = cx.elements_set = false;
    check(weft_gpu_set_vertices(ctx, p, mass.data(), pinned.data()));
    cx.mass.assign(mass.begin(), mass.end());
    cx.pinned.assign(pinned.begin(), pinned.end());
    cx.vertices_set = true;
  }
  const bool same_e = cx.elements_set && cx.static_elems.size() == static_elems.size() &&
                      (static_elems.empty() ||
                       std::memcmp(cx.static_elems.data(), static_elems.data(),
                                   sizeof(weft_element) * static_elems.size()) == 0);
  if (!same_e) {
    cx.elements_set = false;
    check(weft_gpu_set_elements(ctx, static_cast<int64_t>(static_elems.size()), static_elems.data()));
    cx.static_elems = static_elems;
    cx.elements_set = true;
  }
  check(weft_gpu_set_contacts(ctx, static_cast<int64_t>(contacts.size()), contacts.empty() ? nullptr : contacts.data()));
}

// The context's assembled system downloaded into the reference's types.
template <class Real>
AssembledSystem<Real> download_system(Engine& engine, weft_gpu_ctx* ctx, int p,
                                      const std::vector<DevicePartition>& partitions) {
  weft_matrix_info info{};
  check(weft_gpu_matrix_info(ctx, &info));
  std::vector<int64_t> rp(static_cast<std::size_t>(info.block_rows) + 1);
  std::vector<int32_t> cols(static_cast<std::size_t>(info.nnzb));
  std::vector<Real> vals(9 * static_cast<std::size_t>(info.nnzb)), rhs(3 * static_cast<std::size_t>(p));
  if constexpr (std::is_same_v<Real, float>) {
    check(weft_gpu_download_matrix_f32(ctx, rp.data(), cols.data(), vals.data()));
    check(weft_gpu_download_rhs_f32(ctx, rhs.data()));
  } else {
    check(weft_gpu_download_matrix(ctx, rp.data(), cols.data(), vals.data()));
    check(weft_gpu_download_rhs(ctx, rhs.data()));
  }
  AssembledSystem<Real> out{to_partitioned<Real>(info.block_rows, rp, cols, vals, partitions),
                            DistVector<Real>(&engine, partitions)};
  for (const auto& part : partitions) {
    auto local = out.rhs.local(part.device_id);
    std::copy(rhs.begin() + 3 * part.begin, rhs.begin() + 3 * part.end, local.begin());
  }
  return out;
}

// fill_matrix<Real> (assembly.hpp:74-77): same signature and results. The
// static prefix of in.elements (everything before the first Contact
// element, i.e. build_elements' list, physics.hpp:53-54) is cached on the
// device across calls; the contact elements are uploaded every call.
template <class Real>
AssembledSystem<Real> fill_matrix(Engine& engine, const DistributedElements& /*dist*/, const SystemInputs& in,
                                  const std::vector<DevicePartition>& partitions) {
  {
    if (in.dt <= 0.0) throw DimensionError("fill_matrix: dt must be positive");
    Lease lease = acquire(engine);
    weft_gpu_ctx* ctx = lease.get();
    const int p = partitions.empty() ? 0 : partitions.back().end;
    std::vector<weft_element> stat, cont;
    stat.reserve(in.elements.size());
    bool in_contacts = false;
    for (const auto& e : in.elements) {
      in_contacts = in_contacts || e.kind == ElementKind::Contact;
      (in_contacts ? cont : stat).push_back(to_flat(e));
    }
    sync_inputs(lease.c, p, in.mass, in.pinned, stat, cont);
    const auto xc = flat3(in.x_current), xa = flat3(in.x_advanced), v = flat3(in.velocity);
    const int jm = in.mode == JacobianMode::Exact ? WEFT_JAC_EXACT : WEFT_JAC_SPD_PROJECTED;
    if constexpr (std::is_same_v<Real, float>)  // fill_matrix<float>: one rank
      check(weft_gpu_fill_matrix_f32(ctx, xc.data(), xa.data(), v.data(), in.dt, jm));
    else
      check(weft_gpu_fill_matrix(ctx, xc.data(), xa.data(), v.data(), in.dt, jm));
    return download_system<Real>(engine, ctx, p, partitions);
  }
}

// step_system<Real> (physics.hpp:44-69): build_elements (the reference's own
// host function, physics.cpp:5-63) runs once per (mesh, material, gravity,
// wind) and its list stays on the device; per call only the contact
// elements and the state (x, v) go up, x_adv = x + dt v and the assembly run
// on the GPU (weft_gpu_step_system). The cache is keyed by the mesh's
// address and rest-position storage plus the material/load values: a
// caller that mutates a mesh in place between calls must use a new mesh
// object (the reference's Simulator keeps its mesh const, driver.cpp:148).
template <class Real>
AssembledSystem<Real> step_system(Engine& engine, const ClothMesh& mesh, const SimState& state,
                                  const MaterialParams& params, std::span<const std::uint8_t> pinned,
                                  std::vector<AssemblyElement> contact_elements, double dt, const Vec3& gravity,
                                  const Vec3& wind, JacobianMode mode = JacobianMode::SpdProjected) {
  {
    if (dt <= 0.0) throw DimensionError("fill_matrix: dt must be positive");
    const int p = mesh.vertex_count();
    if (state.x.size() != static_cast<std::size_t>(p) || state.v.size() != static_cast<std::size_t>(p))
      throw DimensionError("step_system: state size != vertex count");
    Lease lease = acquire(engine);
    Context& cx = lease.c;
    weft_gpu_ctx* ctx = lease.get();
    const std::vector<double> key{params.stretch_warp, params.stretch_weft, params.shear, params.bend,
                                  params.density, params.damping, params.air_drag, gravity[0], gravity[1],
                                  gravity[2], wind[0], wind[1], wind[2],
                                  static_cast<double>(reinterpret_cast<std::uintptr_t>(mesh.rest_positions.data())),
                                  static_cast<double>(mesh.triangle_count())};
    std::vector<weft_element> stat;
    const bool cached = cx.elements_set && cx.mesh_key == &mesh && cx.elem_params == key;
    if (cached) {
      stat = cx.static_elems;  // what the device holds
    } else {
      const auto elems = build_elements(mesh, params, gravity, wind);
      stat.reserve(elems.size());
      for (const auto& e : elems) stat.push_back(to_flat(e));
    }
    std::vector<weft_element> cont;
    cont.reserve(contact_elements.size());
    for (const auto& e : contact_elements) cont.push_back(to_flat(e));
    cx.mesh_key = nullptr;
    sync_inputs(cx, p, mesh.vertex_mass, pinned, stat, cont);
    cx.mesh_key = &mesh;
    cx.elem_params = key;
    const auto x = flat3(state.x), v = flat3(state.v);
    const int jm = mode == JacobianMode::Exact ? WEFT_JAC_EXACT : WEFT_JAC_SPD_PROJECTED;
    if constexpr (std::is_same_v<Real, float>)
      check(weft_gpu_step_system_f32(ctx, x.data(), v.data(), dt, jm));
    else
      check(weft_gpu_step_system(ctx, x.data(), v.data(), dt, jm));
    return download_system<Real>(engine, ctx, p, make_partitions(p, engine.devices()));
  }
}

// spmv_serial<Real> (bell.hpp:83-84, bell.cpp:147-153): y = A x on one
// device, slots in ascending order per row (BellMatrix::multiply_into,
// bell.cpp:87-129) — the one-partition GPU SpMV, bitwise.
template <class Real>
std::vector<Real> spmv_serial(const BellMatrix<Real>& a, std::span<const Real> x) {
  {
    if (static_cast<int>(x.size()) != a.rows()) throw DimensionError("spmv_serial: dim(x) != rows");
    Lease lease = acquire(1);
    weft_gpu_ctx* ctx = lease.get();
    std::vector<int64_t> rp(static_cast<std::size_t>(a.block_rows()) + 1, 0);
    std::vector<int32_t> cols;
    std::vector<Real> vals;
    for (int r = 0; r < a.block_rows(); ++r) {
      for (int s = 0; s < a.ell_width(); ++s) {
        const int32_t c = a.col_at(r, s);
        if (c == BellMatrix<Real>::kNoBlock) break;
        cols.push_back(c);
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) vals.push_back(a.value_at(r, s, i, j));
      }
      rp[static_cast<std::size_t>(r) + 1] = static_cast<int64_t>(cols.size());
    }
    std::vector<Real> y(x.size(), Real(0));
    if (a.block_rows() == 0) return y;
    lease.c.vertices_set = lease.c.elements_set = false;  // set_matrix replaces the assembled system
    check(set_matrix_r(ctx, a.block_rows(), rp.data(), cols.data(), vals.data()));
    check(spmv_r(ctx, x.data(), y.data()));
    return y;
  }
}

// spmv_pipelined<Real> (sparse.hpp:72-101).
template <class Real>
void spmv_pipelined(Engine& engine, const PartitionedMatrix<Real>& a, const ValidatedSchedule& sched,
                    const DistVector<Real>& x, DistVector<Real>& y, SpmvWorkspace<Real>& /*ws*/) {
  {
    if (engine.devices() != a.devices || sched.devices() != a.devices)
      throw DimensionError("spmv_pipelined: engine/schedule/matrix device counts differ");
    Lease lease = acquire(engine);
    weft_gpu_ctx* ctx = lease.get();
    upload_partitioned(lease.c, a);
    const auto xg = x.gather();
    std::vector<Real> yg(xg.size());
    check(spmv_r(ctx, xg.data(), yg.data()));
    for (const auto& part : a.partitions) {
      auto local = y.local(part.device_id);
      std::copy(yg.begin() + 3 * part.begin, yg.begin() + 3 * part.end, local.begin());
    }
  }
}

// pcg_solve<Real> (solver.hpp:36-178).
template <class Real>
PcgReport pcg_solve(Engine& engine, const PartitionedMatrix<Real>& a, const ValidatedSchedule& /*sched*/,
                    const DistVector<Real>& b, DistVector<Real>& x, const PcgConfig& config) {
  {
    if (engine.devices() != a.devices) throw DimensionError("pcg_solve: engine/matrix device count mismatch");
    Lease lease = acquire(engine);
    weft_gpu_ctx* ctx = lease.get();
    upload_partitioned(lease.c, a);
    const auto bg = b.gather();
    std::vector<Real> xg(bg.size());
    weft_pcg_config cfg{config.rel_tolerance, config.max_iterations,
                        config.preconditioner == Preconditioner::None ? WEFT_PRECOND_NONE : WEFT_PRECOND_BLOCK_JACOBI};
    std::vector<double> hist(static_cast<std::size_t>(std::max(config.max_iterations, 1)));
    std::vector<double> phist(hist.size());
    weft_pcg_report rep{0, 0, 0.0, hist.data(), phist.data()};
    if constexpr (std::is_same_v<Real, float>)  // pcg_solve<float>
      check(weft_gpu_pcg_f32(ctx, bg.data(), xg.data(), &cfg, &rep));
    else
      check(weft_gpu_pcg(ctx, bg.data(), xg.data(), &cfg, &rep));
    for (const auto& part : a.partitions) {
      auto local = x.local(part.device_id);
      std::copy(xg.begin() + 3 * part.begin, xg.begin() + 3 * part.end, local.begin());
    }
    PcgReport out;
    out.iterations = rep.iterations;
    out.converged = rep.converged != 0;
    out.rel_residual = rep.rel_residual;
    out.residual_history.assign(hist.begin(), hist.begin() + rep.iterations);
    out.precond_norm_history.assign(phist.begin(), phist.begin() + rep.iterations);
    if (engine.options().instrument != nullptr && bg.size()) {  // solver.hpp:171-175 (not for b = 0)
      bool zero = true;
      for (Real v : bg) zero = zero && v == Real(0);
      if (!zero) {
        std::ostringstream os;
        os << "event=pcg iterations=" << out.iterations << " rel_residual=" << out.rel_residual
           << " converged=" << (out.converged ? 1 : 0);
        engine.log_line(os.str());
      }
    }
    return out;
  }
}

// build_grid (collision.cpp:118-179): the device grid downloaded into the
// reference's HashGrid / WorkloadTable types.
inline GridBuildResult build_grid(const CollisionSoup& soup, std::span<const Vec3> x_begin, std::span<const Vec3> x_end,
                                  CollisionMode mode, const CollisionParams& params, int cuda_device = 0) {
  Lease lease = acquire(1, cuda_device);
  weft_gpu_ctx* ctx = lease.get();
  std::vector<int32_t> tris(3 * soup.triangles.size());
  for (std::size_t t = 0; t < soup.triangles.size(); ++t)
    for (int c = 0; c < 3; ++c) tris[3 * t + static_cast<std::size_t>(c)] = soup.triangles[t][static_cast<std::size_t>(c)];
  check(weft_gpu_set_soup(ctx, soup.vertex_count, static_cast<int32_t>(soup.triangles.size()), tris.data()));
  const auto x0 = flat3(x_begin), x1 = flat3(x_end);
  check(weft_gpu_build_grid(ctx, x0.data(), x1.data(),
                            mode == CollisionMode::Continuous ? WEFT_CONTINUOUS : WEFT_DISCRETE, params.thickness,
                            params.cell_scale));
  weft_grid_info info{};
  check(weft_gpu_grid_info(ctx, &info));
  std::vector<uint64_t> keys(static_cast<std::size_t>(info.cells));
  std::vector<int64_t> off(static_cast<std::size_t>(info.cells) + 1), prefix(off.size());
  std::vector<int32_t> cell_tris(static_cast<std::size_t>(info.entries));
  std::vector<int64_t> boxes(6 * soup.triangles.size());
  check(weft_gpu_download_grid(ctx, keys.data(), off.data(), cell_tris.data(), prefix.data(), boxes.data()));
  GridBuildResult out;
  out.grid.cell_size = info.cell_size;
  out.grid.cell_keys = keys;
  for (int64_t c = 0; c < info.cells; ++c) {
    out.grid.cell_tris.emplace_back(cell_tris.begin() + off[static_cast<std::size_t>(c)],
                                    cell_tris.begin() + off[static_cast<std::size_t>(c) + 1]);
    const int64_t s = off[static_cast<std::size_t>(c) + 1] - off[static_cast<std::size_t>(c)];
    out.table.counts.push_back(s * (s - 1) / 2);
  }
  out.table.prefix = prefix;
  out.table.total = prefix.back();
  out.grid.tri_boxes.resize(soup.triangles.size());
  for (std::size_t t = 0; t < soup.triangles.size(); ++t)
    for (int c = 0; c < 6; ++c) out.grid.tri_boxes[t][static_cast<std::size_t>(c)] = boxes[6 * t + static_cast<std::size_t>(c)];
  return out;
}

// collide (collision.cpp:391-417): broad + narrow phase on the GPU, results
// in the reference's NarrowPhaseResult (sorted, deduplicated). The soup's
// movable flags are honoured; `engine` only selects the context.
inline NarrowPhaseResult collide(Engine& engine, const CollisionSoup& soup, std::span<const Vec3> x_begin,
                                 std::span<const Vec3> x_end, CollisionMode mode, const CollisionParams& params,
                                 CollideTimes* /*times*/ = nullptr) {
  Lease lease = acquire(engine);
  weft_gpu_ctx* ctx = lease.get();
  std::vector<int32_t> tris(3 * soup.triangles.size());
  for (std::size_t t = 0; t < soup.triangles.size(); ++t)
    for (int c = 0; c < 3; ++c) tris[3 * t + static_cast<std::size_t>(c)] = soup.triangles[t][static_cast<std::size_t>(c)];
  check(weft_gpu_set_soup(ctx, soup.vertex_count, static_cast<int32_t>(soup.triangles.size()), tris.data()));
  check(weft_gpu_set_soup_movable(ctx, soup.movable.data()));
  const auto x0 = flat3(x_begin), x1 = flat3(x_end);
  const bool ccd = mode == CollisionMode::Continuous;
  int64_t n = 0;
  check(weft_gpu_collide(ctx, x0.data(), x1.data(), ccd ? WEFT_CONTINUOUS : WEFT_DISCRETE, params.thickness,
                         params.cell_scale, &n));
  std::vector<int32_t> kab(3 * static_cast<std::size_t>(n));
  std::vector<double> vals(8 * static_cast<std::size_t>(n));
  check(weft_gpu_download_contacts(ctx, kab.data(), vals.data()));
  NarrowPhaseResult out;
  for (int64_t i = 0; i < n; ++i) {
    const auto kind = kab[3 * i] == 0 ? FeatureKind::VertexFace : FeatureKind::EdgeEdge;
    const double* v = &vals[8 * i];
    const Vec3 nrm(v[1], v[2], v[3]);
    const std::array<double, 4> w{v[4], v[5], v[6], v[7]};
    if (ccd) out.impacts.push_back(Impact{kind, kab[3 * i + 1], kab[3 * i + 2], v[0], nrm, w});
    else out.proximities.push_back(Proximity{kind, kab[3 * i + 1], kab[3 * i + 2], v[0], nrm, w});
  }
  return out;
}

inline void set_soup(weft_gpu_ctx* ctx, const CollisionSoup& soup) {
  std::vector<int32_t> tris(3 * soup.triangles.size());
  for (std::size_t t = 0; t < soup.triangles.size(); ++t)
    for (int c = 0; c < 3; ++c) tris[3 * t + static_cast<std::size_t>(c)] = soup.triangles[t][static_cast<std::size_t>(c)];
  check(weft_gpu_set_soup(ctx, soup.vertex_count, static_cast<int32_t>(soup.triangles.size()), tris.data()));
  check(weft_gpu_set_soup_movable(ctx, soup.movable.data()));
}

// build_zones (response.cpp:108-162) on the GPU: same zones, same ids, same
// impact lists and sorted movable vertex lists. Uses the context of Engine(1).
inline std::vector<ImpactZone> build_zones(const std::vector<Impact>& impacts, const CollisionSoup& soup) {
  Lease lease = acquire(1);
  weft_gpu_ctx* ctx = lease.get();
  set_soup(ctx, soup);
  const int64_t n = static_cast<int64_t>(impacts.size());
  std::vector<int32_t> kab(3 * impacts.size() + 3), iz(impacts.size() + 1);
  for (int64_t i = 0; i < n; ++i) {
    kab[3 * i] = impacts[static_cast<std::size_t>(i)].kind == FeatureKind::VertexFace ? 0 : 1;
    kab[3 * i + 1] = impacts[static_cast<std::size_t>(i)].a;
    kab[3 * i + 2] = impacts[static_cast<std::size_t>(i)].b;
  }
  int32_t nz = 0;
  int64_t nv = 0;
  check(weft_gpu_build_zones(ctx, n, kab.data(), iz.data(), &nz, &nv));
  std::vector<int32_t> off(static_cast<std::size_t>(nz) + 1), verts(static_cast<std::size_t>(nv) + 1);
  check(weft_gpu_zone_vertices(ctx, off.data(), verts.data()));
  std::vector<ImpactZone> zones(static_cast<std::size_t>(nz));
  for (int32_t z = 0; z < nz; ++z) {
    zones[static_cast<std::size_t>(z)].id = z;
    zones[static_cast<std::size_t>(z)].vertices.assign(verts.begin() + off[static_cast<std::size_t>(z)],
                                                        verts.begin() + off[static_cast<std::size_t>(z) + 1]);
  }
  for (int64_t i = 0; i < n; ++i) zones[static_cast<std::size_t>(iz[static_cast<std::size_t>(i)])].impacts.push_back(static_cast<int>(i));
  return zones;
}

// distribute_zones (response.cpp:164-182).
inline std::vector<std::vector<int>> distribute_zones(const std::vector<ImpactZone>& zones, int devices) {
  std::vector<int32_t> sizes(zones.size() + 1), dev(zones.size() + 1);
  for (std::size_t z = 0; z < zones.size(); ++z) sizes[z] = static_cast<int32_t>(zones[z].vertices.size());
  check(weft_distribute_zones(static_cast<int32_t>(zones.size()), sizes.data(), devices, dev.data()));
  // the assignment order of the greedy loop: descending size, stable
  std::vector<int> order(zones.size());
  for (std::size_t z = 0; z < zones.size(); ++z) order[z] = static_cast<int>(z);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sizes[static_cast<std::size_t>(a)] > sizes[static_cast<std::size_t>(b)]; });
  std::vector<std::vector<int>> out(static_cast<std::size_t>(devices));
  for (int z : order) out[static_cast<std::size_t>(dev[static_cast<std::size_t>(z)])].push_back(z);
  return out;
}

// resolve_zones (response.cpp:338-400): CCD rounds and zone solves on the GPU;
// x_candidate is updated in place (also when ZoneFailure is thrown, like the
// reference). Bitwise the reference's positions and report.
inline ZoneResolveReport resolve_zones(Engine& engine, const CollisionSoup& soup, std::span<const Vec3> x_begin,
                                       std::vector<Vec3>& x_candidate, std::span<const double> vertex_mass,
                                       const CollisionParams& cparams, const ZoneSolveParams& zparams,
                                       CollideTimes* /*times*/ = nullptr) {
  Lease lease = acquire(engine);
  weft_gpu_ctx* ctx = lease.get();
  set_soup(ctx, soup);
  const auto xb = flat3(x_begin);
  auto xc = flat3(x_candidate);
  const weft_zone_params zp{zparams.clearance, zparams.initial_penalty, zparams.inner_tolerance,
                            zparams.al_iterations, zparams.inner_iterations, zparams.outer_cap,
                            zparams.retry_cap, zparams.max_correction_factor};
  weft_zone_report rep{};
  const bool instrument = engine.options().instrument != nullptr;
  if (instrument) check(weft_gpu_set_instrument(ctx, 1));
  const weft_status st = weft_gpu_resolve_zones(ctx, xb.data(), xc.data(), vertex_mass.data(), cparams.thickness,
                                                cparams.cell_scale, &zp, &rep);
  if (instrument) {  // the per-round event=zones lines (response.cpp:383-388)
    int64_t n = 0;
    check(weft_gpu_take_log(ctx, nullptr, 0, &n));
    std::string lines(static_cast<std::size_t>(n) + 1, '\0');
    check(weft_gpu_take_log(ctx, lines.data(), n + 1, &n));
    check(weft_gpu_set_instrument(ctx, 0));
    std::istringstream is(lines.substr(0, static_cast<std::size_t>(n)));
    for (std::string ln; std::getline(is, ln);)
      if (!ln.empty()) engine.log_line(ln);
  }
  if (st == WEFT_OK || st == WEFT_ERR_ZONE)
    for (std::size_t v = 0; v < x_candidate.size(); ++v) x_candidate[v] = Vec3(xc[3 * v], xc[3 * v + 1], xc[3 * v + 2]);
  check(st);
  ZoneResolveReport out;
  out.outer_iterations = rep.outer_iterations;
  out.zone_count = rep.zone_count;
  out.max_zone_vertices = rep.max_zone_vertices;
  out.impacts_resolved = static_cast<int>(rep.impacts_resolved);
  out.first_round_impacts = static_cast<int>(rep.first_round_impacts);
  return out;
}

}  // namespace weft::gpu
