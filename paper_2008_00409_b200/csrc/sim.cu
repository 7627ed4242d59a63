// sim.cu — C-ABI for assembly and broad phase, and the device-resident
// hot-path step (Simulator::step_impl stages 1-4 plus the CCD broad phase,
// proj/src/driver.cpp:96-215; narrow phase and impact zones are out of
// scope for this tier).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "ctx.cuh"

namespace weft_gpu {
namespace {

// x_adv = x + dt v (physics.hpp:54-55)
__global__ void k_advance(int64_t n, const double* __restrict__ x, const double* __restrict__ v, double dt,
                          double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = x[i] + dt * v[i];
}

// v += dv; x_cand = x + dt v (driver.cpp:165-176) over entries [i0, i1)
// (this rank's rows)
// dv: Real (float under Precision::Single; v_cand += double(dv), driver.cpp:166-170)
template <class T>
__global__ void k_candidate(int64_t i0, int64_t i1, const double* __restrict__ x, double* __restrict__ v,
                            const T* __restrict__ dv, double dt, double* __restrict__ xc) {
  const int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= i1) return;
  const double vi = v[i] + static_cast<double>(dv[i]);
  v[i] = vi;
  xc[i] = x[i] + dt * vi;
}

__global__ void k_movable(int p, const uint8_t* __restrict__ pinned, uint8_t* __restrict__ movable) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < p) movable[i] = pinned[i] ? 0 : 1;
}

void upload_vec(Ctx& c, DBuf<double>& dst, const double* src, size_t n) {
  dst.resize(n);
  if (n) WG_CUDA(cudaMemcpyAsync(dst.data(), src, n * sizeof(double), cudaMemcpyDefault, c.stream));
}

}  // namespace
}  // namespace weft_gpu

using weft_gpu::Ctx;
using weft_gpu::Error;

// Shares the boundary's error convention (capi.cu).
extern "C" weft_status weft_gpu_internal_set_error(const char* msg, weft_status s);

namespace {
template <class F>
weft_status guard2(weft_gpu_ctx* ctx, F&& f) {
  try {
    if (!ctx) throw Error(WEFT_ERR_INVALID, "null context");
    WG_CUDA(cudaSetDevice(ctx->c.device));
    f(ctx->c);
    return WEFT_OK;
  } catch (const Error& e) {
    return weft_gpu_internal_set_error(e.what(), e.status);
  } catch (const std::exception& e) {
    return weft_gpu_internal_set_error(e.what(), WEFT_ERR_INVALID);
  }
}
}  // namespace

extern "C" {

weft_status weft_gpu_set_vertices(weft_gpu_ctx* ctx, int32_t p, const double* mass, const uint8_t* pinned) {
  return guard2(ctx, [&](Ctx& c) { weft_gpu::set_vertices(c, p, mass, pinned); });
}

weft_status weft_gpu_set_elements(weft_gpu_ctx* ctx, int64_t count, const weft_element* elements) {
  return guard2(ctx, [&](Ctx& c) { weft_gpu::set_elements(c, count, elements); });
}

weft_status weft_gpu_set_contacts(weft_gpu_ctx* ctx, int64_t count, const weft_element* contacts) {
  return guard2(ctx, [&](Ctx& c) { weft_gpu::set_contacts(c, count, contacts); });
}

weft_status weft_gpu_fill_matrix(weft_gpu_ctx* ctx, const double* x_cur, const double* x_adv, const double* velocity,
                                 double dt, int32_t jac_mode) {
  return guard2(ctx, [&](Ctx& c) {
    const size_t n = 3 * static_cast<size_t>(c.p);
    weft_gpu::upload_vec(c, c.x_cur, x_cur, n);
    weft_gpu::upload_vec(c, c.x_adv, x_adv, n);
    weft_gpu::upload_vec(c, c.vel, velocity, n);
    weft_gpu::fill_matrix(c, c.x_cur.data(), c.x_adv.data(), c.vel.data(), dt, jac_mode);
  });
}

weft_status weft_gpu_fill_matrix_f32(weft_gpu_ctx* ctx, const double* x_cur, const double* x_adv,
                                     const double* velocity, double dt, int32_t jac_mode) {
  return guard2(ctx, [&](Ctx& c) {
    const size_t n = 3 * static_cast<size_t>(c.p);
    weft_gpu::upload_vec(c, c.x_cur, x_cur, n);
    weft_gpu::upload_vec(c, c.x_adv, x_adv, n);
    weft_gpu::upload_vec(c, c.vel, velocity, n);
    weft_gpu::fill_matrix(c, c.x_cur.data(), c.x_adv.data(), c.vel.data(), dt, jac_mode, true, true);
  });
}

weft_status weft_gpu_step_system_f32(weft_gpu_ctx* ctx, const double* x, const double* v, double dt,
                                     int32_t jac_mode) {
  return guard2(ctx, [&](Ctx& c) {
    const size_t n = 3 * static_cast<size_t>(c.p);
    weft_gpu::upload_vec(c, c.x_cur, x, n);
    weft_gpu::upload_vec(c, c.vel, v, n);
    c.x_adv.resize(n);
    if (n)
      weft_gpu::k_advance<<<weft_gpu::div_up(n, 256), 256, 0, ls(c)>>>(n, c.x_cur.data(), c.vel.data(), dt,
                                                                          c.x_adv.data());
    WG_CUDA(cudaGetLastError());
    weft_gpu::fill_matrix(c, c.x_cur.data(), c.x_adv.data(), c.vel.data(), dt, jac_mode, true, true);
  });
}

weft_status weft_gpu_download_rhs_f32(weft_gpu_ctx* ctx, float* rhs) {
  return guard2(ctx, [&](Ctx& c) {
    if (!c.has_rhs || !c.A.f32) throw Error(WEFT_ERR_INVALID, "download_rhs: no single-precision rhs");
    const size_t o = 3 * static_cast<size_t>(c.row0), m = 3 * static_cast<size_t>(c.row1 - c.row0);
    WG_CUDA(cudaMemcpyAsync(rhs, reinterpret_cast<const float*>(c.rhs.data()) + o, m * sizeof(float),
                            cudaMemcpyDefault, c.stream));
    WG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

weft_status weft_gpu_step_system(weft_gpu_ctx* ctx, const double* x, const double* v, double dt, int32_t jac_mode) {
  return guard2(ctx, [&](Ctx& c) {
    const size_t n = 3 * static_cast<size_t>(c.p);
    weft_gpu::upload_vec(c, c.x_cur, x, n);
    weft_gpu::upload_vec(c, c.vel, v, n);
    c.x_adv.resize(n);
    if (n)
      weft_gpu::k_advance<<<weft_gpu::div_up(n, 256), 256, 0, ls(c)>>>(n, c.x_cur.data(), c.vel.data(), dt,
                                                                          c.x_adv.data());
    WG_CUDA(cudaGetLastError());
    weft_gpu::fill_matrix(c, c.x_cur.data(), c.x_adv.data(), c.vel.data(), dt, jac_mode);
  });
}

weft_status weft_gpu_set_soup(weft_gpu_ctx* ctx, int32_t vertex_count, int32_t tri_count, const int32_t* tris) {
  return guard2(ctx, [&](Ctx& c) { weft_gpu::set_soup(c, vertex_count, tri_count, tris); });
}

weft_status weft_gpu_build_grid(weft_gpu_ctx* ctx, const double* x_begin, const double* x_end, int32_t mode,
                                double thickness, double cell_scale) {
  return guard2(ctx, [&](Ctx& c) {
    const size_t n = 3 * static_cast<size_t>(c.soup_verts);
    if (!x_begin) throw Error(WEFT_ERR_INVALID, "build_grid: x_begin is NULL");
    weft_gpu::upload_vec(c, c.x_cur, x_begin, n);
    const bool ccd = mode == WEFT_CONTINUOUS;
    if (ccd) {
      if (!x_end) throw Error(WEFT_ERR_INVALID, "build_grid: continuous mode needs x_end");
      weft_gpu::upload_vec(c, c.x_adv, x_end, n);
    }
    weft_gpu::build_grid(c, c.x_cur.data(), ccd ? c.x_adv.data() : c.x_cur.data(), mode, thickness, cell_scale);
  });
}

weft_status weft_gpu_set_soup_movable(weft_gpu_ctx* ctx, const uint8_t* movable) {
  return guard2(ctx, [&](Ctx& c) { weft_gpu::set_soup_movable(c, movable); });
}

weft_status weft_gpu_collide(weft_gpu_ctx* ctx, const double* x_begin, const double* x_end, int32_t mode,
                             double thickness, double cell_scale, int64_t* count) {
  return guard2(ctx, [&](Ctx& c) {
    const size_t n = 3 * static_cast<size_t>(c.soup_verts);
    if (!x_begin) throw Error(WEFT_ERR_INVALID, "collide: x_begin is NULL");
    weft_gpu::upload_vec(c, c.x_cur, x_begin, n);
    const bool ccd = mode == WEFT_CONTINUOUS;
    if (ccd) {
      if (!x_end) throw Error(WEFT_ERR_INVALID, "collide: continuous mode needs x_end");
      weft_gpu::upload_vec(c, c.x_adv, x_end, n);
    }
    const double* x1 = ccd ? c.x_adv.data() : c.x_cur.data();
    // replicated grid, this rank's share, merged over the group
    const int64_t nh = weft_gpu::collide(c, c.x_cur.data(), x1, mode, thickness, cell_scale);
    if (count) *count = nh;
  });
}

weft_status weft_gpu_download_contacts(weft_gpu_ctx* ctx, int32_t* kind_ab, double* vals) {
  return guard2(ctx, [&](Ctx& c) { weft_gpu::download_contacts(c, kind_ab, vals); });
}

weft_status weft_gpu_build_zones(weft_gpu_ctx* ctx, int64_t n, const int32_t* kind_ab, int32_t* impact_zone,
                                 int32_t* zone_count, int64_t* vertex_total) {
  return guard2(ctx, [&](Ctx& c) {
    if (n < 0 || (n > 0 && !kind_ab)) throw Error(WEFT_ERR_INVALID, "build_zones: bad impact list");
    if (c.soup_verts == 0 && n > 0) throw Error(WEFT_ERR_INVALID, "build_zones: set the soup first");
    std::vector<unsigned long long> keys(static_cast<size_t>(n));
    const int nedges = static_cast<int>(c.soup_edges.size());
    for (int64_t i = 0; i < n; ++i) {
      const int kind = kind_ab[3 * i], a = kind_ab[3 * i + 1], b = kind_ab[3 * i + 2];
      const bool ok = kind == 0 ? (a >= 0 && a < c.soup_verts && b >= 0 && b < c.soup_tris)
                                : (kind == 1 && a >= 0 && a < nedges && b >= 0 && b < nedges);
      if (!ok) throw Error(WEFT_ERR_DIMENSION, "build_zones: impact " + std::to_string(i) + " out of range");
      keys[static_cast<size_t>(i)] = (static_cast<unsigned long long>(kind) << 62) |
                                     (static_cast<unsigned long long>(a) << 31) | static_cast<unsigned long long>(b);
    }
    weft_gpu::DBuf<unsigned long long>& kd = c.zn_tmp_keys;
    kd.upload(keys.data(), keys.size(), c.stream);
    weft_gpu::DBuf<double> vd;  // weights do not change the zone structure
    vd.resize(8 * static_cast<size_t>(n) + 8);
    vd.zero(c.stream);
    const int32_t nz = weft_gpu::build_zones(c, kd.data(), vd.data(), n);
    if (impact_zone) weft_gpu::download_zones(c, n, impact_zone, nullptr, nullptr);
    WG_CUDA(cudaStreamSynchronize(c.stream));
    if (zone_count) *zone_count = nz;
    if (vertex_total) *vertex_total = c.zn_nzv;
  });
}

weft_status weft_gpu_zone_vertices(weft_gpu_ctx* ctx, int32_t* vert_off, int32_t* verts) {
  return guard2(ctx, [&](Ctx& c) { weft_gpu::download_zones(c, 0, nullptr, vert_off, verts); });
}

weft_status weft_distribute_zones(int32_t zone_count, const int32_t* sizes, int32_t devices, int32_t* device_of) {
  if (zone_count < 0 || devices < 1 || (zone_count > 0 && (!sizes || !device_of))) return WEFT_ERR_INVALID;
  const std::vector<int> sz(sizes, sizes + zone_count);
  const auto asg = weft_gpu::distribute_zones(sz, devices);
  for (int d = 0; d < devices; ++d)
    for (int z : asg[static_cast<size_t>(d)]) device_of[z] = d;
  return WEFT_OK;
}

weft_status weft_gpu_resolve_zones(weft_gpu_ctx* ctx, const double* x_begin, double* x_candidate,
                                   const double* vertex_mass, double thickness, double cell_scale,
                                   const weft_zone_params* params, weft_zone_report* report) {
  return guard2(ctx, [&](Ctx& c) {
    if (!x_begin || !x_candidate || !vertex_mass || !params) throw Error(WEFT_ERR_INVALID, "resolve_zones: NULL argument");
    const size_t n = 3 * static_cast<size_t>(c.soup_verts);
    weft_gpu::upload_vec(c, c.x_cur, x_begin, n);
    weft_gpu::upload_vec(c, c.x_adv, x_candidate, n);
    weft_gpu::upload_vec(c, c.vel, vertex_mass, static_cast<size_t>(c.soup_verts));
    weft_zone_report rep{};
    // like the reference, x_candidate holds the positions reached even when
    // ZoneFailure is raised (resolve_zones mutates it in place)
    auto copy_back = [&]() {
      WG_CUDA(cudaMemcpyAsync(x_candidate, c.x_adv.data(), n * sizeof(double), cudaMemcpyDefault, c.stream));
      WG_CUDA(cudaStreamSynchronize(c.stream));
    };
    try {
      weft_gpu::resolve_zones(c, c.x_cur.data(), c.x_adv.data(), c.vel.data(), thickness, cell_scale, *params, rep,
                              false);
    } catch (const Error& e) {
      if (report) *report = rep;
      if (e.status == WEFT_ERR_ZONE) copy_back();
      throw;
    }
    copy_back();
    if (report) *report = rep;
  });
}

weft_status weft_gpu_grid_info(weft_gpu_ctx* ctx, weft_grid_info* info) {
  return guard2(ctx, [&](Ctx& c) {
    if (!c.has_grid) throw Error(WEFT_ERR_INVALID, "grid_info: build_grid first");
    info->cell_size = c.grid_cell_size;
    info->cells = c.grid_cells;
    info->entries = c.grid_entries;
    info->total = c.grid_total;
  });
}

weft_status weft_gpu_download_grid(weft_gpu_ctx* ctx, uint64_t* cell_keys, int64_t* cell_offsets, int32_t* cell_tris,
                                   int64_t* prefix, int64_t* tri_boxes) {
  return guard2(ctx, [&](Ctx& c) {
    if (!c.has_grid) throw Error(WEFT_ERR_INVALID, "download_grid: build_grid first");
    cudaStream_t s = c.stream;
    if (cell_keys && c.grid_cells)
      WG_CUDA(cudaMemcpyAsync(cell_keys, c.cell_keys.data(), 8 * c.grid_cells, cudaMemcpyDefault, s));
    if (cell_offsets)
      WG_CUDA(cudaMemcpyAsync(cell_offsets, c.cell_off.data(), 8 * (c.grid_cells + 1), cudaMemcpyDefault, s));
    if (cell_tris && c.grid_entries)
      WG_CUDA(cudaMemcpyAsync(cell_tris, c.vals_b.data(), 4 * c.grid_entries, cudaMemcpyDefault, s));
    if (prefix) WG_CUDA(cudaMemcpyAsync(prefix, c.wprefix.data(), 8 * (c.grid_cells + 1), cudaMemcpyDefault, s));
    std::vector<int32_t> lat;
    if (tri_boxes && c.soup_tris) {
      lat.resize(6 * static_cast<size_t>(c.soup_tris));
      WG_CUDA(cudaMemcpyAsync(lat.data(), c.lat.data(), 4 * lat.size(), cudaMemcpyDeviceToHost, s));
    }
    WG_CUDA(cudaStreamSynchronize(s));
    if (tri_boxes)
      for (size_t i = 0; i < lat.size(); ++i) tri_boxes[i] = lat[i];
  });
}

weft_status weft_gpu_candidates(weft_gpu_ctx* ctx, int64_t begin, int64_t end, int64_t* count, int32_t* pairs) {
  return guard2(ctx, [&](Ctx& c) { *count = weft_gpu::candidates(c, begin, end, pairs); });
}

weft_status weft_gpu_sim_set_state(weft_gpu_ctx* ctx, const double* x, const double* v) {
  return guard2(ctx, [&](Ctx& c) {
    if (c.p == 0 || c.n_static == 0) throw Error(WEFT_ERR_INVALID, "sim_set_state: set vertices and elements first");
    // the soup is the cloth (vertices [0, p)) followed by the obstacles'
    // vertices (driver.cpp:73-85), whose positions come per step from
    // weft_gpu_sim_set_obstacles
    if (c.soup_verts < c.p) throw Error(WEFT_ERR_INVALID, "sim_set_state: the soup must start with the cloth");
    if (c.soup_verts > c.p && c.world > 1) throw Error(WEFT_ERR_INVALID, "sim_set_state: obstacles run on one rank");
    const size_t n = 3 * static_cast<size_t>(c.p), ns = 3 * static_cast<size_t>(c.soup_verts);
    if (c.world > 1) {
      weft_gpu::comm_need(c, "sim_set_state");
      weft_gpu::rank_barrier(c);  // no peer may still be reading the state being replaced
    }
    c.sim_x.resize(ns);
    c.sim_v.resize(ns);
    WG_CUDA(cudaMemcpyAsync(c.sim_x.data(), x, n * sizeof(double), cudaMemcpyDefault, c.stream));
    WG_CUDA(cudaMemcpyAsync(c.sim_v.data(), v, n * sizeof(double), cudaMemcpyDefault, c.stream));
    c.sim_xc.resize(ns);
    c.sim_xc.n = ns;
    // movable = !pinned for the cloth, 0 for obstacle vertices
    c.soup_movable.resize(static_cast<size_t>(c.soup_verts));
    if (c.soup_verts > c.p) WG_CUDA(cudaMemsetAsync(c.soup_movable.data() + c.p, 0, c.soup_verts - c.p, c.stream));
    weft_gpu::k_movable<<<weft_gpu::div_up(c.p, 256), 256, 0, ls(c)>>>(c.p, c.pinned.data(), c.soup_movable.data());
    // soup masses (driver.cpp:143-144): the cloth's, 1.0 for obstacle vertices
    c.soup_mass.resize(static_cast<size_t>(c.soup_verts));
    WG_CUDA(cudaMemcpyAsync(c.soup_mass.data(), c.mass.data(), c.p * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
    if (c.soup_verts > c.p) {
      const std::vector<double> ones(static_cast<size_t>(c.soup_verts - c.p), 1.0);
      WG_CUDA(cudaMemcpyAsync(c.soup_mass.data() + c.p, ones.data(), ones.size() * sizeof(double),
                              cudaMemcpyHostToDevice, c.stream));
    }
    WG_CUDA(cudaStreamSynchronize(c.stream));
    c.has_state = true;
    c.obstacles_set = c.soup_verts == c.p;
  });
}

weft_status weft_gpu_sim_set_obstacles(weft_gpu_ctx* ctx, double dt, const double* x_begin, const double* x_end) {
  return guard2(ctx, [&](Ctx& c) {
    if (!c.has_state) throw Error(WEFT_ERR_INVALID, "sim_set_obstacles: sim_set_state first");
    const int no = c.soup_verts - c.p;
    if (no == 0) return;
    if (!x_begin || !x_end || !(dt > 0.0)) throw Error(WEFT_ERR_INVALID, "sim_set_obstacles: bad arguments");
    const size_t n = 3 * static_cast<size_t>(no), o = 3 * static_cast<size_t>(c.p);
    std::vector<double> b(n), e(n), vel(n);
    WG_CUDA(cudaMemcpy(b.data(), x_begin, n * sizeof(double), cudaMemcpyDefault));
    WG_CUDA(cudaMemcpy(e.data(), x_end, n * sizeof(double), cudaMemcpyDefault));
    for (size_t i = 0; i < n; ++i) vel[i] = (e[i] - b[i]) / dt;  // driver.cpp:126-128
    WG_CUDA(cudaMemcpyAsync(c.sim_x.data() + o, b.data(), n * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    WG_CUDA(cudaMemcpyAsync(c.sim_xc.data() + o, e.data(), n * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    WG_CUDA(cudaMemcpyAsync(c.sim_v.data() + o, vel.data(), n * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    WG_CUDA(cudaStreamSynchronize(c.stream));
    c.obstacles_set = true;
  });
}

weft_status weft_gpu_sim_step(weft_gpu_ctx* ctx, const weft_sim_params* prm, weft_step_report* rep) {
  return guard2(ctx, [&](Ctx& c) {
    if (!c.has_state) throw Error(WEFT_ERR_INVALID, "sim_step: sim_set_state first");
    if (!c.obstacles_set) throw Error(WEFT_ERR_INVALID, "sim_step: obstacle positions missing (sim_set_obstacles)");
    cudaStream_t s = c.stream;
    const int64_t n = 3 * static_cast<int64_t>(c.p);
    const double dt = prm->dt;
    const bool f32 = prm->precision == 1;
    if (f32 && c.world > 1) throw Error(WEFT_ERR_INVALID, "sim_step: Precision::Single runs on one rank");
    cudaEvent_t* ev = c.ev;
    // the grid is replicated on every rank (collision.cpp:397-399); each
    // rank walks its split_workload share of the pair space (:181-192)
    auto share = [&](int64_t total, int64_t& b, int64_t& e) {
      const int64_t base = total / c.world, extra = total % c.world;
      b = c.rank * base + std::min<int64_t>(c.rank, extra);
      e = b + base + (c.rank < extra ? 1 : 0);
    };
    int64_t wb = 0, we = 0;
    int64_t dcd = 0, nprox = 0, ncont = 0, nimp = 0;
    const bool contacts = prm->contacts != 0;
    if (contacts) {
      // Simulator::step_impl stages 1-2 in full (driver.cpp:132-149): DCD
      // collide, proximities_to_elements, step_system with the contacts. A
      // rank group narrow-phases its shares and merges the hits, so every
      // rank holds all contact elements; each assembles its own rows, whose
      // contact columns may belong to any rank (the PCG pulls them over
      // peer memory: the dynamic contact halo).
      WG_CUDA(cudaEventRecord(c.ev_side[0], s));
      nprox = weft_gpu::collide(c, c.sim_x.data(), c.sim_x.data(), WEFT_DISCRETE, prm->thickness, prm->cell_scale);
      dcd = c.narrow_pairs;
      WG_CUDA(cudaEventRecord(c.ev_side[1], s));
      WG_CUDA(cudaEventRecord(ev[0], s));
      const weft_gpu::ContactParamsDev kp{prm->thickness, prm->stiffness_scale, prm->friction, prm->contact_damping};
      ncont = weft_gpu::contacts_from_proximities(c, c.sim_x.data(), c.sim_v.data(), dt, kp);
      c.x_adv.resize(static_cast<size_t>(n));
      weft_gpu::k_advance<<<weft_gpu::div_up(n, 256), 256, 0, ls(c)>>>(n, c.sim_x.data(), c.sim_v.data(), dt,
                                                                    c.x_adv.data());
      weft_gpu::fill_matrix(c, c.sim_x.data(), c.x_adv.data(), c.sim_v.data(), dt, prm->jac_mode, true, f32);
      WG_CUDA(cudaEventRecord(ev[2], s));
      WG_CUDA(cudaEventRecord(ev[1], s));
    } else if (c.io_vin) {
    // weft_gpu_sim_step_io, one rank: x arrived on the main stream, v is still
    // in flight on the side stream — the DCD broad phase (x only) runs first
    // and hides the v upload; then the assembly at (x, v)
    if (c.n_contacts) weft_gpu::finish_contacts(c, 0);
    WG_CUDA(cudaEventRecord(c.ev_side[0], s));
    weft_gpu::build_grid(c, c.sim_x.data(), c.sim_x.data(), WEFT_DISCRETE, prm->thickness, prm->cell_scale);
    share(c.grid_total, wb, we);
    dcd = weft_gpu::candidates(c, wb, we, nullptr, /*count_only=*/true);
    WG_CUDA(cudaEventRecord(c.ev_side[1], s));
    WG_CUDA(cudaStreamWaitEvent(s, c.ev_side[2], 0));  // v uploaded
    WG_CUDA(cudaEventRecord(ev[0], s));
    c.x_adv.resize(static_cast<size_t>(n));
    weft_gpu::k_advance<<<weft_gpu::div_up(n, 256), 256, 0, ls(c)>>>(n, c.sim_x.data(), c.sim_v.data(), dt,
                                                                  c.x_adv.data());
    weft_gpu::fill_matrix(c, c.sim_x.data(), c.x_adv.data(), c.sim_v.data(), dt, prm->jac_mode, true, f32);
    WG_CUDA(cudaEventRecord(ev[2], s));
    WG_CUDA(cudaEventRecord(ev[1], s));
    } else {
    if (c.n_contacts) weft_gpu::finish_contacts(c, 0);  // no stale contacts from a contacts-mode step
    // 1 + 2. The proximity broad phase (DCD) on x and the assembly of
    // step_system at (x, v) are independent (contacts come from the narrow
    // phase, out of this tier): the assembly is enqueued on the main stream,
    // the broad phase runs on the side stream at the same time (both are
    // latency-bound kernels that leave most of the GPU idle alone).
    WG_CUDA(cudaEventRecord(ev[0], s));  // state ready
    c.x_adv.resize(static_cast<size_t>(n));
    weft_gpu::k_advance<<<weft_gpu::div_up(n, 256), 256, 0, ls(c)>>>(n, c.sim_x.data(), c.sim_v.data(), dt,
                                                                  c.x_adv.data());
    weft_gpu::fill_matrix(c, c.sim_x.data(), c.x_adv.data(), c.sim_v.data(), dt, prm->jac_mode, /*finish=*/false,
                          f32);
    WG_CUDA(cudaEventRecord(ev[2], s));
    // A/B knob (WEFT_SIM_OVERLAP=1): measured no gain on B200 — the
    // assembly's grids fill every SM, so the side-stream broad phase only
    // runs in their gaps — hence serial by default.
    static const bool serial = std::getenv("WEFT_SIM_OVERLAP") == nullptr;
    if (serial) weft_gpu::fill_matrix_finish(c);
    WG_CUDA(cudaStreamWaitEvent(c.side, serial ? ev[2] : ev[0], 0));
    WG_CUDA(cudaEventRecord(c.ev_side[0], c.side));
    c.cur = c.side;
    try {
      weft_gpu::build_grid(c, c.sim_x.data(), c.sim_x.data(), WEFT_DISCRETE, prm->thickness, prm->cell_scale);
      share(c.grid_total, wb, we);
      dcd = weft_gpu::candidates(c, wb, we, nullptr, /*count_only=*/true);
    } catch (...) {
      c.cur = c.stream;
      throw;
    }
    c.cur = c.stream;
    WG_CUDA(cudaEventRecord(c.ev_side[1], c.side));
    weft_gpu::fill_matrix_finish(c);
    WG_CUDA(cudaStreamWaitEvent(s, c.ev_side[1], 0));  // the cooperative PCG gets the whole GPU
    WG_CUDA(cudaEventRecord(ev[1], s));
    }
    // 3. PCG for dv
    const weft_gpu::PcgResult pr =
        f32 ? weft_gpu::pcg_solve_f32(c, reinterpret_cast<const float*>(c.rhs.data()), prm->pcg, nullptr, nullptr)
            : weft_gpu::pcg_solve(c, c.rhs.data(), prm->pcg, nullptr, nullptr);
    WG_CUDA(cudaEventRecord(ev[3], s));
    if (!pr.converged)  // driver.cpp:158-161
      throw Error(WEFT_ERR_SOLVER, "PCG did not converge (residual " + std::to_string(pr.rel_residual) + ")");
    // 4. candidate update. The reference works on a local v_cand and writes
    // the state only at the commit (driver.cpp:163-206), so a frame that
    // throws after this point (ZoneFailure, a peer timeout) leaves (x, v)
    // untouched: v is saved here and restored unless the commit is reached.
    c.sim_vbak.resize(static_cast<size_t>(n));
    WG_CUDA(cudaMemcpyAsync(c.sim_vbak.data(), c.sim_v.data(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    struct VRestore {
      Ctx& c;
      int64_t n;
      bool armed = true;
      ~VRestore() {
        if (!armed) return;
        cudaStreamSynchronize(c.side);
        cudaMemcpyAsync(c.sim_v.data(), c.sim_vbak.data(), n * sizeof(double), cudaMemcpyDeviceToDevice, c.stream);
        cudaStreamSynchronize(c.stream);
      }
    } v_restore{c, n};
    const int64_t i0 = 3 * static_cast<int64_t>(c.row0), i1 = 3 * static_cast<int64_t>(c.row1);
    if (f32) {
      float* dv = reinterpret_cast<float*>(c.xs.data());
      if (pr.iterations == 0) WG_CUDA(cudaMemsetAsync(dv + i0, 0, (i1 - i0) * sizeof(float), s));
      weft_gpu::k_candidate<float><<<weft_gpu::div_up(i1 - i0, 256), 256, 0, ls(c)>>>(
          i0, i1, c.sim_x.data(), c.sim_v.data(), dv, dt, c.sim_xc.data());
    } else {
      if (pr.iterations == 0) WG_CUDA(cudaMemsetAsync(c.xs.data() + i0, 0, (i1 - i0) * sizeof(double), s));
      weft_gpu::k_candidate<double><<<weft_gpu::div_up(i1 - i0, 256), 256, 0, ls(c)>>>(
          i0, i1, c.sim_x.data(), c.sim_v.data(), c.xs.data(), dt, c.sim_xc.data());
    }
    if (c.world > 1) weft_gpu::exchange_state(c);  // all rows of v and x_cand on every rank
    WG_CUDA(cudaEventRecord(ev[4], s));
    const bool io_out_early = c.io_xout && !contacts;  // v and x_cand are final here
    if (io_out_early) {  // read them back on the side stream while the CCD broad phase runs
      WG_CUDA(cudaStreamWaitEvent(c.side, ev[4], 0));
      WG_CUDA(cudaMemcpyAsync(c.io_vout, c.sim_v.data(), n * sizeof(double), cudaMemcpyDefault, c.side));
      WG_CUDA(cudaMemcpyAsync(c.io_xout, c.sim_xc.data(), n * sizeof(double), cudaMemcpyDefault, c.side));
      WG_CUDA(cudaEventRecord(c.ev_side[3], c.side));
    }
    // 5. impact broad phase (CCD) over begin -> candidate
    int64_t ccd = 0;
    weft_zone_report zr{};
    float tz = 0;
    if (contacts) {
      nimp = weft_gpu::collide(c, c.sim_x.data(), c.sim_xc.data(), WEFT_CONTINUOUS, prm->thickness, prm->cell_scale);
      ccd = c.narrow_pairs;
      if (prm->zones) {
        // 5-6. resolve_zones (driver.cpp:181-191): its first CCD round is
        // the collide above; 7. the commit's velocity correction (:195-204)
        WG_CUDA(cudaEventRecord(c.ev_side[2], s));
        c.zn_pre.resize(static_cast<size_t>(n));
        WG_CUDA(cudaMemcpyAsync(c.zn_pre.data(), c.sim_xc.data(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        weft_gpu::resolve_zones(c, c.sim_x.data(), c.sim_xc.data(), c.soup_mass.data(), prm->thickness,
                                prm->cell_scale, prm->zone, zr, /*have_first=*/true);
        weft_gpu::zone_commit(c, c.sim_xc.data(), c.zn_pre.data(), dt, c.sim_v.data());
        WG_CUDA(cudaEventRecord(c.ev_side[3], s));
        WG_CUDA(cudaEventSynchronize(c.ev_side[3]));
        cudaEventElapsedTime(&tz, c.ev_side[2], c.ev_side[3]);
      }
    } else {
      weft_gpu::build_grid(c, c.sim_x.data(), c.sim_xc.data(), WEFT_CONTINUOUS, prm->thickness, prm->cell_scale);
      share(c.grid_total, wb, we);
      ccd = weft_gpu::candidates(c, wb, we, nullptr, /*count_only=*/true);
    }
    WG_CUDA(cudaEventRecord(ev[5], s));
    // 7. commit
    v_restore.armed = false;
    std::swap(c.sim_x.ptr, c.sim_xc.ptr);
    std::swap(c.sim_x.cap, c.sim_xc.cap);
    c.obstacles_set = c.soup_verts == c.p;  // obstacle positions are per step
    if (c.io_xout) {
      if (io_out_early) {
        WG_CUDA(cudaEventSynchronize(c.ev_side[3]));
      } else {  // contacts / zones change v and x up to the commit
        WG_CUDA(cudaMemcpyAsync(c.io_vout, c.sim_v.data(), n * sizeof(double), cudaMemcpyDefault, s));
        WG_CUDA(cudaMemcpyAsync(c.io_xout, c.sim_x.data(), n * sizeof(double), cudaMemcpyDefault, s));
      }
    }
    WG_CUDA(cudaEventSynchronize(ev[5]));
    if (c.io_xout && !io_out_early) WG_CUDA(cudaStreamSynchronize(s));
    float tdcd = 0, tasm = 0, t13 = 0, t45 = 0;
    cudaEventElapsedTime(&tdcd, c.ev_side[0], c.ev_side[1]);  // overlapped with the assembly
    cudaEventElapsedTime(&tasm, ev[0], ev[2]);
    cudaEventElapsedTime(&t13, ev[1], ev[3]);
    cudaEventElapsedTime(&t45, ev[4], ev[5]);
    if (rep) {
      rep->pcg_iterations = pr.iterations;
      rep->pcg_converged = pr.converged;
      rep->pcg_residual = pr.rel_residual;
      rep->dcd_candidates = dcd;
      rep->ccd_candidates = ccd;
      rep->ms_broad = tdcd + t45;
      rep->ms_assemble = tasm;
      rep->ms_solve = t13;
      rep->proximities = nprox;
      rep->contact_elements = ncont;
      rep->impacts = nimp;
      rep->zone_count = zr.zone_count;
      rep->zone_outer = zr.outer_iterations;
      rep->ms_zones = tz;
      // the full Simulator::step_impl ran its seven stages in canonical order
      rep->stages = contacts && prm->zones ? 7 : 0;
    }
  });
}

weft_status weft_gpu_sim_step_io(weft_gpu_ctx* ctx, const double* x_in, const double* v_in,
                                 const weft_sim_params* prm, double* x_out, double* v_out, weft_step_report* rep) {
  if (!ctx) return WEFT_ERR_INVALID;
  Ctx& c = ctx->c;
  if (c.has_state && c.soup_verts != c.p) {
    // obstacles: the cloth's x and v only — the obstacle positions of this
    // step stay as weft_gpu_sim_set_obstacles gave them
    weft_status st = guard2(ctx, [&](Ctx& cc) {
      if (!x_in || !v_in) throw Error(WEFT_ERR_INVALID, "sim_step_io: NULL state buffer");
      const size_t n = 3 * static_cast<size_t>(cc.p);
      WG_CUDA(cudaMemcpyAsync(cc.sim_x.data(), x_in, n * sizeof(double), cudaMemcpyDefault, cc.stream));
      WG_CUDA(cudaMemcpyAsync(cc.sim_v.data(), v_in, n * sizeof(double), cudaMemcpyDefault, cc.stream));
      WG_CUDA(cudaStreamSynchronize(cc.stream));
    });
    if (st == WEFT_OK) st = weft_gpu_sim_step(ctx, prm, rep);
    if (st == WEFT_OK) st = weft_gpu_sim_get_state(ctx, x_out, v_out);
    return st;
  }
  if (!c.has_state || !prm || prm->contacts || !x_in || !v_in || !x_out || !v_out || c.world > 1) {
    // the plain sequence (contacts mode, rank groups, missing state)
    weft_status st = weft_gpu_sim_set_state(ctx, x_in, v_in);
    if (st == WEFT_OK) st = weft_gpu_sim_step(ctx, prm, rep);
    if (st == WEFT_OK) st = weft_gpu_sim_get_state(ctx, x_out, v_out);
    return st;
  }
  const weft_status st0 = guard2(ctx, [&](Ctx& cc) {
    const size_t n = 3 * static_cast<size_t>(cc.p);
    WG_CUDA(cudaMemcpyAsync(cc.sim_x.data(), x_in, n * sizeof(double), cudaMemcpyDefault, cc.stream));
    WG_CUDA(cudaEventRecord(cc.ev_side[2], cc.stream));
    WG_CUDA(cudaStreamWaitEvent(cc.side, cc.ev_side[2], 0));  // the previous step is done with v
    WG_CUDA(cudaMemcpyAsync(cc.sim_v.data(), v_in, n * sizeof(double), cudaMemcpyDefault, cc.side));
    WG_CUDA(cudaEventRecord(cc.ev_side[2], cc.side));
  });
  if (st0 != WEFT_OK) return st0;
  c.io_vin = v_in;
  c.io_xout = x_out;
  c.io_vout = v_out;
  const weft_status st = weft_gpu_sim_step(ctx, prm, rep);
  c.io_vin = nullptr;
  c.io_xout = c.io_vout = nullptr;
  if (st != WEFT_OK) cudaStreamSynchronize(c.side);
  return st;
}

weft_status weft_gpu_sim_get_state(weft_gpu_ctx* ctx, double* x, double* v) {
  return guard2(ctx, [&](Ctx& c) {
    if (!c.has_state) throw Error(WEFT_ERR_INVALID, "sim_get_state: no state");
    const size_t n = 3 * static_cast<size_t>(c.p);
    if (x) WG_CUDA(cudaMemcpyAsync(x, c.sim_x.data(), n * sizeof(double), cudaMemcpyDefault, c.stream));
    if (v) WG_CUDA(cudaMemcpyAsync(v, c.sim_v.data(), n * sizeof(double), cudaMemcpyDefault, c.stream));
    WG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

}  // extern "C"
