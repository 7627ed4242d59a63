// mesh.cpp — one-time host precompute of the static element data the
// device assembly consumes: rest data, hinges and lumped masses of a cloth
// mesh, and the build_elements list. Host setup, not the per-step hot path
// ("mesh — one-time host precompute; its outputs are static
// device inputs"). Restates proj/src/mesh.cpp:14-212 and
// proj/src/physics.cpp:5-63 in the reference's floating-point association
// (compiled with -ffp-contract=off); the hinge edge order of the reference's
// std::map is reproduced with a stable sort by (a, b).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/weft_gpu.h"
#include "../../include/weft_mesh.h"

namespace {

thread_local std::string g_err;

struct SceneError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct V {
  double x, y, z;
};
V sub(V a, V b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V add(V a, V b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
V scl(double s, V a) { return {s * a.x, s * a.y, s * a.z}; }
V divs(V a, double s) { return {a.x / s, a.y / s, a.z / s}; }
double dot(V a, V b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
V cross(V a, V b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
double norm(V a) { return std::sqrt(dot(a, a)); }

constexpr double kAreaEpsilon = 1e-12;  // mesh.cpp:14

struct TriRest {
  double pwu[3] = {0, 0, 0}, pwv[3] = {0, 0, 0}, area = 0.0;
  bool degenerate = false;
};

struct Hinge {
  int verts[4];
  double rest_angle, stiffness_scale;
};

}  // namespace

struct weft_mesh {
  std::vector<V> rest;
  std::vector<std::array<int, 3>> tris;
  std::vector<std::array<int, 2>> edges;
  std::vector<TriRest> tri_rest;
  std::vector<Hinge> hinges;
  std::vector<double> vertex_area, vertex_mass;
};

namespace {

double triangle_area(V a, V b, V c) { return 0.5 * norm(cross(sub(b, a), sub(c, a))); }  // mesh.cpp:16-18

// dihedral_angle (elements.cpp:94-104)
double dihedral_angle(V x0, V x1, V x2, V x3) {
  const V e = sub(x1, x0);
  const V na = cross(e, sub(x2, x0));
  const V nb = cross(sub(x3, x0), e);
  const double elen = norm(e);
  if (dot(na, na) < 1e-24 || dot(nb, nb) < 1e-24 || elen < 1e-12) return 0.0;
  const double s = dot(cross(na, nb), e) / elen;
  const double c = dot(na, nb);
  return std::atan2(s, c);
}

// Mixed Voronoi areas (mesh.cpp:22-60)
std::vector<double> voronoi_areas(const std::vector<V>& x, const std::vector<std::array<int, 3>>& tris) {
  std::vector<double> area(x.size(), 0.0);
  for (const auto& t : tris) {
    const V a = x[static_cast<size_t>(t[0])], b = x[static_cast<size_t>(t[1])], c = x[static_cast<size_t>(t[2])];
    const double full = triangle_area(a, b, c);
    if (full < kAreaEpsilon) continue;
    auto corner_cos = [](V tip, V p, V q) {
      const V u = sub(p, tip), v = sub(q, tip);
      return dot(u, v) / (norm(u) * norm(v));
    };
    const double ca = corner_cos(a, b, c), cb = corner_cos(b, c, a), cc = corner_cos(c, a, b);
    if (ca < 0.0 || cb < 0.0 || cc < 0.0) {
      for (int k = 0; k < 3; ++k) {
        const double cos_k = k == 0 ? ca : (k == 1 ? cb : cc);
        area[static_cast<size_t>(t[static_cast<size_t>(k)])] += cos_k < 0.0 ? full / 2.0 : full / 4.0;
      }
      continue;
    }
    auto cot = [](double cv) { return cv / std::sqrt(std::max(1e-16, 1.0 - cv * cv)); };
    const V bc = sub(b, c), ca_ = sub(c, a), ab = sub(a, b);
    const double la2 = dot(bc, bc), lb2 = dot(ca_, ca_), lc2 = dot(ab, ab);
    area[static_cast<size_t>(t[0])] += (lb2 * cot(cb) + lc2 * cot(cc)) / 8.0;
    area[static_cast<size_t>(t[1])] += (lc2 * cot(cc) + la2 * cot(ca)) / 8.0;
    area[static_cast<size_t>(t[2])] += (la2 * cot(ca) + lb2 * cot(cb)) / 8.0;
  }
  return area;
}

// triangle_rest (mesh.cpp:62-84)
TriRest triangle_rest(V r0, V r1, V r2) {
  TriRest rest;
  rest.area = triangle_area(r0, r1, r2);
  if (rest.area < kAreaEpsilon) {
    rest.degenerate = true;
    return rest;
  }
  const V e1 = sub(r1, r0), e2 = sub(r2, r0);
  const double u1 = norm(e1);
  const V u_hat = divs(e1, u1);
  const double u2 = dot(e2, u_hat);
  const double v2 = norm(sub(e2, scl(u2, u_hat)));
  const double det = u1 * v2;
  const double a = v2 / det, b = -u2 / det;
  const double c = 0.0, d = u1 / det;
  rest.pwu[0] = -a - c;
  rest.pwu[1] = a;
  rest.pwu[2] = c;
  rest.pwv[0] = -b - d;
  rest.pwv[1] = b;
  rest.pwv[2] = d;
  return rest;
}

// compute_rest_data (mesh.cpp:86-137)
void compute_rest_data(weft_mesh& m) {
  m.tri_rest.clear();
  for (const auto& t : m.tris)
    m.tri_rest.push_back(triangle_rest(m.rest[static_cast<size_t>(t[0])], m.rest[static_cast<size_t>(t[1])],
                                       m.rest[static_cast<size_t>(t[2])]));
  struct Rec {
    int a, b, tri, opp;
  };
  std::vector<Rec> recs;
  recs.reserve(3 * m.tris.size());
  for (int ti = 0; ti < static_cast<int>(m.tris.size()); ++ti) {
    const auto& t = m.tris[static_cast<size_t>(ti)];
    for (int k = 0; k < 3; ++k) {
      int a = t[static_cast<size_t>(k)], b = t[static_cast<size_t>((k + 1) % 3)];
      const int opp = t[static_cast<size_t>((k + 2) % 3)];
      if (a > b) std::swap(a, b);
      recs.push_back({a, b, ti, opp});
    }
  }
  // std::map<edge, vector<(tri, opp)>> iteration order == stable sort by key
  std::stable_sort(recs.begin(), recs.end(),
                   [](const Rec& x, const Rec& y) { return x.a != y.a ? x.a < y.a : x.b < y.b; });
  m.edges.clear();
  m.hinges.clear();
  for (size_t i = 0; i < recs.size();) {
    size_t j = i;
    while (j < recs.size() && recs[j].a == recs[i].a && recs[j].b == recs[i].b) ++j;
    m.edges.push_back({recs[i].a, recs[i].b});
    if (j - i == 2) {
      const Rec& r0 = recs[i];
      const Rec& r1 = recs[i + 1];
      if (!m.tri_rest[static_cast<size_t>(r0.tri)].degenerate && !m.tri_rest[static_cast<size_t>(r1.tri)].degenerate) {
        Hinge h;
        h.verts[0] = r0.a;
        h.verts[1] = r0.b;
        h.verts[2] = r0.opp;
        h.verts[3] = r1.opp;
        const auto P = [&](int v) { return m.rest[static_cast<size_t>(v)]; };
        h.rest_angle = dihedral_angle(P(r0.a), P(r0.b), P(r0.opp), P(r1.opp));
        const V ev = sub(P(r0.b), P(r0.a));
        const double e2 = dot(ev, ev);
        const double areas = m.tri_rest[static_cast<size_t>(r0.tri)].area + m.tri_rest[static_cast<size_t>(r1.tri)].area;
        h.stiffness_scale = 3.0 * e2 / std::max(areas, kAreaEpsilon);
        m.hinges.push_back(h);
      }
    }
    i = j;
  }
  m.vertex_area = voronoi_areas(m.rest, m.tris);
}

// ClothMesh::build (mesh.cpp:141-172)
weft_mesh* build_mesh(std::vector<V> verts, std::vector<std::array<int, 3>> tris, double density) {
  if (density <= 0.0) throw SceneError("cloth density must be positive");
  auto m = std::make_unique<weft_mesh>();
  m->rest = std::move(verts);
  m->tris = std::move(tris);
  const int p = static_cast<int>(m->rest.size());
  for (const auto& t : m->tris) {
    for (int v : t)
      if (v < 0 || v >= p) throw SceneError("triangle vertex index out of range");
    if (t[0] == t[1] || t[1] == t[2] || t[0] == t[2]) throw SceneError("triangle with repeated vertex");
  }
  {  // manifold check: an edge may border at most two triangles
    std::vector<std::array<int, 2>> es;
    es.reserve(3 * m->tris.size());
    for (const auto& t : m->tris)
      for (int k = 0; k < 3; ++k) {
        int a = t[static_cast<size_t>(k)], b = t[static_cast<size_t>((k + 1) % 3)];
        if (a > b) std::swap(a, b);
        es.push_back({a, b});
      }
    std::sort(es.begin(), es.end());
    for (size_t i = 2; i < es.size(); ++i)
      if (es[i] == es[i - 2]) throw SceneError("non-manifold edge in cloth mesh");
  }
  compute_rest_data(*m);
  m->vertex_mass.resize(static_cast<size_t>(p));
  for (int v = 0; v < p; ++v) {
    m->vertex_mass[static_cast<size_t>(v)] = density * m->vertex_area[static_cast<size_t>(v)];
    if (m->vertex_mass[static_cast<size_t>(v)] <= 0.0)
      throw SceneError("vertex " + std::to_string(v) + " has zero mass (isolated or degenerate)");
  }
  return m.release();
}

template <class F>
weft_status guard(F&& f) {
  try {
    f();
    return WEFT_OK;
  } catch (const SceneError& e) {
    g_err = e.what();
    return WEFT_ERR_DIMENSION;
  } catch (const std::exception& e) {
    g_err = e.what();
    return WEFT_ERR_INVALID;
  }
}

}  // namespace

extern "C" {

const char* weft_mesh_last_error(void) { return g_err.c_str(); }

weft_status weft_mesh_build(int32_t nverts, const double* verts, int32_t ntris, const int32_t* tris, double density,
                            weft_mesh** out) {
  return guard([&] {
    std::vector<V> v(static_cast<size_t>(nverts));
    for (int i = 0; i < nverts; ++i) v[static_cast<size_t>(i)] = {verts[3 * i], verts[3 * i + 1], verts[3 * i + 2]};
    std::vector<std::array<int, 3>> t(static_cast<size_t>(ntris));
    for (int i = 0; i < ntris; ++i) t[static_cast<size_t>(i)] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
    *out = build_mesh(std::move(v), std::move(t), density);
  });
}

// make_grid_mesh (mesh.cpp:187-212)
weft_status weft_mesh_grid(int32_t nx, int32_t ny, double width, double height, const double* origin, double density,
                           weft_mesh** out) {
  return guard([&] {
    if (nx < 2 || ny < 2) throw SceneError("grid mesh needs at least 2x2 vertices");
    std::vector<V> verts;
    verts.reserve(static_cast<size_t>(nx) * static_cast<size_t>(ny));
    const V o{origin[0], origin[1], origin[2]};
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) verts.push_back(add(o, V{width * i / (nx - 1), height * j / (ny - 1), 0.0}));
    std::vector<std::array<int, 3>> tris;
    auto id = [nx](int i, int j) { return j * nx + i; };
    for (int j = 0; j + 1 < ny; ++j)
      for (int i = 0; i + 1 < nx; ++i) {
        if ((i + j) % 2 == 0) {
          tris.push_back({id(i, j), id(i + 1, j), id(i + 1, j + 1)});
          tris.push_back({id(i, j), id(i + 1, j + 1), id(i, j + 1)});
        } else {
          tris.push_back({id(i, j), id(i + 1, j), id(i, j + 1)});
          tris.push_back({id(i + 1, j), id(i + 1, j + 1), id(i, j + 1)});
        }
      }
    *out = build_mesh(std::move(verts), std::move(tris), density);
  });
}

weft_status weft_mesh_info(const weft_mesh* m, int32_t* verts, int32_t* tris, int32_t* hinges, int32_t* edges) {
  return guard([&] {
    *verts = static_cast<int32_t>(m->rest.size());
    *tris = static_cast<int32_t>(m->tris.size());
    *hinges = static_cast<int32_t>(m->hinges.size());
    *edges = static_cast<int32_t>(m->edges.size());
  });
}

weft_status weft_mesh_copy(const weft_mesh* m, double* rest, int32_t* tris, double* tri_rest, uint8_t* tri_degenerate,
                           int32_t* hinge_verts, double* hinge_data, double* vertex_area, double* vertex_mass) {
  return guard([&] {
    for (size_t v = 0; v < m->rest.size(); ++v) {
      if (rest) {
        rest[3 * v] = m->rest[v].x;
        rest[3 * v + 1] = m->rest[v].y;
        rest[3 * v + 2] = m->rest[v].z;
      }
      if (vertex_area) vertex_area[v] = m->vertex_area[v];
      if (vertex_mass) vertex_mass[v] = m->vertex_mass[v];
    }
    for (size_t t = 0; t < m->tris.size(); ++t) {
      for (int c = 0; c < 3; ++c) {
        if (tris) tris[3 * t + static_cast<size_t>(c)] = m->tris[t][static_cast<size_t>(c)];
        if (tri_rest) {
          tri_rest[7 * t + static_cast<size_t>(c)] = m->tri_rest[t].pwu[c];
          tri_rest[7 * t + 3 + static_cast<size_t>(c)] = m->tri_rest[t].pwv[c];
        }
      }
      if (tri_rest) tri_rest[7 * t + 6] = m->tri_rest[t].area;
      if (tri_degenerate) tri_degenerate[t] = m->tri_rest[t].degenerate ? 1 : 0;
    }
    for (size_t k = 0; k < m->hinges.size(); ++k) {
      for (int c = 0; c < 4; ++c)
        if (hinge_verts) hinge_verts[4 * k + static_cast<size_t>(c)] = m->hinges[k].verts[c];
      if (hinge_data) {
        hinge_data[2 * k] = m->hinges[k].rest_angle;
        hinge_data[2 * k + 1] = m->hinges[k].stiffness_scale;
      }
    }
  });
}

// build_elements (physics.cpp:5-63): triangles, hinges, vertices.
weft_status weft_build_elements(const weft_mesh* m, const double* material, const double* gravity, const double* wind,
                                weft_element* out, int64_t cap, int64_t* count) {
  return guard([&] {
    const double stretch_warp = material[0], stretch_weft = material[1], shear = material[2], bend = material[3];
    const double damping = material[5], air_drag = material[6];
    const V g{gravity[0], gravity[1], gravity[2]}, w{wind[0], wind[1], wind[2]};
    int64_t n = 0;
    auto emit = [&](const weft_element& e) {
      if (out && n < cap) out[n] = e;
      ++n;
    };
    for (size_t t = 0; t < m->tris.size(); ++t) {
      const TriRest& r = m->tri_rest[t];
      if (r.degenerate) continue;
      weft_element e{};
      e.kind = WEFT_STRETCH;
      e.stencil_size = 3;
      e.stencil[0] = m->tris[t][0];
      e.stencil[1] = m->tris[t][1];
      e.stencil[2] = m->tris[t][2];
      e.stencil[3] = -1;
      e.damping = damping;
      for (int c = 0; c < 3; ++c) {
        e.data[c] = r.pwu[c];
        e.data[3 + c] = r.pwv[c];
      }
      e.data[6] = r.area;
      e.data[7] = stretch_warp;
      e.data[8] = stretch_weft;
      e.data[9] = shear;
      emit(e);
    }
    for (const Hinge& h : m->hinges) {
      weft_element e{};
      e.kind = WEFT_BEND;
      e.stencil_size = 4;
      for (int c = 0; c < 4; ++c) e.stencil[c] = h.verts[c];
      e.damping = damping;
      e.data[0] = h.rest_angle;
      e.data[1] = bend * h.stiffness_scale;
      emit(e);
    }
    for (size_t v = 0; v < m->rest.size(); ++v) {
      weft_element e{};
      e.kind = WEFT_EXTERNAL;
      e.stencil_size = 1;
      e.stencil[0] = static_cast<int32_t>(v);
      e.stencil[1] = e.stencil[2] = e.stencil[3] = -1;
      const V f = add(scl(m->vertex_mass[v], g), scl(m->vertex_area[v], w));
      e.data[0] = f.x;
      e.data[1] = f.y;
      e.data[2] = f.z;
      e.data[3] = air_drag * m->vertex_area[v];
      emit(e);
    }
    *count = n;
  });
}

void weft_mesh_destroy(weft_mesh* m) { delete m; }

}  // extern "C"
