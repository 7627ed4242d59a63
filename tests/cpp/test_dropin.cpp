// Runs reference-style checks through the C++ drop-in (weft::gpu::*),
// comparing against the reference's own CPU functions on the reference's
// own fixture generators (src/oracle). Built by `make -C oracle dropin`
// against the unmodified reference objects; executed by
// tests/test_gpu_dropin.py on a GPU box.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include "oracle/collision_oracle.hpp"
#include "oracle/physics_oracle.hpp"
#include "oracle/sparse_oracle.hpp"
#include "weft/physics.hpp"
#include "weft_dropin.hpp"

using namespace weft;

namespace {

Eigen::MatrixXd dense(const PartitionedMatrix<double>& m) { return oracle::bell_to_dense(gather_matrix(m)); }

}  // namespace

TEST_CASE("drop-in fill_matrix equals the reference fill_matrix (bitwise matrix, 1e-12 rhs), n in {1,2,4}") {
  oracle::Rng rng(22);
  for (int trial = 0; trial < 6; ++trial) {
    auto mesh = oracle::random_cloth(rng, 7);
    const int p = mesh.vertex_count();
    SimState state = SimState::rest(mesh);
    for (auto& v : state.v) v = rng.vec3(-0.3, 0.3);
    std::vector<std::uint8_t> pinned(static_cast<std::size_t>(p), 0);
    pinned[0] = 1;
    MaterialParams params;
    params.damping = 0.001;
    const auto elements = build_elements(mesh, params, Vec3(0, 0, -9.81), Vec3::Zero());
    std::vector<Vec3> adv(state.x.size());
    for (std::size_t i = 0; i < adv.size(); ++i) adv[i] = state.x[i] + 0.01 * state.v[i];
    SystemInputs in;
    in.elements = elements;
    in.x_current = state.x;
    in.x_advanced = adv;
    in.velocity = state.v;
    in.mass = mesh.vertex_mass;
    in.pinned = pinned;
    in.dt = 0.01;
    for (int n : {1, 2, 4}) {
      CAPTURE(trial);
      CAPTURE(n);
      Engine engine(n);
      const auto parts = make_partitions(p, n);
      const auto dist = distribute_elements(elements, parts);
      const auto ref = fill_matrix<double>(engine, dist, in, parts);
      const auto gpu = gpu::fill_matrix<double>(engine, dist, in, parts);
      CHECK((dense(ref.matrix) - dense(gpu.matrix)).cwiseAbs().maxCoeff() == 0.0);
      const auto rb = ref.rhs.gather(), gb = gpu.rhs.gather();
      double scale = 1e-300, err = 0.0;
      for (std::size_t i = 0; i < rb.size(); ++i) {
        scale = std::max(scale, std::abs(rb[i]));
        err = std::max(err, std::abs(rb[i] - gb[i]));
      }
      CHECK(err <= 1e-12 * scale);
    }
  }
}

TEST_CASE("drop-in spmv_pipelined is bitwise equal to the order-matched serial oracle") {
  oracle::Rng rng(6);
  for (int n : {1, 2, 4}) {
    Engine engine(n);
    ValidatedSchedule sched = n == 1 ? ValidatedSchedule() : ValidatedSchedule(generate_work_queues(FatTree::make(n)), n);
    for (int trial = 0; trial < 10; ++trial) {
      const int rows = rng.uniform_int(n, 40);
      const auto global = oracle::random_bell(rng, rows, 3);
      const auto parts = make_partitions(rows, n);
      const auto split = partition_matrix(global, parts);
      std::vector<double> xg(static_cast<std::size_t>(3 * rows));
      for (auto& v : xg) v = rng.uniform(-2.0, 2.0);
      DistVector<double> x(&engine, parts), y(&engine, parts);
      for (const auto& part : parts)
        std::copy(xg.begin() + 3 * part.begin, xg.begin() + 3 * part.end, x.local(part.device_id).begin());
      SpmvWorkspace<double> ws(n, split.padded_len);
      gpu::spmv_pipelined(engine, split, sched, x, y, ws);
      CHECK(y.gather() == oracle::spmv_partitioned_serial<double>(split, sched, xg));
    }
  }
}

TEST_CASE("drop-in pcg_solve: hand-solved 2x2, non-SPD error, cloth system vs reference") {
  {
    std::vector<BlockEntry<double>> entries(1);
    entries[0].m = {4, 1, 0, 1, 3, 0, 0, 0, 1};
    const auto a = BellMatrix<double>::from_entries(1, entries);
    Engine engine(1);
    const auto parts = make_partitions(1, 1);
    const auto split = partition_matrix(a, parts);
    DistVector<double> b(&engine, parts), x(&engine, parts);
    b.local(0)[0] = 1;
    b.local(0)[1] = 2;
    PcgConfig cfg;
    cfg.rel_tolerance = 1e-12;
    const auto rep = gpu::pcg_solve(engine, split, ValidatedSchedule(), b, x, cfg);
    CHECK(rep.converged);
    CHECK(x.gather()[0] == doctest::Approx(1.0 / 11.0).epsilon(1e-10));
    CHECK(x.gather()[1] == doctest::Approx(7.0 / 11.0).epsilon(1e-10));
  }
  {
    std::vector<BlockEntry<double>> entries(1);
    entries[0].m = {-1, 0, 0, 0, -1, 0, 0, 0, -1};
    const auto a = BellMatrix<double>::from_entries(1, entries);
    Engine engine(1);
    const auto parts = make_partitions(1, 1);
    DistVector<double> b(&engine, parts), x(&engine, parts);
    b.fill(1.0);
    PcgConfig cfg;
    cfg.preconditioner = Preconditioner::None;
    CHECK_THROWS_AS(gpu::pcg_solve(engine, partition_matrix(a, parts), ValidatedSchedule(), b, x, cfg), SolverError);
  }
  oracle::Rng rng(35);
  auto mesh = oracle::random_cloth(rng, 7);
  const int p = mesh.vertex_count();
  SimState state = SimState::rest(mesh);
  for (auto& v : state.v) v = rng.vec3(-0.3, 0.3);
  std::vector<std::uint8_t> pinned(static_cast<std::size_t>(p), 0);
  pinned[0] = 1;
  for (int n : {1, 2}) {
    Engine engine(n);
    const auto sys = step_system<double>(engine, mesh, state, MaterialParams{}, pinned, {}, 1.0 / 150.0,
                                         Vec3(0, 0, -9.81), Vec3::Zero());
    ValidatedSchedule sched = n == 1 ? ValidatedSchedule() : ValidatedSchedule(generate_work_queues(FatTree::make(n)), n);
    PcgConfig cfg;
    cfg.rel_tolerance = 1e-10;
    DistVector<double> xr(&engine, sys.matrix.partitions), xgpu(&engine, sys.matrix.partitions);
    const auto rr = pcg_solve(engine, sys.matrix, sched, sys.rhs, xr, cfg);
    const auto rg = gpu::pcg_solve(engine, sys.matrix, sched, sys.rhs, xgpu, cfg);
    CHECK(rg.converged);
    CHECK(std::abs(rg.iterations - rr.iterations) <= 2);
    const auto a = xr.gather(), g = xgpu.gather();
    double scale = 1e-300, err = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
      scale = std::max(scale, std::abs(a[i]));
      err = std::max(err, std::abs(a[i] - g[i]));
    }
    CHECK(err <= 1e-8 * scale);
  }
}

TEST_CASE("drop-in build_grid equals the reference build_grid bit for bit") {
  oracle::Rng rng(43);
  for (int trial = 0; trial < 4; ++trial) {
    const auto scene = oracle::random_two_cloth_scene(rng, 8);
    for (CollisionMode mode : {CollisionMode::Discrete, CollisionMode::Continuous}) {
      CollisionParams params;
      params.thickness = 0.01;
      const auto ref = build_grid(scene.soup, scene.x_begin, scene.x_end, mode, params);
      const auto gpu = gpu::build_grid(scene.soup, scene.x_begin, scene.x_end, mode, params);
      CHECK(ref.grid.cell_size == gpu.grid.cell_size);
      CHECK(ref.grid.cell_keys == gpu.grid.cell_keys);
      CHECK(ref.grid.cell_tris == gpu.grid.cell_tris);
      CHECK(ref.grid.tri_boxes == gpu.grid.tri_boxes);
      CHECK(ref.table.counts == gpu.table.counts);
      CHECK(ref.table.prefix == gpu.table.prefix);
      CHECK(ref.table.total == gpu.table.total);
    }
  }
}

TEST_CASE("drop-in collide equals the reference collide (hits, bitwise values)") {
  oracle::Rng rng(44);
  for (int trial = 0; trial < 4; ++trial) {
    const auto scene = oracle::random_two_cloth_scene(rng, 8);
    for (CollisionMode mode : {CollisionMode::Discrete, CollisionMode::Continuous}) {
      CollisionParams params;
      params.thickness = mode == CollisionMode::Discrete ? 0.1 : 0.01;
      for (int n : {1, 2}) {
        Engine engine(n);
        const auto ref = collide(engine, scene.soup, scene.x_begin, scene.x_end, mode, params);
        const auto gpu = gpu::collide(engine, scene.soup, scene.x_begin, scene.x_end, mode, params);
        REQUIRE(ref.proximities.size() == gpu.proximities.size());
        REQUIRE(ref.impacts.size() == gpu.impacts.size());
        for (std::size_t i = 0; i < ref.proximities.size(); ++i) {
          const auto &a = ref.proximities[i], &b = gpu.proximities[i];
          CHECK((a.kind == b.kind && a.a == b.a && a.b == b.b && a.gap == b.gap && a.normal == b.normal &&
                 a.weights == b.weights));
        }
        for (std::size_t i = 0; i < ref.impacts.size(); ++i) {
          const auto &a = ref.impacts[i], &b = gpu.impacts[i];
          CHECK((a.kind == b.kind && a.a == b.a && a.b == b.b && a.toi == b.toi && a.normal == b.normal &&
                 a.weights == b.weights));
        }
      }
    }
  }
}

TEST_CASE("drop-in build_zones / distribute_zones / resolve_zones equal the reference (bitwise positions)") {
  // test_response.cpp:189-216 scene (resolves) and random_two_cloth_scene
  // (test_response.cpp:218-240 recipe; the reference gives up: ZoneFailure)
  auto soup = CollisionSoup::build({{0, 1, 2}, {3, 4, 5}}, 6, std::vector<std::uint8_t>(6, 1));
  std::vector<Vec3> x0 = {Vec3(-1, -1, 0), Vec3(2, -1, 0), Vec3(0.2, 2, 0),
                          Vec3(0.2, 0.2, 0.05), Vec3(1.5, 0.3, 0.5), Vec3(0.2, 1.5, 0.5)};
  std::vector<Vec3> x1 = x0;
  x1[3] = Vec3(0.2, 0.2, -0.08);
  std::vector<double> mass(6, 0.1);
  CollisionParams cparams;
  cparams.thickness = 0.01;
  ZoneSolveParams zparams;
  zparams.clearance = 0.005;
  Engine engine(2);
  auto xr = x1, xg = x1;
  const auto rr = resolve_zones(engine, soup, x0, xr, mass, cparams, zparams);
  const auto rg = gpu::resolve_zones(engine, soup, x0, xg, mass, cparams, zparams);
  CHECK(rr.outer_iterations == rg.outer_iterations);
  CHECK(rr.zone_count == rg.zone_count);
  CHECK(rr.first_round_impacts == rg.first_round_impacts);
  CHECK(xr == xg);

  oracle::Rng rng(52);
  for (int trial = 0; trial < 3; ++trial) {
    const auto scene = oracle::random_two_cloth_scene(rng, 6 + 2 * trial);
    std::vector<double> m(static_cast<std::size_t>(scene.soup.vertex_count), 0.05);
    const auto brute = collide(engine, scene.soup, scene.x_begin, scene.x_end, CollisionMode::Continuous,
                               CollisionParams{});
    const auto zr = build_zones(brute.impacts, scene.soup);
    const auto zg = gpu::build_zones(brute.impacts, scene.soup);
    REQUIRE(zr.size() == zg.size());
    for (std::size_t z = 0; z < zr.size(); ++z) {
      CHECK(zr[z].impacts == zg[z].impacts);
      CHECK(zr[z].vertices == zg[z].vertices);
    }
    CHECK(distribute_zones(zr, 3) == gpu::distribute_zones(zg, 3));
    std::string er, eg;
    auto a = scene.x_end, b = scene.x_end;
    try {
      resolve_zones(engine, scene.soup, scene.x_begin, a, m, CollisionParams{}, ZoneSolveParams{});
    } catch (const ZoneFailure& e) {
      er = e.what();
    }
    try {
      gpu::resolve_zones(engine, scene.soup, scene.x_begin, b, m, CollisionParams{}, ZoneSolveParams{});
    } catch (const ZoneFailure& e) {
      eg = e.what();
    }
    CHECK(er == eg);
    CHECK(a == b);
  }
}

namespace {

// Two stacked grid layers in DCD proximity (contacts every step).
ClothMesh two_layer_cloth(int nx, double spacing, double gap) {
  std::vector<Vec3> verts;
  std::vector<std::array<int, 3>> tris;
  for (int layer = 0; layer < 2; ++layer) {
    const auto g = make_grid_mesh(nx, nx, spacing * (nx - 1), spacing * (nx - 1), Vec3(0, 0, layer * gap), 0.15);
    const int off = static_cast<int>(verts.size());
    verts.insert(verts.end(), g.rest_positions.begin(), g.rest_positions.end());
    for (const auto& t : g.triangles) tris.push_back({t[0] + off, t[1] + off, t[2] + off});
  }
  return ClothMesh::build(std::move(verts), std::move(tris), 0.15);
}

template <class V>
double max_rel_err(const V& a, const V& b) {
  double scale = 1e-300, err = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    scale = std::max(scale, std::abs(a[i]));
    err = std::max(err, std::abs(a[i] - b[i]));
  }
  return err / scale;
}

}  // namespace

TEST_CASE("drop-in spmv_serial is bitwise the reference spmv_serial") {
  oracle::Rng rng(61);
  for (int trial = 0; trial < 8; ++trial) {
    const int rows = rng.uniform_int(1, 60);
    const auto a = oracle::random_bell(rng, rows, 4);
    std::vector<double> x(static_cast<std::size_t>(3 * rows));
    for (auto& v : x) v = rng.uniform(-2.0, 2.0);
    CHECK(spmv_serial<double>(a, x) == gpu::spmv_serial<double>(a, x));
  }
  const auto a = oracle::random_bell(rng, 5, 2);
  std::vector<double> bad(4);
  CHECK_THROWS_AS(gpu::spmv_serial<double>(a, bad), DimensionError);
}

TEST_CASE("drop-in step_system equals the reference step_system, with contacts, across repeated calls") {
  const auto mesh = two_layer_cloth(9, 0.004, 0.003);
  const int p = mesh.vertex_count();
  std::vector<std::uint8_t> pinned(static_cast<std::size_t>(p), 0);
  pinned[0] = pinned[8] = 1;
  const auto soup = CollisionSoup::build(mesh.triangles, p, std::vector<std::uint8_t>(static_cast<std::size_t>(p), 1));
  MaterialParams params;
  params.damping = 0.001;
  params.air_drag = 0.2;
  oracle::Rng rng(62);
  const double dt = 1.0 / 240.0;
  for (int n : {1, 2}) {
    Engine engine(n);
    SimState state = SimState::rest(mesh);
    for (int call = 0; call < 4; ++call) {
      CAPTURE(n);
      CAPTURE(call);
      for (auto& v : state.v) v = rng.vec3(-0.2, 0.2);
      CollisionParams cp;
      cp.thickness = 0.005;
      const auto prox = collide(engine, soup, state.x, state.x, CollisionMode::Discrete, cp);
      ContactParams kp;
      kp.thickness = 0.005;
      const auto contacts = proximities_to_elements(prox.proximities, soup, state.x, state.v, mesh.vertex_mass, dt, kp);
      REQUIRE(!contacts.empty());
      const auto ref = step_system<double>(engine, mesh, state, params, pinned, contacts, dt, Vec3(0, 0, -9.81),
                                           Vec3(0.5, 0, 0));
      const auto gpu = gpu::step_system<double>(engine, mesh, state, params, pinned, contacts, dt, Vec3(0, 0, -9.81),
                                                Vec3(0.5, 0, 0));
      CHECK((dense(ref.matrix) - dense(gpu.matrix)).cwiseAbs().maxCoeff() == 0.0);
      CHECK(max_rel_err(ref.rhs.gather(), gpu.rhs.gather()) <= 1e-12);
      // the cached static list must follow a material change
      if (call == 2) params.shear *= 2.0;
    }
  }
}

TEST_CASE("a Simulator-style loop on the drop-ins tracks the reference loop") {
  // driver.cpp:132-206 without impact zones: DCD collide -> contact
  // elements -> step_system -> pcg_solve -> v += dv, x += dt v, with every
  // hot-path call swapped for weft::gpu:: in the second loop.
  const auto mesh = two_layer_cloth(10, 0.004, 0.003);
  const int p = mesh.vertex_count();
  std::vector<std::uint8_t> pinned(static_cast<std::size_t>(p), 0);
  for (int i = 0; i < 10; ++i) pinned[static_cast<std::size_t>(90 + i)] = pinned[static_cast<std::size_t>(190 + i)] = 1;
  const auto soup = CollisionSoup::build(mesh.triangles, p, std::vector<std::uint8_t>(pinned.size(), 1));
  const double dt = 1.0 / 240.0;
  const int n = 2;
  Engine engine(n);
  ValidatedSchedule sched(generate_work_queues(FatTree::make(n)), n);
  PcgConfig cfg;
  cfg.rel_tolerance = 1e-10;
  cfg.max_iterations = 4000;  // tol 1e-10 on the contact-stiffened system needs more than the default 400
  CollisionParams cp;
  cp.thickness = 0.005;
  ContactParams kp;
  kp.thickness = 0.005;
  SimState sr = SimState::rest(mesh), sg = sr;
  for (int step = 0; step < 6; ++step) {
    CAPTURE(step);
    const auto pr = collide(engine, soup, sr.x, sr.x, CollisionMode::Discrete, cp);
    const auto pg = gpu::collide(engine, soup, sg.x, sg.x, CollisionMode::Discrete, cp);
    CHECK(pr.proximities.size() == pg.proximities.size());
    const auto cr = proximities_to_elements(pr.proximities, soup, sr.x, sr.v, mesh.vertex_mass, dt, kp);
    const auto cg = proximities_to_elements(pg.proximities, soup, sg.x, sg.v, mesh.vertex_mass, dt, kp);
    const auto ar = step_system<double>(engine, mesh, sr, MaterialParams{}, pinned, cr, dt, Vec3(0, 0, -9.81),
                                        Vec3::Zero());
    const auto ag = gpu::step_system<double>(engine, mesh, sg, MaterialParams{}, pinned, cg, dt, Vec3(0, 0, -9.81),
                                             Vec3::Zero());
    DistVector<double> dr(&engine, ar.matrix.partitions), dg(&engine, ag.matrix.partitions);
    const auto rr = pcg_solve(engine, ar.matrix, sched, ar.rhs, dr, cfg);
    const auto rg = gpu::pcg_solve(engine, ag.matrix, sched, ag.rhs, dg, cfg);
    REQUIRE(rr.converged);
    REQUIRE(rg.converged);
    const auto vr = dr.gather(), vg = dg.gather();
    for (int i = 0; i < p; ++i) {
      for (int c = 0; c < 3; ++c) {
        sr.v[static_cast<std::size_t>(i)][c] += vr[static_cast<std::size_t>(3 * i + c)];
        sg.v[static_cast<std::size_t>(i)][c] += vg[static_cast<std::size_t>(3 * i + c)];
      }
      sr.x[static_cast<std::size_t>(i)] += dt * sr.v[static_cast<std::size_t>(i)];
      sg.x[static_cast<std::size_t>(i)] += dt * sg.v[static_cast<std::size_t>(i)];
    }
    std::vector<double> xr, xg;
    for (int i = 0; i < p; ++i)
      for (int c = 0; c < 3; ++c) {
        xr.push_back(sr.x[static_cast<std::size_t>(i)][c]);
        xg.push_back(sg.x[static_cast<std::size_t>(i)][c]);
      }
    // the north_star tolerance is 1e-5 relative; the dot products' association
    // differs by design, so the loops agree to round-off growth
    const double err = max_rel_err(xr, xg);
    CAPTURE(err);
    CHECK(err <= 1e-6);
  }
}

TEST_CASE("Precision::Single drop-ins: spmv_pipelined<float> bitwise, pcg_solve<float> and step_system<float> track the reference") {
  oracle::Rng rng(31);
  for (int n : {1, 2}) {
    Engine engine(n);
    ValidatedSchedule sched = n == 1 ? ValidatedSchedule() : ValidatedSchedule(generate_work_queues(FatTree::make(n)), n);
    const int rows = 30;
    const auto g64 = oracle::random_bell(rng, rows, 3);
    std::vector<BlockEntry<float>> entries;
    for (int r = 0; r < rows; ++r)
      for (int s = 0; s < g64.ell_width(); ++s) {
        const auto c = g64.col_at(r, s);
        if (c == BellMatrix<double>::kNoBlock) break;
        BlockEntry<float> e;
        e.row = r;
        e.col = c;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) e.m[static_cast<std::size_t>(3 * i + j)] = static_cast<float>(g64.value_at(r, s, i, j));
        entries.push_back(e);
      }
    const auto parts = make_partitions(rows, n);
    const auto split = partition_matrix(BellMatrix<float>::from_entries(rows, entries), parts);
    std::vector<float> xg(static_cast<std::size_t>(3 * rows));
    for (auto& v : xg) v = static_cast<float>(rng.uniform(-1.0, 1.0));
    DistVector<float> x(&engine, parts), y(&engine, parts), yr(&engine, parts);
    for (const auto& part : parts)
      std::copy(xg.begin() + 3 * part.begin, xg.begin() + 3 * part.end, x.local(part.device_id).begin());
    SpmvWorkspace<float> ws(n, split.padded_len);
    gpu::spmv_pipelined(engine, split, sched, x, y, ws);
    spmv_pipelined(engine, split, sched, x, yr, ws);
    CHECK(y.gather() == yr.gather());
  }
  // step_system<float> + pcg_solve<float> on a small cloth vs the reference's
  const auto mesh = make_grid_mesh(12, 12, 0.2, 0.2, Vec3(0, 0, 0), 0.15);
  MaterialParams mat;
  std::vector<std::uint8_t> pinned(static_cast<std::size_t>(mesh.vertex_count()), 0);
  for (int i = 0; i < 12; ++i) pinned[static_cast<std::size_t>(i)] = 1;
  SimState st = SimState::rest(mesh);
  for (auto& v : st.v) v = Vec3(rng.uniform(-0.1, 0.1), rng.uniform(-0.1, 0.1), rng.uniform(-0.1, 0.1));
  for (int n : {1, 2}) {
    Engine engine(n);
    ValidatedSchedule sched = n == 1 ? ValidatedSchedule() : ValidatedSchedule(generate_work_queues(FatTree::make(n)), n);
    const Vec3 g(0, 0, -9.81), w(0, 0, 0);
    auto sg = gpu::step_system<float>(engine, mesh, st, mat, pinned, {}, 1.0 / 240, g, w);
    auto sr = step_system<float>(engine, mesh, st, mat, pinned, {}, 1.0 / 240, g, w);
    const auto mg = gather_matrix(sg.matrix), mr = gather_matrix(sr.matrix);
    CHECK(mg.block_rows() == mr.block_rows());
    bool same = true;
    for (int r = 0; r < mr.block_rows(); ++r)
      for (int s = 0; s < mr.ell_width(); ++s) {
        if (mr.col_at(r, s) != mg.col_at(r, s)) same = false;
        if (mr.col_at(r, s) == BellMatrix<float>::kNoBlock) break;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) same = same && mr.value_at(r, s, i, j) == mg.value_at(r, s, i, j);
      }
    CHECK(same);  // SpdProjected: bitwise
    PcgConfig cfg;
    cfg.rel_tolerance = 1e-5;
    DistVector<float> dg(&engine, sg.matrix.partitions), dr(&engine, sr.matrix.partitions);
    const auto rg = gpu::pcg_solve(engine, sg.matrix, sched, sg.rhs, dg, cfg);
    const auto rr = pcg_solve(engine, sr.matrix, sched, sr.rhs, dr, cfg);
    CHECK(rg.converged);
    CHECK(std::abs(rg.iterations - rr.iterations) <= 2);
    const auto a = dg.gather(), b = dr.gather();
    double diff = 0.0, mag = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
      diff = std::max(diff, std::abs(static_cast<double>(a[i]) - static_cast<double>(b[i])));
      mag = std::max(mag, std::abs(static_cast<double>(b[i])));
    }
    CHECK(diff <= 1e-3 * mag);
  }
}
