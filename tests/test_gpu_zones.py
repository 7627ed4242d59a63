"""Impact zones on the GPU vs the compiled reference:
build_zones (response.cpp:108-162) bitwise zone structure, resolve_zones
(:338-400) bitwise positions / reports / ZoneFailure messages (golden fixtures
from oracle/_ref + live comparisons), the known answers of
proj/tests/test_response.cpp:99-270, and the full step_impl with zones
(driver.cpp:96-215) vs the reference step."""
import glob
import os

import numpy as np
import pytest

from oracle_bindings import REF, RefError, RefSim

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
REPORT = ("outer_iterations", "zone_count", "max_zone_vertices", "impacts_resolved", "first_round_impacts")


@pytest.fixture(scope="module")
def weft():
    from paper_2008_00409_b200 import weft as w
    return w


def vf(a, b):
    return (0, a, b)


def gpu_zones(weft, nv, tris, kab, movable=None):
    with weft.Engine(1) as eng:
        eng.set_soup(nv, np.asarray(tris, np.int32))
        if movable is not None:
            eng.set_soup_movable(movable)
        return eng.build_zones(np.asarray(kab, np.int32))


def test_zone_construction_known_answers(weft):
    """test_response.cpp:99-127."""
    tris = [[0, 1, 2], [3, 4, 5], [6, 7, 8]]
    iz, zv = gpu_zones(weft, 12, tris, [vf(9, 0), vf(9, 1)])
    assert len(zv) == 1 and list(iz) == [0, 0]
    assert list(zv[0]) == [0, 1, 2, 3, 4, 5, 9]
    iz, zv = gpu_zones(weft, 12, tris, [vf(9, 0), vf(10, 2)])
    assert len(zv) == 2 and list(iz) == [0, 1]
    iz, zv = gpu_zones(weft, 12, tris, [vf(9, 0), vf(9, 1), vf(10, 1)])
    assert len(zv) == 1 and list(iz) == [0, 0, 0]


def test_zone_distribution_known_answers(weft):
    """test_response.cpp:144-172 (host logic behind the C-ABI)."""
    assert [len(a) for a in weft.distribute_zones([3, 3, 3, 3], 4)] == [1, 1, 1, 1]
    assert weft.distribute_zones([8, 1, 1, 1, 1], 2) == [[0], [1, 2, 3, 4]]
    a = weft.distribute_zones([100], 4)
    assert a[0] == [0] and a[1] == []


def random_impacts(rng, nv, tris, n, edges_count):
    kinds = rng.integers(0, 2, n)
    out = np.zeros((n, 3), np.int32)
    for i, k in enumerate(kinds):
        if k == 0:
            out[i] = (0, rng.integers(0, nv), rng.integers(0, len(tris)))
        else:
            a, b = sorted(rng.choice(edges_count, 2, replace=False))
            out[i] = (1, a, b)
    return out


def soup_edge_count(tris):
    e = set()
    for t in tris:
        for k in range(3):
            a, b = int(t[k]), int(t[(k + 1) % 3])
            e.add((min(a, b), max(a, b)))
    return len(e)


@pytest.mark.ref
@pytest.mark.parametrize("seed,nx,n", [(1, 6, 20), (2, 12, 200), (3, 30, 3000), (4, 60, 20000)])
def test_build_zones_vs_reference(weft, seed, nx, n):
    """Random impact lists on a pinned grid soup: identical zone ids per
    impact and identical sorted movable vertex lists (union-find on the
    device vs the reference's sequential union-find)."""
    from paper_2008_00409_b200 import scenes
    sc = scenes.layered_cloth(1, nx, seed=seed)
    nv = len(sc.verts)
    rng = np.random.default_rng(seed)
    kab = random_impacts(rng, nv, sc.tris, n, soup_edge_count(sc.tris))
    mv = (1 - sc.pinned).astype(np.uint8)
    iz, zv = gpu_zones(weft, nv, sc.tris, kab, mv)
    rz, rv = REF.build_zones(nv, sc.tris, kab, mv)
    assert np.array_equal(iz, rz)
    assert len(zv) == len(rv) and all(np.array_equal(a, b) for a, b in zip(zv, rv))
    # zone vertex sets are disjoint (test_response.cpp:129-142)
    allv = np.concatenate(zv) if zv else np.zeros(0, np.int32)
    assert len(np.unique(allv)) == len(allv)


def resolve_gpu(weft, nv, tris, x0, x1, mass, mv, th, zp):
    with weft.Engine(2) as eng:
        eng.set_soup(nv, np.asarray(tris, np.int32))
        eng.set_soup_movable(mv)
        prm = weft.ZoneParams(*[float(zp[0]), float(zp[1]), float(zp[2]), int(zp[3]), int(zp[4]), int(zp[5]),
                                int(zp[6]), float(zp[7])])
        try:
            xc, rep = eng.resolve_zones(x0, x1, mass, th, 1.5, prm)
            return 0, "", xc, rep
        except weft.ZoneFailure as e:
            return 7, str(e), e.x_candidate, e.report


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "zones_*.npz"))))
def test_resolve_zones_vs_reference_golden(weft, path):
    g = dict(np.load(path))
    st, msg, xc, rep = resolve_gpu(weft, int(g["nv"]), g["tris"], g["x0"], g["x1"], g["mass"], g["movable"],
                                   float(g["thickness"]), g["params"])
    assert st == int(g["status"]) and msg == str(g["message"])
    if st == 0:
        assert [getattr(rep, f) for f in REPORT] == g["report"].tolist()
    assert np.array_equal(xc, g["x_out"]), float(np.abs(xc - g["x_out"]).max())


@pytest.mark.ref
@pytest.mark.parametrize("layers,nx,seed,amp", [(2, 20, 11, 0.5), (3, 24, 12, 0.6), (2, 64, 13, 0.45)])
def test_resolve_zones_vs_reference_live(weft, layers, nx, seed, amp):
    from paper_2008_00409_b200 import scenes
    sc = scenes.layered_cloth(layers, nx, seed=seed)
    nv = len(sc.verts)
    x0 = sc.verts.reshape(-1).copy()
    x1 = x0 + np.random.default_rng(seed).uniform(-amp, amp, x0.shape) * sc.spacing
    mv = (1 - sc.pinned).astype(np.uint8)
    mass = np.random.default_rng(seed + 1).uniform(5e-4, 2e-3, nv)
    zp = [0.5 * sc.thickness, 10.0, 1e-8, 25, 64, 10, 3, 8.0]
    rs, rmsg, rx, rrep = REF.resolve_zones(nv, sc.tris, mass, x0, x1, thickness=sc.thickness, devices=2, params=zp,
                                           movable=mv)
    st, msg, xc, rep = resolve_gpu(weft, nv, sc.tris, x0, x1, mass, mv, sc.thickness, zp)
    assert (st, msg) == (rs, rmsg)
    if st == 0:
        assert rrep["first_round_impacts"] > 0
        assert {f: getattr(rep, f) for f in REPORT} == rrep
    assert np.array_equal(xc, rx), float(np.abs(xc - rx).max())


def kat_scene():
    tris = np.array([[0, 1, 2], [3, 4, 5]], np.int32)
    x0 = np.array([[-1, -1, 0], [2, -1, 0], [0.2, 2, 0], [0.2, 0.2, 0.05], [1.5, 0.3, 0.5], [0.2, 1.5, 0.5]], float)
    x1 = x0.copy()
    x1[3] = (0.2, 0.2, -0.08)
    return tris, x0.reshape(-1), x1.reshape(-1)


def test_resolve_zones_known_answers(weft):
    """test_response.cpp:174-216,242-270: zero impacts leave positions
    untouched; one vertex-face penetration is resolved (<= 5 outer rounds,
    clean re-CCD, vertex-face separation >= 0.9 clearance); only zone
    vertices move."""
    tris, x0, _ = kat_scene()
    with weft.Engine(1) as eng:
        eng.set_soup(6, tris)
        x1 = x0 + np.tile([0.01, 0.0, 0.0], 6)
        xc, rep = eng.resolve_zones(x0, x1, np.full(6, 0.1), 0.005, 1.5, weft.ZoneParams())
        assert rep.outer_iterations == 0 and np.array_equal(xc, x1)
    tris, x0, x1 = kat_scene()
    with weft.Engine(2) as eng:
        eng.set_soup(6, tris)
        kab, _ = eng.collide(x0, x1, 1, 0.01)
        assert len(kab) > 0
        _, zv = eng.build_zones(kab)
        in_zone = np.zeros(6, bool)
        in_zone[np.concatenate(zv)] = True
        xc, rep = eng.resolve_zones(x0, x1, np.full(6, 0.1), 0.01, 1.5, weft.ZoneParams(clearance=0.005))
        assert 1 <= rep.outer_iterations <= 5
        kab2, _ = eng.collide(x0, xc, 1, 0.01)
        assert len(kab2) == 0
    x = xc.reshape(-1, 3)
    # vertex 3 above the plane of triangle 0 by at least 0.9 * clearance
    n = np.cross(x[1] - x[0], x[2] - x[0])
    n /= np.linalg.norm(n)
    assert abs(np.dot(x[3] - x[0], n)) >= 0.9 * 0.005
    assert np.array_equal(xc.reshape(-1, 3)[~in_zone], x1.reshape(-1, 3)[~in_zone])
    if REF is not None:
        st, msg, rx, rrep = REF.resolve_zones(6, tris, np.full(6, 0.1), x0, x1, thickness=0.01, devices=2,
                                              params=[0.005, 10.0, 1e-8, 25, 64, 10, 3, 8.0])
        assert st == 0 and np.array_equal(xc, rx)


@pytest.mark.ref
@pytest.mark.parametrize("layers,nx,thf,seed,steps", [(2, 16, 2.0, 3, 4), (2, 24, 1.5, 4, 3)])
def test_sim_steps_with_zones_match_reference(weft, layers, nx, thf, seed, steps):
    """The full Simulator::step_impl (driver.cpp:96-215): DCD -> contacts ->
    assembly -> PCG -> candidate -> CCD + resolve_zones -> commit with the
    velocity correction, on the device vs the compiled reference. The PCG's
    dot association differs (tree vs sequential sums), so the bar is the
    north_star state tolerance, and failures must happen at the same step
    (the reference's cloth model tangles on these pinned layered scenes: its
    zone solver gives up within a few steps, ZoneFailure)."""
    from paper_2008_00409_b200 import scenes
    sc = scenes.layered_cloth(layers, nx, seed=seed)
    th = thf * sc.thickness
    mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
    p = mesh.vertex_count
    eng = weft.Engine(1)
    eng.set_vertices(mesh.vertex_mass, sc.pinned)
    eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
    eng.set_soup(p, sc.tris)
    x0 = sc.verts.reshape(-1).copy()
    eng.sim_set_state(x0, np.zeros_like(x0))
    ref = RefSim(REF, sc.verts, sc.tris, sc.pinned, sc.density, sc.material, 2)
    zp = weft.ZoneParams(clearance=0.5 * th)
    params = weft.SimParams(sc.dt, th, 1.5, weft.PcgConfig(1e-9, 3000), weft.JAC_SPD, contacts=1, zones=1, zone=zp)
    zoned = 0
    for k in range(steps):
        try:
            rr = ref.step_contacts(sc.dt, th, tol=1e-9, max_it=3000, zones=zp.as_array())
        except RefError as e:
            with pytest.raises(weft.ZoneFailure) as ei:
                eng.sim_step(params)
            # the surviving zone ids come from a chaotic 10-round solve over
            # states that agree to the tolerance, not bitwise: same failure,
            # same message up to the id list
            head = "impact zones unresolved after 10 outer iterations; zone ids:"
            assert str(e).startswith(head) and str(ei.value).startswith(head)
            break
        rg = eng.sim_step(params)
        assert rg.proximities == rr["proximities"] and rg.contact_elements == rr["contacts"]
        assert rg.impacts == rr["impacts"]
        assert (rg.zone_count, rg.zone_outer) == (rr["zone_count"], rr["zone_outer"])
        zoned += rg.zone_count
        xg = np.zeros(3 * p)
        vg = np.zeros(3 * p)
        eng.sim_get_state(xg, vg)
        xr, vr = ref.get_state()
        assert np.abs(xg - xr).max() <= 1e-5 * np.abs(xr).max()
        assert np.abs(vg - vr).max() <= 1e-5 * max(np.abs(vr).max(), 1e-12) + 1e-12
    if thf == 1.5:
        assert zoned > 0  # at least one step resolved zones before any failure
    ref.close()
    eng.close()
