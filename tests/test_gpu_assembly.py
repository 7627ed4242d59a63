"""GPU assembly parity: pattern, matrix and rhs bitwise vs the reference
(golden fixtures) and the C oracle, in SpdProjected and Exact modes. The
hinge angle uses a correctly rounded atan2 and the reference glibc's, which
is not (tests/test_hinge_atan2.py): they agree on these inputs; at config D
a handful of near-midpoint hinges differ by one ulp (test_gpu_configD.py
counts them)."""
import glob
import os

import numpy as np
import pytest

from oracle_bindings import ELEMENT_DTYPE, JAC_EXACT, JAC_SPD, ORACLE
from problems import contact_elements, hinge_atan2_split_vertices, with_drag

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def weft():
    from paper_2008_00409_b200 import weft as w
    return w


def gpu_fill(weft, n, elems, x, xa, v, mass, pinned, dt, mode, contacts=None):
    eng = weft.Engine(n)
    eng.set_vertices(mass, pinned)
    eng.set_elements(elems)
    if contacts is not None:
        eng.set_contacts(contacts)
    eng.fill_matrix(x, xa, v, dt, mode)
    m = eng.download_matrix()
    m.rhs = eng.download_rhs()
    return eng, m


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "assembly_*.npz"))))
@pytest.mark.parametrize("mode,tag", [(JAC_SPD, "spd"), (JAC_EXACT, "exact")])
@pytest.mark.parametrize("n", [1, 2, 4])
def test_assembly_vs_reference_golden(weft, path, mode, tag, n):
    g = dict(np.load(path))
    elems = g["elems"].view(ELEMENT_DTYPE)
    # split the reference's single list into static + contacts (contacts last)
    k = int(np.argmax(elems["kind"] == 4)) if np.any(elems["kind"] == 4) else len(elems)
    eng, m = gpu_fill(weft, n, elems[:k], g["x"], g["x_adv"], g["v"], g["mass"], g["pinned"], float(g["dt"]), mode,
                      elems[k:] if k < len(elems) else None)
    assert np.array_equal(m.row_ptr, g[f"{tag}_row_ptr"]) and np.array_equal(m.cols, g[f"{tag}_cols"])
    # Exact mode scales the bend Hessian by (theta - theta0) and the rhs
    # carries the bend force: both go through the hinge atan2 and are
    # bitwise on these fixtures.
    assert np.array_equal(m.vals.view(np.int64), g[f"{tag}_vals"].view(np.int64))
    assert np.array_equal(m.rhs.view(np.int64), g[f"{tag}_rhs"].view(np.int64)), \
        f"{int((m.rhs != g[f'{tag}_rhs']).sum())} rhs entries differ (hinge atan2 1-ulp case?)"
    eng.close()


def test_hinge_atan2_device_equals_host(weft):
    """The device build of cr::atan2 is bitwise the host build (no
    contraction or fast-math difference between them)."""
    import ctypes
    lib = weft.LIB
    rng = np.random.default_rng(4)
    n = 1 << 20
    y = np.concatenate([rng.uniform(-1, 1, n), rng.uniform(-1e-6, 1e-6, n), rng.uniform(-1, 1, n) * 1e-200])
    x = np.concatenate([rng.uniform(-1, 1, n), rng.uniform(1e-5, 1e-4, n), rng.uniform(-1, 1, n) * 1e200])
    host, dev = np.empty_like(y), np.empty_like(y)
    p = lambda a: ctypes.c_void_p(a.ctypes.data)
    assert lib.weft_hinge_atan2_host(ctypes.c_int64(len(y)), p(y), p(x), p(host)) == 0
    eng = weft.Engine(1)
    assert lib.weft_gpu_hinge_atan2(eng._ctx, ctypes.c_int64(len(y)), p(y), p(x), p(dev)) == 0
    eng.close()
    assert np.array_equal(host.view(np.int64), dev.view(np.int64))


def layered_problem(weft, layers=3, nx=24, contacts=40, seed=5, drag=True, damping=0.002):
    from paper_2008_00409_b200 import scenes
    sc = scenes.layered_cloth(layers, nx, seed=seed)
    mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
    mat = list(sc.material)
    mat[5] = damping
    rng = np.random.default_rng(seed)
    elems = mesh.build_elements(tuple(mat))
    if drag:
        elems = with_drag(elems, rng)
    p = mesh.vertex_count
    x = sc.verts.reshape(-1) + rng.uniform(-1e-4, 1e-4, 3 * p)
    v = rng.uniform(-0.2, 0.2, 3 * p)
    dt = sc.dt
    xa = x + dt * v
    cts = contact_elements(rng, p, contacts) if contacts else None
    return dict(elems=elems, contacts=cts, x=x, xa=xa, v=v, mass=mesh.vertex_mass, pinned=sc.pinned, dt=dt)


def assert_bitwise_but_split_hinges(m, o, pr):
    """Bitwise, except rows/blocks touching a hinge whose angle glibc rounds
    differently from the correctly rounded atan2 (one ulp of the angle)."""
    dv = np.nonzero((m.vals.view(np.int64) != o.vals.view(np.int64)).reshape(len(m.cols), -1).any(axis=1))[0]
    dr = np.nonzero(m.rhs.view(np.int64) != o.rhs.view(np.int64))[0]
    if len(dv) == 0 and len(dr) == 0:
        return
    split = hinge_atan2_split_vertices(pr["elems"], [pr["x"], pr["xa"]])
    rows_r = set((dr // 3).tolist())
    assert rows_r <= split, sorted(rows_r - split)[:10]
    blk = dv
    brow = np.searchsorted(m.row_ptr, blk, side="right") - 1
    bad = [(int(r), int(c)) for r, c in zip(brow, m.cols[blk]) if int(r) not in split or int(c) not in split]
    assert not bad, bad[:10]
    rel = np.abs(m.rhs - o.rhs).max() / np.abs(o.rhs).max()
    assert rel <= 1e-12


@pytest.mark.parametrize("contacts", [0, 50])
@pytest.mark.parametrize("mode", [JAC_SPD, JAC_EXACT])
def test_assembly_vs_oracle_layered(weft, contacts, mode):
    pr = layered_problem(weft, contacts=contacts)
    full = pr["elems"] if pr["contacts"] is None else np.concatenate([pr["elems"], pr["contacts"]])
    o = ORACLE.fill_matrix(full, pr["x"], pr["xa"], pr["v"], pr["mass"], pr["pinned"], pr["dt"], mode)
    mats = []
    for n in (1, 2, 4):
        eng, m = gpu_fill(weft, n, pr["elems"], pr["x"], pr["xa"], pr["v"], pr["mass"], pr["pinned"], pr["dt"], mode,
                          pr["contacts"])
        assert np.array_equal(m.row_ptr, o.row_ptr) and np.array_equal(m.cols, o.cols)
        assert_bitwise_but_split_hinges(m, o, pr)
        mats.append(m)
        eng.close()
    # partition independence of the gathered matrix (test_assembly.cpp:263-280)
    assert all(np.array_equal(mats[0].vals, mm.vals) and np.array_equal(mats[0].rhs, mm.rhs) for mm in mats)


def test_contacts_change_per_step(weft):
    pr = layered_problem(weft, contacts=0, seed=9)
    rng = np.random.default_rng(3)
    eng = weft.Engine(2)
    eng.set_vertices(pr["mass"], pr["pinned"])
    eng.set_elements(pr["elems"])
    p = len(pr["mass"])
    for step, count in enumerate([30, 0, 80, 5]):
        cts = contact_elements(rng, p, count) if count else np.zeros(0, ELEMENT_DTYPE)
        eng.set_contacts(cts)
        eng.fill_matrix(pr["x"], pr["xa"], pr["v"], pr["dt"])
        m = eng.download_matrix()
        full = np.concatenate([pr["elems"], cts])
        o = ORACLE.fill_matrix(full, pr["x"], pr["xa"], pr["v"], pr["mass"], pr["pinned"], pr["dt"])
        assert np.array_equal(m.cols, o.cols) and np.array_equal(m.vals, o.vals), step
    eng.close()


def test_step_system_matches_fill(weft):
    pr = layered_problem(weft, contacts=10, seed=4)
    eng = weft.Engine(1)
    eng.set_vertices(pr["mass"], pr["pinned"])
    eng.set_elements(pr["elems"])
    eng.set_contacts(pr["contacts"])
    eng.step_system(pr["x"], pr["v"], pr["dt"])
    a = eng.download_matrix()
    eng.fill_matrix(pr["x"], pr["x"] + pr["dt"] * pr["v"], pr["v"], pr["dt"])
    b = eng.download_matrix()
    assert np.array_equal(a.vals, b.vals)
    eng.close()


def test_assembly_errors(weft):
    from problems import contact_elements as ce
    eng = weft.Engine(1)
    eng.set_vertices(np.array([0.0]), np.array([0], np.uint8))
    eng.set_elements(np.zeros(0, ELEMENT_DTYPE))
    with pytest.raises(weft.DimensionError, match="fill_matrix: vertex 0 has non-positive mass"):
        eng.fill_matrix(np.zeros(3), np.zeros(3), np.zeros(3), 0.01)
    with pytest.raises(weft.DimensionError, match="dt must be positive"):
        eng.fill_matrix(np.zeros(3), np.zeros(3), np.zeros(3), 0.0)
    bad = ce(np.random.default_rng(0), 8, 1)
    bad["stencil_size"] = 1
    bad["stencil"][0] = [7, -1, -1, -1]
    with pytest.raises(weft.DimensionError, match="stencil vertex 7 outside all partitions"):
        eng.set_elements(bad)
    eng.close()


def test_gravity_and_pinned_known_answers(weft):
    # test_assembly.cpp:130-154 and :297-321
    ext = np.zeros(1, ELEMENT_DTYPE)
    ext["kind"] = 3
    ext["stencil_size"] = 1
    ext["stencil"] = [0, -1, -1, -1]
    ext["data"][0, :3] = [0.0, 0.0, 2.5 * -9.81]
    eng = weft.Engine(1)
    eng.set_vertices(np.array([2.5]), np.array([0], np.uint8))
    eng.set_elements(ext)
    eng.fill_matrix(np.zeros(3), np.zeros(3), np.zeros(3), 0.01)
    m = eng.download_matrix()
    assert np.array_equal(m.vals[0], (2.5 * np.eye(3)).reshape(9))
    rhs = eng.download_rhs()
    assert rhs[0] == 0.0 and rhs[1] == 0.0 and rhs[2] == pytest.approx(0.01 * 2.5 * -9.81, rel=1e-15)
    # spring between a pinned and a free vertex
    spring = np.zeros(3, ELEMENT_DTYPE)
    spring["kind"] = [2, 3, 3]
    spring["stencil_size"] = [2, 1, 1]
    spring["stencil"] = [[0, 1, -1, -1], [0, -1, -1, -1], [1, -1, -1, -1]]
    spring["data"][0, :2] = [0.5, 100.0]
    spring["data"][1:, 2] = -9.81
    eng.set_vertices(np.array([1.0, 1.0]), np.array([1, 0], np.uint8))
    eng.set_elements(spring)
    eng.fill_matrix(np.array([0, 0, 0, 0.7, 0, 0.0]), np.array([0, 0, 0, 0.7, 0, 0.0]), np.zeros(6), 0.01)
    m = eng.download_matrix()
    rhs = eng.download_rhs()
    assert list(m.cols) == [0, 1] and np.array_equal(m.vals[0], np.eye(3).reshape(9))
    assert np.all(rhs[:3] == 0.0)
    eng.close()
