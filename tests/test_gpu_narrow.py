"""Narrow phase vs the compiled reference's collide
(collision.cpp:391-417): identical (kind, a, b) hit sets, bitwise gap / toi,
normals and weights; known answers of proj/tests/test_collision.cpp."""
import glob
import os

import numpy as np
import pytest

from oracle_bindings import CONTINUOUS, DISCRETE, REF

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def weft():
    from paper_2008_00409_b200 import weft as w
    return w


def gpu_collide(weft, nv, tris, x0, x1, mode, thickness, movable=None):
    with weft.Engine(1) as eng:
        eng.set_soup(nv, tris)
        if movable is not None:
            eng.set_soup_movable(movable)
        return eng.collide(x0, x1, mode, thickness)


def assert_same(kab, vals, rk, rv):
    assert kab.shape == rk.shape and np.array_equal(kab, rk)
    assert np.array_equal(vals, rv), float(np.abs(vals - rv).max())


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "narrow_*.npz"))))
def test_narrow_vs_reference_golden(weft, path):
    g = dict(np.load(path))
    kab, vals = gpu_collide(weft, int(g["nv"]), g["tris"], g["x0"], g["x1"], int(g["mode"]), float(g["thickness"]),
                            g["movable"])
    assert_same(kab, vals, g["kab"], g["vals"])


@pytest.mark.ref
@pytest.mark.parametrize("seed", [41, 42, 43, 44])
@pytest.mark.parametrize("mode,thickness", [(DISCRETE, 0.05), (DISCRETE, 0.2), (CONTINUOUS, 0.01)])
def test_narrow_vs_reference_two_cloth(weft, seed, mode, thickness):
    nv, tris, x0, x1 = REF.two_cloth_scene(seed, 8)
    rk, rv = REF.collide(nv, tris, x0, x1, mode, thickness)
    kab, vals = gpu_collide(weft, nv, tris, x0, x1, mode, thickness)
    assert_same(kab, vals, rk, rv)


@pytest.mark.ref
@pytest.mark.parametrize("mode", [DISCRETE, CONTINUOUS])
def test_narrow_vs_reference_layered_pinned(weft, mode):
    from paper_2008_00409_b200 import scenes
    sc = scenes.layered_cloth(3, 14, seed=8)
    rng = np.random.default_rng(4)
    x0 = sc.verts.reshape(-1)
    x1 = x0 + rng.uniform(-0.6, 0.6, x0.shape) * sc.spacing
    movable = (1 - sc.pinned).astype(np.uint8)
    th = 2 * sc.thickness
    rk, rv = REF.collide(len(sc.verts), sc.tris, x0, x1, mode, th, movable=movable)
    assert len(rk) > 100
    kab, vals = gpu_collide(weft, len(sc.verts), sc.tris, x0, x1, mode, th, movable)
    assert_same(kab, vals, rk, rv)


def test_known_answers(weft):
    # vertex crossing a static triangle hits at t = 0.5 (test_collision.cpp:62-68)
    x0 = np.array([[-1, -1, 0], [2, -1, 0], [0, 2, 0], [0, 0, 1], [5, 5, 5], [5, 6, 5]], float)
    x1 = x0.copy()
    x1[3] = [0, 0, -1]
    tris = np.array([[0, 1, 2], [3, 4, 5]], np.int32)
    kab, vals = gpu_collide(weft, 6, tris, x0.reshape(-1), x1.reshape(-1), CONTINUOUS, 0.005)
    vf = [i for i in range(len(kab)) if kab[i, 0] == 0 and kab[i, 1] == 3 and kab[i, 2] == 0]
    assert len(vf) == 1
    assert abs(vals[vf[0], 0] - 0.5) <= 1e-12 and vals[vf[0], 3] > 0.99
    # DCD point-triangle distance and weights (test_collision.cpp:88-102)
    x = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0.25, 0.25, 0.05], [3, 3, 3], [3, 4, 3]], float)
    kab, vals = gpu_collide(weft, 6, tris, x.reshape(-1), None, DISCRETE, 0.1)
    i = [k for k in range(len(kab)) if tuple(kab[k]) == (0, 3, 0)]
    assert len(i) == 1 and abs(vals[i[0], 0] - 0.05) < 1e-12 and abs(vals[i[0], 5] - 0.5) < 1e-12
    # immovable-only pairs are skipped (test_collision.cpp:251-262)
    x = np.array([[0, 0, 0], [0.1, 0, 0], [0, 0.1, 0], [0.02, 0.02, 0.001], [0.12, 0.02, 0.001],
                  [0.02, 0.12, 0.001]], float)
    kab, _ = gpu_collide(weft, 6, tris, x.reshape(-1), None, DISCRETE, 0.005, np.zeros(6, np.uint8))
    assert len(kab) == 0
    kab, _ = gpu_collide(weft, 6, tris, x.reshape(-1), None, DISCRETE, 0.005)
    assert len(kab) > 0


APPEND_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from paper_2008_00409_b200 import scenes, weft
sc = scenes.layered_cloth(3, 30, seed=8)
rng = np.random.default_rng(4)
x0 = sc.verts.reshape(-1)
x1 = x0 + rng.uniform(-0.6, 0.6, x0.shape) * sc.spacing
out = []
with weft.Engine(1) as eng:
    eng.set_soup(len(sc.verts), sc.tris)
    for mode, th in ((weft.DISCRETE, 2 * sc.thickness), (weft.CONTINUOUS, 1e-9)):
        kab, vals = eng.collide(x0, x1, mode, th)
        out += [kab.astype(np.float64).ravel(), vals.ravel()]
np.save(sys.argv[2], np.concatenate(out))
"""


@pytest.mark.parametrize("env", [{"WEFT_WALK_CAP": "64"}, {"WEFT_WALK_APPEND": "0"},
                                 {"WEFT_NARROW_TWO": "0"}, {"WEFT_NARROW_TWO": "3", "WEFT_NARROW_FCAP": "64"}])
def test_append_feed_overflow_and_ordered_feed(tmp_path, env):
    """The order-free narrow-phase feed (append mode of the candidate walk)
    re-run after overflowing a tiny first capacity, the two-pass ordered feed,
    the fused one-kernel narrow phase and the two-pass (features, then tests)
    narrow phase re-run after overflowing its feature buffer all give the
    default run's hits bit for bit (each in its own process: the switches
    are read once)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for tag, e in (("default", {}), ("variant", env)):
        out = str(tmp_path / f"{tag}.npy")
        r = subprocess.run([sys.executable, "-c", APPEND_SCRIPT, root, out], env={**os.environ, **e},
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[tag] = np.load(out)
    assert len(res["default"]) > 1000
    assert np.array_equal(res["default"].view(np.int64), res["variant"].view(np.int64))
