"""GPU broad phase: grid + candidate pairs bit-exact vs the reference
(golden fixtures) and the C oracle."""
import glob
import os

import numpy as np
import pytest

from oracle_bindings import CONTINUOUS, DISCRETE, ORACLE

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def weft():
    from paper_2008_00409_b200 import weft as w
    return w


def check_grid(g, ref, pairs_ref, eng, devices=(1, 2, 4)):
    assert g.cell_size == ref.cell_size
    for f in ("tri_boxes", "cell_keys", "cell_offsets", "cell_tris", "prefix"):
        assert np.array_equal(getattr(g, f), getattr(ref, f)), f
    pairs = eng.candidates()
    assert np.array_equal(pairs, pairs_ref)
    from paper_2008_00409_b200 import weft as w
    for n in devices:
        parts = [eng.candidates(b, e) for b, e in w.split_workload(g.total, n)]
        assert np.array_equal(np.concatenate(parts), pairs_ref)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "grid_*.npz"))))
@pytest.mark.parametrize("mode,tag", [(DISCRETE, "dcd"), (CONTINUOUS, "ccd")])
def test_grid_vs_reference_golden(weft, path, mode, tag):
    gd = dict(np.load(path))
    with weft.Engine(1) as eng:
        eng.set_soup(int(gd["nv"]), gd["tris"])
        eng.build_grid(gd["x0"], gd["x1"], mode=mode, thickness=0.01)
        g = eng.download_grid(len(gd["tris"]))
        ref = weft.HashGrid(float(gd[f"{tag}_cell_size"]), gd[f"{tag}_cell_keys"], gd[f"{tag}_cell_offsets"],
                            gd[f"{tag}_cell_tris"], gd[f"{tag}_prefix"], gd[f"{tag}_tri_boxes"])
        check_grid(g, ref, gd[f"{tag}_pairs"], eng)


@pytest.mark.parametrize("mode", [DISCRETE, CONTINUOUS])
@pytest.mark.parametrize("layers,nx", [(1, 60), (3, 45)])
def test_grid_vs_oracle_layered(weft, mode, layers, nx):
    from paper_2008_00409_b200 import scenes
    sc = scenes.layered_cloth(layers, nx, seed=11)
    rng = np.random.default_rng(2)
    x0 = sc.verts.reshape(-1)
    x1 = x0 + rng.uniform(-0.002, 0.002, x0.shape) + np.tile([0.0, 0.0, -0.003], sc.vertex_count)
    og = ORACLE.build_grid(sc.tris, x0, x1, mode=mode, thickness=sc.thickness)
    pairs = ORACLE.candidates()
    with weft.Engine(1) as eng:
        eng.set_soup(sc.vertex_count, sc.tris)
        eng.build_grid(x0, x1, mode=mode, thickness=sc.thickness)
        g = eng.download_grid(sc.tri_count)
        check_grid(g, og, pairs, eng)
    ORACLE.free_grid()


def test_hot_cell_and_single_triangle(weft):
    # test_collision.cpp:104-109 and :158-198
    rng = np.random.default_rng(42)
    x = []
    for _ in range(10):
        j = rng.uniform(-1e-4, 1e-4, 3)
        x += [np.array([0.04, 0.04, 0.04]) + j, np.array([0.09, 0.04, 0.04]) + j, np.array([0.04, 0.09, 0.04]) + j]
    x = np.concatenate(x)
    tris = np.arange(30, dtype=np.int32).reshape(10, 3)
    with weft.Engine(1) as eng:
        eng.set_soup(30, tris)
        eng.build_grid(x)
        info = eng.grid_info()
        assert info.cells == 1 and info.total == 45
        ranges = weft.split_workload(info.total, 4)
        assert max(e - b for b, e in ranges) - min(e - b for b, e in ranges) <= 1
        assert sum(len(eng.candidates(b, e)) for b, e in ranges) == 45
        eng.set_soup(3, np.array([[0, 1, 2]], np.int32))
        eng.build_grid(np.array([0, 0, 0, 0.1, 0, 0, 0, 0.1, 0.0]))
        assert eng.grid_info().total == 0 and len(eng.candidates()) == 0


def _serial(d):
    s = 0.0
    for v in d.tolist():
        s += v
    return s


@pytest.mark.parametrize("case", ["uniform", "equal_third", "equal_binary", "few_bits", "logwide", "zeros", "tiny",
                                  "nan", "sizes"])
def test_exact_serial_sum(weft, case):
    import ctypes as C
    rng = np.random.default_rng(7)
    n = 1_650_000
    if case == "uniform":
        ds = [rng.uniform(0, 0.02, n)]
    elif case == "equal_third":
        ds = [np.full(n, 1.0 / 3.0)]
    elif case == "equal_binary":
        ds = [np.full(n, 0.0125), np.full(300_000, 0.5)]
    elif case == "few_bits":
        ds = [rng.integers(0, 64, n) * 2.0 ** -10, rng.integers(0, 3, 200_000) * 0.75]
    elif case == "logwide":
        ds = [10.0 ** rng.uniform(-10, 10, 200_000)]
    elif case == "zeros":
        d = rng.uniform(0, 1, 100_000)
        d[:5000] = 0.0
        d[50_000:60_000] = 0.0
        ds = [d]
    elif case == "tiny":
        ds = [rng.uniform(0, 1e-305, 50_000), np.concatenate([np.full(100, 5e-324), rng.uniform(0, 1, 1000)])]
    elif case == "nan":
        d = rng.uniform(0, 1, 40_000)
        d[20_000] = np.nan
        e = rng.uniform(0, 1, 40_000)
        e[30_000] = np.inf
        ds = [d, e]
    else:
        ds = [rng.uniform(0, 1, m) for m in (0, 1, 2, 31, 33, 16383, 16384, 16385, 50_000)]
    with weft.Engine(1) as eng:
        for d in ds:
            d = np.ascontiguousarray(d, np.float64)
            s = _serial(d)
            mean = s / len(d) if len(d) else 1.0
            want = 1e-9 if mean < 1e-9 else mean
            for fast in (0, 1):
                me, sn = C.c_double(), C.c_double()
                assert weft.LIB.weft_gpu_test_serial_sum(eng._ctx, C.c_int32(len(d)), d.ctypes.data_as(C.c_void_p),
                                                          C.c_int32(fast), C.byref(me), C.byref(sn)) == 0
                assert (sn.value == s) or (np.isnan(sn.value) and np.isnan(s))
                assert (me.value == want) or (np.isnan(me.value) and np.isnan(want)), (fast, len(d), me.value, want)
