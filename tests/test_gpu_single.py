"""Precision::Single (driver.hpp:13, Real = float) on the GPU vs the
compiled reference's float instantiations: spmv_pipelined<float> bitwise
(the same float products and sums in the same order), the FP32 known answer
of test_sparsemat.cpp:172-219 (float SpMV within 2 ulp of the double one),
pcg_solve<float> (float vectors, double dots) by iterations and solution."""
import numpy as np
import pytest

from gen import random_block_csr, random_spd
from oracle_bindings import REF, System

pytestmark = [pytest.mark.gpu, pytest.mark.ref]


@pytest.fixture(scope="module")
def weft():
    from paper_2008_00409_b200 import weft as w
    return w


def f32(s: System) -> System:
    return System(s.rows, s.row_ptr, s.cols, np.asarray(s.vals, np.float32))


def csr(w, s: System):
    return w.BlockCsr(s.rows, s.row_ptr, s.cols, s.vals)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("seed", range(3))
def test_spmv_f32_bitwise_vs_reference(weft, n, seed):
    rng = np.random.default_rng(500 + seed)
    rows = int(rng.integers(n, 300))
    s = f32(random_block_csr(rng, rows, 3, empty_rows=0.05 * (seed % 2)))
    x = rng.uniform(-2, 2, 3 * rows).astype(np.float32)
    with weft.Engine(n) as eng:
        y = eng.spmv_pipelined(csr(weft, s), x)
        assert y.dtype == np.float32
        m = eng.download_matrix()
        assert m.vals.dtype == np.float32
    assert np.array_equal(y, REF.spmv_f32(s, x, n))


def test_spmv_f32_known_answer_random_bell(weft):
    """test_sparsemat.cpp:172-219: oracle::random_bell(Rng(8), 9, 2) rebuilt in
    float, x ~ U(-1, 1) as float, Engine(2): the reference's float pipelined
    SpMV is within 2 ulp of its serial float oracle; the GPU's equals the
    reference's bitwise."""
    s64 = REF.random_bell(8, 9, 2)
    s = f32(s64)
    x = np.random.default_rng(8).uniform(-1, 1, 27).astype(np.float32)
    with weft.Engine(2) as eng:
        y = eng.spmv_pipelined(csr(weft, s), x)
    yr = REF.spmv_f32(s, x, 2)
    assert np.array_equal(y, yr)
    yd = REF.spmv(System(s.rows, s.row_ptr, s.cols, np.asarray(s.vals, np.float64)), x.astype(np.float64), 2)
    assert np.all(np.abs(y.astype(np.float64) - yd) <= 1e-5 * (1.0 + np.abs(yd)))


@pytest.mark.parametrize("n", [1, 2, 4])
@pytest.mark.parametrize("seed", range(3))
def test_pcg_f32_vs_reference(weft, n, seed):
    rng = np.random.default_rng(800 + seed)
    s = f32(random_spd(rng, int(rng.integers(20, 60))))
    b = rng.uniform(-1, 1, 3 * s.rows).astype(np.float32)
    with weft.Engine(n) as eng:
        x, rep = eng.pcg_solve(csr(weft, s), b, weft.PcgConfig(1e-5, 2000))
    xr, rr = REF.pcg_f32(s, b, n, tol=1e-5, max_it=2000)
    assert x.dtype == np.float32 and rep.converged and rr["converged"]
    assert abs(rep.iterations - rr["iterations"]) <= max(1, 0.05 * rr["iterations"])
    assert np.abs(x - xr).max() <= 1e-4 * np.abs(xr).max()


def test_pcg_f32_zero_rhs_and_non_spd(weft):
    rng = np.random.default_rng(3)
    s = f32(random_spd(rng, 10))
    with weft.Engine(1) as eng:
        x, rep = eng.pcg_solve(csr(weft, s), np.zeros(30, np.float32), weft.PcgConfig(1e-6, 100))
        assert rep.converged and rep.iterations == 0 and not x.any()
        neg = System(s.rows, s.row_ptr, s.cols, -np.asarray(s.vals, np.float32))
        with pytest.raises(weft.SolverError, match="non-positive curvature at iteration 1"):
            eng.pcg_solve(csr(weft, neg), np.ones(30, np.float32), weft.PcgConfig(1e-6, 100))


@pytest.mark.parametrize("contacts", [0, 50])
@pytest.mark.parametrize("mode", ["spd", "exact"])
def test_fill_matrix_f32_vs_reference(weft, contacts, mode):
    """fill_matrix<float>: each contribution computed in double, cast to
    float, added in float (assembly.hpp:163,196,212) — pattern and
    SpdProjected values bitwise the reference's float instantiation; the
    Exact bend Hessian and the rhs go through atan2 (CUDA vs glibc) and may
    differ in the last float bit."""
    from oracle_bindings import JAC_EXACT, JAC_SPD
    from test_gpu_assembly import layered_problem
    jm = JAC_SPD if mode == "spd" else JAC_EXACT
    pr = layered_problem(weft, contacts=contacts)
    full = pr["elems"] if pr["contacts"] is None else np.concatenate([pr["elems"], pr["contacts"]])
    for n in (1, 2):
        ref = REF.fill_matrix(full, pr["x"], pr["xa"], pr["v"], pr["mass"], pr["pinned"], pr["dt"], jm, n=n,
                              single=True)
        with weft.Engine(n) as eng:
            eng.set_vertices(pr["mass"], pr["pinned"])
            eng.set_elements(pr["elems"])
            if pr["contacts"] is not None:
                eng.set_contacts(pr["contacts"])
            eng.fill_matrix(pr["x"], pr["xa"], pr["v"], pr["dt"], jm, single=True)
            m = eng.download_matrix()
            rhs = eng.download_rhs()
        assert m.vals.dtype == np.float32 and rhs.dtype == np.float32
        assert np.array_equal(m.row_ptr, ref.row_ptr) and np.array_equal(m.cols, ref.cols)
        rv = ref.vals.astype(np.float32)
        if jm == JAC_SPD:
            assert np.array_equal(m.vals.reshape(rv.shape), rv)
        else:
            assert np.abs(m.vals.reshape(rv.shape) - rv).max() <= 4e-7 * np.abs(rv).max()
        rr = ref.rhs.astype(np.float32)
        assert np.abs(rhs - rr).max() <= 4e-7 * max(np.abs(rr).max(), 1e-30)


def test_step_f32_vs_reference_simulator(weft):
    """Precision::Single through the whole device step (step_impl<float>,
    driver.cpp:92-94): a scene with precision "single" on the GPU Simulator
    vs the reference Simulator, frame by frame."""
    import json
    from oracle_bindings import RefScene
    from paper_2008_00409_b200 import scene as S
    from scenes_gen import SCENES
    spec = dict(SCENES["drape_sphere"])
    spec["precision"] = "single"
    spec["frames"] = 12
    text = json.dumps(spec)
    sc = S.parse_scene(text)
    assert sc.config.precision == "single"
    sim = S.Simulator(sc)
    rs = RefScene(REF, text=text)
    for k in range(sc.config.frames):
        rr = rs.step()
        r = sim.step()
        assert (r.proximities, r.contacts, r.impacts, r.zone_count) == (
            rr["proximities"], rr["contacts"], rr["impacts"], rr["zone_count"]), k
        assert abs(r.pcg_iterations - rr["pcg_iterations"]) <= max(2, 0.05 * rr["pcg_iterations"]), k
    x, v = sim.state()
    xr, vr = rs.state()
    scale = np.abs(xr).max()
    assert np.abs(x.reshape(-1) - xr).max() <= 1e-5 * scale
    assert np.abs(v.reshape(-1) - vr).max() <= 1e-3 * max(np.abs(vr).max(), 1e-12)
    rs.close()
    sim.close()
