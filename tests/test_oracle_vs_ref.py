"""Pins the C restatement (oracle/liboracle.so) bit-for-bit against the
compiled reference (oracle/_ref/libweft_ref.so). CPU only."""
import numpy as np
import pytest

from oracle_bindings import CONTINUOUS, DISCRETE, JAC_EXACT, JAC_SPD, ORACLE, REF
from problems import cloth_problem

pytestmark = pytest.mark.ref


def same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("mode", [JAC_SPD, JAC_EXACT])
def test_fill_matrix_bitwise(seed, mode):
    pr = cloth_problem(REF, 100 + seed, 6, contacts=6 if seed % 2 else 0, drag=seed % 3 == 0)
    args = (pr["elems"], pr["x"], pr["x_adv"], pr["v"], pr["mass"], pr["pinned"], pr["dt"], mode)
    o = ORACLE.fill_matrix(*args)
    for n in (1, 2, 4):
        r = REF.fill_matrix(*args, n=n)
        assert same(o.row_ptr, r.row_ptr) and same(o.cols, r.cols)
        assert same(o.vals, r.vals), np.abs(o.vals - r.vals).max()
        assert same(o.rhs, r.rhs), np.abs(o.rhs - r.rhs).max()


@pytest.mark.parametrize("seed", range(6))
def test_spmv_bitwise(seed):
    s = REF.random_bell(200 + seed, 5 + 7 * seed, 3)
    x = np.random.default_rng(seed).uniform(-2, 2, 3 * s.rows)
    for n in (1, 2, 4):
        if s.rows < n:
            continue
        assert same(ORACLE.spmv(s, x, n), REF.spmv(s, x, n))


@pytest.mark.parametrize("n", [1, 2, 4])
def test_pcg_bitwise_on_cloth(n):
    pr = cloth_problem(REF, 300 + n, 7, contacts=4)
    s = ORACLE.fill_matrix(pr["elems"], pr["x"], pr["x_adv"], pr["v"], pr["mass"], pr["pinned"], pr["dt"])
    xo, ro = ORACLE.pcg(s, s.rhs, n, tol=1e-10)
    xr, rr = REF.pcg(s, s.rhs, n, tol=1e-10)
    assert ro["iterations"] == rr["iterations"] and ro["converged"] and rr["converged"]
    assert same(xo, xr)
    assert same(ro["residual_history"], rr["residual_history"])


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("mode", [DISCRETE, CONTINUOUS])
def test_broad_phase_bitwise(seed, mode):
    nv, tris, x0, x1 = REF.two_cloth_scene(400 + seed, 8)
    g_r = REF.build_grid(nv, tris, x0, x1, mode=mode, thickness=0.01)
    g_o = ORACLE.build_grid(tris, x0, x1, mode=mode, thickness=0.01)
    assert g_o.cell_size == g_r.cell_size
    for k in ("tri_boxes", "cell_keys", "cell_offsets", "cell_tris", "prefix"):
        assert same(getattr(g_o, k), getattr(g_r, k)), k
    for dev in (1, 2, 4):
        b, e = REF.split(g_r, dev)
        for lo, hi in zip(b, e):
            assert same(ORACLE.candidates(lo, hi), REF.candidates(g_r, lo, hi))
    # candidate set == {t1 < t2 : lattice boxes overlap}
    bx = g_o.tri_boxes
    ov = np.all(np.maximum(bx[:, None, :3], bx[None, :, :3]) <= np.minimum(bx[:, None, 3:], bx[None, :, 3:]), axis=2)
    i, j = np.nonzero(np.triu(ov, 1))
    brute = set(zip(i.tolist(), j.tolist()))
    got = set(map(tuple, ORACLE.candidates().tolist()))
    assert got == brute and len(ORACLE.candidates()) == len(brute)
    ORACLE.free_grid()
    REF.free_grid(g_r)
