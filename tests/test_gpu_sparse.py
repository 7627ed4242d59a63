"""GPU SpMV / PCG parity against the CPU oracle (bitwise for SpMV)."""
import numpy as np
import pytest

from gen import banded_block_csr, random_block_csr, random_spd, to_dense
from oracle_bindings import ORACLE, System

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def weft():
    from paper_2008_00409_b200 import weft as w
    return w


def csr(w, s: System):
    return w.BlockCsr(s.rows, s.row_ptr, s.cols, s.vals)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("seed", range(5))
def test_spmv_bitwise_vs_oracle(weft, n, seed):
    rng = np.random.default_rng(1000 + seed)
    rows = int(rng.integers(n, 300))
    s = random_block_csr(rng, rows, 3, empty_rows=0.05 * (seed % 2))
    x = rng.uniform(-2, 2, 3 * rows)
    with weft.Engine(n) as eng:
        y = eng.spmv_pipelined(csr(weft, s), x)
    assert np.array_equal(y, ORACLE.spmv(s, x, n))


@pytest.mark.parametrize("n", [1, 4])
def test_spmv_large_banded(weft, n):
    rng = np.random.default_rng(7)
    s = banded_block_csr(rng, 50_000, offsets=(-301, -300, -1, 0, 1, 300, 301))
    x = rng.uniform(-1, 1, 3 * s.rows)
    with weft.Engine(n) as eng:
        y = eng.spmv_pipelined(csr(weft, s), x)
    assert np.array_equal(y, ORACLE.spmv(s, x, n))


def test_spmv_identity_and_zero(weft):
    rng = np.random.default_rng(3)
    rows = 10
    ident = System(rows, np.arange(rows + 1, dtype=np.int64), np.arange(rows, dtype=np.int32),
                   np.tile(np.eye(3).reshape(9), (rows, 1)))
    x = rng.uniform(-2, 2, 3 * rows)
    for n in (1, 2, 4):
        with weft.Engine(n) as eng:
            assert np.array_equal(eng.spmv_pipelined(csr(weft, ident), x), x)
    zero = System(4, np.zeros(5, np.int64), np.zeros(0, np.int32), np.zeros((0, 9)))
    with weft.Engine(1) as eng:
        assert np.all(eng.spmv_pipelined(csr(weft, zero), np.full(12, 3.0)) == 0.0)
        with pytest.raises(weft.DimensionError):
            eng.spmv_pipelined(None, np.zeros(11))


def test_matrix_roundtrip(weft):
    rng = np.random.default_rng(5)
    s = random_block_csr(rng, 77, 4)
    with weft.Engine(2) as eng:
        eng.set_matrix(csr(weft, s))
        back = eng.download_matrix()
    assert np.array_equal(back.row_ptr, s.row_ptr)
    assert np.array_equal(back.cols, s.cols)
    assert np.array_equal(back.vals, s.vals)


def test_pcg_identity_one_iteration(weft):
    ident = System(3, np.arange(4, dtype=np.int64), np.arange(3, dtype=np.int32), np.tile(np.eye(3).reshape(9), (3, 1)))
    b = np.arange(1, 10, dtype=np.float64)
    with weft.Engine(1) as eng:
        x, rep = eng.pcg_solve(csr(weft, ident), b)
    assert rep.converged and rep.iterations == 1
    assert np.array_equal(x, b)


def test_pcg_hand_solved_2x2(weft):
    s = System(1, np.array([0, 1], np.int64), np.array([0], np.int32), np.array([[4, 1, 0, 1, 3, 0, 0, 0, 1.0]]))
    with weft.Engine(1) as eng:
        x, rep = eng.pcg_solve(csr(weft, s), np.array([1.0, 2.0, 0.0]), weft.PcgConfig(1e-12))
    assert rep.converged
    assert x[0] == pytest.approx(1 / 11, rel=1e-10)
    assert x[1] == pytest.approx(7 / 11, rel=1e-10)
    assert x[2] == 0.0


def test_pcg_zero_rhs_and_non_spd(weft):
    ident = System(4, np.arange(5, dtype=np.int64), np.arange(4, dtype=np.int32), np.tile(np.eye(3).reshape(9), (4, 1)))
    with weft.Engine(1) as eng:
        x, rep = eng.pcg_solve(csr(weft, ident), np.zeros(12))
        assert rep.converged and rep.iterations == 0 and np.all(x == 0)
    neg = System(1, np.array([0, 1], np.int64), np.array([0], np.int32), np.array([-np.eye(3).reshape(9)]))
    with weft.Engine(1) as eng:
        with pytest.raises(weft.SolverError, match="non-positive curvature at iteration 1 \\(matrix not SPD\\)"):
            eng.pcg_solve(csr(weft, neg), np.ones(3), weft.PcgConfig(preconditioner=weft.PRECOND_NONE))


@pytest.mark.parametrize("n", [1, 2, 4])
@pytest.mark.parametrize("seed", range(4))
def test_pcg_random_spd_vs_oracle_and_direct(weft, n, seed):
    rng = np.random.default_rng(2000 + seed)
    rows = int(rng.integers(max(n, 2), 30))
    s = random_spd(rng, rows)
    b = rng.uniform(-1, 1, 3 * rows)
    x_direct = np.linalg.solve(to_dense(s), b)
    with weft.Engine(n) as eng:
        x, rep = eng.pcg_solve(csr(weft, s), b, weft.PcgConfig(1e-10))
    xo, ro = ORACLE.pcg(s, b, n, tol=1e-10)
    assert rep.converged
    scale = max(1e-12, np.abs(x_direct).max())
    assert np.abs(x - x_direct).max() <= 1e-6 * scale
    assert np.abs(x - xo).max() <= 1e-8 * scale
    assert abs(rep.iterations - ro["iterations"]) <= 1
    # preconditioned residual norm is monotone (test_solver.cpp:178-197)
    ph = rep.precond_norm_history
    assert np.all(ph[1:] <= ph[:-1] * (1 + 1e-12)) or n > 1


def test_pcg_bitwise_deterministic(weft):
    rng = np.random.default_rng(33)
    s = random_spd(rng, 17)
    b = rng.uniform(-1, 1, 51)
    with weft.Engine(4) as eng:
        x1, _ = eng.pcg_solve(csr(weft, s), b)
        x2, _ = eng.pcg_solve(None, b)
    assert np.array_equal(x1, x2)


_SOLVE_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from gen import random_spd
from paper_2008_00409_b200 import weft
rng = np.random.default_rng(31)
s = random_spd(rng, 300)
b = rng.uniform(-1, 1, 3 * s.rows)
out = {}
for n in (2, 4, 8):
    with weft.Engine(n) as eng:
        x, rep = eng.pcg_solve(weft.BlockCsr(s.rows, s.row_ptr, s.cols, s.vals), b, weft.PcgConfig(1e-10, 2000))
    out[f"x{n}"], out[f"it{n}"], out[f"h{n}"] = x, np.array(rep.iterations), rep.residual_history
np.savez(sys.argv[2], **out)
"""


def test_pcg_persistent_rows_equals_graph(weft, tmp_path):
    """The multi-partition solve as one cooperative kernel per rank
    (k_pcg_persistent_rows) walks the graph path's virtual blocks: iterates,
    residual histories and solutions are bitwise the two-kernel graph's
    (WEFT_PCG_ROWS=0)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for flag in ("0", "1"):
        out = tmp_path / f"rows{flag}.npz"
        subprocess.run([sys.executable, "-c", _SOLVE_SCRIPT, root, str(out)], check=True,
                       env=dict(os.environ, WEFT_PCG_ROWS=flag), timeout=300)
        res[flag] = dict(np.load(out))
    for k in res["0"]:
        assert np.array_equal(res["0"][k], res["1"][k]), k
