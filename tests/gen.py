"""Deterministic numpy generators for parity inputs (TEST INFRASTRUCTURE)."""
from __future__ import annotations

import numpy as np

from oracle_bindings import System


def random_block_csr(rng: np.random.Generator, rows: int, extra: int, diag=True, empty_rows=0.0) -> System:
    """Random 3x3-block matrix in the spirit of oracle::random_bell
    (src/oracle/sparse_oracle.cpp:7-23): diagonal + `extra` random columns
    per row, duplicates dropped, U(-1,1) values; optional empty rows."""
    row_ptr = [0]
    cols = []
    for r in range(rows):
        if empty_rows and rng.random() < empty_rows:
            row_ptr.append(len(cols))
            continue
        cs = set([r] if diag else [])
        for _ in range(extra):
            cs.add(int(rng.integers(0, rows)))
        cols.extend(sorted(cs))
        row_ptr.append(len(cols))
    nnzb = len(cols)
    return System(rows, np.array(row_ptr, np.int64), np.array(cols, np.int32), rng.uniform(-1, 1, (nnzb, 9)))


def banded_block_csr(rng: np.random.Generator, rows: int, offsets=(-2, -1, 0, 1, 2)) -> System:
    row_ptr = [0]
    cols = []
    for r in range(rows):
        cs = sorted({r + o for o in offsets if 0 <= r + o < rows})
        cols.extend(cs)
        row_ptr.append(len(cols))
    return System(rows, np.array(row_ptr, np.int64), np.array(cols, np.int32), rng.uniform(-1, 1, (len(cols), 9)))


def to_dense(s: System) -> np.ndarray:
    d = np.zeros((3 * s.rows, 3 * s.rows))
    for r in range(s.rows):
        for k in range(s.row_ptr[r], s.row_ptr[r + 1]):
            c = s.cols[k]
            d[3 * r:3 * r + 3, 3 * c:3 * c + 3] += s.vals[k].reshape(3, 3)
    return d


def from_dense(a: np.ndarray) -> System:
    rows = a.shape[0] // 3
    row_ptr = [0]
    cols = []
    vals = []
    for i in range(rows):
        for j in range(rows):
            blk = a[3 * i:3 * i + 3, 3 * j:3 * j + 3]
            if np.abs(blk).max() == 0.0:
                continue
            cols.append(j)
            vals.append(blk.reshape(9))
        row_ptr.append(len(cols))
    return System(rows, np.array(row_ptr, np.int64), np.array(cols, np.int32), np.array(vals).reshape(-1, 9))


def random_spd(rng: np.random.Generator, rows: int) -> System:
    """A = B^T B + 0.5 I from a sparse random B (test_solver.cpp:35-54)."""
    b = to_dense(random_block_csr(rng, rows, 2))
    return from_dense(b.T @ b + 0.5 * np.eye(3 * rows))
