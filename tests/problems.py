"""Seeded test problems shared by the CPU and GPU parity tests (TEST
INFRASTRUCTURE). Mirrors the reference's fixture recipes:
random_problem (proj/tests/test_assembly.cpp:55-71), random_contact
(proj/tests/test_physics.cpp:62-83), random_spd (test_solver.cpp:35-54)."""
from __future__ import annotations

import numpy as np

from oracle_bindings import CONTACT, ELEMENT_DTYPE, EXTERNAL


def contact_elements(rng: np.random.Generator, p: int, count: int, pinned=None, friction=True) -> np.ndarray:
    """Random contact elements (ContactData, elements.hpp:51-62) over p
    vertices, weights summing to zero as for a vertex-face proximity."""
    out = np.zeros(count, ELEMENT_DTYPE)
    for k in range(count):
        ss = int(rng.integers(1, 5))
        stencil = rng.choice(p, size=ss, replace=False)
        n = rng.uniform(-1, 1, 3)
        n /= np.linalg.norm(n)
        w = np.zeros(4)
        w[0] = 1.0
        if ss > 1:
            r = rng.uniform(0.1, 1.0, ss - 1)
            w[1:ss] = -r / r.sum()
        e = out[k]
        e["kind"] = CONTACT
        e["stencil_size"] = ss
        e["stencil"][:] = -1
        e["stencil"][:ss] = stencil
        e["damping"] = 0.0 if k % 3 else 0.001
        d = e["data"]
        d[0:3] = n
        d[3:7] = w
        d[7] = rng.uniform(-0.01, 0.01)  # bias
        d[8] = 0.01  # activation
        d[9] = rng.uniform(100.0, 1000.0)
        d[10] = 0.3
        d[11] = rng.uniform(0.0, 2.0) if (friction and k % 2 == 0) else 0.0
        d[12] = 1.0
        d[13:16] = rng.uniform(-0.1, 0.1, 3)
    return out


def with_drag(elems: np.ndarray, rng: np.random.Generator, frac=0.5) -> np.ndarray:
    """Gives a fraction of External elements a positive drag (ExternalData)."""
    elems = elems.copy()
    ext = np.nonzero(elems["kind"] == EXTERNAL)[0]
    pick = ext[rng.random(len(ext)) < frac]
    elems["data"][pick, 3] = rng.uniform(0.01, 0.5, len(pick))
    return elems


def cloth_problem(ref, seed: int, max_side: int = 6, contacts: int = 0, damping=0.001, drag=False):
    """random_problem of test_assembly.cpp:55-71 built through the compiled
    reference (mesh, rest data, build_elements), numpy-seeded perturbations."""
    rng = np.random.default_rng(seed)
    mesh = ref.random_cloth(seed, max_side)
    p = len(mesh["vertex_mass"])
    x = mesh["rest"] + rng.uniform(-0.02, 0.02, 3 * p)
    v = rng.uniform(-0.5, 0.5, 3 * p)
    dt = float(rng.uniform(0.005, 0.02))
    x_adv = x + dt * v
    pinned = np.zeros(p, np.uint8)
    if p > 4:
        pinned[int(rng.integers(0, p))] = 1
    elems = ref.build_elements(mesh, material=(400.0, 400.0, 60.0, 2e-5, 0.15, damping, 0.0))
    if drag:
        elems = with_drag(elems, rng)
    if contacts:
        elems = np.concatenate([elems, contact_elements(rng, p, contacts)])
    mass = mesh["vertex_mass"].copy()
    ref.free_mesh(mesh)
    return dict(elems=elems, x=x, x_adv=x_adv, v=v, mass=mass, pinned=pinned, dt=dt, p=p)


def hinge_atan2_split_vertices(elems: np.ndarray, positions) -> set:
    """Vertices of the bend elements whose hinge angle is a case where glibc's
    atan2 (the reference, proj/src/elements.cpp:116) and the library's
    correctly rounded atan2 disagree, at any of the given position arrays.

    (s, c) are formed exactly as dihedral_angle does it (elements.cpp:105-117,
    same operation order; numpy float64 elementwise ops round like the
    library's -fmad=false build), then both atan2s are evaluated: glibc via
    math.atan2, the library's via its host build."""
    import ctypes
    import math
    import os
    lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "paper_2008_00409_b200", "libweft_gpu.so"))
    bends = elems[elems["kind"] == 1]
    st = bends["stencil"]
    out = set()
    for pos in positions:
        x = np.asarray(pos, dtype=np.float64).reshape(-1, 3)
        x0, x1, x2, x3 = (x[st[:, i]] for i in range(4))
        cross = lambda a, b: np.stack([a[:, 1] * b[:, 2] - a[:, 2] * b[:, 1], a[:, 2] * b[:, 0] - a[:, 0] * b[:, 2],
                                       a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]], 1)
        dot = lambda a, b: a[:, 0] * b[:, 0] + a[:, 1] * b[:, 1] + a[:, 2] * b[:, 2]
        e = x1 - x0
        na = cross(e, x2 - x0)
        nb = cross(x3 - x0, e)
        s = np.ascontiguousarray(dot(cross(na, nb), e) / np.sqrt(dot(e, e)))
        c = np.ascontiguousarray(dot(na, nb))
        mine = np.empty_like(s)
        assert lib.weft_hinge_atan2_host(ctypes.c_int64(len(s)), ctypes.c_void_p(s.ctypes.data),
                                         ctypes.c_void_p(c.ctypes.data), ctypes.c_void_p(mine.ctypes.data)) == 0
        glibc = np.array([math.atan2(a, b) for a, b in zip(s.tolist(), c.tolist())])
        for k in np.nonzero(mine != glibc)[0]:
            out.update(int(v) for v in st[k])
    return out
