"""ctypes bindings to the CPU oracle (TEST INFRASTRUCTURE).

Two libraries, both built by `make -C oracle` (and by __graft_entry__.build()):

* ``oracle/liboracle.so`` — the C restatement of the reference hot path
  (oracle/weft_oracle.c). Always buildable from repo sources.
* ``oracle/_ref/libweft_ref.so`` — the unmodified reference engine compiled
  against oracle/shim (only where /root/reference exists; the built file
  travels with the gpurun snapshot). ``REF`` is None when it is absent.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libweft_ref.so")

STRETCH, BEND, SPRING, EXTERNAL, CONTACT = range(5)
JAC_EXACT, JAC_SPD = 0, 1
DISCRETE, CONTINUOUS = 0, 1
PRECOND_NONE, PRECOND_BJ = 0, 1

ELEMENT_DTYPE = np.dtype(
    [("kind", "<i4"), ("stencil_size", "<i4"), ("stencil", "<i4", (4,)), ("damping", "<f8"), ("data", "<f8", (18,))],
    align=True,
)
assert ELEMENT_DTYPE.itemsize == 176


class PcgConfig(C.Structure):
    _fields_ = [("rel_tolerance", C.c_double), ("max_iterations", C.c_int32), ("preconditioner", C.c_int32)]


class PcgReport(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("rel_residual", C.c_double),
        ("residual_history", C.POINTER(C.c_double)),
        ("precond_norm_history", C.POINTER(C.c_double)),
    ]


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class System:
    """Global block-CSR system (ascending columns), values row-major 3x3."""

    rows: int
    row_ptr: np.ndarray
    cols: np.ndarray
    vals: np.ndarray  # (nnzb, 9)
    rhs: np.ndarray | None = None


@dataclass
class Grid:
    cell_size: float
    tri_boxes: np.ndarray  # (T, 6) int64
    cell_keys: np.ndarray  # uint64
    cell_offsets: np.ndarray  # int64, cells+1
    cell_tris: np.ndarray  # int32
    prefix: np.ndarray  # int64, cells+1

    @property
    def total(self) -> int:
        return int(self.prefix[-1])


# --------------------------------------------------------------------------
# C restatement
# --------------------------------------------------------------------------
class _OrcSystem(C.Structure):
    _fields_ = [
        ("rows", C.c_int32),
        ("nnzb", C.c_int64),
        ("row_ptr", C.POINTER(C.c_int64)),
        ("cols", C.POINTER(C.c_int32)),
        ("vals", C.POINTER(C.c_double)),
        ("rhs", C.POINTER(C.c_double)),
    ]


class _OrcGrid(C.Structure):
    _fields_ = [
        ("tri_count", C.c_int32),
        ("cell_size", C.c_double),
        ("tri_boxes", C.POINTER(C.c_int64)),
        ("cells", C.c_int64),
        ("cell_keys", C.POINTER(C.c_uint64)),
        ("cell_offsets", C.POINTER(C.c_int64)),
        ("cell_tris", C.POINTER(C.c_int32)),
        ("prefix", C.POINTER(C.c_int64)),
        ("total", C.c_int64),
    ]


def _arr(p, n, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(p, shape=(n,)).astype(dtype, copy=True)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = L = C.CDLL(path)
        L.orc_fill_matrix.restype = C.c_int32
        L.orc_pcg.restype = C.c_int32
        L.orc_candidates.restype = C.c_int64
        L.orc_owner.restype = C.c_int32
        L.orc_work_queues.restype = C.c_int32
        L.orc_dihedral_angle.restype = C.c_double
        L.orc_rng_uniform.restype = C.c_double
        L.orc_rng_raw.restype = C.c_uint64

    def partitions(self, p: int, n: int):
        b = np.zeros(n, np.int32)
        e = np.zeros(n, np.int32)
        self.lib.orc_make_partitions(C.c_int32(p), C.c_int32(n), ptr(b), ptr(e))
        return b, e

    def work_queues(self, n: int):
        m = max(n - 1, 1)
        peer = np.zeros(n * m, np.int32)
        vec = np.zeros(n * m, np.int32)
        if self.lib.orc_work_queues(C.c_int32(n), ptr(peer), ptr(vec)) != 0:
            raise ValueError("n must be a power of two")
        return peer.reshape(n, m)[:, : n - 1], vec.reshape(n, m)[:, : n - 1]

    def spmv(self, s: System, x: np.ndarray, n: int = 1) -> np.ndarray:
        y = np.zeros(3 * s.rows)
        self.lib.orc_spmv(
            C.c_int32(s.rows), ptr(s.row_ptr), ptr(s.cols), ptr(np.ascontiguousarray(s.vals)), C.c_int32(n),
            ptr(np.ascontiguousarray(x, np.float64)), ptr(y),
        )
        return y

    def pcg(self, s: System, b: np.ndarray, n: int = 1, tol=1e-4, max_it=400, precond=PRECOND_BJ):
        x = np.zeros(3 * s.rows)
        hist = np.zeros(max(max_it, 1))
        phist = np.zeros(max(max_it, 1))
        cfg = PcgConfig(tol, max_it, precond)
        rep = PcgReport(0, 0, 0.0, hist.ctypes.data_as(C.POINTER(C.c_double)), phist.ctypes.data_as(C.POINTER(C.c_double)))
        err = C.create_string_buffer(256)
        st = self.lib.orc_pcg(
            C.c_int32(s.rows), ptr(s.row_ptr), ptr(s.cols), ptr(np.ascontiguousarray(s.vals)), C.c_int32(n),
            ptr(np.ascontiguousarray(b, np.float64)), ptr(x), C.byref(cfg), C.byref(rep), err,
        )
        if st != 0:
            raise RuntimeError(err.value.decode())
        return x, dict(iterations=rep.iterations, converged=bool(rep.converged), rel_residual=rep.rel_residual,
                       residual_history=hist[: rep.iterations].copy(), precond_norm_history=phist[: rep.iterations].copy())

    def fill_matrix(self, elems, x_cur, x_adv, vel, mass, pinned, dt, mode=JAC_SPD) -> System:
        p = len(mass)
        out = _OrcSystem()
        err = C.create_string_buffer(256)
        st = self.lib.orc_fill_matrix(
            C.c_int32(p), C.c_int64(len(elems)), ptr(elems), ptr(x_cur), ptr(x_adv), ptr(vel), ptr(mass),
            ptr(pinned), C.c_double(dt), C.c_int32(mode), C.byref(out), err,
        )
        if st != 0:
            raise ValueError(err.value.decode())
        s = System(
            p, _arr(out.row_ptr, p + 1, np.int64), _arr(out.cols, out.nnzb, np.int32),
            _arr(out.vals, 9 * out.nnzb, np.float64).reshape(-1, 9), _arr(out.rhs, 3 * p, np.float64),
        )
        self.lib.orc_free_system(C.byref(out))
        return s

    def element_eval(self, elem, x, v, mode=JAC_SPD):
        f = np.zeros(12)
        j = np.zeros(144)
        fr = np.zeros(12)
        vd = np.zeros(144)
        e = np.ascontiguousarray(elem, ELEMENT_DTYPE)
        self.lib.orc_element_force(ptr(e), ptr(x), ptr(f))
        self.lib.orc_element_jacobian(ptr(e), ptr(x), C.c_int32(mode), ptr(j))
        self.lib.orc_element_friction(ptr(e), ptr(v), ptr(fr))
        self.lib.orc_element_velocity_damping(ptr(e), ptr(vd))
        return f, j, fr, vd

    def build_grid(self, tris, x0, x1=None, mode=DISCRETE, thickness=0.005, cell_scale=1.5) -> Grid:
        g = _OrcGrid()
        x1 = x0 if x1 is None else x1
        self.lib.orc_build_grid(
            C.c_int32(len(tris)), ptr(np.ascontiguousarray(tris, np.int32)), ptr(np.ascontiguousarray(x0, np.float64)),
            ptr(np.ascontiguousarray(x1, np.float64)), C.c_int32(mode), C.c_double(thickness), C.c_double(cell_scale),
            C.byref(g),
        )
        T, cells = len(tris), g.cells
        entries = int(np.ctypeslib.as_array(g.cell_offsets, shape=(cells + 1,))[-1]) if cells else 0
        out = Grid(
            g.cell_size, _arr(g.tri_boxes, 6 * T, np.int64).reshape(-1, 6), _arr(g.cell_keys, cells, np.uint64),
            _arr(g.cell_offsets, cells + 1, np.int64), _arr(g.cell_tris, entries, np.int32),
            _arr(g.prefix, cells + 1, np.int64),
        )
        self._last_grid = g  # keep for candidates
        self._grid_owner = out
        return out

    def candidates(self, begin=None, end=None) -> np.ndarray:
        g = self._last_grid
        begin = 0 if begin is None else begin
        end = g.total if end is None else end
        n = self.lib.orc_candidates(C.byref(g), C.c_int64(begin), C.c_int64(end), None)
        pairs = np.zeros(2 * max(n, 1), np.int32)
        self.lib.orc_candidates(C.byref(g), C.c_int64(begin), C.c_int64(end), ptr(pairs))
        return pairs[: 2 * n].reshape(-1, 2)

    def free_grid(self):
        if getattr(self, "_last_grid", None) is not None:
            self.lib.orc_free_grid(C.byref(self._last_grid))
            self._last_grid = None


# --------------------------------------------------------------------------
# The compiled reference
# --------------------------------------------------------------------------
class Ref:
    def __init__(self, path: str = REF_SO):
        self.lib = L = C.CDLL(path)
        for name in ("ref_fill_matrix", "ref_random_bell", "ref_grid_mesh", "ref_build_mesh", "ref_random_cloth",
                     "ref_build_grid"):
            getattr(L, name).restype = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_build_elements.restype = C.c_int64
        L.ref_grid_candidates.restype = C.c_int64
        L.ref_collide.restype = C.c_int64
        L.ref_spmv.restype = C.c_int32
        L.ref_pcg.restype = C.c_int32
        L.ref_two_cloth_scene.restype = C.c_int32
        for name in ("ref_system_info", "ref_system_copy", "ref_system_free", "ref_mesh_info", "ref_mesh_copy",
                     "ref_mesh_free", "ref_grid_info", "ref_grid_copy", "ref_grid_free", "ref_grid_split",
                     "ref_build_elements", "ref_grid_candidates"):
            getattr(L, name).argtypes = None
        L.ref_system_free.argtypes = [C.c_void_p]
        L.ref_mesh_free.argtypes = [C.c_void_p]
        L.ref_grid_free.argtypes = [C.c_void_p]

    def _system(self, h) -> System:
        rows = C.c_int32()
        nnzb = C.c_int64()
        self.lib.ref_system_info(C.c_void_p(h), C.byref(rows), C.byref(nnzb))
        r, k = rows.value, nnzb.value
        s = System(r, np.zeros(r + 1, np.int64), np.zeros(max(k, 1), np.int32), np.zeros((max(k, 1), 9)), np.zeros(max(3 * r, 1)))
        self.lib.ref_system_copy(C.c_void_p(h), ptr(s.row_ptr), ptr(s.cols), ptr(s.vals), ptr(s.rhs))
        s.cols, s.vals, s.rhs = s.cols[:k], s.vals[:k], s.rhs[: 3 * r]
        self.lib.ref_system_free(C.c_void_p(h))
        return s

    def fill_matrix(self, elems, x_cur, x_adv, vel, mass, pinned, dt, mode=JAC_SPD, n=1, single=False) -> System:
        """fill_matrix<double>, or fill_matrix<float> with single=True (values
        and rhs returned as the float values, exact in float64)."""
        st = C.c_int32()
        fn = self.lib.ref_fill_matrix_f32 if single else self.lib.ref_fill_matrix
        fn.restype = C.c_void_p
        h = fn(
            C.c_int32(len(mass)), C.c_int32(n), C.c_int64(len(elems)), ptr(elems), ptr(x_cur), ptr(x_adv), ptr(vel),
            ptr(mass), ptr(pinned), C.c_double(dt), C.c_int32(mode), C.byref(st),
        )
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        return self._system(h)

    def random_bell(self, seed: int, rows: int, extra: int) -> System:
        return self._system(self.lib.ref_random_bell(C.c_uint64(seed), C.c_int32(rows), C.c_int32(extra)))

    def spmv(self, s: System, x, n=1):
        y = np.zeros(3 * s.rows)
        st = self.lib.ref_spmv(C.c_int32(s.rows), ptr(s.row_ptr), ptr(s.cols), ptr(np.ascontiguousarray(s.vals)),
                               C.c_int32(n), ptr(np.ascontiguousarray(x, np.float64)), ptr(y))
        if st:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return y

    def spmv_f32(self, s: System, x, n=1):
        """spmv_pipelined<float> (Precision::Single); s.vals as float32."""
        y = np.zeros(3 * s.rows, np.float32)
        st = self.lib.ref_spmv_f32(C.c_int32(s.rows), ptr(s.row_ptr), ptr(s.cols),
                                   ptr(np.ascontiguousarray(s.vals, np.float32)), C.c_int32(n),
                                   ptr(np.ascontiguousarray(x, np.float32)), ptr(y))
        if st:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return y

    def pcg_f32(self, s: System, b, n=1, tol=1e-4, max_it=400, precond=PRECOND_BJ):
        """pcg_solve<float> (Precision::Single)."""
        x = np.zeros(3 * s.rows, np.float32)
        hist = np.zeros(max(max_it, 1))
        phist = np.zeros(max(max_it, 1))
        cfg = PcgConfig(tol, max_it, precond)
        rep = PcgReport(0, 0, 0.0, hist.ctypes.data_as(C.POINTER(C.c_double)), phist.ctypes.data_as(C.POINTER(C.c_double)))
        st = self.lib.ref_pcg_f32(C.c_int32(s.rows), ptr(s.row_ptr), ptr(s.cols),
                                  ptr(np.ascontiguousarray(s.vals, np.float32)), C.c_int32(n),
                                  ptr(np.ascontiguousarray(b, np.float32)), ptr(x), C.byref(cfg), C.byref(rep))
        if st:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return x, dict(iterations=rep.iterations, converged=bool(rep.converged), rel_residual=rep.rel_residual,
                       residual_history=hist[: rep.iterations].copy())

    def pcg(self, s: System, b, n=1, tol=1e-4, max_it=400, precond=PRECOND_BJ):
        x = np.zeros(3 * s.rows)
        hist = np.zeros(max(max_it, 1))
        phist = np.zeros(max(max_it, 1))
        cfg = PcgConfig(tol, max_it, precond)
        rep = PcgReport(0, 0, 0.0, hist.ctypes.data_as(C.POINTER(C.c_double)), phist.ctypes.data_as(C.POINTER(C.c_double)))
        st = self.lib.ref_pcg(C.c_int32(s.rows), ptr(s.row_ptr), ptr(s.cols), ptr(np.ascontiguousarray(s.vals)),
                              C.c_int32(n), ptr(np.ascontiguousarray(b, np.float64)), ptr(x), C.byref(cfg), C.byref(rep))
        if st:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return x, dict(iterations=rep.iterations, converged=bool(rep.converged), rel_residual=rep.rel_residual,
                       residual_history=hist[: rep.iterations].copy(), precond_norm_history=phist[: rep.iterations].copy())

    # meshes -------------------------------------------------------------
    def _mesh(self, h):
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        nv, nt, nh, ne = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        self.lib.ref_mesh_info(C.c_void_p(h), C.byref(nv), C.byref(nt), C.byref(nh), C.byref(ne))
        nv, nt, nh = nv.value, nt.value, nh.value
        m = dict(
            rest=np.zeros(3 * nv), tris=np.zeros(3 * nt, np.int32), tri_rest=np.zeros(7 * nt),
            tri_degenerate=np.zeros(nt, np.uint8), hinge_verts=np.zeros(4 * nh, np.int32),
            hinge_data=np.zeros(2 * nh), vertex_area=np.zeros(nv), vertex_mass=np.zeros(nv),
        )
        self.lib.ref_mesh_copy(C.c_void_p(h), *(ptr(m[k]) for k in (
            "rest", "tris", "tri_rest", "tri_degenerate", "hinge_verts", "hinge_data", "vertex_area", "vertex_mass")))
        m["tris"] = m["tris"].reshape(-1, 3)
        m["tri_rest"] = m["tri_rest"].reshape(-1, 7)
        m["hinge_verts"] = m["hinge_verts"].reshape(-1, 4)
        m["hinge_data"] = m["hinge_data"].reshape(-1, 2)
        m["_handle"] = h
        return m

    def grid_mesh(self, nx, ny, w, h, origin=(0.0, 0.0, 0.0), density=0.15):
        return self._mesh(self.lib.ref_grid_mesh(C.c_int32(nx), C.c_int32(ny), C.c_double(w), C.c_double(h),
                                                 *(C.c_double(o) for o in origin), C.c_double(density)))

    def build_mesh(self, verts, tris, density):
        verts = np.ascontiguousarray(verts, np.float64)
        tris = np.ascontiguousarray(tris, np.int32)
        return self._mesh(self.lib.ref_build_mesh(C.c_int32(len(verts) // 3 if verts.ndim == 1 else len(verts)),
                                                  ptr(verts), C.c_int32(len(tris)), ptr(tris), C.c_double(density)))

    def random_cloth(self, seed, max_side):
        return self._mesh(self.lib.ref_random_cloth(C.c_uint64(seed), C.c_int32(max_side)))

    def build_elements(self, mesh, material=(400.0, 400.0, 60.0, 2e-5, 0.15, 0.002, 0.0), gravity=(0, 0, -9.81),
                       wind=(0, 0, 0)):
        h = C.c_void_p(mesh["_handle"])
        mat = np.array(material, np.float64)
        g = np.array(gravity, np.float64)
        w = np.array(wind, np.float64)
        n = self.lib.ref_build_elements(h, ptr(mat), ptr(g), ptr(w), None, C.c_int64(0))
        out = np.zeros(n, ELEMENT_DTYPE)
        self.lib.ref_build_elements(h, ptr(mat), ptr(g), ptr(w), ptr(out), C.c_int64(n))
        return out

    def free_mesh(self, mesh):
        self.lib.ref_mesh_free(C.c_void_p(mesh.pop("_handle")))

    def element_eval(self, elem, x, v, mode=JAC_SPD):
        f, j, fr, vd = np.zeros(12), np.zeros(144), np.zeros(12), np.zeros(144)
        e = np.ascontiguousarray(elem, ELEMENT_DTYPE)
        self.lib.ref_element_eval(ptr(e), C.c_int32(len(x) // 3), ptr(x), ptr(v), C.c_int32(mode), ptr(f), ptr(j),
                                  ptr(fr), ptr(vd))
        return f, j, fr, vd

    # broad phase ----------------------------------------------------------
    def build_grid(self, vertex_count, tris, x0, x1=None, mode=DISCRETE, thickness=0.005, cell_scale=1.5):
        tris = np.ascontiguousarray(tris, np.int32)
        h = self.lib.ref_build_grid(C.c_int32(vertex_count), C.c_int32(len(tris)), ptr(tris),
                                    ptr(np.ascontiguousarray(x0, np.float64)),
                                    ptr(None if x1 is None else np.ascontiguousarray(x1, np.float64)),
                                    C.c_int32(mode), C.c_double(thickness), C.c_double(cell_scale))
        cs, cells, entries, total = C.c_double(), C.c_int64(), C.c_int64(), C.c_int64()
        self.lib.ref_grid_info(C.c_void_p(h), C.byref(cs), C.byref(cells), C.byref(entries), C.byref(total))
        nc, ne = cells.value, entries.value
        g = Grid(cs.value, np.zeros((len(tris), 6), np.int64), np.zeros(nc, np.uint64), np.zeros(nc + 1, np.int64),
                 np.zeros(max(ne, 1), np.int32), np.zeros(nc + 1, np.int64))
        self.lib.ref_grid_copy(C.c_void_p(h), ptr(g.cell_keys), ptr(g.cell_offsets), ptr(g.cell_tris), ptr(g.prefix),
                               ptr(g.tri_boxes))
        g.cell_tris = g.cell_tris[:ne]
        g._handle = h
        return g

    def candidates(self, g: Grid, begin=None, end=None):
        begin = 0 if begin is None else begin
        end = g.total if end is None else end
        h = C.c_void_p(g._handle)
        n = self.lib.ref_grid_candidates(h, C.c_int64(begin), C.c_int64(end), None)
        pairs = np.zeros(2 * max(n, 1), np.int32)
        self.lib.ref_grid_candidates(h, C.c_int64(begin), C.c_int64(end), ptr(pairs))
        return pairs[: 2 * n].reshape(-1, 2)

    def split(self, g: Grid, devices):
        b = np.zeros(devices, np.int64)
        e = np.zeros(devices, np.int64)
        self.lib.ref_grid_split(C.c_void_p(g._handle), C.c_int32(devices), ptr(b), ptr(e))
        return b, e

    def free_grid(self, g: Grid):
        self.lib.ref_grid_free(C.c_void_p(g._handle))

    def collide(self, vertex_count, tris, x0, x1=None, mode=DISCRETE, thickness=0.005, cell_scale=1.5, devices=2,
                movable=None):
        """collide (collision.cpp:391-417) -> (kab (n, 3) int32: kind, a, b; vals (n, 8): gap|toi,
        normal xyz, weights 0..3), sorted and deduplicated by (kind, a, b)."""
        tris = np.ascontiguousarray(tris, np.int32)
        x0 = np.ascontiguousarray(x0, np.float64)
        x1 = None if x1 is None else np.ascontiguousarray(x1, np.float64)
        mv = None if movable is None else np.ascontiguousarray(movable, np.uint8)
        args = (C.c_int32(vertex_count), C.c_int32(len(tris)), ptr(tris), ptr(mv), ptr(x0), ptr(x1), C.c_int32(mode),
                C.c_double(thickness), C.c_double(cell_scale), C.c_int32(devices))
        n = self.lib.ref_collide(*args, C.c_int64(0), None, None)
        if n < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        kab = np.zeros((max(n, 1), 3), np.int32)
        vals = np.zeros((max(n, 1), 8))
        self.lib.ref_collide(*args, C.c_int64(n), ptr(kab), ptr(vals))
        return kab[:n], vals[:n]

    def build_zones(self, vertex_count, tris, kab, movable=None):
        """build_zones (response.cpp:108-162) -> (impact_zone, per-zone vertex lists)."""
        tris = np.ascontiguousarray(tris, np.int32)
        kab = np.ascontiguousarray(kab, np.int32).reshape(-1, 3)
        mv = None if movable is None else np.ascontiguousarray(movable, np.uint8)
        n = len(kab)
        iz = np.zeros(max(n, 1), np.int32)
        cap_off, cap_v = n + 1, 4 * n + 1
        off = np.zeros(cap_off, np.int32)
        verts = np.zeros(cap_v, np.int32)
        nz = self.lib.ref_build_zones(C.c_int32(vertex_count), C.c_int32(len(tris)), ptr(tris), ptr(mv),
                                      C.c_int64(n), ptr(kab), ptr(iz), C.c_int64(cap_off), ptr(off),
                                      C.c_int64(cap_v), ptr(verts))
        if nz < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return iz[:n], [verts[off[z]:off[z + 1]].copy() for z in range(nz)]

    def resolve_zones(self, vertex_count, tris, mass, x_begin, x_cand, thickness=0.005, cell_scale=1.5,
                      devices=2, params=None, movable=None):
        """resolve_zones (response.cpp:338-400) -> (status, message, corrected
        candidate, report dict). params: the 8 ZoneSolveParams values."""
        tris = np.ascontiguousarray(tris, np.int32)
        mv = None if movable is None else np.ascontiguousarray(movable, np.uint8)
        xc = np.ascontiguousarray(x_cand, np.float64).reshape(-1).copy()
        zp = np.asarray(params if params is not None else [0.0025, 10.0, 1e-8, 25, 64, 10, 3, 8.0], np.float64)
        rep = np.zeros(5, np.int64)
        st = self.lib.ref_resolve_zones(C.c_int32(vertex_count), C.c_int32(len(tris)), ptr(tris), ptr(mv),
                                        ptr(np.ascontiguousarray(mass, np.float64)),
                                        ptr(np.ascontiguousarray(x_begin, np.float64).reshape(-1)), ptr(xc),
                                        C.c_double(thickness), C.c_double(cell_scale), C.c_int32(devices), ptr(zp),
                                        ptr(rep))
        msg = self.lib.ref_last_error().decode() if st else ""
        keys = ("outer_iterations", "zone_count", "max_zone_vertices", "impacts_resolved", "first_round_impacts")
        return st, msg, xc, dict(zip(keys, rep.tolist()))

    def two_cloth_scene(self, seed, max_side):
        tc = C.c_int32()
        nv = self.lib.ref_two_cloth_scene(C.c_uint64(seed), C.c_int32(max_side), C.byref(tc), None, None, None)
        tris = np.zeros(3 * tc.value, np.int32)
        x0 = np.zeros(3 * nv)
        x1 = np.zeros(3 * nv)
        self.lib.ref_two_cloth_scene(C.c_uint64(seed), C.c_int32(max_side), C.byref(tc), ptr(tris), ptr(x0), ptr(x1))
        return nv, tris.reshape(-1, 3), x0, x1


ORACLE = Oracle() if os.path.exists(ORACLE_SO) else None
REF = Ref() if os.path.exists(REF_SO) else None


class RefError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


class RefSim:
    """The reference's hot-path step (oracle/ref_harness.cpp ref_sim_*)."""

    def __init__(self, ref: Ref, verts, tris, pinned, density, material, devices):
        L = ref.lib
        L.ref_sim_create.restype = C.c_void_p
        L.ref_sim_step.restype = C.c_int32
        for name in ("ref_sim_set_state", "ref_sim_get_state", "ref_sim_step", "ref_sim_free"):
            getattr(L, name).argtypes = None
        self.ref = ref
        v = np.ascontiguousarray(verts, np.float64).reshape(-1)
        t = np.ascontiguousarray(tris, np.int32).reshape(-1)
        mat = np.array(material, np.float64)
        self.p = len(v) // 3
        self.h = L.ref_sim_create(C.c_int32(self.p), ptr(v), C.c_int32(len(t) // 3), ptr(t),
                                  ptr(np.ascontiguousarray(pinned, np.uint8)), C.c_double(density), ptr(mat),
                                  C.c_int32(devices))
        if not self.h:
            raise RuntimeError(L.ref_last_error().decode())

    def set_state(self, x, v):
        self.ref.lib.ref_sim_set_state(C.c_void_p(self.h), ptr(np.ascontiguousarray(x, np.float64)),
                                       ptr(np.ascontiguousarray(v, np.float64)))

    def get_state(self):
        x = np.zeros(3 * self.p)
        v = np.zeros(3 * self.p)
        self.ref.lib.ref_sim_get_state(C.c_void_p(self.h), ptr(x), ptr(v))
        return x, v

    def step(self, dt, thickness, cell_scale=1.5, tol=1e-4, max_it=400):
        prm = np.array([dt, thickness, cell_scale, tol, max_it], np.float64)
        out = np.zeros(8)
        st = self.ref.lib.ref_sim_step(C.c_void_p(self.h), ptr(prm), ptr(out))
        if st:
            raise RuntimeError(self.ref.lib.ref_last_error().decode())
        keys = ("pcg_iterations", "pcg_converged", "pcg_residual", "dcd_candidates", "ccd_candidates", "ms_broad",
                "ms_assemble", "ms_solve")
        return dict(zip(keys, out.tolist()))

    def time_functions(self, dt, thickness, cell_scale=1.5, reps=3):
        """Median ms of fill_matrix, spmv_pipelined and build_grid (DCD) on
        the current state (ref_sim_time_functions)."""
        L = self.ref.lib
        L.ref_sim_time_functions.restype = C.c_int32
        prm = np.array([dt, thickness, cell_scale], np.float64)
        out = np.zeros(3)
        st = L.ref_sim_time_functions(C.c_void_p(self.h), ptr(prm), C.c_int32(reps), ptr(out))
        if st:
            raise RuntimeError(L.ref_last_error().decode())
        return {"fill_matrix_ms": out[0], "spmv_pipelined_ms": out[1], "build_grid_ms": out[2]}

    def step_contacts(self, dt, thickness, cell_scale=1.5, tol=1e-4, max_it=400, stiffness_scale=4.0,
                      friction=0.2, damping=0.0, zones=None):
        """Simulator::step_impl (ref_sim_step_contacts): without impact
        zones, or with them when `zones` = the 8 zone parameters
        (ref_resolve_zones order)."""
        L = self.ref.lib
        L.ref_sim_step_contacts.restype = C.c_int32
        zp = np.zeros(8) if zones is None else np.asarray(zones, np.float64)
        prm = np.concatenate([[dt, thickness, cell_scale, tol, max_it, stiffness_scale, friction, damping,
                               0.0 if zones is None else 1.0], zp])
        out = np.zeros(8)
        st = L.ref_sim_step_contacts(C.c_void_p(self.h), ptr(prm), ptr(out))
        if st:
            raise RefError(st, L.ref_last_error().decode())
        keys = ("pcg_iterations", "pcg_converged", "pcg_residual", "proximities", "contacts", "impacts",
                "zone_count", "zone_outer")
        return dict(zip(keys, out.tolist()))

    def close(self):
        if self.h:
            self.ref.lib.ref_sim_free(C.c_void_p(self.h))
            self.h = None


class RefScene:
    """The reference's scene loader and Simulator (oracle/ref_harness.cpp ref_scene_*)."""

    CONFIG = ("dt", "frames", "devices", "gx", "gy", "gz", "wx", "wy", "wz", "seed", "stretch_warp", "stretch_weft",
              "shear", "bend", "density", "damping", "air_drag", "thickness", "cell_scale", "stiffness_scale",
              "friction", "clearance_fraction", "contact_damping", "rel_tolerance", "max_iterations",
              "block_jacobi", "zone_outer_cap", "zone_initial_penalty", "double")

    def __init__(self, ref: Ref, text: str | None = None, path: str | None = None, base_dir: str = "."):
        L = self.lib = ref.lib
        L.ref_scene_load.restype = C.c_void_p
        L.ref_scene_save_obj.restype = C.c_int64
        L.ref_scene_step.restype = C.c_int32
        src = (text if text is not None else path).encode()
        self.h = L.ref_scene_load(src, C.c_int32(1 if text is not None else 0), base_dir.encode())
        if not self.h:
            raise RefError(7, L.ref_last_error().decode())
        cnt = np.zeros(3 + 3 * 16, np.int32)
        L.ref_scene_info(C.c_void_p(self.h), ptr(cnt), C.c_int32(16))
        self.nverts, self.ntris, self.nobs = int(cnt[0]), int(cnt[1]), int(cnt[2])
        self.obs_counts = [tuple(int(v) for v in cnt[3 + 3 * o:6 + 3 * o]) for o in range(self.nobs)]

    def config(self) -> dict:
        cfg = np.zeros(len(self.CONFIG))
        self.lib.ref_scene_config(C.c_void_p(self.h), ptr(cfg))
        return dict(zip(self.CONFIG, cfg.tolist()))

    def cloth(self):
        v = np.zeros(3 * self.nverts)
        t = np.zeros(3 * self.ntris, np.int32)
        pin = np.zeros(self.nverts, np.uint8)
        self.lib.ref_scene_cloth(C.c_void_p(self.h), ptr(v), ptr(t), ptr(pin))
        return v, t.reshape(-1, 3), pin

    def obstacle(self, o: int, t: float):
        nv, nt, _ = self.obs_counts[o]
        v = np.zeros(3 * nv)
        tr = np.zeros(3 * nt, np.int32)
        self.lib.ref_scene_obstacle(C.c_void_p(self.h), C.c_int32(o), C.c_double(t), ptr(v), ptr(tr))
        return v.reshape(-1, 3), tr.reshape(-1, 3)

    def step(self, devices: int = 0) -> dict:
        out = np.zeros(10)
        st = self.lib.ref_scene_step(C.c_void_p(self.h), C.c_int32(devices), ptr(out))
        if st:
            raise RefError(st, self.lib.ref_last_error().decode())
        keys = ("frame", "time", "pcg_iterations", "pcg_residual", "proximities", "contacts", "impacts",
                "zone_count", "zone_outer", "committed")
        return dict(zip(keys, out.tolist()))

    def state(self):
        x = np.zeros(3 * self.nverts)
        v = np.zeros(3 * self.nverts)
        self.lib.ref_scene_state(C.c_void_p(self.h), ptr(x), ptr(v))
        return x, v

    def instrument(self):
        """Instrument the Simulator (created at the first step)."""
        self.lib.ref_scene_instrument(C.c_void_p(self.h))

    def take_log(self) -> str:
        self.lib.ref_scene_take_log.restype = C.c_int64
        n = self.lib.ref_scene_take_log(C.c_void_p(self.h), None, C.c_int64(0))
        buf = C.create_string_buffer(n + 1)
        self.lib.ref_scene_take_log(C.c_void_p(self.h), buf, C.c_int64(n + 1))
        return buf.value.decode()

    def save_obj(self) -> str:
        n = self.lib.ref_scene_save_obj(C.c_void_p(self.h), None, C.c_int64(0))
        buf = C.create_string_buffer(int(n))
        self.lib.ref_scene_save_obj(C.c_void_p(self.h), buf, C.c_int64(n))
        return buf.raw.decode()

    def close(self):
        if self.h:
            self.lib.ref_scene_free(C.c_void_p(self.h))
            self.h = None
