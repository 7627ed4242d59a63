"""Python host mirror of the reference hot-path interface over the C-ABI
(include/weft_gpu.h). Names, argument meaning and error behaviour follow the
reference C++ (proj/include/weft/*.hpp):

* ``Engine(devices)``                 — weft::Engine(n) (exec.hpp:83-128): a GPU
                                         context with n logical row partitions.
* ``Engine.spmv_pipelined(A, x)``     — spmv_pipelined (sparse.hpp:72-101)
* ``Engine.pcg_solve(A, b, cfg)``     — pcg_solve (solver.hpp:36-178)
* ``Engine.fill_matrix(...)``         — fill_matrix (assembly.hpp:74-220)
* ``Engine.step_system(...)``         — step_system (physics.hpp:44-69)
* ``Engine.build_grid(...)``          — build_grid (collision.cpp:118-179)
* ``Engine.candidates(...)``          — narrow_phase_range's candidate walk
                                         (collision.cpp:329-378)
* ``split_workload``, ``make_partitions``, ``generate_work_queues``.

Errors raise the Python counterparts of the reference's exception classes
(``DimensionError``, ``SolverError``, ``ExecError``, ...) with the reference's
message text. The CUDA library is mandatory: importing this module on a box
without ``libweft_gpu.so`` raises, there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WEFT_LIB") or os.path.join(_PKG, "libweft_gpu.so")  # WEFT_LIB: dev variants only

STRETCH, BEND, SPRING, EXTERNAL, CONTACT = range(5)
JAC_EXACT, JAC_SPD = 0, 1
DISCRETE, CONTINUOUS = 0, 1
PRECOND_NONE, PRECOND_BLOCK_JACOBI = 0, 1

ELEMENT_DTYPE = np.dtype(
    [("kind", "<i4"), ("stencil_size", "<i4"), ("stencil", "<i4", (4,)), ("damping", "<f8"), ("data", "<f8", (18,))],
    align=True,
)


class Error(RuntimeError):
    """weft::Error (common.hpp:16-20)."""


class DimensionError(Error):
    pass


class SolverError(Error):
    pass


class ExecError(Error):
    pass


class TopologyError(Error):
    pass


class ScheduleError(Error):
    pass


class ZoneFailure(Error):
    """weft::ZoneFailure (response.hpp:8-11)."""


_ERRORS = {1: DimensionError, 2: SolverError, 3: ExecError, 4: TopologyError, 5: ScheduleError, 6: Error,
           7: ZoneFailure}


class Options(C.Structure):
    _fields_ = [("cuda_device", C.c_int32), ("partitions", C.c_int32), ("part_begin", C.c_int32),
                ("part_end", C.c_int32)]


class PcgConfig(C.Structure):
    """PcgConfig (solver.hpp:17-21)."""

    _fields_ = [("rel_tolerance", C.c_double), ("max_iterations", C.c_int32), ("preconditioner", C.c_int32)]

    def __init__(self, rel_tolerance=1e-4, max_iterations=400, preconditioner=PRECOND_BLOCK_JACOBI):
        super().__init__(rel_tolerance, max_iterations, preconditioner)


class _PcgReport(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("rel_residual", C.c_double),
                ("residual_history", C.POINTER(C.c_double)), ("precond_norm_history", C.POINTER(C.c_double))]


class MatrixInfo(C.Structure):
    _fields_ = [("block_rows", C.c_int32), ("max_row_blocks", C.c_int32), ("nnzb", C.c_int64),
                ("padded_slots", C.c_int64)]


class RankInfo(C.Structure):
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("first_row", C.c_int32), ("rows", C.c_int32),
                ("global_rows", C.c_int32)]


IPC_HANDLE_BYTES = 64


def rank_partitions(partitions: int, world: int, rank: int):
    """Partition range [begin, end) of `rank` in a group of `world` ranks
    over `partitions` logical partitions (equal contiguous ranges)."""
    if world < 1 or partitions % world != 0 or not 0 <= rank < world:
        raise TopologyError(f"{partitions} partitions cannot be split over {world} ranks")
    span = partitions // world
    return rank * span, (rank + 1) * span


def exchange_handles(mine: bytes, world: int, group=None) -> list:
    """All ranks' window handles in rank order (torch.distributed
    all_gather_object; the bytes are opaque, any backend works)."""
    import torch.distributed as dist
    if dist.get_world_size(group) != world:
        raise TopologyError(f"process group has {dist.get_world_size(group)} ranks, the engine expects {world}")
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    return allh


def rank_share(total: int, world: int, rank: int):
    """This rank's range of split_workload(total, world) (collision.cpp:
    181-192): the pair-space share a rank walks in the replicated broad
    phase (csrc/sim.cu mirrors it)."""
    base, extra = divmod(total, world)
    b = rank * base + min(rank, extra)
    return b, b + base + (1 if rank < extra else 0)


class GridInfo(C.Structure):
    _fields_ = [("cell_size", C.c_double), ("cells", C.c_int64), ("entries", C.c_int64), ("total", C.c_int64)]


class ZoneParams(C.Structure):
    """ZoneSolveParams (response.hpp:46-60), the reference's defaults."""
    _fields_ = [("clearance", C.c_double), ("initial_penalty", C.c_double), ("inner_tolerance", C.c_double),
                ("al_iterations", C.c_int32), ("inner_iterations", C.c_int32), ("outer_cap", C.c_int32),
                ("retry_cap", C.c_int32), ("max_correction_factor", C.c_double)]

    def __init__(self, clearance=0.0025, initial_penalty=10.0, inner_tolerance=1e-8, al_iterations=25,
                 inner_iterations=64, outer_cap=10, retry_cap=3, max_correction_factor=8.0):
        super().__init__(clearance, initial_penalty, inner_tolerance, al_iterations, inner_iterations, outer_cap,
                         retry_cap, max_correction_factor)

    def as_array(self):
        return np.array([self.clearance, self.initial_penalty, self.inner_tolerance, self.al_iterations,
                         self.inner_iterations, self.outer_cap, self.retry_cap, self.max_correction_factor])


class ZoneReport(C.Structure):
    """ZoneResolveReport (response.hpp:62-68)."""
    _fields_ = [("outer_iterations", C.c_int32), ("zone_count", C.c_int32), ("max_zone_vertices", C.c_int32),
                ("impacts_resolved", C.c_int64), ("first_round_impacts", C.c_int64)]


class SimParams(C.Structure):
    _fields_ = [("dt", C.c_double), ("thickness", C.c_double), ("cell_scale", C.c_double), ("pcg", PcgConfig),
                ("jac_mode", C.c_int32), ("contacts", C.c_int32), ("stiffness_scale", C.c_double),
                ("friction", C.c_double), ("contact_damping", C.c_double), ("zones", C.c_int32),
                ("zone", ZoneParams), ("precision", C.c_int32)]

    def __init__(self, dt=1.0 / 240.0, thickness=0.005, cell_scale=1.5, pcg=None, jac_mode=1, contacts=0,
                 stiffness_scale=4.0, friction=0.2, contact_damping=0.0, zones=0, zone=None, precision=0):
        """SimConfig subset (driver.hpp:30-45): collision, ContactParams
        (response.hpp:13-21) and ZoneSolveParams defaults of the reference;
        the zone clearance follows Simulator's rule clearance_fraction (0.5) *
        thickness (driver.cpp:87-89) unless `zone` is given."""
        if zone is None:
            zone = ZoneParams(clearance=0.5 * thickness)
        super().__init__(dt, thickness, cell_scale, pcg if pcg is not None else PcgConfig(), jac_mode, contacts,
                         stiffness_scale, friction, contact_damping, zones, zone, precision)


class StepReport(C.Structure):
    _fields_ = [("pcg_iterations", C.c_int32), ("pcg_converged", C.c_int32), ("pcg_residual", C.c_double),
                ("dcd_candidates", C.c_int64), ("ccd_candidates", C.c_int64), ("ms_broad", C.c_double),
                ("ms_assemble", C.c_double), ("ms_solve", C.c_double), ("proximities", C.c_int64),
                ("contact_elements", C.c_int64), ("impacts", C.c_int64), ("zone_count", C.c_int32),
                ("zone_outer", C.c_int32), ("ms_zones", C.c_double), ("stages", C.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2008_00409_b200.build` "
                          "(no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    lib.weft_gpu_last_error.restype = C.c_char_p
    return lib


LIB = _load()


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(C.c_void_p)
    if hasattr(a, "data_ptr"):  # torch tensor (device or host)
        return C.c_void_p(a.data_ptr())
    raise TypeError(type(a))


def _check(status: int):
    if status != 0:
        msg = LIB.weft_gpu_last_error().decode()
        raise _ERRORS.get(status, Error)(msg)


def _f64(a):
    return np.ascontiguousarray(a, np.float64).reshape(-1)


def _state_buf(a, n: int, what: str, output: bool):
    """A state buffer handed to the library as a raw pointer: exactly n
    contiguous float64 values (numpy array or torch tensor, host or device).
    Inputs given as other array-likes are converted; anything the library
    could read or write past the end of is rejected."""
    if a is None:
        raise Error(f"{what}: buffer is None")
    if hasattr(a, "data_ptr") and not isinstance(a, np.ndarray):
        import torch
        if a.dtype != torch.float64 or not a.is_contiguous() or a.numel() != n:
            raise DimensionError(f"{what}: need a contiguous float64 tensor of {n} values "
                                 f"(got {a.dtype}, {a.numel()} values, contiguous={a.is_contiguous()})")
        return a
    if not isinstance(a, np.ndarray):
        if output:
            raise Error(f"{what}: output must be a numpy array or a torch tensor")
        a = np.asarray(a)
    if output:
        if a.dtype != np.float64 or not a.flags.c_contiguous or not a.flags.writeable or a.size != n:
            raise DimensionError(f"{what}: need a writable C-contiguous float64 array of {n} values "
                                 f"(got {a.dtype}, {a.size} values)")
        return a
    a = _f64(a)
    if a.size != n:
        raise DimensionError(f"{what}: need {n} values, got {a.size}")
    return a


# ---------------------------------------------------------------------------
# free functions
# ---------------------------------------------------------------------------
def make_partitions(vertex_count: int, devices: int):
    """make_partitions (exec.cpp:10-23) -> list of (begin, end)."""
    b = np.zeros(devices, np.int32)
    e = np.zeros(devices, np.int32)
    _check(LIB.weft_make_partitions(C.c_int32(vertex_count), C.c_int32(devices), _ptr(b), _ptr(e)))
    return list(zip(b.tolist(), e.tolist()))


def generate_work_queues(devices: int):
    """generate_work_queues(FatTree::make(n)) (topology.cpp:79-89) -> per
    device list of (peer, vec)."""
    m = max(devices - 1, 1)
    peer = np.zeros(devices * m, np.int32)
    vec = np.zeros(devices * m, np.int32)
    _check(LIB.weft_work_queues(C.c_int32(devices), _ptr(peer), _ptr(vec)))
    return [list(zip(peer[d * (devices - 1):(d + 1) * (devices - 1)].tolist(),
                     vec[d * (devices - 1):(d + 1) * (devices - 1)].tolist())) for d in range(devices)]


def distribute_zones(sizes, devices: int):
    """distribute_zones (response.cpp:164-182) -> per device list of zone ids."""
    sz = np.ascontiguousarray(sizes, np.int32)
    dev = np.zeros(max(len(sz), 1), np.int32)
    _check(LIB.weft_distribute_zones(C.c_int32(len(sz)), _ptr(sz), C.c_int32(devices), _ptr(dev)))
    out = [[] for _ in range(devices)]
    order = sorted(range(len(sz)), key=lambda z: -int(sz[z]))  # assignment order (stable)
    for z in order:
        out[int(dev[z])].append(z)
    return out


def split_workload(total: int, devices: int):
    """split_workload (collision.cpp:181-192) -> list of (begin, end)."""
    b = np.zeros(devices, np.int64)
    e = np.zeros(devices, np.int64)
    _check(LIB.weft_split_workload(C.c_int64(total), C.c_int32(devices), _ptr(b), _ptr(e)))
    return list(zip(b.tolist(), e.tolist()))


@dataclass
class BlockCsr:
    """Global 3x3-block matrix, ascending columns; values (nnzb, 9) row-major."""

    rows: int
    row_ptr: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    rhs: np.ndarray | None = None


@dataclass
class PcgReport:
    """PcgReport (solver.hpp:23-29)."""

    iterations: int = 0
    rel_residual: float = 0.0
    converged: bool = False
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    precond_norm_history: np.ndarray = field(default_factory=lambda: np.zeros(0))


@dataclass
class HashGrid:
    """HashGrid + WorkloadTable (collision.hpp:59-70) as flat arrays."""

    cell_size: float
    cell_keys: np.ndarray
    cell_offsets: np.ndarray
    cell_tris: np.ndarray
    prefix: np.ndarray
    tri_boxes: np.ndarray

    @property
    def total(self) -> int:
        return int(self.prefix[-1]) if len(self.prefix) else 0


class Engine:
    """A GPU context with ``devices`` logical row partitions (weft::Engine).

    ``world``/``rank`` > 1 make it one rank of a group (one process per GPU)
    holding partitions ``rank_partitions(devices, world, rank)``; call
    ``attach_peers`` once the vertex count is known (after set_vertices or
    set_matrix)."""

    def __init__(self, devices: int = 1, cuda_device: int = 0, world: int = 1, rank: int = 0):
        self._ctx = C.c_void_p()
        b, e = rank_partitions(devices, world, rank)
        opts = Options(cuda_device, devices, b, e)
        _check(LIB.weft_gpu_create(C.byref(opts), C.byref(self._ctx)))
        self.devices = devices
        self.world = world
        self.rank = rank

    def close(self):
        if self._ctx:
            _check(LIB.weft_gpu_destroy(self._ctx))
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- rank group ---------------------------------------------------------
    def rank_info(self) -> RankInfo:
        info = RankInfo()
        _check(LIB.weft_gpu_rank_info(self._ctx, C.byref(info)))
        return info

    def comm_export(self) -> bytes:
        h = (C.c_ubyte * IPC_HANDLE_BYTES)()
        _check(LIB.weft_gpu_comm_export(self._ctx, h))
        return bytes(h)

    def comm_attach(self, handles):
        if len(handles) != self.world or any(len(h) != IPC_HANDLE_BYTES for h in handles):
            raise Error("comm_attach: need one handle per rank")
        buf = (C.c_ubyte * (IPC_HANDLE_BYTES * self.world)).from_buffer_copy(b"".join(handles))
        _check(LIB.weft_gpu_comm_attach(self._ctx, buf))

    def attach_peers(self, group=None):
        """Exports this rank's window and maps every peer's, exchanging the
        handle bytes through torch.distributed (any backend)."""
        self.comm_attach(exchange_handles(self.comm_export(), self.world, group))

    # -- sparse -------------------------------------------------------------
    def set_matrix(self, m: BlockCsr):
        """float32 values: a Precision::Single system (BellMatrix<float>);
        spmv_pipelined / pcg_solve then take and return float32 vectors."""
        rp = _ptr(np.ascontiguousarray(m.row_ptr, np.int64))
        cl = _ptr(np.ascontiguousarray(m.cols, np.int32))
        if np.asarray(m.vals).dtype == np.float32:
            v32 = np.ascontiguousarray(m.vals, np.float32)
            _check(LIB.weft_gpu_set_matrix_f32(self._ctx, C.c_int32(m.rows), rp, cl, _ptr(v32)))
            self._f32 = True
        else:
            _check(LIB.weft_gpu_set_matrix(self._ctx, C.c_int32(m.rows), rp, cl, _ptr(_f64(m.vals))))
            self._f32 = False

    def spmv_pipelined(self, m: BlockCsr | None, x) -> np.ndarray:
        if m is not None:
            self.set_matrix(m)
        rows = self.rank_info().global_rows
        if getattr(self, "_f32", False):
            x = np.ascontiguousarray(x, np.float32)
            if len(x) != 3 * rows:
                raise DimensionError("spmv_pipelined: dim(x) != rows")
            y = np.zeros(3 * rows, np.float32)
            _check(LIB.weft_gpu_spmv_f32(self._ctx, _ptr(x), _ptr(y)))
            return y
        x = _f64(x)
        if len(x) != 3 * rows:
            raise DimensionError("spmv_pipelined: dim(x) != rows")
        y = np.zeros(3 * rows)
        _check(LIB.weft_gpu_spmv(self._ctx, _ptr(x), _ptr(y)))
        return y

    def matrix_info(self) -> MatrixInfo:
        info = MatrixInfo()
        _check(LIB.weft_gpu_matrix_info(self._ctx, C.byref(info)))
        return info

    def download_matrix(self) -> BlockCsr:
        info = self.matrix_info()
        rp = np.zeros(info.block_rows + 1, np.int64)
        cols = np.zeros(max(info.nnzb, 1), np.int32)
        if getattr(self, "_f32", False):
            vals = np.zeros(max(info.nnzb, 1) * 9, np.float32)
            _check(LIB.weft_gpu_download_matrix_f32(self._ctx, _ptr(rp), _ptr(cols), _ptr(vals)))
        else:
            vals = np.zeros(max(info.nnzb, 1) * 9)
            _check(LIB.weft_gpu_download_matrix(self._ctx, _ptr(rp), _ptr(cols), _ptr(vals)))
        return BlockCsr(info.block_rows, rp, cols[: info.nnzb], vals[: 9 * info.nnzb].reshape(-1, 9))

    def download_rhs(self) -> np.ndarray:
        info = self.matrix_info()
        if getattr(self, "_f32", False):
            rhs = np.zeros(3 * info.block_rows, np.float32)
            _check(LIB.weft_gpu_download_rhs_f32(self._ctx, _ptr(rhs)))
            return rhs
        rhs = np.zeros(3 * info.block_rows)
        _check(LIB.weft_gpu_download_rhs(self._ctx, _ptr(rhs)))
        return rhs

    def pcg_solve(self, m: BlockCsr | None, b, config: PcgConfig | None = None):
        """pcg_solve; ``m=None`` uses the context's current (assembled)
        matrix, ``b=None`` its assembled rhs. Returns (x, PcgReport)."""
        if m is not None:
            self.set_matrix(m)
        config = config or PcgConfig()
        n = 3 * self.rank_info().global_rows
        f32 = getattr(self, "_f32", False)
        x = np.zeros(n, np.float32 if f32 else np.float64)
        hist = np.zeros(max(config.max_iterations, 1))
        phist = np.zeros(max(config.max_iterations, 1))
        rep = _PcgReport(0, 0, 0.0, hist.ctypes.data_as(C.POINTER(C.c_double)),
                         phist.ctypes.data_as(C.POINTER(C.c_double)))
        if f32:
            bb = None if b is None else np.ascontiguousarray(b, np.float32)
            _check(LIB.weft_gpu_pcg_f32(self._ctx, _ptr(bb), _ptr(x), C.byref(config), C.byref(rep)))
        else:
            bb = None if b is None else _f64(b)
            _check(LIB.weft_gpu_pcg(self._ctx, _ptr(bb), _ptr(x), C.byref(config), C.byref(rep)))
        return x, PcgReport(rep.iterations, rep.rel_residual, bool(rep.converged), hist[: rep.iterations].copy(),
                            phist[: rep.iterations].copy())

    # -- assembly -----------------------------------------------------------
    def set_vertices(self, mass, pinned):
        mass = _f64(mass)
        pinned = np.ascontiguousarray(pinned, np.uint8)
        _check(LIB.weft_gpu_set_vertices(self._ctx, C.c_int32(len(mass)), _ptr(mass), _ptr(pinned)))

    def set_elements(self, elements):
        e = np.ascontiguousarray(elements, ELEMENT_DTYPE)
        _check(LIB.weft_gpu_set_elements(self._ctx, C.c_int64(len(e)), _ptr(e)))

    def set_contacts(self, contacts):
        e = np.ascontiguousarray(contacts if contacts is not None else np.zeros(0, ELEMENT_DTYPE), ELEMENT_DTYPE)
        _check(LIB.weft_gpu_set_contacts(self._ctx, C.c_int64(len(e)), _ptr(e)))

    def fill_matrix(self, x_current, x_advanced, velocity, dt: float, mode: int = JAC_SPD, single: bool = False):
        """fill_matrix over the context's static + contact elements; the
        system stays resident (download_matrix / download_rhs to read).
        single: fill_matrix<float> (Precision::Single)."""
        fn = LIB.weft_gpu_fill_matrix_f32 if single else LIB.weft_gpu_fill_matrix
        _check(fn(self._ctx, _ptr(_f64(x_current)), _ptr(_f64(x_advanced)), _ptr(_f64(velocity)), C.c_double(dt),
                  C.c_int32(mode)))
        self._f32 = bool(single)

    def step_system(self, x, v, dt: float, mode: int = JAC_SPD, single: bool = False):
        fn = LIB.weft_gpu_step_system_f32 if single else LIB.weft_gpu_step_system
        _check(fn(self._ctx, _ptr(_f64(x)), _ptr(_f64(v)), C.c_double(dt), C.c_int32(mode)))
        self._f32 = bool(single)

    # -- broad phase --------------------------------------------------------
    def set_soup(self, vertex_count: int, tris):
        t = np.ascontiguousarray(tris, np.int32).reshape(-1)
        _check(LIB.weft_gpu_set_soup(self._ctx, C.c_int32(vertex_count), C.c_int32(len(t) // 3), _ptr(t)))

    def build_grid(self, x_begin, x_end=None, mode: int = DISCRETE, thickness: float = 0.005,
                   cell_scale: float = 1.5):
        xb = _f64(x_begin)
        xe = None if x_end is None else _f64(x_end)
        _check(LIB.weft_gpu_build_grid(self._ctx, _ptr(xb), _ptr(xe), C.c_int32(mode), C.c_double(thickness),
                                       C.c_double(cell_scale)))

    def grid_info(self) -> GridInfo:
        info = GridInfo()
        _check(LIB.weft_gpu_grid_info(self._ctx, C.byref(info)))
        return info

    def download_grid(self, tri_count: int) -> HashGrid:
        info = self.grid_info()
        keys = np.zeros(info.cells, np.uint64)
        off = np.zeros(info.cells + 1, np.int64)
        tris = np.zeros(max(info.entries, 1), np.int32)
        prefix = np.zeros(info.cells + 1, np.int64)
        boxes = np.zeros(6 * max(tri_count, 1), np.int64)
        _check(LIB.weft_gpu_download_grid(self._ctx, _ptr(keys), _ptr(off), _ptr(tris), _ptr(prefix), _ptr(boxes)))
        return HashGrid(info.cell_size, keys, off, tris[: info.entries], prefix, boxes[: 6 * tri_count].reshape(-1, 6))

    def candidates(self, begin: int | None = None, end: int | None = None) -> np.ndarray:
        info = self.grid_info()
        begin = 0 if begin is None else begin
        end = info.total if end is None else end
        n = C.c_int64()
        _check(LIB.weft_gpu_candidates(self._ctx, C.c_int64(begin), C.c_int64(end), C.byref(n), None))
        pairs = np.zeros(2 * max(n.value, 1), np.int32)
        _check(LIB.weft_gpu_candidates(self._ctx, C.c_int64(begin), C.c_int64(end), C.byref(n), _ptr(pairs)))
        return pairs[: 2 * n.value].reshape(-1, 2)

    # -- narrow phase ----------------------------------------
    def set_soup_movable(self, movable=None):
        m = None if movable is None else np.ascontiguousarray(movable, np.uint8)
        _check(LIB.weft_gpu_set_soup_movable(self._ctx, _ptr(m)))

    def collide(self, x_begin, x_end=None, mode: int = DISCRETE, thickness: float = 0.005, cell_scale: float = 1.5):
        """collide (collision.cpp:391-417): broad + narrow phase, sorted and
        deduplicated by (kind, a, b). Returns (kab (n, 3) int32: kind 0 =
        VertexFace / 1 = EdgeEdge, a, b; vals (n, 8): gap|toi, normal xyz,
        weights 0..3)."""
        xb = x_begin if hasattr(x_begin, "data_ptr") else _f64(x_begin)
        xe = None if x_end is None else (x_end if hasattr(x_end, "data_ptr") else _f64(x_end))
        n = C.c_int64()
        _check(LIB.weft_gpu_collide(self._ctx, _ptr(xb), _ptr(xe), C.c_int32(mode), C.c_double(thickness),
                                    C.c_double(cell_scale), C.byref(n)))
        kab = np.zeros((max(n.value, 1), 3), np.int32)
        vals = np.zeros((max(n.value, 1), 8))
        _check(LIB.weft_gpu_download_contacts(self._ctx, _ptr(kab), _ptr(vals)))
        return kab[: n.value], vals[: n.value]

    # -- impact zones (response.cpp:108-400) --------------------------------
    def build_zones(self, kab):
        """build_zones (response.cpp:108-162) over (kind, a, b) impacts on
        the soup -> (impact_zone (n,), list of per-zone movable vertices)."""
        kab = np.ascontiguousarray(kab, np.int32).reshape(-1, 3)
        n = len(kab)
        iz = np.zeros(max(n, 1), np.int32)
        nz = C.c_int32()
        nv = C.c_int64()
        _check(LIB.weft_gpu_build_zones(self._ctx, C.c_int64(n), _ptr(kab), _ptr(iz), C.byref(nz), C.byref(nv)))
        off = np.zeros(nz.value + 1, np.int32)
        verts = np.zeros(max(nv.value, 1), np.int32)
        _check(LIB.weft_gpu_zone_vertices(self._ctx, _ptr(off), _ptr(verts)))
        return iz[:n], [verts[off[z]:off[z + 1]].copy() for z in range(nz.value)]

    def resolve_zones(self, x_begin, x_candidate, vertex_mass, thickness: float = 0.005, cell_scale: float = 1.5,
                      params: "ZoneParams | None" = None):
        """resolve_zones (response.cpp:338-400): returns (corrected
        candidate positions, ZoneReport); raises ZoneFailure like the
        reference (with .x_candidate = the positions it left behind)."""
        xc = _f64(x_candidate).copy()
        rep = ZoneReport()
        prm = params if params is not None else ZoneParams()
        try:
            _check(LIB.weft_gpu_resolve_zones(self._ctx, _ptr(_f64(x_begin)), _ptr(xc), _ptr(_f64(vertex_mass)),
                                              C.c_double(thickness), C.c_double(cell_scale), C.byref(prm),
                                              C.byref(rep)))
        except ZoneFailure as e:  # the positions reached, as the reference leaves them
            e.x_candidate, e.report = xc, rep
            raise
        return xc, rep

    # -- device-resident step -----------------------------------------------
    def _state_len(self) -> int:
        return 3 * self.rank_info().global_rows

    def sim_set_state(self, x, v):
        n = self._state_len()
        x = _state_buf(x, n, "sim_set_state: x", False)
        v = _state_buf(v, n, "sim_set_state: v", False)
        _check(LIB.weft_gpu_sim_set_state(self._ctx, _ptr(x), _ptr(v)))

    def sim_set_obstacles(self, dt: float, x_begin, x_end):
        """Obstacle vertex positions at the step's start and end (soup
        vertices after the cloth's; driver.cpp:113-131)."""
        _check(LIB.weft_gpu_sim_set_obstacles(self._ctx, C.c_double(dt), _ptr(_f64(x_begin)), _ptr(_f64(x_end))))

    def sim_step(self, params: SimParams) -> StepReport:
        rep = StepReport()
        _check(LIB.weft_gpu_sim_step(self._ctx, C.byref(params), C.byref(rep)))
        return rep

    def sim_step_io(self, x_in, v_in, params: SimParams, x_out, v_out) -> StepReport:
        """weft_gpu_sim_step_io: upload (x, v), one step, read (x, v) back,
        with the copies overlapped with the broad phases."""
        n = self._state_len()
        x_in = _state_buf(x_in, n, "sim_step_io: x_in", False)
        v_in = _state_buf(v_in, n, "sim_step_io: v_in", False)
        x_out = _state_buf(x_out, n, "sim_step_io: x_out", True)
        v_out = _state_buf(v_out, n, "sim_step_io: v_out", True)
        rep = StepReport()
        _check(LIB.weft_gpu_sim_step_io(self._ctx, _ptr(x_in), _ptr(v_in), C.byref(params), _ptr(x_out), _ptr(v_out),
                                        C.byref(rep)))
        return rep

    def sim_get_state(self, x=None, v=None):
        n = self._state_len()
        x = None if x is None else _state_buf(x, n, "sim_get_state: x", True)
        v = None if v is None else _state_buf(v, n, "sim_get_state: v", True)
        _check(LIB.weft_gpu_sim_get_state(self._ctx, _ptr(x), _ptr(v)))


# ---------------------------------------------------------------------------
# static mesh precompute (include/weft_mesh.h) — one-time host setup
# ---------------------------------------------------------------------------
LIB.weft_mesh_last_error.restype = C.c_char_p
LIB.weft_mesh_destroy.argtypes = [C.c_void_p]

DEFAULT_MATERIAL = (400.0, 400.0, 60.0, 2e-5, 0.15, 0.002, 0.0)  # MaterialParams (physics.hpp:8-16)


def _mcheck(status: int):
    if status != 0:
        raise (DimensionError if status == 1 else Error)(LIB.weft_mesh_last_error().decode())


class ClothMesh:
    """ClothMesh (mesh.hpp:13-52): rest data, hinges, lumped masses."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        nv, nt, nh, ne = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _mcheck(LIB.weft_mesh_info(self._h, C.byref(nv), C.byref(nt), C.byref(nh), C.byref(ne)))
        nv, nt, nh = nv.value, nt.value, nh.value
        self.rest = np.zeros(3 * nv)
        self.triangles = np.zeros((nt, 3), np.int32)
        self.tri_rest = np.zeros((nt, 7))
        self.tri_degenerate = np.zeros(nt, np.uint8)
        self.hinge_verts = np.zeros((nh, 4), np.int32)
        self.hinge_data = np.zeros((nh, 2))
        self.vertex_area = np.zeros(nv)
        self.vertex_mass = np.zeros(nv)
        _mcheck(LIB.weft_mesh_copy(self._h, _ptr(self.rest), _ptr(self.triangles), _ptr(self.tri_rest),
                                   _ptr(self.tri_degenerate), _ptr(self.hinge_verts), _ptr(self.hinge_data),
                                   _ptr(self.vertex_area), _ptr(self.vertex_mass)))

    @property
    def vertex_count(self) -> int:
        return len(self.vertex_mass)

    @classmethod
    def build(cls, vertices, triangles, density: float) -> "ClothMesh":
        v = _f64(vertices)
        t = np.ascontiguousarray(triangles, np.int32).reshape(-1)
        h = C.c_void_p()
        _mcheck(LIB.weft_mesh_build(C.c_int32(len(v) // 3), _ptr(v), C.c_int32(len(t) // 3), _ptr(t),
                                    C.c_double(density), C.byref(h)))
        return cls(h)

    @classmethod
    def grid(cls, nx: int, ny: int, width: float, height: float, origin=(0.0, 0.0, 0.0), density: float = 0.15):
        """make_grid_mesh (mesh.cpp:187-212)."""
        h = C.c_void_p()
        o = np.array(origin, np.float64)
        _mcheck(LIB.weft_mesh_grid(C.c_int32(nx), C.c_int32(ny), C.c_double(width), C.c_double(height), _ptr(o),
                                   C.c_double(density), C.byref(h)))
        return cls(h)

    def build_elements(self, material=DEFAULT_MATERIAL, gravity=(0.0, 0.0, -9.81), wind=(0.0, 0.0, 0.0)):
        """build_elements (physics.cpp:5-63): triangles, hinges, vertices."""
        mat = np.array(material, np.float64)
        g = np.array(gravity, np.float64)
        w = np.array(wind, np.float64)
        n = C.c_int64()
        _mcheck(LIB.weft_build_elements(self._h, _ptr(mat), _ptr(g), _ptr(w), None, C.c_int64(0), C.byref(n)))
        out = np.zeros(n.value, ELEMENT_DTYPE)
        _mcheck(LIB.weft_build_elements(self._h, _ptr(mat), _ptr(g), _ptr(w), _ptr(out), C.c_int64(n.value),
                                        C.byref(n)))
        return out

    def __del__(self):
        if getattr(self, "_h", None) and LIB is not None:
            try:
                LIB.weft_mesh_destroy(self._h)
            except Exception:
                pass
            self._h = None


class GpuStats(C.Structure):
    _fields_ = [("launches", C.c_int64), ("spmv_launches", C.c_int64), ("spmv_ms", C.c_double),
                ("pcg_solves", C.c_int64), ("pcg_iterations", C.c_int64), ("pcg_ms", C.c_double),
                ("pcg_bytes", C.c_double)]


def _engine_profile(self, enable: bool = True):
    _check(LIB.weft_gpu_profile(self._ctx, C.c_int32(1 if enable else 0)))


def _engine_stats(self) -> GpuStats:
    st = GpuStats()
    _check(LIB.weft_gpu_stats(self._ctx, C.byref(st)))
    return st


def _engine_stream(self) -> int:
    s = C.c_void_p()
    _check(LIB.weft_gpu_get_stream(self._ctx, C.byref(s)))
    return s.value or 0


def _engine_set_instrument(self, on: bool = True):
    """EngineOptions::instrument: record the reference's solver event lines
    (event=pcg, event=zones) — take them with take_log()."""
    _check(LIB.weft_gpu_set_instrument(self._ctx, C.c_int32(1 if on else 0)))


def _engine_take_log(self) -> str:
    n = C.c_int64()
    _check(LIB.weft_gpu_take_log(self._ctx, None, C.c_int64(0), C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(LIB.weft_gpu_take_log(self._ctx, buf, C.c_int64(n.value + 1), C.byref(n)))
    return buf.value.decode()


Engine.set_instrument = _engine_set_instrument
Engine.take_log = _engine_take_log
Engine.profile = _engine_profile
Engine.stats = _engine_stats
Engine.stream = _engine_stream
