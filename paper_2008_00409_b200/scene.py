"""Scene files, mesh I/O and the simulation driver of the reference, on the
B200 library (SURVEY §8(f) #4 wire formats + the Simulator that runs them).

Host-side mirror of the reference's scene / driver layer, so a user of the
reference can load the same JSON scenes and run them on the GPU:

* parse_scene / load_scene      — proj/src/scene.cpp:45-178 (same keys,
  defaults, generators, pins and SceneError messages)
* make_uv_sphere / make_funnel / make_box / load_obj / save_obj
                                — proj/src/mesh.cpp:214-337
* Obstacle.positions_at         — proj/src/driver.cpp:14-43 (keyframe
  interpolation, AngleAxisd rotation in the Eigen shim's association)
* RunReport.write_csv           — proj/src/scene.cpp:180-190
* Simulator                     — proj/src/driver.cpp:55-215: the soup is the
  cloth followed by the obstacles, every step is ONE device-resident
  weft_gpu_sim_step (DCD narrow phase -> contacts -> assembly -> PCG -> CCD
  -> impact zones -> commit) with the obstacle positions of the step.

Vector arithmetic follows the reference's left-to-right association so
generated meshes and obstacle positions are bitwise the reference's.
"""
from __future__ import annotations

import json
import math
import os
import time as _time
from dataclasses import dataclass, field

import numpy as np

from . import weft


class SceneError(weft.Error):
    """weft::SceneError (common.hpp:44-47)."""


# ---------------------------------------------------------------- config
@dataclass
class Material:  # MaterialParams (physics.hpp:8-16)
    stretch_warp: float = 400.0
    stretch_weft: float = 400.0
    shear: float = 60.0
    bend: float = 2e-5
    density: float = 0.15
    damping: float = 0.002
    air_drag: float = 0.0

    def as_tuple(self):
        return (self.stretch_warp, self.stretch_weft, self.shear, self.bend, self.density, self.damping,
                self.air_drag)


@dataclass
class SimConfig:  # SimConfig (driver.hpp:31-45) with its member defaults
    dt: float = 1.0 / 150.0
    frames: int = 100
    devices: int = 1
    precision: str = "double"
    gravity: tuple = (0.0, 0.0, -9.81)
    wind: tuple = (0.0, 0.0, 0.0)
    material: Material = field(default_factory=Material)
    thickness: float = 0.005           # CollisionParams
    cell_scale: float = 1.5
    stiffness_scale: float = 4.0       # ContactParams (response.hpp:13-21)
    friction: float = 0.2
    clearance_fraction: float = 0.5
    contact_damping: float = 0.0
    rel_tolerance: float = 1e-4        # PcgConfig (solver.hpp:15-21)
    max_iterations: int = 400
    preconditioner: str = "block-jacobi"
    zones: weft.ZoneParams = field(default_factory=weft.ZoneParams)
    seed: int = 0


# ---------------------------------------------------------------- meshes
@dataclass
class TriSoup:
    vertices: np.ndarray  # (n, 3) float64
    triangles: np.ndarray  # (m, 3) int32


def _add(a, b):
    return (a[0] + b[0], a[1] + b[1], a[2] + b[2])


def _scl(s, a):
    return (s * a[0], s * a[1], s * a[2])


def _soup(verts, tris) -> TriSoup:
    return TriSoup(np.array(verts, np.float64).reshape(-1, 3), np.array(tris, np.int32).reshape(-1, 3))


def make_uv_sphere(center, radius: float, stacks: int, slices: int) -> TriSoup:
    """mesh.cpp:214-237."""
    v = [_add(center, (0.0, 0.0, radius))]
    for i in range(1, stacks):
        phi = math.pi * i / stacks
        for j in range(slices):
            theta = 2.0 * math.pi * j / slices
            sp = math.sin(phi)
            v.append(_add(center, _scl(radius, (sp * math.cos(theta), sp * math.sin(theta), math.cos(phi)))))
    v.append(_add(center, (0.0, 0.0, -radius)))
    bottom = len(v) - 1

    def ring(i, j):
        return 1 + (i - 1) * slices + (j % slices)

    t = [(0, ring(1, j), ring(1, j + 1)) for j in range(slices)]
    for i in range(1, stacks - 1):
        for j in range(slices):
            t.append((ring(i, j), ring(i + 1, j), ring(i + 1, j + 1)))
            t.append((ring(i, j), ring(i + 1, j + 1), ring(i, j + 1)))
    t += [(bottom, ring(stacks - 1, j + 1), ring(stacks - 1, j)) for j in range(slices)]
    return _soup(v, t)


def make_funnel(top_center, top_radius: float, bottom_radius: float, height: float, segments: int) -> TriSoup:
    """mesh.cpp:239-262: cone plus a collar below the neck."""
    v = []
    collar = 0.35 * height

    def add_ring(radius, z):
        for j in range(segments):
            theta = 2.0 * math.pi * j / segments
            v.append(_add(top_center, (radius * math.cos(theta), radius * math.sin(theta), z)))

    add_ring(top_radius, 0.0)
    add_ring(bottom_radius, -height)
    add_ring(bottom_radius, -height - collar)

    def ring(r, j):
        return r * segments + (j % segments)

    t = []
    for r in range(2):
        for j in range(segments):
            t.append((ring(r, j), ring(r, j + 1), ring(r + 1, j)))
            t.append((ring(r, j + 1), ring(r + 1, j + 1), ring(r + 1, j)))
    return _soup(v, t)


def make_box(center, half) -> TriSoup:
    """mesh.cpp:264-276."""
    v = [_add(center, (half[0] if i & 1 else -half[0], half[1] if i & 2 else -half[1], half[2] if i & 4 else -half[2]))
         for i in range(8)]
    faces = [(0, 2, 3, 1), (4, 5, 7, 6), (0, 1, 5, 4), (2, 6, 7, 3), (0, 4, 6, 2), (1, 3, 7, 5)]
    t = []
    for f in faces:
        t.append((f[0], f[1], f[2]))
        t.append((f[0], f[2], f[3]))
    return _soup(v, t)


def load_obj(path: str) -> TriSoup:
    """mesh.cpp:278-318: "v x y z" and "f a b c ..." records (i, i/t, i/t/n;
    negative = relative), polygons fan-triangulated."""
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise SceneError(f"cannot open mesh file: {path}") from None
    verts, tris = [], []
    for no, line in enumerate(lines, 1):
        items = line.split()
        if not items:
            continue
        if items[0] == "v":
            try:
                verts.append((float(items[1]), float(items[2]), float(items[3])))
            except (IndexError, ValueError):
                raise SceneError(f"{path}:{no}: malformed vertex record") from None
        elif items[0] == "f":
            ids = []
            for it in items[1:]:
                head = it.split("/")[0]
                try:
                    k = int(head)
                except ValueError:
                    k = 0
                if k == 0:
                    raise SceneError(f"{path}:{no}: malformed face record")
                ids.append(k - 1 if k > 0 else len(verts) + k)
            if len(ids) < 3:
                raise SceneError(f"{path}:{no}: face with <3 vertices")
            for k in range(1, len(ids) - 1):
                tris.append((ids[0], ids[k], ids[k + 1]))
    for t in tris:
        for v in t:
            if v < 0 or v >= len(verts):
                raise SceneError(f"{path}: face index out of range")
    return _soup(verts, tris)


def save_obj(out, positions, triangles) -> None:
    """mesh.cpp:320-332: "v %.17g %.17g %.17g" lines then 1-based faces.
    `out`: a path or a text stream."""
    if isinstance(out, (str, os.PathLike)):
        try:
            with open(out, "w") as f:
                save_obj(f, positions, triangles)
        except OSError:
            raise SceneError(f"cannot write mesh file: {out}") from None
        return
    pos = np.asarray(positions, np.float64).reshape(-1, 3)
    out.write("".join("v %s %s %s\n" % (_g17(p[0]), _g17(p[1]), _g17(p[2])) for p in pos))
    out.write("".join(f"f {t[0] + 1} {t[1] + 1} {t[2] + 1}\n" for t in np.asarray(triangles).reshape(-1, 3)))


def _g17(x: float) -> str:
    return "%.17g" % float(x)


# ---------------------------------------------------------------- obstacles
@dataclass
class Keyframe:
    time: float = 0.0
    translate: tuple = (0.0, 0.0, 0.0)
    axis: tuple = (0.0, 0.0, 1.0)
    angle: float = 0.0
    center: tuple = (0.0, 0.0, 0.0)


@dataclass
class Obstacle:
    shape: TriSoup
    keyframes: list = field(default_factory=list)

    def positions_at(self, t: float) -> np.ndarray:
        """Obstacle::positions_at (driver.cpp:22-43)."""
        out = self.shape.vertices.copy()
        if not self.keyframes:
            return out
        kf = self.keyframes
        if t <= kf[0].time:
            k = kf[0]
        elif t >= kf[-1].time:
            k = kf[-1]
        else:
            hi = 1
            while kf[hi].time < t:
                hi += 1
            a, b = kf[hi - 1], kf[hi]
            d = b.time - a.time
            u = (t - a.time) / (d if 1e-12 < d else 1e-12)  # std::max(1e-12, d)
            k = Keyframe(a.time, _add(_scl(1.0 - u, a.translate), _scl(u, b.translate)), b.axis,
                         (1.0 - u) * a.angle + u * b.angle, b.center)
        rot = _axis_angle(k.axis, k.angle)
        for i in range(len(out)):
            p = out[i]
            q = (p[0] - k.center[0], p[1] - k.center[1], p[2] - k.center[2])
            r = [(rot[m][0] * q[0] + rot[m][1] * q[1]) + rot[m][2] * q[2] for m in range(3)]
            out[i] = [(r[m] + k.center[m]) + k.translate[m] for m in range(3)]
        return out


def _axis_angle(axis, angle):
    """axis_angle (driver.cpp:14-18) with Eigen::AngleAxisd::toRotationMatrix
    in the shim's association (oracle/shim/Eigen/Dense)."""
    ln = math.sqrt((axis[0] * axis[0] + axis[1] * axis[1]) + axis[2] * axis[2])
    if ln < 1e-12 or angle == 0.0:
        return [[1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]
    ax = (axis[0] / ln, axis[1] / ln, axis[2] / ln)
    sn = math.sin(angle)
    s_ax = (sn * ax[0], sn * ax[1], sn * ax[2])
    c = math.cos(angle)
    c1 = (1.0 - c) * ax[0], (1.0 - c) * ax[1], (1.0 - c) * ax[2]
    m = [[0.0] * 3 for _ in range(3)]
    tmp = c1[0] * ax[1]
    m[0][1] = tmp - s_ax[2]
    m[1][0] = tmp + s_ax[2]
    tmp = c1[0] * ax[2]
    m[0][2] = tmp + s_ax[1]
    m[2][0] = tmp - s_ax[1]
    tmp = c1[1] * ax[2]
    m[1][2] = tmp - s_ax[0]
    m[2][1] = tmp + s_ax[0]
    m[0][0] = c1[0] * ax[0] + c
    m[1][1] = c1[1] * ax[1] + c
    m[2][2] = c1[2] * ax[2] + c
    return m


# ---------------------------------------------------------------- scenes
@dataclass
class Scene:
    name: str
    cloth: weft.ClothMesh
    pinned: np.ndarray
    obstacles: list
    config: SimConfig
    grid: tuple | None = None  # (nx, ny) for grid cloths


def _vec3(j, fallback=(0.0, 0.0, 0.0)):
    if j is None:
        return fallback
    if not isinstance(j, list) or len(j) != 3:
        raise SceneError("expected a 3-element array")
    return (float(j[0]), float(j[1]), float(j[2]))


def _soup_of(j, base_dir) -> TriSoup:
    if "obj" in j:
        return load_obj(os.path.join(base_dir, j["obj"]))
    if "sphere" in j:
        s = j["sphere"]
        return make_uv_sphere(_vec3(s.get("center")), s.get("radius", 0.1), s.get("stacks", 12), s.get("slices", 18))
    if "funnel" in j:
        f = j["funnel"]
        return make_funnel(_vec3(f.get("top_center")), f.get("top_radius", 0.3), f.get("bottom_radius", 0.08),
                           f.get("height", 0.3), f.get("segments", 24))
    if "box" in j:
        b = j["box"]
        return make_box(_vec3(b.get("center")), _vec3(b.get("half_extents")))
    raise SceneError("mesh spec needs one of: obj, sphere, funnel, box")


def parse_scene(text: str, base_dir: str = ".") -> Scene:
    """parse_scene (scene.cpp:45-165)."""
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise SceneError(f"scene parse error: {e}") from None
    cfg = SimConfig()
    cfg.dt = float(j.get("dt", 1.0 / 150.0))
    cfg.frames = int(j.get("frames", 100))
    cfg.devices = int(j.get("devices", 1))
    cfg.gravity = _vec3(j.get("gravity"), (0.0, 0.0, -9.81))
    cfg.wind = _vec3(j.get("wind"), (0.0, 0.0, 0.0))
    cfg.seed = int(j.get("seed", 0))
    cfg.precision = j.get("precision", "double")
    if cfg.precision not in ("double", "single"):
        raise SceneError(f"precision must be 'single' or 'double', got '{cfg.precision}'")
    if "material" in j:
        m, mat = j["material"], cfg.material
        mat.stretch_warp = float(m.get("stretch", mat.stretch_warp))
        mat.stretch_weft = float(m.get("stretch_weft", mat.stretch_warp))
        mat.shear = float(m.get("shear", mat.shear))
        mat.bend = float(m.get("bend", mat.bend))
        mat.density = float(m.get("density", mat.density))
        mat.damping = float(m.get("damping", mat.damping))
        mat.air_drag = float(m.get("air_drag", mat.air_drag))
    if "collision" in j:
        c = j["collision"]
        cfg.thickness = float(c.get("thickness", cfg.thickness))
        cfg.cell_scale = float(c.get("cell_scale", cfg.cell_scale))
        cfg.stiffness_scale = float(c.get("contact_stiffness_scale", cfg.stiffness_scale))
        cfg.friction = float(c.get("friction", cfg.friction))
        cfg.clearance_fraction = float(c.get("clearance_fraction", cfg.clearance_fraction))
    if "solver" in j:
        s = j["solver"]
        cfg.rel_tolerance = float(s.get("tolerance", cfg.rel_tolerance))
        cfg.max_iterations = int(s.get("max_iterations", cfg.max_iterations))
        cfg.preconditioner = s.get("preconditioner", "block-jacobi")
        if cfg.preconditioner not in ("none", "block-jacobi"):
            raise SceneError(f"unknown preconditioner '{cfg.preconditioner}'")
    if "zones" in j:
        z = j["zones"]
        cfg.zones.outer_cap = int(z.get("outer_cap", cfg.zones.outer_cap))
        cfg.zones.initial_penalty = float(z.get("initial_penalty", cfg.zones.initial_penalty))
    if "cloth" not in j:
        raise SceneError("scene has no 'cloth' section")
    cj = j["cloth"]
    grid = None
    if "grid" in cj:
        g = cj["grid"]
        grid = (int(g.get("nx", 20)), int(g.get("ny", 20)))
        if grid[0] < 2 or grid[1] < 2:
            raise SceneError("grid mesh needs at least 2x2 vertices")
        cloth = weft.ClothMesh.grid(grid[0], grid[1], float(g.get("width", 0.5)), float(g.get("height", 0.5)),
                                    _vec3(g.get("origin")), cfg.material.density)
    elif "obj" in cj:
        soup = load_obj(os.path.join(base_dir, cj["obj"]))
        cloth = weft.ClothMesh.build(soup.vertices, soup.triangles, cfg.material.density)
    else:
        raise SceneError("cloth section needs 'grid' or 'obj'")
    p = cloth.vertex_count
    pinned = np.zeros(p, np.uint8)
    for v in cj.get("pins", []):
        if v < 0 or v >= p:
            raise SceneError("pin index out of range")
        pinned[v] = 1
    if cj.get("pin_top_edge", False):  # grid convention: the last row is the top edge
        g = cj["grid"]
        nx, ny = int(g.get("nx", 20)), int(g.get("ny", 20))
        pinned[(ny - 1) * nx:(ny - 1) * nx + nx] = 1
    if cj.get("pin_corners", False):
        g = cj["grid"]
        nx, ny = int(g.get("nx", 20)), int(g.get("ny", 20))
        pinned[(ny - 1) * nx] = 1
        pinned[ny * nx - 1] = 1
    obstacles = []
    for oj in j.get("obstacles", []):
        kfs = [Keyframe(float(k.get("time", 0.0)), _vec3(k.get("translate")), _vec3(k.get("rotate_axis"), (0.0, 0.0, 1.0)),
                        float(k.get("rotate_angle", 0.0)), _vec3(k.get("rotate_center")))
               for k in oj.get("keyframes", [])]
        obstacles.append(Obstacle(_soup_of(oj, base_dir), kfs))
    return Scene(j.get("name", "scene"), cloth, pinned, obstacles, cfg, grid)


def load_scene(path: str) -> Scene:
    """load_scene (scene.cpp:167-178)."""
    try:
        text = open(path).read()
    except OSError:
        raise SceneError(f"cannot open scene file: {path}") from None
    try:
        return parse_scene(text, os.path.dirname(path) or ".")
    except SceneError as e:
        raise SceneError(f"{path}: {e}") from None


# ---------------------------------------------------------------- reports
@dataclass
class FrameReport:  # driver.hpp:47-63
    frame: int = 0
    time: float = 0.0
    integrate_ms: float = 0.0
    broad_ms: float = 0.0
    narrow_ms: float = 0.0
    zones_ms: float = 0.0
    pcg_iterations: int = 0
    pcg_residual: float = 0.0
    proximities: int = 0
    contacts: int = 0
    impacts: int = 0
    zone_count: int = 0
    zone_outer: int = 0
    committed: bool = False
    stage_trace: list = field(default_factory=list)


def canonical_stage_order() -> list:
    """The per-step stage order instrumentation asserts (driver.cpp:49-53)."""
    return ["proximity_dcd", "assemble", "solve", "candidate", "ccd", "zones", "commit"]


def _g10(x) -> str:
    """ostream << double with precision(10) (default float format = %.10g)."""
    return "%.10g" % x


@dataclass
class RunReport:
    frames: list = field(default_factory=list)
    wall_seconds: float = 0.0
    devices: int = 1

    def write_csv(self, out) -> None:
        """RunReport::write_csv (scene.cpp:180-190)."""
        out.write("frame,time,integrate_ms,broad_ms,narrow_ms,zones_ms,pcg_iterations,pcg_residual,"
                  "proximities,contacts,impacts,zones,zone_outer,committed\n")
        for f in self.frames:
            out.write(",".join([str(f.frame), _g10(f.time), _g10(f.integrate_ms), _g10(f.broad_ms),
                                _g10(f.narrow_ms), _g10(f.zones_ms), str(f.pcg_iterations), _g10(f.pcg_residual),
                                str(f.proximities), str(f.contacts), str(f.impacts), str(f.zone_count),
                                str(f.zone_outer), "1" if f.committed else "0"]) + "\n")


# ---------------------------------------------------------------- driver
class Simulator:
    """Simulator (driver.cpp:55-215) on one GPU: the state stays on the
    device; step() issues one weft_gpu_sim_step (the whole step_impl)."""

    def __init__(self, scene: Scene, devices: int | None = None, cuda_device: int = 0, instrument=None):
        """instrument: a writable text stream (EngineOptions::instrument): the
        reference's event lines — stage (driver.cpp:104-111), pcg
        (solver.hpp:171-175) and zones (response.cpp:383-388) — in its
        order and format."""
        self.scene = scene
        cfg = scene.config
        self.mesh = scene.cloth
        p = self.mesh.vertex_count
        self.engine = weft.Engine(devices or cfg.devices, cuda_device=cuda_device)
        self.instrument = instrument
        if instrument is not None:
            self.engine.set_instrument(True)
        self.engine.set_vertices(self.mesh.vertex_mass, scene.pinned)
        self.engine.set_elements(self.mesh.build_elements(cfg.material.as_tuple(), cfg.gravity, cfg.wind))
        tris = [np.asarray(self.mesh.triangles, np.int32).reshape(-1, 3)]
        off = p
        for ob in scene.obstacles:  # CollisionSoup: cloth then obstacles (driver.cpp:73-85)
            tris.append(ob.shape.triangles + off)
            off += len(ob.shape.vertices)
        self.soup_vertices = off
        self.engine.set_soup(off, np.concatenate(tris))
        self.engine.set_soup_movable(np.concatenate([1 - scene.pinned, np.zeros(off - p, np.uint8)]))
        x0 = np.asarray(self.mesh.rest, np.float64).reshape(-1)
        self.engine.sim_set_state(x0, np.zeros_like(x0))
        self.time = 0.0
        self.frame = 0
        zp = weft.ZoneParams(*[getattr(cfg.zones, f) for f, _ in weft.ZoneParams._fields_])
        zp.clearance = cfg.clearance_fraction * cfg.thickness  # driver.cpp:87-89
        pc = weft.PcgConfig(cfg.rel_tolerance, cfg.max_iterations,
                            weft.PRECOND_BLOCK_JACOBI if cfg.preconditioner == "block-jacobi" else weft.PRECOND_NONE)
        self.params = weft.SimParams(cfg.dt, cfg.thickness, cfg.cell_scale, pc, weft.JAC_SPD, contacts=1,
                                     stiffness_scale=cfg.stiffness_scale, friction=cfg.friction,
                                     contact_damping=cfg.contact_damping, zones=1, zone=zp,
                                     precision=1 if cfg.precision == "single" else 0)  # step_impl<Real>

    def _obstacles_at(self, t: float) -> np.ndarray:
        if not self.scene.obstacles:
            return np.zeros(0)
        return np.concatenate([ob.positions_at(t).reshape(-1) for ob in self.scene.obstacles])

    def step(self) -> FrameReport:
        dt = self.scene.config.dt
        if self.scene.obstacles:
            self.engine.sim_set_obstacles(dt, self._obstacles_at(self.time), self._obstacles_at(self.time + dt))
        t0 = _time.perf_counter()
        try:
            r = self.engine.sim_step(self.params)
        except weft.Error as e:
            # the stages the reference logged before it threw: up to the solve
            # for a solver error, up to the zones for a zone failure
            last = "zones" if isinstance(e, weft.ZoneFailure) else "solve"
            order = canonical_stage_order()
            self._log_frame(order[:order.index(last) + 1])
            raise
        stages = canonical_stage_order()[:r.stages]
        self._log_frame(stages)
        if stages != canonical_stage_order():  # driver.cpp:211-213
            raise weft.ExecError(f"frame {self.frame}: stage order violated")
        rep = FrameReport(self.frame, self.time, r.ms_assemble + r.ms_solve, r.ms_broad, 0.0, r.ms_zones,
                          r.pcg_iterations, r.pcg_residual, r.proximities, r.contact_elements, r.impacts,
                          r.zone_count, r.zone_outer, True, stages)
        rep.wall_ms = 1e3 * (_time.perf_counter() - t0)
        self.time += dt
        self.frame += 1
        return rep

    def _log_frame(self, stages):
        """Writes the frame's instrument lines: each stage as it starts, the
        solver's events after the stage that emits them."""
        if self.instrument is None:
            return
        events = [ln for ln in self.engine.take_log().splitlines() if ln]
        for name in stages:
            self.instrument.write(f"event=stage frame={self.frame} name={name}\n")
            kind = {"solve": "event=pcg ", "zones": "event=zones "}.get(name)
            if kind:
                for ln in events:
                    if ln.startswith(kind):
                        self.instrument.write(ln + "\n")

    def state(self):
        p = self.mesh.vertex_count
        x, v = np.zeros(3 * p), np.zeros(3 * p)
        self.engine.sim_get_state(x, v)
        return x.reshape(-1, 3), v.reshape(-1, 3)

    def run(self, frames: int | None = None) -> RunReport:
        rep = RunReport(devices=self.engine.partitions if hasattr(self.engine, "partitions") else 1)
        t0 = _time.perf_counter()
        for _ in range(frames if frames is not None else self.scene.config.frames):
            rep.frames.append(self.step())
        rep.wall_seconds = _time.perf_counter() - t0
        return rep

    def close(self):
        self.engine.close()
