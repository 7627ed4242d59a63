"""Synthetic scenes at the BASELINE configurations:
stacked grid layers of `make_grid_mesh` topology (proj/src/mesh.cpp:187-212),
jittered rest shape (as oracle::random_cloth, physics_oracle.cpp:90-101),
top edge of every layer pinned (scene.cpp:137-142), layers 1.5 x thickness
apart so they are in DCD proximity from step 0, v0 = 0.

Material of the configurations: the MaterialParams defaults (physics.hpp:8-16)
with the stretch and shear stiffness scaled by CONFIG_STRETCH_SCALE. The
reference's stretch / shear conditions are area-weighted (C = a(|w|-1) and
C = a w_u.w_v, elements.cpp:170-172), so a stiffness acts with the squared
rest area: the default 400 N/m is calibrated for ~1 cm triangles (the
reference's scenes, scenes/sphere.json) and cannot carry a hanging sheet of
5 mm triangles — the sheet free-falls, its top row over-stretches and the
run diverges after ~10 steps, identically in both arms. Scaled x1024 the
same sheet runs a stable trajectory (measured >= 40 steps at config D with
the compiled reference) at the same PCG work (~163 iterations per step)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# name -> (layers, nx): BASELINE.md §2 table
CONFIGS = {
    "A": (1, 100),    # 100x100 sheet, ~20K triangles
    "B": (3, 309),    # Zoey-scale, 569,184 triangles
    "C": (2, 501),    # Kimono-scale, 1,000,000 triangles
    "D": (3, 525),    # Kneel-scale, 1,647,456 triangles
    # E: the 0.5M-10M triangle sweep (BASELINE.json configs[4])
    "E05": (1, 501),  # 500,000 triangles, one layer
    "E1": (1, 708),   # 1,000,416 triangles, one layer
    "E3": (3, 708),   # 3,001,248 triangles
    "E5": (4, 792),   # 5,004,504 triangles
    "E10": (4, 1119), # 9,999,392 triangles
}


@dataclass
class Scene:
    verts: np.ndarray      # (p, 3) rest = initial positions
    tris: np.ndarray       # (T, 3) int32
    pinned: np.ndarray     # (p,) uint8
    layers: int
    nx: int
    spacing: float
    thickness: float
    dt: float
    density: float = 0.15
    material: tuple = (400.0, 400.0, 60.0, 2e-5, 0.15, 0.002, 0.0)
    gravity: tuple = (0.0, 0.0, -9.81)

    @property
    def vertex_count(self) -> int:
        return len(self.verts)

    @property
    def tri_count(self) -> int:
        return len(self.tris)


def grid_tris(nx: int, ny: int, offset: int = 0) -> np.ndarray:
    """Triangles of make_grid_mesh (alternating quad diagonals)."""
    j, i = np.meshgrid(np.arange(ny - 1), np.arange(nx - 1), indexing="ij")
    i = i.reshape(-1)
    j = j.reshape(-1)
    a = j * nx + i
    b = j * nx + i + 1
    c = (j + 1) * nx + i + 1
    d = (j + 1) * nx + i
    even = (i + j) % 2 == 0
    t = np.empty((len(a), 2, 3), np.int64)
    t[even, 0] = np.stack([a, b, c], 1)[even]
    t[even, 1] = np.stack([a, c, d], 1)[even]
    t[~even, 0] = np.stack([a, b, d], 1)[~even]
    t[~even, 1] = np.stack([b, c, d], 1)[~even]
    return (t.reshape(-1, 3) + offset).astype(np.int32)


CONFIG_STRETCH_SCALE = 1024.0


def layered_cloth(layers: int, nx: int, spacing: float = 0.005, seed: int = 20240810, jitter: float = 0.15,
                  dt: float = 1.0 / 240.0, hanging: bool = True, stretch_scale: float = 1.0) -> Scene:
    width = spacing * (nx - 1)
    thickness = 0.5 * spacing
    dz = 1.5 * thickness
    rng = np.random.default_rng(seed)
    gi, gj = np.meshgrid(np.arange(nx), np.arange(nx), indexing="xy")
    base = np.stack([width * gi.reshape(-1) / (nx - 1), width * gj.reshape(-1) / (nx - 1),
                     np.zeros(nx * nx)], 1)
    if hanging:  # sheet in the x-z plane, grid row j = nx-1 on top (pinned), layers stacked along y
        base = base[:, [0, 2, 1]]
    verts, tris, pinned = [], [], []
    for k in range(layers):
        v = base.copy()
        v[:, 1 if hanging else 2] = k * dz
        v += rng.uniform(-jitter * spacing, jitter * spacing, v.shape)
        verts.append(v)
        tris.append(grid_tris(nx, nx, k * nx * nx))
        pin = np.zeros(nx * nx, np.uint8)
        pin[(nx - 1) * nx:] = 1  # pin_top_edge: last grid row
        pinned.append(pin)
    mat = list(Scene.material)
    mat[0] *= stretch_scale
    mat[1] *= stretch_scale
    mat[2] *= stretch_scale
    return Scene(np.concatenate(verts), np.concatenate(tris), np.concatenate(pinned), layers, nx, spacing,
                 thickness, dt, material=tuple(mat))


def config(name: str, seed: int = 20240810) -> Scene:
    layers, nx = CONFIGS[name]
    return layered_cloth(layers, nx, seed=seed, stretch_scale=CONFIG_STRETCH_SCALE)
