"""Runs N device-resident steps of a config and prints per-step stats."""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2008_00409_b200 import scenes, weft  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "B"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
import os
sp = float(os.environ.get("SPACING", "0.005"))
dt = float(os.environ.get("DT", str(1.0 / 240.0)))
layers, nx = scenes.CONFIGS[cfg]
sc = scenes.layered_cloth(layers, nx, spacing=sp, dt=dt)
mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
p = mesh.vertex_count
eng = weft.Engine(1)
eng.set_vertices(mesh.vertex_mass, sc.pinned)
eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
eng.set_soup(p, sc.tris)
x0 = sc.verts.reshape(-1).copy()
eng.sim_set_state(x0, np.zeros_like(x0))
prm = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-4, 400), weft.JAC_SPD)
x = np.zeros(3 * p)
v = np.zeros(3 * p)
for k in range(n):
    t0 = time.perf_counter()
    try:
        r = eng.sim_step(prm)
    except Exception as e:
        print("step", k, "failed:", e)
        break
    t1 = time.perf_counter()
    eng.sim_get_state(x, v)
    g = eng.grid_info()
    print(f"step {k}: {1e3*(t1-t0):.2f} ms wall | broad {r.ms_broad:.2f} asm {r.ms_assemble:.2f} solve {r.ms_solve:.2f} | "
          f"it {r.pcg_iterations} res {r.pcg_residual:.2e} | dcd {r.dcd_candidates} ccd {r.ccd_candidates} | "
          f"cells {g.cells} entries {g.entries} W {g.total} | max|x-x0| {np.abs(x-x0).max():.3e} max|v| {np.abs(v).max():.3e}",
          flush=True)
