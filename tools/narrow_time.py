"""Times weft_gpu_collide (broad + narrow phase) on a config's replayed state."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_2008_00409_b200 import scenes, weft  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "D"
sc = scenes.config(cfg)
mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
p = mesh.vertex_count
eng = weft.Engine(1)
eng.set_vertices(mesh.vertex_mass, sc.pinned)
eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
eng.set_soup(p, sc.tris)
eng.set_soup_movable(1 - sc.pinned)
x0 = sc.verts.reshape(-1).copy()
eng.sim_set_state(x0, np.zeros_like(x0))
prm = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-4, 400), weft.JAC_SPD)
for _ in range(2):
    eng.sim_step(prm)
x = np.zeros(3 * p)
v = np.zeros(3 * p)
eng.sim_get_state(x, v)
xc = x + sc.dt * v
for mode, name, xe in ((weft.DISCRETE, "DCD", None), (weft.CONTINUOUS, "CCD", xc)):
    for k in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        kab, vals = eng.collide(x, xe, mode, sc.thickness)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(f"  {name} call {k}: {1e3 * (t1 - t0):.1f} ms", flush=True)
    g = eng.grid_info()
    print(f"{name}: {1e3 * (t1 - t0):.1f} ms wall (incl. H2D of x, D2H of hits) | W {g.total} | hits {len(kab)} "
          f"(VF {(kab[:, 0] == 0).sum()}, EE {(kab[:, 0] == 1).sum()})", flush=True)
