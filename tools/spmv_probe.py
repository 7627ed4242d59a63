"""ncu target for the standalone SpMV: config D, `steps` device-resident steps
from rest (the bench's trajectory), then `reps` y = A x through weft_gpu_spmv
on the last assembled system (x ~ U(-1, 1)).

  ncu --set full -k regex:k_spmv -c 1 python tools/spmv_probe.py D 2 3
"""
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2008_00409_b200 import scenes, weft  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "D"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
sc = scenes.config(cfg, seed=20240810)
mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
p = mesh.vertex_count
eng = weft.Engine(1)
eng.set_vertices(mesh.vertex_mass, sc.pinned)
eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
eng.set_soup(p, sc.tris)
x0 = sc.verts.reshape(-1).copy()
eng.sim_set_state(x0, np.zeros_like(x0))
prm = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-4, 400), weft.JAC_SPD)
for _ in range(steps):
    eng.sim_step(prm)
xr = np.random.default_rng(0).uniform(-1.0, 1.0, 3 * p)
for _ in range(reps):
    y = eng.spmv_pipelined(None, xr)
print("spmv", float(np.abs(y).sum()))
