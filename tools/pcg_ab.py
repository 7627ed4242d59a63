"""A/B timing of library variants (WEFT_LIB=...): config D, the bench's
replayed state (2 steps from rest), median device time of the PCG stage over
8 replayed steps. Prints one line per run."""
import hashlib
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_00409_b200 import scenes, weft  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "D"
sc = scenes.config(cfg, seed=20240810)
mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
p = mesh.vertex_count
eng = weft.Engine(int(os.environ.get("PARTS", "1")))
eng.set_vertices(mesh.vertex_mass, sc.pinned)
eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
eng.set_soup(p, sc.tris)
x0 = sc.verts.reshape(-1).copy()
eng.sim_set_state(x0, np.zeros_like(x0))
prm = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-4, 400), weft.JAC_SPD)
for _ in range(2):
    eng.sim_step(prm)
xs, vs = np.zeros(3 * p), np.zeros(3 * p)
eng.sim_get_state(xs, vs)
solve, asm, broad, its = [], [], [], []
for k in range(9):
    eng.sim_set_state(xs, vs)
    r = eng.sim_step(prm)
    if k:
        solve.append(r.ms_solve)
        asm.append(r.ms_assemble)
        broad.append(r.ms_broad)
        its.append(r.pcg_iterations)
ms = statistics.median(solve)
xo, vo = np.zeros(3 * p), np.zeros(3 * p)
eng.sim_get_state(xo, vo)
digest = hashlib.sha1(xo.tobytes() + vo.tobytes()).hexdigest()[:12]
print(f"{os.environ.get('WEFT_LIB', 'default')} parts={os.environ.get('PARTS', '1')} persistent={os.environ.get('WEFT_PCG_PERSISTENT', '1')} rows={os.environ.get('WEFT_PCG_ROWS', '1')}: solve {ms:.3f} ms ({1e3 * ms / its[-1]:.1f} us/it, {its[-1]} its) "
      f"asm {statistics.median(asm):.3f} broad {statistics.median(broad):.3f} state {digest}", flush=True)
