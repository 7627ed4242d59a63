"""Times the contacts-mode step (DCD narrow phase -> contacts -> assembly ->
PCG -> CCD narrow phase) on a config's replayed state."""
import sys

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
x0 = sc.verts.reshape(-1).copy()
eng.sim_set_state(x0, np.zeros_like(x0))
hot = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-4, 400), weft.JAC_SPD)
full = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-4, 400), weft.JAC_SPD, contacts=1)
for _ in range(2):
    eng.sim_step(hot)
xs = torch.empty(3 * p, dtype=torch.float64, device="cuda")
vs = torch.empty(3 * p, dtype=torch.float64, device="cuda")
eng.sim_get_state(xs, vs)
stream = torch.cuda.ExternalStream(eng.stream())
for k in range(5):
    eng.sim_set_state(xs, vs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    try:
        r = eng.sim_step(full)
    except weft.Error as e:
        print("step failed:", e)
        break
    e1.record(stream)
    e1.synchronize()
    print(f"contacts step {k}: {e0.elapsed_time(e1):.1f} ms | prox {r.proximities} contacts {r.contact_elements} "
          f"impacts {r.impacts} | its {r.pcg_iterations} | broad {r.ms_broad:.1f} asm {r.ms_assemble:.1f} "
          f"solve {r.ms_solve:.1f}", flush=True)
info = eng.matrix_info()
print(f"matrix: rows {info.block_rows} nnzb {info.nnzb} padded {info.padded_slots} max_len {info.max_row_blocks}")
