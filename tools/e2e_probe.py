"""Dev probe: where the end-to-end step's extra time goes (config D):
device-resident sim_step vs sim_step_io with pinned host buffers, and the
bare H2D / D2H copy times of one state vector on the context stream."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_00409_b200 import scenes, weft  # noqa: E402

sc = scenes.config("D")
mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
p = mesh.vertex_count
eng = weft.Engine(1)
eng.set_vertices(mesh.vertex_mass, sc.pinned)
eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
eng.set_soup(p, sc.tris)
x0 = sc.verts.reshape(-1).copy()
eng.sim_set_state(x0, np.zeros_like(x0))
prm = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-4, 400), weft.JAC_SPD)
for _ in range(3):
    eng.sim_step(prm)
stream = torch.cuda.ExternalStream(eng.stream())
xs = torch.empty(3 * p, dtype=torch.float64, device="cuda")
vs = torch.empty(3 * p, dtype=torch.float64, device="cuda")
eng.sim_get_state(xs, vs)


def timed(f, n=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(n):
        f()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / n


def dev():
    eng.sim_set_state(xs, vs)  # outside-stream copies are D2D here
    eng.sim_step(prm)


xa, va = xs.cpu().pin_memory(), vs.cpu().pin_memory()
xb = torch.empty(3 * p, dtype=torch.float64, pin_memory=True)
vb = torch.empty(3 * p, dtype=torch.float64, pin_memory=True)


def io():
    return eng.sim_step_io(xa, va, prm, xb, vb)


with torch.cuda.stream(stream):
    hb = torch.empty(3 * p, dtype=torch.float64, pin_memory=True)
    db = torch.empty(3 * p, dtype=torch.float64, device="cuda")
    h2d = timed(lambda: db.copy_(hb, non_blocking=True), 10)
    d2h = timed(lambda: hb.copy_(db, non_blocking=True), 10)
print(f"state vector {24 * p / 1e6:.1f} MB: H2D {h2d:.3f} ms ({24 * p / h2d / 1e6:.1f} GB/s), "
      f"D2H {d2h:.3f} ms ({24 * p / d2h / 1e6:.1f} GB/s)")
print(f"set_state + sim_step (device copies): {timed(dev):.3f} ms")
print(f"sim_step_io (pinned host buffers):    {timed(io):.3f} ms")
eng.sim_set_state(xs, vs)
r = eng.sim_step(prm)
print(f"device step stage ms: broad {r.ms_broad:.3f} assemble {r.ms_assemble:.3f} solve {r.ms_solve:.3f} its {r.pcg_iterations}")
r = io()
print(f"io step stage ms:     broad {r.ms_broad:.3f} assemble {r.ms_assemble:.3f} solve {r.ms_solve:.3f} its {r.pcg_iterations}")
