"""Times the plain SpMV and the PCG of the assembled config-D system with
CUDA events on the context stream (device pointers, no host copies)."""
import os
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
x = sc.verts.reshape(-1).copy()
v = np.zeros_like(x)
eng.step_system(x, v, sc.dt)
info = eng.matrix_info()
alg = info.nnzb * 76 + info.block_rows * (4 + 48)
xd = torch.rand(3 * p, dtype=torch.float64, device="cuda")
yd = torch.empty_like(xd)
stream = torch.cuda.ExternalStream(eng.stream())
for _ in range(3):
    weft.LIB.weft_gpu_spmv(eng._ctx, weft._ptr(xd), weft._ptr(yd))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 50
e0.record(stream)
for _ in range(n):
    weft.LIB.weft_gpu_spmv(eng._ctx, weft._ptr(xd), weft._ptr(yd))
e1.record(stream)
e1.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"spmv {ms*1e3:.1f} us/launch (incl. 2 D2D copies of x,y), alg {alg/1e6:.0f} MB -> {alg/ms/1e6:.0f} GB/s "
      f"(pair={os.environ.get('WEFT_SPMV_PAIR', '0')})")
for _ in range(2):
    eng.pcg_solve(None, None)
e0.record(stream)
xs, rep = eng.pcg_solve(None, None)
e1.record(stream)
e1.synchronize()
print(f"pcg {e0.elapsed_time(e1):.2f} ms, {rep.iterations} its, {e0.elapsed_time(e1)/rep.iterations*1e3:.1f} us/it")
eng.profile(True)
eng.pcg_solve(None, None)
st = eng.stats()
print(f"profiled pcg spmv {st.spmv_ms/st.spmv_launches*1e3:.1f} us/launch over {st.spmv_launches}")
