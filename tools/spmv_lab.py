"""Driver of tools/spmv_lab.cu on the config-D pattern (not product code)."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_00409_b200 import scenes, weft  # noqa: E402

so = os.path.join(ROOT, "tools", "libspmv_lab.so")
if not os.path.exists(so):
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false",
                    "-Xcompiler", "-fPIC", "-shared", "-o", so, os.path.join(ROOT, "tools", "spmv_lab.cu")], check=True)
lib = C.CDLL(so)
sc = scenes.config(sys.argv[1] if len(sys.argv) > 1 else "D")
mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
p = mesh.vertex_count
keys = [np.arange(p, dtype=np.int64) * (p + 1)]
for st in (mesh.triangles, mesh.hinge_verts):
    for a in range(st.shape[1]):
        for b in range(st.shape[1]):
            keys.append(st[:, a].astype(np.int64) * p + st[:, b])
k = np.unique(np.concatenate(keys))
r, c = k // p, k % p
pin = sc.pinned.astype(bool)
keep = (~pin[r] & ~pin[c]) | (r == c)
r, c = r[keep], c[keep]
row_ptr = np.zeros(p + 1, np.int64)
np.add.at(row_ptr, r + 1, 1)
row_ptr = np.cumsum(row_ptr)
cols = c.astype(np.int32)
rng = np.random.default_rng(0)
vals = rng.uniform(-1, 1, 9 * len(cols))
x = rng.uniform(-1, 1, 3 * p)
alg = len(cols) * 76 + p * 52
for sorted_ in (0, 1):
    y = np.zeros(3 * p)
    t = np.zeros(64, np.float32)
    rc = lib.lab_run(C.c_int(p), row_ptr.ctypes.data_as(C.c_void_p), cols.ctypes.data_as(C.c_void_p),
                     vals.ctypes.data_as(C.c_void_p), x.ctypes.data_as(C.c_void_p), C.c_int(sorted_),
                     y.ctypes.data_as(C.c_void_p), t.ctypes.data_as(C.c_void_p))
    assert rc == 0
    print(f"sorted={sorted_} slots={int(t[4])} (nnzb {len(cols)}) k0 {t[0]*1e3:.1f} us {alg/t[0]/1e6:.0f} GB/s", flush=True)
    names = ["C4S4W4B1v3", "C2S5W8B1v3", "C1S4W8B2v3", "C1S6W8B2v3", "C1S4W16B1v3", "C2S3W8B2v3", "C1S8W8B1v3",
             "C1S4W8B2v4", "C1S6W8B2v4", "C2S3W8B2v4", "C1S3W8B3v4", "C2S4W4B3v4"]
    for i in range(int(t[15])):
        tt = t[16 + 2 * i]
        print(f"   k2 {names[i]}: {tt*1e3:.1f} us {alg/tt/1e6:.0f} GB/s mismatch {int(t[17 + 2 * i])}", flush=True)
    alg2 = len(cols) * 76 + p * 76
    print(f"   pcg-form: 2-vector gather {t[5]*1e3:.1f} us {alg2/t[5]/1e6:.0f} GB/s | +dot {t[6]*1e3:.1f} us "
          f"{alg2/t[6]/1e6:.0f} GB/s | +dot after L2 flush {(t[7]-t[8])*1e3:.1f} us {alg2/(t[7]-t[8])/1e6:.0f} GB/s "
          f"(flush {t[8]*1e3:.1f} us)", flush=True)
    if sorted_:
        print(f"   gather layouts (L2 hints, 256-bit): z only {t[9]*1e3:.1f} us | z, p two arrays {t[10]*1e3:.1f} us | "
              f"z|p 64-byte records {t[11]*1e3:.1f} us", flush=True)
