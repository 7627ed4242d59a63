"""Driver of tools/symlab.cu on the config-D pattern (dev experiment, not product code):
plain SELL-32 SpMV vs reading lower-triangle blocks from their upper mirrors."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_00409_b200 import scenes, weft  # noqa: E402

so = os.path.join(ROOT, "tools", "libsymlab.so")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false",
                "-Xcompiler", "-fPIC", "-shared", "-o", so, os.path.join(ROOT, "tools", "symlab.cu")], check=True)
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
row_len = np.bincount(r, minlength=p)
row_ptr = np.concatenate([[0], np.cumsum(row_len)])
kk = np.arange(len(r)) - row_ptr[r]
slices = (p + 31) // 32
slen_pad = np.zeros(slices * 32, np.int64)
slen_pad[:p] = row_len
slice_len = slen_pad.reshape(slices, 32).max(1)
sbase = np.concatenate([[0], np.cumsum(slice_len * 32)]).astype(np.int64)
slots = int(sbase[-1])
addr = sbase[r // 32] + kk * 32 + (r % 32)
cols = np.zeros(slots, np.int32)
cols[addr] = c
# partner of (r, c) is (c, r)
pk = np.searchsorted(k, c * p + r)
assert np.array_equal(k[pk], c * p + r)
paddr = addr[pk]
lower = c < r
mirror = np.full(slots, -1, np.int32)
mirror[addr[lower]] = paddr[lower]
kp = np.full(slots, 255, np.uint8)
kp[addr[lower]] = kk[pk][lower]
rng = np.random.default_rng(0)
vals = rng.uniform(-1, 1, (slots, 3, 3))
vals[addr[lower]] = np.transpose(vals[paddr[lower]], (0, 2, 1))
vals = np.ascontiguousarray(vals.reshape(-1))
x = rng.uniform(-1, 1, 3 * p)
y = np.zeros(9 * p)
t = np.zeros(8, np.float32)
rc = lib.symlab_run(C.c_int(p), C.c_int64(slots), sbase.ctypes.data_as(C.c_void_p),
                    row_len.astype(np.int32).ctypes.data_as(C.c_void_p), cols.ctypes.data_as(C.c_void_p),
                    mirror.ctypes.data_as(C.c_void_p), kp.ctypes.data_as(C.c_void_p), vals.ctypes.data_as(C.c_void_p),
                    x.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), t.ctypes.data_as(C.c_void_p))
assert rc == 0, rc
y = y.reshape(3, -1)
nnz = len(r)
print(f"config {sys.argv[1] if len(sys.argv) > 1 else 'D'}: rows {p} nnzb {nnz} slots {slots} lower {int(lower.sum())}")
for m, name in enumerate(["plain", "mirror int32", "mirror k' byte"]):
    print(f"  {name:16s} {t[m]*1e3:7.1f} us  bitwise {np.array_equal(y[0], y[m])}")
