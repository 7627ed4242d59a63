"""Dev probe: device time of the exact serial-order cell-size sum
(weft_gpu_test_serial_sum) on config D's DCD box diagonals, with the chunk
map fast path on / off, and with a large first term (no early crossings)."""
import ctypes as C
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_00409_b200 import scenes, weft  # noqa: E402

sc = scenes.config(sys.argv[1] if len(sys.argv) > 1 else "D")
p = sc.verts[sc.tris]
lo = p.min(1) - 0.5 * sc.thickness
hi = p.max(1) + 0.5 * sc.thickness
d = np.sqrt(((hi - lo) ** 2).sum(1))
lib = weft.LIB
with weft.Engine(1) as eng:
    for name, v in (("D diag", d), ("D diag, first term 1e3", np.concatenate([[1e3], d[1:]]))):
        for fast in (1, 0):
            ex, nv = C.c_double(), C.c_double()
            arr = np.ascontiguousarray(v)
            for rep in range(3):
                t0 = time.perf_counter()
                lib.weft_gpu_test_serial_sum(eng._ctx, C.c_int32(len(arr)), arr.ctypes.data_as(C.c_void_p),
                                             C.c_int32(fast), C.byref(ex), C.byref(nv))
                t1 = time.perf_counter()
            print(f"{name} fast={fast}: wall {1e3 * (t1 - t0):.2f} ms (incl. upload + naive serial sum) "
                  f"exact==naive {ex.value == nv.value / len(arr)}", flush=True)
