"""CPU-only checks of the drop-in boundary: libweft_gpu.so loads without a
GPU and exports every entry point include/*.h declares (no compute calls)."""
import ctypes
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2008_00409_b200", "libweft_gpu.so")

DECL = re.compile(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(weft_[a-z0-9_]+)\s*\(", re.M)


def declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        with open(h) as f:
            src = re.sub(r"/\*.*?\*/", "", f.read(), flags=re.S)
        names.update(DECL.findall(src))
    return sorted(names)


def test_headers_declare_entry_points():
    names = declared()
    assert "weft_gpu_create" in names and "weft_gpu_pcg" in names and "weft_mesh_build" in names
    assert len(names) >= 30


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, f"declared in include/*.h but not exported: {missing}"


def test_pure_host_entry_points():
    # Entry points that need no device: partitions, work queues, split.
    lib = ctypes.CDLL(LIB)
    b = (ctypes.c_int32 * 4)()
    e = (ctypes.c_int32 * 4)()
    assert lib.weft_make_partitions(10, 4, b, e) == 0
    assert list(b) == [0, 3, 6, 8] and list(e) == [3, 6, 8, 10]  # exec.cpp:10-23
    peer = (ctypes.c_int32 * 12)()
    vec = (ctypes.c_int32 * 12)()
    assert lib.weft_work_queues(4, peer, vec) == 0
    # test_topology.cpp:37-40: Q0 = [(1,1),(2,2),(1,3)]
    assert list(zip(peer[0:3], vec[0:3])) == [(1, 1), (2, 2), (1, 3)]
    assert lib.weft_work_queues(3, peer, vec) != 0  # not a power of two
    lib.weft_gpu_last_error.restype = ctypes.c_char_p
    assert b"power of two" in lib.weft_gpu_last_error().lower() or lib.weft_gpu_last_error()
    bb = (ctypes.c_int64 * 3)()
    ee = (ctypes.c_int64 * 3)()
    assert lib.weft_split_workload(ctypes.c_int64(10), 3, bb, ee) == 0
    assert [ee[i] - bb[i] for i in range(3)] in ([4, 3, 3], [3, 3, 4], [3, 4, 3])
    assert bb[0] == 0 and ee[2] == 10
