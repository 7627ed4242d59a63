"""How often three double atan2s agree on real hinge inputs.

For the bend elements of a scene (default config D: 3 x 525^2 layered cloth,
2.4 M hinges) at the rest state and at perturbed states (vertices moved by
up to `--amp` metres), forms each hinge's (s, c) exactly like
dihedral_angle (proj/src/elements.cpp:105-117) and compares
  glibc       math.atan2 (what the reference computes),
  cr          the library's correctly rounded atan2 (host build),
  cr_device   the same on the GPU (weft_gpu_hinge_atan2),
  cuda        CUDA's libdevice atan2 (torch.atan2 on a float64 CUDA tensor),
printing the disagreement rates as one JSON line.

  python tools/atan2_agreement.py [--config D] [--amp 1e-3] [--states 3]
"""
import argparse
import ctypes
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def hinge_sc(st, x):
    x0, x1, x2, x3 = (x[st[:, i]] for i in range(4))
    cross = lambda a, b: np.stack([a[:, 1] * b[:, 2] - a[:, 2] * b[:, 1], a[:, 2] * b[:, 0] - a[:, 0] * b[:, 2],
                                   a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]], 1)
    dot = lambda a, b: a[:, 0] * b[:, 0] + a[:, 1] * b[:, 1] + a[:, 2] * b[:, 2]
    e = x1 - x0
    na = cross(e, x2 - x0)
    nb = cross(x3 - x0, e)
    s = dot(cross(na, nb), e) / np.sqrt(dot(e, e))
    c = dot(na, nb)
    return np.ascontiguousarray(s), np.ascontiguousarray(c)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="D")
    ap.add_argument("--amp", type=float, default=1e-3)
    ap.add_argument("--states", type=int, default=3)
    args = ap.parse_args()
    from paper_2008_00409_b200 import scenes, weft
    sc = scenes.config(args.config, seed=1)
    mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
    elems = mesh.build_elements(tuple(sc.material))
    st = elems[elems["kind"] == 1]["stencil"]
    lib = weft.LIB
    p = lambda a: ctypes.c_void_p(a.ctypes.data)
    rng = np.random.default_rng(0)
    counts = {"hinges": 0, "cr_vs_glibc": 0, "cuda_vs_glibc": 0, "cuda_vs_cr": 0, "cr_device_vs_cr": 0}
    eng = None
    try:
        import torch
        gpu = torch.cuda.is_available()
    except ImportError:
        gpu = False
    if gpu:
        eng = weft.Engine(1)
    base = sc.verts.reshape(-1, 3)
    for k in range(args.states):
        x = base if k == 0 else base + rng.uniform(-args.amp, args.amp, base.shape)
        s, c = hinge_sc(st, x)
        glibc = np.array([math.atan2(a, b) for a, b in zip(s.tolist(), c.tolist())])
        cr = np.empty_like(s)
        assert lib.weft_hinge_atan2_host(ctypes.c_int64(len(s)), p(s), p(c), p(cr)) == 0
        counts["hinges"] += len(s)
        counts["cr_vs_glibc"] += int((cr != glibc).sum())
        if gpu:
            cu = torch.atan2(torch.from_numpy(s).cuda(), torch.from_numpy(c).cuda()).cpu().numpy()
            dev = np.empty_like(s)
            assert lib.weft_gpu_hinge_atan2(eng._ctx, ctypes.c_int64(len(s)), p(s), p(c), p(dev)) == 0
            counts["cuda_vs_glibc"] += int((cu != glibc).sum())
            counts["cuda_vs_cr"] += int((cu != cr).sum())
            counts["cr_device_vs_cr"] += int((dev != cr).sum())
    if eng is not None:
        eng.close()
    n = counts["hinges"]
    out = {"config": args.config, "states": args.states, "amp_m": args.amp, "gpu": gpu, **counts,
           "rate_cr_vs_glibc": counts["cr_vs_glibc"] / n}
    if gpu:
        out["rate_cuda_vs_glibc"] = counts["cuda_vs_glibc"] / n
    print(json.dumps(out))


if __name__ == "__main__":
    main()
