"""The opt-in mirrored persistent solve (WEFT_PCG_MIRROR=1, csrc/sparse.cu
k_pcg_persistent<..., kMir>): lower-triangle blocks that are bitwise the
transpose of their upper twin are read from the twin. The products are the
same bits; only the wavefront order of the per-warp partial dot products
differs from the default kernel. Each variant runs in its own process (the
switch is read once per process)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2008_00409_b200 import scenes, weft
sc = scenes.config("B", seed=3)
mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
p = mesh.vertex_count
eng = weft.Engine(1)
eng.set_vertices(mesh.vertex_mass, sc.pinned)
eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
eng.set_soup(p, sc.tris)
x0 = sc.verts.reshape(-1).copy()
eng.sim_set_state(x0, np.zeros_like(x0))
prm = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-8, 2000), weft.JAC_SPD)
its = [eng.sim_step(prm).pcg_iterations for _ in range(3)]
x, v = np.zeros(3 * p), np.zeros(3 * p)
eng.sim_get_state(x, v)
np.save(sys.argv[2], np.concatenate([x, v]))
print(json.dumps({"its": its}))
"""


def run(tmp_path, tag, env):
    out = str(tmp_path / f"{tag}.npy")
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, out], env={**os.environ, **env}, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    import numpy as np
    return json.loads(r.stdout.strip().splitlines()[-1])["its"], np.load(out)


def test_mirrored_solve_matches_default(tmp_path):
    import numpy as np
    its_d, s_d = run(tmp_path, "default", {"WEFT_PCG_MIRROR": "0"})
    its_m, s_m = run(tmp_path, "mirror", {"WEFT_PCG_MIRROR": "1"})
    assert all(abs(a - b) <= 1 for a, b in zip(its_d, its_m)), (its_d, its_m)
    scale = np.abs(s_d).max()
    assert np.abs(s_m - s_d).max() <= 1e-9 * scale
