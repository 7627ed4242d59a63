"""Dev: runs the config trajectory from rest on the GPU and prints per-step
PCG iterations, candidate counts and max |v| (stability check of the bench
scene, paper_2008_00409_b200/scenes.py)."""
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_00409_b200 import scenes, weft  # noqa: E402


def main(config="D", steps=60):
    sc = scenes.config(config)
    mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
    elems = mesh.build_elements(sc.material, sc.gravity)
    p = mesh.vertex_count
    params = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-4, 400, weft.PRECOND_BLOCK_JACOBI),
                            weft.JAC_SPD)
    with weft.Engine(1) as eng:
        eng.set_vertices(mesh.vertex_mass, sc.pinned)
        eng.set_elements(elems)
        eng.set_soup(p, sc.tris)
        eng.sim_set_state(sc.verts.reshape(-1), np.zeros(3 * p))
        x, v = np.zeros(3 * p), np.zeros(3 * p)
        for k in range(steps):
            r = eng.sim_step(params)
            eng.sim_get_state(x, v)
            print(k, r.pcg_iterations, r.dcd_candidates, r.ccd_candidates, f"vmax {np.abs(v).max():.3g}",
                  f"ms {r.ms_broad + r.ms_assemble + r.ms_solve:.1f}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "D", int(sys.argv[2]) if len(sys.argv) > 2 else 60)
