"""Device-resident hot-path step vs the compiled reference's step
(oracle/ref_harness.cpp ref_sim_step): positions and velocities within
1e-5 relative after N steps (north_star tolerance), broad-phase candidate
counts equal."""
import numpy as np
import pytest

from oracle_bindings import REF, RefSim

pytestmark = [pytest.mark.gpu, pytest.mark.ref]


@pytest.fixture(scope="module")
def weft():
    from paper_2008_00409_b200 import weft as w
    return w


@pytest.mark.parametrize("layers,nx,steps,tol", [(1, 24, 6, 1e-9), (3, 16, 5, 1e-9), (2, 20, 4, 1e-4)])
def test_sim_steps_match_reference(weft, layers, nx, steps, tol):
    from paper_2008_00409_b200 import scenes
    sc = scenes.layered_cloth(layers, nx, seed=3)
    mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
    p = mesh.vertex_count
    eng = weft.Engine(1)
    eng.set_vertices(mesh.vertex_mass, sc.pinned)
    eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
    eng.set_soup(p, sc.tris)
    x0 = sc.verts.reshape(-1).copy()
    eng.sim_set_state(x0, np.zeros_like(x0))
    ref = RefSim(REF, sc.verts, sc.tris, sc.pinned, sc.density, sc.material, 2)
    params = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(tol, 3000), weft.JAC_SPD)
    for k in range(steps):
        rg = eng.sim_step(params)
        rr = ref.step(sc.dt, sc.thickness, tol=tol, max_it=3000)
        if k == 0:
            assert rg.dcd_candidates == rr["dcd_candidates"]
        assert abs(rg.pcg_iterations - rr["pcg_iterations"]) <= max(2, 0.02 * rr["pcg_iterations"])
    xg = np.zeros(3 * p)
    vg = np.zeros(3 * p)
    eng.sim_get_state(xg, vg)
    xr, vr = ref.get_state()
    assert np.abs(xg - xr).max() <= 1e-5 * np.abs(xr).max()
    assert np.abs(vg - vr).max() <= 1e-5 * max(np.abs(vr).max(), 1e-12) + 1e-12
    ref.close()
    eng.close()
