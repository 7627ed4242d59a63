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


@pytest.mark.parametrize("layers,nx,steps", [(2, 16, 3), (3, 12, 3)])
def test_sim_steps_with_contacts_match_reference(weft, layers, nx, steps):
    """Simulator::step_impl without impact zones (driver.cpp:132-149 +
    candidate update + CCD): DCD narrow phase -> proximities_to_elements ->
    step_system with contacts -> PCG, on the device, vs the compiled
    reference (oracle/ref_harness.cpp ref_sim_step_contacts)."""
    from paper_2008_00409_b200 import scenes
    sc = scenes.layered_cloth(layers, nx, seed=3)
    th = 2 * sc.thickness  # layers and in-layer features within reach: many contacts
    mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
    p = mesh.vertex_count
    eng = weft.Engine(1)
    eng.set_vertices(mesh.vertex_mass, sc.pinned)
    eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
    eng.set_soup(p, sc.tris)
    x0 = sc.verts.reshape(-1).copy()
    eng.sim_set_state(x0, np.zeros_like(x0))
    ref = RefSim(REF, sc.verts, sc.tris, sc.pinned, sc.density, sc.material, 2)
    params = weft.SimParams(sc.dt, th, 1.5, weft.PcgConfig(1e-9, 3000), weft.JAC_SPD, contacts=1)
    for k in range(steps):
        rg = eng.sim_step(params)
        rr = ref.step_contacts(sc.dt, th, tol=1e-9, max_it=3000)
        assert rg.proximities == rr["proximities"] and rg.contact_elements == rr["contacts"]
        assert rr["contacts"] > 100
        assert rg.impacts == rr["impacts"]
        # the stiffer contact system at tol 1e-9 amplifies the dot-product
        # association difference (tree vs sequential sums) into a few
        # iterations; the state tolerance below is the bar
        assert abs(rg.pcg_iterations - rr["pcg_iterations"]) <= max(2, 0.05 * rr["pcg_iterations"])
    xg = np.zeros(3 * p)
    vg = np.zeros(3 * p)
    eng.sim_get_state(xg, vg)
    xr, vr = ref.get_state()
    assert np.abs(xg - xr).max() <= 1e-5 * np.abs(xr).max()
    assert np.abs(vg - vr).max() <= 1e-5 * max(np.abs(vr).max(), 1e-12) + 1e-12
    # back to the hot-path step: no stale contacts
    r = eng.sim_step(weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-6, 3000), weft.JAC_SPD))
    assert r.contact_elements == 0 and r.pcg_converged
    ref.close()
    eng.close()


def test_sim_step_io_equals_set_step_get(weft):
    """weft_gpu_sim_step_io (copies overlapped with the broad phases) gives
    bitwise the results of sim_set_state + sim_step + sim_get_state."""
    from paper_2008_00409_b200 import scenes
    sc = scenes.layered_cloth(2, 24, seed=4)
    mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
    p = mesh.vertex_count
    x0 = sc.verts.reshape(-1).copy()
    v0 = np.random.default_rng(1).uniform(-0.01, 0.01, 3 * p)
    prm = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-8, 2000), weft.JAC_SPD)
    outs = []
    for io in (False, True):
        eng = weft.Engine(1)
        eng.set_vertices(mesh.vertex_mass, sc.pinned)
        eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
        eng.set_soup(p, sc.tris)
        eng.sim_set_state(x0, v0)
        x, v = x0.copy(), v0.copy()
        xo, vo = np.zeros(3 * p), np.zeros(3 * p)
        reps = []
        for _ in range(3):
            if io:
                reps.append(eng.sim_step_io(x, v, prm, xo, vo))
            else:
                eng.sim_set_state(x, v)
                reps.append(eng.sim_step(prm))
                eng.sim_get_state(xo, vo)
            x, v = xo.copy(), vo.copy()
        outs.append((x, v, [(r.pcg_iterations, r.dcd_candidates, r.ccd_candidates) for r in reps]))
        eng.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]
