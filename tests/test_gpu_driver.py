"""The known answers of the reference's driver tests
(proj/tests/test_driver.cpp:23-198) on the GPU Simulator
(paper_2008_00409_b200/scene.py -> one weft_gpu_sim_step per frame)."""
import numpy as np
import pytest

from oracle_bindings import CONTINUOUS, REF

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_2008_00409_b200 import scene, weft
    return scene, weft


def quiet_scene(S, weft, nx, w, origin, devices=1, pins=(), gravity=(0.0, 0.0, -9.81), obstacles=(), **coll):
    """quiet_config (test_driver.cpp:14-19): dt 1/150, the given devices."""
    cfg = S.SimConfig(dt=1.0 / 150.0, devices=devices, gravity=gravity)
    cfg.material.density = 0.2
    for k, v in coll.items():
        setattr(cfg, k, v)
    cloth = weft.ClothMesh.grid(nx, nx, w, w, origin, 0.2)
    pinned = np.zeros(nx * nx, np.uint8)
    pinned[list(pins)] = 1
    return S.Scene("t", cloth, pinned, list(obstacles), cfg, (nx, nx))


def test_flat_cloth_without_gravity_stays_at_rest(mods):
    """test_driver.cpp:23-38."""
    S, weft = mods
    sc = quiet_scene(S, weft, 6, 0.3, (0.0, 0.0, 0.0), gravity=(0.0, 0.0, 0.0))
    sim = S.Simulator(sc)
    for _ in range(3):
        assert sim.step().committed
    x, v = sim.state()
    assert np.abs(x - sc.cloth.rest.reshape(-1, 3)).max() <= 1e-12 and np.abs(v).max() <= 1e-12
    sim.close()


def test_single_free_vertex_gains_exactly_dt_g(mods):
    """test_driver.cpp:40-52: one vertex of mass 1, dt 1/64, g = -10:
    after 8 steps v_z == 8 * dt * -10 exactly."""
    _, weft = mods
    e = np.zeros(1, weft.ELEMENT_DTYPE)
    e["kind"] = weft.EXTERNAL
    e["stencil_size"] = 1
    e["stencil"] = (0, -1, -1, -1)
    e["data"][0, :4] = (0.0, 0.0, 1.0 * -10.0, 0.0)  # m g, no drag (physics.cpp:45-60)
    with weft.Engine(1) as eng:
        eng.set_vertices(np.array([1.0]), np.array([0], np.uint8))
        eng.set_elements(e)
        eng.set_soup(1, np.zeros((0, 3), np.int32))
        eng.sim_set_state(np.zeros(3), np.zeros(3))
        prm = weft.SimParams(1.0 / 64.0, 0.005, 1.5, weft.PcgConfig(1e-4, 400), weft.JAC_SPD, contacts=1, zones=1)
        for _ in range(8):
            eng.sim_step(prm)
        x, v = np.zeros(3), np.zeros(3)
        eng.sim_get_state(x, v)
    assert v[2] == 8 * (1.0 / 64.0) * -10.0 and v[0] == 0.0


@pytest.mark.parametrize("n", [1, 2])
def test_identical_runs_identical_trajectories(mods, n):
    """test_driver.cpp:100-117 (bitwise)."""
    S, weft = mods
    finals = []
    for _ in range(2):
        sim = S.Simulator(quiet_scene(S, weft, 8, 0.3, (0.0, 0.0, 0.2), devices=n, pins=(56, 63)))
        for _ in range(5):
            sim.step()
        finals.append(sim.state()[0])
        sim.close()
    assert np.array_equal(finals[0], finals[1])


def test_device_count_changes_timings_not_trajectories(mods):
    """test_driver.cpp:119-136: Engine(1) vs Engine(4) within 1e-6."""
    S, weft = mods
    finals = []
    for n in (1, 4):
        sim = S.Simulator(quiet_scene(S, weft, 8, 0.3, (0.0, 0.0, 0.2), devices=n, pins=(56, 63)))
        for _ in range(10):
            sim.step()
        finals.append(sim.state()[0])
        sim.close()
    scale = np.maximum(1.0, np.linalg.norm(finals[0], axis=1))
    assert (np.linalg.norm(finals[0] - finals[1], axis=1) / scale).max() <= 1e-6


def test_cloth_on_sphere_commits_only_penetration_free_frames(mods):
    """test_driver.cpp:155-198: every committed frame passes a CCD audit of
    the soup (the compiled reference's collide where available, else the
    GPU's), zone rounds <= 10, and the cloth ends on the sphere."""
    S, weft = mods
    sphere = S.Obstacle(S.make_uv_sphere((0.0, 0.0, -0.05), 0.1, 10, 14))
    sc = quiet_scene(S, weft, 12, 0.4, (-0.2, -0.2, 0.12), devices=2, obstacles=[sphere], thickness=0.008,
                     stiffness_scale=1.0)
    sim = S.Simulator(sc)
    obs = sphere.positions_at(0.0)
    tris = np.concatenate([sc.cloth.triangles, sphere.shape.triangles + 144]).astype(np.int32)
    nv = 144 + len(obs)
    movable = np.concatenate([np.ones(144, np.uint8), np.zeros(len(obs), np.uint8)])
    with weft.Engine(1) as audit:
        audit.set_soup(nv, tris)
        audit.set_soup_movable(movable)
        for _ in range(12):
            before = sim.state()[0]
            rep = sim.step()
            assert rep.committed and rep.zone_outer <= 10
            after = sim.state()[0]
            x0 = np.concatenate([before, obs]).reshape(-1)
            x1 = np.concatenate([after, obs]).reshape(-1)
            if REF is not None:
                kab, _ = REF.collide(nv, tris, x0, x1, CONTINUOUS, 0.008, movable=movable)
            else:
                kab, _ = audit.collide(x0, x1, weft.CONTINUOUS, 0.008)
            assert len(kab) == 0
    assert sim.state()[0][77, 2] < 0.12
    sim.close()
