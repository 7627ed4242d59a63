"""Scene files and mesh I/O vs the compiled reference:
parse_scene / load_scene (scene.cpp:45-178), the mesh generators and OBJ
I/O (mesh.cpp:187-337), Obstacle::positions_at (driver.cpp:22-43) and
RunReport::write_csv (scene.cpp:180-190). Host logic: runs on CPU."""
import glob
import io
import os

import numpy as np
import pytest

from oracle_bindings import REF, RefError, RefScene
from scenes_gen import SCENES, scene_text

REF_SCENES = sorted(glob.glob("/root/reference/proj/scenes/*.json"))


@pytest.fixture(scope="module")
def S():
    from paper_2008_00409_b200 import scene
    return scene


def config_of(sc):
    c, m = sc.config, sc.config.material
    return [c.dt, c.frames, c.devices, *c.gravity, *c.wind, c.seed, *m.as_tuple(), c.thickness, c.cell_scale,
            c.stiffness_scale, c.friction, c.clearance_fraction, c.contact_damping, c.rel_tolerance, c.max_iterations,
            1.0 if c.preconditioner == "block-jacobi" else 0.0, c.zones.outer_cap, c.zones.initial_penalty,
            1.0 if c.precision == "double" else 0.0]


def assert_same_scene(S, sc, rs):
    assert np.array_equal(np.array(config_of(sc), float), np.array(list(rs.config().values())))
    v, t, pin = rs.cloth()
    assert np.array_equal(sc.cloth.rest, v) and np.array_equal(sc.cloth.triangles, t)
    assert np.array_equal(sc.pinned, pin)
    assert len(sc.obstacles) == rs.nobs
    for o, ob in enumerate(sc.obstacles):
        for t_ in (0.0, 0.013, 0.05, 0.1, 0.17, 0.3, 1.0):
            rv, rt = rs.obstacle(o, t_)
            assert np.array_equal(ob.positions_at(t_), rv) and np.array_equal(ob.shape.triangles, rt)
    s = io.StringIO()
    S.save_obj(s, sc.cloth.rest, sc.cloth.triangles)
    assert s.getvalue() == rs.save_obj()


@pytest.mark.ref
@pytest.mark.parametrize("name", sorted(SCENES))
def test_parse_scene_vs_reference(S, name):
    sc = S.parse_scene(scene_text(name))
    rs = RefScene(REF, text=scene_text(name))
    assert_same_scene(S, sc, rs)
    rs.close()


@pytest.mark.ref
@pytest.mark.parametrize("path", REF_SCENES, ids=[os.path.basename(p) for p in REF_SCENES])
def test_load_reference_scene_files(S, path):
    """The reference's own scene files, loaded by both."""
    sc = S.load_scene(path)
    rs = RefScene(REF, path=path)
    assert_same_scene(S, sc, rs)
    rs.close()


def test_scene_errors(S):
    """SceneError messages of parse_scene (scene.cpp:48-150)."""
    cases = [("{", "scene parse error"), ('{"name": "x"}', "scene has no 'cloth' section"),
             ('{"cloth": {}}', "cloth section needs 'grid' or 'obj'"),
             ('{"precision": "half", "cloth": {"grid": {}}}', "precision must be 'single' or 'double', got 'half'"),
             ('{"solver": {"preconditioner": "ilu"}, "cloth": {"grid": {}}}', "unknown preconditioner 'ilu'"),
             ('{"cloth": {"grid": {"nx": 3, "ny": 3}, "pins": [9]}}', None),
             ('{"cloth": {"grid": {"nx": 3, "ny": 3}, "pins": [-1]}}', "pin index out of range"),
             ('{"cloth": {"grid": {}}, "obstacles": [{"cone": {}}]}', "mesh spec needs one of: obj, sphere, funnel, box"),
             ('{"gravity": [1, 2], "cloth": {"grid": {}}}', "expected a 3-element array")]
    for text, msg in cases:
        if msg is None:
            continue
        with pytest.raises(S.SceneError) as ei:
            S.parse_scene(text)
        assert str(ei.value).startswith(msg)
        if REF is not None:
            with pytest.raises(RefError) as er:
                RefScene(REF, text=text)
            assert str(er.value).startswith(msg)


def test_obj_cloth_and_obstacle(S, tmp_path):
    """OBJ sources (mesh.cpp:278-318): quads fan-triangulated, i/t/n forms,
    negative (relative) indices, comments and blank lines."""
    obj = ["# quad sheet", "v 0 0 0", "v 0.1 0 0", "v 0.1 0.1 0.001", "v 0 0.1 0", "", "v 0.2 0 0", "v 0.2 0.1 0",
           "f 1/1/1 2/2/2 3/3/3 4/4/4", "f 2 5 6 3", "f -4 -1 -2"]
    (tmp_path / "sheet.obj").write_text("\n".join(obj) + "\n")
    (tmp_path / "tet.obj").write_text("v 0 0 -0.1\nv 0.1 0 -0.1\nv 0 0.1 -0.1\nv 0 0 -0.05\nf 1 2 3\nf 1 2 4\n"
                                      "f 2 3 4\nf 3 1 4\n")
    text = ('{"cloth": {"obj": "sheet.obj", "pins": [0, 3]}, "obstacles": [{"obj": "tet.obj", "keyframes": '
            '[{"time": 0, "translate": [0, 0, 0]}, {"time": 1, "translate": [0, 0, 0.5]}]}]}')
    (tmp_path / "s.json").write_text(text)
    sc = S.load_scene(str(tmp_path / "s.json"))
    assert sc.cloth.triangles.shape == (5, 3) and sc.pinned.tolist() == [1, 0, 0, 1, 0, 0]
    if REF is not None:
        rs = RefScene(REF, path=str(tmp_path / "s.json"))
        assert_same_scene(S, sc, rs)
        rs.close()
    (tmp_path / "bad.obj").write_text("v 0 0\n")
    with pytest.raises(S.SceneError, match="malformed vertex record"):
        S.load_obj(str(tmp_path / "bad.obj"))
    (tmp_path / "bad2.obj").write_text("v 0 0 0\nv 1 0 0\nf 1 2\n")
    with pytest.raises(S.SceneError, match="face with <3 vertices"):
        S.load_obj(str(tmp_path / "bad2.obj"))


def test_write_csv(S):
    """RunReport::write_csv (scene.cpp:180-190): header and precision(10)."""
    rep = S.RunReport(frames=[S.FrameReport(0, 0.0, 1.25, 0.5, 0.25, 0.0, 12, 9.87654321098e-05, 3, 2, 1, 1, 1, True),
                              S.FrameReport(1, 1 / 240, 2.0, 0.5, 0.25, 0.125, 13, 1e-4, 0, 0, 0, 0, 0, False)])
    out = io.StringIO()
    rep.write_csv(out)
    lines = out.getvalue().splitlines()
    assert lines[0] == ("frame,time,integrate_ms,broad_ms,narrow_ms,zones_ms,pcg_iterations,pcg_residual,"
                        "proximities,contacts,impacts,zones,zone_outer,committed")
    assert lines[1] == "0,0,1.25,0.5,0.25,0,12,9.876543211e-05,3,2,1,1,1,1"
    assert lines[2] == "1,0.004166666667,2,0.5,0.25,0.125,13,0.0001,0,0,0,0,0,0"
