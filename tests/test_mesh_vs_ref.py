"""The product's one-time host mesh precompute (csrc/mesh.cpp) equals the
reference's ClothMesh/build_elements bit for bit. CPU only (loads the
library without touching a GPU)."""
import numpy as np
import pytest

from oracle_bindings import REF

pytestmark = pytest.mark.ref


@pytest.fixture(scope="module")
def weft():
    from paper_2008_00409_b200 import weft as w
    return w


def same_mesh(m, r):
    assert np.array_equal(m.rest, r["rest"])
    assert np.array_equal(m.triangles, r["tris"])
    assert np.array_equal(m.tri_rest, r["tri_rest"])
    assert np.array_equal(m.tri_degenerate, r["tri_degenerate"])
    assert np.array_equal(m.hinge_verts, r["hinge_verts"])
    assert np.array_equal(m.hinge_data, r["hinge_data"])
    assert np.array_equal(m.vertex_area, r["vertex_area"])
    assert np.array_equal(m.vertex_mass, r["vertex_mass"])


@pytest.mark.parametrize("nx,ny", [(2, 2), (3, 5), (10, 7), (40, 40)])
def test_grid_mesh(weft, nx, ny):
    m = weft.ClothMesh.grid(nx, ny, 0.5, 0.4, (-0.25, 0.1, 0.065), 0.15)
    r = REF.grid_mesh(nx, ny, 0.5, 0.4, (-0.25, 0.1, 0.065), 0.15)
    same_mesh(m, r)
    mat = (500.0, 450.0, 50.0, 2e-5, 0.15, 0.003, 0.3)
    e1 = m.build_elements(mat, (0, 0, -9.81), (0.1, 0.2, 0.0))
    e2 = REF.build_elements(r, mat, (0, 0, -9.81), (0.1, 0.2, 0.0))
    assert e1.tobytes() == e2.tobytes()
    REF.free_mesh(r)


@pytest.mark.parametrize("seed", range(6))
def test_jittered_mesh(weft, seed):
    r0 = REF.random_cloth(seed, 9)
    verts, tris = r0["rest"], r0["tris"]
    m = weft.ClothMesh.build(verts, tris, 0.2)
    r = REF.build_mesh(verts, tris, 0.2)
    same_mesh(m, r)
    assert m.build_elements().tobytes() == REF.build_elements(r).tobytes()
    REF.free_mesh(r)
    REF.free_mesh(r0)


def test_scene_errors(weft):
    with pytest.raises(weft.DimensionError, match="repeated vertex"):
        weft.ClothMesh.build(np.zeros(9), [[0, 0, 1]], 0.1)
    with pytest.raises(weft.DimensionError, match="non-manifold"):
        weft.ClothMesh.build(np.random.default_rng(0).random(15), [[0, 1, 2], [0, 1, 3], [0, 1, 4]], 0.1)
    with pytest.raises(weft.DimensionError, match="density"):
        weft.ClothMesh.build(np.zeros(9), [[0, 1, 2]], 0.0)
