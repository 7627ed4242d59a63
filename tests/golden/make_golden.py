"""Generates the golden fixtures under tests/golden/ from the COMPILED
REFERENCE (oracle/_ref/libweft_ref.so, built from the unmodified sources in
/root/reference by `make -C oracle ref`). Run here, where the reference
exists; the .npz files are committed so GPU boxes (no /root/reference) can
check against the reference's own outputs.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_bindings import CONTINUOUS, DISCRETE, JAC_EXACT, JAC_SPD, REF  # noqa: E402
from problems import cloth_problem  # noqa: E402


ZONE_REPORT = ("outer_iterations", "zone_count", "max_zone_vertices", "impacts_resolved", "first_round_impacts")
# ("two", seed, side) | ("layered", layers, nx, seed, amplitude in grid spacings)
ZONE_CASES = [("two", 52, 6), ("two", 41, 8), ("two", 43, 8), ("layered", 2, 10, 8, 0.6), ("layered", 2, 16, 3, 0.5),
              ("layered", 3, 12, 5, 0.4), ("layered", 3, 30, 2, 0.6)]


def zone_case(case):
    """Inputs of a resolve_zones case: nv, tris, x_begin, x_candidate, mass,
    movable, thickness, the 8 ZoneSolveParams values."""
    if case[0] == "two":
        nv, tris, x0, x1 = REF.two_cloth_scene(case[1], case[2])
        # test_response.cpp:218-240: mass 0.05, default parameters
        return nv, tris, x0, x1, np.full(nv, 0.05), np.ones(nv, np.uint8), 0.005, [0.0025, 10.0, 1e-8, 25, 64, 10, 3,
                                                                                  8.0]
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_2008_00409_b200 import scenes
    _, layers, nx, seed, amp = case
    sc = scenes.layered_cloth(layers, nx, seed=seed)
    x0 = sc.verts.reshape(-1).copy()
    x1 = x0 + np.random.default_rng(4).uniform(-amp, amp, x0.shape) * sc.spacing
    nv = len(sc.verts)
    return (nv, sc.tris, x0, x1, np.full(nv, 1e-3), (1 - sc.pinned).astype(np.uint8), sc.thickness,
            [0.5 * sc.thickness, 10.0, 1e-8, 25, 64, 10, 3, 8.0])


def main():
    assert REF is not None, "oracle/_ref/libweft_ref.so missing: make -C oracle ref"
    # assembly: random_cloth problems (test_assembly.cpp:55-71 recipe) with
    # contacts / drag, both Jacobian modes, reference fill_matrix at n = 2.
    for k, (seed, contacts, drag) in enumerate([(11, 0, False), (12, 5, True), (13, 9, False), (14, 3, True)]):
        pr = cloth_problem(REF, seed, 7, contacts=contacts, drag=drag)
        out = dict(elems=pr["elems"].view(np.uint8), x=pr["x"], x_adv=pr["x_adv"], v=pr["v"], mass=pr["mass"],
                   pinned=pr["pinned"], dt=np.array(pr["dt"]))
        for mode, tag in ((JAC_SPD, "spd"), (JAC_EXACT, "exact")):
            s = REF.fill_matrix(pr["elems"], pr["x"], pr["x_adv"], pr["v"], pr["mass"], pr["pinned"], pr["dt"], mode, n=2)
            out[f"{tag}_row_ptr"], out[f"{tag}_cols"], out[f"{tag}_vals"], out[f"{tag}_rhs"] = s.row_ptr, s.cols, s.vals, s.rhs
        x, rep = REF.pcg(REF.fill_matrix(pr["elems"], pr["x"], pr["x_adv"], pr["v"], pr["mass"], pr["pinned"], pr["dt"]),
                         out["spd_rhs"], 2, tol=1e-10)
        out["pcg_x"], out["pcg_iterations"] = x, np.array(rep["iterations"])
        np.savez_compressed(os.path.join(HERE, f"assembly_{k}.npz"), **out)
    # broad phase: random_two_cloth_scene (collision_oracle.cpp:110-138).
    for k, seed in enumerate([41, 42, 43]):
        nv, tris, x0, x1 = REF.two_cloth_scene(seed, 8)
        out = dict(nv=np.array(nv), tris=tris, x0=x0, x1=x1)
        for mode, tag in ((DISCRETE, "dcd"), (CONTINUOUS, "ccd")):
            g = REF.build_grid(nv, tris, x0, x1, mode=mode, thickness=0.01)
            out[f"{tag}_cell_size"] = np.array(g.cell_size)
            for f in ("tri_boxes", "cell_keys", "cell_offsets", "cell_tris", "prefix"):
                out[f"{tag}_{f}"] = getattr(g, f)
            out[f"{tag}_pairs"] = REF.candidates(g)
            REF.free_grid(g)
        np.savez_compressed(os.path.join(HERE, f"grid_{k}.npz"), **out)
    # narrow phase: collide (collision.cpp:391-417) on random_two_cloth_scene
    # (DCD at two thicknesses, CCD) and on a pinned layered cloth.
    k = 0
    for seed, mode, th in [(41, DISCRETE, 0.05), (43, DISCRETE, 0.2), (41, CONTINUOUS, 0.01), (43, CONTINUOUS, 0.01)]:
        nv, tris, x0, x1 = REF.two_cloth_scene(seed, 8)
        kab, vals = REF.collide(nv, tris, x0, x1, mode, th)
        np.savez_compressed(os.path.join(HERE, f"narrow_{k}.npz"), nv=np.array(nv), tris=tris, x0=x0, x1=x1,
                            mode=np.array(mode), thickness=np.array(th), movable=np.ones(nv, np.uint8), kab=kab,
                            vals=vals)
        k += 1
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_2008_00409_b200 import scenes
    sc = scenes.layered_cloth(2, 10, seed=8)
    x0 = sc.verts.reshape(-1)
    x1 = x0 + np.random.default_rng(4).uniform(-0.6, 0.6, x0.shape) * sc.spacing
    mv = (1 - sc.pinned).astype(np.uint8)
    for mode in (DISCRETE, CONTINUOUS):
        kab, vals = REF.collide(len(sc.verts), sc.tris, x0, x1, mode, 2 * sc.thickness, movable=mv)
        np.savez_compressed(os.path.join(HERE, f"narrow_{k}.npz"), nv=np.array(len(sc.verts)), tris=sc.tris, x0=x0,
                            x1=x1, mode=np.array(mode), thickness=np.array(2 * sc.thickness), movable=mv, kab=kab,
                            vals=vals)
        k += 1
    # impact zones: resolve_zones (response.cpp:338-400) on random_two_cloth_scene
    # (ZoneFailure cases: the positions left behind and the message are pinned
    # too) and on pinned layered cloths with a perturbed candidate.
    for k, case in enumerate(ZONE_CASES):
        nv, tris, x0, x1, mass, mv, th, zp = zone_case(case)
        st, msg, xc, rep = REF.resolve_zones(nv, tris, mass, x0, x1, thickness=th, devices=2, params=zp, movable=mv)
        np.savez_compressed(os.path.join(HERE, f"zones_{k}.npz"), nv=np.array(nv), tris=tris, x0=x0, x1=x1,
                            mass=mass, movable=mv, thickness=np.array(th), params=np.asarray(zp), status=np.array(st),
                            message=np.array(msg), x_out=xc, report=np.array([rep[f] for f in ZONE_REPORT]))
    # scenes (scene.cpp) run by the reference Simulator (driver.cpp:55-215):
    # per-frame counts and the final state (tests/scenes_gen.py scenes)
    from oracle_bindings import RefError, RefScene
    from scenes_gen import SCENES, scene_text
    for name in SCENES:
        rs = RefScene(REF, text=scene_text(name))
        frames, failure = [], ""
        for _ in range(int(rs.config()["frames"])):
            try:
                r = rs.step()
            except RefError as e:  # the scene's last frame fails in the reference (config_A)
                failure = str(e)
                break
            frames.append([r["pcg_iterations"], r["proximities"], r["contacts"], r["impacts"], r["zone_count"],
                           r["zone_outer"]])
        x, v = rs.state()
        extra = {"failure": np.array(failure)} if failure else {"obj": np.array(rs.save_obj())}
        np.savez_compressed(os.path.join(HERE, f"scene_{name}.npz"), text=np.array(scene_text(name)),
                            frames=np.array(frames, np.int64), x=x, v=v, **extra)
        rs.close()
    # SpMV: oracle::random_bell (sparse_oracle.cpp:7-23), pipelined at n = 1, 2, 4.
    for k, (seed, rows) in enumerate([(5, 7), (6, 40)]):
        s = REF.random_bell(seed, rows, 3)
        x = np.random.default_rng(seed).uniform(-2, 2, 3 * rows)
        out = dict(rows=np.array(rows), row_ptr=s.row_ptr, cols=s.cols, vals=s.vals, x=x)
        for n in (1, 2, 4):
            out[f"y{n}"] = REF.spmv(s, x, n)
        np.savez_compressed(os.path.join(HERE, f"spmv_{k}.npz"), **out)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
