"""One rank of a multi-process run of the hot path (TEST INFRASTRUCTURE,
driven by tests/test_gpu_multirank.py). Every rank builds the same seeded
problems, runs them as one rank of a group (Engine(n, world=W, rank=R)),
and saves the rows it owns; the test stitches the ranks together and
compares with a single-process run of the same partitions (bitwise).

    python tests/mp_rank.py OUT_DIR  (env: RANK, WORLD_SIZE, MASTER_ADDR,
                                      MASTER_PORT, WEFT_DEVICE, WEFT_PARTS)
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))


def problems():
    """The seeded inputs every rank (and the single-process check) uses."""
    from gen import random_block_csr, random_spd
    from paper_2008_00409_b200 import scenes

    rng = np.random.default_rng(77)
    spmv = random_block_csr(rng, 157, 4)
    x = rng.uniform(-2, 2, 3 * spmv.rows)
    spd = random_spd(rng, 23)
    b = rng.uniform(-1, 1, 3 * spd.rows)
    sc = scenes.layered_cloth(2, 14, seed=9)
    return dict(spmv=spmv, x=x, spd=spd, b=b, scene=sc)


def run(eng_factory, world, rank, attach, steps=3):
    """Runs every task on an engine from eng_factory(); returns a dict of
    results (full-length vectors: only this rank's rows are meaningful)."""
    from paper_2008_00409_b200 import weft

    pr = problems()
    out = {}
    # -- SpMV (spmv_pipelined)
    eng = eng_factory()
    s = pr["spmv"]
    eng.set_matrix(weft.BlockCsr(s.rows, s.row_ptr, s.cols, s.vals))
    attach(eng)
    out["spmv_y"] = eng.spmv_pipelined(None, pr["x"])
    out["spmv_y2"] = eng.spmv_pipelined(None, 0.5 * pr["x"])  # second call: sequence numbers advance
    engines = [eng]
    # -- PCG (pcg_solve)
    eng = eng_factory()
    s = pr["spd"]
    eng.set_matrix(weft.BlockCsr(s.rows, s.row_ptr, s.cols, s.vals))
    attach(eng)
    xs, rep = eng.pcg_solve(None, pr["b"], weft.PcgConfig(1e-10, 500))
    out["pcg_x"] = xs
    out["pcg_iterations"] = np.array(rep.iterations)
    out["pcg_residual"] = np.array(rep.rel_residual)
    out["pcg_hist"] = rep.residual_history
    engines.append(eng)
    # -- assembly + device-resident steps (step_system, PCG, broad phases)
    sc = pr["scene"]
    mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
    p = mesh.vertex_count
    eng = eng_factory()
    eng.set_vertices(mesh.vertex_mass, sc.pinned)
    attach(eng)
    eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
    eng.set_soup(p, sc.tris)
    x0 = sc.verts.reshape(-1).copy()
    rng = np.random.default_rng(5)
    v0 = rng.uniform(-0.05, 0.05, 3 * p)
    eng.step_system(x0, v0, sc.dt)
    m = eng.download_matrix()
    info = eng.rank_info()
    out["asm_first_row"] = np.array(info.first_row)
    out["asm_row_ptr"], out["asm_cols"], out["asm_vals"] = m.row_ptr, m.cols, m.vals
    out["asm_rhs"] = eng.download_rhs()
    # PCG on the assembled system (its own rhs)
    xa, rep = eng.pcg_solve(None, None, weft.PcgConfig(1e-8, 1000))
    out["asm_pcg_x"], out["asm_pcg_its"] = xa, np.array(rep.iterations)
    eng.sim_set_state(x0, v0)
    params = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-8, 3000), weft.JAC_SPD)
    dcd, ccd, its = [], [], []
    for _ in range(steps):
        try:
            r = eng.sim_step(params)
        except weft.Error as e:
            out["sim_error"] = np.array(str(e))
            break
        dcd.append(r.dcd_candidates)
        ccd.append(r.ccd_candidates)
        its.append(r.pcg_iterations)
    xg = np.zeros(3 * p)
    vg = np.zeros(3 * p)
    eng.sim_get_state(xg, vg)
    out["sim_x"], out["sim_v"] = xg, vg
    out["sim_dcd"], out["sim_ccd"], out["sim_its"] = np.array(dcd), np.array(ccd), np.array(its)
    engines.append(eng)
    # -- the whole Simulator::step_impl (driver.cpp:96-215): DCD collide
    # (shares merged over the ranks), contact elements, step_system with the
    # contacts (inter-layer contact columns cross the partition cut: the
    # dynamic contact halo of the PCG), CCD collide, impact zones
    eng = eng_factory()
    eng.set_vertices(mesh.vertex_mass, sc.pinned)
    attach(eng)
    eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
    eng.set_soup(p, sc.tris)
    # from rest: the pinned layers stay untangled (WEFT_CON_V0=1: the
    # jittered v0, whose tangled layers end in ZoneFailure — the error path)
    eng.sim_set_state(x0, v0 if os.environ.get("WEFT_CON_V0") == "1" else np.zeros_like(x0))
    params = weft.SimParams(sc.dt, 2 * sc.thickness, 1.5, weft.PcgConfig(1e-8, 3000), weft.JAC_SPD, contacts=1,
                            zones=1)
    rows, wall = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        try:
            r = eng.sim_step(params)
        except weft.Error as e:
            out["con_error"] = np.array(str(e))
            wall.append(time.perf_counter() - t0)
            break
        wall.append(time.perf_counter() - t0)
        rows.append([r.proximities, r.contact_elements, r.impacts, r.zone_count, r.pcg_iterations,
                     r.dcd_candidates, r.ccd_candidates])
    eng.sim_get_state(xg, vg)
    out["con_x"], out["con_v"], out["con_counts"] = xg.copy(), vg.copy(), np.array(rows, dtype=np.int64)
    out["con_wall_s"] = np.array(wall)
    engines.append(eng)
    return out, engines


def main():
    import torch.distributed as dist

    from paper_2008_00409_b200 import weft

    out_dir = sys.argv[1]
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    device = int(os.environ.get("WEFT_DEVICE", "0"))
    parts = int(os.environ.get("WEFT_PARTS", str(world)))
    dist.init_process_group("gloo")
    res, engines = run(lambda: weft.Engine(parts, cuda_device=device, world=world, rank=rank), world, rank,
                       lambda e: e.attach_peers())
    dist.barrier()  # nobody unmaps a window a peer may still read
    for e in engines:
        e.close()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
