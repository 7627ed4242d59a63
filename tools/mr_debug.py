"""Debug driver: two ranks on cuda:0, repeated PCG solves on the assembled system."""
import os, subprocess, sys, socket
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))

def rank_main():
    import torch.distributed as dist
    from paper_2008_00409_b200 import weft, scenes
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    sc = scenes.layered_cloth(2, 14, seed=9)
    mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
    p = mesh.vertex_count
    eng = weft.Engine(2, world=world, rank=rank) if world > 1 else weft.Engine(2)
    eng.set_vertices(mesh.vertex_mass, sc.pinned)
    if world > 1: eng.attach_peers()
    eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
    eng.set_soup(p, sc.tris)
    x0 = sc.verts.reshape(-1).copy()
    v0 = np.random.default_rng(5).uniform(-0.05, 0.05, 3 * p)
    for k in range(3):
        eng.step_system(x0, v0, sc.dt)
        xa, rep = eng.pcg_solve(None, None, weft.PcgConfig(1e-8, 1000))
        print(f"rank {rank} solve {k}: its {rep.iterations} res {rep.rel_residual:.3e} sum {np.abs(xa).sum():.17g}", flush=True)
    eng.sim_set_state(x0, v0)
    params = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-8, 1000), weft.JAC_SPD)
    for k in range(3):
        try:
            r = eng.sim_step(params)
            print(f"rank {rank} step {k}: its {r.pcg_iterations} res {r.pcg_residual:.3e} dcd {r.dcd_candidates}", flush=True)
        except Exception as e:
            print(f"rank {rank} step {k}: {e}", flush=True)
            break
    dist.barrier()
    eng.close()
    dist.destroy_process_group()

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "rank":
        rank_main()
    else:
        world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
        ps = [subprocess.Popen([sys.executable, __file__, "rank"], env=dict(os.environ, RANK=str(r), WORLD_SIZE=str(world),
              MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))) for r in range(world)]
        for q in ps: q.wait(timeout=300)
