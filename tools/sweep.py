"""Size sweep on one GPU (BASELINE.json configs[4]: 0.5M-10M triangles): for
each config, the bench's hot-path step (DCD + count, assembly, PCG, CCD +
count) along the trajectory from rest (3 warm-up steps, then 6 timed with
CUDA events), the persistent PCG kernel's HBM roofline, the narrow-phase
DCD time, and the compiled reference's CPU step on the same trajectory
(oracle/_ref, Engine(largest power of two <= host cores); 1 warm-up step,
up to 2 timed within a wall budget). One JSON line per config.

    python tools/sweep.py [A E05 B ...] > profiles/r02_sweep_1gpu.jsonl
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_00409_b200 import scenes, weft  # noqa: E402


def peak():
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        return float(json.load(f)["hbm_gbs"])


def run(cfg: str, steps: int = 6, warmup: int = 3):
    sc = scenes.config(cfg)
    mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
    p = mesh.vertex_count
    eng = weft.Engine(1)
    eng.set_vertices(mesh.vertex_mass, sc.pinned)
    eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
    eng.set_soup(p, sc.tris)
    x0 = sc.verts.reshape(-1).copy()
    eng.sim_set_state(x0, np.zeros_like(x0))
    prm = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-4, 400), weft.JAC_SPD)
    stream = torch.cuda.ExternalStream(eng.stream())
    for _ in range(warmup):
        eng.sim_step(prm)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    reps = [eng.sim_step(prm) for _ in range(steps)]
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    eng.profile(True)
    eng.sim_step(prm)
    st = eng.stats()
    eng.profile(False)
    xs = torch.empty(3 * p, dtype=torch.float64, device="cuda")
    vs = torch.empty(3 * p, dtype=torch.float64, device="cuda")
    eng.sim_get_state(xs, vs)
    info = eng.matrix_info()
    pcg_gbs = st.pcg_bytes / (st.pcg_ms * 1e-3) / 1e9 if st.pcg_solves else None
    eng.set_soup_movable(1 - sc.pinned)
    eng.collide(xs, None, weft.DISCRETE, sc.thickness)
    n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0.record(stream)
    kab, _ = eng.collide(xs, None, weft.DISCRETE, sc.thickness)
    n1.record(stream)
    n1.synchronize()
    out = {
        "config": cfg, "layers": sc.layers, "nx": sc.nx, "triangles": sc.tri_count, "vertices": p,
        "nnzb": info.nnzb, "steps_per_s": 1e3 / ms, "ms_per_step": ms,
        "stage_ms": {"broad": statistics.mean(r.ms_broad for r in reps),
                     "assemble": statistics.mean(r.ms_assemble for r in reps),
                     "solve": statistics.mean(r.ms_solve for r in reps)},
        "pcg_iterations": statistics.mean(r.pcg_iterations for r in reps),
        "pcg_kernel_gbs": pcg_gbs, "pcg_roofline_frac": pcg_gbs / peak() if pcg_gbs else None,
        "narrow_dcd_ms": n0.elapsed_time(n1), "dcd_hits": int(len(kab)),
        "gpu_mem_gb": torch.cuda.mem_get_info()[1] / 1e9 - torch.cuda.mem_get_info()[0] / 1e9,
    }
    eng.close()
    if REF_BUDGET > 0:
        from bench import run_reference_steps
        sec, n, rinfo = run_reference_steps(sc, 2, 1, REF_BUDGET)
        if sec:
            out["cpu_reference"] = {"steps_per_s": 1.0 / sec, "timed_steps": n, "threads": 2 * rinfo["devices"],
                                    "engine_devices": rinfo["devices"], "cpu_model": rinfo["cpu_model"],
                                    "pcg_iterations": rinfo["pcg_iterations"]}
            out["gpu_over_cpu_reference"] = (1e3 / ms) * sec
        else:
            out["cpu_reference"] = rinfo
    return out


REF_BUDGET = float(os.environ.get("SWEEP_REF_BUDGET_S", "150"))

if __name__ == "__main__":
    cfgs = sys.argv[1:] or ["A", "E05", "B", "C", "D", "E3", "E5", "E10"]
    for cfg in cfgs:
        try:
            print(json.dumps(run(cfg)), flush=True)
        except Exception as e:  # a config whose scene diverges must not stop the sweep
            print(json.dumps({"config": cfg, "error": str(e)}), flush=True)
