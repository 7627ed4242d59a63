#!/usr/bin/env python
"""Hot-path benchmark (driver contract).

A step = one pass of the implicit-integration hot path over the synthetic
Kneel-scale cloth (BASELINE config D: 3 x 525^2 grid layers, 1,647,456
triangles, 826,875 vertices): DCD broad phase (grid + candidate pairs),
step_system assembly, block-Jacobi PCG (tol 1e-4), candidate update, CCD
broad phase (grid + candidate pairs), commit. Narrow phase / impact zones
are out of this tier's scope in both arms. The run is a
trajectory from rest: W warm-up steps, then K timed steps continuing it
(config material: paper_2008_00409_b200/scenes.py, stable for >= 40 steps).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

GPU arm: `value` is device-resident steps/s (CUDA events on the context's
stream, max over ranks); `e2e` is the same K steps through the C-ABI with the
state (x, v) copied from pinned host memory to the device and back every
step. Reference arm: the unmodified reference (oracle/_ref, compiled from
/root/reference) running the same trajectory on the host cores with
Engine(n) threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sim steps/sec at 1.65M-tri cloth, 1/2/4/8 B200; SpMV+assembly HBM GB/s vs peak"
UNIT = "steps/s"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["gpu", "reference"], default="gpu")
    ap.add_argument("--config", default="D", help="scene config (A/B/C/D, BASELINE.md §2)")
    ap.add_argument("--seed", type=int, default=20240810)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-narrow", action="store_true", help="skip the narrow-phase timing")
    ap.add_argument("--ref-budget-s", type=float, default=240.0, help="wall budget of the reference arm")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- clocks
class Clocks:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    every 10 ms in a background thread (short timed regions still get many
    samples), `nvidia-smi -lms 100` when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks.mem,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, device: int):
        import threading
        self.p = None
        self.sm, self.mx, self.reasons = [], [], set()
        self.stop_evt = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def run():
                while not self.stop_evt.is_set():
                    self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                    self.mx.append(float(mx))
                    bits = get_reasons(h)
                    for name, b in self.BITS.items():
                        if bits & b:
                            self.reasons.add(name)
                    self.stop_evt.wait(0.01)

            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
            self.nvml = True
            return
        except Exception:
            self.nvml = False
        self.f = tempfile.NamedTemporaryFile("w+", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(device)], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.nvml:
            self.stop_evt.set()
            self.t.join()
            return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                    "sm_max_mhz": max(self.mx) if self.mx else None, "reasons": sorted(self.reasons),
                    "samples": len(self.sm), "source": "nvml 10 ms"}
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.f.read().splitlines():
            parts = [s.strip() for s in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi 100 ms"}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def pcg_traffic_per_launch(config: str, iterations: float):
    """DRAM bytes of one k_pcg_persistent launch from the committed ncu
    --set full capture, scaled to this run's iteration count, or None."""
    path = os.path.join(ROOT, "profiles", "pcg_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f).get(config)
    if not d:
        return None
    return d["dram_bytes_per_launch"] / d["iterations"] * iterations


# ---------------------------------------------------------------- scene
def make_scene(config: str, seed: int):
    from paper_2008_00409_b200 import scenes
    return scenes.config(config, seed=seed)


# ---------------------------------------------------------------- reference
def ref_devices():
    n = os.cpu_count() or 1
    d = 1
    while d * 2 <= min(n, 32):
        d *= 2
    return d, n


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_steps(sc, steps: int, warmup: int, budget_s: float, functions: bool = False):
    """The compiled reference's hot-path step (oracle/ref_harness.cpp
    ref_sim_step) along the trajectory from rest: `warmup` untimed steps,
    then up to `steps` timed ones within `budget_s` of wall time. Returns
    (mean seconds per timed step, timed steps, info)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bindings import REF, RefSim
    if REF is None:
        return None, 0, {"unavailable": "oracle/_ref/libweft_ref.so not built (needs /root/reference at build time)"}
    devices, nproc = ref_devices()
    t_start = time.time()
    sim = RefSim(REF, sc.verts, sc.tris, sc.pinned, sc.density, sc.material, devices)
    for _ in range(warmup):
        sim.step(sc.dt, sc.thickness)
    times, reps = [], []
    for k in range(steps):
        t0 = time.perf_counter()
        r = sim.step(sc.dt, sc.thickness)
        dt = time.perf_counter() - t0
        times.append(dt)
        reps.append(r)
        if time.time() - t_start + dt > budget_s:
            break
    info = {"devices": devices, "nproc": nproc, "last": reps[-1] if reps else {}, "cpu_model": cpu_model(),
            "pcg_iterations": [int(r["pcg_iterations"]) for r in reps]}
    if functions:
        info["functions_median_ms"] = sim.time_functions(sc.dt, sc.thickness, reps=3)
    sim.close()
    return statistics.mean(times), len(times), info


def reference_arm(args, rank, world):
    if rank != 0:
        return
    sc = make_scene(args.config, args.seed)
    sec, n, info = run_reference_steps(sc, args.steps, args.warmup, args.ref_budget_s, functions=True)
    if sec is None:
        print(json.dumps({"impl": "reference", "unavailable": info["unavailable"]}), flush=True)
        return
    value = 1.0 / sec
    sample = (f"steps {args.warmup}..{args.warmup + n - 1} of the config {args.config} trajectory from rest "
              f"({args.warmup} untimed warm-up steps first), reference Engine({info['devices']}) = "
              f"{2 * info['devices']} threads on {info['nproc']} host cores ({info['cpu_model']})")
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": n, "warmup": args.warmup,
        "ms_per_step": 1e3 * sec, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"config {args.config}: {sc.layers} x {sc.nx}^2 layered cloth, {sc.tri_count} tris, "
                               f"{sc.vertex_count} verts, trajectory from rest", "dt": sc.dt, "pcg_tol": 1e-4,
                   "material": sc.material, "reference_stage_ms_last_step": info["last"],
                   "pcg_iterations": info["pcg_iterations"],
                   "functions_median_ms": info["functions_median_ms"],
                   "functions_note": "SURVEY 8(d): medians of 3 at the state after the timed steps; fill_matrix "
                                     "over step_system's inputs, one spmv_pipelined y = A x, one DCD build_grid",
                   "cpu_model": info["cpu_model"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["devices"], "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------- zones
ZONE_SCENE = (3, 160, 0.1, 0.8)  # layers, nx, fraction of vertices perturbed, amplitude (grid spacings)


def zone_case(seed: int = 7):
    """A resolve_zones workload: a pinned layered cloth whose candidate
    positions push a random subset of vertices through their neighbours."""
    import numpy as np
    from paper_2008_00409_b200 import scenes
    layers, nx, frac, amp = ZONE_SCENE
    sc = scenes.layered_cloth(layers, nx, seed=seed)
    rng = np.random.default_rng(seed)
    x0 = sc.verts.reshape(-1).copy()
    x1 = x0.copy()
    pick = rng.random(len(sc.verts)) < frac
    d = rng.uniform(-amp, amp, (len(sc.verts), 3)) * sc.spacing
    x1.reshape(-1, 3)[pick] += d[pick]
    mv = (1 - sc.pinned).astype(np.uint8)
    mass = np.full(len(sc.verts), 1e-3)
    return sc, x0, x1, mv, mass


def body_proxy_bench(weft, stream, steps: int = 12):
    """BASELINE.json configs[2] as written: the Kimono-scale layered cloth
    (config C, 2 x 501^2, 1 M triangles) on a body proxy — a uv-sphere
    obstacle (mesh.cpp:214-237) pressed into the hanging layers at 0.5 m/s —
    through the whole Simulator::step_impl on the device (contacts, CCD, impact
    zones, the kinematic obstacle given per step as driver.cpp:113-131 does).
    Informational (not the headline config); one GPU."""
    import numpy as np
    import torch
    from paper_2008_00409_b200 import scene as S
    from paper_2008_00409_b200 import scenes
    sc = scenes.config("C")
    mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
    p = mesh.vertex_count
    xs = sc.verts
    radius = 0.4
    ycl = float(xs[:, 1].max())
    center = (float(xs[:, 0].mean()), ycl + radius + 1.5 * sc.thickness, float(xs[:, 2].mean()))
    body = S.make_uv_sphere(center, radius, 48, 96)
    bv = np.asarray(body.vertices, np.float64).reshape(-1, 3)
    bt = np.asarray(body.triangles, np.int32).reshape(-1, 3) + p
    speed = 0.2  # m/s toward the cloth (-y): within the contact thickness from the start
    out = {"workload": f"config C ({sc.layers} x {sc.nx}^2, {sc.tri_count} tris) + uv-sphere body proxy "
                       f"r = {radius} m ({len(bt)} tris) moving into the cloth at {speed} m/s",
           "note": "weft_gpu_sim_step(contacts=1, zones=1) after weft_gpu_sim_set_obstacles, trajectory from rest; "
                   "median device time of steps 2..; informational"}
    times, reps = [], []
    try:
        with weft.Engine(1) as eng:
            eng.set_vertices(mesh.vertex_mass, sc.pinned)
            eng.set_elements(mesh.build_elements(sc.material, sc.gravity))
            eng.set_soup(p + len(bv), np.concatenate([sc.tris, bt]))
            x0 = sc.verts.reshape(-1).copy()
            eng.sim_set_state(x0, np.zeros_like(x0))
            prm = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-4, 400), weft.JAC_SPD, contacts=1,
                                 zones=1)
            st = torch.cuda.ExternalStream(eng.stream())
            for k in range(steps):
                b0 = bv - np.array([0.0, speed * sc.dt * k, 0.0])
                b1 = bv - np.array([0.0, speed * sc.dt * (k + 1), 0.0])
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                eng.sim_set_obstacles(sc.dt, b0.reshape(-1), b1.reshape(-1))
                r = eng.sim_step(prm)
                e1.record(st)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
                reps.append(r)
            out.update({"ms": statistics.median(times[2:]), "ms_all": times,
                        "proximities": [int(r.proximities) for r in reps],
                        "contact_elements": [int(r.contact_elements) for r in reps],
                        "impacts": [int(r.impacts) for r in reps], "zones": [int(r.zone_count) for r in reps],
                        "pcg_iterations": [int(r.pcg_iterations) for r in reps]})
    except weft.Error as e:
        out["error"] = f"step {len(times)}: {e}"
        if len(times) > 2:
            out.update({"ms": statistics.median(times[2:]), "ms_all": times,
                        "proximities": [int(r.proximities) for r in reps],
                        "contact_elements": [int(r.contact_elements) for r in reps],
                        "impacts": [int(r.impacts) for r in reps], "zones": [int(r.zone_count) for r in reps]})
    return out


def zone_bench(weft, stream, with_ref: bool):
    """Impact zones: resolve_zones (CCD rounds + zone
    solves) on the GPU vs the compiled reference on the same input; both
    outputs must be bitwise equal."""
    import numpy as np
    import torch
    sc, x0, x1, mv, mass = zone_case()
    prm = weft.ZoneParams(clearance=0.5 * sc.thickness)
    out = {"workload": f"{ZONE_SCENE[0]} x {ZONE_SCENE[1]}^2 layered cloth ({sc.tri_count} tris), "
                       f"{ZONE_SCENE[2]:.0%} of the vertices displaced by up to {ZONE_SCENE[3]} grid spacings"}
    with weft.Engine(1) as eng:
        eng.set_soup(len(sc.verts), sc.tris)
        eng.set_soup_movable(mv)
        times, res = [], None
        for k in range(4):
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            try:
                res = eng.resolve_zones(x0, x1, mass, sc.thickness, 1.5, prm)
            except weft.ZoneFailure as e:
                res = (e.x_candidate, e.report)
                out["zone_failure"] = str(e)[:120]
            t1.record(stream)
            t1.synchronize()
            if k:
                times.append(t0.elapsed_time(t1))
        xc, rep = res
        out.update({"gpu_ms": statistics.median(times), "first_round_impacts": rep.first_round_impacts,
                    "outer_iterations": rep.outer_iterations, "zones": rep.zone_count,
                    "max_zone_vertices": rep.max_zone_vertices,
                    "note": "weft_gpu_resolve_zones incl. its CCD rounds and host<->device copies of the positions; "
                            "median of 3 after one warm-up"})
    if with_ref:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_bindings import REF
        if REF is not None:
            devices, _ = ref_devices()
            t = time.perf_counter()
            st, msg, rx, rrep = REF.resolve_zones(len(sc.verts), sc.tris, mass, x0, x1, thickness=sc.thickness,
                                                  devices=devices, params=prm.as_array(), movable=mv)
            out["reference_ms"] = 1e3 * (time.perf_counter() - t)
            out["reference_devices"] = devices
            out["bitwise_equal"] = bool(np.array_equal(rx, xc))
    return out


# ---------------------------------------------------------------- GPU arm
def gpu_arm(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    # WEFT_BENCH_ONE_GPU=1: every rank on cuda:0 with gloo plumbing — a
    # functional check of the rank-group path on a 1-GPU box (time-sliced
    # contexts; its timings are meaningless).
    one_gpu = os.environ.get("WEFT_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    backend = "gloo" if one_gpu else "nccl"
    if world > 1 and not dist.is_initialized():
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2008_00409_b200 import weft

    sc = make_scene(args.config, args.seed)
    mesh = weft.ClothMesh.build(sc.verts, sc.tris, sc.density)
    elems = mesh.build_elements(sc.material, sc.gravity)
    p = mesh.vertex_count
    # one logical partition per rank: the rows of the cloth are split over
    # the GPUs (strong scaling of the one 1.65M-triangle problem)
    eng = weft.Engine(world, cuda_device=local, world=world, rank=rank)
    eng.set_vertices(mesh.vertex_mass, sc.pinned)
    if world > 1:
        eng.attach_peers()
    eng.set_elements(elems)
    eng.set_soup(p, sc.tris)
    x0 = sc.verts.reshape(-1).copy()
    v0 = np.zeros_like(x0)
    eng.sim_set_state(x0, v0)
    params = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-4, 400, weft.PRECOND_BLOCK_JACOBI),
                            weft.JAC_SPD)
    stream = torch.cuda.ExternalStream(eng.stream(), device=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def reduce_over_ranks(v: float, op) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if backend == "gloo" else "cuda")
        dist.all_reduce(t, op=op)
        return float(t.item())

    def max_over_ranks(v: float) -> float:
        return reduce_over_ranks(v, dist.ReduceOp.MAX)

    # warm-up: the first W steps of the trajectory from rest
    for _ in range(args.warmup):
        eng.sim_step(params)
    # the trajectory state at the start of the timed region (device copy):
    # the e2e leg and the profiled replay restart from it
    xs = torch.empty(3 * p, dtype=torch.float64, device="cuda")
    vs = torch.empty(3 * p, dtype=torch.float64, device="cuda")
    eng.sim_get_state(xs, vs)
    torch.cuda.synchronize()

    # ---- device-resident timed region: steps W .. W+K-1
    barrier()
    launches0 = eng.stats().launches
    clocks = Clocks(local)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    reps = [eng.sim_step(params) for _ in range(args.steps)]
    ev1.record(stream)
    ev1.synchronize()
    barrier()
    clk = clocks.stop()
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    launches = eng.stats().launches - launches0
    xk = torch.empty_like(xs)
    eng.sim_get_state(xk, None)
    torch.cuda.synchronize()
    # Kernel timing for the roofline, CUDA events on the context stream in a
    # profiled replay of the first two timed steps: the one-partition solve
    # is ONE persistent kernel (timed whole); the multi-partition solve runs
    # as a CUDA graph, so its SpMV launches are timed one by one (chunked
    # launches, identical kernels and inputs).
    eng.sim_set_state(xs, vs)
    eng.profile(True)
    for _ in range(2):
        eng.sim_step(params)
    st = eng.stats()
    eng.profile(False)
    info = eng.matrix_info()

    # ---- end-to-end through the C-ABI with host buffers: the same K steps
    # from the same state, (x, v) uploaded from pinned host memory and the
    # step's result read back every step, the output of step k fed to k+1
    e2e = None
    if not args.no_e2e:
        xa, va = xs.cpu().pin_memory(), vs.cpu().pin_memory()
        xb = torch.empty(3 * p, dtype=torch.float64, pin_memory=True)
        vb = torch.empty(3 * p, dtype=torch.float64, pin_memory=True)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            # H2D of the step's inputs, the step, D2H of its result (one call:
            # weft_gpu_sim_step_io overlaps the copies with the broad phases)
            eng.sim_step_io(xa, va, params, xb, vb)
            xa, xb = xb, xa
            va, vb = vb, va
        e1.record(stream)
        e1.synchronize()
        barrier()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1))
        # every rank uploads the full state (x, v) and reads it back
        e2e = {"value": args.steps / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": world * 2 * 8 * 3 * p,
               "d2h_bytes_per_step": world * 2 * 8 * 3 * p,
               "same_trajectory_as_value": bool(torch.equal(xa.to(xk.device), xk))}

    # SpMV alone (SURVEY §8(d)'s SpMV microbench): y = A x through
    # weft_gpu_spmv on the assembled system of the last step, x ~ U(-1, 1);
    # the kernel timed by the library's CUDA events (the host copies of x and
    # y are outside them); the 0.69 GB matrix is larger than L2
    spmv = None
    if world == 1:
        xr = np.random.default_rng(args.seed).uniform(-1.0, 1.0, 3 * p)
        for _ in range(3):
            eng.spmv_pipelined(None, xr)
        eng.profile(True)
        for _ in range(20):
            eng.spmv_pipelined(None, xr)
        sst = eng.stats()
        eng.profile(False)
        info_now = eng.matrix_info()
        sp_ms = sst.spmv_ms / max(sst.spmv_launches, 1)
        sp_bytes = 76.0 * info_now.nnzb + 52.0 * info_now.block_rows
        spmv = {"kernel": "k_spmv (weft_gpu_spmv, y = A x in the reference's order)", "launches": int(sst.spmv_launches),
                "ms": sp_ms, "alg_bytes": sp_bytes, "achieved": sp_bytes / sp_ms / 1e6, "unit": "GB/s",
                "bytes_note": "SURVEY 8(d): nnzb (72 values + 4 column) + rows (4 length + 24 x + 24 y)"}

    # narrow phase (not part of the hot-path step): collide()
    # = broad phase + elementary DCD / CCD tests + dedup at the timed region's start state
    narrow = None
    if world == 1 and not args.no_narrow:
        eng.set_soup_movable(1 - sc.pinned)
        xe = xs + sc.dt * vs
        narrow = {}
        for name, mode, x1 in (("dcd", weft.DISCRETE, None), ("ccd", weft.CONTINUOUS, xe)):
            eng.collide(xs, x1, mode, sc.thickness)  # warm-up (buffers)
            times = []
            for _ in range(3):
                n0 = torch.cuda.Event(enable_timing=True)
                n1 = torch.cuda.Event(enable_timing=True)
                n0.record(stream)
                kab, _ = eng.collide(xs, x1, mode, sc.thickness)
                n1.record(stream)
                n1.synchronize()
                times.append(n0.elapsed_time(n1))
            g = eng.grid_info()
            narrow[name] = {"ms": statistics.median(times), "ms_all": times, "raw_pairs": g.total, "hits": int(len(kab)),
                            "vertex_face": int((kab[:, 0] == 0).sum()), "edge_edge": int((kab[:, 0] == 1).sum())}
        narrow["note"] = ("weft_gpu_collide at the timed region's start state (x_end = x + dt v for CCD): grid, candidate walk, "
                          "6 VF + 9 EE tests per candidate pair, radix-sorted dedup; device time incl. the hit "
                          "download; not part of the timed step (out of the hot-path scope in both arms)")

    # Simulator::step_impl minus impact zones (contacts mode): DCD narrow phase
    # -> proximities_to_elements -> assembly with contacts -> PCG -> CCD
    # narrow phase; informational, the headline step is the hot path above
    full = None
    if world == 1 and not args.no_narrow:
        fp = weft.SimParams(sc.dt, sc.thickness, 1.5, weft.PcgConfig(1e-4, 400, weft.PRECOND_BLOCK_JACOBI),
                            weft.JAC_SPD, contacts=1, zones=1)
        ftimes, frep = [], None
        try:
            for k in range(4):
                eng.sim_set_state(xs, vs)
                f0 = torch.cuda.Event(enable_timing=True)
                f1 = torch.cuda.Event(enable_timing=True)
                f0.record(stream)
                frep = eng.sim_step(fp)
                f1.record(stream)
                f1.synchronize()
                if k:
                    ftimes.append(f0.elapsed_time(f1))
            full = {"ms": statistics.median(ftimes), "steps_per_s": 1e3 / statistics.median(ftimes),
                    "proximities": frep.proximities, "contact_elements": frep.contact_elements,
                    "impacts": frep.impacts, "zones": frep.zone_count, "pcg_iterations": frep.pcg_iterations,
                    "stage_ms": {"broad_and_narrow": frep.ms_broad, "contacts_and_assemble": frep.ms_assemble,
                                 "solve": frep.ms_solve, "zones": frep.ms_zones},
                    "note": "weft_gpu_sim_step(contacts=1, zones=1) from the timed region's start state: the whole "
                            "Simulator::step_impl (driver.cpp:96-215) incl. resolve_zones, device-resident; "
                            "median of 3"}
        except weft.Error as e:
            full = {"error": str(e)}
        eng.sim_step(params)  # back to the hot-path step (drops the contacts)

    zones = None
    if world == 1 and not args.no_narrow:
        zones = zone_bench(weft, stream, not args.no_cpu_baseline)
    proxy = None
    if world == 1 and not args.no_narrow:
        proxy = body_proxy_bench(weft, stream)

    # candidate counts: each rank walks its split_workload share
    dcd_total = int(reduce_over_ranks(float(reps[-1].dcd_candidates), dist.ReduceOp.SUM if world > 1 else None))
    ccd_total = int(reduce_over_ranks(float(reps[-1].ccd_candidates), dist.ReduceOp.SUM if world > 1 else None))
    barrier()  # no rank unmaps its window while a peer may still read it
    if rank != 0:
        eng.close()
        return
    value = args.steps / (ms_total / 1e3)  # whole-job steps/s (one step = the whole cloth on all ranks)
    peak, peak_src = peaks()
    if spmv is not None:
        spmv.update({"peak": peak, "frac": spmv["achieved"] / peak, "peak_source": peak_src})
    if st.pcg_solves:
        # k_pcg_persistent: per iteration 76 B per streamed
        # live block (9 FP64 values + int32 column) and per row 268 B (q kept
        # in shared memory) or 316 B (q through HBM), counted by the library.
        kname = "k_pcg_persistent (whole PCG solve, one launch)"
        alg_bytes = st.pcg_bytes / st.pcg_solves  # the library's per-solve algorithmic bytes
        launch_ms = st.pcg_ms / st.pcg_solves
        nlaunch = st.pcg_solves
        traffic = pcg_traffic_per_launch(args.config, st.pcg_iterations / st.pcg_solves)
        if world > 1:  # the rank group's solver: one cooperative launch per rank (its rows only)
            kname = "k_pcg_persistent_rows (rank-group PCG, one cooperative launch per rank)"
            traffic = None  # no ncu capture of the multi-rank kernel (one GPU per gpurun call)
    else:
        # k_pcg_spmv: 9 FP64 values + 1 int32 column per live block; per
        # row: length word, z and p gathered once, q written.
        kname = "k_pcg_spmv"
        alg_bytes = info.nnzb * (9 * 8 + 4) + info.block_rows * (4 + 3 * 8 * 3)
        launch_ms = st.spmv_ms / max(st.spmv_launches, 1)
        nlaunch = st.spmv_launches
        traffic = None  # no committed ncu capture of the multi-partition kernels
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9
    it = [r.pcg_iterations for r in reps]
    # The assembly against the same HBM roofline (SURVEY §8(d) algorithmic
    # bytes per step: inputs x, v 48 B + external/mass/pinned ~41 B per vertex,
    # stretch records ~100 B per triangle, hinge records ~40 B per hinge;
    # outputs 76 B per block + 28 B per row). FP64- and latency-bound
    # element math, not bandwidth-bound: reported, not the dominant kernel.
    nh = len(mesh.hinge_verts)
    asm_bytes = 89.0 * p + 100.0 * len(sc.tris) + 40.0 * nh + 76.0 * info.nnzb + 28.0 * info.block_rows
    asm_ms = statistics.mean(r.ms_assemble for r in reps)
    assembly_roofline = {"alg_bytes_per_step": asm_bytes, "ms": asm_ms,
                         "achieved": asm_bytes / (asm_ms * 1e-3) / 1e9, "peak": None, "unit": "GB/s",
                         "bound": "fp64/latency (element evaluation + ordered per-slot accumulation)"}
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        sec, n, rinfo = run_reference_steps(sc, 3, 0, 60.0)
        if sec is not None:
            cpu = {"value": 1.0 / sec, "unit": UNIT, "cores": rinfo["devices"], "kind": "reference",
                   "sample": f"the first {n} steps of the config {args.config} trajectory from rest by the compiled "
                             f"reference, Engine({rinfo['devices']}) = {2 * rinfo['devices']} threads on "
                             f"{rinfo['nproc']} host cores ({rinfo['cpu_model']})"}
        else:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": rinfo["unavailable"]}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {
            "workload": f"config {args.config}: {sc.layers} x {sc.nx}^2 layered cloth, {sc.tri_count} tris, "
                        f"{p} verts, pinned top edges, dt={sc.dt:.6g}, PCG tol 1e-4 block-Jacobi; every step "
                        f"trajectory from rest: {args.warmup} warm-up steps, then steps {args.warmup}.."
                        f"{args.warmup + args.steps - 1} timed",
            "material": sc.material,
            "parallelism": "single GPU" if world == 1 else (
                f"{world} ranks, one row partition each (make_partitions); PCG halos and ordered dot "
                "reductions over peer memory (CUDA IPC / NVLink), replicated broad phase with split pair ranges"
                + (" [WEFT_BENCH_ONE_GPU: all ranks time-sliced on one GPU, functional check only]" if one_gpu else "")),
            "l2": "inputs larger than L2 (matrix alone ~0.75 GB)",
            "pcg_iterations_mean": statistics.mean(it), "nnzb": info.nnzb, "block_rows": info.block_rows,
            "dcd_candidates": dcd_total, "ccd_candidates": ccd_total,
            "stage_ms_mean": {"broad": statistics.mean(r.ms_broad for r in reps),
                              "assemble": statistics.mean(r.ms_assemble for r in reps),
                              "solve": statistics.mean(r.ms_solve for r in reps)},
            "gpu_launches_per_step": launches / args.steps,
            "narrow_phase": narrow,
            "full_step_contacts": full,
            "impact_zones": zones,
            "body_proxy": proxy,
            "assembly_roofline": assembly_roofline,
            "spmv": spmv,
        },
        "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "alg_bytes_per_launch": alg_bytes,
                     "avg_launch_ms": launch_ms, "launches": nlaunch, "peak_source": peak_src},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
    }
    assembly_roofline["peak"] = peak
    assembly_roofline["frac"] = assembly_roofline["achieved"] / peak
    print(json.dumps(out), flush=True)
    eng.close()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        reference_arm(args, rank, world)
    else:
        gpu_arm(args, rank, world, local)


if __name__ == "__main__":
    main()
