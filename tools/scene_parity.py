import sys, time, numpy as np, ctypes as C
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2008_00409_b200 import scene as S
from scenes_gen import SCENES, scene_text
from oracle_bindings import REF, ptr
L = REF.lib
L.ref_scene_load.restype = C.c_void_p
for name in SCENES:
    txt = scene_text(name)
    sc = S.parse_scene(txt)
    sim = S.Simulator(sc)
    h = L.ref_scene_load(txt.encode(), 1, b".")
    out = np.zeros(10)
    frames = sc.config.frames
    worst = 0.0; msg = ""
    for k in range(frames):
        st = L.ref_scene_step(C.c_void_p(h), C.c_int32(0), ptr(out))
        try:
            r = sim.step()
        except Exception as e:
            msg = f"gpu raised at {k}: {str(e)[:60]} / ref st {st} {L.ref_last_error()[:60] if st else ''}"; break
        if st:
            msg = f"ref raised at {k}: {L.ref_last_error()[:60]}"; break
        xr, vr = np.zeros(3*sim.mesh.vertex_count), np.zeros(3*sim.mesh.vertex_count)
        L.ref_scene_state(C.c_void_p(h), ptr(xr), ptr(vr))
        xg, vg = sim.state()
        ex = np.abs(xg.reshape(-1)-xr).max()/np.abs(xr).max(); ev = np.abs(vg.reshape(-1)-vr).max()/max(np.abs(vr).max(),1e-12)
        worst = max(worst, ex, ev)
        if (r.proximities, r.contacts, r.impacts, r.zone_count) != tuple(int(v) for v in out[[4,5,6,7]]):
            msg += f" counts differ at {k}: gpu {(r.proximities, r.contacts, r.impacts, r.zone_count)} ref {out[[4,5,6,7]]};"
    print(name, frames, "worst rel", f"{worst:.2e}", "last gpu", (r.pcg_iterations, r.proximities, r.contacts, r.impacts, r.zone_count), "ref", out[[2,4,5,6,7]].astype(int), msg, flush=True)
