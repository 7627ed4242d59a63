"""Dev check: the rank group's ZoneFailure path (2 ranks time-sliced on one GPU) vs the single process."""
import os, sys, time, tempfile
sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo")
os.environ["WEFT_CON_V0"] = "1"
import test_gpu_multirank as t
from paper_2008_00409_b200 import weft
import mp_rank
d = tempfile.mkdtemp()
t0 = time.time()
ranks = t.spawn(2, 2, d)
print("spawn s", time.time() - t0)
single, engines = mp_rank.run(lambda: weft.Engine(2), 1, 0, lambda e: None)
print("single", single["con_counts"].tolist(), str(single.get("con_error")), "wall", single["con_wall_s"].tolist())
for r in ranks:
    print("rank", r["con_counts"].tolist(), str(r.get("con_error")), "wall", r["con_wall_s"].tolist())
    import numpy as np
    print(np.array_equal(r["con_x"], single["con_x"]), np.array_equal(r["con_v"], single["con_v"]))
