"""Dev probe: cell occupancy of the DCD / CCD grids of a config at rest
(entries, cells, pair space, triangles-per-cell histogram)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_00409_b200 import scenes, weft  # noqa: E402

sc = scenes.config(sys.argv[1] if len(sys.argv) > 1 else "D")
p = len(sc.verts)
x = sc.verts.reshape(-1).copy()
with weft.Engine(1) as eng:
    eng.set_soup(p, sc.tris)
    for mode, xe in ((weft.DISCRETE, None), (weft.CONTINUOUS, x + 1e-4)):
        eng.build_grid(x, xe, mode, sc.thickness)
        g = eng.download_grid(len(sc.tris))
        s = np.diff(g.cell_offsets)
        pairs = s * (s - 1) // 2
        print(f"mode {mode}: cell {g.cell_size:.4g} entries {s.sum()} cells {len(s)} pairs {pairs.sum()} "
              f"mean s {s.mean():.1f} max s {s.max()}")
        for lo, hi in ((1, 16), (17, 32), (33, 64), (65, 128), (129, 256), (257, 10**9)):
            m = (s >= lo) & (s <= hi)
            print(f"   s in [{lo},{hi}]: cells {m.sum()} pairs {pairs[m].sum()} ({100 * pairs[m].sum() / max(pairs.sum(), 1):.1f}%)")
