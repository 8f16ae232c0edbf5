import sys, numpy as np
sys.path.insert(0, '.')
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import configs as CF, distributed as D
wl = CF.c1_relaxation(3000, seed=1)
st = D.initial_partition(wl.x, wl.y, wl.z, wl.d, 2, 0)
b = np.array([wl.x.min(), wl.y.min(), wl.z.min(), wl.x.max(), wl.y.max(), wl.z.max(), wl.d.max()])
g = D.global_grid(b); grid, dims = g.as_override()
eng = D.GpuRankEngine(E.SimulationParams(**wl.params), device=0)
variant = sys.argv[1]
for rnd in range(3):
    eng.load(st, 3000, rnd)
    if variant in ("override", "both"):
        eng.set_grid_override(grid, dims)
    eng.step()
    out = eng.dump()
    print(variant, "round", rnd, "n", len(out["x"]), "evals", eng.counters(), flush=True)
    if variant in ("redump", "both"):
        st = {k: out[k] for k in st}
