import sys, numpy as np
sys.path.insert(0, '.')
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import configs as CF, distributed as D
wl = CF.c1_relaxation(3000, seed=1)
world = 2
for rank in range(world):
    st = D.initial_partition(wl.x, wl.y, wl.z, wl.d, world, rank)
    other = D.initial_partition(wl.x, wl.y, wl.z, wl.d, world, 1 - rank)
    b = np.array([wl.x.min(), wl.y.min(), wl.z.min(), wl.x.max(), wl.y.max(), wl.z.max(), wl.d.max()])
    g = D.global_grid(b)
    L = D.layer_bounds(int(g.dims[2]), world)
    lay = D.box_layer(other["z"], g)
    gh = D._take(other, np.nonzero(lay == (L[1] if rank == 0 else L[1] - 1))[0])
    gh["flags"] = gh["flags"] | D.FLAG_GHOST
    full = D._concat([st, gh])
    print("rank", rank, "owned", len(st["x"]), "ghosts", len(gh["x"]), "dims", g.dims, flush=True)
    eng = D.GpuRankEngine(E.SimulationParams(**wl.params), device=0)
    eng.load(full, 3000, 0)
    grid, dims = g.as_override()
    print("override", grid, dims, flush=True)
    eng.set_grid_override(grid, dims)
    try:
        eng.sim.environment().update()
        print("env ok", eng.sim.environment().dims(), flush=True)
        eng.step()
        print("step ok", eng.counters(), flush=True)
    except Exception as e:
        print("FAILED", e, flush=True)
        raise
