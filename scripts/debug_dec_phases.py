"""Per-phase host wall time of one decomposed step at world 1 (bench --decompose shape)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import bench
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import distributed as D

os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1)
n = 1 << 26
x, y, z, d, uid, L = bench._slab_workload(n, 1, 0)
sim = E.Simulation(E.SimulationParams(seed=0, simulation_time_step=0.01, record_forces=False, capacity=int(n * 1.3)))
sim.add_agents(x, y, z, d, uid=uid, uid_count=n)
dec = D.DeviceSlabDecomposition(sim, dist, 0, 1, transport="nccl", cap=int(0.06 * n) + (1 << 20))
dec.simulate(3)
T = {}
orig = {k: getattr(dec, k) for k in ("_export", "_exchange", "_import", "_allreduce")}
def wrap(name, f):
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(*a, **k); torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + time.perf_counter() - t0; return r
    return g
for k, f in orig.items(): setattr(dec, k, wrap(k, f))
for meth in ("local_bounds", "simulate", "set_grid_override"):
    setattr(sim, meth, wrap(meth, getattr(sim, meth)))
steps = 5
torch.cuda.synchronize(); t0 = time.perf_counter()
dec.simulate(steps)
torch.cuda.synchronize(); tot = time.perf_counter() - t0
for k, v in sorted(T.items(), key=lambda kv: -kv[1]): print(f"{k:20s} {v / steps * 1e3:8.3f} ms/step")
print(f"total {tot / steps * 1e3:.3f} ms/step")
dist.destroy_process_group()
