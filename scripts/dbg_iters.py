"""Per-iteration device time of c4 with and without neighbour lists (diagnostic)."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import torch
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import configs as CF
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
wl = CF.c4_large_uniform(n)
for lists, skin in ((False, 0.0), (True, 2.7), (True, 4.0)):
    prm = dict(wl.params, record_forces=False, neighbor_list=lists, neighbor_skin=skin)
    sim = E.Simulation(E.SimulationParams(**prm))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    sim.simulate(3)
    sim.synchronize()
    sim.reset_timers(True)
    t0 = time.perf_counter()
    sim.simulate(20)
    sim.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    r = sim.phase_report()
    it = np.array(r.per_iteration_ms)
    print(f"lists={lists} skin={skin}: wall {wall/20:.2f} ms/it, device sum {it.sum()/20:.2f}, per-it", np.round(it, 1).tolist(), sim.list_stats(), flush=True)
    del sim
