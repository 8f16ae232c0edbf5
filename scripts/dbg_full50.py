"""Whole c4 configuration (50 iterations from the initial state) with lists auto vs off (diagnostic)."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import configs as CF
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
cfg = sys.argv[2] if len(sys.argv) > 2 else "c4"
wl = CF.CONFIGS[cfg](n)
steps = wl.steps
for lists in (False, True):
    prm = dict(wl.params, record_forces=False, neighbor_list=lists)
    sim = E.Simulation(E.SimulationParams(**prm))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    sim.synchronize()
    sim.reset_timers(True)
    t0 = time.perf_counter()
    sim.simulate(steps)
    sim.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    r = sim.phase_report()
    it = np.array(r.per_iteration_ms)
    print(f"{cfg} n={n} lists={lists}: {steps} its wall {wall/steps:.3f} ms/it ({n*steps/wall*1e3:.4g} agent-it/s), per-it", np.round(it, 2).tolist(), sim.list_stats(), "evals", sim.report().force_evaluations, flush=True)
    del sim
