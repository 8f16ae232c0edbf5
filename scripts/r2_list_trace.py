"""c4 list policy trace: per-iteration device times (phase events) with the iteration kinds (ABSIM_LIST_TRACE=1)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import configs as CF

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 23
wl = CF.c4_large_uniform(n, seed=0)
prm = dict(wl.params, record_forces=False)
sim = E.Simulation(E.SimulationParams(**prm))
sim.add_agents(wl.x, wl.y, wl.z, wl.d)
sim.reset_timers(True)
t0 = time.time()
sim.simulate(steps)
sim.synchronize()
print("wall %.1f ms for %d steps" % ((time.time() - t0) * 1e3, steps))
r = sim.phase_report()
print("per-iteration ms:", " ".join("%.1f" % v for v in r.per_iteration_ms))
print("phases:", r.per_operation_ms)
print("lists:", sim.list_stats())
sim.reset_timers(False)
t0 = time.time()
sim.simulate(20)
sim.synchronize()
print("untimed (graphs) wall %.1f ms for 20 steps -> %.2f ms/step" % ((time.time() - t0) * 1e3, (time.time() - t0) * 50))
print("lists:", sim.list_stats())
