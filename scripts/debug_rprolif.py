"""Per-iteration host timing of the reference proliferation workload."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import configs as CF

wl = CF.ref_proliferation(32768)
prm = dict(wl.params, capacity=3 * wl.n * 2 ** 7)
sim = E.Simulation(E.SimulationParams(**prm))
sim.add_agents(wl.x, wl.y, wl.z, wl.d)
sim.set_agent_ext(wl.tags, wl.rng_counters)
for it in range(14):
    t0 = time.perf_counter()
    sim.simulate(1)
    sim.synchronize()
    dt = time.perf_counter() - t0
    r = sim.report()
    env = sim.environment()
    print(f"it {it} {dt*1e3:8.2f} ms n={r.final_agent_count} uid_count={r.uid_count} launches={r.kernel_launches}", flush=True)
