import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import configs as CF
wl = CF.ref_proliferation(216)
print(wl.params)
sim = E.Simulation(E.SimulationParams(**wl.params))
sim.add_agents(wl.x, wl.y, wl.z, wl.d)
sim.set_agent_ext(wl.tags, wl.rng_counters)
for k in range(20):
    sim.simulate(1)
    print(k, sim.agent_count(), flush=True)
