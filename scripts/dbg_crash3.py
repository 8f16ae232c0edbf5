import sys, os
sys.path.insert(0, '/root/repo')
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import configs as CF
n = int(sys.argv[1]); sf = int(sys.argv[2]); its = int(sys.argv[3]); warm = int(sys.argv[4]) if len(sys.argv) > 4 else 0
wl = CF.c4_large_uniform(n)
sim = E.Simulation(E.SimulationParams(**dict(wl.params, record_forces=False, neighbor_list=False, sorting_frequency=sf)))
sim.add_agents(wl.x, wl.y, wl.z, wl.d)
try:
    if warm: sim.simulate(warm)
    sim.simulate(its)
    print("ok", sys.argv[1:], os.environ.get("ABSIM_GRAPHS"), flush=True)
except Exception as e:
    print("fail", sys.argv[1:], os.environ.get("ABSIM_GRAPHS"), e, flush=True)
