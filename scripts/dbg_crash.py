import sys
sys.path.insert(0, '/root/repo')
import paper_2301_06984_b200 as E
from paper_2301_06984_b200 import configs as CF
n = int(sys.argv[1]); timing = sys.argv[2] == "1"; lists = sys.argv[3] == "1"
wl = CF.c4_large_uniform(n)
sim = E.Simulation(E.SimulationParams(**dict(wl.params, record_forces=False, neighbor_list=lists)))
sim.add_agents(wl.x, wl.y, wl.z, wl.d)
if timing: sim.reset_timers(True)
for k in range(12):
    try:
        sim.simulate(1 if k < 6 else 5)
    except Exception as e:
        print("fail at call", k, e, flush=True); break
else:
    print("ok", n, timing, lists, sim.list_stats(), flush=True)
