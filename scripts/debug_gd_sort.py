import sys, os, numpy as np
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, R + "/tests")
import paper_2301_06984_b200 as E
from oracle import oracle as O
from paper_2301_06984_b200 import configs as CF
from _util import by_uid
wl = CF.ref_proliferation(216)
prm = dict(wl.params, sorting_frequency=int(sys.argv[1]))
sim = E.Simulation(E.SimulationParams(**prm))
sim.add_agents(wl.x, wl.y, wl.z, wl.d)
sim.set_agent_ext(wl.tags, wl.rng_counters)
p = O.OracleParams(seed=prm["seed"], model=prm["model"], mp=prm["model_params"], sorting_frequency=int(sys.argv[1]))
orc = O.PortSim(p, wl.x, wl.y, wl.z, wl.d); orc.set_tags(wl.tags); orc.set_rng_counters(wl.rng_counters)
for it in range(3):
    sim.simulate(1); orc.simulate(1)
    g, o = by_uid(sim.agents()), by_uid(orc.dump())
    gt, gr = sim.agent_ext()
    bad = np.where(np.abs(g["x"] - o["x"]) > 1e-6)[0]
    print("it", it, "n", len(g["uid"]), "bad", len(bad), "d-mismatch", int(np.sum(np.abs(g["d"] - o["d"]) > 1e-9)))
    for k in bad[:6]:
        print("  uid", int(g["uid"][k]), "gpu", g["x"][k], g["y"][k], g["d"][k], "ref", o["x"][k], o["y"][k], o["d"][k])
