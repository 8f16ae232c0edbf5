"""debug: GrowDivide + remove_self with Morton sorts, one iteration at a time, device vs port (storage keys too)."""
import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2301_06984_b200 as E
from oracle import oracle as O
from paper_2301_06984_b200 import configs as CF
from _util import by_uid
sf = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
wl = CF.ref_proliferation_die(216, p_remove=0.03, sorting_frequency=sf)
wl.params = dict(wl.params, sorting_frequency=sf)
sim = E.Simulation(E.SimulationParams(**wl.params))
sim.add_agents(wl.x, wl.y, wl.z, wl.d)
sim.set_agent_ext(wl.tags, wl.rng_counters)
orc = O.PortSim(O.OracleParams(seed=wl.params["seed"], model=wl.params["model"], mp=wl.params["model_params"],
                               sorting_frequency=sf), wl.x, wl.y, wl.z, wl.d)
for it in range(0, 25, ch):
    sim.simulate(ch)
    orc.simulate(ch)
    g = sim.agents(); keys = sim.storage_keys()
    o = orc.dump()
    order = np.argsort(keys)
    same_set = np.array_equal(np.sort(g["uid"]), np.sort(o["uid"]))
    same_order = len(order) == len(o["uid"]) and np.array_equal(g["uid"][order], o["uid"])
    gb, ob = by_uid(g), by_uid(o)
    dx = np.abs(gb["x"] - ob["x"]).max() if same_set else -1
    r, c = sim.report(), orc.counts()
    print(it, "n", r.final_agent_count, c["agents"], "uidc", r.uid_count, c["uid_count"], "added", r.agents_added, c["agents_added"],
          "removed", r.agents_removed, "set", same_set, "order", same_order, "keys perm", np.array_equal(np.sort(keys), np.arange(len(keys))), "dx %.3g" % dx)
    if same_set and not same_order:
        bad = np.nonzero(g["uid"][order] != o["uid"])[0]
        print("   first order mismatch at slot", bad[:8], "gpu", g["uid"][order][bad[:8]], "ref", o["uid"][bad[:8]])
