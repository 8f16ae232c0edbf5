import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))) + "/tests")
import paper_2301_06984_b200 as E
from oracle import oracle as O
from paper_2301_06984_b200 import configs as CF
from test_reference_models import _compare
static = sys.argv[1] == "1"; sortf = int(sys.argv[2])
wl = CF.ref_proliferation(216)
prm = dict(wl.params, detect_static_agents=static, sorting_frequency=sortf)
sim = E.Simulation(E.SimulationParams(**prm))
sim.add_agents(wl.x, wl.y, wl.z, wl.d)
sim.set_agent_ext(wl.tags, wl.rng_counters)
p = O.OracleParams(seed=prm["seed"], model=prm["model"], mp=prm["model_params"], detect_static=static,
                   sorting_frequency=sortf, fixed_box=prm.get("fixed_box_length", 0.0))
orc = O.PortSim(p, wl.x, wl.y, wl.z, wl.d)
orc.set_tags(wl.tags); orc.set_rng_counters(wl.rng_counters)
for it in range(12):
    sim.simulate(1); orc.simulate(1)
    try:
        _compare(sim, orc, f"it {it}")
    except AssertionError as e:
        print("FAIL at", it, str(e)[:160]); sys.exit(0)
print("OK")
