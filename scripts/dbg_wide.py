import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2301_06984_b200 as E
from oracle import oracle as O
from paper_2301_06984_b200 import configs as CF
from test_gpu_parity import _oparams
from _util import by_uid
for skin, sf in ((9.0, 10), (9.0, 0), (5.0, 0), (3.0, 0)):
    wl = CF.c4_large_uniform(6000, seed=8)
    prm = dict(wl.params, neighbor_skin=skin, sorting_frequency=sf)
    sim = E.Simulation(E.SimulationParams(**prm)); sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    orc = O.PortSim(_oparams(O, prm), wl.x, wl.y, wl.z, wl.d)
    for st in range(6):
        sim.simulate(2); orc.simulate(2)
        g, o = by_uid(sim.agents()), by_uid(orc.dump())
        err = np.max(np.abs(g['x'] - o['x']))
        print(skin, sf, 'after', 2*(st+1), 'maxerr %.3e' % err, 'evals', sim.report().force_evaluations - orc.counts()['force_evaluations'], sim.list_stats(), flush=True)
        if err > 1e-6: break
