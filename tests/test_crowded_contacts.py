"""Crowded neighbourhoods: more contacts per agent than the kernels record.

The walk kernels keep 16 possible contacts per agent in shared memory, the
next 48 in a per-thread spill array, and walk a second time beyond that; the
list step records 24 per agent and re-scans the agent's list beyond. Every
branch must give the reference's forces (mechanics.cpp:10-27, summed over the
same neighbour set, simulation.cpp:463-489): evaluations and partners exact,
positions and forces within 1e-9.
"""
import numpy as np
import pytest

from _util import by_uid
from test_gpu_parity import _oparams, compare_state

pytestmark = pytest.mark.gpu


def _cloud(n, side, seed, d_lo=9.0, d_hi=11.0):
    rng = np.random.default_rng(seed)
    return (rng.uniform(0, side, n), rng.uniform(0, side, n), rng.uniform(0, side, n), rng.uniform(d_lo, d_hi, n))


@pytest.mark.parametrize("n,side,lo,hi", [(3000, 60.0, 17, 64), (1500, 30.0, 65, 10 ** 6)])
@pytest.mark.parametrize("bins", [1, 2])
@pytest.mark.parametrize("lists", [False, "always"])
def test_crowded_contacts(engine, oracle_mod, n, side, lo, hi, bins, lists):
    """side 60: ~20-40 overlapping partners per agent (the spill array);
    side 30: > 64 (the second walk). bins 1 = box walk, 2 = sub-binned fp32
    walk; lists: the list step's contact records and its re-scan."""
    O = oracle_mod
    x, y, z, d = _cloud(n, side, seed=n)
    prm = dict(seed=1, simulation_time_step=0.001, record_forces=True, neighbor_list=lists, neighbor_skin=1.0)
    p = engine.SimulationParams(**prm)
    p.bins_per_box = bins
    sim = engine.Simulation(p)
    sim.add_agents(x, y, z, d)
    orc = O.PortSim(_oparams(O, prm), x, y, z, d)
    for chunk in range(2):
        per = 3 if lists else 1  # the list path needs several iterations per call
        sim.simulate(per)
        orc.simulate(per)
        g, o = sim.agents(), orc.dump()
        compare_state(g, o, what=f"crowded n={n} side={side} chunk {chunk}")
        assert sim.report().force_evaluations == orc.counts()["force_evaluations"]
    partners = by_uid(sim.agents())["partners"]
    assert np.median(partners) >= lo and np.median(partners) <= hi, np.median(partners)
    if lists and side > 50:  # (side 30: > 254 candidates per agent, the lists switch themselves off)
        assert sim.list_stats()["list_steps"] >= 4
