"""In-loop Morton sort path guess: a counting-sort guess whose
code space does not fit the cell table is detected on the device, rolled back
and re-run on the exact radix path. Forced here with the test hook
ABSIM_SORT_GUESS_COUNTING on a flat slab (Morton code space >> cell table)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np, sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + "/tests")
import paper_2301_06984_b200 as E
from oracle import oracle as O
from _util import assert_close, by_uid
rng = np.random.default_rng(4)
n = 3000
x, y = rng.uniform(0, 600, n), rng.uniform(0, 600, n)
z, d = rng.uniform(0, 12, n), rng.uniform(8, 12, n)
sim = E.Simulation(E.SimulationParams(seed=1, simulation_time_step=0.01, sorting_frequency=1))
sim.add_agents(x, y, z, d)
orc = O.PortSim(O.OracleParams(seed=1, dt=0.01, sorting_frequency=1), x, y, z, d)
for step in range(4):
    sim.simulate(1)
    orc.simulate(1)
    g, o = by_uid(sim.agents()), by_uid(orc.dump())
    assert np.array_equal(g["uid"], o["uid"])
    for k in ("x", "y", "z"):
        assert_close(g[k], o[k], 1e-9, 1.0, k)
    assert sim.report().force_evaluations == orc.counts()["force_evaluations"]
print("OK")
"""


@pytest.mark.gpu
def test_counting_guess_rolled_back(engine, oracle_mod):
    env = dict(os.environ, ABSIM_SORT_GUESS_COUNTING="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stderr[-3000:]
    assert "sort retry at iteration" in r.stderr  # the rollback path actually ran
