"""Neighbour lists against the CPU oracle.

Between two environment rebuilds the mechanical step reads per-agent
candidate lists (radius r + skin) instead of walking the cell table. The
reference's neighbour set {j != i : d2 <= r_i^2} (uniform_grid.cpp:172-230,
simulation.cpp:469) does not depend on the grid, so the bars are the usual
ones: force evaluations and partners exact, positions / forces within 1e-9.
The coverage check (2 x accumulated displacement <= skin) runs on the device
before every list step; these tests drive it through every branch: normal
list steps, forced rebuilds (tiny skin), list growth (wide skin) and sort
iterations (config 4's sorting_frequency).
"""
import numpy as np
import pytest

from _util import assert_close, by_uid
from test_gpu_parity import _oparams, compare_state
from paper_2301_06984_b200 import configs as CF

pytestmark = pytest.mark.gpu


def _run_pair(E, O, wl, steps, chunks, **kw):
    prm = dict(wl.params)
    prm.update(kw)
    sim = E.Simulation(E.SimulationParams(**prm))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    orc = O.PortSim(_oparams(O, wl.params), wl.x, wl.y, wl.z, wl.d)
    per = steps // chunks
    for q in range(chunks):
        sim.simulate(per)
        orc.simulate(per)
        compare_state(sim.agents(), orc.dump(), what=f"{wl.name} after {(q + 1) * per}")
        assert sim.report().force_evaluations == orc.counts()["force_evaluations"], f"evals after {(q + 1) * per}"
    return sim, orc


@pytest.mark.parametrize("cfg,n", [("c1", 4096), ("c4", 8192)])
def test_lists_match_oracle(engine, oracle_mod, cfg, n):
    wl = CF.CONFIGS[cfg](n, seed=3)
    sim, _ = _run_pair(engine, oracle_mod, wl, 30, 3, neighbor_list="always")
    st = sim.list_stats()
    assert st["list_steps"] >= 27 and 0 < st["builds"] < 30, st  # a call's last step may re-bin
    # auto policy (lists only while a build serves >= 3 steps): same results, any mix of step kinds
    _run_pair(engine, oracle_mod, wl, 30, 3)


def test_lists_same_as_rebinning(engine, oracle_mod):
    """Lists on and off give the same integers and agree to 1e-9."""
    wl = CF.c4_large_uniform(8192, seed=4)
    out = []
    for nl in ("always", False):
        p = dict(wl.params, neighbor_list=nl)
        sim = engine.Simulation(engine.SimulationParams(**p))
        sim.add_agents(wl.x, wl.y, wl.z, wl.d)
        sim.simulate(25)
        out.append((sim.report().force_evaluations, sim.agents(), sim.list_stats()))
    assert out[0][0] == out[1][0]
    assert out[1][2]["list_steps"] == 0 and out[0][2]["list_steps"] >= 24
    compare_state(out[0][1], out[1][1], what="lists vs re-binning")


def test_tiny_skin_forces_rebuilds(engine, oracle_mod):
    """skin 0.02: no list survives a step. Forced lists rebuild every
    iteration (and the device coverage check rejects the list step the host
    schedules before any displacement is known); the auto policy falls back
    to re-binning. Results stay exact either way."""
    wl = CF.c1_relaxation(3000, seed=7)
    sim, _ = _run_pair(engine, oracle_mod, wl, 20, 2, neighbor_skin=0.02, neighbor_list="always")
    st = sim.list_stats()
    assert st["builds"] >= 15, st
    sim, _ = _run_pair(engine, oracle_mod, wl, 20, 2, neighbor_skin=0.02)
    assert sim.list_stats()["builds"] < st["builds"]


def test_wide_skin_grows_lists(engine, oracle_mod):
    """skin 9 (c4 shape): more than 64 candidates per agent -> the list
    storage grows (or lists switch off beyond 255); still exact."""
    wl = CF.c4_large_uniform(6000, seed=8)
    sim, _ = _run_pair(engine, oracle_mod, wl, 12, 2, neighbor_skin=9.0)
    assert sim.list_stats()["max_candidates"] > 64


def test_list_step_per_agent_evaluations(engine, oracle_mod):
    """The list sweep's per-agent neighbour counts equal the oracle's
    neighbour sets on the same pre-step state (free-running lists, then one
    more list step with per-agent recording)."""
    O = oracle_mod
    wl = CF.c4_large_uniform(8192, seed=9)
    p = dict(wl.params, sorting_frequency=0, neighbor_skin=8.0)  # wide: the lists surely cover step 4
    sim = engine.Simulation(engine.SimulationParams(**p))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    sim.simulate(3)
    pre = sim.agents()
    steps0 = sim.list_stats()["list_steps"]
    sim.record_evaluations(True)
    sim.simulate(1)
    assert sim.list_stats()["list_steps"] == steps0 + 1  # served from the lists
    ev = dict(zip(sim.agents()["uid"].tolist(), sim.evaluations().tolist()))
    orc = O.PortSim(_oparams(O, p), pre["x"], pre["y"], pre["z"], pre["d"])
    st = {k: pre[k] for k in ("uid", "x", "y", "z", "d", "flags", "partners", "volume")}
    orc.load(st, int(pre["uid"].max()) + 1, 3)
    orc.env_update()
    off, nb = orc.neighbors()
    od = orc.dump()
    oev = {int(u): int(off[i + 1] - off[i]) for i, u in enumerate(od["uid"])}
    assert ev == oev
