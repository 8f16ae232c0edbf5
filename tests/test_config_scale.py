"""Parity at BASELINE.json's own sizes, slow.

* c1: 131,072 agents x 100 iterations, free-running against the C port
  (fp64 state within 1e-9, force evaluations exact).
* c2: the 16^3 proliferation lattice through six synchronous doublings
  (> 100k daughters appended in one commit), free-running against the port
  (agent and uid counts, evaluations, state).
* c4: 2^26 agents, teacher-forced on the two Morton-sort iterations 0 and 10:
  cell ids (box_index_of) and every agent's force evaluations — the size of
  its neighbour set at the force radius, from the hot walker itself
  (abs_gpu_record_evaluations) — against the UNMODIFIED reference engine on
  the same state (its multithreaded neighbour counts are order-free).
"""
import numpy as np
import pytest

from _util import assert_close, by_uid
from test_gpu_parity import _oparams, compare_state
from paper_2301_06984_b200 import configs as CF

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_c1_full_scale_free_running(engine, oracle_mod):
    wl = CF.c1_relaxation()  # 131,072 agents
    sim = engine.Simulation(engine.SimulationParams(**wl.params))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    orc = oracle_mod.PortSim(_oparams(oracle_mod, wl.params), wl.x, wl.y, wl.z, wl.d)
    for q in range(4):
        sim.simulate(25)
        orc.simulate(25)
        assert sim.report().force_evaluations == orc.counts()["force_evaluations"], f"evals after {25 * (q + 1)}"
    compare_state(sim.agents(), orc.dump(), what="c1 131072 x 100")


def test_c2_through_division_bursts(engine, oracle_mod):
    wl = CF.c2_proliferation(16)  # 4096 cells, synchronous doublings ~21 iterations apart
    prm = dict(wl.params, capacity=300_000)
    sim = engine.Simulation(engine.SimulationParams(**prm))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    orc = oracle_mod.PortSim(_oparams(oracle_mod, wl.params), wl.x, wl.y, wl.z, wl.d)
    largest_burst, n_prev = 0, wl.n
    it = 0
    while orc.counts()["agents"] < 200_000:
        sim.simulate(7)
        orc.simulate(7)
        it += 7
        r, c = sim.report(), orc.counts()
        assert (r.final_agent_count, r.uid_count, r.force_evaluations) == \
               (c["agents"], c["uid_count"], c["force_evaluations"]), f"iteration {it}"
        largest_burst = max(largest_burst, c["agents"] - n_prev)
        n_prev = c["agents"]
        assert it < 200
    assert largest_burst > 100_000
    compare_state(sim.agents(), orc.dump(), what=f"c2 after {it}")


def _ref_counts_and_cells(O, st):
    """Reference engine on a downloaded state (agents created in uid order):
    per-uid box_index_of and force-query neighbour counts."""
    n = len(st["uid"])
    u = st["uid"].astype(np.int64)
    arrs = {}
    for k in ("x", "y", "z", "d"):  # scatter into uid order (a permutation of 0..n-1)
        a = np.empty(n)
        a[u] = st[k]
        arrs[k] = a
    ref = O.RefSim(O.OracleParams(seed=0, dt=0.01), arrs["x"], arrs["y"], arrs["z"], arrs["d"])
    grid = ref.env_update()
    cells = ref.cell_ids()
    counts = ref.neighbor_counts()
    ref.close()
    return grid, cells, counts  # indexed by uid (storage order = creation order)


def _gpu_cells(sim):
    env = sim.environment()
    env.update()
    ids = env.cell_ids()
    uid = sim.fields("uid")["uid"]
    out = np.empty(len(uid), np.uint64)
    out[uid.astype(np.int64)] = ids
    return env, out


def test_c4_full_scale_sort_iterations(engine, oracle_mod, have_ref):
    if not have_ref:
        pytest.skip("reference build (oracle/_ref) not present")
    O = oracle_mod
    wl = CF.c4_large_uniform()  # 2^26 agents, Morton sort every 10 iterations
    sim = engine.Simulation(engine.SimulationParams(**dict(wl.params, record_forces=False)))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    n = wl.n
    for target in (0, 10):
        if target:
            sim.simulate(target - sim.iteration)
        pre = sim.fields("uid", "x", "y", "z", "d")
        env, gcells = _gpu_cells(sim)
        grid, rcells, rcounts = _ref_counts_and_cells(O, pre)
        assert np.array_equal(env.origin(), grid["origin"]) and env.box_length() == grid["box"], target
        assert np.array_equal(env.dims(), grid["dims"]), target
        assert np.array_equal(gcells, rcells), f"cell ids at iteration {target}"
        sim.record_evaluations(True)
        e0 = sim.report().force_evaluations
        sim.simulate(1)  # the sort iteration itself (sorting_frequency 10)
        sim.record_evaluations(False)
        ev = sim.evaluations()
        uid = sim.fields("uid")["uid"].astype(np.int64)
        gev = np.empty(n, np.uint32)
        gev[uid] = ev
        assert np.array_equal(gev, rcounts), f"per-agent evaluations at iteration {target}"
        assert sim.report().force_evaluations - e0 == int(rcounts.sum(dtype=np.uint64))
