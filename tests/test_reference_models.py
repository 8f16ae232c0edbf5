"""The reference's own behaviour models on the device:
models::GrowDivide and models::Cohere (models.hpp:15-64) on the reference's
own population builders (models.cpp:21-61), against the C oracle (pinned
bit-exact to the unmodified reference in test_oracle.py) and the reference
itself when its build is present. Integer state (agent/uid counts, tags,
RandomStream counters, force evaluations) is exact; positions within
1e-9 (cos/sin of the division axis and the Cohere centroid sum order are
the non-bit-portable terms)."""
import numpy as np
import pytest

from _util import assert_close, by_uid
from paper_2301_06984_b200 import configs as CF

pytestmark = pytest.mark.gpu


def _oracle(O, wl):
    prm = wl.params
    p = O.OracleParams(seed=prm["seed"], model=prm["model"], mp=prm["model_params"],
                       fixed_box=prm.get("fixed_box_length", 0.0))
    s = O.PortSim(p, wl.x, wl.y, wl.z, wl.d)
    s.set_tags(wl.tags)
    s.set_rng_counters(wl.rng_counters)
    return s, p


def _gpu(E, wl):
    sim = E.Simulation(E.SimulationParams(**wl.params))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    sim.set_agent_ext(wl.tags, wl.rng_counters)
    return sim


def _compare(sim, orc, what):
    g = sim.agents()
    g["tag"], g["rngc"] = sim.agent_ext()
    o = orc.dump()
    o["tag"], o["rngc"] = orc.tags(), orc.rng_counters()
    g, o = by_uid(g), by_uid(o)
    assert np.array_equal(g["uid"], o["uid"]), f"{what}: uid sets"
    for k in ("tag", "rngc"):
        assert np.array_equal(g[k], o[k]), f"{what}: {k}"
    for k in ("x", "y", "z", "d"):
        assert_close(g[k], o[k], 1e-9, 1.0, f"{what} {k}")
    r, c = sim.report(), orc.counts()
    assert (r.final_agent_count, r.uid_count, r.agents_added) == (c["agents"], c["uid_count"], c["agents_added"])
    assert r.force_evaluations == c["force_evaluations"], what


def test_growdivide_reference_lattice(engine, oracle_mod, have_ref):
    O = oracle_mod
    wl = CF.ref_proliferation(216)
    sim = _gpu(engine, wl)
    orc, p = _oracle(O, wl)
    ref = O.RefSim.builtin(p, "proliferation", 216) if have_ref else None
    for chunk in range(4):
        sim.simulate(5)
        orc.simulate(5)
        _compare(sim, orc, f"grow-divide after {5 * (chunk + 1)}")
        if ref is not None:
            ref.simulate(5)
            assert ref.counts()["agents"] == sim.report().final_agent_count
    assert sim.report().final_agent_count > 216


def test_cohere_reference_clustering(engine, oracle_mod, have_ref):
    O = oracle_mod
    wl = CF.ref_clustering(3000, seed=7)
    sim = _gpu(engine, wl)
    orc, p = _oracle(O, wl)
    for chunk in range(3):
        sim.simulate(4)
        orc.simulate(4)
        _compare(sim, orc, f"cohere after {4 * (chunk + 1)}")
    if have_ref:  # the reference's own builder gives the same start state
        ref = O.RefSim.builtin(p, "clustering", 3000)
        ref.simulate(12)
        g, r = by_uid(sim.agents()), by_uid(ref.dump())
        assert np.array_equal(g["uid"], r["uid"])
        assert_close(g["x"], r["x"], 1e-9, 1.0, "cohere vs reference x")


def test_cohere_radius_exceeds_box(engine):
    """uniform_grid.cpp:176-181: a query radius above the box length fails."""
    wl = CF.ref_clustering(500, seed=1)
    prm = {**wl.params, "fixed_box_length": 0.0}  # box = largest diameter (10) < 30
    sim = engine.Simulation(engine.SimulationParams(**prm))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    with pytest.raises(ValueError, match="query radius"):
        sim.simulate(1)


@pytest.mark.parametrize("graphs", ["1", "0"])
def test_growdivide_static_combined(engine, oracle_mod, graphs):
    """Divisions + static detection together, replayed through CUDA graphs or
    launched directly: capacity and cell-table growth mid-run (device
    rollbacks), behaviour agents listed past the static pre-pass."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = f"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + "/tests")
import paper_2301_06984_b200 as E
from oracle import oracle as O
from paper_2301_06984_b200 import configs as CF
from test_reference_models import _compare
wl = CF.ref_proliferation(216)
prm = dict(wl.params, detect_static_agents=True)
sim = E.Simulation(E.SimulationParams(**prm))
sim.add_agents(wl.x, wl.y, wl.z, wl.d)
sim.set_agent_ext(wl.tags, wl.rng_counters)
p = O.OracleParams(seed=prm["seed"], model=prm["model"], mp=prm["model_params"], detect_static=True,
                   fixed_box=prm.get("fixed_box_length", 0.0))
orc = O.PortSim(p, wl.x, wl.y, wl.z, wl.d)
orc.set_tags(wl.tags)
orc.set_rng_counters(wl.rng_counters)
for chunk in range(4):
    sim.simulate(4)
    orc.simulate(4)
    _compare(sim, orc, f"after {{4 * (chunk + 1)}}")
    assert sim.report().force_skips == orc.counts()["force_skips"]
assert sim.report().final_agent_count > 216
print("OK")
"""
    env = dict(os.environ, ABSIM_GRAPHS=graphs)
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("model,sf", [(5, 3), (7, 0), (7, 4)])
def test_additions_after_reordering(engine, oracle_mod, model, sf):
    """Daughter uids follow the reference's storage order (commit.cpp:186-222)
    after Morton sorts and removals: the device carries each agent's slot in
    that order (Soa::skey) through every move, ranks dividing parents by it
    and applies remove_agents_parallel (commit.cpp:14-106) to it. GrowDivide
    with sorts, GrowDivide + remove_self, both together, against the port
    (pinned to the reference in test_oracle.py)."""
    O = oracle_mod
    wl = CF.ref_proliferation_die(216, p_remove=0.03, sorting_frequency=sf) if model == 7 else CF.ref_proliferation(216)
    wl.params = dict(wl.params, sorting_frequency=sf)
    sim = _gpu(engine, wl)
    orc = O.PortSim(O.OracleParams(seed=wl.params["seed"], model=wl.params["model"], mp=wl.params["model_params"],
                                   sorting_frequency=sf), wl.x, wl.y, wl.z, wl.d)
    for chunk in range(5):
        sim.simulate(5)
        orc.simulate(5)
        _compare(sim, orc, f"model {model} sf {sf} after {5 * (chunk + 1)}")
    r = sim.report()
    assert r.agents_added > 0 and (model != 7 or r.agents_removed > 0)


def test_api_removal_then_divisions(engine, oracle_mod):
    """abs_gpu_remove in the caller's list order (the reference's removal
    vector gives the hole order), then more GrowDivide iterations: survivors'
    slots and the later daughters' uids match the port."""
    O = oracle_mod
    wl = CF.ref_proliferation(216)
    sim = _gpu(engine, wl)
    orc, _ = _oracle(O, wl)
    sim.simulate(6)
    orc.simulate(6)
    d = orc.dump()
    rng = np.random.default_rng(3)
    slots = rng.choice(len(d["uid"]), size=40, replace=False).astype(np.uint32)
    sim.remove_agents(d["uid"][slots])
    orc.remove(slots)
    for chunk in range(3):
        sim.simulate(5)
        orc.simulate(5)
        _compare(sim, orc, f"after removal + {5 * (chunk + 1)}")
