"""Golden fixtures produced by the unmodified reference engine
(tests/golden/make_golden.py). CPU: the C oracle reproduces them bit for bit.
GPU: the sm_100a path reproduces them within the parity bars."""
import glob
import os

import numpy as np
import pytest

from _util import assert_close, by_uid
from paper_2301_06984_b200 import configs as CF

HERE = os.path.dirname(os.path.abspath(__file__))
FILES = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))
FACTORIES = {
    "c1_n2048_s0": lambda: CF.c1_relaxation(2048, seed=0),
    "c2_side4_s0": lambda: CF.c2_proliferation(side=4, seed=0),
    "c3_n2000_s0": lambda: CF.c3_spheroid(2000, seed=0),
    "c4_n2048_s0": lambda: CF.c4_large_uniform(2048, seed=0),
}


def _name(path):
    return os.path.splitext(os.path.basename(path))[0]


def _oparams(O, wl):
    prm = wl.params
    return O.OracleParams(seed=prm.get("seed", 42), dt=prm.get("simulation_time_step", 0.1),
                          detect_static=prm.get("detect_static_agents", False),
                          model=prm.get("model", 0), mp=prm.get("model_params", [0.0] * 8),
                          sorting_frequency=prm.get("sorting_frequency", 0))


def test_fixtures_present():
    assert set(map(_name, FILES)) == set(FACTORIES)


@pytest.mark.parametrize("path", FILES, ids=_name)
def test_port_reproduces_golden(oracle_mod, path):
    G = np.load(path)
    wl = FACTORIES[_name(path)]()
    s = oracle_mod.PortSim(_oparams(oracle_mod, wl), wl.x, wl.y, wl.z, wl.d, wl.mask)
    g = s.env_update()
    assert np.array_equal(g["origin"], G["origin"]) and g["box"] == G["box"] and g["dmax"] == G["dmax"]
    assert np.array_equal(g["dims"], G["dims"])
    assert np.array_equal(s.cell_ids(), G["cell_id"])
    off, nbr = s.neighbors()
    assert np.array_equal(off, G["nbr_offsets"]) and np.array_equal(nbr, G["nbr_uids"])
    s.simulate(int(G["steps"]))
    d = s.dump()
    for k in d:
        assert np.array_equal(d[k], G[f"final_{k}"]), k


@pytest.mark.gpu
@pytest.mark.parametrize("path", FILES, ids=_name)
def test_gpu_reproduces_golden(engine, path):
    G = np.load(path)
    wl = FACTORIES[_name(path)]()
    sim = engine.Simulation(engine.SimulationParams(**wl.params, bins_per_box=2))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d, behaviour_mask=wl.mask)
    env = sim.environment()
    env.update()
    assert np.array_equal(env.origin(), G["origin"]) and env.box_length() == G["box"]
    assert env.largest_agent_diameter() == G["dmax"] and np.array_equal(env.dims(), G["dims"])
    a = sim.agents()
    got = dict(zip(a["uid"].tolist(), env.cell_ids().tolist()))
    assert got == dict(zip(G["cell_uid"].tolist(), G["cell_id"].tolist()))
    off, nbr = env.neighbors()
    gn = {int(u): tuple(nbr[off[i]:off[i + 1]].tolist()) for i, u in enumerate(a["uid"])}
    on = {int(u): tuple(G["nbr_uids"][G["nbr_offsets"][i]:G["nbr_offsets"][i + 1]].tolist())
          for i, u in enumerate(G["cell_uid"])}
    assert gn == on
    sim.simulate(int(G["steps"]))
    r = sim.report()
    assert [r.final_agent_count, r.uid_count, r.iterations, r.force_evaluations, r.force_skips,
            r.agents_added] == G["counts"].tolist()
    g = by_uid(sim.agents())
    o = by_uid({k[6:]: G[k] for k in G.files if k.startswith("final_")})
    assert np.array_equal(g["uid"], o["uid"])
    for k in ("x", "y", "z", "d", "volume"):
        assert_close(g[k], o[k], 1e-9, 1.0, k)
    for k in ("fx", "fy", "fz"):
        assert_close(g[k], o[k], 1e-9, 2.0, k)
    assert np.array_equal(g["partners"], o["partners"])
    assert np.array_equal(g["flags"], o["flags"])
