"""EnvironmentKind (params.hpp:9): the brute-force environment
(BruteForceEnvironment, environment.hpp:53-80) and the kd-tree environment
(KdTreeEnvironment, kdtree_env.cpp:8-86) as the comparison baselines of the
paper's grid-vs-tree study, against the unmodified reference's own
brute-force and kd-tree environments."""
import numpy as np
import pytest

from _util import assert_close, by_uid
from paper_2301_06984_b200 import configs as CF

K = 2.0


def _rp(O, wl, env, **kw):
    prm = wl.params
    args = dict(seed=prm.get("seed", 0), dt=prm.get("simulation_time_step", 0.1),
                detect_static=prm.get("detect_static_agents", False), env=env)
    args.update(kw)
    return O.OracleParams(**args)


def _nbr_map(uid, off, nb):
    return {int(u): tuple(nb[off[i]:off[i + 1]].tolist()) for i, u in enumerate(uid)}


def test_params_validation(engine):
    E = engine
    with pytest.raises(ValueError):
        E.SimulationParams(environment="octree", simulation_time_step=0.01).validate()
    E.SimulationParams(environment="kdtree").validate()
    with pytest.raises(ValueError):  # params.cpp:52-55
        E.SimulationParams(environment="brute_force", sorting_frequency=10).validate()
    E.SimulationParams(environment="brute_force").validate()


def test_reference_environments_agree(oracle_mod, have_ref):
    """Pin: the reference's brute-force and kd-tree environments give its
    grid's neighbour sets and states (criterion 1 / test_grid.cpp:163-212)."""
    O = oracle_mod
    if not have_ref:
        pytest.skip("reference build unavailable")
    wl = CF.c1_relaxation(1500, seed=5)
    sims = [O.RefSim(_rp(O, wl, env), wl.x, wl.y, wl.z, wl.d) for env in (0, 1, 2)]
    for s in sims:
        s.simulate(4)
    dumps = [by_uid(s.dump()) for s in sims]
    for d in dumps[1:]:
        assert np.array_equal(d["uid"], dumps[0]["uid"])
        for k in ("x", "y", "z"):
            assert_close(d[k], dumps[0][k], 1e-9, 1.0, k)
        assert np.array_equal(d["partners"], dumps[0]["partners"])
    assert sims[1].counts()["force_evaluations"] == sims[0].counts()["force_evaluations"]
    maps = []
    for s in sims:
        s.env_update()
        o, u = s.neighbors()
        maps.append(_nbr_map(s.dump()["uid"], o, u))
    assert maps[0] == maps[1] == maps[2]


@pytest.mark.gpu
@pytest.mark.parametrize("static", [False, True])
def test_gpu_brute_force_matches_reference(engine, oracle_mod, have_ref, static):
    E, O = engine, oracle_mod
    if not have_ref:
        pytest.skip("reference build unavailable")
    wl = CF.c1_relaxation(2048, seed=3)
    ref = O.RefSim(_rp(O, wl, 1, detect_static=static), wl.x, wl.y, wl.z, wl.d)
    sim = E.Simulation(E.SimulationParams(**{**wl.params, "environment": "brute_force",
                                             "detect_static_agents": static}))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    for step in range(5):
        ref.simulate(1)
        sim.simulate(1)
        g, o = by_uid(sim.agents()), by_uid(ref.dump())
        assert np.array_equal(g["uid"], o["uid"])
        for k in ("x", "y", "z"):
            assert_close(g[k], o[k], 1e-9, 1.0, f"step {step} {k}")
        for k in ("fx", "fy", "fz"):
            assert_close(g[k], o[k], 1e-9, K, f"step {step} {k}")
        assert np.array_equal(g["partners"], o["partners"]), step
        r = sim.report()
        c = ref.counts()
        assert r.force_evaluations == c["force_evaluations"] and r.force_skips == c["force_skips"], step
    env = sim.environment()
    assert env.name() == "brute_force" and env.max_query_radius() == float("inf")
    env.update()
    assert env.largest_agent_diameter() == float(np.max(sim.agents()["d"]))
    go, gu = env.neighbors()
    ro, ru = ref.neighbors()
    assert _nbr_map(sim.agents()["uid"], go, gu) == _nbr_map(ref.dump()["uid"], ro, ru)
    with pytest.raises(E.AbsimError):
        env.cell_ids()  # no cells without a grid


@pytest.mark.gpu
def test_gpu_brute_force_equals_grid(engine):
    """Same population, both environments: identical integer outputs."""
    E = engine
    wl = CF.c4_large_uniform(1 << 13, seed=2)
    out = []
    for env in ("uniform_grid", "brute_force"):
        sim = E.Simulation(E.SimulationParams(**{**wl.params, "environment": env, "sorting_frequency": 0}))
        sim.add_agents(wl.x, wl.y, wl.z, wl.d)
        sim.simulate(3)
        out.append((by_uid(sim.agents()), sim.report().force_evaluations))
    (a, ea), (b, eb) = out
    assert ea == eb
    assert np.array_equal(a["partners"], b["partners"])
    for k in ("x", "y", "z"):
        assert_close(a[k], b[k], 1e-9, 1.0, k)


@pytest.mark.gpu
def test_gpu_brute_force_static_known_answer(engine):
    """test_scheduler.cpp:464-488 under the brute-force environment: a settled
    3x3x3 lattice costs 108 evaluations, then all 27 agents are skipped."""
    E = engine
    g = np.arange(3) * 10.0
    x, y, z = (a.ravel() for a in np.meshgrid(g, g, g, indexing="ij"))
    sim = E.Simulation(E.SimulationParams(detect_static_agents=True, environment="brute_force"))
    sim.add_agents(x, y, z, np.full(27, 10.0))
    sim.simulate(1)
    r = sim.report()
    assert r.force_evaluations == 108 and r.force_skips == 0
    sim.simulate(1)
    r = sim.report()
    assert r.force_evaluations == 108 and r.force_skips == 27


@pytest.mark.gpu
def test_gpu_brute_force_edge_cases(engine):
    E = engine
    sim = E.Simulation(E.SimulationParams(environment="brute_force"))
    sim.simulate(3)  # empty population
    assert sim.report().final_agent_count == 0
    sim.add_agents([0.0, 1e6], [0.0, 0.0], [0.0, 0.0], [10.0, 10.0])  # far apart: no grid budget in brute force
    sim.simulate(2)
    assert sim.report().force_evaluations == 0
    a = by_uid(sim.agents())
    assert a["x"].tolist() == [0.0, 1e6]


# ---- kd-tree environment (KdTreeEnvironment, kdtree_env.cpp:8-86) on the device ----

@pytest.mark.gpu
@pytest.mark.parametrize("static", [False, True])
@pytest.mark.parametrize("n", [20, 2048, 30000])
def test_gpu_kdtree_matches_reference(engine, oracle_mod, have_ref, static, n):
    """The device kd-tree (balanced median splits on the widest axis, leaves of
    32, rebuilt every update) against the UNMODIFIED reference's kd-tree
    environment: states, forces, partners, evaluation / skip counts per step,
    and the neighbour sets as sorted uid lists. n = 20 is a single leaf,
    2048 has 6 levels, 30000 has 10 with uneven ranges."""
    E, O = engine, oracle_mod
    if not have_ref:
        pytest.skip("reference build unavailable")
    wl = CF.c1_relaxation(n, seed=3)
    ref = O.RefSim(_rp(O, wl, 2, detect_static=static), wl.x, wl.y, wl.z, wl.d)
    sim = E.Simulation(E.SimulationParams(**{**wl.params, "environment": "kdtree", "detect_static_agents": static}))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    for step in range(4):
        ref.simulate(1)
        sim.simulate(1)
        g, o = by_uid(sim.agents()), by_uid(ref.dump())
        assert np.array_equal(g["uid"], o["uid"])
        for k in ("x", "y", "z"):
            assert_close(g[k], o[k], 1e-9, 1.0, f"step {step} {k}")
        for k in ("fx", "fy", "fz"):
            assert_close(g[k], o[k], 1e-9, K, f"step {step} {k}")
        assert np.array_equal(g["partners"], o["partners"]), step
        r, c = sim.report(), ref.counts()
        assert r.force_evaluations == c["force_evaluations"] and r.force_skips == c["force_skips"], step
    env = sim.environment()
    assert env.name() == "kdtree" and env.max_query_radius() == float("inf")
    env.update()
    go, gu = env.neighbors()
    ref.env_update()  # the reference's tree holds copies of the positions (kdtree_env.cpp:13-16)
    ro, ru = ref.neighbors()
    assert _nbr_map(sim.agents()["uid"], go, gu) == _nbr_map(ref.dump()["uid"], ro, ru)
    with pytest.raises(E.AbsimError):
        env.cell_ids()  # no cells without a grid


@pytest.mark.gpu
def test_gpu_kdtree_equals_grid_and_handles_degenerate_clouds(engine):
    """Same population under the grid and the tree: identical integers. Then
    clouds that stress the splits: all agents on a line (two axes of zero
    width), many coincident coordinates (ties at the median), a growing
    population (c2: the tree is rebuilt from the new agent count every step)."""
    E = engine
    wl = CF.c4_large_uniform(1 << 13, seed=2)
    out = []
    for env in ("uniform_grid", "kdtree"):
        sim = E.Simulation(E.SimulationParams(**{**wl.params, "environment": env, "sorting_frequency": 0}))
        sim.add_agents(wl.x, wl.y, wl.z, wl.d)
        sim.simulate(3)
        out.append((by_uid(sim.agents()), sim.report().force_evaluations))
    (a, ea), (b, eb) = out
    assert ea == eb and np.array_equal(a["partners"], b["partners"])
    for k in ("x", "y", "z"):
        assert_close(a[k], b[k], 1e-9, 1.0, k)
    rng = np.random.default_rng(0)
    n = 5000
    clouds = {
        "line": (np.arange(n) * 4.0, np.zeros(n), np.zeros(n)),
        "ties": (rng.integers(0, 12, n) * 9.0, rng.integers(0, 12, n) * 9.0, rng.integers(0, 12, n) * 9.0),
    }
    for name, (x, y, z) in clouds.items():
        res = []
        for env in ("brute_force", "kdtree"):
            sim = E.Simulation(E.SimulationParams(simulation_time_step=0.01, environment=env))
            sim.add_agents(x, y, z, np.full(n, 10.0))
            sim.simulate(2)
            res.append((by_uid(sim.agents()), sim.report().force_evaluations))
        assert res[0][1] == res[1][1], name
        assert np.array_equal(res[0][0]["partners"], res[1][0]["partners"]), name
    wl = CF.c2_proliferation(4)
    res = []
    for env in ("uniform_grid", "kdtree"):
        sim = E.Simulation(E.SimulationParams(**{**wl.params, "environment": env}))
        sim.add_agents(wl.x, wl.y, wl.z, wl.d)
        sim.simulate(45)  # two doublings
        res.append((by_uid(sim.agents()), sim.report()))
    assert res[0][1].final_agent_count == res[1][1].final_agent_count > 64
    assert res[0][1].force_evaluations == res[1][1].force_evaluations
    assert np.array_equal(res[0][0]["uid"], res[1][0]["uid"])
    for k in ("x", "y", "z", "d"):
        assert_close(res[0][0][k], res[1][0][k], 1e-9, 1.0, k)
