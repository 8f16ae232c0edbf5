"""CPU: pin the C restatement (oracle/absim_oracle.c) against the unmodified
reference (oracle/_ref, built from /root/reference/proj/src) and against the
reference's own known answers (proj/tests/*.cpp)."""
import math

import numpy as np
import pytest

from paper_2301_06984_b200 import configs as CF
from _util import by_uid, contact_cases

FIELDS = ["uid", "x", "y", "z", "d", "fx", "fy", "fz", "partners", "flags", "volume"]


def _pair(O, wl, **extra):
    prm = dict(wl.params)
    p = O.OracleParams(seed=prm.get("seed", 42), dt=prm.get("simulation_time_step", 0.1),
                       detect_static=prm.get("detect_static_agents", False),
                       model=prm.get("model", 0), mp=prm.get("model_params", [0.0] * 8),
                       sorting_frequency=prm.get("sorting_frequency", 0), **extra)
    return p


def _bitwise(a, b):
    da, db = a.dump(), b.dump()
    for k in FIELDS:
        assert np.array_equal(da[k], db[k]), k
    assert a.counts() == b.counts()


@pytest.mark.parametrize("case", ["c1", "c1_static", "c2", "c3", "c4"])
def test_port_bitwise_equals_reference(oracle_mod, have_ref, case):
    O = oracle_mod
    if not have_ref:
        pytest.skip("reference build unavailable")
    if case.startswith("c1"):
        wl = CF.c1_relaxation(2500, seed=1)
        steps = 6
    elif case == "c2":
        wl = CF.c2_proliferation(side=4, seed=2)
        steps = 60
    elif case == "c3":
        wl = CF.c3_spheroid(3000, seed=3)
        steps = 5
    else:
        wl = CF.c4_large_uniform(3000, seed=4)
        steps = 12
    p = _pair(O, wl)
    if case == "c1_static":
        p.detect_static = True
        p.threshold = 5.0
    ref = O.RefSim(p, wl.x, wl.y, wl.z, wl.d, wl.mask)
    port = O.PortSim(p, wl.x, wl.y, wl.z, wl.d, wl.mask)
    g1, g2 = ref.env_update(), port.env_update()
    for k in ("origin", "box", "dmax", "dims", "indexed"):
        assert np.array_equal(np.asarray(g1[k]), np.asarray(g2[k])), k
    assert np.array_equal(ref.cell_ids(), port.cell_ids())
    o1, u1 = ref.neighbors()
    o2, u2 = port.neighbors()
    assert np.array_equal(o1, o2) and np.array_equal(u1, u2)
    ref.simulate(steps)
    port.simulate(steps)
    _bitwise(ref, port)


@pytest.mark.parametrize("static", [False, True])
def test_port_contact_boundaries_equal_reference(oracle_mod, have_ref, static):
    """Exact decision boundaries (coincident centres, touching pairs,
    d2 == r^2, agents on box faces; tests/_util.py:contact_cases): the port
    reproduces the reference bit for bit, so the GPU test of the same cases
    (test_gpu_parity.py) is pinned to the reference through it."""
    O = oracle_mod
    if not have_ref:
        pytest.skip("reference build unavailable")
    x, y, z, d = contact_cases()
    p = O.OracleParams(seed=3, dt=0.01, detect_static=static, model=0, mp=[0.0] * 8,
                       sorting_frequency=0, threshold=0.0, fixed_box=0.0)
    ref = O.RefSim(p, x, y, z, d)
    port = O.PortSim(p, x, y, z, d)
    g1, g2 = ref.env_update(), port.env_update()
    for k in ("origin", "box", "dmax", "dims", "indexed"):
        assert np.array_equal(np.asarray(g1[k]), np.asarray(g2[k])), k
    assert np.array_equal(ref.cell_ids(), port.cell_ids())
    o1, u1 = ref.neighbors()
    o2, u2 = port.neighbors()
    assert np.array_equal(o1, o2) and np.array_equal(u1, u2)
    ref.simulate(4)
    port.simulate(4)
    _bitwise(ref, port)
    c = port.counts()
    if static:  # the zero-force pairs (touching, d2 == r^2, past r) settle and are skipped
        assert c["force_skips"] > 0
    else:  # 44 evaluations per step: 2 per pair, 1 for the past-r pair (only its d = 14 side sees it)
        assert c["force_evaluations"] == 4 * 44 and c["force_skips"] == 0


@pytest.mark.parametrize("k,max_disp,threshold", [(5.0, 0.5, 0.0), (2.0, 3.0, 4.0), (0.5, 0.05, 1.0)])
def test_port_mechanics_parameters_equal_reference(oracle_mod, have_ref, k, max_disp, threshold):
    """repulsion_coefficient / max_displacement / force_threshold away from
    their defaults (params.hpp:17-52): port == reference bit for bit."""
    O = oracle_mod
    if not have_ref:
        pytest.skip("reference build unavailable")
    wl = CF.c1_relaxation(3000, seed=11)
    p = O.OracleParams(seed=11, dt=0.1, k=k, max_disp=max_disp, threshold=threshold)
    ref = O.RefSim(p, wl.x, wl.y, wl.z, wl.d)
    port = O.PortSim(p, wl.x, wl.y, wl.z, wl.d)
    ref.simulate(3)
    port.simulate(3)
    _bitwise(ref, port)


def test_port_sort_equals_reference(oracle_mod, have_ref):
    O = oracle_mod
    if not have_ref:
        pytest.skip("reference build unavailable")
    wl = CF.c1_relaxation(1500, seed=7)
    p = _pair(O, wl)
    ref = O.RefSim(p, wl.x, wl.y, wl.z, wl.d)
    port = O.PortSim(p, wl.x, wl.y, wl.z, wl.d)
    ref.sort()
    port.env_update()
    port.sort()
    assert np.array_equal(ref.dump()["uid"], port.dump()["uid"])


# ---- known answers from the reference's own tests ------------------------

def test_morton_known_answers(oracle_mod):
    O = oracle_mod
    assert O.morton_encode3(0, 0, 0) == 0  # test_morton.cpp:72-79
    assert O.morton_encode3(1, 1, 1) == 7
    assert O.morton_encode3(1, 0, 0) == 1
    assert O.morton_encode3(0, 1, 0) == 2
    assert O.morton_encode3(0, 0, 1) == 4
    assert O.morton_encode3(2, 3, 5) == 286
    assert O.morton_encode3(0x1FFFFF, 0x1FFFFF, 0x1FFFFF) == 0x7FFFFFFFFFFFFFFF
    with pytest.raises(ValueError):
        O.morton_encode3(1 << 21, 0, 0)
    rng = np.random.default_rng(7)
    for _ in range(200):
        x, y, z = (int(v) for v in rng.integers(0, 1 << 21, 3))
        assert O.morton_decode3(O.morton_encode3(x, y, z)) == (x, y, z)


def _enumerate_runs(dims):
    codes = []
    for z in range(dims[2]):
        for y in range(dims[1]):
            for x in range(dims[0]):
                if dims[2] == 1:
                    c = 0
                    for i in range(31):
                        c |= ((x >> i) & 1) << (2 * i) | ((y >> i) & 1) << (2 * i + 1)
                else:
                    c = 0
                    for i in range(21):
                        c |= ((x >> i) & 1) << (3 * i) | ((y >> i) & 1) << (3 * i + 1) | ((z >> i) & 1) << (3 * i + 2)
                codes.append(c)
    codes.sort()
    table, prev = [], None
    for r, c in enumerate(codes):
        if c - r != prev:
            table.append((r, c - r))
            prev = c - r
    return table


def test_offsets_table_known_answers(oracle_mod):
    O = oracle_mod
    assert O.offsets_table([3, 3, 1]) == [(0, 0), (5, 1), (6, 2), (8, 4)]  # test_morton.cpp:137-149
    assert O.offsets_table([4, 4, 1]) == [(0, 0)]
    for dims in ([3, 2, 2], [5, 7, 3], [9, 9, 9], [1, 6, 2], [8, 3, 1]):
        assert O.offsets_table(dims) == _enumerate_runs(dims)


def test_prefix_sum(oracle_mod):
    O = oracle_mod
    v, t = O.exclusive_scan([1, 2, 3])
    assert t == 6 and list(v) == [0, 1, 3]
    rng = np.random.default_rng(13)
    a = rng.integers(0, 1000, 100000)
    v, t = O.exclusive_scan(a)
    assert t == int(a.sum()) and np.array_equal(v, np.concatenate([[0], np.cumsum(a)[:-1]]))


def test_removal_worked_example(oracle_mod):
    """test_commit.cpp:99-119: removing slots {1,4,6} of 7 leaves [u0,u5,u2,u3]."""
    O = oracle_mod
    x = np.arange(7, dtype=float)
    s = O.PortSim(O.OracleParams(), x, np.zeros(7), np.zeros(7), np.ones(7))
    s.remove([1, 4, 6])
    assert list(s.dump()["uid"]) == [0, 5, 2, 3]
    s2 = O.PortSim(O.OracleParams(), np.arange(6, dtype=float), np.zeros(6), np.zeros(6), np.ones(6))
    s2.remove([1, 5])  # test_commit.cpp:263-289 (before the append)
    assert list(s2.dump()["uid"]) == [0, 4, 2, 3]


def _lattice(s, spacing):
    pts = [(x * spacing, y * spacing, z * spacing) for x in range(s) for y in range(s) for z in range(s)]
    return [np.array(v, dtype=float) for v in zip(*pts)]


def test_static_lattice_known_answer(oracle_mod):
    """test_scheduler.cpp:464-488: 27 touching agents -> 108 evals, then skips."""
    O = oracle_mod
    x, y, z = _lattice(3, 10.0)
    s = O.PortSim(O.OracleParams(detect_static=True), x, y, z, np.full(27, 10.0))
    s.simulate(1)
    c = s.counts()
    assert c["force_evaluations"] == 108 and c["force_skips"] == 0
    s.simulate(1)
    c = s.counts()
    assert c["force_evaluations"] == 108 and c["force_skips"] == 27
    s.simulate(1)
    assert s.counts()["force_skips"] == 54
    assert (s.dump()["flags"] & 1).sum() == 27


def test_cancelling_triple_known_answer(oracle_mod):
    """test_scheduler.cpp:490-519."""
    O = oracle_mod
    s = O.PortSim(O.OracleParams(detect_static=True, threshold=10.0), np.array([0.0, 10.0, 20.0]),
                  np.zeros(3), np.zeros(3), np.full(3, 12.0))
    s.simulate(1)
    assert s.counts()["force_evaluations"] == 4 and s.counts()["force_skips"] == 0
    s.simulate(2)
    assert s.counts()["force_evaluations"] == 8 and s.counts()["force_skips"] == 4
    d = by_uid(s.dump())
    assert sorted(int(u) for u, f in zip(d["uid"], d["flags"]) if f & 1) == [0, 2]
    assert list(d["x"]) == [0.0, 10.0, 20.0]


def test_static_front_known_answer(oracle_mod, have_ref):
    """test_scheduler.cpp:521-534: growth wakes shells; {18,19,20,24,25,26} stay static."""
    O = oracle_mod
    x, y, z = _lattice(3, 10.0)
    mask = np.array([1 if (i // 9 == 0 and (i // 3) % 3 == 1) else 0 for i in range(27)], np.uint8)
    p = O.OracleParams(detect_static=True, model=O.MODEL_GROW, mp=[0.5, 20.0])
    s = O.PortSim(p, x, y, z, np.full(27, 10.0), mask)
    s.simulate(3)
    d = by_uid(s.dump())
    assert sorted(int(u) for u, f in zip(d["uid"], d["flags"]) if f & 1) == [18, 19, 20, 24, 25, 26]
    if have_ref:  # the reference's own builder gives the same population
        r = O.RefSim.builtin(p, "static_front", 27)
        r.simulate(3)
        _bitwise(r, s)


def test_grid_floor_clamp_known_answer(oracle_mod):
    """test_grid.cpp:68-86: (19.999,20,39.9) -> (0,1,1); far corner clamps."""
    O = oracle_mod
    x = np.array([0.0, 100.0, 19.999, 100.0])
    y = np.array([0.0, 100.0, 20.0, 100.0])
    z = np.array([0.0, 100.0, 39.9, 100.0])
    s = O.PortSim(O.OracleParams(fixed_box=20.0), x, y, z, np.full(4, 10.0))
    g = s.env_update()
    assert list(g["dims"]) == [6, 6, 6] and list(g["origin"]) == [0, 0, 0]
    ids = s.cell_ids()
    assert ids[2] == 0 + 6 * (1 + 6 * 1)
    assert ids[3] == 5 + 6 * (5 + 6 * 5)


def test_errors_match_reference(oracle_mod):
    O = oracle_mod
    s = O.PortSim(O.OracleParams(fixed_box=5.0), np.zeros(2), np.zeros(2), np.zeros(2), np.full(2, 10.0))
    with pytest.raises(RuntimeError, match="fixed box"):
        s.simulate(1)
    s = O.PortSim(O.OracleParams(), np.array([0.0, math.inf]), np.zeros(2), np.zeros(2), np.full(2, 10.0))
    with pytest.raises(RuntimeError, match="not finite"):
        s.simulate(1)
    with pytest.raises(RuntimeError, match="diameter"):
        O.PortSim(O.OracleParams(), np.zeros(1), np.zeros(1), np.zeros(1), np.zeros(1))


# ---- the reference's own behaviour models ---------------------
def _port_from(O, wl, **kw):
    prm = wl.params
    p = O.OracleParams(seed=prm["seed"], model=prm["model"], mp=prm["model_params"],
                       fixed_box=prm.get("fixed_box_length", 0.0), **kw)
    s = O.PortSim(p, wl.x, wl.y, wl.z, wl.d)
    s.set_tags(wl.tags)
    s.set_rng_counters(wl.rng_counters)
    return s, p


def _same_state(a, b, what):
    da, db = a.dump(), b.dump()
    for k in ("uid", "x", "y", "z", "d", "partners", "flags"):
        assert np.array_equal(da[k], db[k]), f"{what}: {k}"
    assert np.array_equal(a.tags(), b.tags()), f"{what}: tags"
    assert np.array_equal(a.rng_counters(), b.rng_counters()), f"{what}: rng counters"
    assert a.counts() == b.counts(), f"{what}: counts"


def test_growdivide_matches_reference_builder(oracle_mod, have_ref):
    """models::GrowDivide on the reference's own build_proliferation lattice:
    daughters from the agent's RandomStream (cos/sin), tags and counters."""
    if not have_ref:
        pytest.skip("reference build unavailable")
    O = oracle_mod
    wl = CF.ref_proliferation(64)
    port, p = _port_from(O, wl)
    ref = O.RefSim.builtin(p, "proliferation", 64)
    for chunk in range(4):
        ref.simulate(6)
        port.simulate(6)
        _same_state(ref, port, f"grow-divide after {6 * (chunk + 1)}")
    assert ref.counts()["agents"] > 64


def test_cohere_matches_reference_builder(oracle_mod, have_ref):
    """models::Cohere on the reference's own build_clustering population
    (tags uid % 2, box pinned to the attraction radius)."""
    if not have_ref:
        pytest.skip("reference build unavailable")
    O = oracle_mod
    wl = CF.ref_clustering(600, seed=7)
    port, p = _port_from(O, wl)
    ref = O.RefSim.builtin(p, "clustering", 600)
    d0 = ref.dump()
    assert np.array_equal(d0["x"], wl.x) and np.array_equal(ref.tags(), wl.tags)
    assert np.array_equal(ref.rng_counters(), wl.rng_counters)
    for chunk in range(3):
        ref.simulate(4)
        port.simulate(4)
        _same_state(ref, port, f"cohere after {4 * (chunk + 1)}")


@pytest.mark.parametrize("model,sf", [(5, 3), (7, 0), (7, 3)])
def test_reordered_storage_matches_reference(oracle_mod, have_ref, model, sf):
    """Daughter uids and removal slots follow the reference's storage order
    after Morton sorts (sorting_frequency) and removals (remove_self, commit:
    removals before additions, commit.cpp:164-225): GrowDivide with sorts,
    GrowDivide + removals, both together; port == unmodified reference."""
    if not have_ref:
        pytest.skip("reference build unavailable")
    O = oracle_mod
    wl = CF.ref_proliferation_die(216, p_remove=0.03, sorting_frequency=sf) if model == 7 else CF.ref_proliferation(216)
    prm = dict(wl.params, sorting_frequency=sf)
    p = O.OracleParams(seed=prm["seed"], model=prm["model"], mp=prm["model_params"], sorting_frequency=sf)
    port = O.PortSim(p, wl.x, wl.y, wl.z, wl.d)
    port.set_tags(wl.tags)
    port.set_rng_counters(wl.rng_counters)
    ref = O.RefSim(p, wl.x, wl.y, wl.z, wl.d)  # fresh agents: tags and stream counters 0, as the lattice's
    assert not wl.tags.any() and not wl.rng_counters.any()
    for chunk in range(5):
        ref.simulate(5)
        port.simulate(5)
        _same_state(ref, port, f"model {model} sf {sf} after {5 * (chunk + 1)}")
    c = ref.counts()
    assert c["agents_added"] > 0 and (model != 7 or c["agents_removed"] > 0)
