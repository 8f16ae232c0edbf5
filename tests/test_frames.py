"""abs_gpu_run_frames (the host-boundary pipeline used for the end-to-end
number): every frame must equal upload -> simulate -> download of the same
inputs, i.e. the oracle run on those inputs, while frames overlap their
copies with compute."""
import numpy as np
import pytest

from _util import assert_close
from paper_2301_06984_b200 import configs as CF

pytestmark = pytest.mark.gpu


def _oracle_positions(O, wl, iterations):
    prm = wl.params
    orc = O.PortSim(O.OracleParams(seed=prm.get("seed", 0), dt=prm.get("simulation_time_step", 0.1)),
                    wl.x, wl.y, wl.z, wl.d)
    orc.simulate(iterations)
    o = orc.dump()
    i = np.argsort(o["uid"])
    return {k: o[k][i] for k in ("uid", "x", "y", "z")}


@pytest.mark.parametrize("iterations", [1, 3])
def test_frames_match_oracle(engine, oracle_mod, iterations):
    E, O = engine, oracle_mod
    wls = [CF.c1_relaxation(3000 + 500 * f, seed=f) for f in range(3)]
    sim = E.Simulation(E.SimulationParams(**{**wls[0].params, "record_forces": False}))
    outs = [tuple(np.zeros(len(w.x) + 7) for _ in range(3)) for w in wls]
    uids = [np.zeros(len(w.x) + 7, np.uint64) for w in wls]
    counts = sim.run_frames([(w.x, w.y, w.z, w.d) for w in wls], outs, iterations=iterations, uids=uids)
    assert counts == [len(w.x) for w in wls]
    for w, o, u, n in zip(wls, outs, uids, counts):
        ref = _oracle_positions(O, w, iterations)
        i = np.argsort(u[:n])
        assert np.array_equal(u[:n][i], ref["uid"])
        for k, a in zip("xyz", o):
            assert_close(a[:n][i], ref[k], 1e-9, 1.0, f"frame {k}")


def test_frames_equal_sequential_api(engine):
    E = engine
    wl = CF.c4_large_uniform(1 << 15, seed=3)
    prm = {**wl.params, "record_forces": False, "sorting_frequency": 2}
    seq = E.Simulation(E.SimulationParams(**prm))
    want = []
    for f in range(4):  # the per-frame sequence the pipeline replaces
        seq.add_agents(wl.x, wl.y, wl.z, wl.d)
        seq.set_iteration(5 + 2 * f)
        seq.simulate(2)
        a = seq.agents()
        i = np.argsort(a["uid"])
        want.append((a["x"][i], a["y"][i], a["z"][i]))
    sim = E.Simulation(E.SimulationParams(**prm))
    outs = [tuple(np.zeros(wl.n) for _ in range(3)) for _ in range(4)]
    uids = [np.zeros(wl.n, np.uint64) for _ in range(4)]
    sim.run_frames([(wl.x, wl.y, wl.z, wl.d)] * 4, outs, iterations=2, first_iteration=5, uids=uids)
    for f in range(4):
        i = np.argsort(uids[f])
        assert np.array_equal(uids[f][i], np.arange(wl.n, dtype=np.uint64))
        for k in range(3):
            assert_close(outs[f][k][i], want[f][k], 1e-9, 1.0, f"frame {f}")
    assert sim.iteration == 5 + 2 * 4


def test_frames_output_capacity_error(engine):
    E = engine
    wl = CF.c1_relaxation(2000, seed=1)
    sim = E.Simulation(E.SimulationParams(**wl.params))
    outs = [tuple(np.zeros(100) for _ in range(3))]
    with pytest.raises(E.AbsimError):
        sim.run_frames([(wl.x, wl.y, wl.z, wl.d)], outs)


def test_frames_with_divisions(engine):
    """A model that adds agents inside a frame (models::GrowDivide): outputs
    grow past the input count and still equal the sequential API."""
    E = engine
    wl = CF.ref_proliferation(216)
    prm = {**wl.params, "record_forces": False}
    seq = E.Simulation(E.SimulationParams(**prm))
    seq.add_agents(wl.x, wl.y, wl.z, wl.d)
    seq.set_iteration(0)
    seq.simulate(7)
    a = seq.agents()
    i = np.argsort(a["uid"])
    sim = E.Simulation(E.SimulationParams(**prm))
    cap = 8 * wl.n
    outs = [tuple(np.zeros(cap) for _ in range(3)) for _ in range(2)]
    uids = [np.zeros(cap, np.uint64) for _ in range(2)]
    counts = sim.run_frames([(wl.x, wl.y, wl.z, wl.d)] * 2, outs, iterations=7, first_iteration=0, uids=uids)
    assert counts[0] > wl.n
    # frame 0 starts at iteration 0 like the sequential run
    n = counts[0]
    assert n == len(a["uid"])
    j = np.argsort(uids[0][:n])
    assert np.array_equal(uids[0][:n][j], a["uid"][i])
    for k, o in zip("xyz", outs[0]):
        assert_close(o[:n][j], a[k][i], 1e-9, 1.0, f"divisions {k}")


def test_frames_edge_cases(engine):
    """Empty frames and a one-agent frame (uniform_grid.cpp:66-72: N = 0 gives
    dims {1,1,1}); a lone agent has no neighbours and does not move."""
    E = engine
    sim = E.Simulation(E.SimulationParams(simulation_time_step=0.01))
    e = np.zeros(0)
    one = (np.array([1.0]), np.array([2.0]), np.array([3.0]), np.array([10.0]))
    outs = [tuple(np.zeros(4) for _ in range(3)) for _ in range(3)]
    counts = sim.run_frames([(e, e, e, e), one, (e, e, e, e)], outs, iterations=2)
    assert counts == [0, 1, 0]
    assert (outs[1][0][0], outs[1][1][0], outs[1][2][0]) == (1.0, 2.0, 3.0)
    assert sim.report().force_evaluations == 0
