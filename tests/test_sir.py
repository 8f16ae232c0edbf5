"""Config 5 (SIR on a periodic cube, absim_models.h). The reference has no
periodic boundaries; the unmodified reference engine runs the
model with ghost images at the faces through its public hooks
(oracle/ref_harness.cpp, RefSir), which pins the C port bit for bit
(positions, states, infection iterations, S/I/R counts per step); the GPU
is then checked against the port."""
import numpy as np
import pytest

from _util import by_uid
from paper_2301_06984_b200 import configs as CF


def _oparams(O, wl):
    prm = wl.params
    return O.OracleParams(seed=prm["seed"], model=prm["model"], mp=prm["model_params"])


@pytest.mark.parametrize("n,steps,threads", [(3000, 45, 1), (12000, 30, 4)])
def test_sir_port_equals_reference(oracle_mod, have_ref, n, steps, threads):
    """The port's SIR restatement against the reference engine (ghost images):
    identical per-step S/I/R counts, states, infection iterations and
    positions; the step count crosses the recovery time (20)."""
    if not have_ref:
        pytest.skip("reference build (oracle/_ref) not present")
    O = oracle_mod
    wl = CF.c5_sir(n, seed=5)
    p = _oparams(O, wl)
    port = O.PortSim(p, wl.x, wl.y, wl.z, wl.d)
    p.threads = threads
    ref = O.RefSirSim(p, wl.x, wl.y, wl.z)
    hist = []
    for _ in range(steps):
        port.simulate(1)
        hist.append(port.sir_counts())
    ref.simulate(steps)
    assert np.array_equal(ref.count_history(), np.array(hist, np.uint64))
    r = by_uid(ref.dump())
    o = port.dump()
    o["state"], o["t"] = port.sir_state()
    o = by_uid({k: o[k] for k in ("uid", "x", "y", "z", "state", "t")})
    assert np.array_equal(r["uid"], o["uid"])
    for k in ("x", "y", "z", "state", "t"):
        assert np.array_equal(r[k], o[k]), k
    assert hist[-1][2] > 0 and hist[-1][1] > 0


def test_sir_oracle_invariants(oracle_mod):
    O = oracle_mod
    wl = CF.c5_sir(20000, seed=3)
    s = O.PortSim(_oparams(O, wl), wl.x, wl.y, wl.z, wl.d)
    st0, _ = s.sir_state()
    init_inf = int((st0 == 1).sum())
    assert 100 <= init_inf <= 300  # ~1 %
    L = wl.params["model_params"][0]
    prev_r = 0
    for step in range(25):
        s.simulate(1)
        S, I, R = s.sir_counts()
        assert S + I + R == wl.n
        assert R >= prev_r  # recovered never leave R
        prev_r = R
        d = s.dump()
        assert (d["x"] >= 0).all() and (d["x"] <= L).all()
    st, ti = s.sir_state()
    assert R >= init_inf  # every initial infection has recovered after 20 steps
    assert (ti[st == 1] >= 5).all()


@pytest.mark.gpu
def test_sir_gpu_bit_exact(engine, oracle_mod):
    O = oracle_mod
    wl = CF.c5_sir(30000, seed=1)
    sim = engine.Simulation(engine.SimulationParams(**wl.params))
    sim.add_agents(wl.x, wl.y, wl.z, wl.d)
    orc = O.PortSim(_oparams(O, wl), wl.x, wl.y, wl.z, wl.d)
    for step in range(30):
        sim.simulate(1)
        orc.simulate(1)
        assert sim.sir_counts() == orc.sir_counts(), f"counts at step {step}"
    g = sim.agents()
    gs, gt = sim.sir_state()
    g["state"], g["t"] = gs, gt
    o = orc.dump()
    os_, ot = orc.sir_state()
    o["state"], o["t"] = os_, ot
    g, o = by_uid(g), by_uid(o)
    assert np.array_equal(g["uid"], o["uid"])
    for k in ("x", "y", "z", "state", "t"):
        assert np.array_equal(g[k], o[k]), k
    assert sim.sir_counts()[2] > 0


@pytest.mark.gpu
def test_sir_rejects_small_box(engine):
    with pytest.raises(ValueError):
        engine.Simulation(engine.SimulationParams(model=engine.MODEL_SIR, model_params=[4.0, 2.0, 1.0, 20.0, 0.1]))
