"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED
reference engine (oracle/_ref/libabsim_ref.so, built from
/root/reference/proj/src by oracle/Makefile) on small seeded cases.

Run in the build container (needs the reference build):
    python tests/golden/make_golden.py
The .npz files are committed; the GPU box never needs /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2301_06984_b200 import configs as CF  # noqa: E402

CASES = {
    # name: (workload factory, steps, extra oracle params)
    "c1_n2048_s0": (lambda: CF.c1_relaxation(2048, seed=0), 10, {}),
    "c2_side4_s0": (lambda: CF.c2_proliferation(side=4, seed=0), 60, {}),
    "c3_n2000_s0": (lambda: CF.c3_spheroid(2000, seed=0), 6, {}),
    "c4_n2048_s0": (lambda: CF.c4_large_uniform(2048, seed=0), 12, {}),
}


def oparams(wl):
    prm = wl.params
    return O.OracleParams(seed=prm.get("seed", 42), dt=prm.get("simulation_time_step", 0.1),
                          detect_static=prm.get("detect_static_agents", False),
                          model=prm.get("model", 0), mp=prm.get("model_params", [0.0] * 8),
                          sorting_frequency=prm.get("sorting_frequency", 0))


def make(name):
    factory, steps, _ = CASES[name]
    wl = factory()
    ref = O.RefSim(oparams(wl), wl.x, wl.y, wl.z, wl.d, wl.mask)
    g = ref.env_update()
    cell = ref.cell_ids()
    off, nbr = ref.neighbors()
    uid0 = ref.dump()["uid"]
    ref.simulate(steps)
    out = ref.dump()
    c = ref.counts()
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"),
        steps=steps, origin=g["origin"], box=g["box"], dmax=g["dmax"], dims=g["dims"],
        cell_uid=uid0, cell_id=cell, nbr_offsets=off, nbr_uids=nbr,
        counts=np.array([c[k] for k in ("agents", "uid_count", "iterations", "force_evaluations",
                                        "force_skips", "agents_added")], np.uint64),
        **{f"final_{k}": v for k, v in out.items()})
    print(name, c)


if __name__ == "__main__":
    for n in CASES:
        make(n)
