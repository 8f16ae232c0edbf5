"""Shared test helpers."""
import numpy as np


def by_uid(dump: dict) -> dict:
    order = np.argsort(dump["uid"], kind="stable")
    return {k: v[order] for k, v in dump.items()}


def assert_close(got, ref, rel=1e-9, floor=1.0, what=""):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    tol = rel * np.maximum(np.abs(ref), floor)
    bad = np.abs(got - ref) > tol
    assert not bad.any(), (f"{what}: {bad.sum()} mismatches, worst "
                           f"{np.max(np.abs(got - ref) / np.maximum(np.abs(ref), floor)):.3e}")


def contact_cases():
    """Isolated pairs on a 40-unit lattice (no cross-site interaction, dmax 14),
    one decision boundary per kind, with integer coordinates so every distance
    is exact in fp64:
      0 coincident centres (random direction, test_mechanics.cpp:55-72)
      1 touching, |d| = 0.5(da+db) = 10: overlap == 0 -> zero force, still an
        evaluation (mechanics.cpp:17-19)
      2 d2 == r^2 = (0.5(10+14))^2 = 144: inclusive neighbour (uniform_grid.cpp:223)
      3 one unit past r: not a neighbour
      4 overlapping by 4 on a diagonal (dist = 6 = sqrt(36) exactly: (2,4,4))
      5 overlapping pair with one agent exactly on a box face (x = origin + 14k,
        the floor boundary of box_index_of, uniform_grid.cpp:28-37)."""
    xs, ys, zs, ds = [], [], [], []
    site = 0
    for kind in range(6):
        for rep in range(4):
            bx, by, bz = 40.0 * (site % 5), 40.0 * ((site // 5) % 5), 40.0 * (site // 25)
            site += 1
            a = (bx, by, bz)
            if kind == 0:
                b, da, db = a, 10.0, 10.0
            elif kind == 1:
                b, da, db = (bx + 10.0, by, bz), 10.0, 10.0
            elif kind == 2:
                b, da, db = (bx, by + 12.0, bz), 10.0, 14.0
            elif kind == 3:
                b, da, db = (bx, by, bz + 13.0), 10.0, 14.0
            elif kind == 4:
                b, da, db = (bx + 2.0, by + 4.0, bz + 4.0), 10.0, 10.0
            else:
                a = (-200.0 + 14.0 * (15 + 3 * rep), by, bz + 100.0)
                b, da, db = (a[0] - 3.0, by, bz + 100.0), 10.0, 12.0
            for p, d in ((a, da), (b, db)):
                xs.append(p[0]); ys.append(p[1]); zs.append(p[2]); ds.append(d)
    # one agent with d = dmax at the lattice origin fixes the box length at 14
    xs.append(-200.0); ys.append(-200.0); zs.append(-200.0); ds.append(14.0)
    return [np.array(v, dtype=np.float64) for v in (xs, ys, zs, ds)]
