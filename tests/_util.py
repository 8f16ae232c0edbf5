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
