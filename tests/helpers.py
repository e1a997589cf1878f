"""Shared helpers for the parity tests (test infrastructure)."""
import hashlib
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")


def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


def digest(st):
    h = hashlib.sha256()
    for a in (st.H, st.HUx, st.HUy):
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def assert_bitwise(a, b, what=""):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, what
    diff = bits(a) != bits(b)
    if diff.any():
        k = int(np.flatnonzero(diff)[0])
        raise AssertionError(f"{what}: {int(diff.sum())} cells differ; first k={k}: {a.reshape(-1)[k]!r} vs {b.reshape(-1)[k]!r}")


def assert_state_bitwise(s1, s2, what=""):
    for f in ("H", "HUx", "HUy"):
        assert_bitwise(getattr(s1, f), getattr(s2, f), f"{what} {f}")
    assert s1.t == s2.t, f"{what} t {s1.t!r} vs {s2.t!r}"


def make(stepper_cls, sc, **kw):
    s = stepper_cls(sc.terrain, sc.params, sc.control, sc.options, **kw)
    if sc.wind.any():
        s.set_wind(sc.wind)
    if sc.sources:
        s.set_sources(sc.sources)
    return s


def golden_factories():
    from paper_1705_00614_b200 import scenarios as S
    return {
        "c1_dry_n0": lambda: S.dam_break_1d(False, 0.0),
        "c1_wet_n002": lambda: S.dam_break_1d(True, 0.02),
        "c1_dry_n002_capped": lambda: S.dam_break_1d(False, 0.02),
        "c2_128": lambda: S.circular_dam_break(128, 8.0, 16),
        "flood64_all_physics": lambda: S.floodplain(64, 50.0),
        "lake128": lambda: S.lake_at_rest(128),
    }
