"""Host-side logic of bench.py (no GPU): the algorithmic byte model the roofline divides by, and
the whole-host oracle fan-out of the CPU baseline."""
import numpy as np
import pytest

import bench
import workloads as W


def test_byte_model_matches_survey_and_stored_form():
    """SURVEY §8 D.3 prints B_min for the 3x3 director form (cfg3 302.0, cfg4 291.5 B per
    element-step); the stored form (d1, d2: DESIGN §4) removes 2 x 3 x 8 = 48 B per element."""
    for name, n, survey in (("cfg3", 64, 302.0), ("cfg4", 8, 291.5)):
        w = W.make(name, n_rods=n)
        assert bench.b_min_per_el_step(w, 12.0) == pytest.approx(survey, abs=1e-9)
        assert bench.b_min_per_el_step(w) == pytest.approx(survey - 48.0, abs=1e-9)
    w = W.make("cfg4", n_rods=8)
    N = 64.0
    assert bench.b_min_per_el_step(w) == pytest.approx((16 * (6 * (N + 1) + 9 * N) + 128) / N)


def test_oracle_fanout_counts_all_work():
    w = W.make("cfg2", n_rods=12)
    r = bench.oracle_fanout_rate(w, 2, 3)
    assert r["value"] > 0 and r["cores"] >= 1
    assert f"x 3 steps" in r["sample"]
    n = min(w.n_rods, 2 * r["cores"])
    assert f"{n} seeded rods" in r["sample"]
