"""CPU: the cascade-depth frontier oracle (oracle/frontier.py) reproduces the
reference's frontier_compare / two_stage_points / three_stage_points bit for bit
on the golden fixtures (tests/golden/make_golden_frontier.py)."""

import numpy as np
import pytest

from oracle import frontier as of
from tests.goldens import catalog_from_doc, frontier_cases

CASES = frontier_cases()


@pytest.mark.parametrize("name", ["jitter00", "jitter05", "wide", "default", "wide_dupgrid"])
def test_oracle_report_matches_reference(name):
    d = CASES[name]
    cat = catalog_from_doc(d["catalog"])
    gap, e2, e3, n2, n3 = of.compare(cat.variants, np.asarray(d["h"]), tuple(d["thresholds"]))
    r = d["report"]
    assert (n2, n3) == (r["n_two"], r["n_three"])
    assert [list(p) for p in e2] == r["envelope_two"]
    assert [list(p) for p in e3] == r["envelope_three"]
    assert gap == r["gap"]


@pytest.mark.parametrize("name", ["jitter00", "wide", "wide_dupgrid"])
def test_oracle_points_match_reference(name):
    d = CASES[name]
    cat = catalog_from_doc(d["catalog"])
    h, thr = np.asarray(d["h"]), tuple(d["thresholds"])
    got2 = [[a, b, list(c)] for a, b, c in of.two_stage(cat.variants, h, thr)]
    got3 = [[a, b, list(c)] for a, b, c in of.three_stage(cat.variants, h, thr)]
    assert got2 == d["two"]
    assert got3 == d["three"]


def test_envelope_helpers_edge_cases():
    assert of.envelope([(1.0, 2.0), (1.0, 1.0), (2.0, 0.5)]) == [(1.0, 1.0), (2.0, 0.5)]
    # collinear middle point is dropped (on the chord)
    assert of.envelope([(0.0, 0.0), (1.0, 1.0), (2.0, 2.0)]) == [(0.0, 0.0), (2.0, 2.0)]
    hull = [(0.0, 1.0), (2.0, 0.0)]
    assert of.envelope_at(hull, 1.0) == 0.5 and of.envelope_at(hull, 3.0) == float("inf")
    assert of.gap(hull, [(5.0, 0.0), (6.0, 0.0)]) == 0.0
