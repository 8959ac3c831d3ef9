"""Pin the CPU oracle to the genuine reference's outputs (golden fixtures).

CPU-only.  The fixtures were produced by cascadesim itself
(tests/golden/make_golden.py); passing here means the oracle that every GPU
parity test trusts reproduces the reference bit for bit."""

import random

import numpy as np
import pytest

from oracle import grid as og
from oracle import planner as op
from paper_2509_00642_b200.catalog import select_candidates
from tests.goldens import (PROFILE_CASES, catalog_from_doc, load_json, load_npz, row_tuples,
                           rows_ns, scores_of)


def _pool(doc):
    cat = catalog_from_doc(doc["catalog"])
    pool = select_candidates(cat, doc["eps"], doc["eps"])
    assert [v.id for v in pool] == doc.get("pool", [v.id for v in pool])
    return pool


@pytest.mark.parametrize("variant", ["default", "bypass01", "unsorted", "duplicates",
                                     "negzero", "dense33"])
def test_oracle_matches_reference_conftest160(variant):
    doc = load_json("conftest160")
    rec = load_npz("conftest160")
    pool = _pool(doc)
    case = doc["variants"][variant]
    rows = og.profile_rows(pool, rec["h"], noise=rec["noise"], thresholds=case["thresholds"])
    assert rows == row_tuples(case["table"])


def test_oracle_scores_match_stored_scores():
    rec = load_npz("c1")
    doc = load_json("c1")
    pool = _pool(doc)
    _, scores = og.model_arrays(pool, rec["h"], rec["noise"])
    for mid, s in scores_of(rec).items():
        assert np.array_equal(scores[mid], s)


def test_oracle_matches_reference_c1():
    doc = load_json("c1")
    rec = load_npz("c1")
    pool = _pool(doc)
    rows = og.profile_rows(pool, rec["h"], scores=scores_of(rec), thresholds=doc["thresholds"])
    assert len(rows) == 374
    assert rows == row_tuples(doc["table"])


@pytest.mark.parametrize("name", PROFILE_CASES)
def test_oracle_matches_reference_synthetic(name):
    doc = load_json(name)
    rec = load_npz(name)
    pool = _pool(doc)
    rows = og.profile_rows(pool, rec["h"], scores=scores_of(rec), thresholds=doc["thresholds"])
    assert rows == row_tuples(doc["table"])


def test_pareto_kats():
    for case in load_json("pareto_kats")["cases"]:
        lat = [r[0] for r in case["rows"]]
        qual = [r[1] for r in case["rows"]]
        assert og.pareto_keep(lat, qual) == case["kept"]


@pytest.mark.parametrize("n", list(range(1, 140)) + [255, 256, 257, 1000, 4099, 65537, 100003])
def test_pairwise_sum_is_numpy(n):
    rng = np.random.default_rng(n)
    a = rng.uniform(18.0, 40.0, n)
    assert og.pairwise_sum(a.tolist()) == float(np.add.reduce(a))
    assert og.pairwise_sum(a.tolist()) / n == float(a.mean())
    leaves = og.pairwise_leaves(n)
    assert sum(m for _, m in leaves) == n
    assert all(lo2 == lo1 + m1 for (lo1, m1), (lo2, _) in zip(leaves, leaves[1:]))


def _check_plan(got, want):
    assert got["row_index"] == want["row_index"]
    assert got["workers"] == want["workers"]
    assert got["batches"] == want["batches"]
    assert got["path_latency_s"] == want["path_latency_s"]
    assert got["fidelity_cost"] == want["fidelity_cost"]
    assert got["infeasible"] == want["infeasible"]


def test_oracle_planner_random200():
    cases = load_json("planner_random200")["cases"]
    kinds = set()
    for case in cases:
        cat = catalog_from_doc(case["catalog"])
        rows = rows_ns(case["rows"])
        for fn, key, err in ((op.solve, "solve", "solve_error"), (op.brute_force, "brute", "brute_error")):
            try:
                got = fn(rows, cat, case["lam"], case["queues"], case["workers"], case["t_slo"],
                         case["alpha"])
            except op.OraclePlannerError as exc:
                assert case[key] is None and case[err] == str(exc)
                kinds.add("refused")
                continue
            _check_plan(got, case[key])
            kinds.add("infeasible" if got["infeasible"] else "feasible")
            if not got["infeasible"]:
                assert op.audit(got, rows[got["row_index"]], cat, case["workers"],
                                case["t_slo"], case["alpha"]) == []
    assert kinds == {"refused", "infeasible", "feasible"}


def test_oracle_planner_conftest_sweep():
    doc = load_json("planner_conftest")
    cat = catalog_from_doc(doc["catalog"])
    rows = rows_ns(doc["table"]["rows"])
    for pt in doc["points"]:
        got = op.solve(rows, cat, pt["lam"], pt["queues"], pt["workers"], pt["t_slo"], pt["alpha"])
        _check_plan(got, pt["solve"])


def test_oracle_planner_rejects_negative_demand():
    doc = load_json("planner_conftest")
    cat = catalog_from_doc(doc["catalog"])
    with pytest.raises(op.OraclePlannerError, match="negative demand"):
        op.solve(rows_ns(doc["table"]["rows"]), cat, -1.0)
    random.Random(0)
