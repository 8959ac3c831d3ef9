"""GPU parity: libhadis_b200 vs the reference (golden fixtures) and the oracle.

Every test here runs the CUDA path through the C ABI (via the package's
ctypes layer) and compares with the reference's own outputs or with the CPU
oracle on the same seeded inputs."""

import math
import random

import numpy as np
import pytest

from oracle import grid as og
from oracle import planner as op
from paper_2509_00642_b200 import (GridProfiler, default_catalog, pareto_prune, profile_records,
                                   solve, solve_many)
from paper_2509_00642_b200.catalog import select_candidates
from paper_2509_00642_b200.planner import PlannerError
from paper_2509_00642_b200.profiler import GridSpec, light_scores
from tests.goldens import (PROFILE_CASES, catalog_from_doc, load_json, load_npz, row_tuples,
                           rows_ns, scores_of)

pytestmark = pytest.mark.gpu


def tuples(table):
    return [(r.light_id, r.heavy_id, r.theta, r.tau, r.r_light, r.r_heavy, r.fidelity_cost,
             r.mean_latency_s) for r in table.rows]


def assert_rows_close(got, want, rel=1e-9):
    """Identical membership/order, bit-exact counts-derived fields, fid within rel."""
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g[:6] == w[:6] and g[7] == w[7], (g, w)
        assert math.isclose(g[6], w[6], rel_tol=rel, abs_tol=0.0), (g, w)


def _golden_pool(doc):
    cat = catalog_from_doc(doc["catalog"])
    return cat, select_candidates(cat, doc["eps"], doc["eps"])


@pytest.mark.parametrize("variant", ["default", "bypass01", "unsorted", "duplicates", "negzero",
                                     "dense33"])
@pytest.mark.parametrize("exact", [True, False])
def test_conftest160_matches_reference(gpu_device, variant, exact):
    doc = load_json("conftest160")
    rec = load_npz("conftest160")
    cat, pool = _golden_pool(doc)
    case = doc["variants"][variant]
    table = profile_records(cat, rec["h"], scores=scores_of(rec), thresholds=case["thresholds"],
                            exact_fid=exact)
    want = row_tuples(case["table"])
    if exact:
        assert tuples(table) == want
    else:
        assert_rows_close(tuples(table), want)


@pytest.mark.parametrize("name", ("c1",) + PROFILE_CASES)
@pytest.mark.parametrize("exact", [True, False])
def test_golden_profiles_match_reference(gpu_device, name, exact):
    doc = load_json(name)
    rec = load_npz(name)
    cat, pool = _golden_pool(doc)
    table = profile_records(cat, rec["h"], scores=scores_of(rec), thresholds=doc["thresholds"],
                            eps_latency=doc["eps"], eps_quality=doc["eps"], exact_fid=exact)
    want = row_tuples(doc["table"])
    if exact:
        assert tuples(table) == want
    else:
        assert_rows_close(tuples(table), want)


@pytest.mark.parametrize("seed,n,k,hmode", [(1, 1, 5, "u"), (2, 7, 9, "u"), (3, 300, 17, "ties"),
                                            (4, 1000, 40, "u"), (5, 4000, 64, "ties"),
                                            (6, 2500, 33, "clip"), (7, 129, 128, "u"),
                                            (8, 50, 1, "u"), (9, 50, 2, "ties"),
                                            (10, 64, 3, "const"), (11, 200, 6, "grid"),
                                            (12, 333, 12, "sparse")])
def test_random_records_match_oracle(gpu_device, seed, n, k, hmode):
    """Edge cases as the reference's tests have them: one record, one or two
    thresholds, all-equal hardness, hardness exactly on the thresholds, a
    non-uniform (guided-binning) grid."""
    rng = np.random.default_rng(seed)
    cat = default_catalog()
    pool = select_candidates(cat, 0.1, 0.1)
    if hmode == "ties":
        h = rng.choice(np.round(rng.uniform(0.0, 1.0, 37), 2), n)
    elif hmode == "const":
        h = np.full(n, 0.37)
    elif hmode == "grid":
        h = rng.choice(np.linspace(0.0, 1.0, k), n)
    else:
        h = rng.uniform(0.0, 1.0, n)
    sigma = 0.3 if hmode == "clip" else 0.05
    noise = rng.normal(0.0, sigma, n)
    if hmode == "sparse":
        thr = tuple(rng.permutation(np.round(np.sort(rng.uniform(0.0, 1.0, k)) ** 3, 6)).tolist())
    else:
        thr = tuple(rng.permutation(np.linspace(0.0, 1.0, k)).tolist())
    want = og.profile_rows(pool, h, noise=noise, thresholds=thr)
    got = profile_records(pool, h, noise=noise, thresholds=thr, exact_fid=True)
    assert tuples(got) == want
    got2 = profile_records(pool, h, noise=noise, thresholds=thr, exact_fid=False)
    assert_rows_close(tuples(got2), want)


def test_fid_exact_kernel_is_numpy(gpu_device):
    import torch
    from paper_2509_00642_b200 import _lib
    rng = np.random.default_rng(3)
    lib = _lib.load()
    for n in (1, 5, 8, 127, 128, 129, 1000, 4099, 65537, 1000003):
        h = rng.uniform(0, 1, n)
        s = rng.uniform(0, 1, (2, n))
        cells = [(0, 0.3, 0.5, 30.0, 8.0, 25.0, 3.0), (1, 0.0, 1.0, 36.0, 12.0, 23.0, 3.0),
                 (1, 0.7, 0.2, 31.0, 8.0, 26.0, 5.0)]
        dev = torch.device("cuda")
        d_h = torch.from_numpy(h).to(dev)
        d_s = torch.from_numpy(s).to(dev)
        slot = torch.tensor([c[0] for c in cells], dtype=torch.int32, device=dev)
        th = torch.tensor([c[1] for c in cells], dtype=torch.float64, device=dev)
        ta = torch.tensor([c[2] for c in cells], dtype=torch.float64, device=dev)
        par = torch.tensor([c[3:] for c in cells], dtype=torch.float64, device=dev)
        out = torch.empty(len(cells), dtype=torch.float64, device=dev)
        _lib.check(lib.hadis_fid_exact(_lib.ptr(d_h), _lib.ptr(d_s), n, len(cells), _lib.ptr(slot),
                                       _lib.ptr(th), _lib.ptr(ta), _lib.ptr(par), _lib.ptr(out),
                                       _lib.stream_handle()), "fid_exact")
        got = out.cpu().tolist()
        for c, g in zip(cells, got):
            heavy = (h > c[1]) | (s[c[0]] < c[2])
            want = float(np.where(heavy, c[5] + c[6] * h, c[3] + c[4] * h).mean())
            assert g == want, (n, c)


def test_pareto_prune_kats(gpu_device):
    for case in load_json("pareto_kats")["cases"]:
        rows = [tuple(r) + (i,) for i, r in enumerate(case["rows"])]
        kept = pareto_prune(rows, key=lambda r: (r[0], r[1]))
        assert [r[2] for r in kept] == case["kept"]
    assert pareto_prune([(1.0, 5.0), (2.0, 4.0), (1.5, 6.0)]) == [(1.0, 5.0), (2.0, 4.0)]
    assert pareto_prune([]) == []


@pytest.mark.parametrize("n", [1, 2, 3, 100, 2047, 2048, 2049, 5000, 70001])
def test_pareto_prune_random(gpu_device, n):
    rng = random.Random(n)
    rows = [(rng.choice([0.5, 1.0, rng.uniform(0, 10)]), rng.choice([1.0, rng.uniform(0, 10)]))
            for _ in range(n)]
    got = pareto_prune(rows)
    want = [rows[i] for i in og.pareto_keep([r[0] for r in rows], [r[1] for r in rows])]
    assert got == want


def _plan_matches(plan, want, rows):
    assert plan.row == rows[want["row_index"]]
    assert plan.workers == want["workers"]
    assert plan.batches == want["batches"]
    assert plan.path_latency_s == want["path_latency_s"]
    assert plan.fidelity_cost == want["fidelity_cost"]
    assert plan.infeasible == want["infeasible"]


def test_planner_random200_matches_reference(gpu_device):
    cases = load_json("planner_random200")["cases"]
    for case in cases:
        cat = catalog_from_doc(case["catalog"])
        rows = rows_ns(case["rows"])
        try:
            plan = solve(rows, cat, case["lam"], case["queues"], case["workers"], case["t_slo"],
                         case["alpha"])
        except PlannerError as exc:
            assert case["solve"] is None and case["solve_error"] == str(exc)
            continue
        _plan_matches(plan, case["solve"], rows)


def test_planner_conftest_sweep_matches_reference(gpu_device):
    doc = load_json("planner_conftest")
    cat = catalog_from_doc(doc["catalog"])
    rows = rows_ns(doc["table"]["rows"])
    pts = doc["points"]
    plans = solve_many(rows, cat, [p["lam"] for p in pts], [p["queues"] for p in pts],
                       [p["workers"] for p in pts], [p["t_slo"] for p in pts], 1.5)
    for plan, pt in zip(plans, pts):
        _plan_matches(plan, pt["solve"], rows)


def test_planner_errors(gpu_device):
    doc = load_json("planner_conftest")
    cat = catalog_from_doc(doc["catalog"])
    rows = rows_ns(doc["table"]["rows"])
    with pytest.raises(PlannerError, match="negative demand"):
        solve(rows, cat, -1.0)
    dead = rows_ns([dict(doc["table"]["rows"][0], r_light=0.0, r_heavy=0.0)])
    # a row with no load is trivially feasible (zero workers), as in the reference
    plan = solve(dead, cat, 3.0)
    want = op.solve(dead, cat, 3.0)
    _plan_matches(plan, want, dead)
    # ... but when nothing meets the SLO the fallback has no serveable row
    with pytest.raises(PlannerError, match="no serveable rows"):
        solve(dead, cat, 3.0, t_slo=0.01)
    with pytest.raises(op.OraclePlannerError, match="no serveable rows"):
        op.solve(dead, cat, 3.0, t_slo=0.01)


def test_planner_sweep_vs_oracle_on_gpu_table(gpu_device):
    rng = np.random.default_rng(11)
    cat = default_catalog()
    h = rng.uniform(0.05, 0.9, 20000)
    noise = rng.normal(0, 0.05, 20000)
    table = profile_records(cat, h, noise=noise, thresholds=tuple(i / 31 for i in range(32)))
    pr = random.Random(5)
    lams = [pr.uniform(0, 120) for _ in range(60)] + [0.0]
    ts = [pr.choice([5.0, 15.0, 30.0, 60.0, 90.0]) for _ in lams]
    ws = [pr.choice([1, 2, 3, 8, 16]) for _ in lams]
    qs = [({m: pr.uniform(0, 40) for m in cat.ids() if pr.random() < 0.5} if pr.random() < 0.5
           else {}) for _ in lams]
    plans = solve_many(table, cat, lams, qs, ws, ts, 1.5)
    for plan, lam, t, w, q in zip(plans, lams, ts, ws, qs):
        want = op.solve(table.rows, cat, lam, q, w, t, 1.5)
        _plan_matches(plan, want, table.rows)


@pytest.mark.slow
def test_c2_scale_properties(gpu_device):
    """c2 shape (4 models, 1M records, 256 thresholds): size-independent checks."""
    rng = np.random.default_rng(20261017)
    cat = default_catalog()
    pool = select_candidates(cat, 0.1, 0.1)
    n = 1_000_000
    h = rng.uniform(0.05, 0.9, n)
    noise = rng.normal(0.0, 0.05, n)
    thr = tuple(i / 255 for i in range(256))
    scores = light_scores(pool, h, noise)
    prof = GridProfiler(pool, h, scores)
    dt = prof.run(thr)
    from paper_2509_00642_b200.profiler import rows_from_device
    rows = rows_from_device(dt, pool, thr)
    assert len(rows) == dt.n_rows > 0
    by_pair = {}
    for r in rows:
        by_pair.setdefault((r.light_id, r.heavy_id), []).append(r)
    assert len(by_pair) == 6
    for prs in by_pair.values():
        keys = [(r.theta, r.tau) for r in prs]
        assert keys == sorted(keys)
        for a in prs:     # frontier property (profiler tests: test_rows_per_pair_form_frontier)
            for b in prs:
                if a is b:
                    continue
                dom = (b.mean_latency_s <= a.mean_latency_s and b.fidelity_cost <= a.fidelity_cost
                       and (b.mean_latency_s < a.mean_latency_s or b.fidelity_cost < a.fidelity_cost))
                assert not dom or a.theta == 1.0
    # bit-exact counts / latency and 1e-9 fidelity on a sample of rows, via numpy
    cost, sc = og.model_arrays(pool, h, noise)
    ids = {v.id: v for v in pool}
    for r in random.Random(1).sample(rows, 12):
        lt, hv = ids[r.light_id], ids[r.heavy_id]
        nb, nr, rl, rh, fid, lat = og.cell_stats(h, sc[lt.id], cost[lt.id], cost[hv.id],
                                                 lt.latency_s[1], hv.latency_s[1], r.theta, r.tau)
        assert (r.r_light, r.r_heavy, r.mean_latency_s) == (rl, rh, lat)
        assert math.isclose(r.fidelity_cost, fid, rel_tol=1e-9)


@pytest.mark.parametrize("layout", ["bucketed", "original"])
def test_k1_layouts_agree(gpu_device, layout):
    """Both K1 paths (row-bucketed record store / original order with L2
    atomics) give the same table as the oracle."""
    rng = np.random.default_rng(99)
    cat = default_catalog()
    pool = select_candidates(cat, 0.1, 0.1)
    n = 50_000
    h = rng.choice(np.round(rng.uniform(0.0, 1.0, 500), 3), n)
    noise = rng.normal(0.0, 0.08, n)
    thr = tuple(i / 47 for i in range(48))
    prof = GridProfiler(pool, h, light_scores(pool, h, noise), layout=layout)
    from paper_2509_00642_b200.profiler import rows_from_device
    got = [(r.light_id, r.heavy_id, r.theta, r.tau, r.r_light, r.r_heavy, r.fidelity_cost,
            r.mean_latency_s) for r in rows_from_device(prof.run(thr), pool, thr)]
    want = og.profile_rows(pool, h, noise=noise, thresholds=thr)
    assert_rows_close(got, want)


@pytest.mark.parametrize("n,thr_k,shift_case", [(100_001, 48, "odd"), (262_144, 64, "wide"),
                                                 (3, 5, "tiny"), (70_000, 1024, "k1024"),
                                                 (50_000, 200, "random"), (50_000, 64, "clustered")])
def test_bucketed_histograms_bitexact(gpu_device, n, thr_k, shift_case):
    """The row-bucketed store + K1 give bit-identical prefix tables to the
    global-atomic K1 on adversarial records: hardness exactly on thresholds,
    0.0 and 1.0, one row holding > 32768 records (chunked, atomics), odd n
    (scalar loads), scores on thresholds and at the clip bounds."""
    import torch
    rng = np.random.default_rng(n + thr_k)
    cat = default_catalog()
    pool = select_candidates(cat, 0.1, 0.1)
    thr = tuple(i / (thr_k - 1) for i in range(thr_k))      # uniform-grid binning path
    if shift_case == "random":                               # guided (<= 2 per guide bucket)
        thr = tuple(sorted(set(np.round(rng.uniform(0, 1, thr_k), 6).tolist())))
    elif shift_case == "clustered":                          # general guided search
        thr = tuple(sorted(set((0.5 + rng.uniform(-1e-4, 1e-4, thr_k)).tolist() + [0.0, 1.0])))
    h = rng.uniform(0.0, 1.0, n)
    pick = rng.random(n)
    h[pick < 0.2] = rng.choice(np.asarray(thr), int((pick < 0.2).sum()))
    h[(pick >= 0.2) & (pick < 0.6)] = thr[len(thr) // 2] + 1e-9   # one heavy row
    h[pick > 0.98] = 0.0
    h[pick > 0.99] = 1.0
    sc = rng.uniform(0.0, 1.0, (len(pool) - 1, n))
    sc[:, ::7] = rng.choice(np.asarray(thr), sc[:, ::7].shape)
    sc[:, ::11] = 0.0
    sc[:, ::13] = 1.0
    tabs = {}
    for layout in ("bucketed", "original"):
        prof = GridProfiler(pool, h, sc, layout=layout)
        st = prof.launch(prof.plan(thr))
        prof.finish(st)
        tabs[layout] = (st["cnt"].clone(), st["hsum"].clone())
    torch.cuda.synchronize()
    assert torch.equal(tabs["bucketed"][0], tabs["original"][0])
    assert torch.equal(tabs["bucketed"][1], tabs["original"][1])


def test_bucketed_rejects_bad_hardness(gpu_device):
    from paper_2509_00642_b200.profiler import ProfileError
    cat = default_catalog()
    pool = select_candidates(cat, 0.1, 0.1)
    h = np.linspace(0.0, 1.0, 1000)
    h[17] = 1.5
    prof = GridProfiler(pool, h, np.full((len(pool) - 1, 1000), 0.5))
    with pytest.raises(ProfileError):
        prof.run((0.0, 0.5, 1.0))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_profile_equals_single(gpu_device, world):
    """torchrun world ranks (gloo, sharing the box's GPU): pair-sharded
    profiling + all-gather merge reproduces the 1-process table exactly."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HADIS_DIST_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone",
                          "--nproc-per-node", str(world), os.path.join(root, "tools",
                                                                       "check_sharded.py")],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "sharded OK" in out.stdout


# ------------------------------------------------ cascade-depth frontier (f1)

def _frontier_case(name):
    from tests.goldens import frontier_cases
    d = frontier_cases()[name]
    return d, catalog_from_doc(d["catalog"]), np.asarray(d["h"]), tuple(d["thresholds"])


def _hull_close(got, want, tol=1e-9):
    """Envelopes agree as functions: values at every breakpoint of both."""
    from paper_2509_00642_b200.frontier import envelope_value
    want = [tuple(p) for p in want]
    xs = sorted({x for x, _ in got} | {x for x, _ in want})
    lo, hi = max(got[0][0], want[0][0]), min(got[-1][0], want[-1][0])
    assert abs(got[0][0] - want[0][0]) <= tol and abs(got[-1][0] - want[-1][0]) <= tol
    for x in xs:
        if lo <= x <= hi:
            assert abs(envelope_value(got, x) - envelope_value(want, x)) <= tol * max(1.0, abs(x))


@pytest.mark.parametrize("name", ["jitter%02d" % s for s in range(20)] +
                         ["wide", "default", "default_k33_n2000", "wide_dupgrid"])
def test_frontier_compare_matches_reference(gpu_device, name):
    from paper_2509_00642_b200.frontier import frontier_compare
    d, cat, h, thr = _frontier_case(name)
    rep = frontier_compare(cat, h=h, thresholds=thr)
    r = d["report"]
    assert (rep.n_two, rep.n_three) == (r["n_two"], r["n_three"])
    assert abs(rep.gap - r["gap"]) <= 1e-9
    _hull_close(list(rep.envelope_two), r["envelope_two"])
    _hull_close(list(rep.envelope_three), r["envelope_three"])


@pytest.mark.parametrize("name", ["jitter00", "wide", "wide_dupgrid"])
def test_cascade_points_match_reference(gpu_device, name):
    """Two-stage points bit-exact (latency and numpy-exact fidelity); three-stage
    latency bit-exact, fidelity within 1e-12 relative."""
    from paper_2509_00642_b200.frontier import three_stage_points, two_stage_points
    d, cat, h, thr = _frontier_case(name)
    two = two_stage_points(cat.variants, h, thr)
    assert [[p.latency_s, p.fidelity_cost, list(p.detail)] for p in two] == d["two"]
    three = three_stage_points(cat.variants, h, thr)
    assert len(three) == len(d["three"])
    for p, (lat, fid, det) in zip(three, d["three"]):
        assert p.latency_s == lat and list(p.detail) == det
        assert math.isclose(p.fidelity_cost, fid, rel_tol=1e-12)


def test_frontier_errors(gpu_device):
    from paper_2509_00642_b200.frontier import FrontierError, frontier_compare, lower_envelope
    cat = default_catalog()
    with pytest.raises(FrontierError):
        frontier_compare(cat, h=np.array([0.5, 1.5]))
    with pytest.raises(FrontierError):
        lower_envelope([])


def test_graph_replay_matches_eager(gpu_device):
    """The CUDA-graph replay of the whole pipeline returns the eager table, twice
    (static buffers reused), and tracks new record values written in place."""
    import torch
    rng = np.random.default_rng(11)
    cat = default_catalog()
    pool = select_candidates(cat, 0.1, 0.1)
    n = 20_000
    h = rng.uniform(0.05, 0.9, n)
    noise = rng.normal(0.0, 0.05, n)
    thr = tuple(i / 63 for i in range(64))
    prof = GridProfiler(pool, h, light_scores(pool, h, noise))
    plan = prof.plan(thr)
    eager = prof.run(thr)
    replay = prof.graph(plan)
    for _ in range(2):
        got = replay()
        assert got.n_rows == eager.n_rows
        for f in ("pair", "theta_pos", "tau_pos", "r_light", "r_heavy", "fid", "lat"):
            assert torch.equal(getattr(got, f), getattr(eager, f)), f
    h2 = rng.uniform(0.05, 0.9, n)
    prof.h.copy_(torch.from_numpy(h2))
    prof.scores.copy_(torch.from_numpy(light_scores(pool, h2, noise)))
    fresh = GridProfiler(pool, h2, light_scores(pool, h2, noise)).run(thr)
    got = replay()
    assert got.n_rows == fresh.n_rows
    assert torch.equal(got.fid, fresh.fid) and torch.equal(got.lat, fresh.lat)


# --------------------------------- online consumers of the allocation search (f4)

def test_planner_modes_match_reference(gpu_device):
    """Every make_planner mode (online, cache-d/dq, clipper, proteus, diffserve)
    over a 120-epoch (demand, backlog) sequence equals the reference's plans
    field by field (tests/golden/make_golden_planner_modes.py)."""
    from paper_2509_00642_b200.planner import PlannerError, make_planner
    from paper_2509_00642_b200.profiler import CascadeRow
    doc = load_json("planner_conftest")
    modes = load_json("planner_modes")
    cat = default_catalog()
    rows = tuple(CascadeRow(**r) for r in doc["table"]["rows"])

    class T:                                       # table stand-in: .rows is all planners use
        pass
    table = T()
    table.rows = rows
    for key, want_list in modes["runs"].items():
        mode, workers, t_slo = key.split("|")
        fn = make_planner(mode, table, cat, workers=int(workers), t_slo=float(t_slo), alpha=1.5)
        for ep, want in zip(modes["epochs"], want_list):
            if "error" in want:
                with pytest.raises(PlannerError):
                    fn(ep["lam"], dict(ep["queues"]))
                continue
            plan, info = fn(ep["lam"], dict(ep["queues"]))
            w = want["plan"]
            got_row = {k: getattr(plan.row, k) for k in w["row"]}
            assert got_row == w["row"], (key, ep)
            assert (plan.workers, plan.batches, plan.infeasible, plan.label) == \
                (w["workers"], w["batches"], w["infeasible"], w["label"]), (key, ep)
            assert plan.path_latency_s == w["path_latency_s"], (key, ep)
            assert plan.fidelity_cost == w["fidelity_cost"] and plan.lam == w["lam"]
            assert plan.queues == w["queues"] and info == want["info"], (key, ep)


def test_fallback_plan_and_negative_demand_match_reference(gpu_device):
    """fallback_plan over explicit (index, row) pairs -- including negative
    demand, which only ``solve`` rejects (planner.py:170-222) -- equals the
    reference's plans field by field."""
    from paper_2509_00642_b200.planner import PlannerError, fallback_plan, solve_many
    from paper_2509_00642_b200.profiler import CascadeRow
    doc = load_json("planner_conftest")
    modes = load_json("planner_modes")
    cat = default_catalog()
    rows = tuple(CascadeRow(**r) for r in doc["table"]["rows"])
    indexed = list(enumerate(rows))
    for case in modes["fallback"]:
        plan = fallback_plan(indexed, cat, case["lam"], dict(case["queues"]), case["workers"],
                             30.0, 1.5, "fb")
        w = case["plan"]
        assert {k: getattr(plan.row, k) for k in w["row"]} == w["row"], case
        assert (plan.workers, plan.batches, plan.infeasible, plan.label) == \
            (w["workers"], w["batches"], w["infeasible"], w["label"]), case
        assert plan.path_latency_s == w["path_latency_s"], case
    with pytest.raises(PlannerError, match="solve: negative demand"):
        solve_many(rows, cat, [1.0, -0.5])


# ------------------------------------------------ router weight sweep (f3)

@pytest.mark.parametrize("name", ["separable80", "noisy600", "noisy3000"])
def test_tune_weights_matches_reference(gpu_device, name):
    from paper_2509_00642_b200.router import tune_weights_features
    d = {x["name"]: x for x in load_json("router")}[name]
    arr = load_npz("router")
    w, thr, acc = tune_weights_features(arr[name + ":features"], arr[name + ":labels"])
    assert (list(w), thr, acc) == (d["weights"], d["threshold"], d["acc"])


def test_tune_weights_per_vector_matches_reference(gpu_device):
    import torch
    from paper_2509_00642_b200 import _lib
    from paper_2509_00642_b200.router import _weight_grid
    d = {x["name"]: x for x in load_json("router")}["separable80"]
    arr = load_npz("router")
    mat, lab = arr["separable80:features"], arr["separable80:labels"]
    grid = _weight_grid(mat.shape[1], (0.0, 1.0, 2.0))
    dev = torch.device("cuda")
    acc = torch.empty(len(grid), dtype=torch.float64, device=dev)
    thr = torch.empty(len(grid), dtype=torch.float64, device=dev)
    p = _lib.ptr
    d_x = torch.from_numpy(np.ascontiguousarray(mat)).to(dev)     # held until the sync below
    d_l = torch.from_numpy(lab.astype(np.uint8)).to(dev)
    d_w = torch.tensor(grid, dtype=torch.float64, device=dev)
    _lib.check(_lib.load().hadis_tune_weights(p(d_x), p(d_l), mat.shape[0], mat.shape[1], p(d_w),
                                              len(grid), int(lab.sum()), p(acc), p(thr),
                                              _lib.stream_handle()), "tune_weights")
    got = list(zip(acc.cpu().tolist(), thr.cpu().tolist()))
    assert [list(x) for x in got] == d["per_vector"]


def test_tune_weights_rejects_degenerate(gpu_device):
    from paper_2509_00642_b200.router import RouterError, tune_weights_features
    with pytest.raises(RouterError):
        tune_weights_features(np.zeros((2, 8)), [0, 0])


def test_table_pipeline_matches_single_builds(gpu_device):
    """Streaming builds (double-buffered H2D / graph / D2H) return, for each
    record set, exactly the rows of a standalone build."""
    import torch
    from paper_2509_00642_b200.profiler import TablePipeline
    rng = np.random.default_rng(13)
    cat = default_catalog()
    pool = select_candidates(cat, 0.1, 0.1)
    n = 30_000
    thr = tuple(i / 47 for i in range(48))
    sets = []
    for _ in range(5):
        h = rng.uniform(0.05, 0.9, n)
        sc = light_scores(pool, h, rng.normal(0.0, 0.05, n))
        sets.append((torch.from_numpy(h).pin_memory(), torch.from_numpy(sc).pin_memory()))
    pipe = TablePipeline(pool, n, len(pool) - 1, thr)
    pipe.warm(*sets[0])
    for i, (h_pin, sc_pin) in enumerate(sets):
        want = GridProfiler(pool, h_pin.numpy(), sc_pin.numpy()).run(thr)
        rows = {}
        got = pipe.run([(h_pin, sc_pin)], on_rows=lambda k, r: rows.update(r))
        assert got[0][1] == want.n_rows
        for f in TablePipeline.FIELDS:
            assert torch.equal(rows[f], getattr(want, f).cpu()), (i, f)
    res = pipe.run(sets)                     # all five in flight
    assert [r[0] for r in res] == list(range(5))


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c3", "c4"])
def test_full_scale_properties(gpu_device, name):
    """BASELINE c3 / c4 at full size (8 / 16 models, 10M records, 512^2 / 1024^2 grid):
    per-pair (theta, tau) order, no table row dominated by another (theta = max
    rows excepted, profiler.py:168-173), and on sampled cells, numpy's
    profiler.py:146-165 arithmetic: table rows match it (bit-exact counts and
    latency, fid 1e-9) and cells outside the table are weakly dominated by a row."""
    from paper_2509_00642_b200 import synth
    cfg = synth.CONFIGS[name]
    pool, h, noise, scores = synth.records(cfg)
    thr = cfg.thresholds
    dt = GridProfiler(pool, h, scores).run(thr)
    assert dt.n_rows > 0 and len(dt.pairs) == cfg.n_pairs
    pair = dt.pair.cpu().numpy()
    tp, cp = dt.theta_pos.cpu().numpy(), dt.tau_pos.cpu().numpy()
    lat, fid = dt.lat.cpu().numpy(), dt.fid.cpu().numpy()
    rl, rh = dt.r_light.cpu().numpy(), dt.r_heavy.cpu().numpy()
    K = len(thr)
    assert np.all(np.diff(pair) >= 0)
    starts = np.searchsorted(pair, np.arange(len(dt.pairs) + 1))
    for p in range(len(dt.pairs)):
        a, b = starts[p], starts[p + 1]
        assert b > a
        key = tp[a:b].astype(np.int64) * K + cp[a:b]
        assert np.all(np.diff(key) > 0)                     # (theta, tau) order, no duplicates
        o = np.lexsort((fid[a:b], lat[a:b]))
        f = fid[a:b][o]
        prev_min = np.minimum.accumulate(np.concatenate(([np.inf], f[:-1])))
        free = np.asarray(thr)[tp[a:b][o]] != max(thr)
        assert np.all(f[free] < prev_min[free])              # strictly below all cheaper rows
    rng = random.Random(4)
    for _ in range(30):
        p = rng.randrange(len(dt.pairs))
        i, j = dt.pairs[p]
        lt, hv = pool[i], pool[j]
        lc = lt.base_quality_cost + lt.hardness_penalty * h
        hc = hv.base_quality_cost + hv.hardness_penalty * h
        a, b = starts[p], starts[p + 1]
        rows = dict(zip((tp[a:b].astype(np.int64) * K + cp[a:b]).tolist(), range(a, b)))
        member = list(rows)[rng.randrange(len(rows))]
        for cell in (member, rng.randrange(K * K)):
            th, ta = thr[cell // K], thr[cell % K]
            nb, nr, r_l, r_h, f_c, l_c = og.cell_stats(h, scores[i], lc, hc, lt.latency_s[1],
                                                       hv.latency_s[1], th, ta)
            if cell in rows:
                r = rows[cell]
                assert (rl[r], rh[r], lat[r]) == (r_l, r_h, l_c)
                assert math.isclose(fid[r], f_c, rel_tol=1e-9)
            else:
                dom = (lat[a:b] <= l_c) & (fid[a:b] <= f_c * (1 + 1e-9))
                assert dom.any(), (p, cell)


def test_brute_force_solve_matches_reference(gpu_device):
    """brute_force_solve on every golden instance, the overload fallback included."""
    from paper_2509_00642_b200.planner import brute_force_solve
    for case in load_json("planner_random200")["cases"]:
        cat = catalog_from_doc(case["catalog"])
        rows = rows_ns(case["rows"])
        try:
            plan = brute_force_solve(rows, cat, case["lam"], case["queues"], case["workers"],
                                     case["t_slo"], case["alpha"])
        except PlannerError as exc:
            assert case["brute"] is None and case["brute_error"] == str(exc)
            continue
        _plan_matches(plan, case["brute"], rows)


@pytest.mark.parametrize("models,n,k", [(24, 2000, 9), (40, 801, 5)])
def test_large_pool_matches_oracle(gpu_device, models, n, k):
    """Large pools (276 / 780 pairs; light groups of up to 39 heavy partners, an
    odd record count on the scalar-load path) against the oracle, bit-exact rows
    in exact mode."""
    from paper_2509_00642_b200 import synth
    cat = synth.geometric_catalog(models)
    pool = select_candidates(cat, 1e-9, 1e-9)
    assert len(pool) == models
    rng = np.random.default_rng(models)
    h = rng.uniform(0.0, 1.0, n)
    noise = rng.normal(0.0, 0.05, n)
    thr = tuple(np.linspace(0.0, 1.0, k).tolist())
    want = og.profile_rows(pool, h, noise=noise, thresholds=thr)
    got = profile_records(pool, h, noise=noise, thresholds=thr, exact_fid=True)
    assert tuples(got) == want


@pytest.mark.parametrize("k,n", [(2047, 5001), (2600, 4001)])
def test_max_grid_layouts_agree(gpu_device, k, n):
    """Grids at / past the row-bucketed store's limit (2047 distinct thresholds;
    2600 takes the global-atomic K1): both K1 layouts give the same table, in
    (theta, tau) order, and sampled rows match numpy's cell arithmetic."""
    from paper_2509_00642_b200.profiler import rows_from_device
    rng = np.random.default_rng(k)
    cat = default_catalog()
    pool = select_candidates(cat, 0.1, 0.1)[:3]
    h = rng.uniform(0.0, 1.0, n)
    noise = rng.normal(0.0, 0.05, n)
    thr = tuple(i / (k - 1) for i in range(k))
    scores = light_scores(pool, h, noise)
    tables = []
    for layout in (("bucketed", "original") if k <= 2047 else ("original",)):
        prof = GridProfiler(pool, h, scores, layout=layout)
        tables.append([(r.light_id, r.heavy_id, r.theta, r.tau, r.r_light, r.r_heavy,
                        r.fidelity_cost, r.mean_latency_s)
                       for r in rows_from_device(prof.run(thr), pool, thr)])
    assert all(t == tables[0] for t in tables[1:])
    rows = tables[0]
    assert rows
    cost, sc = og.model_arrays(pool, h, noise)
    ids = {v.id: v for v in pool}
    for r in random.Random(k).sample(rows, 8):
        lt, hv = ids[r[0]], ids[r[1]]
        _, _, rl, rh, fid, lat = og.cell_stats(h, sc[lt.id], cost[lt.id], cost[hv.id],
                                               lt.latency_s[1], hv.latency_s[1], r[2], r[3])
        assert (r[4], r[5], r[7]) == (rl, rh, lat)
        assert math.isclose(r[6], fid, rel_tol=1e-9)


@pytest.mark.parametrize("case", ["one_row", "two_rows_8193", "tiny_n2"])
def test_skewed_rows_match_oracle(gpu_device, case):
    """Row-bucketed store edge cases: every record in one theta-row (K1 splits the
    row across CTAs: atomic flush + separate row scan), a record count just past
    a scatter tile with five light models (two quads), two records."""
    from paper_2509_00642_b200 import synth
    rng = np.random.default_rng(7)
    if case == "one_row":
        pool = select_candidates(default_catalog(), 0.1, 0.1)
        n = 100_000
        h = np.full(n, 0.4321)
    elif case == "two_rows_8193":
        pool = select_candidates(synth.geometric_catalog(6), 1e-9, 1e-9)
        n = 8193
        h = rng.choice([0.25, 0.75], n)
    else:
        pool = select_candidates(synth.geometric_catalog(6), 1e-9, 1e-9)
        n = 2
        h = np.array([0.1, 0.9])
    noise = rng.normal(0.0, 0.05, n)
    thr = tuple(np.linspace(0.0, 1.0, 9).tolist())
    want = og.profile_rows(pool, h, noise=noise, thresholds=thr)
    got = profile_records(pool, h, noise=noise, thresholds=thr, exact_fid=True)
    assert tuples(got) == want


def test_odd_scores_match_oracle(gpu_device):
    """Caller-supplied scores outside [0, 1], NaN, and exactly on thresholds: the
    tau-bins follow numpy's `s < tau` (NaN never rejects)."""
    rng = np.random.default_rng(12)
    pool = select_candidates(default_catalog(), 0.1, 0.1)
    n = 3001
    h = rng.uniform(0.0, 1.0, n)
    thr = tuple(np.linspace(0.0, 1.0, 11).tolist())
    sc = {}
    for v in pool[:-1]:
        s = rng.uniform(-0.2, 1.2, n)
        s[rng.integers(0, n, 50)] = np.nan
        s[rng.integers(0, n, 200)] = rng.choice(thr, 200)
        sc[v.id] = s
    want = og.profile_rows(pool, h, scores=sc, thresholds=thr)
    got = profile_records(pool, h, scores=np.stack([sc[v.id] for v in pool[:-1]]),
                          thresholds=thr, exact_fid=True)
    assert tuples(got) == want


def test_solve_many_past_one_launch(gpu_device):
    """More points than one device launch takes (65535): chunked launches give the
    same plans as the reference-order oracle on a sample, in input order."""
    doc = load_json("planner_conftest")
    cat = catalog_from_doc(doc["catalog"])
    rows = rows_ns(doc["table"]["rows"])
    pr = random.Random(3)
    lams = [pr.uniform(0.0, 150.0) for _ in range(70_001)]
    plans = solve_many(rows, cat, lams, None, 8, 60.0, 1.5)
    assert len(plans) == len(lams)
    for i in [0, 1, 65534, 65535, 65536, 70_000] + pr.sample(range(len(lams)), 14):
        _plan_matches(plans[i], op.solve(rows, cat, lams[i], {}, 8, 60.0, 1.5), rows)


def test_profiler_reuse_across_grids(gpu_device):
    """One GridProfiler, alternating threshold grids and pair subsets (plans,
    workspaces and record stores are reused or regrown): every run equals a
    fresh profiler's run."""
    from paper_2509_00642_b200.profiler import pair_list
    rng = np.random.default_rng(21)
    pool = select_candidates(default_catalog(), 0.1, 0.1)
    n = 20_001
    h = rng.uniform(0.0, 1.0, n)
    scores = light_scores(pool, h, rng.normal(0.0, 0.05, n))
    shared = GridProfiler(pool, h, scores)
    pairs = pair_list(pool)
    jobs = [(tuple(i / 63 for i in range(64)), None), (tuple(i / 15 for i in range(16)), None),
            (tuple(i / 200 for i in range(201)), pairs[2:5]), (tuple(i / 63 for i in range(64)),
                                                                pairs[:1])]
    for thr, prs in jobs + jobs[::-1]:
        got = shared.run(thr, pairs=prs)
        want = GridProfiler(pool, h, scores).run(thr, pairs=prs)
        assert got.n_rows == want.n_rows
        for f in ("pair", "theta_pos", "tau_pos", "r_light", "r_heavy", "fid", "lat"):
            assert torch_equal(getattr(got, f), getattr(want, f)), f


def torch_equal(a, b):
    import torch
    return bool(torch.equal(a, b))


@pytest.mark.parametrize("workers", [0, 1, 2, 64])
def test_planner_worker_extremes(gpu_device, workers):
    """Worker budgets at the edges (none, one, two, more than any row needs)
    against the oracle: same plan or the same PlannerError message."""
    doc = load_json("planner_conftest")
    cat = catalog_from_doc(doc["catalog"])
    rows = rows_ns(doc["table"]["rows"])
    for lam in (0.0, 0.3, 3.0, 40.0, 400.0):
        for t_slo in (5.0, 60.0):
            try:
                want = op.solve(rows, cat, lam, {"sd35-turbo": 7.0}, workers, t_slo, 1.5)
            except Exception as exc:          # oracle raises the reference's error text
                with pytest.raises(PlannerError, match=str(exc).split(":")[0]):
                    solve(rows, cat, lam, {"sd35-turbo": 7.0}, workers, t_slo, 1.5)
                continue
            plan = solve(rows, cat, lam, {"sd35-turbo": 7.0}, workers, t_slo, 1.5)
            _plan_matches(plan, want, rows)


# ------------------------------------------------ capacities, pipelines, devices

def _dt_arrays(dt):
    return {f: getattr(dt, f).cpu().numpy() for f in ("pair", "theta_pos", "tau_pos", "r_light",
                                                      "r_heavy", "fid", "lat")}


@pytest.mark.parametrize("name", ["ties3000", "cross1500"])
def test_exact_capacity_grows_and_cub_request_sort(gpu_device, name):
    """An exact-request capacity below the need grows (no 'retries exhausted'),
    and capacities above one CTA's bitonic sort take the CUB radix-sort path;
    both give the same table as the default capacities."""
    doc = load_json(name)
    rec = load_npz(name)
    cat, pool = _golden_pool(doc)
    sc = scores_of(rec)
    prof = GridProfiler(pool, rec["h"], np.stack([sc[v.id] for v in pool[:-1]]))
    plan = prof.plan(doc["thresholds"])
    base = _dt_arrays(prof.run(doc["thresholds"]))
    cand, _, out = plan.caps
    plan.caps = (cand, 1, out)
    dt = prof.finish(prof.launch(plan))
    assert all(np.array_equal(base[k], v) for k, v in _dt_arrays(dt).items())
    plan.caps = (cand, 8192, out)
    dt = prof.finish(prof.launch(plan))
    assert all(np.array_equal(base[k], v) for k, v in _dt_arrays(dt).items())


def test_table_pipeline_delivers_every_set(gpu_device):
    """TablePipeline: each record set's rows reach the callback (no set
    overwrites another), equal to a one-shot build of the same records."""
    import torch
    from paper_2509_00642_b200.profiler import TablePipeline
    cat = default_catalog()
    pool = select_candidates(cat, 0.1, 0.1)
    thr = tuple(i / 31 for i in range(32))
    sets, want = [], []
    for seed in range(5):
        rng = np.random.default_rng(100 + seed)
        h = rng.uniform(0.05, 0.9, 20000)
        sc = light_scores(pool, h, rng.normal(0.0, 0.05, 20000))
        sets.append((torch.from_numpy(h).pin_memory(), torch.from_numpy(sc).pin_memory()))
        want.append(_dt_arrays(GridProfiler(pool, h, sc).run(thr)))
    pipe = TablePipeline(pool, 20000, len(pool) - 1, thr)
    pipe.warm(*sets[0])
    got = {}
    res = pipe.run(sets, on_rows=lambda i, rows: got.__setitem__(
        i, {f: v.numpy().copy() for f, v in rows.items()}))
    assert [r[0] for r in res] == list(range(5))
    for i in range(5):
        assert all(np.array_equal(want[i][f], got[i][f]) for f in want[i]), i


def test_graph_replay_survives_workspace_reallocation(gpu_device):
    """A captured replay keeps its own buffers: a later, larger run on the same
    profiler (new workspace) does not corrupt the replay's results."""
    cat = default_catalog()
    pool = select_candidates(cat, 0.1, 0.1)
    rng = np.random.default_rng(5)
    h = rng.uniform(0.05, 0.9, 30000)
    sc = light_scores(pool, h, rng.normal(0.0, 0.05, 30000))
    prof = GridProfiler(pool, h, sc)
    small = tuple(i / 15 for i in range(16))
    replay = prof.graph(prof.plan(small))
    want = _dt_arrays(replay())
    prof.run(tuple(i / 200 for i in range(201)))       # bigger grid: reallocates workspace
    got = _dt_arrays(replay())
    assert all(np.array_equal(want[k], v) for k, v in got.items())


@pytest.mark.gpu
def test_bench_multi_rank_line(gpu_device):
    """bench.py's N > 1 arm under torchrun (2 ranks, gloo, sharing the box's
    GPU): the timed step (local build + slab all-gather + merge kernel) runs
    and rank 0 prints one JSON line whose table has the 1-rank row count."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    args = ["--config", "c2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
            "--no-allocation"]
    one = subprocess.run([sys.executable, os.path.join(root, "bench.py")] + args,
                         capture_output=True, text=True, timeout=900)
    assert one.returncode == 0, one.stderr[-3000:]
    env = dict(os.environ, HADIS_DIST_BACKEND="gloo")
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone",
                          "--nproc-per-node", "2", os.path.join(root, "bench.py"), "--gpus", "2"]
                         + args, capture_output=True, text=True, env=env, timeout=900)
    assert two.returncode == 0, two.stderr[-3000:]
    l1 = json.loads([x for x in one.stdout.splitlines() if x.startswith("{")][-1])
    l2 = json.loads([x for x in two.stdout.splitlines() if x.startswith("{")][-1])
    assert l2["n_gpus"] == 2 and l2["value"] > 0 and l2["ms_per_step"] > 0
    assert l2["config"]["rows"] == l1["config"]["rows"]
    assert "merge" in l2 and l2["merge"]["slab_row_bytes"] == 24
    # the same sharded step over NCCL (one rank: process group, all-gather of the
    # slab, merge kernel) -- the collective path the multi-GPU runs take
    env = dict(os.environ, HADIS_BENCH_SHARDED="1", HADIS_DIST_BACKEND="nccl")
    nccl = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone",
                           "--nproc-per-node", "1", os.path.join(root, "bench.py")] + args,
                          capture_output=True, text=True, env=env, timeout=900)
    assert nccl.returncode == 0, nccl.stderr[-3000:]
    l3 = json.loads([x for x in nccl.stdout.splitlines() if x.startswith("{")][-1])
    assert l3["config"]["rows"] == l1["config"]["rows"] and "merge" in l3
