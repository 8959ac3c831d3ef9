"""Parity at BASELINE scale (SURVEY §8 d, configs c2-c5), against the CPU
oracle run over the box's host cores (forked processes, numpy per cell --
the reference's own arithmetic, profiler.py:138-174 and planner.py:113-227).

* c2 (4 models, 1M records, 256^2 grid): the WHOLE table, row for row.
* c5 (1000-point re-plan sweep over the c2 table): 100 points without and
  100 with seeded per-model backlogs U(0, 40), plan for plan.
* c3 / c4 (8 / 16 models, 10M records, 512^2 / 1024^2): 2000 completeness
  probes each -- cells drawn uniformly and next to emitted rows, evaluated
  exactly with numpy; a probe must be emitted iff the reference's prune
  (catalog.py:171-192, plus the theta = max sub-frontier, profiler.py:166-174)
  keeps it against the table's rows, and emitted probes must carry the
  reference's values (bit-exact counts / latency, fidelity within 1e-9).
"""

import math
import multiprocessing as mp
import os
import random

import numpy as np
import pytest

from oracle import grid as og
from oracle import planner as op
from paper_2509_00642_b200 import synth
from paper_2509_00642_b200.planner import solve_many
from paper_2509_00642_b200.profiler import GridProfiler, profile_records, rows_from_device

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

PROCS = max(1, os.cpu_count() or 1)


def tuples(rows):
    return [(r.light_id, r.heavy_id, r.theta, r.tau, r.r_light, r.r_heavy, r.fidelity_cost,
             r.mean_latency_s) for r in rows]


def test_c2_full_table_equals_oracle(gpu_device):
    cfg = synth.CONFIGS["c2"]
    pool, h, noise, scores = synth.records(cfg)
    table = profile_records(pool, h, scores=scores, thresholds=cfg.thresholds, exact_fid=True)
    sc = {v.id: scores[i] for i, v in enumerate(pool[:-1])}
    want = og.profile_rows_parallel(pool, h, sc, cfg.thresholds, PROCS)
    got = tuples(table.rows)
    assert len(got) == len(want) == 44299
    assert got == want


# ------------------------------------------------------------------ c5

_SOLVE = None


def _oracle_point(args):
    rows, cat, W = _SOLVE
    lam, slo, queues = args
    return op.solve(rows, cat, lam, queues, W, slo, 1.5)


def test_c5_points_equal_oracle(gpu_device):
    global _SOLVE
    cfg = synth.CONFIGS["c2"]
    pool, h, noise, scores = synth.records(cfg)
    prof = GridProfiler(pool, h, scores)
    dt = prof.run(cfg.thresholds)
    rows = rows_from_device(dt, pool, cfg.thresholds)
    assert len(rows) == 44299
    cat = cfg.catalog()
    lams, slos, _ = synth.replan_points(1000)
    _, _, backlog = synth.replan_points(1000, backlog=True, models=[v.id for v in cat.variants])
    pick = list(range(0, 1000, 10))                      # 100 points across the sweep
    points = [(lams[k], slos[k], {}) for k in pick] + \
        [(lams[k], slos[k], backlog[k]) for k in pick]
    plans = solve_many(rows, cat, [p[0] for p in points], [p[2] for p in points], cfg.workers,
                       [p[1] for p in points], 1.5)
    _SOLVE = (rows, cat, cfg.workers)
    try:
        with mp.get_context("fork").Pool(PROCS) as pool_:
            want = pool_.map(_oracle_point, points, chunksize=1)
    finally:
        _SOLVE = None
    for (lam, slo, q), plan, w in zip(points, plans, want):
        assert rows[w["row_index"]] is plan.row, (lam, slo, q)
        assert plan.workers == w["workers"] and plan.batches == w["batches"], (lam, slo)
        assert plan.path_latency_s == w["path_latency_s"], (lam, slo)
        assert plan.infeasible == w["infeasible"], (lam, slo)
    assert len(want) == 200


# ------------------------------------------------------------ c3 / c4

_PROBE = None


def _probe_job(job):
    """Exact cell values (profiler.py:146-165) for one (pair, theta) and taus."""
    h, scores, pool, pairs, thr = _PROBE
    p, ti, tis = job
    i, j = pairs[p]
    lt, hv = pool[i], pool[j]
    lc = lt.base_quality_cost + lt.hardness_penalty * h
    hc = hv.base_quality_cost + hv.hardness_penalty * h
    vals = og.theta_row(h, scores[i], lc, hc, lt.latency_s[1], hv.latency_s[1], thr[ti],
                        [thr[t] for t in tis])
    return [(p, ti, t, v) for t, v in zip(tis, vals)]


def _exact_cells(cells, h, scores, pool, pairs, thr):
    """{(pair, theta_pos, tau_pos): cell_stats tuple} over the host cores."""
    global _PROBE
    jobs = {}
    for p, ti, t in cells:
        jobs.setdefault((p, ti), set()).add(t)
    _PROBE = (h, scores, pool, pairs, thr)
    try:
        with mp.get_context("fork").Pool(PROCS) as pool_:
            parts = pool_.map(_probe_job, [(p, ti, sorted(ts)) for (p, ti), ts in jobs.items()],
                              chunksize=1)
    finally:
        _PROBE = None
    return {(p, ti, t): v for part in parts for p, ti, t, v in part}


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_full_scale_completeness_probes(gpu_device, name):
    cfg = synth.CONFIGS[name]
    pool, h, noise, scores = synth.records(cfg)
    thr = cfg.thresholds
    K = len(thr)
    top = K - 1                                       # thresholds are sorted: theta = max
    dt = GridProfiler(pool, h, scores).run(thr)
    pair = dt.pair.cpu().numpy()
    tp, cp = dt.theta_pos.cpu().numpy().astype(np.int64), dt.tau_pos.cpu().numpy().astype(np.int64)
    lat, fid = dt.lat.cpu().numpy(), dt.fid.cpu().numpy()
    rl, rh = dt.r_light.cpu().numpy(), dt.r_heavy.cpu().numpy()
    starts = np.searchsorted(pair, np.arange(len(dt.pairs) + 1))
    rng = random.Random(20261017)
    probes = set()
    while len(probes) < 1000:                         # uniform cells
        probes.add((rng.randrange(len(dt.pairs)), rng.randrange(K), rng.randrange(K)))
    while len(probes) < 2000:                         # next to emitted rows
        r = rng.randrange(dt.n_rows)
        dti, dta = rng.choice(((0, 1), (0, -1), (1, 0), (-1, 0), (1, 1), (-1, -1)))
        ti, ta = int(tp[r]) + dti, int(cp[r]) + dta
        if 0 <= ti < K and 0 <= ta < K:
            probes.add((int(pair[r]), ti, ta))
    exact = _exact_cells(sorted(probes), h, scores, pool, dt.pairs, thr)

    ambiguous = []
    verdicts = []
    for (p, ti, ta), v in exact.items():
        _, _, e_rl, e_rh, e_fid, e_lat = v
        a, b = starts[p], starts[p + 1]
        idx = np.searchsorted(tp[a:b] * K + cp[a:b], ti * K + ta)
        emitted = idx < b - a and tp[a + idx] == ti and cp[a + idx] == ta
        if emitted:
            r = a + idx
            assert (rl[r], rh[r], lat[r]) == (e_rl, e_rh, e_lat), (name, p, ti, ta)
            assert math.isclose(fid[r], e_fid, rel_tol=1e-9), (name, p, ti, ta)
        # rows ordered before the probe in the prune's (lat, fid, index) order.
        # Twins -- rows with the probe's own (r_light, r_heavy), i.e. the same
        # non-bypassed and heavy sets (duplicate theta rows / empty tau bins) --
        # have numpy's fid exactly: equal values, ordered by grid index.
        G = tp[a:b] * K + cp[a:b]
        others = G != ti * K + ta
        L, F, G = lat[a:b][others], fid[a:b][others], G[others]
        twin = (rl[a:b][others] == e_rl) & (rh[a:b][others] == e_rh)
        F = np.where(twin, e_fid, F)
        near = (np.abs(F - e_fid) <= 1e-9 * abs(e_fid)) & ~twin
        if np.any(near & (L <= e_lat)):
            ambiguous.append((p, ti, ta))                # fidelity too close to call on fid*
            continue
        before = (L < e_lat) | ((L == e_lat) & ((F < e_fid) | (twin & (G < ti * K + ta))))
        killed = np.any(before & (F <= e_fid))
        keep = not killed
        if ti == top:                                    # theta = max sub-frontier
            nb = tp[a:b][others] == top
            keep = keep or not np.any(before & nb & (F <= e_fid))
        verdicts.append(((p, ti, ta), bool(keep), bool(emitted)))
    wrong = [v for v in verdicts if v[1] != v[2]]
    assert not wrong, wrong[:10]
    assert len(verdicts) >= 1900, len(ambiguous)
    assert sum(v[2] for v in verdicts) > 100          # the probes reach the frontier
