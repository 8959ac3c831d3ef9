"""Oracle: grid evaluator + Pareto extractor of the cascade profiler.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Array-level restatement of ``cascadesim.profiler.profile_config`` after its
text phase: given the selected pool, per-query hardness ``h`` and per-model
scores (both in ``stable_text_key`` order), reproduce the table rows the
reference emits.  Every arithmetic expression keeps the reference's numpy op
order so results are bit-identical to the reference on the same records.

Model objects are duck-typed: anything with ``id``, ``latency_s`` (dict
batch -> seconds), ``base_quality_cost``, ``hardness_penalty`` and
``accept_params`` works (the reference's ``ModelVariant`` or ours).
"""

from __future__ import annotations

import math

import numpy as np

ROW_FIELDS = ("light_id", "heavy_id", "theta", "tau", "r_light", "r_heavy",
              "fidelity_cost", "mean_latency_s")


def model_arrays(pool, h, noise):
    """Per-model cost and discriminator-score arrays (profiler.py:133-137).

    cost_m  = base_m + pen_m * h                       (numpy, elementwise)
    score_m = clip(1 / (1 + exp(-(a_m - s_m * h))) + noise, 0, 1)
    """
    h = np.asarray(h, dtype=np.float64)
    noise = np.asarray(noise, dtype=np.float64)
    cost, score = {}, {}
    for v in pool:
        cost[v.id] = v.base_quality_cost + v.hardness_penalty * h
        a, slope = v.accept_params
        curve = 1.0 / (1.0 + np.exp(-(a - slope * h)))
        score[v.id] = np.clip(curve + noise, 0.0, 1.0)
    return cost, score


def light_heavy_pairs(pool):
    """Ordered (light, heavy) pairs, light strictly faster (profiler.py:141-143)."""
    order = sorted(pool, key=lambda v: (v.latency_s[1], v.id))
    return [(order[i], order[j]) for i in range(len(order))
            for j in range(i + 1, len(order))]


def pareto_keep(lat, qual):
    """Indices kept by ``catalog.pareto_prune`` (catalog.py:171-192), in its
    output order: sort by (latency, quality, original index), keep a row iff
    its quality is strictly below every quality seen before it."""
    order = sorted(range(len(lat)), key=lambda i: (lat[i], qual[i], i))
    kept, best = [], math.inf
    for i in order:
        if qual[i] < best:
            kept.append(i)
            best = qual[i]
    return kept


def cell_stats(h, light_score, light_cost, heavy_cost, lat_light, lat_heavy, theta, tau,
               bypass=None, n_bypass=None):
    """One grid cell exactly as profiler.py:146-165 computes it.

    ``bypass`` / ``n_bypass`` are the per-theta values the reference computes
    once (``bypass_at[theta]``, profiler.py:138, and ``n_bypass`` per theta
    row, :146-147); pass them when evaluating a whole theta row.
    Returns (n_bypass, n_reject, r_light, r_heavy, fid, mean_lat)."""
    n = h.shape[0]
    if bypass is None:
        bypass = h > theta
    if n_bypass is None:
        n_bypass = int(bypass.sum())
    reject = ~bypass & (light_score < tau)
    n_reject = int(reject.sum())
    heavy = bypass | reject
    fid = float(np.where(heavy, heavy_cost, light_cost).mean())
    lat = ((n - n_bypass) * lat_light + (n_bypass + n_reject) * lat_heavy) / n
    return (n_bypass, n_reject, (n - n_bypass) / n, (n_bypass + n_reject) / n, fid, lat)


def theta_row(h, light_score, light_cost, heavy_cost, lat_light, lat_heavy, theta, taus):
    """Every tau cell of one theta row, with the reference's per-theta hoisting
    (profiler.py:138, 145-149)."""
    bypass = h > theta
    n_bypass = int(bypass.sum())
    return [cell_stats(h, light_score, light_cost, heavy_cost, lat_light, lat_heavy, theta, tau,
                       bypass, n_bypass) for tau in taus]


def pair_grid(h, light, heavy, cost, score, thresholds):
    """Every (theta, tau) cell of one pair, in grid order (index = i*K + j)."""
    cells = []
    for theta in thresholds:
        for tau, (nb, nr, rl, rh, fid, lat) in zip(thresholds, theta_row(
                h, score[light.id], cost[light.id], cost[heavy.id], light.latency_s[1],
                heavy.latency_s[1], theta, thresholds)):
            cells.append((light.id, heavy.id, theta, tau, rl, rh, fid, lat))
    return cells


def pair_frontier(cells, thresholds):
    """Frontier + theta=max no-bypass sub-frontier, merged and sorted by
    (theta, tau) as profiler.py:166-174 does (dict semantics included)."""
    lat = [c[7] for c in cells]
    fid = [c[6] for c in cells]
    front = [cells[i] for i in pareto_keep(lat, fid)]
    top = max(thresholds)
    nb_cells = [c for c in cells if c[2] == top]
    nb_front = [nb_cells[i] for i in pareto_keep([c[7] for c in nb_cells],
                                                 [c[6] for c in nb_cells])]
    merged = {(c[2], c[3]): c for c in front}
    for c in nb_front:
        merged.setdefault((c[2], c[3]), c)
    return [merged[k] for k in sorted(merged)]


def profile_rows(pool, h, noise=None, thresholds=(), scores=None):
    """All table rows (tuples in ROW_FIELDS order) for a pool.

    Give either ``noise`` (scores derived as the reference does) or explicit
    ``scores`` (dict model id -> float64[N]); ``h`` must be in the same
    (``stable_text_key``) order as the reference would use.
    """
    thresholds = tuple(float(t) for t in thresholds)
    h = np.asarray(h, dtype=np.float64)
    if scores is None:
        cost, scores = model_arrays(pool, h, noise)
    else:
        cost = {v.id: v.base_quality_cost + v.hardness_penalty * h for v in pool}
        scores = {k: np.asarray(s, dtype=np.float64) for k, s in scores.items()}
    rows = []
    for light, heavy in light_heavy_pairs(pool):
        cells = pair_grid(h, light, heavy, cost, scores, thresholds)
        rows.extend(pair_frontier(cells, thresholds))
    return rows


_PAR = None


def _par_rows(job):
    h, cost, scores, pairs, thresholds = _PAR
    pi, t0, t1 = job
    light, heavy = pairs[pi]
    out = []
    for theta in thresholds[t0:t1]:
        for tau, (nb, nr, rl, rh, fid, lat) in zip(thresholds, theta_row(
                h, scores[light.id], cost[light.id], cost[heavy.id], light.latency_s[1],
                heavy.latency_s[1], theta, thresholds)):
            out.append((light.id, heavy.id, theta, tau, rl, rh, fid, lat))
    return pi, t0, out


def profile_rows_parallel(pool, h, scores, thresholds, procs):
    """profile_rows with the cell grid split over ``procs`` forked processes
    (jobs = (pair, theta block)); the per-pair frontier runs in the parent.
    Same values as profile_rows (each cell is the same numpy computation)."""
    import multiprocessing as mp
    global _PAR
    thresholds = tuple(float(t) for t in thresholds)
    h = np.asarray(h, dtype=np.float64)
    cost = {v.id: v.base_quality_cost + v.hardness_penalty * h for v in pool}
    scores = {k: np.asarray(s, dtype=np.float64) for k, s in scores.items()}
    pairs = light_heavy_pairs(pool)
    K = len(thresholds)
    step = max(1, K // 32)
    jobs = [(pi, t0, min(K, t0 + step)) for pi in range(len(pairs)) for t0 in range(0, K, step)]
    _PAR = (h, cost, scores, pairs, thresholds)
    try:
        with mp.get_context("fork").Pool(procs) as pool_:
            parts = pool_.map(_par_rows, jobs, chunksize=1)
    finally:
        _PAR = None
    by_pair = {}
    for pi, t0, cells in sorted(parts, key=lambda x: (x[0], x[1])):
        by_pair.setdefault(pi, []).extend(cells)
    rows = []
    for pi in range(len(pairs)):
        rows.extend(pair_frontier(by_pair[pi], thresholds))
    return rows


# ---------------------------------------------------------------------------
# numpy pairwise summation (what ``ndarray.mean`` does for contiguous float64)

_PW_BLOCK = 128


def pairwise_sum(a, lo=0, n=None):
    """Bit-exact restatement of numpy's float64 pairwise reduction.

    numpy sums a contiguous float64 array by recursive halving (split point
    rounded down to a multiple of 8) until a block has <= 128 elements; such
    a block is summed with 8 interleaved accumulators combined as
    ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the <8 tail added in order;
    blocks shorter than 8 are summed left to right from 0.0.  Checked against
    ``np.add.reduce`` for n in 1..300 and up to 1e6 (tests/test_oracle_golden.py).
    """
    if n is None:
        n = len(a)
    if n < 8:
        acc = 0.0
        for i in range(lo, lo + n):
            acc += a[i]
        return acc
    if n <= _PW_BLOCK:
        r = [a[lo + j] for j in range(8)]
        i = 8
        stop = n - (n % 8)
        while i < stop:
            for j in range(8):
                r[j] += a[lo + i + j]
            i += 8
        acc = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            acc += a[lo + i]
            i += 1
        return acc
    half = n // 2
    half -= half % 8
    return pairwise_sum(a, lo, half) + pairwise_sum(a, lo + half, n - half)


def pairwise_leaves(n):
    """Leaf blocks (offset, length) of the pairwise recursion, left to right."""
    out = []
    stack = [(0, n)]
    while stack:
        lo, m = stack.pop()
        if m <= _PW_BLOCK:
            out.append((lo, m))
            continue
        half = m // 2
        half -= half % 8
        stack.append((lo + half, m - half))
        stack.append((lo, half))
    return out
