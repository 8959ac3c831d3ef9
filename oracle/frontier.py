"""CPU oracle (test infrastructure only) for the cascade-depth frontier, SURVEY §8 f1.

A numpy restatement of pkg/src/cascadesim/frontier.py:
  * two-stage points  (frontier.py:60-85): for light i < heavy j in latency
    order, theta, tau: bypass = h > theta, reject = !bypass & s_i < tau,
    fid = sum(where(heavy, c_j, c_i)) / n, lat = ((n-nb) L_i + (nb+nr) L_j) / n;
  * three-stage points (frontier.py:88-120): light i < middle j < heavy k,
    theta, tau1, tau2, fid = (sum c_i[on_light] + sum c_j[on_middle] +
    sum c_k[on_heavy]) / n, lat = (#!bypass L_i + #reject1 L_j + #heavy L_k) / n;
  * lower convex envelope (frontier.py:123-143), piecewise-linear evaluation
    (:146-155) and the max gap over the shared range (:158-168).
Scores are noise free: s = 1 / (1 + exp(-(a - s h))), costs c = b + p h.
Pinned bitwise to the reference's output on tests/golden/frontier.json
(generator: tests/golden/make_golden_frontier.py).
"""

from __future__ import annotations

import math

import numpy as np


def model_curves(variants, h):
    """Per model (in the given order): cost and accept-score arrays."""
    costs, scores = [], []
    for v in variants:
        a, s = v.accept_params
        costs.append(v.base_quality_cost + v.hardness_penalty * h)
        scores.append(1.0 / (1.0 + np.exp(-(a - s * h))))
    return costs, scores


def by_latency(variants):
    return sorted(variants, key=lambda v: (v.latency_s[1], v.id))


def two_stage(variants, h, thresholds):
    """[(lat, fid, (light id, heavy id, theta, tau))] in the reference's order."""
    vs = by_latency(variants)
    costs, scores = model_curves(vs, h)
    n = len(h)
    out = []
    for i in range(len(vs)):
        for j in range(i + 1, len(vs)):
            Li, Lj = vs[i].latency_s[1], vs[j].latency_s[1]
            for theta in thresholds:
                by = h > theta
                nb = int(np.count_nonzero(by))
                for tau in thresholds:
                    rej = np.logical_and(np.logical_not(by), scores[i] < tau)
                    nr = int(np.count_nonzero(rej))
                    heavy = np.logical_or(by, rej)
                    fid = float(np.where(heavy, costs[j], costs[i]).sum()) / n
                    lat = ((n - nb) * Li + (nb + nr) * Lj) / n
                    out.append((lat, fid, (vs[i].id, vs[j].id, theta, tau)))
    return out


def three_stage(variants, h, thresholds):
    vs = by_latency(variants)
    costs, scores = model_curves(vs, h)
    n = len(h)
    out = []
    m = len(vs)
    for i in range(m):
        for j in range(i + 1, m):
            for k in range(j + 1, m):
                Li, Lj, Lk = vs[i].latency_s[1], vs[j].latency_s[1], vs[k].latency_s[1]
                for theta in thresholds:
                    by = h > theta
                    keep = np.logical_not(by)
                    for t1 in thresholds:
                        r1 = np.logical_and(keep, scores[i] < t1)
                        for t2 in thresholds:
                            r2 = np.logical_and(r1, scores[j] < t2)
                            light = np.logical_and(keep, np.logical_not(r1))
                            middle = np.logical_and(r1, np.logical_not(r2))
                            heavy = np.logical_or(by, r2)
                            fid = float(costs[i][light].sum() + costs[j][middle].sum()
                                        + costs[k][heavy].sum()) / n
                            lat = (float(np.count_nonzero(keep)) * Li
                                   + float(np.count_nonzero(r1)) * Lj
                                   + float(np.count_nonzero(heavy)) * Lk) / n
                            out.append((lat, fid, (vs[i].id, vs[j].id, vs[k].id, theta, t1, t2)))
    return out


def envelope(points):
    """Lower convex hull of (lat, fid) pairs: lowest fid per latency, then a
    monotone chain that drops vertices on or above the chord."""
    xy = sorted(set(points))
    if not xy:
        raise ValueError("envelope: no points")
    first = []
    for x, y in xy:
        if first and first[-1][0] == x:
            continue
        first.append((x, y))
    hull = []
    for x, y in first:
        while len(hull) >= 2:
            (x1, y1), (x2, y2) = hull[-2], hull[-1]
            if (y2 - y1) * (x - x1) >= (y - y1) * (x2 - x1):
                hull.pop()
            else:
                break
        hull.append((x, y))
    return hull


def envelope_at(hull, x):
    if x < hull[0][0] or x > hull[-1][0]:
        return math.inf
    for (x1, y1), (x2, y2) in zip(hull, hull[1:]):
        if x1 <= x <= x2:
            return min(y1, y2) if x2 == x1 else y1 + (y2 - y1) * (x - x1) / (x2 - x1)
    return hull[-1][1]


def gap(hull_a, hull_b):
    lo = max(hull_a[0][0], hull_b[0][0])
    hi = min(hull_a[-1][0], hull_b[-1][0])
    if hi < lo:
        return 0.0
    xs = sorted({x for x, _ in hull_a} | {x for x, _ in hull_b} | {lo, hi})
    return max(envelope_at(hull_a, x) - envelope_at(hull_b, x) for x in xs if lo <= x <= hi)


def compare(variants, h, thresholds):
    """(gap, envelope_two, envelope_three, n_two, n_three)."""
    p2 = two_stage(variants, h, thresholds)
    p3 = three_stage(variants, h, thresholds)
    e2 = envelope([(a, b) for a, b, _ in p2])
    e3 = envelope([(a, b) for a, b, _ in p3])
    return gap(e2, e3), e2, e3, len(p2), len(p3)
