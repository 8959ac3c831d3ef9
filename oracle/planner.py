"""Oracle: allocation search of the online planner.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Plain-Python restatement of ``cascadesim.planner`` (planner.py:81-321):
``solve`` -> ``_solve_over_rows`` -> ``_evaluate_row`` with the
``fallback_plan`` overload path, the exhaustive ``brute_force_solve`` and the
``validate_plan`` auditor.  Rows are duck-typed (``light_id``, ``heavy_id``,
``r_light``, ``r_heavy``, ``fidelity_cost``); catalogs need ``by_id`` and
``batch_sizes``.  Results are returned as plain dicts so tests can compare
them field by field with the GPU planner and with golden fixtures.
"""

from __future__ import annotations

import math

SLACK = 1e-9          # planner.py:32
RATE_FLOOR = 0.01     # planner.py:33


class OraclePlannerError(ValueError):
    pass


def shares_of(row):
    """CascadeRow.shares (profiler.py:58-61): merged when light == heavy."""
    out = {row.light_id: row.r_light}
    out[row.heavy_id] = out.get(row.heavy_id, 0.0) + row.r_heavy
    return out


def models_of(row):
    return [row.light_id] if row.light_id == row.heavy_id else [row.light_id, row.heavy_id]


def drain(q, rate, alpha):
    """queue_delay (planner.py:81-85)."""
    if q <= 0:
        return 0.0
    return alpha * q / max(rate, RATE_FLOOR)


def path_latency(row, catalog, batches, lam, queues, alpha):
    """sum(lat + d) over the row's models (planner.py:93-104, 138-139)."""
    shares = shares_of(row)
    total = 0
    for m in models_of(row):
        lat = catalog.by_id(m).latency_s[batches[m]]
        total = total + (lat + drain(queues.get(m, 0.0), lam * shares[m], alpha))
    return total


def min_workers(rate, mu):
    """planner.py:107-110."""
    if rate <= 0:
        return 1
    return max(1, math.ceil((rate - SLACK) / mu))


def batch_combos(active, batch_sizes):
    combos = [()]
    for _ in active:
        combos = [c + (b,) for c in combos for b in batch_sizes]
    return combos


def best_for_row(row, catalog, lam, queues, workers, t_slo, alpha):
    """_evaluate_row (planner.py:113-148): min (total, path), first wins."""
    shares = shares_of(row)
    models = models_of(row)
    active = [m for m in models if shares[m] > 0]
    inactive = [m for m in models if shares[m] <= 0]
    best = None
    for combo in batch_combos(active, catalog.batch_sizes):
        batches = dict(zip(active, combo))
        for m in inactive:
            batches[m] = catalog.batch_sizes[0]
        x = {}
        for m in models:
            if shares[m] > 0:
                x[m] = min_workers(lam * shares[m], catalog.by_id(m).throughput_qps[batches[m]])
            else:
                x[m] = 0
        total = sum(x.values())
        if total > workers:
            continue
        path = path_latency(row, catalog, batches, lam, queues, alpha)
        if path > t_slo + SLACK:
            continue
        if best is None or (total, path) < best[0]:
            best = ((total, path), batches, x)
    return best


def _plan(row, idx, workers_map, batches, lam, queues, path, infeasible):
    return {"row_index": idx, "light_id": row.light_id, "heavy_id": row.heavy_id,
            "theta": row.theta, "tau": row.tau,
            "workers": dict(workers_map), "batches": dict(batches), "lam": lam,
            "queues": dict(queues), "fidelity_cost": row.fidelity_cost,
            "path_latency_s": path, "infeasible": infeasible}


def overload(rows, catalog, lam, queues, workers, alpha):
    """fallback_plan (planner.py:170-214): max bottleneck capacity."""
    best = None
    for idx, row in rows:
        shares = shares_of(row)
        models = models_of(row)
        active = [m for m in models if shares[m] > 0]
        if not active:
            continue
        lat_l = catalog.by_id(row.light_id).latency_s[1]
        lat_h = catalog.by_id(row.heavy_id).latency_s[1]
        for combo in batch_combos(active, catalog.batch_sizes):
            batches = dict(zip(active, combo))
            for m in models:
                batches.setdefault(m, catalog.batch_sizes[0])
            mus = {m: catalog.by_id(m).throughput_qps[batches[m]] for m in active}
            if len(active) == 1:
                splits = [{active[0]: workers}]
            else:
                splits = [{active[0]: i, active[1]: workers - i} for i in range(1, workers)]
            for x in splits:
                cap = min(x[m] * mus[m] / shares[m] for m in active)
                key = (-cap, lat_l, lat_h, idx)
                if best is None or key < best[0]:
                    full = {m: x.get(m, 0) for m in models}
                    path = path_latency(row, catalog, batches, lam, queues, alpha)
                    best = (key, row, idx, batches, full, path)
    if best is None:
        raise OraclePlannerError("fallback: no serveable rows")
    _, row, idx, batches, x, path = best
    return _plan(row, idx, x, batches, lam, queues, path, True)


def solve(rows, catalog, lam, queues=None, workers=16, t_slo=60.0, alpha=1.5):
    """planner.solve (planner.py:217-227) over ``rows`` (a sequence)."""
    if lam < 0:
        raise OraclePlannerError("solve: negative demand")
    queues = queues or {}
    indexed = list(enumerate(rows))
    best = None
    for idx, row in indexed:
        got = best_for_row(row, catalog, lam, queues, workers, t_slo, alpha)
        if got is None:
            continue
        (total, path), batches, x = got
        key = (row.fidelity_cost, total, path, idx)
        if best is None or key < best[0]:
            best = (key, row, idx, batches, x, path)
    if best is None:
        return overload(indexed, catalog, lam, queues, workers, alpha)
    _, row, idx, batches, x, path = best
    return _plan(row, idx, x, batches, lam, queues, path, False)


def brute_force(rows, catalog, lam, queues=None, workers=16, t_slo=60.0, alpha=1.5):
    """brute_force_solve (planner.py:230-288): every worker split."""
    if len(rows) > 200 or workers > 16 or len(catalog.batch_sizes) > 5:
        raise OraclePlannerError("oracle-too-large")
    queues = queues or {}
    best = None
    for idx, row in enumerate(rows):
        shares = shares_of(row)
        models = models_of(row)
        active = [m for m in models if shares[m] > 0]
        if not active:
            continue
        for combo in batch_combos(active, catalog.batch_sizes):
            batches = dict(zip(active, combo))
            for m in models:
                batches.setdefault(m, catalog.batch_sizes[0])
            if len(active) == 1:
                options = [{active[0]: a} for a in range(1, workers + 1)]
            else:
                options = [{active[0]: a, active[1]: b} for a in range(1, workers + 1)
                           for b in range(1, workers + 1 - a)]
            for xa in options:
                if any(xa[m] * catalog.by_id(m).throughput_qps[batches[m]]
                       < lam * shares[m] - SLACK for m in active):
                    continue
                x = {m: xa.get(m, 0) for m in models}
                total = sum(x.values())
                if total > workers:
                    continue
                path = path_latency(row, catalog, batches, lam, queues, alpha)
                if path > t_slo + SLACK:
                    continue
                key = (row.fidelity_cost, total, path, idx)
                if best is None or key < best[0]:
                    best = (key, row, idx, batches, x, path)
    if best is None:
        return overload(list(enumerate(rows)), catalog, lam, queues, workers, alpha)
    _, row, idx, batches, x, path = best
    return _plan(row, idx, x, batches, lam, queues, path, False)


def audit(plan, row, catalog, workers=16, t_slo=60.0, alpha=1.5):
    """validate_plan (planner.py:291-321): list of violated constraints."""
    problems = []
    if sum(plan["workers"].values()) > workers:
        problems.append("worker-budget")
    shares = shares_of(row)
    for m in models_of(row):
        need = plan["lam"] * shares.get(m, 0.0)
        x = plan["workers"].get(m, 0)
        b = plan["batches"].get(m)
        if b is None:
            problems.append(f"missing-batch: {m}")
            continue
        mu = catalog.by_id(m).throughput_qps[b]
        if need > 0 and x * mu < need - SLACK:
            problems.append(f"capacity: {m}")
        if need > 0 and x < 1:
            problems.append(f"no-workers: {m}")
    path = path_latency(row, catalog, plan["batches"], plan["lam"], plan["queues"], alpha)
    if path > t_slo + SLACK:
        problems.append("path-latency")
    return problems
