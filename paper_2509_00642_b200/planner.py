"""Online allocation search on the GPU: drop-in for cascadesim.planner.solve.

Public surface mirrors pkg/src/cascadesim/planner.py:
``Plan`` (:40-78), ``PlannerError`` (:36), ``queue_delay`` (:81),
``update_estimate`` (:88), ``solve`` (:217-227), ``fallback_plan``
(:170-214), the consumers ``PlanCache`` / ``cached_solve`` (:328-367), the
baselines ``clipper_plan`` / ``proteus_plan`` / ``diffserve_plan``
(:387-500) and every ``make_planner`` mode (:443-479), the audit helpers
``brute_force_solve`` / ``validate_plan`` (:230-325, host arithmetic, as in the
reference), plus the batched ``solve_many`` used by re-plan sweeps.  Every (demand, SLO) point is decided
on the device by ``hadis_solve_many`` with the reference's exact float64
expressions and tie-breaks; this module only moves rows/points to the device
and turns the per-point result back into ``Plan`` objects.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib

DEFAULT_WORKERS = 16
DEFAULT_T_SLO_S = 60.0
DEFAULT_QUEUE_ALPHA = 1.5
EWMA_WEIGHT = 0.3
SOLVER_DELAY_S = 0.03
_RATE_FLOOR = 0.01
_SLACK = 1e-9
_MAX_POINTS_PER_LAUNCH = 65535


class PlannerError(ValueError):
    pass


@dataclass(frozen=True)
class Plan:
    row: object
    workers: dict
    batches: dict
    lam: float
    queues: dict
    fidelity_cost: float
    path_latency_s: float
    infeasible: bool = False
    label: str = "online"

    @property
    def total_workers(self) -> int:
        return sum(self.workers.values())

    def pair_models(self) -> list:
        models = [self.row.light_id]
        if self.row.heavy_id != self.row.light_id:
            models.append(self.row.heavy_id)
        return models

    def describe(self) -> dict:
        return {
            "label": self.label, "light": self.row.light_id, "heavy": self.row.heavy_id,
            "theta": self.row.theta, "tau": self.row.tau, "r_light": self.row.r_light,
            "r_heavy": self.row.r_heavy, "workers": dict(sorted(self.workers.items())),
            "batches": dict(sorted(self.batches.items())), "lam": self.lam,
            "queues": dict(sorted(self.queues.items())), "fidelity_cost": self.fidelity_cost,
            "path_latency_s": self.path_latency_s, "infeasible": self.infeasible,
        }


def queue_delay(queue_len: float, rate_qps: float, alpha: float = DEFAULT_QUEUE_ALPHA) -> float:
    """Drain-time estimate for a backlog (planner.py:81-85)."""
    if queue_len <= 0:
        return 0.0
    return alpha * queue_len / max(rate_qps, _RATE_FLOOR)


def update_estimate(estimate: float, observed: float, weight: float = EWMA_WEIGHT) -> float:
    """EWMA demand tracker (planner.py:88-90)."""
    return weight * observed + (1.0 - weight) * estimate


def row_arrays(rows, index):
    """Planner inputs of a row sequence: (light, heavy) catalog indices
    int32[R][2], shares float64[R][2] (r_light, r_heavy) and fidelity
    float64[R].  A columnar ``CascadeRows`` table is converted column-wise
    (no row objects); unknown model ids raise CatalogError as the reference
    catalog lookup does."""
    from .profiler import CascadeRows
    try:
        if isinstance(rows, CascadeRows):
            pair, pair_ids, r_l, r_h, fid = rows.columns()
            pm = np.array([(index[a], index[b]) for a, b in pair_ids], dtype=np.int32)
            rm = np.ascontiguousarray(pm.reshape(-1, 2)[pair.astype(np.int64)])
            share = np.ascontiguousarray(np.stack([r_l, r_h], axis=1))
            fid = np.ascontiguousarray(fid)
        else:
            rm = np.array([(index[r.light_id], index[r.heavy_id]) for r in rows],
                          dtype=np.int32).reshape(-1, 2)
            share = np.array([(r.r_light, r.r_heavy) for r in rows],
                             dtype=np.float64).reshape(-1, 2)
            fid = np.array([r.fidelity_cost for r in rows], dtype=np.float64)
    except KeyError as exc:
        from .catalog import CatalogError
        raise CatalogError(f"unknown-variant: {exc.args[0]!r}") from None
    return rm, share, fid


class DeviceRows:
    """A table's rows and its catalog's latency/throughput tables in HBM.

    Built once per (rows, catalog) and reused for every planning call; ``rows``
    is any sequence of CascadeRow-like objects (ours or the reference's)."""

    def __init__(self, rows, catalog, device=None):
        torch = _lib.torch_cuda()
        self.torch = torch
        from .profiler import CascadeRows
        self.rows = rows if isinstance(rows, CascadeRows) else tuple(rows)
        self.catalog = catalog
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.device = dev
        ids = [v.id for v in catalog.variants]
        self.model_ids = ids
        bs = tuple(catalog.batch_sizes)
        self.batch_sizes = bs
        if not self.rows:
            raise PlannerError("fallback: no serveable rows")
        rm, share, fid = row_arrays(self.rows, {m: i for i, m in enumerate(ids)})
        variants = [catalog.by_id(m) for m in ids]
        lat = np.array([[v.latency_s[b] for b in bs] for v in variants], dtype=np.float64)
        mu = np.array([[v.throughput_qps[b] for b in bs] for v in variants], dtype=np.float64)
        lat1 = np.array([v.latency_s.get(1, np.nan) for v in variants], dtype=np.float64)
        self.d_model = torch.from_numpy(rm).to(dev)
        self.d_share = torch.from_numpy(share).to(dev)
        self.d_fid = torch.from_numpy(fid).to(dev)
        self.d_batch = torch.tensor(bs, dtype=torch.int32, device=dev)
        self.d_lat = torch.from_numpy(lat).to(dev)
        self.d_mu = torch.from_numpy(mu).to(dev)
        self.d_lat1 = torch.from_numpy(lat1).to(dev)
        self._ws = None

    @classmethod
    def from_device_table(cls, dt, pool, catalog):
        """Planner rows straight from a profiler DeviceTable (no host row
        objects): light/heavy catalog indices per pair, shares and fidelity stay
        on the device.  ``rows`` is left empty; plans carry row indices."""
        torch = _lib.torch_cuda()
        self = cls.__new__(cls)
        self.torch = torch
        self.catalog = catalog
        self.device = dt.pair.device
        ids = [v.id for v in catalog.variants]
        self.model_ids = ids
        index = {m: i for i, m in enumerate(ids)}
        self.batch_sizes = tuple(catalog.batch_sizes)
        pm = torch.tensor([(index[pool[i].id], index[pool[j].id]) for i, j in dt.pairs],
                          dtype=torch.int32, device=self.device)
        self.d_model = pm[dt.pair.long()].contiguous()
        self.d_share = torch.stack([dt.r_light, dt.r_heavy], dim=1).contiguous()
        self.d_fid = dt.fid.contiguous()
        variants = [catalog.by_id(m) for m in ids]
        bs = self.batch_sizes
        self.d_batch = torch.tensor(bs, dtype=torch.int32, device=self.device)
        self.d_lat = torch.tensor([[v.latency_s[b] for b in bs] for v in variants],
                                  dtype=torch.float64, device=self.device)
        self.d_mu = torch.tensor([[v.throughput_qps[b] for b in bs] for v in variants],
                                 dtype=torch.float64, device=self.device)
        self.d_lat1 = torch.tensor([v.latency_s.get(1, float("nan")) for v in variants],
                                   dtype=torch.float64, device=self.device)
        self.rows = ()
        self.n_rows = int(dt.n_rows)
        self._ws = None
        return self

    def queue_matrix(self, queues_list):
        q = np.zeros((len(queues_list), len(self.model_ids)), dtype=np.float64)
        col = {m: i for i, m in enumerate(self.model_ids)}
        for p, queues in enumerate(queues_list):
            for m, v in (queues or {}).items():
                if m in col:
                    q[p, col[m]] = v
        return q

    def launch(self, lam, t_slo, workers, qmat, alpha, stream=None):
        """Enqueue one batched solve; returns device result tensors."""
        torch = self.torch
        dev = self.device
        P = int(lam.shape[0])
        lib = _lib.load()
        if torch.cuda.current_device() != dev.index and dev.index is not None:
            with torch.cuda.device(dev):
                return self.launch(lam, t_slo, workers, qmat, alpha, stream)
        n_rows = len(self.rows) if self.rows else self.n_rows
        ws_bytes = lib.hadis_solve_workspace_bytes(P, n_rows)
        if self._ws is None or self._ws.numel() < ws_bytes:
            self._ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        out = dict(row=torch.empty(P, dtype=torch.int32, device=dev),
                   x=torch.empty(2 * P, dtype=torch.int32, device=dev),
                   b=torch.empty(2 * P, dtype=torch.int32, device=dev),
                   path=torch.empty(P, dtype=torch.float64, device=dev),
                   flags=torch.empty(P, dtype=torch.int32, device=dev))
        p = _lib.ptr
        _lib.check(lib.hadis_solve_many(
            n_rows, p(self.d_model), p(self.d_share), p(self.d_fid), len(self.model_ids),
            len(self.batch_sizes), p(self.d_batch), p(self.d_lat), p(self.d_mu), p(self.d_lat1), P,
            p(lam), p(t_slo), p(workers), p(qmat), float(alpha), p(out["row"]), p(out["x"]),
            p(out["b"]), p(out["path"]), p(out["flags"]), p(self._ws), ws_bytes,
            _lib.stream_handle(stream, dev)), "hadis_solve_many")
        return out

    def solve_arrays(self, lams, t_slos, workers, queues_list, alpha):
        """Host arrays in, host result arrays out (one device round trip per chunk)."""
        torch = self.torch
        dev = self.device
        lams = np.asarray(lams, dtype=np.float64)
        t_slos = np.asarray(t_slos, dtype=np.float64)
        workers = np.asarray(workers, dtype=np.int32)
        qmat = self.queue_matrix(queues_list)
        res = {k: [] for k in ("row", "x", "b", "path", "flags")}
        for s in range(0, lams.shape[0], _MAX_POINTS_PER_LAUNCH):
            e = min(lams.shape[0], s + _MAX_POINTS_PER_LAUNCH)
            out = self.launch(torch.from_numpy(lams[s:e]).to(dev),
                              torch.from_numpy(t_slos[s:e]).to(dev),
                              torch.from_numpy(workers[s:e]).to(dev),
                              torch.from_numpy(qmat[s:e]).to(dev), alpha)
            for k in res:
                res[k].append(out[k].cpu().numpy())
        return {k: np.concatenate(v) for k, v in res.items()}


def _plan_from(dr: DeviceRows, res, p, lam, queues, label):
    flags = int(res["flags"][p])
    ri = int(res["row"][p])
    if ri < 0:
        raise PlannerError("fallback: no serveable rows")
    row = dr.rows[ri]
    infeasible = bool(flags & 1)
    xl, xh = int(res["x"][2 * p]), int(res["x"][2 * p + 1])
    bl, bh = int(res["b"][2 * p]), int(res["b"][2 * p + 1])
    shares = {row.light_id: row.r_light}
    shares[row.heavy_id] = shares.get(row.heavy_id, 0.0) + row.r_heavy
    if row.light_id == row.heavy_id:
        models, x, b = [row.light_id], {row.light_id: xl}, {row.light_id: bl}
    else:
        models = [row.light_id, row.heavy_id]
        x = {row.light_id: xl, row.heavy_id: xh}
        b = {row.light_id: bl, row.heavy_id: bh}
    active = [m for m in models if shares[m] > 0]
    # dict insertion order as the reference builds it (active models first)
    batches = {m: b[m] for m in active}
    for m in models:
        batches.setdefault(m, b[m])
    workers_map = {m: x[m] for m in models}
    return Plan(row=row, workers=workers_map, batches=batches, lam=lam,
                queues=dict(queues or {}), fidelity_cost=row.fidelity_cost,
                path_latency_s=float(res["path"][p]), infeasible=infeasible, label=label)


_CACHE: dict = {}


def device_rows(rows, catalog) -> DeviceRows:
    """Cached DeviceRows for a (rows, catalog) pair (rebuilt when either changes)."""
    key = (id(rows), id(catalog))
    hit = _CACHE.get(key)
    if hit is not None and hit.catalog is catalog and \
            (hit.rows is rows or hit.rows == tuple(rows)):
        return hit
    if len(_CACHE) > 32:
        _CACHE.clear()
    dr = DeviceRows(rows, catalog)
    _CACHE[key] = dr
    return dr


def solve_many(table, catalog, lams, queues=None, workers=DEFAULT_WORKERS, t_slo=DEFAULT_T_SLO_S,
               alpha=DEFAULT_QUEUE_ALPHA, label="online"):
    """planner.solve for many points at once; scalars broadcast, lists are per point.
    Like ``solve`` (planner.py:221-222), a negative demand raises PlannerError."""
    lams = [float(x) for x in lams]
    if any(x < 0 for x in lams):
        raise PlannerError("solve: negative demand")
    return _solve_points(table, catalog, lams, queues, workers, t_slo, alpha, label)


def _solve_points(table, catalog, lams, queues, workers, t_slo, alpha, label):
    """_solve_over_rows + fallback_plan (planner.py:151-214) per point, any demand."""
    lams = [float(x) for x in lams]
    P = len(lams)
    t_slos = [float(t_slo)] * P if np.isscalar(t_slo) else [float(x) for x in t_slo]
    ws = [int(workers)] * P if np.isscalar(workers) else [int(x) for x in workers]
    qs = [queues] * P if (queues is None or isinstance(queues, dict)) else list(queues)
    rows = table.rows if hasattr(table, "rows") else table
    dr = device_rows(rows, catalog)
    res = dr.solve_arrays(lams, t_slos, ws, qs, alpha)
    return [_plan_from(dr, res, p, lams[p], qs[p], label) for p in range(P)]


def solve(table, catalog, lam: float, queues=None, workers: int = DEFAULT_WORKERS,
          t_slo: float = DEFAULT_T_SLO_S, alpha: float = DEFAULT_QUEUE_ALPHA,
          label: str = "online") -> Plan:
    """Pick the feasible table row with the lowest fidelity cost (planner.py:217-227)."""
    if lam < 0:
        raise PlannerError("solve: negative demand")
    return solve_many(table, catalog, [lam], queues, workers, t_slo, alpha, label)[0]


def _row_models(row) -> list:
    return [row.light_id] if row.light_id == row.heavy_id else [row.light_id, row.heavy_id]


def _row_shares(row) -> dict:
    out = {row.light_id: row.r_light}
    out[row.heavy_id] = out.get(row.heavy_id, 0.0) + row.r_heavy
    return out


def _path_latency(row, catalog, batches, lam, queues, alpha) -> float:
    """sum(latency + drain) over the path's unique models, the reference's
    left-to-right float order (planner.py:93-104 summed as at :136-140)."""
    shares = _row_shares(row)
    total = 0
    for m in _row_models(row):
        variant = catalog.by_id(m)
        total = total + (variant.latency_s[batches[m]]
                         + queue_delay(queues.get(m, 0.0), lam * shares[m], alpha))
    return total


def brute_force_solve(table, catalog, lam: float, queues=None, workers: int = DEFAULT_WORKERS,
                      t_slo: float = DEFAULT_T_SLO_S, alpha: float = DEFAULT_QUEUE_ALPHA) -> Plan:
    """Exhaustive cross-check of ``solve`` (planner.py:230-288): every worker
    split, not only the minimal one, same key (fid, total workers, path, row
    index).  An audit aid on small instances, computed on the host exactly as
    the reference does; the overload branch is the device ``fallback_plan``."""
    rows = list(table.rows if hasattr(table, "rows") else table)
    if len(rows) > 200 or workers > 16 or len(catalog.batch_sizes) > 5:
        raise PlannerError("oracle-too-large: brute force capped at "
                           "200 rows / 16 workers / 5 batch sizes")
    queues = queues or {}
    best = None
    for idx, row in enumerate(rows):
        shares = _row_shares(row)
        models = _row_models(row)
        active = [m for m in models if shares[m] > 0]
        if not active:
            continue
        combos = [()]
        for _ in active:
            combos = [c + (b,) for c in combos for b in catalog.batch_sizes]
        for combo in combos:
            batches = dict(zip(active, combo))
            for m in models:
                batches.setdefault(m, catalog.batch_sizes[0])
            if len(active) == 1:
                splits = [{active[0]: a} for a in range(1, workers + 1)]
            else:
                splits = [{active[0]: a, active[1]: b} for a in range(1, workers + 1)
                          for b in range(1, workers + 1 - a)]
            for xa in splits:
                if any(xa[m] * catalog.by_id(m).throughput_qps[batches[m]]
                       < lam * shares[m] - _SLACK for m in active):
                    continue
                x = {m: xa.get(m, 0) for m in models}
                total = sum(x.values())
                if total > workers:
                    continue
                path = _path_latency(row, catalog, batches, lam, queues, alpha)
                if path > t_slo + _SLACK:
                    continue
                key = (row.fidelity_cost, total, path, idx)
                if best is None or key < best[0]:
                    best = (key, row, batches, x, path)
    if best is None:
        return fallback_plan(list(enumerate(rows)), catalog, lam, queues, workers, t_slo, alpha,
                             "online")
    _, row, batches, x, path = best
    return Plan(row=row, workers=x, batches=batches, lam=lam, queues=dict(queues),
                fidelity_cost=row.fidelity_cost, path_latency_s=path, infeasible=False,
                label="online")


def validate_plan(plan: Plan, catalog, workers: int = DEFAULT_WORKERS,
                  t_slo: float = DEFAULT_T_SLO_S, alpha: float = DEFAULT_QUEUE_ALPHA) -> list:
    """Independent feasibility audit of a plan (planner.py:291-321): the
    violated constraints as the reference's human-readable strings."""
    problems = []
    if plan.total_workers > workers:
        problems.append(f"worker-budget: {plan.total_workers} > {workers}")
    shares = _row_shares(plan.row)
    for m in plan.pair_models():
        share = shares.get(m, 0.0)
        x = plan.workers.get(m, 0)
        batch = plan.batches.get(m)
        if batch is None:
            problems.append(f"missing-batch: {m}")
            continue
        variant = catalog.by_id(m)
        if batch not in variant.latency_s:
            problems.append(f"unprofiled-batch: {m} b={batch}")
            continue
        need = plan.lam * share
        cap = x * variant.throughput_qps[batch]
        if need > 0 and cap < need - _SLACK:
            problems.append(f"capacity: {m} x={x} covers {cap:.6f} qps < {need:.6f}")
        if need > 0 and x < 1:
            problems.append(f"no-workers: {m} has load but x=0")
    path = _path_latency(plan.row, catalog, plan.batches, plan.lam, plan.queues, alpha)
    if path > t_slo + _SLACK:
        problems.append(f"path-latency: {path:.6f} > {t_slo}")
    return problems


def fallback_plan(indexed_rows, catalog, lam, queues, workers, t_slo, alpha, label):
    """Overload plan over explicit (index, row) pairs (planner.py:170-214).

    Runs the same device search with an SLO no plan can meet, so the
    fallback branch decides; indices are the caller's."""
    indexed_rows = list(indexed_rows)
    if not indexed_rows:
        raise PlannerError("fallback: no serveable rows")
    rows = [r for _, r in indexed_rows]
    order = sorted(range(len(indexed_rows)), key=lambda i: indexed_rows[i][0])
    ordered = [rows[i] for i in order]
    return _solve_points(ordered, catalog, [lam], queues, workers, -float("inf"), alpha, label)[0]


@dataclass
class PlanCache:
    """Reuse plans for nearby states instead of re-solving each epoch
    (planner.py:328-351): mode 'd' keys on the binned demand estimate, 'dq'
    also on the binned total backlog."""

    mode: str
    demand_bin_qps: float = 10.0
    queue_bin: int = 12
    entries: dict = field(default_factory=dict)
    hits: int = 0
    misses: int = 0

    def __post_init__(self) -> None:
        if self.mode not in ("d", "dq"):
            raise PlannerError(f"cache mode must be 'd' or 'dq', got {self.mode!r}")

    def key(self, lam: float, queues) -> tuple:
        demand_key = int(lam // self.demand_bin_qps)
        if self.mode == "d":
            return (demand_key,)
        return (demand_key, int(sum((queues or {}).values()) // self.queue_bin))


def cached_solve(cache: PlanCache, table, catalog, lam: float, queues=None,
                 workers: int = DEFAULT_WORKERS, t_slo: float = DEFAULT_T_SLO_S,
                 alpha: float = DEFAULT_QUEUE_ALPHA):
    """Solve through the cache (planner.py:354-367); returns (plan, was_cache_hit)."""
    key = cache.key(lam, queues)
    hit = cache.entries.get(key)
    if hit is not None:
        cache.hits += 1
        return hit, True
    plan = solve(table, catalog, lam, queues, workers, t_slo, alpha)
    cache.entries[key] = plan
    cache.misses += 1
    return plan, False


def expected_cost_uniform(variant) -> float:
    """Mean quality cost over hardness uniform on [0, 1] (quality.py:68-70)."""
    return variant.base_quality_cost + 0.5 * variant.hardness_penalty


def _single_model_row(variant, theta: float = 1.0):
    """Synthetic no-cascade row: one model serves everything (planner.py:373-384)."""
    from .profiler import CascadeRow
    return CascadeRow(light_id=variant.id, heavy_id=variant.id, theta=theta, tau=0.0,
                      r_light=1.0, r_heavy=0.0, fidelity_cost=expected_cost_uniform(variant),
                      mean_latency_s=variant.latency_s[1])


_SLACK = 1e-9


def clipper_plan(catalog, which: str, lam: float, queues=None, workers: int = DEFAULT_WORKERS,
                 t_slo: float = DEFAULT_T_SLO_S, alpha: float = DEFAULT_QUEUE_ALPHA) -> Plan:
    """Static single-model cluster (planner.py:387-421): all workers on the
    fastest ('light') or slowest ('heavy') variant at the largest batch whose
    path latency fits the deadline; flagged infeasible when demand exceeds
    that capacity.  A handful of scalar comparisons: host arithmetic."""
    if which not in ("light", "heavy"):
        raise PlannerError(f"clipper_plan: which must be light/heavy, got {which!r}")
    ordered = catalog.sorted_by_latency()
    variant = ordered[0] if which == "light" else ordered[-1]
    row = _single_model_row(variant)
    queues = queues or {}
    wait = queue_delay(queues.get(variant.id, 0.0), lam, alpha)
    fits = [b for b in catalog.batch_sizes if variant.latency_s[b] + wait <= t_slo + _SLACK]
    chosen = fits[-1] if fits else catalog.batch_sizes[0]
    infeasible = not fits or lam > workers * variant.throughput_qps[chosen] + _SLACK
    return Plan(row=row, workers={variant.id: workers}, batches={variant.id: chosen}, lam=lam,
                queues=dict(queues), fidelity_cost=row.fidelity_cost,
                path_latency_s=variant.latency_s[chosen] + wait, infeasible=infeasible,
                label=f"clipper-{which}")


def proteus_plan(catalog, lam: float, queues=None, workers: int = DEFAULT_WORKERS,
                 t_slo: float = DEFAULT_T_SLO_S, alpha: float = DEFAULT_QUEUE_ALPHA,
                 eps_latency: float = 0.1, eps_quality: float = 0.1) -> Plan:
    """Accuracy-scaling baseline (planner.py:424-440): the same device search
    over one single-model row per candidate variant."""
    from .catalog import select_candidates
    rows = [_single_model_row(v) for v in select_candidates(catalog, eps_latency, eps_quality)]
    return _solve_points(rows, catalog, [lam], queues, workers, t_slo, alpha, "proteus")[0]


def diffserve_plan(table, catalog, lam: float, queues=None, workers: int = DEFAULT_WORKERS,
                   t_slo: float = DEFAULT_T_SLO_S, alpha: float = DEFAULT_QUEUE_ALPHA,
                   light_id: str = "sd35-turbo", heavy_id: str = "sd35-large") -> Plan:
    """Fixed-pair discriminator cascade, no bypass (planner.py:482-500): the
    device search over the table's no-bypass rows of one pair."""
    max_theta = max(r.theta for r in table.rows)
    rows = [r for r in table.rows if r.light_id == light_id and r.heavy_id == heavy_id
            and r.theta == max_theta]
    if not rows:
        raise PlannerError(f"diffserve_plan: table has no rows for pair {light_id}/{heavy_id}")
    return _solve_points(rows, catalog, [lam], queues, workers, t_slo, alpha, "diffserve")[0]


PLANNER_MODES = ("online", "cache-d", "cache-dq", "clipper-light", "clipper-heavy", "proteus",
                 "diffserve")


def make_planner(mode: str, table, catalog, workers: int = DEFAULT_WORKERS,
                 t_slo: float = DEFAULT_T_SLO_S, alpha: float = DEFAULT_QUEUE_ALPHA, **kwargs):
    """(lam, queues) -> (Plan, info) callable for the simulator (planner.py:443-479):
    'online' re-solves each epoch on the device, 'cache-d'/'cache-dq' reuse
    plans keyed on binned demand (and backlog), the rest are the baselines."""
    if mode == "online":
        def fn(lam, queues):
            return solve(table, catalog, lam, queues, workers, t_slo, alpha), {}
        return fn
    if mode in ("cache-d", "cache-dq"):
        cache = PlanCache(mode=mode.split("-")[1], **kwargs)

        def fn(lam, queues):
            plan, hit = cached_solve(cache, table, catalog, lam, queues, workers, t_slo, alpha)
            return plan, {"cache_hit": hit}
        return fn
    if mode in ("clipper-light", "clipper-heavy"):
        which = mode.split("-")[1]

        def fn(lam, queues):
            return clipper_plan(catalog, which, lam, queues, workers, t_slo, alpha), {}
        return fn
    if mode == "proteus":
        def fn(lam, queues):
            return proteus_plan(catalog, lam, queues, workers, t_slo, alpha), {}
        return fn
    if mode == "diffserve":
        def fn(lam, queues):
            return diffserve_plan(table, catalog, lam, queues, workers, t_slo, alpha,
                                  **kwargs), {}
        return fn
    raise PlannerError(f"unknown planner mode {mode!r}; pick from {PLANNER_MODES}")
