"""Model catalog types, candidate selection and the generic Pareto prune.

Host-side mirror of the parts of ``cascadesim.catalog`` the profiling path
consumes (reference: pkg/src/cascadesim/catalog.py).  The value types are
field-compatible with the reference's, and every function accepts either our
objects or the reference's (duck typing on ``id``, ``latency_s``,
``throughput_qps``, ``base_quality_cost``, ``hardness_penalty``,
``accept_params``), so a cascadesim user can hand its own ``Catalog`` to
``profile_config`` / ``solve`` unchanged.

``select_candidates`` (catalog.py:199-271) stays on the host: it is O(M^2)
over at most a few dozen variants.  ``pareto_prune``
(catalog.py:171-192) runs on the GPU (``hadis_pareto_prune`` in the C ABI).
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass

DEFAULT_BATCH_SIZES = (1, 2, 4, 8, 16)
DEFAULT_BATCH_BETA = 0.25
_REL_TOL = 1e-9


class CatalogError(ValueError):
    """Catalog validation failure (same type name/role as the reference's)."""


@dataclass(frozen=True)
class ModelVariant:
    """One serveable variant (catalog.py:28-45)."""

    id: str
    latency_s: dict
    throughput_qps: dict
    base_quality_cost: float
    hardness_penalty: float
    accept_params: tuple

    def batch_sizes(self) -> tuple:
        return tuple(sorted(self.latency_s))


@dataclass(frozen=True)
class Catalog:
    """A pool of variants over one batch-size set (catalog.py:48-87)."""

    variants: tuple
    batch_sizes: tuple = DEFAULT_BATCH_SIZES
    calibrated: bool = False

    def __post_init__(self) -> None:
        check_catalog(self)

    def by_id(self, variant_id: str):
        for v in self.variants:
            if v.id == variant_id:
                return v
        raise CatalogError(f"unknown-variant: {variant_id!r}")

    def ids(self) -> tuple:
        return tuple(v.id for v in self.variants)

    def sorted_by_latency(self) -> tuple:
        return tuple(sorted(self.variants, key=_light_first))

    def content_hash(self) -> str:
        return catalog_hash(self)


def _light_first(v):
    return (v.latency_s[1], v.id)


def catalog_hash(cat) -> str:
    """16-hex provenance hash of the calibrated numbers (catalog.py:70-87).

    Works on any catalog-shaped object so tables profiled from a reference
    ``Catalog`` carry the same hash the reference would write."""
    doc = {
        "batch_sizes": list(cat.batch_sizes),
        "calibrated": cat.calibrated,
        "variants": [{
            "id": v.id,
            "latency_s": {str(b): repr(v.latency_s[b]) for b in sorted(v.latency_s)},
            "base_quality_cost": repr(v.base_quality_cost),
            "hardness_penalty": repr(v.hardness_penalty),
            "accept_params": [repr(v.accept_params[0]), repr(v.accept_params[1])],
        } for v in cat.variants],
    }
    return hashlib.sha256(json.dumps(doc, sort_keys=True).encode("utf-8")).hexdigest()[:16]


def scaled_batch_profile(latency_b1, batch_sizes=DEFAULT_BATCH_SIZES, beta=DEFAULT_BATCH_BETA):
    """L(b) = L(1) * (1 + beta * (b - 1)) (catalog.py:90-100)."""
    if latency_b1 <= 0:
        raise CatalogError("latency_b1 must be positive")
    if beta <= 0:
        raise CatalogError("beta must be positive")
    return {b: latency_b1 * (1.0 + beta * (b - 1)) for b in batch_sizes}


def make_variant(variant_id, latency_s, base_quality_cost, hardness_penalty, accept_params):
    """Variant with throughput_qps = b / L(b) (catalog.py:103-119)."""
    lat = dict(sorted(latency_s.items()))
    return ModelVariant(id=variant_id, latency_s=lat,
                        throughput_qps={b: b / l for b, l in lat.items()},
                        base_quality_cost=base_quality_cost,
                        hardness_penalty=hardness_penalty,
                        accept_params=accept_params)


def batch_latency(variant, batch: int) -> float:
    """Exact latency lookup; an unprofiled batch size is an error (catalog.py:163-168)."""
    try:
        return variant.latency_s[batch]
    except KeyError:
        raise CatalogError(f"batch-not-profiled: {variant.id} b={batch}") from None


def load_catalog(path: str) -> Catalog:
    """Catalog from the reference's YAML file format (catalog.py:289-331): same
    keys (batch_sizes, batch_scaling_beta, calibrated, variants[] with id,
    base_quality_cost, hardness_penalty, accept_params and latency_s table or
    latency_b1) and the same first-violation messages."""
    import yaml
    with open(path, "r", encoding="utf-8") as fh:
        raw = yaml.safe_load(fh)
    if not isinstance(raw, dict):
        raise CatalogError("catalog file: top level must be a mapping")
    batch_sizes = tuple(raw.get("batch_sizes", DEFAULT_BATCH_SIZES))
    beta = float(raw.get("batch_scaling_beta", DEFAULT_BATCH_BETA))
    entries = raw.get("variants")
    if not isinstance(entries, list) or not entries:
        raise CatalogError("variants: must be a non-empty list")
    variants = []
    for i, entry in enumerate(entries):
        where = f"variants[{i}]"
        if not isinstance(entry, dict):
            raise CatalogError(f"{where}: must be a mapping")
        try:
            fields = (entry["id"], float(entry["base_quality_cost"]),
                      float(entry["hardness_penalty"]),
                      tuple(float(x) for x in entry["accept_params"]))
        except KeyError as exc:
            raise CatalogError(f"{where}.{exc.args[0]}: missing") from None
        vid, cost, penalty, accept = fields
        if len(accept) != 2:
            raise CatalogError(f"{where}.accept_params: expected [a, s]")
        lat = entry.get("latency_s")
        if isinstance(lat, dict):
            latency = {int(b): float(x) for b, x in lat.items()}
            missing = [b for b in batch_sizes if b not in latency]
            if tuple(sorted(latency)) != batch_sizes and missing:
                raise CatalogError(f"{where}.latency_s: missing batch sizes {missing}")
        elif "latency_b1" in entry:
            latency = scaled_batch_profile(float(entry["latency_b1"]), batch_sizes, beta)
        else:
            raise CatalogError(f"{where}.latency_s: give a table or latency_b1")
        variants.append(make_variant(vid, latency, cost, penalty, (accept[0], accept[1])))
    return Catalog(variants=tuple(variants), batch_sizes=batch_sizes,
                   calibrated=bool(raw.get("calibrated", False)))


def check_catalog(cat) -> None:
    """Validation rules and messages of catalog.py:122-160."""
    if not cat.variants:
        raise CatalogError("variants: empty pool")
    if list(cat.batch_sizes) != sorted(set(cat.batch_sizes)):
        raise CatalogError("batch_sizes: must be strictly increasing")
    seen = set()
    for i, v in enumerate(cat.variants):
        where = f"variants[{i}] ({v.id})"
        if v.id in seen:
            raise CatalogError(f"{where}.id: duplicate")
        seen.add(v.id)
        if tuple(sorted(v.latency_s)) != tuple(cat.batch_sizes):
            raise CatalogError(f"{where}.latency_s: batch sizes {sorted(v.latency_s)} "
                               f"do not match catalog set {list(cat.batch_sizes)}")
        prev = 0.0
        for b in cat.batch_sizes:
            lat = v.latency_s[b]
            if lat <= prev:
                raise CatalogError(f"{where}.latency_s[{b}]: not strictly increasing")
            prev = lat
            mu = v.throughput_qps.get(b)
            if mu is None:
                raise CatalogError(f"{where}.throughput_qps[{b}]: missing")
            if abs(mu * lat - b) > _REL_TOL * b:
                raise CatalogError(f"{where}.throughput_qps[{b}]: {mu!r} is not b/latency")
        if v.base_quality_cost <= 0:
            raise CatalogError(f"{where}.base_quality_cost: must be positive")
        if v.hardness_penalty < 0:
            raise CatalogError(f"{where}.hardness_penalty: must be non-negative")
        if v.accept_params[1] <= 0:
            raise CatalogError(f"{where}.accept_params: slope must be positive")
    if cat.calibrated:
        order = sorted(cat.variants, key=_light_first)
        for lighter, heavier in zip(order, order[1:]):
            if not heavier.base_quality_cost < lighter.base_quality_cost:
                raise CatalogError(
                    f"variants ({heavier.id}): calibrated catalogs need strictly "
                    f"lower quality cost than the faster {lighter.id}")


def default_catalog() -> Catalog:
    """The shipped four-variant diffusion catalog (catalog.py:274-286)."""
    table = (("sdxl-lightning", 0.5, 36.0, 12.0, (2.0, 4.0)),
             ("sd35-turbo", 1.3, 31.0, 8.0, (2.6, 4.0)),
             ("sd35-medium", 13.0, 26.0, 5.0, (3.2, 4.0)),
             ("sd35-large", 27.0, 23.0, 3.0, (3.6, 4.0)))
    return Catalog(variants=tuple(make_variant(name, scaled_batch_profile(l1), cost, pen, acc)
                                  for name, l1, cost, pen, acc in table),
                   calibrated=True)


def _close(a, b, eps):
    return abs(a - b) <= eps * max(abs(a), abs(b))


def select_candidates(catalog, eps_latency: float, eps_quality: float) -> list:
    """Adjacency / dominance / redundancy pruning (catalog.py:199-271).

    Operates on the (b=1 latency, base quality cost) point of each variant and
    returns survivors light to heavy, id breaking latency ties."""
    for name, eps in (("eps_latency", eps_latency), ("eps_quality", eps_quality)):
        if not (0.0 < eps < 0.5):
            raise CatalogError(f"{name}: must lie in (0, 0.5)")
    pool = list(catalog.variants)
    if not pool:
        raise CatalogError("variants: empty pool")
    pt = {id(v): (v.latency_s[1], v.base_quality_cost) for v in pool}

    # variants that are the unique minimum on either axis can never be merged away
    keep_always = set()
    for axis in (0, 1):
        values = sorted(p[axis] for p in pt.values())
        if values.count(values[0]) == 1:
            keep_always.add(min(pool, key=lambda v: pt[id(v)][axis]).id)

    groups = []
    for v in pool:
        lv, qv = pt[id(v)]
        home = next((g for g in groups
                     if all(_close(lv, pt[id(w)][0], eps_latency)
                            and _close(qv, pt[id(w)][1], eps_quality) for w in g)), None)
        if home is None:
            groups.append([v])
        else:
            home.append(v)
    alive = []
    for g in groups:
        rep = min(g, key=lambda v: v.id)
        alive.extend(v for v in g if v is rep or v.id in keep_always)
    position = {id(v): i for i, v in enumerate(pool)}
    alive.sort(key=lambda v: position[id(v)])

    def beats(a, b):
        (la, qa), (lb, qb) = pt[id(a)], pt[id(b)]
        return (la <= lb and qa < qb) or (la < lb and qa <= qb)

    alive = [v for v in alive if not any(beats(o, v) for o in alive if o is not v)]

    costs = [pt[id(v)][1] for v in alive]
    span = max(costs) - min(costs)
    if span > 0:
        pruned = True
        while pruned and len(alive) > 2:
            pruned = False
            ordered = sorted(alive, key=_light_first)
            for left, mid, right in zip(ordered, ordered[1:], ordered[2:]):
                (l0, q0), (lm, qm), (l1, q1) = pt[id(left)], pt[id(mid)], pt[id(right)]
                if abs(qm - (q0 + (q1 - q0) * (lm - l0) / (l1 - l0))) <= eps_quality * span:
                    alive.remove(mid)
                    pruned = True
                    break
    return sorted(alive, key=_light_first)


def pareto_prune(rows, key=None):
    """Latency/quality Pareto frontier of tagged rows (catalog.py:171-192).

    Same contract as the reference: ``key(row) -> (latency, quality)``
    (default: the row itself is the pair); a row survives iff its quality is
    strictly below that of every row sorted before it by (latency, quality,
    original index); the result is in that sorted order.  The sort and the
    strict prefix-min run on the GPU (``hadis_pareto_prune``)."""
    rows = list(rows)
    if key is None:
        key = lambda r: (r[0], r[1])  # noqa: E731
    if not rows:
        return []
    from . import _lib
    lat, qual = zip(*(key(r)[:2] for r in rows))
    kept = _lib.pareto_prune_indices(lat, qual)
    return [rows[i] for i in kept]
