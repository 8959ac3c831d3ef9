"""Generate golden fixtures from the genuine reference (cascadesim 0.1.0).

Run in the build container only (needs /root/reference; it never travels):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Everything written here is produced by the reference's own public functions:
``profile_config`` (pkg/src/cascadesim/profiler.py:107), ``pareto_prune``
(catalog.py:171), ``solve`` / ``brute_force_solve`` (planner.py:217/230) and
the acceptance-suite instance generator (pkg/tests/test_acceptance.py:122-173,
re-implemented below with the same RNG call sequence).  Records (hardness and
keyed noise, in ``stable_text_key`` order) and the per-model scores computed
from them with the reference's numpy expression (profiler.py:133-137) are
stored next to the reference's output rows, so the GPU path can be fed the
exact bytes the reference consumed.

Synthetic record sets (router-like ties, 8-model catalogs, crossing costs)
are pushed through the genuine ``profile_config`` by replacing
``router.hardness`` and ``stream_normal`` inside ``cascadesim.profiler`` with
lookups keyed by prompt text -- the method SURVEY.md §7.1(ii) verified to be
identical to an unpatched run.
"""

from __future__ import annotations

import json
import os
import random
import sys
from dataclasses import asdict

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from cascadesim import catalog as rcat  # noqa: E402
from cascadesim import planner as rplan  # noqa: E402
from cascadesim import profiler as rprof  # noqa: E402
from cascadesim import router as rrouter  # noqa: E402
from cascadesim.seeds import stable_text_key, stream_normal  # noqa: E402
from cascadesim.workload import gen_prompts  # noqa: E402


def cat_doc(cat):
    return {
        "batch_sizes": list(cat.batch_sizes),
        "calibrated": cat.calibrated,
        "variants": [{
            "id": v.id,
            "latency_s": {str(b): x for b, x in v.latency_s.items()},
            "throughput_qps": {str(b): x for b, x in v.throughput_qps.items()},
            "base_quality_cost": v.base_quality_cost,
            "hardness_penalty": v.hardness_penalty,
            "accept_params": list(v.accept_params),
        } for v in cat.variants],
    }


def table_doc(table):
    prov = asdict(table.provenance)
    prov["thresholds"] = list(prov["thresholds"])
    return {"provenance": prov, "rows": [asdict(r) for r in table.rows]}


def scores_for(pool, h, noise):
    out = {}
    for v in pool:
        a, s = v.accept_params
        out[v.id] = np.clip(1.0 / (1.0 + np.exp(-(a - s * h))) + noise, 0.0, 1.0)
    return out


def text_records(prompts, seed, sigma=0.05):
    texts = sorted(prompts, key=stable_text_key)
    lex = rrouter.load_lexicons()
    h = np.array([rrouter.hardness(t, None, lex) for t in texts])
    noise = np.array([stream_normal(seed, stable_text_key(t), "disc", sigma=sigma) for t in texts])
    return texts, h, noise


def save_records(name, pool, h, noise):
    arrays = {"h": h, "noise": noise}
    for mid, s in scores_for(pool, h, noise).items():
        arrays["score:" + mid] = s
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)


def dump(name, doc):
    with open(os.path.join(HERE, name + ".json"), "w", encoding="utf-8") as fh:
        json.dump(doc, fh, indent=0, sort_keys=True)
        fh.write("\n")


class Patched:
    """Feed synthetic (h, noise) records through the genuine profile_config."""

    def __init__(self, h_by_text, noise_by_text):
        self.h, self.noise = h_by_text, noise_by_text

    def __enter__(self):
        self.saved = (rprof.router.hardness, rprof.stream_normal)
        rprof.router.hardness = lambda t, w=None, lex=None: self.h[t]
        key_to_text = {stable_text_key(t): t for t in self.h}
        rprof.stream_normal = lambda seed, key, ch, sigma=1.0: self.noise[key_to_text[key]]
        return self

    def __exit__(self, *exc):
        rprof.router.hardness, rprof.stream_normal = self.saved


def synthetic_case(name, cat, h_values, noise_values, thresholds, eps=0.1, seed=0):
    texts = [f"synthetic query {i:07d}" for i in range(len(h_values))]
    order = sorted(range(len(texts)), key=lambda i: stable_text_key(texts[i]))
    h = np.asarray(h_values, dtype=np.float64)[order]
    noise = np.asarray(noise_values, dtype=np.float64)[order]
    sorted_texts = [texts[i] for i in order]
    with Patched(dict(zip(sorted_texts, h.tolist())), dict(zip(sorted_texts, noise.tolist()))):
        table = rprof.profile_config(cat, texts, seed=seed, eps_latency=eps,
                                     eps_quality=eps, thresholds=thresholds)
    pool = rcat.select_candidates(cat, eps, eps)
    save_records(name, pool, h, noise)
    doc = {"catalog": cat_doc(cat), "eps": eps, "seed": seed, "thresholds": list(thresholds),
           "pool": [v.id for v in pool], "table": table_doc(table)}
    dump(name, doc)
    print(f"{name}: n={len(h)} K={len(thresholds)} pool={len(pool)} rows={len(table.rows)}")
    return table


def geometric_catalog(m, l0=0.5, growth=1.45):
    """SURVEY.md §8(d) c3/c4 family: L_{k+1}=1.45 L_k, cost_{k+1}=cost_k-4/1.15^k."""
    variants, lat, cost = [], l0, 40.0
    for k in range(m):
        variants.append(rcat.make_variant(
            f"g{k:02d}", rcat.scaled_batch_profile(lat), cost, 12.0 * 0.85 ** k,
            (2.0 + 0.12 * k, 4.0)))
        lat *= growth
        cost -= 4.0 / 1.15 ** k
    return rcat.Catalog(variants=tuple(variants), calibrated=True)


# --------------------------------------------------------------------- planner

def random_instance(rng):
    """pkg/tests/test_acceptance.py:122-173 (same RNG call order)."""
    n_var = rng.choice((2, 3))
    sizes = (1,) + tuple(sorted(rng.sample((2, 4, 8), rng.randint(0, 2))))
    variants = []
    lat = rng.uniform(0.2, 1.2)
    cost = rng.uniform(32.0, 42.0)
    for k in range(n_var):
        latency = {b: lat * (1.0 + 0.25 * (b - 1)) for b in sizes}
        variants.append(rcat.make_variant(f"m{k}", latency, cost, rng.uniform(0.5, 10.0),
                                          (rng.uniform(1.2, 3.8), 4.0)))
        lat *= rng.uniform(1.8, 4.5)
        cost -= rng.uniform(1.0, 5.0)
    cat = rcat.Catalog(variants=tuple(variants), batch_sizes=sizes, calibrated=True)
    ids = [v.id for v in cat.sorted_by_latency()]
    pairs = [(a, b) for i, a in enumerate(ids) for b in ids[i + 1:]]
    rng.shuffle(pairs)
    pairs = pairs[:3]
    rows = []
    for _ in range(rng.randint(1, 20)):
        light_id, heavy_id = rng.choice(pairs)
        bypass = 1.0 if rng.random() < 0.15 else rng.uniform(0.0, 1.0)
        reroute = rng.uniform(0.0, 1.0 - bypass)
        rows.append(rprof.CascadeRow(
            light_id=light_id, heavy_id=heavy_id, theta=1.0 - bypass, tau=rng.random(),
            r_light=1.0 - bypass, r_heavy=bypass + reroute,
            fidelity_cost=rng.uniform(18.0, 40.0), mean_latency_s=rng.uniform(0.3, 8.0)))
    prov = rprof.TableProvenance(catalog_hash=cat.content_hash(), prompts_hash="synthetic",
                                 n_prompts=0, seed=0, noise_sigma=0.0, thresholds=(0.0, 1.0),
                                 eps_latency=0.1, eps_quality=0.1)
    table = rprof.CascadeTable(rows=tuple(rows), provenance=prov)
    budget = rng.randint(1, 8)
    pick = rng.random()
    if pick < 0.1:
        lam = 0.0
    elif pick < 0.5:
        lam = rng.uniform(0.05, 2.0)
    else:
        lam = rng.uniform(2.0, 30.0)
    t_slo = rng.uniform(1.0, 10.0) if rng.random() < 0.5 else rng.uniform(10.0, 120.0)
    queues = {}
    if rng.random() < 0.5:
        for v in variants:
            if rng.random() < 0.5:
                queues[v.id] = rng.uniform(0.0, 40.0)
    return cat, table, lam, budget, t_slo, queues


def plan_doc(plan, table):
    if plan is None:
        return None
    idx = next(i for i, r in enumerate(table.rows) if r is plan.row)
    return {"row_index": idx, "workers": plan.workers, "batches": {k: int(v) for k, v in plan.batches.items()},
            "lam": plan.lam, "queues": plan.queues, "fidelity_cost": plan.fidelity_cost,
            "path_latency_s": plan.path_latency_s, "infeasible": plan.infeasible,
            "label": plan.label}


def try_solve(fn, *a, **kw):
    try:
        return fn(*a, **kw), None
    except rplan.PlannerError as exc:
        return None, str(exc)


def planner_cases():
    rng = random.Random(20260819)
    cases = []
    for _ in range(200):
        cat, table, lam, budget, t_slo, queues = random_instance(rng)
        fast, ferr = try_solve(rplan.solve, table, cat, lam, queues=queues, workers=budget, t_slo=t_slo)
        slow, serr = try_solve(rplan.brute_force_solve, table, cat, lam, queues=queues,
                               workers=budget, t_slo=t_slo)
        cases.append({"catalog": cat_doc(cat), "rows": [asdict(r) for r in table.rows],
                      "lam": lam, "workers": budget, "t_slo": t_slo, "alpha": 1.5,
                      "queues": queues, "solve": plan_doc(fast, table), "solve_error": ferr,
                      "brute": plan_doc(slow, table), "brute_error": serr})
    dump("planner_random200", {"cases": cases})
    print("planner_random200: 200 instances")


def planner_sweep(table, cat, name):
    pts = []
    rng = random.Random(7)
    for lam in (0.0, 0.4, 1.0, 3.0, 5.0, 8.5, 17.0, 23.0, 42.0, 61.0, 86.0, 140.0):
        for workers in (3, 8, 16):
            for t_slo in (10.0, 30.0, 60.0, 90.0):
                queues = {}
                if rng.random() < 0.4:
                    for v in cat.variants:
                        if rng.random() < 0.5:
                            queues[v.id] = rng.uniform(0.0, 40.0)
                plan, err = try_solve(rplan.solve, table, cat, lam, queues=queues,
                                      workers=workers, t_slo=t_slo)
                pts.append({"lam": lam, "workers": workers, "t_slo": t_slo, "alpha": 1.5,
                            "queues": queues, "solve": plan_doc(plan, table), "solve_error": err})
    dump(name, {"catalog": cat_doc(cat), "table": table_doc(table), "points": pts})
    print(f"{name}: {len(pts)} points over {len(table.rows)} rows")


def pareto_kats():
    cases = [[[1.0, 5.0], [2.0, 4.0], [1.5, 6.0]],
             [[1.0, 5.0], [2.0, 4.0], [3.0, 3.0]],
             [[1.0, 5.0], [1.0, 5.0]],
             [[2.0, 1.0], [2.0, 1.0], [1.0, 3.0], [1.0, 2.0], [3.0, 0.5], [0.0, 0.0], [-0.0, 0.0]]]
    rng = random.Random(11)
    for n in (1, 2, 5, 40, 300, 5000):
        cases.append([[rng.choice((0.5, 1.0, rng.uniform(0.1, 100))),
                       rng.choice((2.0, 3.0, rng.uniform(0.1, 100)))] for _ in range(n)])
    out = []
    for c in cases:
        tagged = [(x[0], x[1], i) for i, x in enumerate(c)]
        kept = rcat.pareto_prune(tagged, key=lambda r: (r[0], r[1]))
        out.append({"rows": c, "kept": [r[2] for r in kept]})
    dump("pareto_kats", {"cases": out})
    print(f"pareto_kats: {len(out)} cases")


def main():
    cat = rcat.default_catalog()

    # conftest fixture: 160 prompts, seed 42, default grid (pkg/tests/conftest.py:8-21)
    prompts = gen_prompts(160, seed=42)
    texts, h, noise = text_records(prompts, 42)
    table = rprof.profile_config(cat, prompts, seed=42)
    pool = rcat.select_candidates(cat, 0.1, 0.1)
    save_records("conftest160", pool, h, noise)
    variants = {}
    for label, thr in (("default", rprof.THRESHOLD_GRID), ("bypass01", (0.0, 1.0)),
                       ("unsorted", (0.5, 0.1, 0.9, 0.3, 0.7)),
                       ("duplicates", (0.2, 0.6, 0.2, 1.0, 0.6)),
                       ("negzero", (-0.0, 0.25, 0.0, 0.75)),
                       ("dense33", tuple(i / 32 for i in range(33)))):
        t = rprof.profile_config(cat, prompts, seed=42, thresholds=thr)
        variants[label] = {"thresholds": list(thr), "table": table_doc(t)}
    dump("conftest160", {"catalog": cat_doc(cat), "seed": 42, "eps": 0.1,
                         "pool": [v.id for v in pool],
                         "prompts_hash": rprof.prompts_hash(texts),
                         "catalog_hash": cat.content_hash(), "variants": variants})
    print(f"conftest160: rows={len(table.rows)}")
    planner_sweep(table, cat, "planner_conftest")

    # c1: (sd35-turbo, sd35-large), gen_prompts(5000, seed=0), seed 0, K=64
    c1cat = rcat.Catalog(variants=(cat.by_id("sd35-turbo"), cat.by_id("sd35-large")), calibrated=True)
    prompts = gen_prompts(5000, seed=0)
    texts, h, noise = text_records(prompts, 0)
    thr = tuple(i / 63 for i in range(64))
    t1 = rprof.profile_config(c1cat, prompts, seed=0, thresholds=thr)
    save_records("c1", rcat.select_candidates(c1cat, 0.1, 0.1), h, noise)
    dump("c1", {"catalog": cat_doc(c1cat), "seed": 0, "eps": 0.1, "thresholds": list(thr),
                "prompts_hash": rprof.prompts_hash(texts), "table": table_doc(t1)})
    print(f"c1: rows={len(t1.rows)}")

    # router-like ties: resample real hardness values (SURVEY.md §8d last paragraph)
    rng = np.random.default_rng(20261017)
    _, real_h, _ = text_records(gen_prompts(512, seed=5), 5)
    synthetic_case("ties3000", cat, rng.choice(real_h, 3000), rng.normal(0.0, 0.05, 3000),
                   tuple(i / 23 for i in range(24)))
    # 8-model geometric catalog, eps 1e-3 so all 8 survive
    synthetic_case("geo8", geometric_catalog(8), rng.uniform(0.05, 0.9, 2000),
                   rng.normal(0.0, 0.05, 2000), tuple(i / 15 for i in range(16)), eps=1e-3)
    # costs that cross inside [0, 1] (at h=0.25): heavy is worse on hard prompts
    cross = rcat.Catalog(variants=(
        rcat.make_variant("x-light", rcat.scaled_batch_profile(1.0), 27.0, 2.0, (0.0, 0.5)),
        rcat.make_variant("x-heavy", rcat.scaled_batch_profile(4.0), 25.0, 10.0, (3.0, 4.0))),
        calibrated=False)
    synthetic_case("cross1500", cross, rng.choice(np.round(rng.uniform(0, 0.45, 40), 3), 1500),
                   rng.normal(0.0, 0.2, 1500), tuple(i / 19 for i in range(20)))

    planner_cases()
    pareto_kats()


if __name__ == "__main__":
    main()
