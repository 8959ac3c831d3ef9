"""Restatement of the reference acceptance suite's randomized solver instance
generator (pkg/tests/test_acceptance.py:122-173, same RNG call order) over
this package's types.  Test infrastructure."""

from paper_2509_00642_b200.catalog import Catalog, catalog_hash, make_variant
from paper_2509_00642_b200.profiler import CascadeRow, CascadeTable, TableProvenance


def random_instance(rng):
    n_var = rng.choice((2, 3))
    sizes = (1,) + tuple(sorted(rng.sample((2, 4, 8), rng.randint(0, 2))))
    variants = []
    lat = rng.uniform(0.2, 1.2)
    cost = rng.uniform(32.0, 42.0)
    for k in range(n_var):
        latency = {b: lat * (1.0 + 0.25 * (b - 1)) for b in sizes}
        variants.append(make_variant(f"m{k}", latency, cost, rng.uniform(0.5, 10.0),
                                     (rng.uniform(1.2, 3.8), 4.0)))
        lat *= rng.uniform(1.8, 4.5)
        cost -= rng.uniform(1.0, 5.0)
    cat = Catalog(variants=tuple(variants), batch_sizes=sizes, calibrated=True)
    ids = [v.id for v in cat.sorted_by_latency()]
    pairs = [(a, b) for i, a in enumerate(ids) for b in ids[i + 1:]]
    rng.shuffle(pairs)
    pairs = pairs[:3]
    rows = []
    for _ in range(rng.randint(1, 20)):
        light_id, heavy_id = rng.choice(pairs)
        bypass = 1.0 if rng.random() < 0.15 else rng.uniform(0.0, 1.0)
        reroute = rng.uniform(0.0, 1.0 - bypass)
        rows.append(CascadeRow(light_id=light_id, heavy_id=heavy_id, theta=1.0 - bypass,
                               tau=rng.random(), r_light=1.0 - bypass,
                               r_heavy=bypass + reroute,
                               fidelity_cost=rng.uniform(18.0, 40.0),
                               mean_latency_s=rng.uniform(0.3, 8.0)))
    prov = TableProvenance(catalog_hash=catalog_hash(cat), prompts_hash="synthetic",
                           n_prompts=0, seed=0, noise_sigma=0.0, thresholds=(0.0, 1.0),
                           eps_latency=0.1, eps_quality=0.1)
    table = CascadeTable(rows=tuple(rows), provenance=prov)
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
