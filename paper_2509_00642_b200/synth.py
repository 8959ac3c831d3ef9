"""Synthetic workloads of BASELINE.json's configs.

c1  2 models (sd35-turbo, sd35-large), 5k queries, 64x64 grid
c2  4 models (default catalog), 1M queries, 256x256 grid, planner W=8
c3  8-model geometric catalog (eps 1e-3), 10M queries, 512x512
c4  16-model geometric catalog (eps 1e-6), 10M queries, 1024x1024
c5  1k (demand, SLO) points x the c2 table x all worker splits of 8

Records: numpy default_rng(20261017); h ~ U(0.05, 0.9) (gen_prompts' default
range, workload.py:312), noise ~ N(0, 0.05); scores with the reference's
expression (profiler.py:137); thresholds i / (K - 1).  The data is synthetic
(there is no network for real prompt sets) and labelled so in bench output.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .catalog import Catalog, default_catalog, make_variant, scaled_batch_profile, select_candidates
from .profiler import light_scores

SEED = 20261017


def geometric_catalog(m: int, l0: float = 0.5, growth: float = 1.45) -> Catalog:
    """L_{k+1} = 1.45 L_k, cost_{k+1} = cost_k - 4/1.15^k, pen = 12 * 0.85^k,
    accept = (2.0 + 0.12 k, 4.0), beta 0.25, batches (1, 2, 4, 8, 16)."""
    variants, lat, cost = [], l0, 40.0
    for k in range(m):
        variants.append(make_variant(f"g{k:02d}", scaled_batch_profile(lat), cost,
                                     12.0 * 0.85 ** k, (2.0 + 0.12 * k, 4.0)))
        lat *= growth
        cost -= 4.0 / 1.15 ** k
    return Catalog(variants=tuple(variants), calibrated=True)


@dataclass(frozen=True)
class Config:
    name: str
    n_models: int
    n_queries: int
    k: int
    eps: float
    workers: int = 8

    @property
    def thresholds(self):
        return tuple(i / (self.k - 1) for i in range(self.k))

    def catalog(self) -> Catalog:
        if self.name == "c1":
            cat = default_catalog()
            return Catalog(variants=(cat.by_id("sd35-turbo"), cat.by_id("sd35-large")),
                           calibrated=True)
        if self.n_models == 4:
            return default_catalog()
        return geometric_catalog(self.n_models)

    def pool(self):
        pool = select_candidates(self.catalog(), self.eps, self.eps)
        assert len(pool) == self.n_models, (self.name, len(pool))
        return pool

    @property
    def n_pairs(self) -> int:
        return self.n_models * (self.n_models - 1) // 2

    @property
    def cells(self) -> int:
        return self.n_pairs * self.k * self.k


CONFIGS = {
    "c1": Config("c1", 2, 5_000, 64, 0.1),
    "c2": Config("c2", 4, 1_000_000, 256, 0.1),
    "c3": Config("c3", 8, 10_000_000, 512, 1e-3),
    "c4": Config("c4", 16, 10_000_000, 1024, 1e-6),
}


def records(cfg: Config, seed: int = SEED):
    """(pool, h float64[N], noise float64[N], scores float64[M-1, N])."""
    rng = np.random.default_rng(seed)
    h = rng.uniform(0.05, 0.9, cfg.n_queries)
    noise = rng.normal(0.0, 0.05, cfg.n_queries)
    pool = cfg.pool()
    return pool, h, noise, light_scores(pool, h, noise)


def replan_points(n_points: int = 1000, seed: int = SEED, backlog: bool = False, models=()):
    """c5: 250 demand values x T_slo in {15, 30, 60, 90}."""
    lams, slos = [], []
    for i in range(n_points // 4):
        for t in (15.0, 30.0, 60.0, 90.0):
            lams.append(0.1 * (i + 1))
            slos.append(t)
    queues = [{} for _ in lams]
    if backlog:
        rng = np.random.default_rng(seed)
        queues = [{m: float(rng.uniform(0.0, 40.0)) for m in models} for _ in lams]
    return lams, slos, queues
