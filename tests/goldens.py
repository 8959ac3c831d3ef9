"""Loaders for the golden fixtures written by tests/golden/make_golden.py."""

from __future__ import annotations

import json
import os
from types import SimpleNamespace

import numpy as np

from paper_2509_00642_b200.catalog import Catalog, ModelVariant

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_json(name):
    with open(os.path.join(GOLDEN, name + ".json"), encoding="utf-8") as fh:
        return json.load(fh)


def load_npz(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def catalog_from_doc(doc):
    variants = tuple(ModelVariant(
        id=v["id"],
        latency_s={int(b): x for b, x in v["latency_s"].items()},
        throughput_qps={int(b): x for b, x in v["throughput_qps"].items()},
        base_quality_cost=v["base_quality_cost"],
        hardness_penalty=v["hardness_penalty"],
        accept_params=tuple(v["accept_params"])) for v in doc["variants"])
    return Catalog(variants=variants, batch_sizes=tuple(doc["batch_sizes"]),
                   calibrated=doc["calibrated"])


def row_tuples(table_doc):
    return [(r["light_id"], r["heavy_id"], r["theta"], r["tau"], r["r_light"], r["r_heavy"],
             r["fidelity_cost"], r["mean_latency_s"]) for r in table_doc["rows"]]


def rows_ns(rows):
    return [SimpleNamespace(**r) for r in rows]


def scores_of(rec):
    return {k.split(":", 1)[1]: v for k, v in rec.items() if k.startswith("score:")}


PROFILE_CASES = ("ties3000", "geo8", "cross1500")


def frontier_cases():
    return {d["name"]: d for d in load_json("frontier")}


_TEXT = None


def load_text():
    """tests/golden/text.json.gz (generator: tests/golden/make_golden_text.py)."""
    global _TEXT
    if _TEXT is None:
        import gzip
        with gzip.open(os.path.join(GOLDEN, "text.json.gz"), "rt", encoding="utf-8") as fh:
            _TEXT = json.load(fh)
    return _TEXT

