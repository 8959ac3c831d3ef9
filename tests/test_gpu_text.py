"""GPU parity of the text -> record step and of the
text-level drop-in ``profile_config`` against the genuine reference's outputs
(tests/golden/text.json.gz, c1/conftest160 goldens, router goldens).

Nothing here needs the reference installed: the prompt texts and every
expected value are committed fixtures."""

import os
import tempfile
from dataclasses import asdict

import numpy as np
import pytest

from oracle import text as ot
from paper_2509_00642_b200 import load_table, profile_config, save_table
from paper_2509_00642_b200 import router as gr
from paper_2509_00642_b200 import text as gt
from paper_2509_00642_b200.catalog import default_catalog
from tests.goldens import catalog_from_doc, load_json, load_npz, load_text, row_tuples

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    return load_text()


def tuples(table):
    return [(r.light_id, r.heavy_id, r.theta, r.tau, r.r_light, r.r_heavy, r.fidelity_cost,
             r.mean_latency_s) for r in table.rows]


def prov_doc(table):
    d = asdict(table.provenance)
    d["thresholds"] = list(d["thresholds"])
    return d


@pytest.mark.parametrize("case", ["edge", "random3000"])
def test_features_and_hardness_bitexact(gpu_device, gold, case):
    c = gold["cases"][case]
    raw, feat, h = gt.text_features(c["texts"])
    _, _, h_alt = gt.text_features(c["texts"], gold["misc"]["alt_weights"])
    for i, row in enumerate(c["rows"]):
        assert raw[i].tolist() == row["raw"], (i, c["texts"][i])
        assert feat[i].tolist() == row["features"], (i, c["texts"][i])
        assert h[i] == row["h"] and h_alt[i] == row["h_alt"], (i, c["texts"][i])
    keys = gt.text_keys(c["texts"])
    assert [str(k) for k in keys] == [r["key"] for r in c["rows"]]


@pytest.mark.parametrize("case", ["edge", "random3000"])
def test_text_records_order_and_noise(gpu_device, gold, case):
    c = gold["cases"][case]
    texts = c["texts"]
    for k, (seed, sigma) in enumerate(gold["misc"]["noise_keys"]):
        rec = gt.text_records(texts, seed, sigma)
        want_order = sorted(range(len(texts)), key=lambda i: ot.stable_text_key(texts[i]))
        assert rec.order.tolist() == want_order
        assert [str(int(x)) for x in rec.keys] == [c["rows"][i]["key"] for i in want_order]
        assert rec.h.tolist() == [c["rows"][i]["h"] for i in want_order]
        assert rec.noise.tolist() == [c["rows"][i]["noise"][k] for i in want_order], (seed, sigma)


@pytest.mark.parametrize("name,seed", [("conftest160", 42), ("c1", 0)])
def test_records_equal_reference_records(gpu_device, gold, name, seed):
    rec = gt.text_records(gold["corpora"][name], seed, 0.05)
    z = load_npz(name)
    assert np.array_equal(rec.h, z["h"]) and np.array_equal(rec.noise, z["noise"])


@pytest.mark.parametrize("variant", ["default", "bypass01", "unsorted", "duplicates", "negzero",
                                     "dense33"])
def test_profile_config_conftest160_equals_reference(gpu_device, gold, variant):
    doc = load_json("conftest160")
    cat = catalog_from_doc(doc["catalog"])
    case = doc["variants"][variant]
    table = profile_config(cat, gold["corpora"]["conftest160"], seed=42,
                           thresholds=case["thresholds"])
    assert tuples(table) == row_tuples(case["table"])
    assert prov_doc(table) == case["table"]["provenance"]


def test_profile_config_c1_equals_reference(gpu_device, gold):
    doc = load_json("c1")
    cat = catalog_from_doc(doc["catalog"])
    prompts = list(reversed(gold["corpora"]["c1"]))          # order must not matter
    table = profile_config(cat, prompts, seed=0, thresholds=doc["thresholds"])
    assert tuples(table) == row_tuples(doc["table"])
    assert prov_doc(table) == doc["table"]["provenance"]


def test_profile_config_edge_texts_equal_reference(gpu_device, gold):
    texts = gold["cases"]["edge"]["texts"] + gold["cases"]["random3000"]["texts"]
    cat = default_catalog()
    t1 = profile_config(cat, texts, seed=3, thresholds=tuple(i / 20 for i in range(21)))
    want = gold["tables"]["edge_random"]
    assert tuples(t1) == row_tuples(want) and prov_doc(t1) == want["provenance"]
    t2 = profile_config(cat, texts, seed=-8, noise_sigma=0.2,
                        weights=gold["misc"]["alt_weights"], thresholds=(0.0, 0.3, 0.3, 0.9, 0.1))
    want = gold["tables"]["edge_random_alt"]
    assert tuples(t2) == row_tuples(want) and prov_doc(t2) == want["provenance"]


def test_save_table_bytes_equal_reference(gpu_device, gold):
    cat = default_catalog()
    table = profile_config(cat, gold["corpora"]["conftest160"], seed=42)
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "t.json")
        save_table(table, path)
        with open(path, encoding="utf-8") as fh:
            assert fh.read() == gold["misc"]["save_table_conftest160"]
        back = load_table(path, catalog=cat)
        assert back == table


def test_router_dropins(gpu_device, gold):
    row = gold["cases"]["edge"]["rows"][3]
    t = gold["cases"]["edge"]["texts"][3]
    assert list(gr.raw_features(t).values()) == row["raw"]
    assert list(gr.features(t)) == row["features"]
    assert gr.hardness(t) == row["h"]
    assert gr.hardness(t, gold["misc"]["alt_weights"]) == row["h_alt"]
    with pytest.raises(gr.RouterError, match="must sum to 1"):
        gr.hardness(t, [0.5] * 8)
    hs = gr.hardness_many(gold["cases"]["random3000"]["texts"])
    assert hs.tolist() == [r["h"] for r in gold["cases"]["random3000"]["rows"]]


@pytest.mark.parametrize("name", ["separable80", "noisy600", "noisy3000"])
def test_tune_weights_on_text_equals_reference(gpu_device, gold, name):
    corpus = [(t, lbl) for t, lbl in gold["corpora"][name]]
    want = next(d for d in load_json("router") if d["name"] == name)
    weights, threshold, acc = gr.tune_weights(corpus)
    assert list(weights) == want["weights"]
    assert threshold == want["threshold"] and acc == want["acc"]
    _, feat, _ = gt.text_features([t for t, _ in corpus])
    assert np.array_equal(feat, load_npz("router")[name + ":features"])
