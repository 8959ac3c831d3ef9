"""Drop-in table contract on the host (SURVEY §8 rows a6 / f2 / b): the
reference's table file (bytes written by its save_table), load_table's
provenance gate and error messages, prompts_hash / stable_text_key values,
and the columnar CascadeRows view behaving as the reference's row tuple."""

import json
import os

import numpy as np
import pytest

from paper_2509_00642_b200 import load_table, save_table
from paper_2509_00642_b200.catalog import Catalog, catalog_hash, default_catalog
from paper_2509_00642_b200.profiler import (CascadeRow, CascadeRows, CascadeTable, ProfileError,
                                            prompts_hash, stable_text_key)
from tests.goldens import load_text


@pytest.fixture(scope="module")
def gold():
    return load_text()


def _write(tmp_path, text):
    path = str(tmp_path / "table.json")
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(text)
    return path


def test_reference_table_file_round_trips_byte_for_byte(tmp_path, gold):
    ref_text = gold["misc"]["save_table_conftest160"]
    table = load_table(_write(tmp_path, ref_text), catalog=default_catalog())
    out = str(tmp_path / "again.json")
    save_table(table, out)
    with open(out, encoding="utf-8") as fh:
        assert fh.read() == ref_text
    assert isinstance(table.rows, tuple) and all(isinstance(r, CascadeRow) for r in table.rows)
    assert table.provenance.catalog_hash == gold["misc"]["catalog_hash_default"]
    assert table.provenance.prompts_hash == gold["misc"]["prompts_hash"]["conftest160"]


def test_provenance_gate_and_malformed_messages(tmp_path, gold):
    path = _write(tmp_path, gold["misc"]["save_table_conftest160"])
    cat = default_catalog()
    other = Catalog(variants=cat.variants[:3], calibrated=True)
    with pytest.raises(ProfileError) as exc:
        load_table(path, catalog=other)
    assert str(exc.value) == gold["misc"]["load_errors"]["mismatch"]
    table = load_table(path, catalog=other, override_provenance=True)
    assert len(table.rows) > 0
    bad = _write(tmp_path, json.dumps({"rows": []}))
    with pytest.raises(ProfileError) as exc:
        load_table(bad)
    assert str(exc.value) == gold["misc"]["load_errors"]["malformed"]


def test_hashes_equal_reference_values(gold):
    assert catalog_hash(default_catalog()) == gold["misc"]["catalog_hash_default"]
    for name, texts in gold["corpora"].items():
        texts = [t if isinstance(t, str) else t[0] for t in texts]
        assert prompts_hash(texts) == gold["misc"]["prompts_hash"][name]
    for text, row in zip(gold["cases"]["random3000"]["texts"],
                         gold["cases"]["random3000"]["rows"]):
        assert str(stable_text_key(text)) == row["key"]


def _columnar():
    rng = np.random.default_rng(3)
    n = 1000
    ids = [("a", "b"), ("a", "c"), ("b", "c")]
    thr = tuple(i / 9 for i in range(10))
    pair = np.sort(rng.integers(0, 3, n)).astype(np.int32)
    th = rng.integers(0, 10, n).astype(np.int32)
    ta = rng.integers(0, 10, n).astype(np.int32)
    vals = [rng.random(n) for _ in range(4)]
    rows = CascadeRows(ids, pair, th, ta, *vals, thr)
    want = tuple(CascadeRow(light_id=ids[p][0], heavy_id=ids[p][1], theta=thr[a], tau=thr[b],
                            r_light=x1, r_heavy=x2, fidelity_cost=f, mean_latency_s=m)
                 for p, a, b, x1, x2, f, m in zip(pair.tolist(), th.tolist(), ta.tolist(),
                                                  *(v.tolist() for v in vals)))
    return rows, want


def test_columnar_rows_behave_as_the_row_tuple(tmp_path):
    rows, want = _columnar()
    assert len(rows) == len(want) and rows == want and want == rows
    assert list(rows) == list(want) and rows[5] == want[5] and rows[-1] == want[-1]
    assert rows[3:9] == want[3:9] and rows[5] is rows[5]
    assert hash(rows) == hash(want)
    with pytest.raises(IndexError):
        rows[len(rows)]
    prov = None
    from paper_2509_00642_b200.profiler import TableProvenance
    prov = TableProvenance(catalog_hash="x", prompts_hash="y", n_prompts=1, seed=0,
                           noise_sigma=0.0, thresholds=(0.0, 1.0), eps_latency=0.1,
                           eps_quality=0.1)
    a, b = str(tmp_path / "a.json"), str(tmp_path / "b.json")
    save_table(CascadeTable(rows=rows, provenance=prov), a)
    save_table(CascadeTable(rows=want, provenance=prov), b)
    assert open(a).read() == open(b).read()
    assert CascadeTable(rows=rows, provenance=prov) == CascadeTable(rows=want, provenance=prov)
    t = CascadeTable(rows=rows, provenance=prov)
    assert t.pairs() == [("a", "b"), ("a", "c"), ("b", "c")]
    assert t.rows_for_pair("a", "c") == [r for r in want if r.heavy_id == "c" and r.light_id == "a"]


def test_planner_row_arrays_columnar_equals_tuple(tmp_path, gold):
    """The planner's host conversion gives the same arrays for a columnar
    CascadeRows table and for the tuple of its rows (catalog indices, not the
    per-pair id list, feed the device rows)."""
    from paper_2509_00642_b200.catalog import CatalogError
    from paper_2509_00642_b200.planner import row_arrays
    table = load_table(_write(tmp_path, gold["misc"]["save_table_conftest160"]),
                       catalog=default_catalog())
    rows = table.rows
    pairs = sorted({(r.light_id, r.heavy_id) for r in rows})
    pid = {p: i for i, p in enumerate(pairs)}
    thr = sorted({r.theta for r in rows} | {r.tau for r in rows})
    tpos = {t: i for i, t in enumerate(thr)}
    cols = CascadeRows(pairs, [pid[(r.light_id, r.heavy_id)] for r in rows],
                       [tpos[r.theta] for r in rows], [tpos[r.tau] for r in rows],
                       [r.r_light for r in rows], [r.r_heavy for r in rows],
                       [r.fidelity_cost for r in rows], [r.mean_latency_s for r in rows], thr)
    assert cols == rows
    index = {v.id: i for i, v in enumerate(default_catalog().variants)}
    a, b = row_arrays(cols, index), row_arrays(rows, index)
    for x, y in zip(a, b):
        assert x.dtype == y.dtype and np.array_equal(x, y)
    with pytest.raises(CatalogError, match="unknown-variant"):
        row_arrays(cols, {k: v for k, v in index.items() if k != pairs[0][0]})
