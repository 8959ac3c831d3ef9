"""CPU: the router weight-sweep oracle (oracle/router.py) reproduces the
reference's tune_weights bit for bit on the golden corpora."""

import numpy as np
import pytest

from oracle import router as orr
from tests.goldens import load_json, load_npz

DOCS = {d["name"]: d for d in load_json("router")}
ARR = load_npz("router")


@pytest.mark.parametrize("name", ["separable80", "noisy600"])
def test_oracle_tune_matches_reference(name):
    d = DOCS[name]
    w, thr, acc = orr.tune(ARR[name + ":features"], ARR[name + ":labels"])
    assert (list(w), thr, acc) == (d["weights"], d["threshold"], d["acc"])


def test_oracle_per_vector_matches_reference():
    d = DOCS["separable80"]
    mat, lab = ARR["separable80:features"], ARR["separable80:labels"]
    grid = orr.weight_grid(mat.shape[1])
    assert len(grid) == len(d["per_vector"]) == 3 ** 8 - 1
    for w, (acc, thr) in list(zip(grid, d["per_vector"]))[::37]:
        assert orr.best_split(mat, lab, w) == (acc, thr)
