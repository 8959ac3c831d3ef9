"""The text -> record oracle (oracle/text.py) against the reference's own outputs
(tests/golden/text.json.gz, c1.npz, conftest160.npz, router.npz).  CPU only."""

import numpy as np
import pytest

from oracle import text as ot
from tests.goldens import load_npz, load_text


@pytest.fixture(scope="module")
def gold():
    return load_text()


@pytest.mark.parametrize("case", ["edge", "random3000"])
def test_per_text_values(gold, case):
    c = gold["cases"][case]
    seeds = gold["misc"]["noise_keys"]
    alt = gold["misc"]["alt_weights"]
    for text, row in zip(c["texts"], c["rows"]):
        assert str(ot.stable_text_key(text)) == row["key"]
        assert list(ot.raw_features(text)) == row["raw"], text
        assert list(ot.features(text)) == row["features"]
        assert ot.hardness(text) == row["h"]
        assert ot.hardness(text, alt) == row["h_alt"]
        assert [ot.stream_normal(s, ot.stable_text_key(text), "disc", sigma=sg)
                for s, sg in seeds] == row["noise"]


@pytest.mark.parametrize("name,seed", [("conftest160", 42), ("c1", 0)])
def test_records_match_record_goldens(gold, name, seed):
    texts, h, noise = ot.text_records(gold["corpora"][name], seed)
    z = load_npz(name)
    assert np.array_equal(np.asarray(h), z["h"])
    assert np.array_equal(np.asarray(noise), z["noise"])


@pytest.mark.parametrize("name", ["separable80", "noisy600", "noisy3000"])
def test_router_features_match(gold, name):
    mat = np.array([ot.features(t) for t, _ in gold["corpora"][name]])
    assert np.array_equal(mat, load_npz("router")[name + ":features"])
