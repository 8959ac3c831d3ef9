"""Golden fixtures for the text -> record step, generated
by the genuine reference (cascadesim 0.1.0):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_text.py

Writes tests/golden/text.json.gz:

* ``corpora``: the prompt texts behind the existing record goldens --
  ``conftest160`` (gen_prompts(160, 42), pkg/tests/conftest.py:8-21; its h /
  noise are in conftest160.npz), ``c1`` (gen_prompts(5000, 0); c1.npz) and the
  router corpora of make_golden_router.py (features in router.npz);
* ``cases``: hand-written edge texts (Unicode whitespace, Kelvin sign,
  punctuation-only tokens, sentence ends, long prompts, phrase overlaps ...)
  plus 3000 seeded random texts, each with the reference's stable_text_key,
  raw_features, features, hardness (default and a non-uniform weight vector)
  and stream_normal noise for several (seed, sigma) keys;
* ``tables``: profile_config on the edge + random texts (default catalog),
  and the exact bytes save_table writes for the conftest160 default table,
  plus the reference's load_table error messages.
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys
import tempfile
from dataclasses import asdict

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, HERE)

from cascadesim import catalog as rcat  # noqa: E402
from cascadesim import profiler as rprof  # noqa: E402
from cascadesim import router as rr  # noqa: E402
from cascadesim.seeds import stable_text_key, stream_normal  # noqa: E402
from cascadesim.workload import gen_prompts  # noqa: E402

from make_golden_router import corpus_cases  # noqa: E402

ALT_WEIGHTS = (0.3, 0.05, 0.2, 0.05, 0.1, 0.1, 0.15, 0.05)
NOISE_KEYS = ((0, 0.05), (7, 0.05), (-5, 1.0), (2 ** 62 + 11, 0.3), (True, 0.05), (42, 0.0))


def edge_texts(lex):
    kword = next(w for w in sorted(lex.word_freq) if "k" in w)
    texts = [
        "", "   ", "\t\n",
        "A red dog. The Blue cat! an old man? Paris is near the river",
        "...!!! ??? ,,, ;:", "! Hello . world", "end. . Next",
        "the the the red red", "a red blue green", "a red blue green the",
        "the red the dog", "a dog a", "an",
        "to the left of the right of in front of on top of next to surrounded by",
        "to the left", "to the left of", "next to to the right of above",
        "in front in front of top of",
        "Émile walks beside the river　Ωmega straße İstanbul",
        "a\tred\ndog\x1cand\x1fthe\x0bcat\x0cnear\rthe\x85house on top of"
        " the hill a b",
        "(The) [quick] {brown} `fox` \"jumps\" 'over' the lazy dog.",
        "THE RED Dog RUNNING Freedom",
        "K", kword.replace("k", "K"), kword.upper().replace("K", "K"),
        "Hello. Ärger Über ǅungla Δelta δelta \U0001d400bc",
        "x" * 100, "1st 2nd 3 red cats 42", "' a.b.c \"",
        "running jumping flying freedom love justice",
        "Zephyr and Myra walk. Orin sings! Elowen? Thane",
        "café naïve résumé the café",
        "a red castle near the river with Myra, " * 60,
        "to the left of " * 40,
        "the " * 500,
    ]
    return texts


def random_texts(lex, n, seed):
    rng = random.Random(seed)
    vocab = (sorted(lex.word_freq) + sorted(lex.adjectives) + sorted(lex.determiners)
             + sorted(lex.abstract) + sorted(lex.actions)
             + [w for p in lex.spatial for w in p] + ["Myra", "Orin", "zzyzx", "quux", "Thane"])
    seps = [" ", " ", " ", "  ", "\t", "\n", " "]
    puncts = ["", "", "", ".", ",", "!", "?", ";", "\"", "'", "(", ")"]
    out = []
    for _ in range(n):
        words = []
        for _ in range(rng.randint(0, 45)):
            w = rng.choice(vocab)
            r = rng.random()
            if r < 0.1:
                w = w.capitalize()
            elif r < 0.13:
                w = w.upper()
            if rng.random() < 0.2:
                w = rng.choice(puncts) + w
            if rng.random() < 0.25:
                w = w + rng.choice(puncts)
            words.append(w)
            words.append(rng.choice(seps))
        out.append("".join(words))
    return out


def per_text(texts, lex):
    rows = []
    for t in texts:
        raw = rr.raw_features(t, lex)
        rows.append({
            "key": str(stable_text_key(t)),
            "raw": [raw[k] for k in rr.FEATURE_NAMES],
            "features": list(rr.features(t, lex)),
            "h": rr.hardness(t, None, lex),
            "h_alt": rr.hardness(t, ALT_WEIGHTS, lex),
            "noise": [stream_normal(seed, stable_text_key(t), "disc", sigma=s)
                      for seed, s in NOISE_KEYS],
        })
    return rows


def table_doc(table):
    prov = asdict(table.provenance)
    prov["thresholds"] = list(prov["thresholds"])
    return {"provenance": prov, "rows": [asdict(r) for r in table.rows]}


def main():
    lex = rr.load_lexicons()
    corpora = {"conftest160": gen_prompts(160, seed=42), "c1": gen_prompts(5000, seed=0)}
    for name, corpus in corpus_cases():
        corpora[name] = [[t, int(lbl)] for t, lbl in corpus]
    edge = edge_texts(lex)
    rand = random_texts(lex, 3000, 99)
    cases = {"edge": {"texts": edge, "rows": per_text(edge, lex)},
             "random3000": {"texts": rand, "rows": per_text(rand, lex)}}

    cat = rcat.default_catalog()
    tables = {}
    tables["edge_random"] = table_doc(rprof.profile_config(
        cat, edge + rand, seed=3, thresholds=tuple(i / 20 for i in range(21))))
    tables["edge_random_alt"] = table_doc(rprof.profile_config(
        cat, edge + rand, seed=-8, noise_sigma=0.2, weights=ALT_WEIGHTS,
        thresholds=(0.0, 0.3, 0.3, 0.9, 0.1)))
    # test_acceptance.py's shared table (scenario.build_table of diurnal.yaml:
    # gen_prompts(2048, 5), seed 5, default grid) -- the c10 solve-latency table
    from cascadesim.scenario import build_table, load_scenario
    sc = load_scenario(os.path.join(REF, "cascadesim", "data", "scenarios", "diurnal.yaml"))
    corpora["shared2048"] = gen_prompts(sc.profile.n_prompts, sc.seed, sc.profile.hardness_range)
    shared = build_table(sc, cat)
    tables["shared2048"] = table_doc(shared)
    misc_shared = {"seed": sc.seed, "noise_sigma": sc.profile.noise_sigma,
                   "eps_latency": sc.profile.eps_latency, "eps_quality": sc.profile.eps_quality}
    conf = rprof.profile_config(cat, corpora["conftest160"], seed=42)
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "t.json")
        rprof.save_table(conf, path)
        with open(path, encoding="utf-8") as fh:
            saved = fh.read()
        errors = {}
        other = rcat.Catalog(variants=cat.variants[:3], calibrated=True)
        try:
            rprof.load_table(path, catalog=other)
        except rprof.ProfileError as exc:
            errors["mismatch"] = str(exc)
        with open(path, "w", encoding="utf-8") as fh:
            json.dump({"rows": []}, fh)
        try:
            rprof.load_table(path)
        except rprof.ProfileError as exc:
            errors["malformed"] = str(exc)
    misc = {"prompts_hash": {name: rprof.prompts_hash([x if isinstance(x, str) else x[0]
                                                        for x in texts])
                             for name, texts in corpora.items()},
            "alt_weights": list(ALT_WEIGHTS),
            "noise_keys": [[seed, s] for seed, s in NOISE_KEYS],
            "save_table_conftest160": saved, "load_errors": errors,
            "catalog_hash_default": cat.content_hash(), "shared2048": misc_shared}
    doc = {"corpora": corpora, "cases": cases, "tables": tables, "misc": misc}
    with gzip.open(os.path.join(HERE, "text.json.gz"), "wt", encoding="utf-8") as fh:
        json.dump(doc, fh, sort_keys=True)
    print({k: len(v) for k, v in corpora.items()}, len(edge), len(rand),
          {k: len(v["rows"]) for k, v in tables.items()})


if __name__ == "__main__":
    main()
