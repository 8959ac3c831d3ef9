"""CPU oracle (test infrastructure only) for the text -> record step, SURVEY §8
rows a1/f3: a plain-Python restatement of

* cascadesim.router ``tokenize`` / ``_rarity`` / ``_count_objects`` /
  ``_count_spatial`` / ``raw_features`` / ``features`` / ``hardness``
  (pkg/src/cascadesim/router.py:92-196), and
* cascadesim.seeds ``_digest`` / ``stream_normal`` / ``stable_text_key``
  (pkg/src/cascadesim/seeds.py:18-55),

over the lexicon data the package ships (paper_2509_00642_b200/data/
lexicons.json, packed from the reference's data/lexicons by
tools/pack_lexicons.py).  Pinned to tests/golden/text.json.gz (generator:
tests/golden/make_golden_text.py, which runs the genuine reference).

Nothing in the product path imports this module.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import re
import struct

FEATURE_CAPS = (40.0, 1.0, 5.0, 1.0, 1.0, 5.0, 5.0, 5.0)       # router.py:31
_PUNCT = ".,;:!?\"'()[]{}`"                                     # router.py:37
_SENTENCE_END = re.compile(r"[.!?]$")                           # router.py:38
_DATA = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "paper_2509_00642_b200", "data", "lexicons.json")


class Lex:
    """router.load_lexicons (router.py:64-87) over the packed data file."""

    def __init__(self, path=_DATA):
        with open(path, encoding="utf-8") as fh:
            files = json.load(fh)["files"]
        self.word_freq = {}
        for line in files["word_frequency.tsv"]:
            word, value = line.split("\t")
            self.word_freq[word] = float(value)
        self.freq_floor = min(self.word_freq.values())
        phrases = [tuple(p.split()) for p in files["spatial_phrases.txt"]]
        phrases.sort(key=lambda p: (-len(p), p))
        self.by_first = {}
        for p in phrases:
            self.by_first.setdefault(p[0], []).append(p)
        self.abstract = frozenset(files["abstract_nouns.txt"])
        self.actions = frozenset(files["action_verbs.txt"])
        self.determiners = frozenset(files["noun_markers.txt"])
        self.adjectives = frozenset(files["adjectives.txt"])


_LEX = None


def lexicons():
    global _LEX
    if _LEX is None:
        _LEX = Lex()
    return _LEX


def tokenize(text):
    """router.py:92-104 -> list of (raw, lower, sentence_initial)."""
    out = []
    start = True
    for raw in text.split():
        word = raw.strip(_PUNCT)
        ends = bool(_SENTENCE_END.search(raw))
        if word:
            out.append((word, word.lower(), start))
            start = ends
        elif ends:
            start = True
    return out


def rarity(word, lex):
    """router.py:107-114."""
    freq = lex.word_freq.get(word)
    if freq is None:
        return 1.0
    freq = min(max(freq, lex.freq_floor), 1.0)
    if freq >= 1.0:
        return 0.0
    return math.log(freq) / math.log(lex.freq_floor)


def count_objects(lowers, lex):
    """router.py:117-131."""
    count, i = 0, 0
    while i < len(lowers):
        if lowers[i] in lex.determiners:
            j = i + 1
            while j < len(lowers) and lowers[j] in lex.adjectives:
                j += 1
            if j < len(lowers) and lowers[j] not in lex.determiners:
                count += 1
                i = j + 1
                continue
        i += 1
    return count


def count_spatial(lowers, lex):
    """router.py:134-151."""
    count, i, n = 0, 0, len(lowers)
    while i < n:
        matched = False
        for phrase in lex.by_first.get(lowers[i], ()):
            k = len(phrase)
            if i + k <= n and tuple(lowers[i:i + k]) == phrase:
                count += 1
                i += k
                matched = True
                break
        if not matched:
            i += 1
    return count


def raw_features(text, lex=None):
    """router.py:154-172, as a tuple in FEATURE_NAMES order."""
    lex = lex or lexicons()
    toks = tokenize(text)
    lowers = [t[1] for t in toks]
    n = len(toks)
    objects = count_objects(lowers, lex)
    adjectives = sum(1 for w in lowers if w in lex.adjectives)
    return (float(n),
            (sum(rarity(w, lex) for w in lowers) / n) if n else 0.0,
            float(objects),
            float(sum(1 for w in lowers if w in lex.abstract)),
            adjectives / max(1, objects),
            float(count_spatial(lowers, lex)),
            float(sum(1 for w in lowers if w in lex.actions)),
            float(sum(1 for raw, _, first in toks if raw[0].isupper() and not first)))


def features(text, lex=None):
    """router.py:175-179."""
    return tuple(min(r / c, 1.0) for r, c in zip(raw_features(text, lex), FEATURE_CAPS))


def hardness(text, weights=None, lex=None):
    """router.py:192-196 (weights already validated)."""
    w = (0.125,) * 8 if weights is None else tuple(float(x) for x in weights)
    vec = features(text, lex)
    return min(1.0, max(0.0, sum(a * b for a, b in zip(w, vec))))


def stable_text_key(text):
    """seeds.py:49-55."""
    return int.from_bytes(hashlib.sha256(text.encode("utf-8")).digest()[:8], "big") >> 1


def digest(parts):
    """seeds.py:18-30."""
    h = hashlib.blake2b(digest_size=16)
    for part in parts:
        if isinstance(part, bool):
            h.update(b"b" + (b"\x01" if part else b"\x00"))
        elif isinstance(part, int):
            h.update(b"i" + struct.pack(">q", part))
        elif isinstance(part, str):
            h.update(b"s" + part.encode("utf-8"))
        else:
            raise TypeError("stream keys must be ints or strings, got %r" % (part,))
        h.update(b"\x1f")
    return h.digest()


def stream_normal(*key, sigma=1.0):
    """seeds.py:38-46."""
    if sigma == 0.0:
        return 0.0
    d = digest(key)
    u1 = (int.from_bytes(d[:8], "big") + 1.0) / (2.0 ** 64 + 2.0)
    u2 = int.from_bytes(d[8:16], "big") / 2.0 ** 64
    return sigma * math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def text_records(prompts, seed, sigma=0.05, weights=None):
    """profiler.py:125-132: texts in key order, hardness and keyed noise."""
    lex = lexicons()
    texts = sorted(prompts, key=stable_text_key)
    h = [hardness(t, weights, lex) for t in texts]
    noise = [stream_normal(seed, stable_text_key(t), "disc", sigma=sigma) for t in texts]
    return texts, h, noise
