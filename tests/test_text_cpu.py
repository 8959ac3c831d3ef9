"""Host logic of the GPU text path (no device calls): the lexicon image, the
digest key packing, the committed Unicode tables, the weight check."""

import ctypes
import os
import struct

import numpy as np

import pytest

from oracle import text as ot
from paper_2509_00642_b200 import _lib, text
from tests.goldens import load_text

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_lexicon_image_layout_matches_the_library():
    assert ctypes.sizeof(text.LexiconImage) == _lib.load().hadis_lexicon_bytes()


def test_lexicon_image_contents():
    lex = text.lexicon()
    img = lex.image
    ref = ot.lexicons()
    words = [img.pool[img.word_off[i]:img.word_off[i] + img.word_len[i]].decode()
             for i in range(img.n_words)]
    assert words == lex.words
    for i, w in enumerate(words):
        slot = text.fnv1a32(w.encode()) & (text.TABLE - 1)
        while img.table[slot] != i:                 # reachable by linear probing
            assert img.table[slot] != -1
            slot = (slot + 1) & (text.TABLE - 1)
        fl = img.word_flags[i]
        assert bool(fl & text.F_DET) == (w in ref.determiners)
        assert bool(fl & text.F_ADJ) == (w in ref.adjectives)
        assert bool(fl & text.F_ABS) == (w in ref.abstract)
        assert bool(fl & text.F_ACT) == (w in ref.actions)
        assert bool(fl & text.F_FREQ) == (w in ref.word_freq)
        assert img.rarity[i] == ot.rarity(w, ref) or not fl & text.F_FREQ
    # phrases in the reference's scan order, grouped by first word
    for first, phrases in ref.by_first.items():
        i = words.index(first)
        got = [tuple(words[img.phrase_words[k][j]] for j in range(img.phrase_len[k]))
               for k in range(img.phrase_begin[i], img.phrase_begin[i] + img.phrase_count[i])]
        assert got == phrases
    assert img.max_phrase_len == max(len(p) for ps in ref.by_first.values() for p in ps)


@pytest.mark.parametrize("part", [0, 7, -5, 2 ** 62 + 11, True, False, "disc", "é"])
def test_digest_parts_match_seeds_packing(part):
    # seeds._digest packs each part then "\x1f"; the oracle restates it
    import hashlib
    h = hashlib.blake2b(digest_size=16)
    h.update(text.digest_part(part))
    assert h.digest() == ot.digest((part,))


def test_digest_part_errors_like_the_reference():
    with pytest.raises(struct.error):
        text.digest_part(2 ** 63)
    with pytest.raises(TypeError, match="stream keys must be ints or strings"):
        text.digest_part(1.5)


def test_committed_unicode_tables_match_this_interpreter():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "gen", os.path.join(ROOT, "tools", "gen_unicode_tables.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    with open(gen.OUT, encoding="utf-8") as fh:
        committed = fh.read()
    assert committed.split("\n", 1)[1] == gen.render().split("\n", 1)[1]


def test_check_weights_messages():
    with pytest.raises(text.RouterError, match="weights: expected 8 values"):
        text.check_weights([1.0])
    with pytest.raises(text.RouterError, match="weights: must be non-negative"):
        text.check_weights([-0.5, 1.5] + [0.0] * 6)
    with pytest.raises(text.RouterError, match="weights: must sum to 1"):
        text.check_weights([0.5] * 8)
    assert text.check_weights([0.125] * 8) == text.DEFAULT_WEIGHTS


def test_pack_texts_offsets():
    blob, offs = text.pack_texts(["", "ab", "é", ""])
    assert offs.tolist() == [0, 0, 2, 4, 4]
    assert bytes(blob[:4]) == b"ab\xc3\xa9"


def test_prompts_hash_and_keys_are_the_reference_values():
    gold = load_text()
    for row, t in zip(gold["cases"]["edge"]["rows"], gold["cases"]["edge"]["texts"]):
        from paper_2509_00642_b200.profiler import stable_text_key
        assert str(stable_text_key(t)) == row["key"]
    from paper_2509_00642_b200.profiler import prompts_hash
    for name, texts in gold["corpora"].items():
        texts = [x if isinstance(x, str) else x[0] for x in texts]
        assert prompts_hash(texts) == gold["misc"]["prompts_hash"][name]
        assert prompts_hash(list(reversed(texts))) == gold["misc"]["prompts_hash"][name]


@pytest.mark.parametrize("texts", [["abc", "", "d e"], ["Émile x", "y", ""], [], [""],
                                   ["plain ascii", "naïve café", "日本"]])
def test_pack_texts_layout(texts):
    """pack_texts (ASCII fast path and the general UTF-8 path): blob = the
    concatenated UTF-8 bytes, offsets = their running byte lengths."""
    from paper_2509_00642_b200.text import pack_texts
    blob, offs = pack_texts(texts)
    enc = [t.encode("utf-8") for t in texts]
    assert offs.tolist() == [0] + list(np.cumsum([len(e) for e in enc]).tolist())
    assert bytes(blob[:offs[-1]]) == b"".join(enc)
