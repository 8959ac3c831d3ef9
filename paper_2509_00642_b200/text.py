"""Text -> records on the GPU.

Host side of ``hadis_text_records`` / ``hadis_text_features`` (csrc/text.cu):
the record prep of ``profile_config`` (reference profiler.py:125-132) --
prompts in ``stable_text_key`` order (seeds.py:49-55), ``router.hardness``
per prompt (router.py:92-196) and the keyed discriminator noise
``stream_normal(seed, key, "disc", sigma)`` (seeds.py:18-46).

What runs where:

* GPU: SHA-256 prompt keys, the stable key sort (CUB radix sort), the
  tokenizer and every lexicon feature, the hardness sum, and the BLAKE2b
  digest that yields stream_normal's two uniforms.
* host: packing the prompts into one UTF-8 byte buffer, the lexicon image
  (built once; rarity values use the host libm like router._rarity), and
  Box-Muller's ``log``/``cos`` through ``hadis_keyed_normal_host`` -- glibc's
  functions, which CPython's math module calls and libdevice does not
  reproduce bit for bit.

The lexicons are the reference's data files, packed into
``data/lexicons.json`` by tools/pack_lexicons.py.
"""

from __future__ import annotations

import ctypes
import hashlib
import json
import math
import os
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib

FEATURE_NAMES = (
    "prompt_length", "token_rarity", "num_objects", "abstractness",
    "attribute_density", "spatial_relations", "action_verbs", "named_entities",
)                                                                     # router.py:20-29
FEATURE_CAPS = (40.0, 1.0, 5.0, 1.0, 1.0, 5.0, 5.0, 5.0)              # router.py:30
DEFAULT_WEIGHTS = tuple(1.0 / len(FEATURE_NAMES) for _ in FEATURE_NAMES)
_PUNCT = ".,;:!?\"'()[]{}`"                                           # router.py:37
_DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "lexicons.json")

TABLE = 2048
MAX_WORDS = 1024
MAX_PHRASES = 128
MAX_PHRASE_LEN = 8
POOL = 16384
MAX_WORD_BYTES = 64
F_DET, F_ADJ, F_ABS, F_ACT, F_FREQ = 1, 2, 4, 8, 16


class RouterError(ValueError):
    pass


def check_weights(weights) -> tuple:
    """router.check_weights (router.py:182-189)."""
    weights = tuple(float(w) for w in weights)
    if len(weights) != len(FEATURE_NAMES):
        raise RouterError(f"weights: expected {len(FEATURE_NAMES)} values")
    if any(w < 0 for w in weights):
        raise RouterError("weights: must be non-negative")
    if abs(sum(weights) - 1.0) > 1e-9:
        raise RouterError("weights: must sum to 1")
    return weights


class LexiconImage(ctypes.Structure):
    """Mirror of ``hadis_lexicon`` (include/hadis_b200.h)."""

    _fields_ = [
        ("rarity", ctypes.c_double * MAX_WORDS),
        ("n_words", ctypes.c_int32), ("n_phrases", ctypes.c_int32),
        ("max_phrase_len", ctypes.c_int32), ("max_word_bytes", ctypes.c_int32),
        ("table", ctypes.c_int16 * TABLE),
        ("word_off", ctypes.c_uint16 * MAX_WORDS),
        ("phrase_begin", ctypes.c_uint16 * MAX_WORDS),
        ("phrase_count", ctypes.c_uint8 * MAX_WORDS),
        ("word_len", ctypes.c_uint8 * MAX_WORDS),
        ("word_flags", ctypes.c_uint8 * MAX_WORDS),
        ("phrase_len", ctypes.c_uint8 * MAX_PHRASES),
        ("phrase_words", (ctypes.c_int16 * MAX_PHRASE_LEN) * MAX_PHRASES),
        ("pool", ctypes.c_char * POOL),
    ]


def fnv1a32(data: bytes) -> int:
    h = 2166136261
    for b in data:
        h = ((h ^ b) * 16777619) & 0xFFFFFFFF
    return h


def _matchable(word: str) -> bool:
    """Can a lowered, punctuation-stripped token ever equal ``word``?"""
    return (bool(word) and word.isascii() and word == word.lower()
            and not any(c.isspace() for c in word)
            and word[0] not in _PUNCT and word[-1] not in _PUNCT)


class Lexicon:
    """router.load_lexicons (router.py:64-87) as the device image."""

    def __init__(self, path: str = _DATA):
        with open(path, encoding="utf-8") as fh:
            files = json.load(fh)["files"]
        freq = {}
        for line in files["word_frequency.tsv"]:
            word, value = line.split("\t")
            freq[word] = float(value)
        self.freq = freq
        self.freq_floor = min(freq.values())
        phrases = [tuple(p.split()) for p in files["spatial_phrases.txt"]]
        phrases.sort(key=lambda p: (-len(p), p))
        sets = {F_DET: files["noun_markers.txt"], F_ADJ: files["adjectives.txt"],
                F_ABS: files["abstract_nouns.txt"], F_ACT: files["action_verbs.txt"]}
        if set(sets[F_DET]) & set(sets[F_ADJ]):
            raise ValueError("lexicons: a word is both a noun marker and an adjective; the "
                             "object counter's two-state scan does not cover that")
        flags = {}
        for bit, words in sets.items():
            for w in words:
                flags[w] = flags.get(w, 0) | bit
        for w in freq:
            flags[w] = flags.get(w, 0) | F_FREQ
        by_first = {}
        for p in phrases:
            if all(_matchable(w) for w in p):       # others can never match a token
                by_first.setdefault(p[0], []).append(p)
        for p in (q for qs in by_first.values() for q in qs):
            for w in p:
                flags.setdefault(w, 0)
        words = sorted(w for w in flags if _matchable(w))
        for w in flags:
            if not w.isascii():
                raise ValueError(f"lexicons: non-ASCII word {w!r} is not supported")
        if len(words) > MAX_WORDS:
            raise ValueError("lexicons: too many words for the device image")
        self.words = words
        self.flags = flags
        self.by_first = by_first
        self.image = self._build()

    def rarity(self, word: str) -> float:
        """router._rarity (router.py:107-114), host libm."""
        f = self.freq.get(word)
        if f is None:
            return 1.0
        f = min(max(f, self.freq_floor), 1.0)
        if f >= 1.0:
            return 0.0
        return math.log(f) / math.log(self.freq_floor)

    def _build(self) -> LexiconImage:
        img = LexiconImage()
        ids = {w: i for i, w in enumerate(self.words)}
        for i in range(TABLE):
            img.table[i] = -1
        pool = bytearray()
        maxw = 0
        for i, w in enumerate(self.words):
            b = w.encode("ascii")
            maxw = max(maxw, len(b))
            if len(b) > MAX_WORD_BYTES:
                raise ValueError(f"lexicons: word {w!r} longer than {MAX_WORD_BYTES} bytes")
            img.word_off[i] = len(pool)
            img.word_len[i] = len(b)
            img.word_flags[i] = self.flags[w]
            img.rarity[i] = self.rarity(w)
            pool += b
            slot = fnv1a32(b) & (TABLE - 1)
            while img.table[slot] != -1:
                slot = (slot + 1) & (TABLE - 1)
            img.table[slot] = i
        if len(pool) > POOL:
            raise ValueError("lexicons: string pool overflow")
        img.pool = bytes(pool)
        k = 0
        maxlen = 0
        for w in self.words:
            ps = self.by_first.get(w, ())
            img.phrase_begin[ids[w]] = k
            img.phrase_count[ids[w]] = len(ps)
            for p in ps:
                if k >= MAX_PHRASES or len(p) > MAX_PHRASE_LEN:
                    raise ValueError("lexicons: spatial phrase table overflow")
                img.phrase_len[k] = len(p)
                for j, pw in enumerate(p):
                    img.phrase_words[k][j] = ids[pw]
                maxlen = max(maxlen, len(p))
                k += 1
        img.n_words, img.n_phrases = len(self.words), k
        img.max_phrase_len, img.max_word_bytes = maxlen, maxw
        return img


_LEXICON = None
_DEVICE_LEX = {}


def lexicon() -> Lexicon:
    global _LEXICON
    if _LEXICON is None:
        _LEXICON = Lexicon()
    return _LEXICON


def device_lexicon(device):
    """The lexicon image as a device byte tensor (built once per device)."""
    torch = _lib.torch_cuda()
    key = str(device)
    t = _DEVICE_LEX.get(key)
    if t is None:
        img = lexicon().image
        raw = np.frombuffer(bytes(img), dtype=np.uint8).copy()
        t = _DEVICE_LEX[key] = torch.from_numpy(raw).to(device)
    return t


def digest_part(part) -> bytes:
    """One packed key part of seeds._digest (seeds.py:18-30)."""
    if isinstance(part, bool):
        return b"b" + (b"\x01" if part else b"\x00") + b"\x1f"
    if isinstance(part, int):
        return b"i" + struct.pack(">q", part) + b"\x1f"
    if isinstance(part, str):
        return b"s" + part.encode("utf-8") + b"\x1f"
    raise TypeError("stream keys must be ints or strings, got %r" % (part,))


def pack_texts(texts):
    """UTF-8 byte buffer + int64 offsets[n + 1] (host numpy)."""
    joined = "".join(texts)
    if joined.isascii():                 # byte lengths = character lengths: one encode
        offs = np.zeros(len(texts) + 1, dtype=np.int64)
        np.cumsum(np.fromiter(map(len, texts), dtype=np.int64, count=len(texts)), out=offs[1:])
        blob = np.frombuffer(bytearray(joined.encode("ascii") or b"\0"), dtype=np.uint8)
        return blob, offs
    enc = [t.encode("utf-8") for t in texts]
    offs = np.zeros(len(enc) + 1, dtype=np.int64)
    np.cumsum(np.fromiter(map(len, enc), dtype=np.int64, count=len(enc)), out=offs[1:])
    blob = np.frombuffer(bytearray(b"".join(enc) or b"\0"), dtype=np.uint8)
    return blob, offs


def _weights_vec(weights):
    return DEFAULT_WEIGHTS if weights is None else tuple(float(w) for w in weights)


@dataclass
class TextRecords:
    order: np.ndarray        # int64[n]: input index of the j-th prompt in key order
    keys: np.ndarray         # uint64[n]: stable_text_key, sorted
    h: np.ndarray            # float64[n] hardness (key order)
    noise: np.ndarray        # float64[n] keyed discriminator noise (key order)
    d_h: object              # the same hardness, device tensor
    stats: dict


def text_records(texts, seed, noise_sigma, weights=None, device=None, raw=False) -> TextRecords:
    """profiler.py:125-132 on the GPU: key order, hardness, keyed noise."""
    torch = _lib.torch_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda")
    lib = _lib.load()
    n = len(texts)
    blob, offs = pack_texts(texts)
    seed_part = digest_part(seed) if noise_sigma != 0.0 else b""
    chan = digest_part("disc")
    d_blob = torch.from_numpy(blob).to(dev)
    d_offs = torch.from_numpy(offs).to(dev)
    d_w = torch.tensor(_weights_vec(weights), dtype=torch.float64, device=dev)
    d_seed = torch.tensor(list(seed_part or b"\0"), dtype=torch.uint8, device=dev)
    d_chan = torch.tensor(list(chan), dtype=torch.uint8, device=dev)
    order = torch.empty(n, dtype=torch.int64, device=dev)
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    d_h = torch.empty(n, dtype=torch.float64, device=dev)
    u = torch.empty((2, n), dtype=torch.float64, device=dev)
    d_raw = torch.empty((n, 8), dtype=torch.float64, device=dev) if raw else None
    ws_bytes = lib.hadis_text_workspace_bytes(n)
    if ws_bytes == 0:
        raise ValueError("text_records: too many prompts for one call")
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    p = _lib.ptr
    _lib.check(lib.hadis_text_records(
        p(d_blob), p(d_offs), n, p(device_lexicon(dev)), p(d_w), p(d_seed), len(seed_part),
        p(d_chan), len(chan), p(order), p(keys), p(d_h), p(u[0]), p(u[1]), p(d_raw), p(ws),
        ws_bytes, _lib.stream_handle()), "hadis_text_records")
    h = d_h.cpu().numpy()
    uu = u.cpu().numpy()
    noise = np.empty(n, dtype=np.float64)
    _lib.check(lib.hadis_keyed_normal_host(
        uu[0].ctypes.data_as(ctypes.c_void_p), uu[1].ctypes.data_as(ctypes.c_void_p), n,
        float(noise_sigma), noise.ctypes.data_as(ctypes.c_void_p), 0), "hadis_keyed_normal_host")
    rec = TextRecords(order=order.cpu().numpy(), keys=keys.cpu().numpy().view(np.uint64), h=h,
                      noise=noise, d_h=d_h, stats={})
    if raw:
        rec.stats["raw"] = d_raw.cpu().numpy()
    return rec


def text_features(texts, weights=None, device=None):
    """(raw [n, 8], features [n, 8], hardness [n]) per prompt, input order."""
    torch = _lib.torch_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda")
    lib = _lib.load()
    n = len(texts)
    blob, offs = pack_texts(texts)
    d_blob = torch.from_numpy(blob).to(dev)
    d_offs = torch.from_numpy(offs).to(dev)
    d_w = torch.tensor(_weights_vec(weights), dtype=torch.float64, device=dev)
    out = torch.empty((2, max(n, 1), 8), dtype=torch.float64, device=dev)
    d_h = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    p = _lib.ptr
    _lib.check(lib.hadis_text_features(p(d_blob), p(d_offs), n, p(device_lexicon(dev)), p(d_w),
                                       None, p(d_h), p(out[0]), p(out[1]), _lib.stream_handle()),
               "hadis_text_features")
    o = out.cpu().numpy()
    return o[0][:n], o[1][:n], d_h.cpu().numpy()[:n]


def text_keys(texts, device=None):
    """stable_text_key of every prompt (GPU SHA-256), input order, as Python ints."""
    torch = _lib.torch_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda")
    n = len(texts)
    blob, offs = pack_texts(texts)
    d_blob = torch.from_numpy(blob).to(dev)
    d_offs = torch.from_numpy(offs).to(dev)
    keys = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    _lib.check(_lib.load().hadis_text_keys(_lib.ptr(d_blob), _lib.ptr(d_offs), n,
                                           _lib.ptr(keys), _lib.stream_handle()),
               "hadis_text_keys")
    return [int(k) for k in keys.cpu().numpy().view(np.uint64)[:n]]


def prompts_hash_sorted(texts_sorted) -> str:
    """profiler.prompts_hash (profiler.py:101-104) of prompts already in key order."""
    return hashlib.sha256("\x1f".join(texts_sorted).encode("utf-8")).hexdigest()[:16]
