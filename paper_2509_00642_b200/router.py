"""Router weight sweep on the GPU: drop-in for cascadesim.router.tune_weights
(pkg/src/cascadesim/router.py:199-234).

``tune_weights(corpus, levels)`` keeps the reference's signature, return value
``(weights, threshold, balanced_acc)`` and error (``RouterError`` on a
degenerate corpus).  Text -> feature vectors runs on the GPU
(``text.text_features``: tokenizer + lexicon features, router.py:92-179);
``tune_weights_features`` takes a feature matrix directly.  The per-text
drop-ins ``raw_features`` / ``features`` / ``hardness`` / ``check_weights``
(router.py:154-196) and the batched ``hardness_many`` use the same kernel.
Every normalized weight vector is scored on the device (``hadis_tune_weights``: one CTA per vector, numpy-exact scores, sort, best
threshold); the reference's sequential "first unless better by 1e-12" rule
then picks the winner on the host over the per-vector results.
"""

from __future__ import annotations

import itertools

import numpy as np

from . import _lib
from .text import (DEFAULT_WEIGHTS, FEATURE_CAPS, FEATURE_NAMES, RouterError,  # noqa: F401
                   check_weights, lexicon, text_features)


def load_lexicons():
    """The packed reference lexicons (router.load_lexicons, router.py:64-87)."""
    return lexicon()


def raw_features(text: str, lex=None) -> dict:
    """router.raw_features (router.py:154-172): uncapped values by feature name."""
    raw, _, _ = text_features([text])
    return {name: float(v) for name, v in zip(FEATURE_NAMES, raw[0].tolist())}


def features(text: str, lex=None) -> tuple:
    """router.features (router.py:175-179)."""
    _, feat, _ = text_features([text])
    return tuple(feat[0].tolist())


def hardness(text: str, weights=None, lex=None) -> float:
    """router.hardness (router.py:192-196)."""
    weights = None if weights is None else check_weights(weights)
    _, _, h = text_features([text], weights)
    return float(h[0])


def hardness_many(texts, weights=None):
    """router.hardness of every text (one kernel launch), float64[n]."""
    weights = None if weights is None else check_weights(weights)
    return text_features(list(texts), weights)[2]


def _weight_grid(n_features, levels):
    grid = []
    for combo in itertools.product(levels, repeat=n_features):
        total = sum(combo)
        if total > 0:
            grid.append(tuple(value / total for value in combo))
    return grid


def tune_weights_features(features, labels, levels=(0.0, 1.0, 2.0)):
    """Best routing weights for a labeled feature matrix [N, F]."""
    torch = _lib.torch_cuda()
    mat = np.ascontiguousarray(np.asarray(features, dtype=np.float64))
    lab = np.asarray(labels, dtype=bool)
    if mat.ndim != 2 or mat.shape[0] != lab.shape[0]:
        raise RouterError("tune_weights: features must be [n_prompts, n_features]")
    if len(lab) < 2 or lab.all() or not lab.any():
        raise RouterError("degenerate-corpus: need both hard and easy examples")
    grid = _weight_grid(mat.shape[1], tuple(float(x) for x in levels))
    if not grid:
        raise RouterError("tune_weights: no non-zero weight vector on the grid")
    dev = torch.device("cuda")
    d_x = torch.from_numpy(mat).to(dev)
    d_l = torch.from_numpy(lab.astype(np.uint8)).to(dev)
    d_w = torch.tensor(grid, dtype=torch.float64, device=dev)
    acc = torch.empty(len(grid), dtype=torch.float64, device=dev)
    thr = torch.empty(len(grid), dtype=torch.float64, device=dev)
    p = _lib.ptr
    _lib.check(_lib.load().hadis_tune_weights(p(d_x), p(d_l), mat.shape[0], mat.shape[1], p(d_w),
                                              len(grid), int(lab.sum()), p(acc), p(thr),
                                              _lib.stream_handle()), "hadis_tune_weights")
    accs, thrs = acc.cpu().tolist(), thr.cpu().tolist()
    best = None                                   # router.py:229-231, in enumeration order
    for a, w, t in zip(accs, grid, thrs):
        if best is None or a > best[0] + 1e-12:
            best = (a, w, t)
    return best[1], best[2], best[0]


def tune_weights(corpus, levels=(0.0, 1.0, 2.0)):
    """Exhaustive grid search for routing weights on a labeled corpus of
    (text, label) pairs; returns (weights, threshold, balanced_acc)."""
    labels = np.array([int(label) for _, label in corpus], dtype=bool)
    if len(corpus) < 2 or labels.all() or not labels.any():
        raise RouterError("degenerate-corpus: need both hard and easy examples")
    _, mat, _ = text_features([text for text, _ in corpus])
    return tune_weights_features(mat, labels, levels)
