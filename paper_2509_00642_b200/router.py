"""Router weight sweep on the GPU: drop-in for cascadesim.router.tune_weights
(pkg/src/cascadesim/router.py:199-234).

``tune_weights(corpus, levels)`` keeps the reference's signature, return value
``(weights, threshold, balanced_acc)`` and error (``RouterError`` on a
degenerate corpus).  Text -> feature vectors stays on the host with the
reference's own ``router.features`` (string processing, like hardness in
``profile_config``); ``tune_weights_features`` takes the feature matrix
directly.  Every normalized weight vector is scored on the device
(``hadis_tune_weights``: one CTA per vector, numpy-exact scores, sort, best
threshold); the reference's sequential "first unless better by 1e-12" rule
then picks the winner on the host over the per-vector results.
"""

from __future__ import annotations

import itertools

import numpy as np

from . import _lib


class RouterError(ValueError):
    pass


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
    try:
        from cascadesim import router as text_router
    except ImportError as exc:  # pragma: no cover - depends on the user's install
        raise ImportError("tune_weights on prompt text needs cascadesim's router.features "
                          "(text -> features); use tune_weights_features otherwise") from exc
    lex = text_router.load_lexicons()
    mat = np.array([text_router.features(text, lex) for text, _ in corpus])
    return tune_weights_features(mat, labels, levels)
