"""CPU oracle (test infrastructure only) for the router weight sweep, SURVEY §8 f3:
a numpy restatement of pkg/src/cascadesim/router.py:199-234 (``tune_weights``)
over a precomputed feature matrix.  Pinned to tests/golden/router.json
(generator: tests/golden/make_golden_router.py)."""

from __future__ import annotations

import itertools

import numpy as np


def weight_grid(n_features, levels=(0.0, 1.0, 2.0)):
    """Normalized weight vectors in itertools.product order (all-zero skipped)."""
    out = []
    for combo in itertools.product(levels, repeat=n_features):
        total = sum(combo)
        if total > 0:
            out.append(tuple(v / total for v in combo))
    return out


def best_split(mat, labels, weights):
    """(balanced accuracy, threshold) of one weight vector at its best cut."""
    labels = np.asarray(labels, dtype=bool)
    n_pos = int(labels.sum())
    n_neg = labels.size - n_pos
    scores = mat @ np.asarray(weights)
    cuts = np.unique(scores)
    cand = np.concatenate(([cuts[0] - 1.0], (cuts[:-1] + cuts[1:]) / 2.0, [cuts[-1] + 1.0]))
    hard = scores[None, :] > cand[:, None]
    acc = ((hard & labels).sum(axis=1) / n_pos + (~hard & ~labels).sum(axis=1) / n_neg) / 2.0
    i = int(np.argmax(acc))
    return float(acc[i]), float(cand[i])


def tune(mat, labels, levels=(0.0, 1.0, 2.0)):
    """(weights, threshold, acc): first vector unless a later one is better by 1e-12."""
    best = None
    for w in weight_grid(mat.shape[1], levels):
        acc, thr = best_split(mat, labels, w)
        if best is None or acc > best[0] + 1e-12:
            best = (acc, w, thr)
    return best[1], best[2], best[0]
