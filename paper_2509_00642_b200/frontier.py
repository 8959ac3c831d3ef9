"""Cascade-depth frontier on the GPU: drop-in for cascadesim.frontier.

Same public surface as pkg/src/cascadesim/frontier.py: ``THRESHOLDS``,
``FrontierError``, ``FrontierPoint``, ``FrontierReport``, ``default_hardness``,
``two_stage_points``, ``three_stage_points``, ``lower_envelope``,
``envelope_value``, ``envelope_gap``, ``frontier_compare``.

Every two-stage (light < heavy) and three-stage (light < middle < heavy)
operating point comes from ``hadis_cascade_points`` (libhadis_b200.so): one
pass bins the population into 3-D (theta-row, tau1-bin, tau2-bin) histograms
per model pair, prefix sums turn them into per-point counts and hardness sums,
and one thread per point evaluates latency (bit-exact, the reference's float
expression) and fidelity.  Two-stage fidelities are then replaced by the
numpy-exact pairwise sums of ``hadis_fid_exact`` (``exact=True``, default);
three-stage fidelities are the fixed-point restatement (within ~1e-15 relative).
The lower convex envelope and the gap run on the host over the points that
can be hull vertices (not beaten in fidelity from both the left and the right).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib

THRESHOLDS = tuple(i / 10 for i in range(11))


class FrontierError(ValueError):
    pass


@dataclass(frozen=True)
class FrontierPoint:
    latency_s: float
    fidelity_cost: float
    detail: tuple  # (model ids..., thresholds...) for reporting


@dataclass(frozen=True)
class FrontierReport:
    gap: float
    envelope_two: tuple
    envelope_three: tuple
    n_two: int
    n_three: int


def default_hardness(n: int = 256) -> np.ndarray:
    """Evenly spread hardness population on (0, 1): bin midpoints (frontier.py:47-49)."""
    return (np.arange(n) + 0.5) / n


def _by_latency(variants):
    return sorted(variants, key=lambda v: (v.latency_s[1], v.id))


def _accept_scores(variants, h):
    """Noise-free accept scores with the reference's numpy expression (frontier.py:52-57)."""
    out = np.empty((len(variants), h.shape[0]), dtype=np.float64)
    for m, v in enumerate(variants):
        a, s = v.accept_params
        out[m] = 1.0 / (1.0 + np.exp(-(a - s * h)))
    return out


class CascadePoints:
    """Device evaluation of every cascade point over the distinct thresholds.

    ``two[p, a, b]`` / ``three[t, a, b, c]`` hold (lat, fid) for pair p /
    triple t (lexicographic over latency-ordered models) and distinct
    threshold ranks a (theta), b (tau / tau1), c (tau2)."""

    def __init__(self, variants, h, thresholds, exact=True):
        torch = _lib.torch_cuda()
        self.variants = _by_latency(variants)
        self.h = np.ascontiguousarray(np.asarray(h, dtype=np.float64))
        thr = tuple(float(t) for t in thresholds)
        if not thr:
            raise FrontierError("frontier: empty threshold grid")
        if any(math.isnan(t) for t in thr):
            raise FrontierError("frontier: NaN thresholds are not supported")
        self.thresholds = thr
        first = {}
        for i, t in enumerate(thr):
            first.setdefault(t, i)
        self.unique = tuple(sorted(first))
        self.rank = np.array([self.unique.index(t) for t in thr], dtype=np.int64)
        n, M, U = self.h.shape[0], len(self.variants), len(self.unique)
        if n == 0:
            raise FrontierError("frontier: empty hardness population")
        if M > 16:
            raise FrontierError("frontier: at most 16 variants are supported")
        dev = torch.device("cuda")
        lib = _lib.load()
        d_h = torch.from_numpy(self.h).to(dev)
        d_s = torch.from_numpy(_accept_scores(self.variants, self.h)).to(dev)
        params = np.array([[v.latency_s[1], v.base_quality_cost, v.hardness_penalty]
                           for v in self.variants], dtype=np.float64)
        d_p = torch.from_numpy(params).to(dev)
        d_u = torch.tensor(self.unique, dtype=torch.float64, device=dev)
        P2, P3 = M * (M - 1) // 2, M * (M - 1) * (M - 2) // 6
        out2 = torch.empty((P2, U, U, 2), dtype=torch.float64, device=dev)
        out3 = torch.empty((max(P3, 1), U, U, U, 2), dtype=torch.float64, device=dev)
        bad = torch.zeros(1, dtype=torch.int32, device=dev)
        ws_bytes = lib.hadis_cascade_workspace_bytes(M, U)
        ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=dev)
        p = _lib.ptr
        st = _lib.stream_handle()
        shift = lib.hadis_hfix_shift(n)
        _lib.check(lib.hadis_cascade_points(p(d_h), p(d_s), n, M, p(d_p), p(d_u), U, shift,
                                            p(out2), p(out3), p(bad), p(ws), ws_bytes, st),
                   "hadis_cascade_points")
        self._d = (d_h, d_s, params, n, U, M)
        if exact and P2:
            out2.view(-1, 2)[:, 1] = self.exact_two(np.arange(P2 * U * U))
        if int(bad.item()):
            raise FrontierError("frontier: hardness must be finite and within [0, 1]")
        self._dev = (out2, out3[:P3])
        self._two = self._three = None

    def exact_two(self, flat):
        """numpy-exact two-stage fidelities (hadis_fid_exact: the pairwise mean of
        where(h > theta | s_i < tau, c_j, c_i)) for flat indices into ``two``."""
        torch = _lib.torch_cuda()
        d_h, d_s, params, n, U, M = self._d
        flat = np.asarray(flat, dtype=np.int64)
        pairs = np.array([(i, j) for i in range(M) for j in range(i + 1, M)], dtype=np.int64)
        pr, a, b = flat // (U * U), flat // U % U, flat % U
        li, hj = pairs[pr, 0], pairs[pr, 1]
        u = np.asarray(self.unique)
        dev = d_h.device
        slot = torch.from_numpy(li.astype(np.int32)).to(dev)
        th = torch.from_numpy(u[a]).to(dev)
        ta = torch.from_numpy(u[b]).to(dev)
        cp = torch.from_numpy(np.stack([params[li, 1], params[li, 2], params[hj, 1],
                                        params[hj, 2]], axis=1)).to(dev)
        fid = torch.empty(flat.size, dtype=torch.float64, device=dev)
        if flat.size:
            p = _lib.ptr
            _lib.check(_lib.load().hadis_fid_exact(p(d_h), p(d_s), n, int(flat.size), p(slot),
                                                   p(th), p(ta), p(cp), p(fid),
                                                   _lib.stream_handle()), "hadis_fid_exact")
        return fid

    @property
    def two(self):
        if self._two is None:
            self._two = self._dev[0].cpu().numpy()
        return self._two

    @property
    def three(self):
        if self._three is None:
            self._three = self._dev[1].cpu().numpy()
        return self._three

    def hull_candidates(self, which, exact_two=False):
        """(lat, fid) of the points that can be lower-envelope vertices: the
        left and right Pareto staircases (hadis_pareto_prune on (lat, fid) and
        (-lat, fid)); every other point is beaten in fidelity from both sides
        and lies strictly above the envelope."""
        torch = _lib.torch_cuda()
        pts = self._dev[0 if which == 2 else 1].reshape(-1, 2)
        lat, fid = pts[:, 0].contiguous(), pts[:, 1].contiguous()
        lib = _lib.load()
        n = int(lat.numel())
        ws_bytes = lib.hadis_pareto_workspace_bytes(n)
        ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=lat.device)
        keep = []
        for x in (lat, -lat):
            idx = torch.empty(n, dtype=torch.int64, device=lat.device)
            cnt = torch.zeros(1, dtype=torch.int64, device=lat.device)
            _lib.check(lib.hadis_pareto_prune(_lib.ptr(x), _lib.ptr(fid), n, _lib.ptr(idx),
                                              _lib.ptr(cnt), _lib.ptr(ws), ws_bytes,
                                              _lib.stream_handle()), "hadis_pareto_prune")
            keep.append(idx[:int(cnt.item())])
        sel = torch.unique(torch.cat(keep))
        f = fid[sel]
        if which == 2 and exact_two:
            f = self.exact_two(sel.cpu().numpy())
        return lat[sel].cpu().numpy(), f.cpu().numpy()

    def two_points(self):
        vs, thr, r = self.variants, self.thresholds, self.rank
        out, p = [], 0
        for i in range(len(vs)):
            for j in range(i + 1, len(vs)):
                for a, theta in zip(r, thr):
                    for b, tau in zip(r, thr):
                        lat, fid = self.two[p, a, b]
                        out.append(FrontierPoint(float(lat), float(fid),
                                                 (vs[i].id, vs[j].id, theta, tau)))
                p += 1
        return out

    def three_points(self):
        vs, thr, r = self.variants, self.thresholds, self.rank
        out, t = [], 0
        M = len(vs)
        for i in range(M):
            for j in range(i + 1, M):
                for k in range(j + 1, M):
                    for a, theta in zip(r, thr):
                        for b, t1 in zip(r, thr):
                            for c, t2 in zip(r, thr):
                                lat, fid = self.three[t, a, b, c]
                                out.append(FrontierPoint(float(lat), float(fid),
                                                         (vs[i].id, vs[j].id, vs[k].id,
                                                          theta, t1, t2)))
                    t += 1
        return out


def two_stage_points(variants, h: np.ndarray, thresholds=THRESHOLDS) -> list:
    """frontier.py:60-85 on the GPU."""
    if len(variants) < 2:
        raise FrontierError("two_stage_points: need at least two variants")
    return CascadePoints(variants, h, thresholds).two_points()


def three_stage_points(variants, h: np.ndarray, thresholds=THRESHOLDS) -> list:
    """frontier.py:88-120 on the GPU."""
    if len(variants) < 3:
        raise FrontierError("three_stage_points: need at least three variants")
    return CascadePoints(variants, h, thresholds).three_points()


def _hull_xy(x, y):
    """Lower convex hull (frontier.py:123-143 semantics) of point arrays:
    lowest y per x, then a monotone chain dropping vertices on or above the
    chord.  Points beaten in y from both sides (a lower-or-equal x with smaller
    y and a greater-or-equal x with smaller y) are strictly above the hull and
    are filtered out first."""
    x = np.asarray(x, dtype=np.float64).ravel()
    y = np.asarray(y, dtype=np.float64).ravel()
    if x.size == 0:
        raise FrontierError("lower_envelope: no points")
    order = np.lexsort((y, x))
    x, y = x[order], y[order]
    first = np.ones(x.size, dtype=bool)
    first[1:] = x[1:] != x[:-1]
    x, y = x[first], y[first]
    left = np.minimum.accumulate(np.concatenate(([np.inf], y[:-1])))
    right = np.minimum.accumulate(np.concatenate((y[1:], [np.inf]))[::-1])[::-1]
    keep = (y < left) | (y < right)
    keep[0] = keep[-1] = True
    hull = []
    for px, py in zip(x[keep].tolist(), y[keep].tolist()):
        while len(hull) >= 2:
            (x1, y1), (x2, y2) = hull[-2], hull[-1]
            if (y2 - y1) * (px - x1) >= (py - y1) * (x2 - x1):
                hull.pop()
            else:
                break
        hull.append((px, py))
    return hull


def lower_envelope(points) -> list:
    """Lower convex hull of (latency, fidelity) points, vertices left to right."""
    pts = list(points)
    if not pts:
        raise FrontierError("lower_envelope: no points")
    return _hull_xy([p.latency_s for p in pts], [p.fidelity_cost for p in pts])


def envelope_value(hull, x: float) -> float:
    """Piecewise-linear value of a hull at x (inf outside its range)."""
    if x < hull[0][0] or x > hull[-1][0]:
        return math.inf
    xs = [a for a, _ in hull]
    i = int(np.searchsorted(xs, x, side="left"))
    if i < len(hull) and hull[i][0] == x:
        # a breakpoint: the segment ending here is evaluated first in the reference
        if i > 0:
            (x1, y1), (x2, y2) = hull[i - 1], hull[i]
            return min(y1, y2) if x2 == x1 else y1 + (y2 - y1) * (x - x1) / (x2 - x1)
        if len(hull) > 1:
            (x1, y1), (x2, y2) = hull[0], hull[1]
            return min(y1, y2) if x2 == x1 else y1 + (y2 - y1) * (x - x1) / (x2 - x1)
        return hull[0][1]
    (x1, y1), (x2, y2) = hull[i - 1], hull[i]
    return y1 + (y2 - y1) * (x - x1) / (x2 - x1)


def envelope_gap(hull_a, hull_b) -> float:
    """max over the shared-range breakpoints of a(x) - b(x)."""
    lo = max(hull_a[0][0], hull_b[0][0])
    hi = min(hull_a[-1][0], hull_b[-1][0])
    if hi < lo:
        return 0.0
    xs = sorted({x for x, _ in hull_a} | {x for x, _ in hull_b} | {lo, hi})
    return max(envelope_value(hull_a, x) - envelope_value(hull_b, x)
               for x in xs if lo <= x <= hi)


def frontier_compare(catalog, h: np.ndarray | None = None, thresholds=THRESHOLDS,
                     exact: bool = True) -> FrontierReport:
    """Compare two-stage and three-stage frontiers on one hardness population
    (frontier.py:171-188)."""
    if h is None:
        h = default_hardness()
    variants = catalog.sorted_by_latency()
    if len(variants) < 2:
        raise FrontierError("two_stage_points: need at least two variants")
    if len(variants) < 3:
        raise FrontierError("three_stage_points: need at least three variants")
    # exact two-stage fidelities only where they matter: the envelope candidates
    cp = CascadePoints(variants, h, thresholds, exact=False)
    env2 = _hull_xy(*cp.hull_candidates(2, exact_two=exact))
    env3 = _hull_xy(*cp.hull_candidates(3))
    K = len(cp.thresholds)
    M = len(cp.variants)
    return FrontierReport(gap=envelope_gap(env2, env3), envelope_two=tuple(env2),
                          envelope_three=tuple(env3), n_two=M * (M - 1) // 2 * K * K,
                          n_three=M * (M - 1) * (M - 2) // 6 * K ** 3)
