"""Offline cascade profiling on the GPU: drop-in for cascadesim.profiler.

Public surface (same names, signatures, return types and error behaviour as
pkg/src/cascadesim/profiler.py):

* ``THRESHOLD_GRID``, ``ProfileError``, ``CascadeRow``, ``TableProvenance``,
  ``CascadeTable`` (profiler.py:30-98) -- field-compatible frozen dataclasses;
* ``profile_config(catalog, prompts, seed, noise_sigma, eps_latency,
  eps_quality, thresholds, weights)`` (profiler.py:107-186);
* ``prompts_hash`` / ``save_table`` / ``load_table`` (profiler.py:101-104,
  189-216), byte-identical JSON layout.

Added array-level entry points (no text needed):

* ``profile_records(pool_or_catalog, h, scores=None, noise=None, ...)`` --
  the same table from per-query records (hardness, light-model scores) that
  the reference derives from prompt text (profiler.py:125-137);
* ``GridProfiler`` -- keeps records resident in HBM and runs the device
  pipeline (K1 histogram, K2 scan, K3/K4 frontier) without host round trips.

What runs where: text -> records (SHA-256 keys, key sort, tokenizer,
lexicon features, hardness, the BLAKE2b noise digest) runs on the GPU
(text.py / csrc/text.cu) with Box-Muller's log/cos on the host libm;
scores are formed with the reference's numpy expression; everything from
the records onward -- bypass/reject counting, every grid cell, the Pareto
extraction and the (theta, tau) merge -- runs in libhadis_b200.so on the
GPU.  The reference package is not needed at run time.
"""

from __future__ import annotations

import hashlib
import json
import math
from collections.abc import Sequence
from dataclasses import asdict, dataclass

import numpy as np

from . import _lib
from .catalog import catalog_hash, select_candidates
from .text import check_weights, prompts_hash_sorted, text_records

THRESHOLD_GRID = tuple(i / 10 for i in range(11))
DEFAULT_NOISE_SIGMA = 0.05


class ProfileError(ValueError):
    pass


@dataclass(frozen=True)
class CascadeRow:
    """One profiled operating point of a light/heavy cascade pair (profiler.py:37-61)."""

    light_id: str
    heavy_id: str
    theta: float
    tau: float
    r_light: float
    r_heavy: float
    fidelity_cost: float
    mean_latency_s: float

    @property
    def bypass_fraction(self) -> float:
        return 1.0 - self.r_light

    @property
    def reroute_fraction(self) -> float:
        return self.r_heavy - self.bypass_fraction

    def shares(self) -> dict:
        out = {self.light_id: self.r_light}
        out[self.heavy_id] = out.get(self.heavy_id, 0.0) + self.r_heavy
        return out


@dataclass(frozen=True)
class TableProvenance:
    catalog_hash: str
    prompts_hash: str
    n_prompts: int
    seed: int
    noise_sigma: float
    thresholds: tuple
    eps_latency: float
    eps_quality: float


@dataclass(frozen=True)
class CascadeTable:
    rows: tuple
    provenance: TableProvenance

    def pairs(self) -> list:
        seen = []
        for row in self.rows:
            pair = (row.light_id, row.heavy_id)
            if pair not in seen:
                seen.append(pair)
        return sorted(seen)

    def rows_for_pair(self, light_id: str, heavy_id: str) -> list:
        return [r for r in self.rows if r.light_id == light_id and r.heavy_id == heavy_id]

    def find_row(self, light_id, heavy_id, theta, tau) -> CascadeRow:
        for r in self.rows_for_pair(light_id, heavy_id):
            if abs(r.theta - theta) < 1e-12 and abs(r.tau - tau) < 1e-12:
                return r
        raise ProfileError(f"row-not-found: {light_id}/{heavy_id} theta={theta} tau={tau}")


# ----------------------------------------------------------------- hashing

def stable_text_key(text: str) -> int:
    """63-bit SHA-256 prompt key (seeds.py:49-55)."""
    return int.from_bytes(hashlib.sha256(text.encode("utf-8")).digest()[:8], "big") >> 1


def prompts_hash(prompts) -> str:
    """Order-free hash of a prompt population (profiler.py:101-104)."""
    blob = "\x1f".join(sorted(prompts, key=stable_text_key)).encode("utf-8")
    return hashlib.sha256(blob).hexdigest()[:16]


# ------------------------------------------------------------- table I/O

def save_table(table: CascadeTable, path: str) -> None:
    """JSON layout of profiler.py:189-196 (indent=1, sort_keys, trailing newline)."""
    doc = {"provenance": asdict(table.provenance), "rows": [asdict(r) for r in table.rows]}
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(doc, fh, indent=1, sort_keys=True)
        fh.write("\n")


def load_table(path: str, catalog=None, override_provenance: bool = False) -> CascadeTable:
    """Reader with the provenance gate of profiler.py:199-216."""
    with open(path, "r", encoding="utf-8") as fh:
        doc = json.load(fh)
    try:
        prov = dict(doc["provenance"])
        prov["thresholds"] = tuple(prov["thresholds"])
        provenance = TableProvenance(**prov)
        rows = tuple(CascadeRow(**r) for r in doc["rows"])
    except (KeyError, TypeError) as exc:
        raise ProfileError(f"table file: malformed ({exc})") from None
    if catalog is not None:
        current = catalog_hash(catalog)
        if provenance.catalog_hash != current and not override_provenance:
            raise ProfileError(
                "provenance-mismatch: table was profiled against catalog "
                f"{provenance.catalog_hash}, current catalog is {current}; "
                "pass override_provenance to use it anyway")
    return CascadeTable(rows=rows, provenance=provenance)


# ------------------------------------------------------ grid description

def _light_first(v):
    return (v.latency_s[1], v.id)


@dataclass(frozen=True)
class GridSpec:
    """Threshold list as given plus its sorted distinct values.

    ``first_pos[r]`` is the first position of the r-th smallest distinct
    value -- the representative the reference's index tie-break keeps."""

    thresholds: tuple
    unique: tuple
    first_pos: tuple

    @staticmethod
    def build(thresholds) -> "GridSpec":
        thr = tuple(float(t) for t in thresholds)
        if not thr:
            raise ProfileError("profile_config: empty threshold grid")
        if any(math.isnan(t) for t in thr):
            raise ProfileError("profile_config: NaN thresholds are not supported")
        first = {}
        for i, t in enumerate(thr):
            first.setdefault(t, i)   # -0.0 and 0.0 share one key, as in the reference's dict
        uniq = tuple(sorted(first))
        return GridSpec(thr, uniq, tuple(first[u] for u in uniq))


def light_scores(pool, h, noise):
    """Discriminator scores of every light-capable pool model (profiler.py:134-137),
    rows in pool latency order (the heaviest model is never a light stage)."""
    h = np.asarray(h, dtype=np.float64)
    noise = np.asarray(noise, dtype=np.float64)
    out = np.empty((len(pool) - 1, h.shape[0]), dtype=np.float64)
    for i, v in enumerate(pool[:-1]):
        a, s = v.accept_params
        out[i] = np.clip(1.0 / (1.0 + np.exp(-(a - s * h))) + noise, 0.0, 1.0)
    return out


def pair_list(pool):
    return [(i, j) for i in range(len(pool)) for j in range(i + 1, len(pool))]


def pair_params(pool, pairs):
    rows = []
    for i, j in pairs:
        lt, hv = pool[i], pool[j]
        rows.append((lt.latency_s[1], hv.latency_s[1], lt.base_quality_cost, lt.hardness_penalty,
                     hv.base_quality_cost, hv.hardness_penalty))
    return np.asarray(rows, dtype=np.float64).reshape(len(pairs), _lib.PAIR_PARAMS)


# --------------------------------------------------------- device pipeline

@dataclass
class DeviceTable:
    """Raw device output of one profiling run (rows in pair-major (theta, tau) order)."""

    pairs: list          # (light pool index, heavy pool index) per local pair id
    n_rows: int
    pair_rows: list      # rows per local pair
    pair: object         # torch int32 [rows]
    theta_pos: object
    tau_pos: object
    r_light: object      # torch float64 [rows]
    r_heavy: object
    fid: object
    lat: object
    stats: dict


class ProfilePlan:
    """Device-resident description of one (threshold grid, pair set) job:
    sorted distinct thresholds, first positions, pair slots/parameters and the
    output/workspace capacities learned from previous runs."""

    def __init__(self, prof, thresholds, pairs):
        torch = prof.torch
        dev = prof.device
        self.grid = GridSpec.build(thresholds)
        self.pairs = pair_list(prof.pool) if pairs is None else list(pairs)
        if not self.pairs:
            raise ProfileError("profile_records: no pairs to profile")
        rows = sorted({prof.row_of(i) for i, _ in self.pairs})     # score rows used
        self.slot0 = rows[0]
        self.n_light = rows[-1] - rows[0] + 1
        self.U = len(self.grid.unique)
        self.P = len(self.pairs)
        self.d_u = torch.tensor(self.grid.unique, dtype=torch.float64, device=dev)
        self.d_first = torch.tensor(self.grid.first_pos, dtype=torch.int32, device=dev)
        self.d_slot = torch.tensor([prof.row_of(i) - self.slot0 for i, _ in self.pairs],
                                   dtype=torch.int32, device=dev)
        self.d_params = torch.from_numpy(pair_params(prof.pool, self.pairs)).to(dev)
        cells = self.U * self.U * self.P
        cand = int(min(cells, max(1 << 20, cells // 8)))
        self.caps = (cand, 2048, int(min(cells, cand + self.U * self.P)))
        self.cells = cells


def grow_caps(plan, caps, stats, out_limit=None):
    """Capacities after an overflow reported in ``stats`` (hadis_frontier_stat),
    or ProfileError for the hard limits.  ``out_limit`` caps the output rows
    (a multi-GPU slab); None = the grid's cell count."""
    of = stats[_lib.ST_OVERFLOW]
    if of & 128:
        raise ProfileError("profile_records: more than 65 pool models per light stage "
                           "is not supported")
    if of & 2:
        raise ProfileError("profile_records: too many exactness-critical cells "
                           f"({stats[_lib.ST_EXACT_CELLS]}); reduce the grid")
    cand_cap, exact_cap, out_cap = caps
    cells = plan.cells
    if of & 16:                   # candidate list
        cand_cap = int(min(cells, max(cand_cap * 4, stats[_lib.ST_CANDIDATES] + 1)))
    if of & (8 | 16):             # output rows (bounded by candidates + nobypass rows)
        out_cap = int(min(cells, max(out_cap * 2, cand_cap + plan.U * plan.P,
                                     stats[_lib.ST_ROWS] + 1)))
        if out_limit is not None:
            out_cap = min(out_cap, out_limit)
    if of & (4 | 32 | 64):        # uncertain decisions / exact requests overflowed
        need = max(stats[_lib.ST_UNCERTAIN], stats[_lib.ST_EXACT_CELLS]) + 1
        exact_cap = int(min(cells * 2, max(exact_cap * 4, need)))
    if (cand_cap, exact_cap, out_cap) == tuple(caps):
        raise ProfileError(f"profile_records: capacity overflow {of:#x} cannot grow")
    return (cand_cap, exact_cap, out_cap)


class GridProfiler:
    """Records resident in HBM + the K1..K4 device pipeline.

    ``h`` is float64[N] and ``scores`` float64[L, N] (row i = pool model i as
    the light stage), both in ``stable_text_key`` order and already on the
    device (torch tensors) or host arrays copied once at construction.
    ``run`` profiles one threshold grid; ``launch``/``finish`` split it into an
    asynchronous enqueue and a synchronising check for pipelined callers."""

    def __init__(self, pool, h, scores, device=None, layout="bucketed", slots=None):
        torch = _lib.torch_cuda()
        self.torch = torch
        self.pool = list(pool)
        if len(self.pool) < 2:
            raise ProfileError("profile_config: need at least two candidate variants")
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.h = torch.as_tensor(h, dtype=torch.float64, device=self.device).contiguous()
        self.scores = torch.as_tensor(scores, dtype=torch.float64, device=self.device).contiguous()
        self.n = int(self.h.shape[0])
        if self.n == 0:
            raise ProfileError("profile_config: empty prompt population")
        # slots: pool light index of each score row when scores hold a subset
        # of the light models (a multi-GPU shard); default row i = pool model i
        self.slots = None if slots is None else [int(x) for x in slots]
        want_rows = len(self.pool) - 1 if self.slots is None else len(self.slots)
        if self.scores.dim() != 2 or self.scores.shape[1] != self.n or \
                self.scores.shape[0] < want_rows:
            raise ProfileError("profile_records: scores must be [n_models - 1, n_records]")
        self._row_of = None if self.slots is None else {m: r for r, m in enumerate(self.slots)}
        self.lib = _lib.load()
        self.shift = self.lib.hadis_hfix_shift(self.n)
        self._ws = None
        self._plans = {}
        if layout not in ("bucketed", "original"):
            raise ValueError("layout must be 'bucketed' or 'original'")
        self.layout = layout
        self.bad = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._stats_pin = None
        self._store = None
        self.sink = None        # sharding.ShardSlab: emit rows into a multi-GPU slab

    def row_of(self, light_index: int) -> int:
        """Score row holding pool model ``light_index`` as the light stage."""
        if self._row_of is None:
            return light_index
        try:
            return self._row_of[light_index]
        except KeyError:
            raise ProfileError(f"profile_records: no score row for light model {light_index}") \
                from None

    def _bucket_store(self, n_light):
        """Row-bucketed record store buffers (hfix u64[n], bs u16 model quads, row plan)."""
        torch = self.torch
        st = self._store
        elems = self.lib.hadis_bs_store_elems(self.n, n_light)
        if st is None or st[1].numel() < elems:
            st = self._store = (torch.empty(self.n, dtype=torch.int64, device=self.device),
                                torch.empty(elems, dtype=torch.int16, device=self.device),
                                torch.empty(self.lib.hadis_row_plan_bytes(1), dtype=torch.uint8,
                                            device=self.device))
        return st

    def plan(self, thresholds=THRESHOLD_GRID, pairs=None) -> ProfilePlan:
        key = (tuple(float(t) for t in thresholds), None if pairs is None else tuple(pairs))
        pl = self._plans.get(key)
        if pl is None:
            pl = self._plans[key] = ProfilePlan(self, thresholds, pairs)
        return pl

    def run(self, thresholds=THRESHOLD_GRID, pairs=None, exact_fid=False, stream=None):
        """Profile ``pairs`` (default: every light<heavy pair); returns a DeviceTable."""
        return self.finish(self.launch(self.plan(thresholds, pairs), exact_fid, stream))

    def launch(self, plan: ProfilePlan, exact_fid=False, stream=None, events=None):
        """See ``_launch``; runs with ``self.device`` current (kernels and the
        default stream belong to the profiler's device, not the caller's)."""
        with self.torch.cuda.device(self.device):
            return self._launch(plan, exact_fid, stream, events)

    def _launch(self, plan: ProfilePlan, exact_fid=False, stream=None, events=None):
        """Enqueue B (row-bucketed record store), K1 (histogram), K2 (2-D scan)
        and K3/K4 (frontier) on ``stream``; no host synchronisation.  ``events``
        (optional list of 6 torch.cuda.Event) brackets B0-B2 | B3 | K1 | K2 | K3+K4."""
        torch = self.torch
        dev = self.device
        st = _lib.stream_handle(stream, dev)
        bins = (plan.U + 1) * (plan.U + 1) * plan.n_light
        # stream None = the current stream at launch time (a captured graph
        # replays on whichever stream is current then, so keep None)
        state = dict(plan=plan, exact_fid=exact_fid, stream=stream,
                     scanned=torch.empty((plan.U + 1) * plan.n_light, dtype=torch.uint8,
                                         device=dev),
                     cnt=torch.empty(bins, dtype=torch.int32, device=dev),
                     hsum=torch.empty(bins, dtype=torch.int64, device=dev),
                     scores=self.scores[plan.slot0:plan.slot0 + plan.n_light])
        p = _lib.ptr
        ev_stream = stream if stream is not None else torch.cuda.current_stream(dev)
        rec = (lambda i: events[i].record(ev_stream)) if events is not None else (lambda i: None)
        rec(0)
        if self.layout == "bucketed" and plan.U < 2048:
            hfix, bs, rplan = self._bucket_store(plan.n_light)
            _lib.check(self.lib.hadis_records_plan(
                p(self.h), self.n, p(plan.d_u), plan.U, self.shift, p(self.bad), p(rplan),
                rplan.numel(), st), "hadis_records_plan")
            rec(1)
            _lib.check(self.lib.hadis_records_scatter(
                p(self.h), p(state["scores"]), self.n, plan.n_light, p(plan.d_u), plan.U,
                self.shift, p(hfix), p(bs), p(rplan), rplan.numel(), st), "hadis_records_scatter")
            rec(2)
            _lib.check(self.lib.hadis_bin_hist_rows(
                p(hfix), p(bs), self.n, plan.n_light, plan.U, p(rplan), p(state["cnt"]),
                p(state["hsum"]), p(state["scanned"]), st), "hadis_bin_hist_rows")
            scanned = state["scanned"]
        else:
            rec(1)
            rec(2)
            _lib.check(self.lib.hadis_bin_hist(p(self.h), p(state["scores"]), self.n, plan.n_light,
                                               p(plan.d_u), plan.U, self.shift, p(state["cnt"]),
                                               p(state["hsum"]), p(self.bad), st), "hadis_bin_hist")
            scanned = None
        rec(3)
        _lib.check(self.lib.hadis_hist_scan(p(state["cnt"]), p(state["hsum"]), plan.n_light,
                                            plan.U, p(scanned), st), "hadis_hist_scan")
        rec(4)
        self._frontier(state, plan.caps)
        rec(5)
        return state

    def graph(self, plan: ProfilePlan, exact_fid=False):
        """Capture the whole device pipeline of ``plan`` (B0..F14, ~40 kernels
        and memsets) into one CUDA graph.  An eager run first learns the
        output capacities; ``replay()`` relaunches the graph and returns the
        DeviceTable (a capacity overflow falls back to an eager rerun inside
        ``finish`` and the graph is re-captured on the next call).
        ``replay.launch()`` / ``replay.state`` expose the asynchronous half
        for pipelined callers (TablePipeline)."""
        torch = self.torch
        self.finish(self.launch(plan, exact_fid))          # learn capacities, allocate
        torch.cuda.synchronize(self.device)
        prof = self

        class Replay:
            def __init__(self):
                self.caps = None
                self.capture()

            def capture(self):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.device(prof.device), torch.cuda.graph(g):
                    state = prof.launch(plan, exact_fid)
                # the graph bakes in raw pointers: own every buffer it touches
                # (the profiler may reallocate its workspace / record store later)
                self.graph, self.state, self.caps = g, state, plan.caps
                self.buffers = (prof._ws, prof._store, prof.h, prof.scores, prof.bad)

            def launch(self):
                """Enqueue one replay on the current stream (no host sync)."""
                if self.caps != plan.caps:
                    self.capture()
                with torch.cuda.device(prof.device):
                    self.graph.replay()
                return self.state

            def __call__(self):
                return prof.finish(self.launch())

        return Replay()

    def _frontier(self, state, caps):
        torch = self.torch
        plan = state["plan"]
        cand_cap, exact_cap, out_cap = caps
        U, P = plan.U, plan.P
        ws_bytes = self.lib.hadis_frontier_workspace_bytes(P, U, cand_cap, exact_cap, out_cap)
        if ws_bytes == 0:
            raise ProfileError("profile_records: invalid frontier sizes")
        if self._ws is None or self._ws.numel() < ws_bytes:
            self._ws = torch.empty(ws_bytes, dtype=torch.uint8, device=self.device)
        dev = self.device
        if self.sink is not None:           # rows go straight into a multi-GPU slab
            out, stats = self.sink.columns(out_cap), self.sink.stats(P)
            stats.zero_()
        else:
            out = dict(pair=torch.empty(out_cap, dtype=torch.int32, device=dev),
                       theta_pos=torch.empty(out_cap, dtype=torch.int32, device=dev),
                       tau_pos=torch.empty(out_cap, dtype=torch.int32, device=dev),
                       r_light=torch.empty(out_cap, dtype=torch.float64, device=dev),
                       r_heavy=torch.empty(out_cap, dtype=torch.float64, device=dev),
                       fid=torch.empty(out_cap, dtype=torch.float64, device=dev),
                       lat=torch.empty(out_cap, dtype=torch.float64, device=dev))
            stats = torch.zeros(_lib.ST_PAIR0 + P + 1, dtype=torch.int64, device=dev)  # + bad
        p = _lib.ptr
        args = (p(state["cnt"]), p(state["hsum"]), self.n, U, self.shift, P, p(plan.d_slot),
                p(plan.d_params), p(plan.d_first), len(plan.grid.thresholds), p(plan.d_u),
                p(self.h), p(state["scores"]), 1 if state["exact_fid"] else 0, p(self._ws),
                ws_bytes, cand_cap, exact_cap, out_cap)
        if self.sink is not None:           # compact rows (the merge rebuilds the rest)
            _lib.check(self.lib.hadis_pair_frontiers_compact(
                *args, p(out["theta_pos"]), p(out["tau_pos"]), p(out["n_light"]),
                p(out["n_heavy"]), p(out["fid"]), p(stats),
                _lib.stream_handle(state["stream"], self.device)), "hadis_pair_frontiers_compact")
        else:
            _lib.check(self.lib.hadis_pair_frontiers(
                *args, p(out["pair"]), p(out["theta_pos"]), p(out["tau_pos"]), p(out["r_light"]),
                p(out["r_heavy"]), p(out["fid"]), p(out["lat"]), p(stats),
                _lib.stream_handle(state["stream"], self.device)), "hadis_pair_frontiers")
        # the record-validation flag rides along, so finish() needs one device read
        with torch.cuda.stream(state["stream"] or torch.cuda.current_stream(self.device)):
            stats[-1:].copy_(self.bad)
        state.update(out=out, stats=stats, caps=caps)

    def finish(self, state) -> DeviceTable:
        """Synchronise, check device-side status, grow capacities and rerun if needed."""
        with self.torch.cuda.device(self.device):
            return self._finish(state)

    def _finish(self, state) -> DeviceTable:
        plan = state["plan"]
        for _ in range(6):
            dev_stats = state["stats"]
            pin = self._stats_pin
            if pin is None or pin.numel() < dev_stats.numel():
                pin = self._stats_pin = self.torch.empty(dev_stats.numel(),
                                                         dtype=self.torch.int64).pin_memory()
            st = state["stream"] or self.torch.cuda.current_stream(self.device)
            with self.torch.cuda.stream(st):
                pin[:dev_stats.numel()].copy_(dev_stats, non_blocking=True)
            st.synchronize()
            stats = pin[:dev_stats.numel()].tolist()
            if stats[-1]:
                raise ProfileError("profile_records: hardness must be finite and within [0, 1]")
            if stats[_lib.ST_OVERFLOW] == 0:
                break
            plan.caps = grow_caps(plan, state["caps"], stats)
            self._frontier(state, plan.caps)
        else:
            raise ProfileError("profile_records: capacity retries exhausted")
        n_rows = stats[_lib.ST_ROWS]
        out = state["out"]
        col = (lambda f: out[f][:n_rows] if f in out else None)   # slab sinks hold compact rows
        return DeviceTable(
            pairs=plan.pairs, n_rows=n_rows,
            pair_rows=stats[_lib.ST_PAIR0:_lib.ST_PAIR0 + plan.P],
            pair=col("pair"), theta_pos=col("theta_pos"), tau_pos=col("tau_pos"),
            r_light=col("r_light"), r_heavy=col("r_heavy"), fid=col("fid"), lat=col("lat"),
            stats={"rows": n_rows, "candidates": stats[_lib.ST_CANDIDATES],
                   "uncertain": stats[_lib.ST_UNCERTAIN],
                   "exact_cells": stats[_lib.ST_EXACT_CELLS]})


class TablePipeline:
    """Streaming table builds for a sequence of record sets (re-profiling
    sweeps): host records in, host row arrays out, double-buffered so that
    the H2D copy of set i, the device build of set i-1 and the D2H copy of
    set i-2's rows run concurrently (PCIe is full duplex; the build is one
    CUDA graph).  Every record set must have the same shape (n, light rows).

    Rows land in pinned host buffers owned by the set's slot (two slots);
    ``run(inputs, on_rows)`` hands each set's rows to ``on_rows(i, rows)``
    once their copy has completed -- ``rows`` maps FIELDS to pinned tensors
    that stay valid until the same slot's next set finishes (two sets later),
    so the callback must consume or copy them."""

    FIELDS = ("pair", "theta_pos", "tau_pos", "r_light", "r_heavy", "fid", "lat")

    def __init__(self, pool, n, n_rows_scores, thresholds, pairs=None, device=None,
                 score_slots=None):
        """score_slots: pool light index of each score row when the record sets
        carry only some light models' scores (a multi-GPU shard)."""
        torch = _lib.torch_cuda()
        self.torch = torch
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.slots = []
        with torch.cuda.device(self.device):
            for _ in range(2):
                d_h = torch.zeros(n, dtype=torch.float64, device=self.device)
                d_sc = torch.zeros((n_rows_scores, n), dtype=torch.float64, device=self.device)
                prof = GridProfiler(pool, d_h, d_sc, device=self.device, slots=score_slots)
                self.slots.append(dict(h=d_h, sc=d_sc, prof=prof,
                                       plan=prof.plan(thresholds, pairs), replay=None,
                                       ev_in=torch.cuda.Event(), ev_comp=torch.cuda.Event(),
                                       ev_out=torch.cuda.Event(), busy=False, out={},
                                       stats_pin=torch.zeros(_lib.ST_PAIR0 + 1,
                                                             dtype=torch.int64).pin_memory(),
                                       bad_pin=torch.zeros(1, dtype=torch.int32).pin_memory()))
            self.s_in = torch.cuda.Stream(device=self.device)
            self.s_comp = torch.cuda.Stream(device=self.device)
            self.s_out = torch.cuda.Stream(device=self.device)

    def warm(self, h_pin, sc_pin):
        """First build of both slots on these records (learns capacities, captures graphs)."""
        with self.torch.cuda.device(self.device):
            for sl in self.slots:
                sl["h"].copy_(h_pin)
                sl["sc"][:sc_pin.shape[0]].copy_(sc_pin)
                sl["replay"] = sl["prof"].graph(sl["plan"])
            self.torch.cuda.synchronize(self.device)

    def _out_buffers(self, sl, n_rows):
        bufs = sl["out"]
        for f in self.FIELDS:
            v = sl["replay"].state["out"][f]
            buf = bufs.get(f)
            if buf is None or buf.numel() < n_rows:
                bufs[f] = self.torch.empty(max(n_rows, 1), dtype=v.dtype).pin_memory()
        return bufs

    def run(self, inputs, on_rows=None):
        """inputs: list of (h_pin, sc_pin) pinned host tensors.  Returns the
        per-set (set index, n_rows, d2h bytes); rows go to ``on_rows``."""
        with self.torch.cuda.device(self.device):
            return self._run(inputs, on_rows)

    def _run(self, inputs, on_rows):
        torch = self.torch
        done = []
        pending = []                                    # (slot index, set index, n_rows)

        def deliver(k, i, n_rows):
            sl = self.slots[k]
            sl["ev_out"].synchronize()
            if on_rows is not None:
                on_rows(i, {f: sl["out"][f][:n_rows] for f in self.FIELDS})

        def finalize(k, i):
            sl = self.slots[k]
            sl["ev_stats"].synchronize()
            stats = sl["stats_pin"].tolist()
            if int(sl["bad_pin"][0]):
                raise ProfileError("profile_records: hardness must be finite and within [0, 1]")
            if stats[_lib.ST_OVERFLOW]:
                raise ProfileError("TablePipeline: capacity overflow; rebuild with warm()")
            n_rows = stats[_lib.ST_ROWS]
            if len(pending) == 2:                        # this slot's previous set: hand it out
                deliver(*pending.pop(0))
            bufs = self._out_buffers(sl, n_rows)
            nbytes = 0
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(sl["ev_comp"])
                for f in self.FIELDS:
                    v = sl["replay"].state["out"][f][:n_rows]
                    bufs[f][:n_rows].copy_(v, non_blocking=True)
                    nbytes += n_rows * v.element_size()
                sl["ev_out"].record(self.s_out)
            pending.append((k, i, n_rows))
            return n_rows, nbytes

        launched = None                                  # (slot index, set index)
        for i, (h_pin, sc_pin) in enumerate(inputs):
            k = i % 2
            sl = self.slots[k]
            with torch.cuda.stream(self.s_in):
                if sl["busy"]:
                    self.s_in.wait_event(sl["ev_comp"])    # the slot's last build read its inputs
                sl["h"].copy_(h_pin, non_blocking=True)
                sl["sc"][:sc_pin.shape[0]].copy_(sc_pin, non_blocking=True)
                sl["ev_in"].record(self.s_in)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(sl["ev_in"])
                if sl["busy"]:
                    self.s_comp.wait_event(sl["ev_out"])  # its previous rows are copied out
                state = sl["replay"].launch()
                sl["ev_comp"].record(self.s_comp)
                sl["stats_pin"][:].copy_(state["stats"][:_lib.ST_PAIR0 + 1], non_blocking=True)
                sl["bad_pin"].copy_(sl["prof"].bad, non_blocking=True)
                sl["ev_stats"] = torch.cuda.Event()
                sl["ev_stats"].record(self.s_comp)
            sl["busy"] = True
            if launched is not None:
                done.append((launched[1],) + finalize(*launched))
            launched = (k, i)
        if launched is not None:
            done.append((launched[1],) + finalize(*launched))
        while pending:
            deliver(*pending.pop(0))
        return done


class CascadeRows(Sequence):
    """The rows of a profiled table, kept columnar (numpy) and turned into
    ``CascadeRow`` objects only when accessed -- an 11M-row c4 table costs one
    D2H copy instead of 11M Python objects.  Behaves as the reference's
    ``tuple[CascadeRow, ...]`` (profiler.py:92-98): len, indexing, slicing,
    iteration, equality with any sequence of rows, hashing; a row fetched
    twice is the same object (plans refer to table rows by identity)."""

    def __init__(self, ids, pair, theta_pos, tau_pos, r_light, r_heavy, fid, lat, thresholds):
        self._ids = list(ids)               # (light_id, heavy_id) per pair id
        self._cols = (np.asarray(pair), np.asarray(theta_pos), np.asarray(tau_pos),
                      np.asarray(r_light, dtype=np.float64),
                      np.asarray(r_heavy, dtype=np.float64),
                      np.asarray(fid, dtype=np.float64), np.asarray(lat, dtype=np.float64))
        self._thr = tuple(float(t) for t in thresholds)
        self._cache = {}

    def __len__(self):
        return int(self._cols[0].shape[0])

    def _row(self, i):
        row = self._cache.get(i)
        if row is None:
            p, a, b, x1, x2, f, m = (c[i] for c in self._cols)
            lid, hid = self._ids[int(p)]
            row = self._cache[i] = CascadeRow(
                light_id=lid, heavy_id=hid, theta=self._thr[int(a)], tau=self._thr[int(b)],
                r_light=float(x1), r_heavy=float(x2), fidelity_cost=float(f),
                mean_latency_s=float(m))
        return row

    def __getitem__(self, i):
        if isinstance(i, slice):
            return tuple(self._row(j) for j in range(*i.indices(len(self))))
        n = len(self)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError("row index out of range")
        return self._row(i)

    def __iter__(self):
        n = len(self)
        step = 1 << 16
        for s0 in range(0, n, step):
            chunk = [c[s0:s0 + step].tolist() for c in self._cols]
            for j, (p, a, b, x1, x2, f, m) in enumerate(zip(*chunk)):
                row = self._cache.get(s0 + j)
                if row is None:
                    lid, hid = self._ids[p]
                    row = CascadeRow(light_id=lid, heavy_id=hid, theta=self._thr[a],
                                     tau=self._thr[b], r_light=x1, r_heavy=x2,
                                     fidelity_cost=f, mean_latency_s=m)
                yield row

    def columns(self):
        """(pair ids, (light_id, heavy_id) per pair id, r_light, r_heavy, fid) as arrays."""
        return self._cols[0], self._ids, self._cols[3], self._cols[4], self._cols[5]

    def __eq__(self, other):
        if isinstance(other, CascadeRows):
            return (self._ids == other._ids and self._thr == other._thr and
                    all(np.array_equal(a, b) for a, b in zip(self._cols, other._cols)))
        if isinstance(other, (tuple, list, Sequence)) and not isinstance(other, str):
            return len(self) == len(other) and all(a == b for a, b in zip(self, other))
        return NotImplemented

    def __hash__(self):
        return hash(tuple(self))

    def __repr__(self):
        return f"CascadeRows({len(self)} rows)"


def rows_from_device(dt: DeviceTable, pool, thresholds, lazy=False):
    """Table rows (host) from a DeviceTable: a tuple of CascadeRow objects, or
    the columnar CascadeRows view (``lazy=True``, one D2H copy per column)."""
    cols = [getattr(dt, f).cpu().numpy() for f in ("pair", "theta_pos", "tau_pos", "r_light",
                                                    "r_heavy", "fid", "lat")]
    ids = [(pool[i].id, pool[j].id) for i, j in dt.pairs]
    rows = CascadeRows(ids, *cols, thresholds)
    return rows if lazy else tuple(rows)


def _pool_of(pool_or_catalog, eps_latency, eps_quality):
    if hasattr(pool_or_catalog, "variants"):
        pool = select_candidates(pool_or_catalog, eps_latency, eps_quality)
    else:
        pool = sorted(pool_or_catalog, key=_light_first)
    if len(pool) < 2:
        raise ProfileError("profile_config: need at least two candidate variants")
    return pool


def profile_records(pool_or_catalog, h, scores=None, noise=None, thresholds=THRESHOLD_GRID,
                    eps_latency=0.1, eps_quality=0.1, exact_fid=False, provenance=None,
                    lazy=True):
    """CascadeTable from per-query records (array-level profile_config).

    ``h``: hardness in [0, 1] per query; ``scores``: dict model id -> float64[N]
    or an array [n_pool - 1, N] (pool latency order); or ``noise`` to derive
    scores exactly as profiler.py:134-137.  Records must be in the order the
    reference would use (``stable_text_key`` order of the prompts) for
    ``exact_fid`` to be bitwise-identical; counts, latencies and membership do
    not depend on order.  ``lazy`` (default) keeps the rows columnar
    (``CascadeRows``: a tuple-like view materialising rows on access)."""
    pool = _pool_of(pool_or_catalog, eps_latency, eps_quality)
    h = np.asarray(h, dtype=np.float64) if not hasattr(h, "is_cuda") else h
    if h.shape[0] == 0:
        raise ProfileError("profile_config: empty prompt population")
    if scores is None:
        if noise is None:
            raise ProfileError("profile_records: give scores or noise")
        scores = light_scores(pool, h, noise)
    elif isinstance(scores, dict):
        scores = np.stack([np.asarray(scores[v.id], dtype=np.float64) for v in pool[:-1]])
    prof = GridProfiler(pool, h, scores)
    dt = prof.run(thresholds, exact_fid=exact_fid)
    rows = rows_from_device(dt, pool, thresholds, lazy=lazy)
    if provenance is None:
        cat = pool_or_catalog if hasattr(pool_or_catalog, "variants") else None
        provenance = TableProvenance(
            catalog_hash=catalog_hash(cat) if cat is not None else "",
            prompts_hash="", n_prompts=prof.n, seed=0, noise_sigma=0.0,
            thresholds=tuple(float(t) for t in thresholds), eps_latency=eps_latency,
            eps_quality=eps_quality)
    return CascadeTable(rows=rows, provenance=provenance)


def profile_config(catalog, prompts, seed: int = 0, noise_sigma: float = DEFAULT_NOISE_SIGMA,
                   eps_latency: float = 0.1, eps_quality: float = 0.1,
                   thresholds=THRESHOLD_GRID, weights=None, exact_fid: bool = True) -> CascadeTable:
    """Drop-in for cascadesim.profiler.profile_config (profiler.py:107-186).

    ``exact_fid`` (default True) recomputes every emitted row's fidelity with
    the numpy-exact emulation so the returned table equals the reference's
    bit for bit; False keeps the fixed-point fidelity (within ~1e-12 relative)."""
    texts = list(prompts)
    if not texts:
        raise ProfileError("profile_config: empty prompt population")
    pool = _pool_of(catalog, eps_latency, eps_quality)
    thr = tuple(float(t) for t in thresholds)
    weights = None if weights is None else check_weights(weights)
    rec = text_records(texts, seed, noise_sigma, weights)
    texts = [texts[i] for i in rec.order.tolist()]
    prov = TableProvenance(catalog_hash=catalog_hash(catalog),
                           prompts_hash=prompts_hash_sorted(texts), n_prompts=len(texts),
                           seed=seed, noise_sigma=noise_sigma, thresholds=thr,
                           eps_latency=eps_latency, eps_quality=eps_quality)
    return profile_records(pool, rec.d_h, scores=light_scores(pool, rec.h, rec.noise),
                           thresholds=thr, exact_fid=exact_fid, provenance=prov)
