"""Multi-GPU profiling and planning: pair-sharded builds + one all-gather merge.

SPEC.md:309-310 calls pair x grid profiling embarrassingly parallel with a
deterministic (pair, theta, tau) reduction order.  One process per GPU:

* ``shard_light_groups`` assigns whole light-model groups of the canonical
  pair list (light < heavy in pool latency order, profiler.py:141-143) to
  ranks longest-first, so every rank reads the score rows of at most a few
  light models; ``shard_pairs`` is the plain contiguous split;
* each rank builds its pairs' frontiers with no data-path collective (a
  pair's frontier needs no other pair's cells), emitting rows straight into
  its slab (``ShardSlab``: frontier stats header + the compact rows of
  ``hadis_pair_frontiers_compact`` -- theta_pos, tau_pos, n_light, n_heavy,
  fid: 24 bytes per row instead of the table's 44, no pack step);
* one ``all_gather_into_tensor`` of the fixed-size slabs (NCCL over NVLink on
  GPUs; gloo moves them through host memory) gives every rank every slab,
  row counts included, so no count round trip precedes it;
* ``hadis_shard_merge`` writes the canonical table on every rank (pairs in
  global order, each pair's rows in its owner's (theta, tau) order; r_light,
  r_heavy, lat rebuilt from the counts with the frontier's own operations)
  without a host round trip; the table is identical for 1/2/4/8 GPUs.

Error consensus: a rank's local failure (bad records, a slab too small, an
exception) is written into its slab header instead of being raised before
the collective; after the all-gather every rank sees every header and raises
(or grows and reruns) identically, so no rank is left waiting in a collective.

``solve_sharded`` splits the (demand, SLO) points into equal chunks, solves
each on its rank's GPU and all-gathers the plan arrays as one float64 tensor.
"""

from __future__ import annotations

import numpy as np

from . import _lib

FIELDS = ("pair", "theta_pos", "tau_pos", "r_light", "r_heavy", "fid", "lat")
_INT_FIELDS = ("pair", "theta_pos", "tau_pos")
SLAB_FIELDS = ("theta_pos", "tau_pos", "n_light", "n_heavy", "fid")   # compact slab rows

ERR_RECORDS, ERR_SLAB, ERR_PROFILE = 1, 2, 4       # host error word bits


def shard_pairs(pairs, world: int, rank: int):
    """Contiguous chunk of ``pairs`` for ``rank`` (all pairs cost the same
    U^2 cells, so equal counts balance the grid work).  Returns (offset, chunk)."""
    n = len(pairs)
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    size = base + (1 if rank < extra else 0)
    return start, list(pairs[start:start + size])


def shard_light_groups(pairs, world: int, rank: int):
    """Balanced shard for ``rank``: pairs grouped by light model (the pairs of
    one light model share its score row, K1 histogram and row staging), whole
    groups assigned longest-first to the least-loaded rank (a group larger than
    an even share is split into even-share chunks).  Cost = pairs + one pair's
    worth per light model (its scatter / K1 / staging).  c4 on 8 ranks:
    {15}, {14, 1}, {13, 2}, ... -- at most two light models per rank.
    Returns (global pair ids, pairs), both in canonical order."""
    groups = {}
    for gi, pr in enumerate(pairs):
        groups.setdefault(pr[0], []).append(gi)
    share = max(1, -(-len(pairs) // world))
    units = []
    for light in sorted(groups):
        ids = groups[light]
        for c in range(0, len(ids), share):
            units.append(ids[c:c + share])
    units.sort(key=lambda u: (-(len(u) + 1), u[0]))
    load = [0] * world
    owned = [[] for _ in range(world)]
    for u in units:
        r = min(range(world), key=lambda i: (load[i], i))
        load[r] += len(u) + 1
        owned[r].extend(u)
    ids = sorted(owned[rank])
    return ids, [pairs[i] for i in ids]


class ShardMap:
    """Who owns which global pair (the same on every rank: the assignment is a
    pure function of the pair list and the world size)."""

    def __init__(self, pairs, world: int):
        self.n_pairs = len(pairs)
        self.world = world
        self.rank_ids = [shard_light_groups(pairs, world, r)[0] for r in range(world)]
        self.pair_rank = np.zeros(self.n_pairs, dtype=np.int32)
        self.pair_local = np.zeros(self.n_pairs, dtype=np.int32)
        for r, ids in enumerate(self.rank_ids):
            for j, g in enumerate(ids):
                self.pair_rank[g], self.pair_local[g] = r, j
        self.rank_npairs = np.array([len(ids) for ids in self.rank_ids], dtype=np.int32)
        # header: frontier stats for up to n_pairs local pairs + record flag, host error word
        self.hdr_words = -(-(_lib.ST_PAIR0 + self.n_pairs + 2) // 32) * 32


class ShardSlab:
    """One rank's slab (include/hadis_b200.h, hadis_shard_slab_bytes): the
    frontier of GridProfiler(sink=slab) writes its stats and rows into it."""

    def __init__(self, torch, hdr_words: int, cap: int, device):
        self.torch = torch
        self.hdr_words, self.cap = hdr_words, int(cap)
        self.nbytes = int(_lib.load().hadis_shard_slab_bytes(hdr_words, self.cap))
        self.buf = torch.zeros(self.nbytes, dtype=torch.uint8, device=device)
        self.header = self.buf[:8 * hdr_words].view(torch.int64)

    def offsets(self):
        return slab_offsets(self.hdr_words, self.cap)

    def columns(self, out_cap=None):
        """Views of the compact row columns (n_light / n_heavy hold uint32 bits)."""
        if out_cap is not None and out_cap != self.cap:
            raise ValueError("ShardSlab: the frontier's out_cap must equal the slab capacity")
        torch, cap = self.torch, self.cap
        out = {}
        for f, off in zip(SLAB_FIELDS, self.offsets()):
            dt, size = (torch.float64, 8) if f == "fid" else (torch.int32, 4)
            out[f] = self.buf[off:off + size * cap].view(dt)
        return out

    def stats(self, n_local_pairs: int):
        return self.header[:_lib.ST_PAIR0 + n_local_pairs + 1]

    def set_error(self, bits: int):
        self.header[self.hdr_words - 1] = bits


def slab_offsets(hdr_words: int, cap: int):
    """Byte offsets of the compact columns SLAB_FIELDS (csrc/shards.cu slab_i32_off /
    slab_f64_off): four 32-bit columns back to back, then fid at an 8-byte boundary."""
    i32 = [8 * hdr_words + 4 * k * cap for k in range(4)]
    return i32 + [(8 * hdr_words + 16 * cap + 7) & ~7]


def all_gather_slab(torch, dist, slab_buf, gathered, group=None):
    """gathered <- every rank's slab (NCCL on device; gloo through host memory)."""
    if dist.get_backend(group) == "gloo":
        host = torch.empty(gathered.numel(), dtype=torch.uint8)
        dist.all_gather_into_tensor(host, slab_buf.cpu(), group=group)
        gathered.copy_(host)
    else:
        dist.all_gather_into_tensor(gathered, slab_buf, group=group)


class ShardedTable:
    """This rank's share of a pair-sharded table build plus the merge.

    ``h``: float64[N] (every rank holds all records); ``scores``: the score
    rows of ``slots`` (pool light indices; None = every light model, row i =
    pool model i).  ``step()`` = local build (one CUDA-graph replay) + local
    status read + one all-gather + the merge kernel + one status read; it
    returns the merged table's columns (device views) on every rank."""

    def __init__(self, pool, h, scores, thresholds, dist, group=None, device=None, slots=None,
                 exact_fid=False, graph=True, headroom=1.125):
        from .profiler import GridProfiler, pair_list
        torch = _lib.torch_cuda()
        self.torch, self.dist, self.group = torch, dist, group
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.pool = list(pool)
        self.thresholds = tuple(float(t) for t in thresholds)
        self.exact_fid = exact_fid
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.pairs = pair_list(self.pool)
        self.map = ShardMap(self.pairs, self.world)
        self.ids = self.map.rank_ids[self.rank]
        self.mine = [self.pairs[g] for g in self.ids]
        self.lib = _lib.load()
        dev = self.device
        self.d_pair_rank = torch.from_numpy(self.map.pair_rank).to(dev)
        self.d_pair_local = torch.from_numpy(self.map.pair_local).to(dev)
        self.d_rank_npairs = torch.from_numpy(self.map.rank_npairs).to(dev)
        from .profiler import pair_params
        self.d_params = torch.from_numpy(pair_params(self.pool, self.pairs)).to(dev)
        self.n_records = int(h.shape[0]) if hasattr(h, "shape") else len(h)
        self.out_stats = torch.zeros(8, dtype=torch.int64, device=dev)
        self.stats_pin = torch.zeros(8, dtype=torch.int64).pin_memory()
        self.hdr_pin = torch.zeros(self.map.hdr_words, dtype=torch.int64).pin_memory()
        self.ws = torch.empty(max(1, self.lib.hadis_shard_merge_workspace_bytes(len(self.pairs))),
                              dtype=torch.uint8, device=dev)
        self.prof = self.plan = self.replay = None
        err = 0
        local_rows = 0
        if self.mine:
            try:
                my_slots = sorted({i for i, _ in self.mine})
                if slots is None:
                    rows = my_slots
                else:
                    pos = {m: r for r, m in enumerate(slots)}
                    rows = [pos[m] for m in my_slots]
                sc = scores[rows] if hasattr(scores, "index_select") else np.asarray(scores)[rows]
                self.prof = GridProfiler(self.pool, h, sc, device=dev, slots=my_slots)
                self.plan = self.prof.plan(self.thresholds, pairs=self.mine)
                local_rows = self.prof.run(self.thresholds, pairs=self.mine,
                                           exact_fid=exact_fid).n_rows
            except Exception as exc:          # reported through the consensus below
                self._local_exc = exc
                err = ERR_PROFILE
        # setup-time agreement on the slab capacity (and on failures)
        agree = torch.tensor([local_rows, err], dtype=torch.int64, device=dev)
        if dist.get_backend(group) == "gloo":
            agree = agree.cpu()
        dist.all_reduce(agree, op=dist.ReduceOp.MAX, group=group)
        if int(agree[1]):
            self._raise(int(agree[1]))
        self.headroom = headroom
        self._alloc(int(int(agree[0]) * headroom) + 1024, graph)

    def _raise(self, err):
        from .profiler import ProfileError
        exc = getattr(self, "_local_exc", None)
        if exc is not None:
            raise exc
        if err & ERR_RECORDS:
            raise ProfileError("profile_records: hardness must be finite and within [0, 1]")
        raise ProfileError("sharded profile: another rank failed to build its shard")

    def _alloc(self, cap, graph):
        torch = self.torch
        self.slab = ShardSlab(torch, self.map.hdr_words, cap, self.device)
        self.gathered = torch.empty(self.world * self.slab.nbytes, dtype=torch.uint8,
                                    device=self.device)
        self.out_cap = self.world * cap
        self.merged = {f: torch.empty(self.out_cap, dtype=torch.int32 if f in _INT_FIELDS
                                      else torch.float64, device=self.device) for f in FIELDS}
        if self.prof is not None:
            self.prof.sink = self.slab
            cand, exact, _ = self.plan.caps
            self.plan.caps = (cand, exact, cap)
            self.replay = self.prof.graph(self.plan, self.exact_fid) if graph else None

    @property
    def gather_bytes(self):
        """Bytes each rank receives per step (the slabs of all ranks)."""
        return self.world * self.slab.nbytes

    def _local(self):
        """Local build + local status (host read); failures go into the header."""
        from .profiler import ProfileError, grow_caps
        if self.prof is None:
            self.slab.header.zero_()
            return
        torch = self.torch
        if self.replay is not None:
            state = self.replay.launch()
        else:
            state = self.prof.launch(self.plan, self.exact_fid)
        n_loc = len(self.mine)
        for _ in range(6):
            hdr = self.slab.stats(n_loc)
            local = self.hdr_pin[:hdr.numel()]
            local.copy_(hdr, non_blocking=True)
            torch.cuda.current_stream(self.device).synchronize()
            st = local.tolist()
            if st[-1]:
                self.slab.set_error(ERR_RECORDS)
                return
            if st[_lib.ST_OVERFLOW] == 0:
                self.slab.set_error(0)
                return
            try:
                caps = grow_caps(self.plan, state["caps"], st, out_limit=self.slab.cap)
            except ProfileError as exc:
                if st[_lib.ST_OVERFLOW] & 8 and state["caps"][2] >= self.slab.cap:
                    self.slab.set_error(ERR_SLAB)      # every rank grows the slab next
                else:
                    self._local_exc = exc
                    self.slab.set_error(ERR_PROFILE)
                return
            self.plan.caps = caps
            self.prof._frontier(state, caps)
        self.slab.set_error(ERR_PROFILE)

    def step(self):
        """Build + merge; returns {field: device column[:rows]} (every rank)."""
        torch = self.torch
        for _ in range(4):
            with torch.cuda.device(self.device):
                self._local()
                all_gather_slab(torch, self.dist, self.slab.buf, self.gathered, self.group)
                self.merge()
                self.stats_pin[:5].copy_(self.out_stats[:5], non_blocking=True)
                torch.cuda.current_stream(self.device).synchronize()
            total, of, bad, err, max_rows = self.stats_pin[:5].tolist()
            if bad or err & ERR_RECORDS:
                self._raise(ERR_RECORDS)
            if err & ERR_PROFILE:
                self._raise(ERR_PROFILE)
            if err & ERR_SLAB or of & 8:               # identical decision on every rank
                self._alloc(int(max(max_rows, self.slab.cap) * 2), self.replay is not None)
                continue
            return {f: self.merged[f][:total] for f in FIELDS}
        self._raise(ERR_PROFILE)

    def merge(self, stream=None):
        """Enqueue hadis_shard_merge on the gathered slabs (no host sync)."""
        p = _lib.ptr
        m = self.merged
        _lib.check(self.lib.hadis_shard_merge(
            p(self.gathered), self.world, self.slab.nbytes, self.slab.cap, self.map.hdr_words,
            p(self.d_pair_rank), p(self.d_pair_local), p(self.d_rank_npairs), len(self.pairs),
            p(self.d_params), self.n_records,
            self.out_cap, p(m["pair"]), p(m["theta_pos"]), p(m["tau_pos"]), p(m["r_light"]),
            p(m["r_heavy"]), p(m["fid"]), p(m["lat"]), p(self.out_stats), p(self.ws),
            self.ws.numel(), _lib.stream_handle(stream, self.device)), "hadis_shard_merge")


def profile_sharded(prof, thresholds, dist, exact_fid=False, group=None):
    """This rank's share of every pair + the merge: returns (pairs, rows dict
    of device columns in canonical order, identical on every rank)."""
    st = ShardedTable(prof.pool, prof.h, prof.scores, thresholds, dist, group=group,
                      device=prof.device, slots=prof.slots, exact_fid=exact_fid, graph=False)
    return st.pairs, st.step()


PLAN_COLS = 7          # row, x_light, x_heavy, b_light, b_heavy, path, flags (float64)


def solve_sharded(table, catalog, lams, queues=None, workers=16, t_slo=60.0, alpha=1.5,
                  dist=None, group=None, label="online"):
    """Allocation search over many (demand, SLO) points on every rank (SURVEY
    §8(e), c5): equal point chunks per rank (points are independent), the
    device search on each rank's GPU, then one all-gather of the plan arrays
    (a [chunk, 7] float64 tensor per rank; integers are exact in float64).
    Returns the plans in input order on every rank."""
    from .planner import PlannerError, _plan_from, device_rows
    torch = _lib.torch_cuda()
    lams = [float(x) for x in lams]
    if any(x < 0 for x in lams):                  # every rank holds every point: same raise
        raise PlannerError("solve: negative demand")
    n = len(lams)

    def per_point(v, cast):
        if v is None or np.isscalar(v) or isinstance(v, dict):
            return [v] * n
        v = list(v)
        return [cast(x) for x in v] if cast else v

    qs = per_point(queues, None)
    ws = per_point(workers, int)
    ts = per_point(t_slo, float)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    chunk = max(1, -(-n // world))
    start, stop = min(n, rank * chunk), min(n, (rank + 1) * chunk)
    rows = table.rows if hasattr(table, "rows") else table
    dr = device_rows(rows, catalog)
    dev = dr.device
    mine = torch.zeros((chunk, PLAN_COLS), dtype=torch.float64, device=dev)
    if stop > start:
        res = dr.solve_arrays(lams[start:stop], ts[start:stop], ws[start:stop], qs[start:stop],
                              alpha)
        k = stop - start
        arr = np.empty((k, PLAN_COLS), dtype=np.float64)
        arr[:, 0] = res["row"]
        arr[:, 1:3] = res["x"].reshape(k, 2)
        arr[:, 3:5] = res["b"].reshape(k, 2)
        arr[:, 5] = res["path"]
        arr[:, 6] = res["flags"]
        mine[:k] = torch.from_numpy(arr).to(dev)
    gloo = dist.get_backend(group) == "gloo"
    send = mine.cpu() if gloo else mine
    everything = torch.empty((world * chunk, PLAN_COLS), dtype=torch.float64,
                             device="cpu" if gloo else dev)
    dist.all_gather_into_tensor(everything, send, group=group)
    g = everything[:n].cpu().numpy()
    res = {"row": g[:, 0].astype(np.int32), "x": g[:, 1:3].astype(np.int32).reshape(-1),
           "b": g[:, 3:5].astype(np.int32).reshape(-1), "path": g[:, 5].copy(),
           "flags": g[:, 6].astype(np.int32)}
    return [_plan_from(dr, res, p, lams[p], qs[p], label) for p in range(n)]
