"""Multi-GPU profiling: pair-sharded grid evaluation + one all-gather merge.

SPEC.md:309-310 calls pair x grid profiling embarrassingly parallel with a
deterministic (pair, theta, tau) reduction order.  One process per GPU:

* ``shard_light_groups`` assigns whole light-model groups of the canonical
  pair list (light < heavy in pool latency order, profiler.py:141-143) to
  ranks longest-first, so every rank reads the score rows of at most a few
  light models; ``shard_pairs`` is the plain contiguous split;
* each rank runs K1..K4 for its pairs (a pair's frontier needs no other
  pair's cells, so nothing is exchanged on the data path);
* ``gather_rows`` packs each rank's emitted rows into one float64 buffer and
  merges them with a single ``all_gather_into_tensor`` (NCCL over NVLink on
  GPUs, gloo in the CPU tests); a stable sort by global pair id restores the
  canonical pair order, so the result is identical to the 1-GPU table.
"""

from __future__ import annotations

FIELDS = ("pair", "theta_pos", "tau_pos", "r_light", "r_heavy", "fid", "lat")


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


def pack_rows(torch, arrays, pair_ids, device):
    """[rows, 7] float64 buffer (pair ids made global; integers are exact in f64).
    ``pair_ids``: an int offset (contiguous shard) or the shard's global ids."""
    n = int(arrays["pair"].shape[0])
    buf = torch.empty((n, len(FIELDS)), dtype=torch.float64, device=device)
    gid = None if isinstance(pair_ids, int) else torch.as_tensor(
        list(pair_ids) or [0], dtype=torch.int64, device=device)
    for j, f in enumerate(FIELDS):
        col = arrays[f].to(device=device)
        if f == "pair":
            col = col.to(torch.float64) + pair_ids if gid is None else \
                gid[col.to(torch.int64)].to(torch.float64)
        buf[:, j] = col.to(torch.float64)
    return buf


def gather_rows(torch, dist, arrays, pair_ids, device, group=None):
    """All-gather every rank's rows; returns dict of concatenated columns
    (float64 for doubles, int64 for ids) in canonical pair order (rows of one
    pair keep their (theta, tau) order: a stable sort by global pair id)."""
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "gloo":      # gloo collectives run on host tensors
        device = torch.device("cpu")
    local = pack_rows(torch, arrays, pair_ids, device)
    n_local = torch.tensor([local.shape[0]], dtype=torch.int64, device=device)
    counts = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(counts, n_local, group=group)
    counts = counts.cpu().tolist()
    width = max(max(counts), 1)
    padded = torch.zeros((width, len(FIELDS)), dtype=torch.float64, device=device)
    padded[:local.shape[0]] = local
    everything = torch.empty((world * width, len(FIELDS)), dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(everything, padded, group=group)
    parts = [everything[r * width:r * width + counts[r]] for r in range(world)]
    merged = torch.cat(parts, dim=0)
    if not isinstance(pair_ids, int):          # non-contiguous shards: canonical pair order
        order = torch.sort(merged[:, 0], stable=True).indices
        merged = merged[order]
    out = {}
    for j, f in enumerate(FIELDS):
        col = merged[:, j]
        out[f] = col.to(torch.int64) if f in ("pair", "theta_pos", "tau_pos") else col
    return out


def profile_sharded(prof, thresholds, dist, exact_fid=False, group=None):
    """Run this rank's share of every pair and merge: returns (pairs, rows dict).
    Shards are whole light-model groups (``shard_light_groups``)."""
    from .profiler import pair_list
    torch = prof.torch
    pairs = pair_list(prof.pool)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    ids, mine = shard_light_groups(pairs, world, rank)
    if mine:
        from .profiler import GridProfiler
        slots = sorted({i for i, _ in mine})
        rows = [prof.row_of(i) for i in slots]
        shard = GridProfiler(prof.pool, prof.h, prof.scores[rows], device=prof.device,
                             layout=prof.layout, slots=slots)
        dt = shard.run(thresholds, pairs=mine, exact_fid=exact_fid)
        arrays = {f: getattr(dt, f) for f in FIELDS}
    else:
        empty_i = torch.empty(0, dtype=torch.int32, device=prof.device)
        empty_d = torch.empty(0, dtype=torch.float64, device=prof.device)
        arrays = {f: (empty_i if f in ("pair", "theta_pos", "tau_pos") else empty_d)
                  for f in FIELDS}
    return pairs, gather_rows(torch, dist, arrays, ids, prof.device, group)


def solve_sharded(table, catalog, lams, queues=None, workers=16, t_slo=60.0, alpha=1.5,
                  dist=None, group=None, label="online"):
    """Allocation search over many (demand, SLO) points on every rank (SURVEY
    §8(e), c5): contiguous point chunks per rank (points are independent),
    ``planner.solve_many`` on each rank's GPU, then one all-gather of the
    plans; the list is in input order on every rank."""
    import numpy as np

    from .planner import solve_many
    lams = [float(x) for x in lams]
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
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    mine = (solve_many(table, catalog, lams[start:stop], qs[start:stop], ws[start:stop],
                       ts[start:stop], alpha, label) if stop > start else [])
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    return [p for part in parts for p in part]
