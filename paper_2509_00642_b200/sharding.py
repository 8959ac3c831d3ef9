"""Multi-GPU profiling: pair-sharded grid evaluation + one all-gather merge.

SPEC.md:309-310 calls pair x grid profiling embarrassingly parallel with a
deterministic (pair, theta, tau) reduction order.  One process per GPU:

* ``shard_pairs`` splits the canonical pair list (light < heavy in pool
  latency order, profiler.py:141-143) into contiguous, cell-balanced chunks,
  so every rank reads only the score rows of its own light models;
* each rank runs K1..K4 for its pairs (a pair's frontier needs no other
  pair's cells, so nothing is exchanged on the data path);
* ``gather_rows`` packs each rank's emitted rows into one float64 buffer and
  merges them with a single ``all_gather_into_tensor`` (NCCL over NVLink on
  GPUs, gloo in the CPU tests); concatenating in rank order is the canonical
  pair order, so the result is identical to the 1-GPU table.
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


def pack_rows(torch, arrays, pair_offset, device):
    """[rows, 7] float64 buffer (pair ids made global; integers are exact in f64)."""
    n = int(arrays["pair"].shape[0])
    buf = torch.empty((n, len(FIELDS)), dtype=torch.float64, device=device)
    for j, f in enumerate(FIELDS):
        col = arrays[f].to(device=device, dtype=torch.float64)
        buf[:, j] = col + pair_offset if f == "pair" else col
    return buf


def gather_rows(torch, dist, arrays, pair_offset, device, group=None):
    """All-gather every rank's rows; returns dict of concatenated columns
    (float64 for doubles, int64 for ids) in canonical (rank = pair) order."""
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "gloo":      # gloo collectives run on host tensors
        device = torch.device("cpu")
    local = pack_rows(torch, arrays, pair_offset, device)
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
    out = {}
    for j, f in enumerate(FIELDS):
        col = merged[:, j]
        out[f] = col.to(torch.int64) if f in ("pair", "theta_pos", "tau_pos") else col
    return out


def profile_sharded(prof, thresholds, dist, exact_fid=False, group=None):
    """Run this rank's share of every pair and merge: returns (pairs, rows dict)."""
    from .profiler import pair_list
    torch = prof.torch
    pairs = pair_list(prof.pool)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    offset, mine = shard_pairs(pairs, world, rank)
    if mine:
        dt = prof.run(thresholds, pairs=mine, exact_fid=exact_fid)
        arrays = {f: getattr(dt, f) for f in FIELDS}
    else:
        empty_i = torch.empty(0, dtype=torch.int32, device=prof.device)
        empty_d = torch.empty(0, dtype=torch.float64, device=prof.device)
        arrays = {f: (empty_i if f in ("pair", "theta_pos", "tau_pos") else empty_d)
                  for f in FIELDS}
    return pairs, gather_rows(torch, dist, arrays, offset, prof.device, group)
