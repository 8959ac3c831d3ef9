"""Multi-process sharding logic on CPU (gloo, world_size 2): the pair split
covers every pair once in canonical order and the all-gather merge of
per-rank rows reproduces the single-process row list exactly."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_00642_b200.sharding import FIELDS, gather_rows, shard_pairs


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n,world", [(1, 2), (6, 2), (28, 8), (120, 8), (120, 3), (5, 8)])
def test_shard_pairs_partition(n, world):
    pairs = [(i, i + 1) for i in range(n)]
    seen = []
    for r in range(world):
        off, chunk = shard_pairs(pairs, world, r)
        assert pairs[off:off + len(chunk)] == chunk
        seen.extend(chunk)
    assert seen == pairs
    sizes = [len(shard_pairs(pairs, world, r)[1]) for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def _rows_for(pair_ids):
    # deterministic fake per-pair rows: pair p has p % 3 + 1 rows
    rows = {f: [] for f in FIELDS}
    for p in pair_ids:
        for k in range(p % 3 + 1):
            rows["pair"].append(p)
            rows["theta_pos"].append(k)
            rows["tau_pos"].append(2 * k + 1)
            rows["r_light"].append(p / 7.0 + k)
            rows["r_heavy"].append(1.0 / (p + k + 1))
            rows["fid"].append(30.0 - p * 0.01 - k / 3.0)
            rows["lat"].append(0.5 + p + k * 1e-3)
    return rows


def _worker(rank, world, port, n_pairs, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pairs = list(range(n_pairs))
    off, mine = shard_pairs(pairs, world, rank)
    rows = _rows_for(mine)
    arrays = {}
    for f in FIELDS:
        if f in ("pair", "theta_pos", "tau_pos"):
            t = torch.tensor(rows[f], dtype=torch.int32)
            arrays[f] = t - off if f == "pair" else t     # local pair ids
        else:
            arrays[f] = torch.tensor(rows[f], dtype=torch.float64)
    merged = gather_rows(torch, dist, arrays, off, torch.device("cpu"))
    if rank == 0:
        torch.save({f: merged[f] for f in FIELDS}, out_path)
    dist.destroy_process_group()


@pytest.mark.parametrize("n_pairs", [6, 7, 1])
def test_gather_rows_gloo_world2(tmp_path, n_pairs):
    out = str(tmp_path / "merged.pt")
    mp.spawn(_worker, args=(2, _free_port(), n_pairs, out), nprocs=2, join=True)
    merged = torch.load(out)
    want = _rows_for(range(n_pairs))
    for f in FIELDS:
        got = merged[f].tolist()
        assert got == want[f], f
