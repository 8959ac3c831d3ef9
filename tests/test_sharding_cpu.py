"""Multi-process sharding logic on CPU (gloo, world_size 2): the pair split
covers every pair once in canonical order and the all-gather merge of
per-rank rows reproduces the single-process row list exactly."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_00642_b200.sharding import FIELDS, gather_rows, shard_light_groups, shard_pairs


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


@pytest.mark.parametrize("models,world", [(16, 8), (16, 2), (16, 3), (8, 8), (4, 8), (16, 16),
                                          (2, 1)])
def test_shard_light_groups_partition(models, world):
    pairs = [(i, j) for i in range(models) for j in range(i + 1, models)]
    seen = []
    loads = []
    for r in range(world):
        ids, mine = shard_light_groups(pairs, world, r)
        assert ids == sorted(ids) and mine == [pairs[i] for i in ids]
        seen.extend(ids)
        loads.append(len(ids))
    assert sorted(seen) == list(range(len(pairs)))
    share = -(-len(pairs) // world)
    assert max(loads) <= share + 1
    if (models, world) == (16, 8):              # c4 on 8 GPUs: {15}, {14, 1}, {13, 2}, ...
        lights = [len({p[0] for p in shard_light_groups(pairs, 8, r)[1]}) for r in range(8)]
        assert loads == [15] * 8 and max(lights) == 2


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


def _worker(rank, world, port, n_pairs, out_path, by_light=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if by_light:                                 # pairs of a 5-model pool, light-group shards
        plist = [(i, j) for i in range(5) for j in range(i + 1, 5)][:n_pairs]
        off, mine_pairs = shard_light_groups(plist, world, rank)
        mine = list(off)
        local_ids = list(range(len(mine)))
    else:
        pairs = list(range(n_pairs))
        off, mine = shard_pairs(pairs, world, rank)
        local_ids = None
    rows = _rows_for(mine)
    if local_ids is not None:                    # rows carry local pair ids 0..len(mine)-1
        rows["pair"] = [mine.index(p) for p in rows["pair"]]
    arrays = {}
    for f in FIELDS:
        if f in ("pair", "theta_pos", "tau_pos"):
            t = torch.tensor(rows[f], dtype=torch.int32)
            arrays[f] = t - off if (f == "pair" and not by_light) else t   # local pair ids
        else:
            arrays[f] = torch.tensor(rows[f], dtype=torch.float64)
    merged = gather_rows(torch, dist, arrays, off, torch.device("cpu"))
    if rank == 0:
        torch.save({f: merged[f] for f in FIELDS}, out_path)
    dist.destroy_process_group()


@pytest.mark.parametrize("n_pairs,by_light", [(6, False), (7, False), (1, False), (10, True),
                                              (7, True)])
def test_gather_rows_gloo_world2(tmp_path, n_pairs, by_light):
    out = str(tmp_path / "merged.pt")
    mp.spawn(_worker, args=(2, _free_port(), n_pairs, out, by_light), nprocs=2, join=True)
    merged = torch.load(out)
    want = _rows_for(range(n_pairs))
    for f in FIELDS:
        got = merged[f].tolist()
        assert got == want[f], f
