"""Multi-process sharding logic on CPU (gloo, world_size 2): the pair split
covers every pair once in canonical order; slabs laid out as the C ABI
defines them (hadis_shard_slab_bytes) travel through the product's
all-gather, and a numpy mirror of hadis_shard_merge over the gathered bytes
reproduces the canonical row list exactly, r_light / r_heavy / lat rebuilt
from the compact rows' counts as IEEE divisions by n (what the kernel's div_n
computes).  (The CUDA merge itself runs in
the GPU test test_sharded_profile_equals_single.)"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import numpy as np

from paper_2509_00642_b200 import _lib
from paper_2509_00642_b200.sharding import (FIELDS, SLAB_FIELDS, ShardMap, all_gather_slab,
                                            shard_light_groups, shard_pairs, slab_offsets)

N_REC = 1000003          # record count of the fake slabs


def _lat_pair(g):
    """Fake (L_light, L_heavy) of global pair g."""
    return 0.25 + g / 13.0, 1.5 + g / 7.0


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


def _rows_for(g):
    """Deterministic fake compact rows of global pair g: g % 3 + 1 rows of
    (theta_pos, tau_pos, n_light, n_heavy, fid)."""
    return [(k, 2 * k + 1, N_REC - 17 * g - k, 3 * g + 11 * k + 1, 30.0 - g * 0.01 - k / 3.0)
            for k in range(g % 3 + 1)]


def _table_row(g, row):
    """The table row the merge must produce from a compact row (profiler order)."""
    th, ta, nl, nh, fid = row
    ll, lh = _lat_pair(g)
    return (th, ta, nl / N_REC, nh / N_REC, fid, (nl * ll + nh * lh) / N_REC)


def _fake_slab(smap, rank, cap):
    hw = smap.hdr_words
    nbytes = _lib.load().hadis_shard_slab_bytes(hw, cap)
    buf = np.zeros(nbytes, dtype=np.uint8)
    hdr = buf[:8 * hw].view(np.int64)
    offs = slab_offsets(hw, cap)
    cols = [buf[offs[k]:offs[k] + 4 * cap].view(np.uint32 if k >= 2 else np.int32)
            for k in range(4)] + [buf[offs[4]:offs[4] + 8 * cap].view(np.float64)]
    r = 0
    for j, g in enumerate(smap.rank_ids[rank]):
        rows = _rows_for(g)
        hdr[_lib.ST_PAIR0 + j] = len(rows)
        for row in rows:
            for k, v in enumerate(row):
                cols[k][r] = v
            r += 1
    hdr[_lib.ST_ROWS] = r
    return buf


def _merge_mirror(gathered, smap, cap):
    """numpy restatement of hadis_shard_merge (csrc/shards.cu) -- test infra."""
    hw = smap.hdr_words
    nbytes = _lib.load().hadis_shard_slab_bytes(hw, cap)
    offs = slab_offsets(hw, cap)
    out = {f: [] for f in FIELDS}
    for g in range(smap.n_pairs):
        r, j = int(smap.pair_rank[g]), int(smap.pair_local[g])
        slab = gathered[r * nbytes:(r + 1) * nbytes]
        hdr = slab[:8 * hw].view(np.int64)
        src = int(hdr[_lib.ST_PAIR0:_lib.ST_PAIR0 + j].sum())
        cnt = int(hdr[_lib.ST_PAIR0 + j])
        cols = [slab[offs[k]:offs[k] + 4 * cap].view(np.uint32 if k >= 2 else np.int32)
                for k in range(4)] + [slab[offs[4]:offs[4] + 8 * cap].view(np.float64)]
        ll, lh = _lat_pair(g)
        for i in range(src, src + cnt):
            th, ta, nl, nh, fid = (c[i].item() for c in cols)
            out["pair"].append(g)
            out["theta_pos"].append(th)
            out["tau_pos"].append(ta)
            out["r_light"].append(float(nl) / N_REC)      # IEEE division = the kernel's div_n
            out["r_heavy"].append(float(nh) / N_REC)
            out["fid"].append(fid)
            out["lat"].append((float(nl) * ll + float(nh) * lh) / N_REC)
    return out


def _worker(rank, world, port, n_models, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pairs = [(i, j) for i in range(n_models) for j in range(i + 1, n_models)]
    smap = ShardMap(pairs, world)
    cap = 64
    slab = torch.from_numpy(_fake_slab(smap, rank, cap))
    gathered = torch.empty(world * slab.numel(), dtype=torch.uint8)
    all_gather_slab(torch, dist, slab, gathered)
    if rank == 0:
        torch.save(_merge_mirror(gathered.numpy(), smap, cap), out_path)
    dist.destroy_process_group()


@pytest.mark.parametrize("n_models", [2, 4, 5, 8])
def test_slab_gather_and_merge_gloo_world2(tmp_path, n_models):
    out = str(tmp_path / "merged.pt")
    mp.spawn(_worker, args=(2, _free_port(), n_models, out), nprocs=2, join=True)
    merged = torch.load(out)
    n_pairs = n_models * (n_models - 1) // 2
    want = {f: [] for f in FIELDS}
    for g in range(n_pairs):
        for row in _rows_for(g):
            want["pair"].append(g)
            for k, f in enumerate(FIELDS[1:]):
                want[f].append(_table_row(g, row)[k])
    for f in FIELDS:
        assert merged[f] == want[f], f


@pytest.mark.parametrize("models,world", [(16, 8), (8, 3), (4, 8), (2, 1)])
def test_shard_map_covers_every_pair_once(models, world):
    pairs = [(i, j) for i in range(models) for j in range(i + 1, models)]
    smap = ShardMap(pairs, world)
    for g in range(len(pairs)):
        r, j = smap.pair_rank[g], smap.pair_local[g]
        assert smap.rank_ids[r][j] == g
    assert smap.rank_npairs.sum() == len(pairs)
    assert smap.hdr_words % 32 == 0 and smap.hdr_words >= _lib.ST_PAIR0 + len(pairs) + 2


@pytest.mark.parametrize("cap", [0, 1, 3, 1000, 12345])
def test_slab_layout_matches_library(cap):
    hw = 160
    nbytes = _lib.load().hadis_shard_slab_bytes(hw, cap)
    offs = slab_offsets(hw, cap)
    assert len(offs) == len(SLAB_FIELDS) == 5
    assert offs[0] == 8 * hw and offs[4] % 8 == 0 and offs[4] >= offs[3] + 4 * cap
    assert offs[-1] + 8 * cap <= nbytes and nbytes % 256 == 0
