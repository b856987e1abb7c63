"""Host-side logic of candidate-axis sharding (no GPU): the cross-shard merge
must reproduce the reference's best_candidate rule (portfolio.hpp:32-61) on
the union of the shards, and the exchange must work over torch.distributed
with world_size 2 (gloo)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2111_14991_b200.sharding import (ShardRecord, TorchComm, merge_shard_records, split_bounds,
                                            sum_in_rank_order)

EI, POI, LCB = 0, 1, 2


def rec(best_pos, best_score, first, nan_mask=0, n=10):
    return ShardRecord(tuple(best_pos), tuple(best_score), first, nan_mask, n, 0.1, 0.2, -0.3, False)


def reference_best(scores, eligible):
    """portfolio.hpp:32-61 restated over a flat score list."""
    best, best_score = -1, 0.0
    for i, (s, e) in enumerate(zip(scores, eligible)):
        if not e:
            continue
        if best == -1 or s > best_score:
            best, best_score = i, s
    return best


def shard_view(scores, eligible, lo, hi):
    idx = [i for i in range(lo, hi) if eligible[i]]
    if not idx:
        return rec([-1, -1, -1], [0, 0, 0], -1, 0, 0)
    first = idx[0]
    nonnan = [i for i in idx if not math.isnan(scores[i])]
    bp, bs = -1, 0.0
    for i in nonnan:
        if bp == -1 or scores[i] > bs:
            bp, bs = i, scores[i]
    nan_mask = 1 if math.isnan(scores[first]) else 0
    return rec([bp, -1, -1], [bs, 0, 0], first, nan_mask, len(idx))


@pytest.mark.parametrize("seed", range(40))
def test_merge_equals_unsharded_best_candidate(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 60))
    scores = list(np.round(rng.normal(size=n), 1))  # coarse: many ties
    for i in range(n):
        if rng.random() < 0.15:
            scores[i] = math.nan
    eligible = list(rng.random(n) > 0.3)
    parts = int(rng.integers(1, 5))
    recs = [shard_view(scores, eligible, *split_bounds(n, parts, r)) for r in range(parts)]
    want = reference_best(scores, eligible)
    if want == -1:
        with pytest.raises(Exception, match="no candidates"):
            merge_shard_records(recs, 1 << EI)
        return
    got = merge_shard_records(recs, 1 << EI)
    assert got.position[EI] == want, (scores, eligible, parts)
    assert got.n_candidates == sum(eligible)


def test_merge_first_nan_wins_and_masks():
    # first eligible candidate (global 3, shard 0) has a NaN EI score: it wins
    recs = [rec([5, 5, 4], [0.5, 0.9, -1.0], 3, nan_mask=1), rec([12, 11, 10], [2.0, 0.1, 3.0], 10)]
    sel = merge_shard_records(recs, 0b111)
    assert sel.position == (3, 5, 10)
    assert math.isnan(sel.score[EI])
    # ties across shards resolve to the lowest position
    recs = [rec([7, -1, -1], [1.5, 0, 0], 2), rec([4, -1, -1], [1.5, 0, 0], 1)]
    assert merge_shard_records(recs, 1 << EI).position[EI] == 4


def test_split_bounds_cover():
    for n in (1, 7, 1000, 1_000_000):
        for parts in (1, 2, 3, 8):
            b = [split_bounds(n, parts, r) for r in range(parts)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(parts - 1))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm(torch.device("cpu"))
        # (1) variance totals, summed in rank order
        tot = np.array([0.5 + rank, 100.0 + rank])
        gsum, gcnt = sum_in_rank_order(comm.allgather(tot))
        # (2) selection records
        mine = rec([10 * rank + 3, -1, 10 * rank + 1], [1.0 + rank, 0.0, -0.5 * rank], 10 * rank, 0, 5)
        recs = [ShardRecord.unpack(a) for a in comm.allgather(mine.pack())]
        sel = merge_shard_records(recs, (1 << EI) | (1 << LCB))
        q.put((rank, gsum, gcnt, sel.position, sel.n_candidates))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange_and_merge():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    for rank, gsum, gcnt, pos, ncand in out:
        assert gsum == 0.5 + 1.5 and gcnt == 201
        assert pos == (13, -1, 1)  # EI: rank 1's 2.0 beats 1.0; LCB: rank 0's 0.0 beats -0.5
        assert ncand == 10
    assert out[0][1:] == out[1][1:]  # identical decision on every rank
