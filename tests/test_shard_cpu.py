"""Host logic of the row-band multi-GPU path (paper_1605_02406_b200/shard.py) on CPU: band partition,
which bucket of which band feeds each band, and the torch.distributed exchange protocol (near buckets
point to point, far buckets by all-gather, all-rank failure on overflow) with the gloo backend at world
sizes 2, 3 and 4 (127.0.0.1 rendezvous).  The device side of the same path is tests/test_band_gpu.py."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1605_02406_b200.shard import DistTransport, band_rows, plan_bands, sources_for


def test_band_rows_partition():
    for h, w in [(2048, 1), (2048, 2), (2048, 3), (1024, 8), (32, 5), (7, 7)]:
        rows = band_rows(h, w)
        assert len(rows) == w and rows[0][0] == 0 and rows[-1][1] == h
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
        sizes = [r1 - r0 for r0, r1 in rows]
        assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1
    with pytest.raises(ValueError):
        band_rows(4, 5)


def test_sources_for():
    # band r is fed by r-1's "above" bucket, r+1's "below" bucket and the far buckets of everyone else
    assert sources_for(0, 1) == (None, None, [], [])
    assert sources_for(0, 3) == (None, (1, 0), [], [(2, 2)])
    assert sources_for(2, 5) == ((1, 1), (3, 0), [(0, 3)], [(4, 2)])
    assert sources_for(4, 5) == ((3, 1), None, [(0, 3), (1, 3), (2, 3)], [])


def test_plan_bands_balances_work():
    import numpy as np
    rng = np.random.default_rng(0)
    W, H = 64, 256
    for world in (1, 2, 3, 5, 8):
        cnt = rng.integers(0, 5000, H) * (rng.random(H) < 0.3)
        cnt[100:120] += 40000                       # a dense stripe
        rows = plan_bands(cnt, W, world, min_rows=8)
        assert len(rows) == world and rows[0][0] == 0 and rows[-1][1] == H
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
        assert all(r1 - r0 >= 8 for r0, r1 in rows)
        cost = cnt * 64.0 + 56.0 * W
        per = [cost[r0:r1].sum() for r0, r1 in rows]
        # each boundary is the first row reaching its share: no band exceeds its share by more than one row
        # (unless the min_rows clamp applies)
        assert max(per) <= cost.sum() / world + cost.max() + 8 * cost.max()
    # uniform rows -> the even partition
    assert plan_bands(np.full(256, 100), W, 4, 8) == [(0, 64), (64, 128), (128, 192), (192, 256)]
    # everything in one row: the clamp keeps min_rows per band
    one = np.zeros(64, np.int64); one[10] = 10 ** 6
    rows = plan_bands(one, W, 4, 8)
    assert all(r1 - r0 >= 8 for r0, r1 in rows) and rows[-1][1] == 64
    with pytest.raises(ValueError):
        plan_bands(np.zeros(20), W, 3, 8)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        t = DistTransport(rank, world, torch.device("cpu"))
        # band b sends (b+1) records to the band below, (b+2) above, 1 further below / above where one exists
        cnt = lambda b: [b + 1 if b > 0 else 0, b + 2 if b < world - 1 else 0, 1 if b > 1 else 0,
                         1 if b < world - 2 else 0]
        rec = lambda src, d, n: torch.arange(4 * n, dtype=torch.float32).view(n, 4) + 1000 * src + 100 * d
        counts = cnt(rank)
        out = [rec(rank, d, counts[d]) for d in range(4)]
        srcs = t.exchange_buckets(out, counts)
        lo_near, hi_near, lo_far, hi_far = sources_for(rank, world)
        expect = ([("lo", lo_near)] if lo_near else []) + ([("hi", hi_near)] if hi_near else [])
        expect += [("lof", x) for x in lo_far] + [("hif", x) for x in hi_far]
        assert [k for k, _, _ in srcs] == [k for k, _ in expect]
        for (kind, got, n), (_, (b, d)) in zip(srcs, expect):
            assert n == cnt(b)[d] and got.shape[0] == n
            assert torch.equal(got, rec(b, d, n)), (rank, kind, b, d)
        # a band reporting an overflow makes every rank raise (nobody waits in a collective)
        from paper_1605_02406_b200 import dog
        with pytest.raises(dog.DogError):
            t.exchange_buckets([rec(rank, d, 0) for d in range(4)], [0, 0, 0, 0], ok=0 if rank == world - 1 else 1)
        out = torch.zeros(world, dtype=torch.int64)
        t.allgather_u64(torch.tensor([10 ** 12 + rank], dtype=torch.int64), out)
        assert out.tolist() == [10 ** 12 + r for r in range(world)]
        # rebalancing exchanges: variable-length all-gather and all-reduce (ShardedFilter.rebalance)
        mine = torch.arange(4 * (rank + 1), dtype=torch.float32).view(rank + 1, 4) + 100 * rank
        got = t.allgather_var(mine)
        assert [g.shape[0] for g in got] == [r + 1 for r in range(world)]
        for r, g in enumerate(got):
            assert torch.equal(g, torch.arange(4 * (r + 1), dtype=torch.float32).view(r + 1, 4) + 100 * r)
        s = t.allreduce_sum(torch.tensor([rank, 1], dtype=torch.int64))
        assert s.tolist() == [world * (world - 1) // 2, world]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_exchange_protocol_gloo(world):
    mp.spawn(_worker, args=(world, _free_port()), nprocs=world, join=True)
