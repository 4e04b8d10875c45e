"""Host logic of the row-band multi-GPU path (paper_1605_02406_b200/shard.py) on CPU: band partition,
neighbour pairing, and the torch.distributed exchange protocol with the gloo backend at world sizes 2
and 3 (127.0.0.1 rendezvous).  The device side of the same path is tests/test_band_gpu.py."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1605_02406_b200.shard import DistTransport, band_rows, neighbour_counts, plan_bands


def test_band_rows_partition():
    for h, w in [(2048, 1), (2048, 2), (2048, 3), (1024, 8), (32, 5), (7, 7)]:
        rows = band_rows(h, w)
        assert len(rows) == w and rows[0][0] == 0 and rows[-1][1] == h
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
        sizes = [r1 - r0 for r0, r1 in rows]
        assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1
    with pytest.raises(ValueError):
        band_rows(4, 5)


def test_neighbour_counts():
    counts = [(0, 5), (3, 7), (2, 0)]         # (down, up) per band, bottom-up
    assert neighbour_counts(counts, 0) == (0, 3)
    assert neighbour_counts(counts, 1) == (5, 2)
    assert neighbour_counts(counts, 2) == (7, 0)


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
        # every band sends (rank+1) records down and (rank+2) up; edge bands send nothing off the grid
        n_down = rank + 1 if rank > 0 else 0
        n_up = rank + 2 if rank < world - 1 else 0
        n_lo, n_hi = t.counts(n_down, n_up)
        assert n_lo == (rank + 1 if rank > 0 else 0) and n_hi == (rank + 2 if rank < world - 1 else 0)
        rec = lambda src, n, tag: torch.arange(4 * n, dtype=torch.float32).view(n, 4) + 1000 * src + tag
        send_down, send_up = rec(rank, n_down, 1), rec(rank, n_up, 2)
        recv_lo, recv_hi = torch.zeros(n_lo, 4), torch.zeros(n_hi, 4)
        t.migrate(send_down, send_up, recv_lo, recv_hi)
        if rank > 0:                               # what the band below sent up
            assert torch.equal(recv_lo, rec(rank - 1, n_lo, 2))
        if rank < world - 1:                       # what the band above sent down
            assert torch.equal(recv_hi, rec(rank + 1, n_hi, 1))
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


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_protocol_gloo(world):
    mp.spawn(_worker, args=(world, _free_port()), nprocs=world, join=True)
