"""Sharded filters against the whole grid and the oracle.

* The library's sharded context (include/dog.h dog_create with n_devices >= 2, dog_step /
  dog_step_sharded, dog_read_cells, dog_set_bands): several row bands on cuda:0, exchanges device to
  device inside the library, no host synchronisation inside a cycle.  Its next state must equal the
  ORACLE's bit for bit (not only the GPU whole-grid filter's), with thin bands and far migrants.
* The one-process-per-GPU driver (paper_1605_02406_b200.shard.ShardedFilter: the path `bench.py --gpus N`
  runs), here two processes sharing cuda:0 with the gloo backend and host-staged collectives (NCCL
  refuses two ranks on one device; no kernel waits on another process's kernel): ShardedFilter.step and
  ShardedFilter.rebalance over 8 cycles, bit for bit against the whole-grid filter.
Requires a CUDA device: run with `-m gpu`."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
from paper_1605_02406_b200 import inputs as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    torch.cuda.set_device(0)


def _bits(a, b, what):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    bad = np.nonzero(a.view(np.uint32).ravel() != b.view(np.uint32).ravel())[0]
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first at {bad[:5]}"


def _state(st):
    return np.stack([st["x"], st["y"], st["vx"], st["vy"]], 1)


def test_sharded_context_matches_the_oracle():
    """cfg1 (32x32, 10k + 1k, moving box), three bands on cuda:0 through dog_step on the sharded context:
    next state, m_F, occupancy and free mass bit-identical to the oracle every cycle; moments within 1e-4."""
    from paper_1605_02406_b200 import dog
    cfg = I.CONFIGS["cfg1"]
    sc = I.scene(cfg)
    kw = dict(cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params())
    f = dog.Filter(cfg.width, cfg.height, cfg.nu, cfg.nu_b, devices=[0, 0, 0], **kw)
    assert f.world == 3 and f.bands()[0] == [(0, 11), (11, 22), (22, 32)]
    o = oracle.Oracle(oracle.Params(width=cfg.width, height=cfg.height, nu=cfg.nu, nu_b=cfg.nu_b,
                                    cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params()))
    for k in range(10):
        meas = sc.frame(k)
        o.step(meas.numpy(), cfg.dt)
        f.step(meas.cuda().contiguous(), cfg.dt)
        so, sg = o.get_state(), f.get_state()
        for key in ("x", "y", "vx", "vy", "m_free"):
            _bits(so[key], sg[key], f"cycle {k}: {key}")
        co, cg = o.read_cells(), f.read_cells()
        _bits(co["occ"], cg["occ"].cpu().numpy(), f"cycle {k}: occ")
        _bits(co["free"], cg["free"].cpu().numpy(), f"cycle {k}: free")
        assert np.allclose(cg["mean"].cpu().numpy(), co["mean"], rtol=1e-4, atol=1e-6), k
        assert np.allclose(cg["cov"].cpu().numpy(), co["cov"], rtol=1e-4, atol=1e-8), k
    f.close()


def test_sharded_thin_bands_and_far_migrants():
    """4x Table I process noise on 64x64 cells and one-row bands: most particles of a thin band leave it
    and many cross more than one band (the far buckets).  dog_step_sharded with per-band measurement rows
    and one stream per band, band boundaries moved by dog_set_bands between cycles: bit-identical to the
    whole-grid filter throughout (nothing is lost)."""
    from paper_1605_02406_b200 import dog
    cfg = I.config("cfg1", width=64, height=64, nu=40_000, nu_b=4_000, sigma_pos=0.08, sigma_vel=3.2)
    sc = I.scene(cfg)
    kw = dict(cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params())
    g = dog.Filter(cfg.width, cfg.height, cfg.nu, cfg.nu_b, **kw)
    f = dog.Filter(cfg.width, cfg.height, cfg.nu, cfg.nu_b, devices=[0, 0, 0, 0], **kw)
    streams = [torch.cuda.Stream() for _ in range(4)]
    plan = {2: [(0, 1), (1, 2), (2, 30), (30, 64)], 5: [(0, 40), (40, 41), (41, 43), (43, 64)],
            7: [(0, 16), (16, 32), (32, 48), (48, 64)]}
    for k in range(10):
        if k in plan:
            f.set_bands(plan[k])
            assert f.bands()[0] == plan[k]
        meas = sc.frame(k, device="cuda").contiguous()
        g.step(meas, cfg.dt)
        rows, _ = f.bands()
        torch.cuda.synchronize()
        f.step_sharded([meas[r0:r1].contiguous() for r0, r1 in rows], cfg.dt, streams)
        for s in streams:
            s.synchronize()
        _bits(_state(f.get_state()), _state(g.get_state()), f"cycle {k}: next state")
        cw = g.read_cells()
        outs = f.read_cells_sharded(streams)
        for (r0, r1), ob in zip(rows, outs):
            sl = slice(r0 * cfg.width, r1 * cfg.width)
            _bits(ob["occ"].cpu().numpy(), cw["occ"][sl].cpu().numpy(), f"cycle {k} rows {r0}-{r1}: occ")
            _bits(ob["free"].cpu().numpy(), cw["free"][sl].cpu().numpy(), f"cycle {k} rows {r0}-{r1}: free")
        full = f.read_cells()
        _bits(full["occ"].cpu().numpy(), cw["occ"].cpu().numpy(), f"cycle {k}: occ (whole-grid readout)")
    f.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _two_process_worker(rank, world, port, cfg_kw, cycles, out_path):
    import torch.distributed as dist
    from paper_1605_02406_b200 import dog, shard
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        cfg = I.config("cfg1", **cfg_kw)
        sc = I.scene(cfg)
        t = shard.DistTransport(rank, world, torch.device("cuda", 0), stage_cpu=True)
        sf = shard.ShardedFilter.from_config(cfg, rank, world, t)
        rebal = {3: None, 5: [(0, 2), (2, cfg.height)]}
        moved = []
        results = []
        for k in range(cycles):
            if k in rebal:
                moved.append(sf.rebalance(rows=rebal[k]))
            meas = sc.frame(k, device="cuda").contiguous()
            sf.step(sf.band_of(meas).contiguous(), cfg.dt)
            torch.cuda.synchronize()
            parts, g0 = sf.f.particles()
            allp = t.allgather_var(torch.from_numpy(parts))
            mf = t.allgather_var(torch.from_numpy(sf.f.m_free()))
            occ = t.allgather_var(sf.f.read_cells()["occ"].cpu())
            if rank == 0:
                results.append((np.concatenate([a.numpy() for a in allp]), np.concatenate([a.numpy() for a in mf]),
                                np.concatenate([a.numpy() for a in occ]), list(sf.rows)))
        if rank == 0:
            import pickle
            with open(out_path, "wb") as fh:
                pickle.dump((results, moved), fh)
    finally:
        dist.destroy_process_group()


def test_sharded_filter_two_processes(tmp_path):
    """ShardedFilter.step + ShardedFilter.rebalance (a plan_bands move, then a forced 2-row band) in two
    processes on cuda:0 over gloo, 8 cycles: state, m_F and occupancy bit-identical to the whole grid."""
    import torch.multiprocessing as mp
    from paper_1605_02406_b200 import dog
    cfg_kw = dict(width=48, height=40, nu=20_000, nu_b=2_000, sigma_vel=1.6)
    cycles = 8
    out = str(tmp_path / "sharded.pkl")
    mp.start_processes(_two_process_worker, args=(2, _free_port(), cfg_kw, cycles, out), nprocs=2, join=True,
                       start_method="spawn")
    import pickle
    with open(out, "rb") as fh:
        results, moved = pickle.load(fh)
    assert moved[1]                              # the forced partition always moves
    cfg = I.config("cfg1", **cfg_kw)
    sc = I.scene(cfg)
    g = dog.Filter.from_config(cfg)
    for k in range(cycles):
        g.step(sc.frame(k, device="cuda").contiguous(), cfg.dt)
        st = g.get_state()
        parts, mf, occ, rows = results[k]
        _bits(parts, _state(st), f"cycle {k}: next state (rows {rows})")
        _bits(mf, st["m_free"], f"cycle {k}: m_F")
        _bits(occ, g.read_cells()["occ"].cpu().numpy(), f"cycle {k}: occ")
    assert results[-1][3][0] == (0, 2)
