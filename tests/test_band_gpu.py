"""Row-band contexts: the union of the bands must reproduce the whole-grid filter bit
for bit -- next state (in global index order), occupancy / free mass and m_F of every cell; velocity
moments within the north-star 1e-4 (their fp64 sums run over the bands' own tiles).  The bands run in
one process on one GPU (paper_1605_02406_b200.shard.LocalBands: phases band after band, exchanges by
device copies), which exercises exactly the device code and the exchange protocol a multi-GPU run uses.
Requires a CUDA device: run with `-m gpu`."""
import numpy as np
import pytest
import torch

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


def run_bands_vs_whole(cfg, world, cycles, frames=None, migrant_cap=None, rebalance=None):
    """rebalance: {cycle: rows or None} -- after that cycle, move the band boundaries (None: plan_bands)."""
    from paper_1605_02406_b200 import dog, shard
    g = dog.Filter.from_config(cfg)
    lb = shard.LocalBands.from_config(cfg, world, migrant_cap=migrant_cap)
    sc = I.scene(cfg) if frames is None else None
    for k in range(cycles):
        if rebalance and (k - 1) in rebalance:
            before = list(lb.rows)
            assert lb.rebalance(min_rows=8, rows=rebalance[k - 1]), (k, before)
            assert lb.rows != before and lb.rows[0][0] == 0 and lb.rows[-1][1] == cfg.height
        meas = (sc.frame(k, device="cuda") if frames is None
                else torch.as_tensor(frames[k]).reshape(cfg.height, cfg.width, 2).cuda())
        g.step(meas.contiguous(), cfg.dt)
        lb.step(meas.contiguous(), cfg.dt)
        torch.cuda.synchronize()
        st = g.get_state()
        whole = np.stack([st["x"], st["y"], st["vx"], st["vy"]], 1)
        parts, spans = lb.particles()
        first = 0
        for g0, n in spans:                     # each band owns a contiguous range of global indices
            if n:
                assert g0 == first, (k, spans)
            first = g0 + n if n else first
        if parts.shape[0]:
            assert parts.shape[0] == cfg.nu, (k, parts.shape)
            _bits(parts, whole, f"cycle {k}: next state")
        cw = g.read_cells()
        for b, f in enumerate(lb.bands):
            r0, r1 = lb.rows[b]
            cb = f.read_cells()
            sl = slice(r0 * cfg.width, r1 * cfg.width)
            _bits(cb["occ"].cpu().numpy(), cw["occ"][sl].cpu().numpy(), f"cycle {k} band {b}: occ")
            _bits(cb["free"].cpu().numpy(), cw["free"][sl].cpu().numpy(), f"cycle {k} band {b}: free")
            _bits(f.m_free(), st["m_free"][sl], f"cycle {k} band {b}: m_F")
            mw, mb = cw["mean"][sl].cpu().numpy(), cb["mean"].cpu().numpy()
            assert np.allclose(mb, mw, rtol=1e-4, atol=1e-6), f"cycle {k} band {b}: mean"
            vw, vb = cw["cov"][sl].cpu().numpy(), cb["cov"].cpu().numpy()
            assert np.allclose(vb, vw, rtol=1e-4, atol=1e-6), f"cycle {k} band {b}: cov"
    return lb


def test_two_bands_cfg1():
    run_bands_vs_whole(I.CONFIGS["cfg1"], 2, 10)


def test_three_bands_multitile_scene():
    """256x256 ray-cast scene, 300k particles (74 tiles), three bands (86/85/85 rows)."""
    cfg = I.config("cfg2", width=256, height=256, nu=300_000, nu_b=30_000, beams=400, movers=6, peds=4,
                   boxes=15)
    run_bands_vs_whole(cfg, 3, 5)


def test_four_bands_fast_movers():
    """Large process noise (4x Table I, SURVEY cfg 5 settings) on a small grid: many migrants per cycle."""
    cfg = I.config("cfg1", width=64, height=64, nu=40_000, nu_b=4_000, sigma_pos=0.08, sigma_vel=3.2)
    run_bands_vs_whole(cfg, 4, 8)


def test_rebalance_bands_bit_exact():
    """NEXT-4 band rebalancing: boundaries moved between cycles -- by plan_bands from the particles per row,
    then to a forced skewed partition -- and the bands keep reproducing the whole grid bit for bit."""
    cfg = I.config("cfg2", width=256, height=256, nu=300_000, nu_b=30_000, beams=400, movers=6, peds=4,
                   boxes=15)
    run_bands_vs_whole(cfg, 3, 7, rebalance={2: None, 4: [(0, 40), (40, 200), (200, 256)]})


def test_doppler_bands_bit_exact():
    """NEXT-1 on row bands: three bands running the Doppler branch (dog_band_assign_doppler) reproduce the
    whole-grid dog_step_doppler bit for bit -- next state in global order, occupancy, m_F."""
    from paper_1605_02406_b200 import dog, shard
    cfg = I.config("cfg2", width=256, height=256, nu=300_000, nu_b=30_000, beams=400, movers=6, peds=4,
                   boxes=15)
    g = dog.Filter.from_config(cfg)
    lb = shard.LocalBands.from_config(cfg, 3)
    sc = I.scene(cfg)
    for k in range(6):
        meas = sc.frame(k, device="cuda").contiguous()
        if k < 2:
            g.step(meas, cfg.dt)
            lb.step(meas, cfg.dt)
        else:
            dop, pA = sc.doppler(k, meas, frac=0.7)
            dop, pA = dop.cuda().contiguous(), pA.cuda().contiguous()
            g.step_doppler(meas, dop, pA, cfg.dt)
            lb.step(meas, cfg.dt, doppler=(dop, pA))
        torch.cuda.synchronize()
        st = g.get_state()
        whole = np.stack([st["x"], st["y"], st["vx"], st["vy"]], 1)
        parts, _ = lb.particles()
        _bits(parts, whole, f"cycle {k}: next state")
        cw = g.read_cells()
        for b, f in enumerate(lb.bands):
            r0, r1 = lb.rows[b]
            sl = slice(r0 * cfg.width, r1 * cfg.width)
            _bits(f.read_cells()["occ"].cpu().numpy(), cw["occ"][sl].cpu().numpy(), f"cycle {k} band {b}: occ")
            _bits(f.m_free(), st["m_free"][sl], f"cycle {k} band {b}: m_F")
            mb, mw = f.read_cells()["mean"].cpu().numpy(), cw["mean"][sl].cpu().numpy()
            assert np.allclose(mb, mw, rtol=1e-4, atol=1e-6), f"cycle {k} band {b}: mean"


def test_exact_bands_bit_exact():
    """NEXT-3 on row bands: three bands running the exact PHD/MIB cycle (dog_band_assign_exact; every cell
    of a band in its list, births over the whole grid on the global born-mass CDF) reproduce the
    whole-grid dog_step_exact bit for bit."""
    from paper_1605_02406_b200 import dog, shard
    cfg = I.config("cfg2", width=128, height=96, nu=60_000, nu_b=6_000, beams=300, movers=3, peds=2, boxes=6)
    g = dog.Filter.from_config(cfg)
    lb = shard.LocalBands.from_config(cfg, 3)
    sc = I.scene(cfg)
    for k in range(6):
        meas = sc.frame(k, device="cuda").contiguous()
        if k < 2:
            g.step(meas, cfg.dt)
            lb.step(meas, cfg.dt)
        else:
            obs = I.Scene.exact_obs(meas)
            g.step_exact(obs, cfg.dt)
            lb.step(meas, cfg.dt, obs=obs)
        torch.cuda.synchronize()
        st = g.get_state()
        whole = np.stack([st["x"], st["y"], st["vx"], st["vy"]], 1)
        parts, _ = lb.particles()
        _bits(parts, whole, f"cycle {k}: next state")
        cw = g.read_cells()
        for b, f in enumerate(lb.bands):
            r0, r1 = lb.rows[b]
            sl = slice(r0 * cfg.width, r1 * cfg.width)
            _bits(f.read_cells()["occ"].cpu().numpy(), cw["occ"][sl].cpu().numpy(), f"cycle {k} band {b}: occ")
