"""GPU parity of the Doppler / association branch (NEXT-1): dog_step_doppler through the C ABI vs the
oracle's orc_step_doppler on the same seeded scene, radar overlay and injected states -- stage dumps
and the next state bit-exact, velocity moments within the north-star 1e-4 relative tolerance.
Requires a CUDA device."""
import numpy as np
import pytest
import torch

import oracle
from paper_1605_02406_b200 import inputs as I

pytestmark = pytest.mark.gpu


def pair(cfg, **over):
    from paper_1605_02406_b200 import dog
    kw = dict(cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params())
    kw.update(over)
    g = dog.Filter(cfg.width, cfg.height, cfg.nu, cfg.nu_b, debug=True, **kw)
    o = oracle.Oracle(oracle.Params(width=cfg.width, height=cfg.height, nu=cfg.nu, nu_b=cfg.nu_b, **kw))
    return o, g


def bits(a, b, what):
    a = np.ascontiguousarray(a); b = np.ascontiguousarray(b)
    if a.dtype == np.float32:
        a, b = a.view(np.uint32), b.view(np.uint32)
    bad = np.nonzero(a != b)[0]
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first at {bad[:5]}: {a[bad[:5]]} vs {b[bad[:5]]}"


def close(a, b, rel, abs_, what):
    a = a.astype(np.float64).reshape(-1); b = b.astype(np.float64).reshape(-1)
    bad = np.nonzero(np.abs(a - b) > rel * np.maximum(np.abs(a), np.abs(b)) + abs_)[0]
    assert bad.size == 0, f"{what}: {bad.size} beyond tolerance, first {bad[:5]}: {a[bad[:5]]} vs {b[bad[:5]]}"


def compare(o, g, nu_b):
    # (PERM and JOINT_IDX are dumps of k_resample_tiles, which this path replaces)
    for n in ("PRED_X", "PRED_Y", "PRED_VX", "PRED_VY", "KEY", "OFFSETS", "RHO_P", "RHO_B", "RP", "RB", "NB"):
        bits(o.dump(n), g.debug(n), n)
    so, sg = o.scalars(), g.scalars()
    for k in ("W", "U", "A", "n_in", "k"):
        assert so[k] == sg[k], (k, so[k], sg[k])
    nslots = nu_b if so["A"] > 0 else 0
    for n in ("BIRTH_X", "BIRTH_Y", "BIRTH_VX", "BIRTH_VY"):
        bits(o.dump(n)[:nslots], g.debug(n)[:nslots], n)
    co = o.read_cells()
    cg = {k: v.cpu().numpy() for k, v in g.read_cells(check=False).items() if k != "status"}
    bits(co["occ"], cg["occ"], "occ")
    close(co["mean"], cg["mean"], 1e-4, 1e-6, "vel_mean")
    close(co["cov"][:, :2], cg["cov"][:, :2], 1e-4, 1e-7, "vel_var")
    scale = np.sqrt(np.abs(co["cov"][:, 0] * co["cov"][:, 1])).astype(np.float64)
    assert np.all(np.abs(co["cov"][:, 2].astype(np.float64) - cg["cov"][:, 2]) <= 1e-4 * scale + 1e-7), "vel_cov"
    sto, stg = o.get_state(), g.get_state()
    for k in ("x", "y", "vx", "vy", "m_free"):
        bits(sto[k], stg[k], "state." + k)
    assert np.float32(sto["w_bar"]).view(np.uint32) == np.float32(stg["w_bar"]).view(np.uint32)


def run(cfg, steps, plain=2, frac=0.5, p_assoc=0.8, sd=0.25, **over):
    """`plain` ordinary cycles to populate the grid, then `steps` Doppler cycles, all in lockstep."""
    o, g = pair(cfg, **over)
    sc = I.scene(cfg)
    n_dop_cells = 0
    for k in range(plain + steps):
        meas = sc.frame(k)
        mg = meas.cuda().contiguous()
        if k < plain:
            o.step(meas.numpy(), cfg.dt)
            g.step(mg, cfg.dt)
            continue
        dop, pA = sc.doppler(k, meas, frac=frac, p_assoc=p_assoc, sd=sd)
        n_dop_cells += int((pA > 0).sum())
        o.step_doppler(meas.numpy(), dop.numpy(), pA.numpy(), cfg.dt)
        g.step_doppler(mg, dop.cuda().contiguous(), pA.cuda().contiguous(), cfg.dt)
        compare(o, g, cfg.nu_b)
    assert n_dop_cells > 0
    return o, g


def test_doppler_cfg1_lockstep():
    """32x32 moving box, 10k + 1k particles: 2 plain cycles, then 8 Doppler cycles -- and the branch
    matters: the same cycles without the Doppler grid end in a different state."""
    cfg = I.CONFIGS["cfg1"]
    o, g = run(cfg, 8, frac=0.7)
    ref = oracle.Oracle(oracle.Params(width=cfg.width, height=cfg.height, nu=cfg.nu, nu_b=cfg.nu_b,
                                      cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params()))
    sc = I.scene(cfg)
    for k in range(10):
        ref.step(sc.frame(k).numpy(), cfg.dt)
    a, b = ref.get_state(), g.get_state()
    assert not np.array_equal(a["vx"], b["vx"])


def test_doppler_multitile_scene():
    """256x256 ray-cast scene, 300k particles (74 sort tiles), sharp and broad likelihoods, p_A = 1."""
    cfg = I.config("cfg2", width=256, height=256, nu=300_000, nu_b=30_000, beams=600, movers=4, peds=3, boxes=15)
    run(cfg, 3, plain=3, frac=0.6, p_assoc=1.0, sd=0.1)
    run(cfg, 2, plain=2, frac=0.3, p_assoc=0.4, sd=2.0)


def test_doppler_all_zero_pA_is_the_plain_cycle():
    """p_A = 0 everywhere: dog_step_doppler reproduces dog_step bit for bit (and the oracle's orc_step)."""
    from paper_1605_02406_b200 import dog
    cfg = I.config("cfg1", width=37, height=23, nu=10_007, nu_b=999)
    sc = I.scene(cfg)
    kw = dict(cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params())
    a = dog.Filter(cfg.width, cfg.height, cfg.nu, cfg.nu_b, **kw)
    b = dog.Filter(cfg.width, cfg.height, cfg.nu, cfg.nu_b, **kw)
    dop = torch.zeros(cfg.C, 4, device="cuda"); pA = torch.zeros(cfg.C, device="cuda")
    for k in range(5):
        m = sc.frame(k).cuda().contiguous()
        a.step(m, cfg.dt)
        b.step_doppler(m, dop, pA, cfg.dt)
        sa, sb = a.get_state(), b.get_state()
        for key in ("x", "y", "vx", "vy", "m_free"):
            bits(sa[key], sb[key], f"cycle {k} {key}")
        ra, rb = a.read_cells(), b.read_cells()
        close(ra["mean"].cpu().numpy(), rb["mean"].cpu().numpy(), 1e-6, 1e-9, "mean")


def test_doppler_without_side_stream(monkeypatch):
    """The same cycles with every kernel on the caller's stream (DOG_NO_FORK: no side stream)."""
    monkeypatch.setenv("DOG_NO_FORK", "1")
    run(I.CONFIGS["cfg1"], 4, frac=0.7)


@pytest.mark.slow
def test_doppler_full_size_cfgT_one_cycle():
    """The bench configuration (cfg T: 2048x2048, 8M + 800k) with the bench's radar overlay: warm the GPU
    filter with plain cycles, inject its state into the oracle, run one Doppler cycle on both, compare
    the next state bit for bit and the moments within 1e-4."""
    from paper_1605_02406_b200 import dog
    cfg = I.CONFIGS["cfgT"]
    sc = I.scene(cfg)
    g = dog.Filter.from_config(cfg)
    for k in range(6):
        g.step(sc.frame(k, device="cuda"), cfg.dt)
    st = g.get_state()
    o = oracle.Oracle(oracle.Params(width=cfg.width, height=cfg.height, nu=cfg.nu, nu_b=cfg.nu_b,
                                    cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params()))
    o.set_state(st["x"], st["y"], st["vx"], st["vy"], st["w_bar"], st["m_free"], st["k"])
    meas = sc.frame(6)
    dop, pA = sc.doppler(6, meas, frac=0.5, p_assoc=0.8, sd=0.25)
    assert int((pA > 0).sum()) > 100
    o.step_doppler(meas.numpy(), dop.numpy(), pA.numpy(), cfg.dt)
    g.step_doppler(meas.cuda().contiguous(), dop.cuda().contiguous(), pA.cuda().contiguous(), cfg.dt)
    sto, stg = o.get_state(), g.get_state()
    for key in ("x", "y", "vx", "vy", "m_free"):
        bits(sto[key], stg[key], "state." + key)
    co = o.read_cells()
    cg = {key: v.cpu().numpy() for key, v in g.read_cells(check=False).items() if key != "status"}
    bits(co["occ"], cg["occ"], "occ")
    close(co["mean"], cg["mean"], 1e-4, 1e-6, "vel_mean")


def test_doppler_incompatible_cells_fall_back():
    """A radial-speed SD so small (1e-5 m/s) that every member of most cells is more than 13.2 SD away,
    so its f32 likelihood underflows to 0 (A-34): those cells take the GS = 0 guard (the mu_A term
    dropped, even split, A-35) -- bit-exact like the rest."""
    cfg = I.config("cfg1", nu=20_000, nu_b=2_000)
    o, g = run(cfg, 4, plain=3, frac=1.0, p_assoc=1.0, sd=1e-5)
    sc = I.scene(cfg)
    _, pA = sc.doppler(6, sc.frame(6), frac=1.0, p_assoc=1.0, sd=1e-5)   # the last cycle's overlay
    off, gs = o.dump("OFFSETS"), o.dump("GS")
    members = np.diff(off.astype(np.int64)) > 0
    doppler_cells = (pA.numpy().reshape(-1) > 0) & members
    assert doppler_cells.sum() > 0 and (gs[doppler_cells] == 0).sum() > 0
