"""GPU parity of the exact PHD/MIB filter with a single-object likelihood (NEXT-3 general form; Eqs. 38,
49-52; A-38): dog_step_exact_lik through the C ABI vs the oracle's orc_step_exact_lik on the
same seeded inputs (inputs.Scene.exact_lik: observation grid, radar overlay as the likelihood) -- stage
dumps (rho_p, rho_b, fixed-point masses, slots), births, occupancy and the next state bit-exact, velocity
moments within the north-star 1e-4.  Requires a CUDA device."""
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


def compare(o, g, nu_b, tag):
    # (PERM and JOINT_IDX are dumps of k_resample_tiles, which the likelihood tiles bypass)
    for n in ("PRED_X", "PRED_Y", "PRED_VX", "PRED_VY", "KEY", "OFFSETS", "RHO_P", "RHO_B", "RP", "RB", "NB"):
        bits(o.dump(n), g.debug(n), f"{tag}: {n}")
    so, sg = o.scalars(), g.scalars()
    for key in ("W", "U", "A", "n_in", "k"):
        assert so[key] == sg[key], (tag, key, so[key], sg[key])
    nslots = nu_b if so["A"] > 0 else 0
    for n in ("BIRTH_X", "BIRTH_Y", "BIRTH_VX", "BIRTH_VY"):
        bits(o.dump(n)[:nslots], g.debug(n)[:nslots], f"{tag}: {n}")
    co = o.read_cells()
    cg = {key: v.cpu().numpy() for key, v in g.read_cells(check=False).items() if key != "status"}
    bits(co["occ"], cg["occ"], f"{tag}: occ")
    bits(co["free"], cg["free"], f"{tag}: free")
    close(co["mean"], cg["mean"], 1e-4, 1e-6, f"{tag}: mean")
    close(co["cov"][:, :2], cg["cov"][:, :2], 1e-4, 1e-7, f"{tag}: vel_var")
    scale = np.sqrt(np.abs(co["cov"][:, 0] * co["cov"][:, 1])).astype(np.float64)
    assert np.all(np.abs(co["cov"][:, 2].astype(np.float64) - cg["cov"][:, 2]) <= 1e-4 * scale + 1e-7), f"{tag}: cov"
    sto, stg = o.get_state(), g.get_state()
    for key in ("x", "y", "vx", "vy"):
        bits(sto[key], stg[key], f"{tag}: state.{key}")
    assert np.float32(sto["w_bar"]).view(np.uint32) == np.float32(stg["w_bar"]).view(np.uint32)


def dev(t):
    return torch.as_tensor(t).cuda().contiguous()


def run(cfg, steps, p_cl=0.02, frac=0.5, p_assoc=0.8, sd=0.25, **over):
    o, g = pair(cfg, **over)
    sc = I.scene(cfg)
    n_lik = 0
    for k in range(steps):
        meas = sc.frame(k)
        obs, lik, pA = sc.exact_lik(k, meas, p_cl=p_cl, frac=frac, p_assoc=p_assoc, sd=sd)
        n_lik += int(((pA > 0) & (obs[..., 0] > 0)).sum())
        o.step_exact_lik(obs.numpy(), lik.numpy(), pA.numpy(), cfg.dt)
        g.step_exact_lik(dev(obs), dev(lik), dev(pA), cfg.dt)
        compare(o, g, cfg.nu_b, f"cycle {k}")
    assert n_lik > 0
    return o, g


def test_exact_lik_cfg1_lockstep():
    """32x32 moving box, 10k + 1k particles, 8 cycles from the empty state."""
    run(I.CONFIGS["cfg1"], 8)


def test_exact_lik_every_return_associated():
    """p_A = 1 on every cell with a return, a sharp likelihood (sd 0.05 m/s): most members far in the
    tail of g, the split carried by the relative fixed point (A-34)."""
    run(I.CONFIGS["cfg1"], 6, frac=1.0, p_assoc=1.0, sd=0.05, p_cl=0.0)


def test_exact_lik_multitile_scene():
    """256x256 ray-cast scene, 300k particles, 30k births: 4 cycles, likelihood cells spread over tiles."""
    cfg = I.config("cfg2", width=256, height=256, nu=300_000, nu_b=30_000, beams=600, movers=4, peds=3, boxes=15)
    run(cfg, 4)


def test_pA_zero_is_step_exact():
    """p_A = 0 everywhere: dog_step_exact_lik is dog_step_exact bit for bit (GPU against GPU)."""
    from paper_1605_02406_b200 import dog
    cfg = I.CONFIGS["cfg1"]
    kw = dict(cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params())
    a = dog.Filter(cfg.width, cfg.height, cfg.nu, cfg.nu_b, **kw)
    b = dog.Filter(cfg.width, cfg.height, cfg.nu, cfg.nu_b, **kw)
    sc = I.scene(cfg)
    for k in range(5):
        meas = sc.frame(k)
        obs, lik, pA = sc.exact_lik(k, meas)
        a.step_exact(dev(obs), cfg.dt)
        b.step_exact_lik(dev(obs), dev(lik), torch.zeros_like(dev(pA)), cfg.dt)
    sa, sb = a.get_state(), b.get_state()
    for key in ("x", "y", "vx", "vy"):
        bits(sa[key], sb[key], key)
    ra, rb = a.read_cells(check=False), b.read_cells(check=False)
    bits(ra["occ"].cpu().numpy(), rb["occ"].cpu().numpy(), "occ")


def test_injected_random_state():
    """A random injected state (velocities N(0, 3^2), half the cells with a measurement, random p_TP,
    p_FP, p_cl, likelihood directions and p_A), two cycles with fresh draws: bit-exact."""
    from paper_1605_02406_b200 import dog
    W, H, nu, nu_b = 96, 80, 60_000, 6_000
    kw = dict(cell_size=0.1, seed=5, v_max=20.0)
    o = oracle.Oracle(oracle.Params(width=W, height=H, nu=nu, nu_b=nu_b, **kw))
    g = dog.Filter(W, H, nu, nu_b, debug=True, **kw)
    rng = np.random.default_rng(21)
    x = rng.uniform(2, W - 2, nu).astype(np.float32); y = rng.uniform(2, H - 2, nu).astype(np.float32)
    vx = rng.normal(0, 3, nu).astype(np.float32); vy = rng.normal(0, 3, nu).astype(np.float32)
    C = W * H
    mf = np.zeros(C, np.float32)
    o.set_state(x, y, vx, vy, np.float32(0.8 / nu), mf, 3)
    g.set_state(x, y, vx, vy, np.float32(0.8 / nu), mf, 3)
    for k in range(2):
        occ = (rng.random(C) < 0.5).astype(np.float32)
        obs = np.stack([occ, rng.uniform(0.6, 0.95, C), rng.uniform(0.01, 0.2, C), rng.uniform(0.01, 0.3, C)],
                       1).astype(np.float32)
        ang = rng.uniform(0, 2 * np.pi, C)
        lik = np.stack([np.cos(ang), np.sin(ang), rng.normal(0, 3, C), rng.uniform(0.3, 1.5, C)], 1).astype(np.float32)
        pA = np.where(rng.random(C) < 0.7, rng.uniform(0.2, 1.0, C), 0.0).astype(np.float32)
        o.step_exact_lik(obs, lik, pA, 0.1)
        g.step_exact_lik(dev(obs), dev(lik), dev(pA), 0.1)
        compare(o, g, nu_b, f"cycle {k}")


@pytest.mark.slow
def test_exact_lik_full_size_cfgT_one_cycle():
    """cfg T (2048x2048, 8M + 800k): the GPU filter warmed with plain and exact cycles, its state injected
    into the oracle, one cycle with the likelihood on both (the bench's launch configuration): births,
    occupancy and the next state bit for bit."""
    from paper_1605_02406_b200 import dog
    cfg = I.CONFIGS["cfgT"]
    sc = I.scene(cfg)
    g = dog.Filter.from_config(cfg)
    for k in range(6):
        g.step(sc.frame(k, device="cuda"), cfg.dt)
    for k in range(6, 8):
        g.step_exact(I.Scene.exact_obs(sc.frame(k, device="cuda")), cfg.dt)
    st = g.get_state()
    o = oracle.Oracle(oracle.Params(width=cfg.width, height=cfg.height, nu=cfg.nu, nu_b=cfg.nu_b,
                                    cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params()))
    o.set_state(st["x"], st["y"], st["vx"], st["vy"], st["w_bar"], st["m_free"], st["k"])
    meas = sc.frame(8)
    obs, lik, pA = sc.exact_lik(8, meas)
    o.step_exact_lik(obs.numpy(), lik.numpy(), pA.numpy(), cfg.dt)
    g.step_exact_lik(dev(obs), dev(lik), dev(pA), cfg.dt)
    sto, stg = o.get_state(), g.get_state()
    for key in ("x", "y", "vx", "vy"):
        bits(sto[key], stg[key], "state." + key)
    co = o.read_cells()
    cg = {key: v.cpu().numpy() for key, v in g.read_cells(check=False).items() if key != "status"}
    bits(co["occ"], cg["occ"], "occ")
    close(co["mean"], cg["mean"], 1e-4, 1e-6, "mean")


def test_no_measurement_gate_and_no_births():
    """p_A > 0 everywhere but no measurement anywhere: dog_step_exact_lik is dog_step_exact bit for bit (the
    gate); and a filter without birth slots (nu_b = 0) runs the likelihood cycle bit-exact vs the oracle."""
    from paper_1605_02406_b200 import dog
    cfg = I.CONFIGS["cfg1"]
    kw = dict(cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params())
    a = dog.Filter(cfg.width, cfg.height, cfg.nu, cfg.nu_b, **kw)
    b = dog.Filter(cfg.width, cfg.height, cfg.nu, cfg.nu_b, **kw)
    sc = I.scene(cfg)
    for k in range(4):
        meas = sc.frame(k)
        obs, lik, pA = sc.exact_lik(k, meas, frac=1.0)
        obs[..., 0] = 0.0
        a.step_exact(dev(obs), cfg.dt)
        b.step_exact_lik(dev(obs), dev(lik), torch.full_like(dev(pA), 0.9), cfg.dt)
    sa, sb = a.get_state(), b.get_state()
    for key in ("x", "y", "vx", "vy"):
        bits(sa[key], sb[key], key)
    run(I.config("cfg1", nu_b=0), 4)
