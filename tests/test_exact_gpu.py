"""GPU parity of the exact PHD/MIB filter (NEXT-3): dog_step_exact through the C ABI vs the oracle's
orc_step_exact on the same seeded scene (observation grids from inputs.Scene.exact_obs) -- stage
dumps, masses, joint indices and the next state bit-exact, velocity moments within 1e-4.  Requires a
CUDA device."""
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


def run(cfg, steps, **over):
    o, g = pair(cfg, **over)
    sc = I.scene(cfg)
    for k in range(steps):
        obs = I.Scene.exact_obs(sc.frame(k))
        o.step_exact(obs.numpy(), cfg.dt)
        g.step_exact(obs.cuda().contiguous(), cfg.dt)
        for n in ("PRED_X", "PRED_Y", "PRED_VX", "PRED_VY", "KEY", "PERM", "OFFSETS", "RHO_P", "RHO_B", "RP", "RB", "NB",
                  "JOINT_IDX"):
            bits(o.dump(n), g.debug(n), f"cycle {k}: {n}")
        so, sg = o.scalars(), g.scalars()
        for key in ("W", "U", "A", "n_in", "k"):
            assert so[key] == sg[key], (k, key, so[key], sg[key])
        nslots = cfg.nu_b if so["A"] > 0 else 0
        for n in ("BIRTH_X", "BIRTH_Y", "BIRTH_VX", "BIRTH_VY"):
            bits(o.dump(n)[:nslots], g.debug(n)[:nslots], f"cycle {k}: {n}")
        co = o.read_cells()
        cg = {key: v.cpu().numpy() for key, v in g.read_cells(check=False).items() if key != "status"}
        bits(co["occ"], cg["occ"], f"cycle {k}: occ")
        bits(co["free"], cg["free"], f"cycle {k}: free")
        close(co["mean"], cg["mean"], 1e-4, 1e-6, f"cycle {k}: mean")
        sto, stg = o.get_state(), g.get_state()
        for key in ("x", "y", "vx", "vy", "m_free"):
            bits(sto[key], stg[key], f"cycle {k}: state.{key}")
    return o, g


def test_exact_cfg1_lockstep():
    """32x32 moving box, 10k + 1k particles, 8 cycles of the exact filter from the empty state."""
    run(I.CONFIGS["cfg1"], 8)


def test_exact_multitile_scene():
    """256x256 ray-cast scene, 300k particles, 30k births spread over the whole grid (every cell has
    r_b > 0): 4 cycles."""
    cfg = I.config("cfg2", width=256, height=256, nu=300_000, nu_b=30_000, beams=600, movers=4, peds=3, boxes=15)
    run(cfg, 4)


@pytest.mark.slow
def test_exact_full_size_cfgT_one_cycle():
    """cfg T (2048x2048, 8M + 800k): the GPU filter warmed with plain cycles, its state injected into the
    oracle, one exact PHD/MIB cycle on both (every cell in the active list): next state bit for bit."""
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
    obs = I.Scene.exact_obs(sc.frame(6))
    o.step_exact(obs.numpy(), cfg.dt)
    g.step_exact(obs.cuda().contiguous(), cfg.dt)
    sto, stg = o.get_state(), g.get_state()
    for key in ("x", "y", "vx", "vy"):
        bits(sto[key], stg[key], "state." + key)
    co = o.read_cells()
    cg = {key: v.cpu().numpy() for key, v in g.read_cells(check=False).items() if key != "status"}
    bits(co["occ"], cg["occ"], "occ")


def test_exact_then_plain_cycles_alternate():
    """Mode switches on one filter: exact cycles (dense list, no PDL), plain Dempster-Shafer cycles
    (compacted list, cluster scan), exact again -- every cycle bit-exact with the oracle."""
    cfg = I.config("cfg2", width=128, height=96, nu=40_000, nu_b=4_000, beams=300, movers=3, peds=2, boxes=6)
    o, g = pair(cfg)
    sc = I.scene(cfg)
    for k, mode in enumerate(["plain", "exact", "exact", "plain", "plain", "exact", "plain"]):
        meas = sc.frame(k)
        if mode == "exact":
            obs = I.Scene.exact_obs(meas)
            o.step_exact(obs.numpy(), cfg.dt)
            g.step_exact(obs.cuda().contiguous(), cfg.dt)
        else:
            o.step(meas.numpy(), cfg.dt)
            g.step(meas.cuda().contiguous(), cfg.dt)
        for n in ("KEY", "OFFSETS", "RHO_P", "RHO_B", "RP", "RB", "NB", "JOINT_IDX"):
            bits(o.dump(n), g.debug(n), f"cycle {k} ({mode}): {n}")
        sto, stg = o.get_state(), g.get_state()
        for key in ("x", "y", "vx", "vy", "m_free"):
            bits(sto[key], stg[key], f"cycle {k} ({mode}): state.{key}")
        co = o.read_cells()
        cg = {key: v.cpu().numpy() for key, v in g.read_cells(check=False).items() if key != "status"}
        bits(co["occ"], cg["occ"], f"cycle {k} ({mode}): occ")
        close(co["mean"], cg["mean"], 1e-4, 1e-6, f"cycle {k} ({mode}): mean")
