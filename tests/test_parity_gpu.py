"""GPU parity: libdog.so (through its C ABI) vs the CPU oracle, element by element, on the same seeded
inputs and the same injected states.  Bit-exact on every integer / index / f32-state output; masses are
expected (and checked) bit-identical; velocity moments within the north-star 1e-4 relative tolerance
(DESIGN.md section 4).  Requires a CUDA device: run with `-m gpu`."""
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
    oracle.build()
    torch.cuda.set_device(0)


def pair(cfg, **over):
    from paper_1605_02406_b200 import dog
    kw = dict(cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params())
    kw.update(over)
    g = dog.Filter(cfg.width, cfg.height, cfg.nu, cfg.nu_b, debug=True, **kw)
    o = oracle.Oracle(oracle.Params(width=cfg.width, height=cfg.height, nu=cfg.nu, nu_b=cfg.nu_b, **kw))
    return o, g


def inject(o, g, st):
    o.set_state(st["x"], st["y"], st["vx"], st["vy"], st["w_bar"], st["m_free"], st["k"])
    g.set_state(st["x"], st["y"], st["vx"], st["vy"], st["w_bar"], st["m_free"], st["k"])


def assert_bits(a, b, what):
    a = np.ascontiguousarray(a); b = np.ascontiguousarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    if a.dtype == np.float32:
        a, b = a.view(np.uint32), b.view(np.uint32)
    bad = np.nonzero(a != b)[0]
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first at {bad[:5]}: {a[bad[:5]]} vs {b[bad[:5]]}"


def rel_close(a, b, rel, abs_, what):
    a = a.astype(np.float64); b = b.astype(np.float64)
    tol = rel * np.maximum(np.abs(a), np.abs(b)) + abs_
    bad = np.nonzero(np.abs(a - b) > tol)[0]
    assert bad.size == 0, f"{what}: {bad.size} beyond tolerance, first {bad[:5]}: {a[bad[:5]]} vs {b[bad[:5]]}"


def compare_cycle(o, g, rc_gpu=None):
    """Stage-by-stage comparison of the last cycle."""
    for n in ("PRED_X", "PRED_Y", "PRED_VX", "PRED_VY", "KEY", "PERM", "OFFSETS", "RHO_P", "RHO_B", "RP",
              "RB", "NB", "JOINT_IDX"):
        assert_bits(o.dump(n), g.debug(n), n)
    so, sg = o.scalars(), g.scalars()
    for k in ("W", "U", "A", "n_in", "k"):
        assert so[k] == sg[k], (k, so[k], sg[k])
    for k in ("w_pred", "w_bar"):
        assert np.float32(so[k]).view(np.uint32) == np.float32(sg[k]).view(np.uint32), k
    nslots = g.nu_b if so["A"] > 0 else 0
    for n in ("BIRTH_X", "BIRTH_Y", "BIRTH_VX", "BIRTH_VY"):
        assert_bits(o.dump(n)[:nslots], g.debug(n)[:nslots], n)
    co = o.read_cells()
    cg = {k: v.cpu().numpy() for k, v in g.read_cells(check=False).items() if k != "status"}
    assert_bits(co["occ"], cg["occ"], "occ")
    assert_bits(co["free"], cg["free"], "free")
    mo, mg = co["mean"].reshape(-1), cg["mean"].reshape(-1)
    rel_close(mo, mg, 1e-4, 1e-6, "vel_mean")
    vo, vg = co["cov"].reshape(-1, 3), cg["cov"].reshape(-1, 3)
    rel_close(vo[:, :2].reshape(-1), vg[:, :2].reshape(-1), 1e-4, 1e-8, "vel_var")
    scale = np.sqrt(np.abs(vo[:, 0] * vo[:, 1])).astype(np.float64)
    assert np.all(np.abs(vo[:, 2].astype(np.float64) - vg[:, 2]) <= 1e-4 * scale + 1e-8), "vel_cov"
    sto, stg = o.get_state(), g.get_state()
    for k in ("x", "y", "vx", "vy", "m_free"):
        assert_bits(sto[k], stg[k], "state." + k)
    assert sto["k"] == stg["k"]


def run_lockstep(cfg, steps, st=None, frames=None, ego=None, **over):
    o, g = pair(cfg, **over)
    if st is not None:
        inject(o, g, st)
    sc = I.scene(cfg) if frames is None else None
    for k in range(steps):
        if ego is not None and k > 0:                        # ego-motion compensation between cycles (NEXT-2)
            dx, dy = ego[k]
            so, sg = o.ego_scroll(dx, dy), g.ego_scroll(dx, dy)
            assert so == sg, (k, so, sg)
            assert o.ego_residual() == g.ego_residual(), k
            a, b = o.get_state(), g.get_state()
            for key in ("x", "y", "vx", "vy", "m_free"):
                assert_bits(a[key], b[key], f"ego scroll {k}: {key}")
        meas = frames[k] if frames is not None else sc.frame(k).numpy()
        o.step(meas, cfg.dt)
        g.step(torch.from_numpy(np.ascontiguousarray(meas, np.float32)).cuda(), cfg.dt)
        compare_cycle(o, g)
    return o, g


def test_cfg1_lockstep_10_cycles():
    """BASELINE configs[0]: 32x32, 10k + 1k particles, moving box, 10 cycles from the empty state."""
    run_lockstep(I.CONFIGS["cfg1"], 10)


def test_ego_motion_compensation():
    """NEXT-2: the grid and the particles scrolled between cycles (positive, negative, zero and sub-cell
    deltas; the residual carries over) -- scroll result and every following cycle bit-exact."""
    rng = np.random.default_rng(11)
    ego = [tuple(rng.uniform(-0.35, 0.35, 2)) for _ in range(8)]
    ego[3] = (0.0, 0.0)
    ego[5] = (0.04, -0.03)
    run_lockstep(I.CONFIGS["cfg1"], 8, ego=ego)


def test_grid_origin_follows_the_ego_shifts():
    """dog_grid's origin (world metres of cell (0, 0)) is kept by the context and moved by -shift * cell_size
    for every applied ego shift (content moves by +shift cells), so world <-> cell stays consistent."""
    from paper_1605_02406_b200 import dog
    cfg = I.CONFIGS["cfg1"]
    f = dog.Filter(cfg.width, cfg.height, cfg.nu, cfg.nu_b, cell_size=cfg.cell_size, origin=(12.5, -3.25))
    assert f.origin() == (12.5, -3.25)
    cs = float(np.float32(cfg.cell_size))
    ox, oy = 12.5, -3.25
    for dx, dy in [(0.35, -0.12), (-0.71, 0.0), (0.04, 0.33), (0.0, 0.0)]:
        sx, sy = f.ego_scroll(dx, dy)
        ox -= sx * cs
        oy -= sy * cs
        assert f.origin() == (ox, oy), (dx, dy, f.origin(), (ox, oy))


def test_sharded_context_keeps_the_origin():
    """A sharded context (two bands on cuda:0) reports the dog_grid origin it was created with."""
    from paper_1605_02406_b200 import dog
    cfg = I.CONFIGS["cfg1"]
    f = dog.Filter(cfg.width, cfg.height, cfg.nu, cfg.nu_b, cell_size=cfg.cell_size, devices=[0, 0],
                   origin=(-7.5, 102.25))
    assert f.origin() == (-7.5, 102.25)
    f.close()


def test_dense_scene_long_list_paths():
    """A cfg-5-like dense scene (i.i.d. measured cells, 4x process noise, p_B 0.1) on 96x96 cells: from
    the third cycle the active list exceeds C/4, so the library switches to the grid-wide list scan and
    the lane-per-cell pair sort, moments and per-slot births -- every stage stays bit-exact with the
    oracle (the switch must not change a result)."""
    cfg = I.config("cfg5", width=96, height=96, nu=120_000, nu_b=30_000)
    o, g = run_lockstep(cfg, 7)
    assert o.scalars()["n_in"] > 0
    n_c = np.diff(o.dump("OFFSETS").astype(np.int64))
    active = int(np.count_nonzero((n_c > 0) | (o.dump("RB") > 0)))
    assert active > cfg.C // 4, (active, cfg.C)              # the run-heavy paths were taken


def test_exact_resampling_fallback_forced(monkeypatch):
    """The exact 128-bit path of F(X) (dog_fcount.cuh), which the fp64 estimates hand over to when they
    land within the margin of an integer (a few members per cycle at cfg T), forced for every member and
    output boundary (DOG_FORCE_EXACT_F): the cycles stay bit-exact with the oracle's binary search."""
    monkeypatch.setenv("DOG_FORCE_EXACT_F", "1")
    run_lockstep(I.config("cfg2", width=128, height=128, nu=120_000, nu_b=12_000, beams=300, movers=3, peds=2,
                          boxes=6), 4)


def test_ragged_sizes():
    """nu not a multiple of 4 / of the 4096-element sort tile, odd nu_b, non-square grid."""
    cfg = I.config("cfg1", width=37, height=23, nu=10_007, nu_b=999)
    run_lockstep(cfg, 6)


def test_no_births():
    """nu_b = 0 with an injected population: no birth kernel, pure persistence."""
    cfg = I.config("cfg1", nu=20_000, nu_b=0)
    rng = np.random.default_rng(3)
    st = I.cells_state(cfg, rng.integers(0, 30, cfg.C) * (rng.random(cfg.C) < 0.5), 0.01, rng=rng,
                       vel=(1.0, -0.5), vel_sd=2.0)
    run_lockstep(cfg, 4, st=st)


def test_multitile_scene():
    """A 256x256 ray-cast scene with 300k particles (74 sort tiles, 16 cell tiles) for 5 cycles."""
    cfg = I.config("cfg2", width=256, height=256, nu=300_000, nu_b=30_000, beams=600, movers=4, peds=3,
                   boxes=15)
    run_lockstep(cfg, 5)


def test_single_cell_holds_everything():
    """One cell holds every particle (one segment spanning every moments range and sort tile)."""
    cfg = I.config("cfg1", width=16, height=16, nu=50_000, nu_b=5_000, sigma_pos=0.0, sigma_vel=0.0)
    counts = np.zeros(cfg.C, np.int64); counts[77] = cfg.nu
    st = I.cells_state(cfg, counts, 1.0 / cfg.nu, vel=(0.0, 0.0), vel_sd=3.0)
    meas = np.zeros((3, cfg.C, 2), np.float32); meas[:, 77, 0] = 0.9; meas[:, :77, 1] = 0.5
    run_lockstep(cfg, 3, st=st, frames=meas)


def test_all_particles_leave_the_grid():
    """Every particle predicted outside (sentinel key C): no persistent mass, births only."""
    cfg = I.config("cfg1", nu=5_000, nu_b=500, sigma_pos=0.0, sigma_vel=0.0)
    st = I.cells_state(cfg, np.r_[np.zeros(cfg.C - 1, int), [cfg.nu]], 1.0 / cfg.nu, vel=(50.0, 0.0))
    meas = np.zeros((2, cfg.C, 2), np.float32); meas[:, 5, 0] = 0.8
    run_lockstep(cfg, 2, st=st, frames=meas)


def test_empty_world_stays_empty():
    cfg = I.CONFIGS["cfg1"]
    meas = np.zeros((3, cfg.C, 2), np.float32); meas[..., 1] = 0.4
    o, g = run_lockstep(cfg, 3, frames=meas)
    assert g.scalars()["W"] == 0


def test_bayesian_injection():
    """The P-BBF setup (p_S = 1, alpha = 1, sigma = 0, p_B = 0) with Bayesian measurements."""
    cfg = I.config("cfg1", nu=1024 * 50, nu_b=0, p_s=1.0, p_b=0.0, sigma_pos=0.0, sigma_vel=0.0,
                   free_tau=float("inf"))
    rng = np.random.default_rng(5)
    st = I.cells_state(cfg, rng.integers(5, 50, cfg.C), 1.0 / 50, rng=rng)
    st["m_free"] = np.clip(1 - st["w_bar"] * np.bincount(
        (st["y"][st["x"] >= 0].astype(int) * 32 + st["x"][st["x"] >= 0].astype(int)), minlength=cfg.C),
        0, 1).astype(np.float32)
    z = rng.uniform(0.05, 0.95, (4, cfg.C)).astype(np.float32)
    frames = np.stack([z, 1 - z], -1).astype(np.float32)
    run_lockstep(cfg, 4, st=st, frames=frames)


def test_invalid_measurement_cells():
    """A-27: NaN / negative / over-unity cells are treated as vacuous on both sides and reported
    as DOG_E_MEAS by the next synchronous call."""
    from paper_1605_02406_b200 import dog
    cfg = I.CONFIGS["cfg1"]
    sc = I.scene(cfg)
    frames = [sc.frame(k).numpy().reshape(-1, 2).copy() for k in range(3)]
    frames[1][3] = [np.nan, 0.1]; frames[1][4] = [-0.1, 0.2]; frames[1][5] = [0.7, 0.6]
    o, g = pair(cfg)
    for k in range(3):
        o.step(frames[k], cfg.dt)
        g.step(torch.from_numpy(frames[k]).cuda(), cfg.dt)
        rc = g.read_cells(check=False)["status"]
        assert rc == (dog.DOG_E_MEAS if k == 1 else dog.DOG_OK)
        compare_cycle(o, g)


def test_resume_bit_exact_and_host_entry():
    """dog_get_state / dog_set_state resume exactly (counter-based RNG), and dog_step_host (host
    buffers, the end-to-end entry) computes the same cycle as dog_step."""
    from paper_1605_02406_b200 import dog
    cfg = I.CONFIGS["cfg1"]
    sc = I.scene(cfg)
    a = dog.Filter.from_config(cfg)
    for k in range(4):
        a.step(sc.frame(k).cuda(), cfg.dt)
    st = a.get_state()
    b = dog.Filter.from_config(cfg)
    b.set_state(st["x"], st["y"], st["vx"], st["vy"], st["w_bar"], st["m_free"], st["k"])
    occ_host = torch.empty(cfg.C).pin_memory()
    for k in range(4, 7):
        a.step(sc.frame(k).cuda(), cfg.dt)
        b.step_host(sc.frame(k).contiguous().pin_memory(), cfg.dt, occ_host)
        assert torch.equal(a.read_cells()["occ"].cpu(), occ_host)
    sa, sb = a.get_state(), b.get_state()
    for k in ("x", "y", "vx", "vy", "m_free"):
        assert_bits(sa[k], sb[k], k)


def test_profile_stages():
    from paper_1605_02406_b200 import dog
    cfg = I.CONFIGS["cfg1"]
    f = dog.Filter.from_config(cfg)
    f.profile_begin(3)
    meas = I.scene(cfg).frame(0).cuda()
    for _ in range(3):
        f.step(meas, cfg.dt)
    stages, n = f.profile_end()
    assert n == 3 and "predict_sort" in stages and "resample" in stages and all(v >= 0 for v in stages.values())


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfgT", "cfg4", "cfg5"])
def test_full_size_one_cycle(name):
    """Every BASELINE.json configuration at its full size -- cfg2 (512x512, 2M + 200k), cfg3 (1024x1024,
    8M + 800k), the bench's cfg T (2048x2048, 8M + 800k), cfg4 (2048x2048, 32M + 3.2M, on one GPU) and
    the cfg5 stress case (1024x1024, 8M + 2M, 4x noise, p_B 0.1) -- in the bench's launch configuration:
    warm the GPU filter for 6 cycles, inject its state into the oracle, run one more cycle on both and
    compare every stage element by element.  Particles predicted within 2^-20 cells of a cell boundary
    are counted and reported separately (north star); their keys are checked like every other one.
    A second filter in the release configuration bench.py times (no debug dumps: the kernels without
    their debug stores) runs the same seven cycles; its next state and readouts must equal the oracle's
    too (bit-exact; moments within 1e-4)."""
    from paper_1605_02406_b200 import dog
    cfg = I.CONFIGS[name]
    sc = I.scene(cfg)
    g = dog.Filter.from_config(cfg, debug=True)
    r = dog.Filter.from_config(cfg)
    for k in range(6):
        m = sc.frame(k, device="cuda")
        g.step(m, cfg.dt)
        r.step(m, cfg.dt)
    st = g.get_state()
    o = oracle.Oracle(oracle.Params(width=cfg.width, height=cfg.height, nu=cfg.nu, nu_b=cfg.nu_b,
                                    cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params()))
    o.set_state(st["x"], st["y"], st["vx"], st["vy"], st["w_bar"], st["m_free"], st["k"])
    meas = sc.frame(6).numpy()
    o.step(meas, cfg.dt)
    g.step(torch.from_numpy(meas).cuda(), cfg.dt)
    px, py = o.dump("PRED_X").astype(np.float64), o.dump("PRED_Y").astype(np.float64)
    near = (np.abs(px - np.round(px)) < 2.0 ** -20) | (np.abs(py - np.round(py)) < 2.0 ** -20)
    assert_bits(o.dump("KEY")[near], g.debug("KEY")[near], "keys of near-boundary particles")
    print(f"{name}: {int(near.sum())} of {cfg.nu} particles within 2^-20 cells of a cell boundary")
    compare_cycle(o, g)
    r.step(torch.from_numpy(meas).cuda(), cfg.dt)
    sto, str_ = o.get_state(), r.get_state()
    for key in ("x", "y", "vx", "vy", "m_free"):
        assert_bits(sto[key], str_[key], "release state." + key)
    co = o.read_cells()
    cr = {key: v.cpu().numpy() for key, v in r.read_cells(check=False).items() if key != "status"}
    assert_bits(co["occ"], cr["occ"], "release occ")
    assert_bits(co["free"], cr["free"], "release free")
    rel_close(co["mean"].reshape(-1), cr["mean"].reshape(-1), 1e-4, 1e-6, "release vel_mean")
    vo, vr = co["cov"].reshape(-1, 3), cr["cov"].reshape(-1, 3)
    rel_close(vo[:, :2].reshape(-1), vr[:, :2].reshape(-1), 1e-4, 1e-8, "release vel_var")
    scale = np.sqrt(np.abs(vo[:, 0] * vo[:, 1])).astype(np.float64)
    assert np.all(np.abs(vo[:, 2].astype(np.float64) - vr[:, 2]) <= 1e-4 * scale + 1e-8), "release vel_cov"
    r.close()


def test_transforms_exhaustive():
    """The kernels' range-specialised division and square root (ln spec, Box-Muller radius) equal IEEE
    div.rn / sqrt.rn on the whole input domain (every odd m in [1, 2^24)), and the packed two-lane
    Box-Muller equals two scalar evaluations over every m and every sincos argument."""
    from paper_1605_02406_b200 import dog
    bad_ln, bad_sqrt, bad_pair, first = dog.check_transforms()
    assert (bad_ln, bad_sqrt, bad_pair) == (0, 0, 0), (bad_ln, bad_sqrt, bad_pair, first)


def test_wide_tile_bounding_box():
    """A sort tile whose particles span more than 2^20 cells of its bounding box (opposite corners of a
    2048 x 1024 grid): the tile sort takes its two-phase path (full keys in global scratch)."""
    cfg = I.config("cfg1", width=2048, height=1024, nu=8192, nu_b=512)
    rng = np.random.default_rng(21)
    i = np.arange(cfg.nu)
    corner = (i % 3 == 0)
    x = np.where(corner, rng.uniform(0, 3, cfg.nu), rng.uniform(2044, 2048, cfg.nu)).astype(np.float32)
    y = np.where(corner, rng.uniform(0, 3, cfg.nu), rng.uniform(1020, 1024, cfg.nu)).astype(np.float32)
    st = dict(x=x, y=y, vx=rng.normal(0, 1, cfg.nu).astype(np.float32), vy=rng.normal(0, 1, cfg.nu).astype(np.float32),
              w_bar=np.float32(1e-4), m_free=np.zeros(cfg.C, np.float32), k=2)
    frames = [np.zeros((cfg.C, 2), np.float32) for _ in range(3)]
    for f in frames:
        f.reshape(cfg.height, cfg.width, 2)[:3, :3, 0] = 0.9
        f.reshape(cfg.height, cfg.width, 2)[1020:, 2044:, 0] = 0.9
    run_lockstep(cfg, 3, st=st, frames=frames)


def test_maximum_width_grid():
    """The widest grid the ABI accepts (65535 columns; the packed (row, col) key uses 16 bits each) with
    particles spread along it: keys, sort (wide bounding boxes) and the whole cycle bit-exact."""
    cfg = I.config("cfg1", width=65535, height=3, nu=20_000, nu_b=1_000)
    rng = np.random.default_rng(5)
    x = rng.uniform(0, cfg.width, cfg.nu).astype(np.float32)
    y = rng.uniform(0, cfg.height, cfg.nu).astype(np.float32)
    x[:50] = np.float32(65534.999)                          # the last column
    st = dict(x=x, y=y, vx=rng.normal(0, 3, cfg.nu).astype(np.float32), vy=rng.normal(0, 1, cfg.nu).astype(np.float32),
              w_bar=np.float32(2e-5), m_free=np.zeros(cfg.C, np.float32), k=1)
    frames = []
    for k in range(2):
        f = np.zeros((cfg.C, 2), np.float32)
        hit = rng.random(cfg.C) < 0.05
        f[hit, 0] = 0.95
        f[~hit, 1] = 0.3
        frames.append(f)
    run_lockstep(cfg, 2, st=st, frames=frames)


def test_grid_of_2_24_cells():
    """4096 x 4096 cells (C = 2^24, the first size past the 40-bit mass fixed point: FX = 38, A-23): a random
    injected state over the whole grid, every cell with a return or a free observation (every cell active),
    two cycles -- keys, masses (R_p, R_b at 2^38), slots, W, the next state bit-exact vs the oracle."""
    import oracle
    assert oracle.fx_bits(4096 * 4096) == 38
    cfg = I.config("cfg1", width=4096, height=4096, nu=2_000_000, nu_b=200_000)
    rng = np.random.default_rng(7)
    st = dict(x=rng.uniform(0, cfg.width, cfg.nu).astype(np.float32),
              y=rng.uniform(0, cfg.height, cfg.nu).astype(np.float32),
              vx=rng.normal(0, 3, cfg.nu).astype(np.float32), vy=rng.normal(0, 3, cfg.nu).astype(np.float32),
              w_bar=np.float32(0.9 * cfg.C / cfg.nu), m_free=np.zeros(cfg.C, np.float32), k=1)
    frames = []
    for k in range(2):
        f = np.zeros((cfg.C, 2), np.float32)
        hit = rng.random(cfg.C) < 0.5
        f[hit, 0] = 0.9
        f[~hit, 1] = 0.4
        frames.append(f)
    run_lockstep(cfg, 2, st=st, frames=frames)


def test_run_to_run_determinism():
    """Two filters with the same seed and inputs agree bit for bit -- state AND velocity moments (every
    floating-point sum on the path has a fixed order: run sums in thread order, warp trees of fixed
    shape, cells combined in tile order) -- including the Doppler and exact branches."""
    from paper_1605_02406_b200 import dog
    cfg = I.config("cfg2", width=256, height=256, nu=300_000, nu_b=30_000, beams=400, movers=6, peds=4, boxes=15)
    sc = I.scene(cfg)
    a, b = dog.Filter.from_config(cfg), dog.Filter.from_config(cfg)
    for k in range(6):
        m = sc.frame(k, device="cuda").contiguous()
        if k < 3:
            a.step(m, cfg.dt); b.step(m, cfg.dt)
        elif k < 5:
            dop, pA = sc.doppler(k, m, frac=0.6)
            dop, pA = dop.cuda().contiguous(), pA.cuda().contiguous()
            a.step_doppler(m, dop, pA, cfg.dt); b.step_doppler(m, dop, pA, cfg.dt)
        else:
            obs = I.Scene.exact_obs(m)
            a.step_exact(obs, cfg.dt); b.step_exact(obs, cfg.dt)
        ra, rb = a.read_cells(), b.read_cells()
        for key in ("occ", "free", "mean", "cov"):
            assert torch.equal(ra[key].view(torch.int32), rb[key].view(torch.int32)), (k, key)
    sa, sb = a.get_state(), b.get_state()
    for key in ("x", "y", "vx", "vy", "m_free"):
        assert np.array_equal(sa[key].view(np.uint32), sb[key].view(np.uint32)), key
