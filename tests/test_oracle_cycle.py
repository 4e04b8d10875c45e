"""Pins of the CPU oracle's full cycle (O1-O7) against closed forms, printed examples, invariants
and brute force.  The expected values never come from the oracle's own formulas; where a step is
re-derived it is through a different formulation (e.g. Dempster's rule by set intersection, the
BBF of Eq. 1, exact rational arithmetic, direct enumeration)."""
import json
import math
import os
import struct
from fractions import Fraction

import numpy as np
import pytest

from paper_1605_02406_b200 import inputs as I
from pinlib import dempster_by_sets, f32, gold, ulp32

TWO40 = 2 ** 40


def mk(orc, **kw):
    base = dict(width=32, height=32, nu=10_000, nu_b=1_000, cell_size=0.1, p_s=0.99, p_b=0.02,
                sigma_pos=0.02, sigma_vel=0.8, sigma_birth_vel=4.0, free_tau=2.0, occ_max=1.0,
                v_max=0.0, seed=2406)
    base.update(kw)
    return orc.Oracle(orc.Params(**base))


def sentinel_state(nu, C):
    return dict(x=np.full(nu, I.SENTINEL_POS, np.float32), y=np.full(nu, I.SENTINEL_POS, np.float32),
                vx=np.zeros(nu, np.float32), vy=np.zeros(nu, np.float32), m_free=np.zeros(C, np.float32))


# ------------------------------------------------------------------------------- O1 predict
def test_predict_noiseless_spec_examples(orc):
    """S:224-226 (Eq. 14, Eq. 39, A-4/A-5): zero noise, T = 0.5 s, 1 m cells:
    p = (10,20), v = (2,-1) -> (11, 19.5); weight 0.4 * p_S 0.99 -> 0.396; a particle leaving the
    grid gets the sentinel key C."""
    ex = gold("spec_examples.json")["predict"]
    o = mk(orc, width=32, height=32, nu=4, nu_b=0, cell_size=1.0, sigma_pos=0.0, sigma_vel=0.0)
    st = sentinel_state(4, 1024)
    st["x"][:2] = [10.0, 31.5]; st["y"][:2] = [20.0, 5.0]
    st["vx"][:2] = [2.0, 2.0]; st["vy"][:2] = [-1.0, 0.0]
    o.set_state(st["x"], st["y"], st["vx"], st["vy"], 0.4, st["m_free"], 0)
    o.step(np.zeros((32, 32, 2), np.float32), ex[0]["T"])
    px, py = o.dump("PRED_X"), o.dump("PRED_Y")
    assert (px[0], py[0]) == tuple(ex[0]["out"])
    assert o.dump("PRED_VX")[0] == 2.0 and o.dump("PRED_VY")[0] == -1.0
    key = o.dump("KEY")
    assert key[0] == 19 * 32 + 11 and key[1] == 1024 and key[2] == 1024
    w_pred = o.scalars()["w_pred"]
    assert abs(float(w_pred) - ex[1]["w_pred"]) <= ulp32(0.396)


def test_predict_noise_is_gaussian_with_table_sd(orc):
    """A-1 (Table I, SD = sigma * T): the residuals (x' - x - v Tc) / s_p and
    (v' - v) / s_v are standard normal (KS), independent across components."""
    from scipy import stats
    o = mk(orc, width=64, height=64, nu=20000, nu_b=0, sigma_pos=0.02, sigma_vel=0.8)
    rng = np.random.default_rng(1)
    st = sentinel_state(20000, 64 * 64)
    st["x"][:] = rng.uniform(10, 50, 20000).astype(np.float32)
    st["y"][:] = rng.uniform(10, 50, 20000).astype(np.float32)
    st["vx"][:] = rng.normal(0, 3, 20000).astype(np.float32)
    st["vy"][:] = rng.normal(0, 3, 20000).astype(np.float32)
    o.set_state(st["x"], st["y"], st["vx"], st["vy"], 1e-4, st["m_free"], 5)
    o.step(np.zeros((64, 64, 2), np.float32), 0.1)
    Tc, s_p, s_v, _ = orc.step_scalars(o.p, 0.1)
    rx = (o.dump("PRED_X").astype(np.float64) - st["x"] - st["vx"] * np.float64(Tc)) / s_p
    rvx = (o.dump("PRED_VX").astype(np.float64) - st["vx"]) / s_v
    rvy = (o.dump("PRED_VY").astype(np.float64) - st["vy"]) / s_v
    for r in (rx, rvx, rvy):
        assert stats.kstest(r, "norm").pvalue > 0.001
    assert abs(np.corrcoef(rvx, rvy)[0, 1]) < 0.03


# ------------------------------------------------------------------------------- O2 assign
def test_assign_spec_example(orc):
    """keys [2,0,2,1] -> stable order [1,3,0,2], cell 2 spans slots [2,4)."""
    ex = gold("spec_examples.json")["sort"][0]
    o = mk(orc, width=3, height=1, nu=4, nu_b=0, cell_size=1.0, sigma_pos=0.0, sigma_vel=0.0)
    st = sentinel_state(4, 3)
    st["x"][:] = [2.5, 0.5, 2.5, 1.5]; st["y"][:] = 0.5
    o.set_state(st["x"], st["y"], st["vx"], st["vy"], 0.1, st["m_free"], 0)
    o.step(np.zeros((1, 3, 2), np.float32), 0.1)
    assert o.dump("KEY").tolist() == ex["keys"]
    assert o.dump("PERM").tolist() == ex["perm"]
    assert o.dump("OFFSETS").tolist() == ex["offsets"]


def run_cfg1(orc, steps=4, **kw):
    cfg = I.CONFIGS["cfg1"]
    o = mk(orc, seed=cfg.seed, **kw)
    sc = I.scene(cfg)
    for k in range(steps):
        o.step(sc.frame(k).numpy(), cfg.dt)
    return o, sc


def test_assign_brute_force_membership(orc):
    """P-SORT: after a realistic cycle, each cell's slot range holds exactly the particles whose key
    is that cell, in ascending input order (stable, A-6); sentinels sort last."""
    o, _ = run_cfg1(orc, steps=3)
    key, perm, off = o.dump("KEY"), o.dump("PERM"), o.dump("OFFSETS")
    C = 1024
    assert sorted(perm.tolist()) == list(range(len(key)))
    for c in range(C):
        members = np.nonzero(key == c)[0]
        assert perm[off[c]:off[c + 1]].tolist() == members.tolist()
    assert np.all(key[perm[off[C]:]] == C)


# ------------------------------------------------------------------------------- O3 cells
def test_cells_against_definitions(orc):
    """Eqs. 61-63, 67-68 per cell, against independent formulations: S_c = n_c w_pred (exact sum of
    equal weights), m_p = min(S_c, 1), m_Fp = min(alpha m_F, 1 - m_p), Dempster by set
    intersection (exact rationals), the birth split in exact arithmetic, rho_p + rho_b = m_O, and
    the fixed point R = floor(rho 2^40) with births only where m_zO > 0."""
    cfg = I.CONFIGS["cfg1"]
    o = mk(orc, seed=cfg.seed)
    sc = I.scene(cfg)
    for k in range(3):
        o.step(sc.frame(k).numpy(), cfg.dt)
    mF_prev = o.get_state()["m_free"].copy()
    meas = sc.frame(3).numpy().reshape(-1, 2)
    o.step(meas, cfg.dt)
    alpha = orc.step_scalars(o.p, cfg.dt)[3]
    w_pred = float(o.scalars()["w_pred"])
    off = o.dump("OFFSETS").astype(np.int64)
    n = np.diff(off)
    S, mp, mfp = o.dump("S"), o.dump("MP"), o.dump("MFP")
    occ, fre, rp, rb = o.dump("OCC"), o.dump("FREE"), o.dump("RHO_P"), o.dump("RHO_B")
    Rp, Rb = o.dump("RP"), o.dump("RB")
    for c in range(1024):
        assert S[c] == f32(float(n[c] * Fraction(w_pred)))
        assert mp[c] == min(S[c], 1.0)
        assert mfp[c] == min(f32(alpha * mF_prev[c]), f32(1.0 - mp[c]))
        eo, ef = dempster_by_sets((float(mp[c]), float(mfp[c])), (float(meas[c, 0]), float(meas[c, 1])))
        k = float(mp[c]) * float(meas[c, 1]) + float(mfp[c]) * float(meas[c, 0])
        tol = 16 * 2.0 ** -24 / max(1 - k, 1e-6)
        assert abs(occ[c] - eo) <= tol and abs(fre[c] - ef) <= tol
        assert abs((rp[c] + rb[c]) - occ[c]) <= 2 * ulp32(occ[c])
        q = Fraction(0.02) * (1 - Fraction(float(mp[c])))
        den = Fraction(float(mp[c])) + q
        exact_rb = Fraction(float(occ[c])) * q / den if den > 0 else 0
        assert abs(rb[c] - float(exact_rb)) <= 4 * ulp32(float(exact_rb)) + 1e-30
        assert Rp[c] == (math.floor(Fraction(float(max(rp[c], 0))) * TWO40) if n[c] > 0 else 0)
        assert Rb[c] == (math.floor(Fraction(float(max(rb[c], 0))) * TWO40) if meas[c, 0] > 0 else 0)
    st = o.get_state()
    assert np.array_equal(st["m_free"], fre)


# ------------------------------------------------------------------------------- O6 moments
def test_moments_spec_examples(orc):
    """S:275-277 (Eqs. 81-84): v_x {1,3} in one cell -> mean 2, var 1; one particle -> var 0;
    v_y = v_x -> cov = var.  Zero noise, p_B = 0, cells kept occupied by the measurement."""
    o = mk(orc, width=4, height=1, nu=3, nu_b=0, cell_size=1.0, sigma_pos=0.0, sigma_vel=0.0, p_b=0.0)
    st = sentinel_state(3, 4)
    st["x"][:] = [0.5, 0.5, 2.5]; st["y"][:] = 0.5
    st["vx"][:] = [1.0, 3.0, 2.5]; st["vy"][:] = [1.0, 3.0, -1.0]
    o.set_state(st["x"], st["y"], st["vx"], st["vy"], 0.2, st["m_free"], 0)
    meas = np.zeros((1, 4, 2), np.float32); meas[0, :, 0] = 0.9
    o.step(meas, 1e-6)
    cells = o.read_cells()
    ex = gold("spec_examples.json")["moments"]
    assert abs(cells["mean"][0, 0] - ex[0]["mean"]) < 1e-6
    assert abs(cells["cov"][0, 0] - ex[0]["var"]) < 1e-5
    assert abs(cells["cov"][0, 2] - cells["cov"][0, 0]) < 1e-6    # v_y = v_x -> cov = var
    assert abs(cells["mean"][2, 0] - ex[1]["mean"]) < 1e-6
    assert abs(cells["cov"][2, 0]) < 1e-5 and abs(cells["cov"][2, 1]) < 1e-5
    assert np.all(cells["mean"][[1, 3]] == 0) and np.all(cells["cov"][[1, 3]] == 0)


def test_moments_brute_force(orc):
    """Moments of a realistic cycle equal direct sample statistics of each cell's predicted particles
    (w' is uniform within a cell), and satisfy cov^2 <= var_x var_y."""
    o, _ = run_cfg1(orc, steps=4)
    off, perm = o.dump("OFFSETS"), o.dump("PERM")
    pvx, pvy = o.dump("PRED_VX").astype(np.float64), o.dump("PRED_VY").astype(np.float64)
    rp = o.dump("RHO_P")
    cells = o.read_cells()
    checked = 0
    for c in range(1024):
        a, b = off[c], off[c + 1]
        if b == a or rp[c] <= 0:
            assert np.all(cells["mean"][c] == 0) and np.all(cells["cov"][c] == 0)
            continue
        idx = perm[a:b]
        vx, vy = pvx[idx], pvy[idx]
        mx, my = vx.mean(), vy.mean()
        assert abs(cells["mean"][c, 0] - mx) <= 1e-5 * max(1, abs(mx))
        assert abs(cells["mean"][c, 1] - my) <= 1e-5 * max(1, abs(my))
        scale = max(1.0, mx * mx + vx.var())
        assert abs(cells["cov"][c, 0] - vx.var()) <= 1e-5 * scale
        assert abs(cells["cov"][c, 1] - vy.var()) <= 1e-5 * max(1.0, my * my + vy.var())
        assert abs(cells["cov"][c, 2] - ((vx - mx) * (vy - my)).mean()) <= 1e-5 * max(1.0, scale)
        checked += 1
    assert checked > 10


# ------------------------------------------------------------------------------- O5 births
def test_births_properties(orc):
    """P-SLOT / P-BIRTH on a realistic cycle: exactly nu_b slots, proportional to the gated born
    mass (floor/ceil of the share), positions strictly inside the slot's cell, velocities
    N(0, sigma_B^2) (KS), slots of a cell contiguous and in cell order."""
    from scipy import stats
    o, _ = run_cfg1(orc, steps=2, nu_b=20000)
    Rb, nb, bcell = o.dump("RB"), o.dump("NB"), o.dump("BIRTH_CELL")
    A = int(sum(int(v) for v in Rb))
    assert A > 0 and int(nb.sum()) == 20000
    for c in np.nonzero(Rb)[0]:
        share = Fraction(20000 * int(Rb[c]), A)
        assert math.floor(share) <= nb[c] <= math.ceil(share)
    assert np.all(np.diff(bcell.astype(np.int64)) >= 0)
    assert np.array_equal(np.bincount(bcell, minlength=1024), nb.astype(np.int64))
    bx, by = o.dump("BIRTH_X"), o.dump("BIRTH_Y")
    col, row = bcell % 32, bcell // 32
    assert np.all(bx >= col) and np.all(bx < col + 1) and np.all(by >= row) and np.all(by < row + 1)
    v = np.concatenate([o.dump("BIRTH_VX"), o.dump("BIRTH_VY")]) / 4.0
    assert stats.kstest(v, "norm").pvalue > 0.001


# ------------------------------------------------------------------------------- O7 resample
def test_resample_step_properties(orc):
    """P-RES on a realistic cycle: selected joint indices are non-decreasing; every joint member gets
    floor/ceil of nu q/W copies; the next state is an exact copy of the selected member; total weight
    is conserved (Eq. 57): nu w_bar = W 2^-40 to one f32 rounding, and W 2^-40 equals the posterior
    mass of represented cells to within C 2^-40 (fixed-point floors)."""
    o, _ = run_cfg1(orc, steps=3)
    off, perm, nb = o.dump("OFFSETS"), o.dump("PERM"), o.dump("NB")
    Rp, Rb, rp, rb = o.dump("RP"), o.dump("RB"), o.dump("RHO_P"), o.dump("RHO_B")
    jidx = o.dump("JOINT_IDX")
    s = o.scalars()
    nu = 10_000
    # rebuild the joint list (cell-interleaved, A-25) and the members' weights
    src, q = [], []
    slot = 0
    for c in range(1024):
        n = int(off[c + 1] - off[c])
        for r in range(n):
            src.append(("p", int(perm[off[c] + r]))); q.append(int(Rp[c]) // n + (r < int(Rp[c]) % n))
        m = int(nb[c])
        for r in range(m):
            src.append(("b", slot)); q.append(int(Rb[c]) // m + (r < int(Rb[c]) % m)); slot += 1
    W = sum(q)
    assert W == s["W"]
    assert np.all(np.diff(jidx.astype(np.int64)) >= 0)
    copies = np.bincount(jidx, minlength=len(q))
    for j in range(len(q)):
        share = Fraction(nu * q[j], W)
        assert math.floor(share) <= copies[j] <= math.ceil(share)
    st = o.get_state()
    px, py = o.dump("PRED_X"), o.dump("PRED_Y")
    bx, by = o.dump("BIRTH_X"), o.dump("BIRTH_Y")
    for i in range(0, nu, 37):
        kind, k = src[jidx[i]]
        if kind == "p":
            assert (st["x"][i], st["y"][i]) == (px[k], py[k])
        else:
            assert (st["x"][i], st["y"][i]) == (bx[k], by[k])
    assert abs(float(st["w_bar"]) * nu - W * 2.0 ** -40) <= nu * ulp32(float(st["w_bar"]))
    mass = sum(Fraction(float(max(rp[c], 0))) for c in range(1024) if off[c + 1] > off[c])
    mass += sum(Fraction(float(max(rb[c], 0))) for c in range(1024) if nb[c] > 0 and Rb[c] > 0)
    assert abs(float(mass) - W * 2.0 ** -40) <= 2 * 1024 * 2.0 ** -40


# ------------------------------------------------------------------------------- whole-cycle closed forms
def bayesian_setup(orc, seed=5, N=100, steps=1):
    """P-BBF setup: 32x32, Bayesian state m_O = n_c w_bar, m_F = 1 - m_O, alpha = 1,
    p_S = 1, sigma = 0, v = 0, p_B = 0, Bayesian measurements (z, 1-z)."""
    rng = np.random.default_rng(seed)
    cfg = I.config("cfg1", nu=1024 * N, nu_b=0, p_s=1.0, p_b=0.0, sigma_pos=0.0, sigma_vel=0.0,
                   free_tau=float("inf"))
    o = mk(orc, width=32, height=32, nu=cfg.nu, nu_b=0, p_s=1.0, p_b=0.0, sigma_pos=0.0, sigma_vel=0.0,
           free_tau=float("inf"))
    counts = rng.integers(5, N, 1024)
    w_bar = np.float32(1.0 / N)
    st = I.cells_state(cfg, counts, w_bar, rng=rng)
    m_O = np.array([f32(float(Fraction(int(n)) * Fraction(float(w_bar)))) for n in counts], np.float32)
    m_F = (np.float32(1.0) - m_O).astype(np.float32)
    o.set_state(st["x"], st["y"], st["vx"], st["vy"], w_bar, m_F, 0)
    return o, rng, m_O


def test_bbf_reduction_one_step(orc):
    """P-BBF (the DS counterpart of the P:795-867 proposition): one cycle equals the binary Bayes
    filter Eq. 1 applied to the realised prior m_p: m_O' = z p / (z p + (1-z)(1-p))."""
    o, rng, m_O = bayesian_setup(orc)
    z = rng.uniform(0.05, 0.95, 1024).astype(np.float32)
    meas = np.stack([z, (1 - z).astype(np.float32)], -1)
    o.step(meas, 0.1)
    p = o.dump("MP").astype(np.float64)
    assert np.array_equal(p.astype(np.float32), m_O)
    zz = z.astype(np.float64)
    bbf = zz * p / (zz * p + (1 - zz) * (1 - p))
    occ = o.read_cells()["occ"]
    assert np.max(np.abs(occ - bbf)) <= 2e-6


def test_bbf_reduction_trajectory(orc):
    """P-BBF over 30 cycles.  Resampling quantises each cell's mass to whole particles, so after the
    first cycle the prior is no longer exactly Bayesian (m_p + m_Fp != 1).  Two closed forms still
    pin every cycle: (a) Dempster's rule with a Bayesian measurement (z, 1-z) is Bayes' rule on the
    prior PLAUSIBILITIES (Shafer 1976): m_O' = z Pl(O) / (z Pl(O) + (1-z) Pl(F)), Pl(O) = 1 - m_Fp,
    Pl(F) = 1 - m_p -- Eq. 1 with the plausibility ratio; (b) systematic resampling moves each cell's
    represented mass R_p 2^-40 by less than one particle weight w_bar = W 2^-40 / nu (Eq. 57)."""
    o, rng, m_O = bayesian_setup(orc, N=100)
    nu = 1024 * 100
    prev = None
    for k in range(30):
        z = rng.uniform(0.1, 0.9, 1024)
        meas = np.stack([z, 1 - z], -1).astype(np.float32)
        o.step(meas, 0.1)
        mp, mfp = o.dump("MP").astype(np.float64), o.dump("MFP").astype(np.float64)
        zz = meas[:, 0].astype(np.float64)
        plo, plf = 1 - mfp, 1 - mp
        ref = zz * plo / (zz * plo + (1 - zz) * plf)
        occ = o.read_cells()["occ"].astype(np.float64)
        assert np.max(np.abs(occ - ref)) <= 4e-6, k
        if prev is not None:
            Rp_prev, wbar = prev
            assert np.all(np.abs(mp - Rp_prev * 2.0 ** -40) <= wbar * (1 + 1e-6) + 1e-7)
        s = o.scalars()
        prev = (o.dump("RP").astype(np.float64), s["W"] * 2.0 ** -40 / nu)


def test_static_fixed_points(orc):
    """P-FIX: repeated free measurement (0, m_zF) on an empty grid converges to
    m_F* = m_zF / (1 - alpha (1 - m_zF)); repeated occupied (m_zO, 0), p_B = 0, injected particles
    converges to m_O* = m_zO / (1 - p_S (1 - m_zO)) (fixed points of Eqs. 61-63)."""
    o = mk(orc, width=8, height=8, nu=64 * 200, nu_b=0, p_b=0.0, sigma_pos=0.0, sigma_vel=0.0)
    cfg = I.config("cfg1", width=8, height=8, nu=64 * 200, nu_b=0)
    st = I.cells_state(cfg, np.r_[np.full(32, 200), np.zeros(32, int)], 1.0 / 400)
    o.set_state(st["x"], st["y"], st["vx"], st["vy"], np.float32(1.0 / 400), st["m_free"], 0)
    meas = np.zeros((64, 2), np.float32)
    meas[:32, 0] = 0.6
    meas[32:, 1] = 0.7
    for k in range(400):
        o.step(meas, 0.1)
    alpha = orc.step_scalars(o.p, 0.1)[3]
    cells = o.read_cells()
    mF_star = 0.7 / (1 - alpha * 0.3)
    mO_star = 0.6 / (1 - 0.99 * 0.4)
    assert np.max(np.abs(cells["free"][32:] - mF_star)) < 1e-5
    W = o.scalars()["W"] * 2.0 ** -40
    assert np.max(np.abs(cells["occ"][:32] - mO_star)) <= 3 * W / (64 * 200) + 1e-5


def test_vacuous_decay(orc):
    """P-DECAY: a vacuous measurement (0,0) with p_B = 0 makes Dempster the identity, so the total
    weight decays exactly by p_S per cycle (Eq. 39) up to fixed-point floors, and m_F by alpha."""
    o = mk(orc, width=16, height=16, nu=256 * 50, nu_b=0, p_b=0.0, sigma_pos=0.0, sigma_vel=0.0)
    cfg = I.config("cfg1", width=16, height=16, nu=256 * 50, nu_b=0)
    rng = np.random.default_rng(2)
    st = I.cells_state(cfg, np.full(256, 50), 1.0 / 64, rng=rng)
    mf0 = rng.uniform(0, 0.2, 256).astype(np.float32)   # below 1 - m_p: the Eq. 62 cap stays inactive
    o.set_state(st["x"], st["y"], st["vx"], st["vy"], np.float32(1.0 / 64), mf0, 0)
    W_prev = 256 * 50 / 64
    mf = mf0.astype(np.float64)
    alpha = orc.step_scalars(o.p, 0.1)[3]
    for k in range(10):
        o.step(np.zeros((256, 2), np.float32), 0.1)
        W = o.scalars()["W"] * 2.0 ** -40
        assert abs(W - 0.99 * W_prev) <= 1e-6 * W_prev + 256 * 2.0 ** -40
        W_prev = W
        mf = mf * alpha
        assert np.max(np.abs(o.read_cells()["free"] - mf)) <= 1e-6


def test_empty_world_and_first_cycle(orc):
    """A-19/A-26: from the empty state, a measurement without occupied evidence keeps the world empty
    (W = 0, all particles at the sentinel); with occupied evidence, cycle 1 is births only and the
    readout equals the measurement (vacuous prior)."""
    o = mk(orc)
    meas = np.zeros((1024, 2), np.float32); meas[:, 1] = 0.5; meas[100, 1] = 0.0
    o.step(meas, 0.1)
    st = o.get_state()
    assert o.scalars()["W"] == 0 and st["w_bar"] == 0 and np.all(st["x"] == I.SENTINEL_POS)
    meas[100, 0] = 0.9; meas[100, 1] = 0.0
    o.step(meas, 0.1)
    cells = o.read_cells()
    assert cells["occ"][100] == np.float32(0.9)
    assert o.dump("NB")[100] == 1000 and o.scalars()["W"] > 0


def test_determinism_and_resume(orc):
    """Counter-based draws (A-20): two runs agree bit for bit, and resuming from get_state/set_state
    reproduces the remaining cycles exactly."""
    a, sc = run_cfg1(orc, steps=3)
    b, _ = run_cfg1(orc, steps=3)
    sa, sb = a.get_state(), b.get_state()
    for k in ("x", "y", "vx", "vy", "m_free"):
        assert np.array_equal(sa[k], sb[k])
    c = mk(orc, seed=I.CONFIGS["cfg1"].seed)
    c.set_state(sa["x"], sa["y"], sa["vx"], sa["vy"], sa["w_bar"], sa["m_free"], sa["k"])
    for k in range(3, 5):
        a.step(sc.frame(k).numpy(), 0.1)
        c.step(sc.frame(k).numpy(), 0.1)
    sa, sc2 = a.get_state(), c.get_state()
    for k in ("x", "y", "vx", "vy", "m_free"):
        assert np.array_equal(sa[k], sc2[k])
