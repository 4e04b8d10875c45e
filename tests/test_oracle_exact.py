"""Pins of the oracle's exact PHD/MIB filter (NEXT-3; section V) in the uniform-likelihood
setting of the section IV-F proposition: the cell update against the generalised binary
Bayes filter it reduces to (SPEC S:340-347 examples: p = 0.5, alpha = 3 -> 0.75; alpha = 1 leaves p;
inverse evidence cancels), and the whole cycle under the proposition's premises (static deterministic
process, p_S = 1, p_B = 0) tracking the BBF recursion cell by cell; plus the SPEC's empty-cell example
and births in unobserved cells."""
import numpy as np
import pytest

import oracle


def bbf(p, alpha):                         # generalised binary Bayes update (Eq. BBF_gen)
    return alpha * p / (alpha * p + (1.0 - p))


def test_cell_update_is_the_bbf_update():
    ex = lambda S, occ, tp, fp: sum(oracle.exact_cell(S, 1.0, 0.0, occ, tp, fp))
    assert abs(ex(0.5, 1.0, 0.9, 0.3) - 0.75) < 1e-7                   # SPEC: p=0.5, alpha=3 -> 0.75
    for p in (0.1, 0.5, 0.93):
        assert abs(ex(p, 1.0, 0.4, 0.4) - p) < 1e-7                    # alpha = 1 (measurement)
        assert abs(ex(p, 0.0, 0.4, 0.4) - p) < 1e-7                    # p_TP = p_FP, no measurement
    p1 = ex(0.5, 1.0, 0.9, 0.3)
    assert abs(ex(p1, 1.0, 0.3, 0.9) - 0.5) < 1e-6                     # alpha = 3 then 1/3
    rng = np.random.default_rng(0)
    for _ in range(2000):
        p = float(np.float32(rng.uniform(0.001, 0.999)))
        tp, fp = (float(np.float32(v)) for v in rng.uniform(0.01, 0.99, 2))
        occ = float(rng.random() < 0.5)
        alpha = tp / fp if occ else (1 - tp) / (1 - fp)
        assert abs(ex(p, occ, tp, fp) - bbf(p, alpha)) < 2e-6, (p, tp, fp, occ)
    # monotone in alpha
    vals = [ex(0.3, 1.0, 0.9, fp) for fp in (0.9, 0.6, 0.3, 0.1, 0.05)]
    assert all(a < b for a, b in zip(vals, vals[1:]))


def test_birth_split_of_the_prediction():
    # r_b+ = p_B (1 - r_p+), both scaled by the same factor (Eqs. 32, 38-41)
    rp, rb = oracle.exact_cell(0.2, 1.0, 0.05, 0.0, 0.5, 0.5)
    assert abs(rp - 0.2) < 1e-7 and abs(rb - 0.05 * 0.8) < 1e-8
    rp, rb = oracle.exact_cell(0.2, 1.0, 0.05, 1.0, 0.9, 0.1)
    rplus = 0.2 + 0.04
    f = 0.9 / (0.1 * (1 - rplus) + 0.9 * rplus)
    assert abs(rp - 0.2 * f) < 1e-6 and abs(rb - 0.04 * f) < 1e-6
    # p_B = 0 and no persistent mass: the cell stays empty
    assert oracle.exact_cell(0.0, 1.0, 0.0, 1.0, 0.9, 0.1) == (0.0, 0.0)


def test_cycle_reduces_to_bbf():
    """Proposition of section IV-F: static deterministic process (no noise, zero velocities, p_S = 1,
    p_B = 0), the occupancy of every cell follows the BBF recursion with alpha from its observations
    (within the quantisation of resampling: ~4000 particles per cell)."""
    W = H = 4
    C = W * H
    per = 4096
    nu = per * C
    p = oracle.Params(width=W, height=H, nu=nu, nu_b=0, cell_size=0.1, p_s=1.0, p_b=0.0, sigma_pos=0.0,
                      sigma_vel=0.0, sigma_birth_vel=0.0, seed=9)
    o = oracle.Oracle(p)
    rng = np.random.default_rng(1)
    p0 = rng.uniform(0.05, 0.95, C)
    w_bar = 1.0 / per                          # cell c holds n_c particles: initial occupancy n_c w_bar = p0_c
    n_c = np.maximum(1, np.round(p0 * per)).astype(np.int64)
    n_c[-1] += nu - n_c.sum()                  # the remaining particles fill the last cell ...
    assert n_c[-1] > 0
    cells = np.repeat(np.arange(C), n_c)
    x = (cells % W + 0.5).astype(np.float32); y = (cells // W + 0.5).astype(np.float32)
    z = np.zeros(nu, np.float32)
    o.set_state(x, y, z, z, np.float32(w_bar), np.zeros(C, np.float32), 0)
    S0 = n_c * np.float32(w_bar)
    ref = np.minimum(S0, 1.0)                  # truncation (occ_max = 1)
    for k in range(15):
        obs = np.zeros((C, 4), np.float32)
        obs[:, 0] = rng.random(C) < 0.5
        obs[:, 1] = rng.uniform(0.3, 0.95, C)
        obs[:, 2] = rng.uniform(0.05, 0.7, C)
        o.step_exact(obs, 0.1)
        occ = o.read_cells()["occ"]
        alpha = np.where(obs[:, 0] > 0, obs[:, 1] / obs[:, 2], (1 - obs[:, 1]) / (1 - obs[:, 2]))
        ref = bbf(ref, alpha)
        # the last cell started saturated (S0 > 1): compare the others
        assert np.all(np.abs(occ[:-1] - ref[:-1]) < 4e-3), (k, np.abs(occ[:-1] - ref[:-1]).max())
        st = o.get_state()
        assert np.all(st["vx"] == 0) and np.all(st["x"] - np.floor(st["x"]) == 0.5)   # nothing moves
        # the resampled cell masses carry the posterior forward: re-derive ref from them (quantisation)
        cnt = np.bincount((np.floor(st["y"]).astype(int) * W + np.floor(st["x"]).astype(int)), minlength=C)
        ref = np.minimum(cnt * np.float64(st["w_bar"]), 1.0)


def test_births_in_unobserved_cells():
    """p_B > 0: born mass and birth slots also in cells without any measurement."""
    W = H = 16
    C = W * H
    p = oracle.Params(width=W, height=H, nu=2000, nu_b=C, cell_size=0.1, p_b=0.02, seed=4)
    o = oracle.Oracle(p)
    obs = np.zeros((C, 4), np.float32)
    obs[:, 1] = 0.05; obs[:, 2] = 0.05                      # unobserved everywhere (alpha = 1)
    o.step_exact(obs, 0.1)
    nb, rb = o.dump("NB"), o.dump("RB")
    assert (rb > 0).all() and nb.sum() == C and (nb > 0).mean() > 0.9
    occ = o.read_cells()["occ"]
    assert np.allclose(occ, 0.02, atol=1e-7)                # r = p_B (1 - 0) from the empty state
