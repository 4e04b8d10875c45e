"""Pins of the oracle's Doppler / association branch (NEXT-1; Eqs. 69-80; SPEC S:161-165,
S:252-266) against the SPEC's worked examples, closed forms and invariants of the cycle:
the exp spec against libm, g against the normal density, Q_j's end points and monotonicity, the
SPEC's two-particle weight example, the nu_A rounding rule, and whole-cycle properties (p_A = 0 is the
plain cycle bit for bit; the joint weight of a cell is R_p exactly; incompatible members get no
copies; associated births move along the measured radial speed; an only-compatible member's velocity
is the cell's mean)."""
import math

import numpy as np
import pytest

import oracle

SENT = -1073741824.0


# ---------------------------------------------------------------- primitives
def test_exp_spec_vs_libm():
    rng = np.random.default_rng(0)
    qs = (-rng.uniform(0, 87, 20000)).astype(np.float32)
    for q in qs:
        e = oracle.exp_spec(float(q))
        assert abs(e / math.exp(float(q)) - 1.0) < 2.5 * 2.0 ** -24, q
    assert oracle.exp_spec(0.0) == 1.0
    assert oracle.exp_spec(-88.0) == 0.0 and oracle.exp_spec(-1e30) == 0.0


def test_doppler_g_spec_examples():
    # v=(5,0), dir=(1,0), radial_speed=5, sd=1 -> 1/sqrt(2 pi)
    assert abs(oracle.doppler_g(5, 0, 1, 0, 5, 1) / (1 / math.sqrt(2 * math.pi)) - 1) < 1e-6
    # v orthogonal to dir, radial_speed 0 -> the same maximum density
    assert oracle.doppler_g(0, 3, 1, 0, 0, 1) == oracle.doppler_g(5, 0, 1, 0, 5, 1)
    # v=(5,0), dir=(1,0), radial_speed=0, sd=1 -> N(5; 0, 1)
    assert abs(oracle.doppler_g(5, 0, 1, 0, 0, 1) / (math.exp(-12.5) / math.sqrt(2 * math.pi)) - 1) < 1e-5
    # closed form on an oblique direction and another SD: e = v.u - v_r
    u = (0.6, 0.8)
    v = (1.5, -2.0)
    e = v[0] * u[0] + v[1] * u[1] - 0.3
    ref = math.exp(-0.5 * (e / 0.7) ** 2) / (0.7 * math.sqrt(2 * math.pi))
    assert abs(oracle.doppler_g(v[0], v[1], u[0], u[1], 0.3, 0.7) / ref - 1) < 1e-5


def test_gfx_fixed_point():
    # A-34: gfx = floor((g / g_max) 2^31) in f32 -- the cell's most likely member holds exactly 2^31
    assert oracle.doppler_gfx(0.5, 0.5) == 1 << 31
    assert oracle.doppler_gfx(0.25, 0.5) == 1 << 30
    assert oracle.doppler_gfx(0.0, 0.5) == 0
    assert oracle.doppler_gfx(0.0, 0.0) == 0                    # every member underflowed: the guard
    g, m = 0.123456, 0.987654
    r = np.float32(np.float32(g) / np.float32(m))
    assert oracle.doppler_gfx(g, m) == math.floor(float(r) * 2 ** 31)
    # tiny likelihoods keep their relative precision (the old absolute 2^-24 quantum floored them to 0)
    assert oracle.doppler_gfx(1e-30, 4e-30) == 1 << 29


def test_weights_concentrate_on_the_nearest_member():
    """Eqs. 71-72 with p_A = 1: each member's share of rho_p is g_j / sum g, however
    small every g is.  Five members of one cell whose velocities sit 6..10 SD from the measured radial
    speed: the nearest one (6 SD) must carry all but ~exp(-6.5) of the mass, and the cell's mean velocity
    is the g-weighted mean computed here from the normal density in fp64 (an independent formulation)."""
    w, h = 8, 8
    sd = 0.25
    t = np.array([6.0, 7.0, 8.0, 9.0, 10.0])
    nu = 5
    vx = (t * sd).astype(np.float32)                             # e = v . u - v_r with u = (1, 0), v_r = 0
    x = np.full(nu, 3.5, np.float32); y = np.full(nu, 4.5, np.float32)
    vy = np.zeros(nu, np.float32)
    p = oracle.Params(width=w, height=h, nu=nu, nu_b=0, cell_size=0.1, seed=3, p_b=0.0,
                      sigma_pos=0.0, sigma_vel=0.0, p_s=1.0)
    o = oracle.Oracle(p)
    o.set_state(x, y, vx, vy, np.float32(0.1), np.zeros(w * h, np.float32), 0)
    C = w * h
    meas = np.zeros((C, 2), np.float32)
    cell = 4 * w + 3
    meas[cell, 0] = 0.9
    dop = np.zeros((C, 4), np.float32); dop[:, 0] = 1.0; dop[:, 3] = sd
    pA = np.zeros(C, np.float32); pA[cell] = 1.0
    o.step_doppler(meas, dop, pA, 1e-9)                          # dt -> 0: positions stay in the cell
    # each member's predicted velocity (sigma_vel = 0: unchanged) and its normal density in fp64
    pv = o.dump("PRED_VX").astype(np.float64)
    g = np.exp(-0.5 * ((pv - 0.0) / sd) ** 2) / (sd * math.sqrt(2 * math.pi))
    assert (g > 0).all() and g.max() < 1e-7                      # every g below the old 2^-24 quantum
    share = g / g.sum()
    gfx, GS = o.dump("GFX"), o.dump("GS")
    assert int(GS[cell]) > 0                                     # not the sum(w~) = 0 guard
    q = gfx.astype(np.float64) / float(GS[cell])
    assert np.allclose(q, share, rtol=1e-6, atol=1e-9)
    assert q[0] > 0.998
    mean = o.read_cells()["mean"][cell]
    ref = float((share * pv).sum())
    assert abs(mean[0] - ref) < 1e-5 * abs(ref) and mean[0] < 1.6  # ~ the nearest member's 1.5 m/s


def test_Q_end_points_monotone_and_closed_forms():
    rng = np.random.default_rng(1)
    for _ in range(200):
        n = int(rng.integers(1, 40))
        gfx = rng.integers(0, 1 << 26, n).astype(np.uint64)
        gfx[rng.random(n) < 0.3] = 0
        if gfx.sum() == 0:
            gfx[0] = 1
        GS = int(gfx.sum())
        Rp = int(rng.integers(1, 1 << 40))
        pA = float(np.float32(rng.random()))
        pre = np.concatenate([[0], np.cumsum(gfx)]).astype(np.uint64)
        Q = [oracle.doppler_Q(Rp, pA, int(pre[j]), GS, j, n) for j in range(n + 1)]
        assert Q[0] == 0 and Q[n] == Rp                          # the cell's mass, exactly
        assert all(Q[j] <= Q[j + 1] for j in range(n))           # nonnegative member weights
        # p_A = 1: Q_j = floor(R_p GS_j / GS); p_A = 0: floor(R_p j / n)  (within one fp64 rounding)
        for j in range(n + 1):
            q1 = oracle.doppler_Q(Rp, 1.0, int(pre[j]), GS, j, n)
            q0 = oracle.doppler_Q(Rp, 0.0, int(pre[j]), GS, j, n)
            assert abs(q1 - Rp * int(pre[j]) // GS) <= 1
            assert abs(q0 - Rp * j // n) <= 1


def test_spec_two_particle_weights():
    # w_pred {0.2, 0.2}, likelihoods {2, 0}, p_A = 1, rho_p = 0.3 -> w = {0.3, 0}
    Rp = math.floor(float(np.float32(0.3)) * 2 ** 40)
    gfx = [oracle.doppler_gfx(2.0, 2.0), oracle.doppler_gfx(0.0, 2.0)]
    GS = sum(gfx)
    Q = [oracle.doppler_Q(Rp, 1.0, g, GS, j, 2) for j, g in enumerate([0, gfx[0], GS])]
    assert (Q[1] - Q[0], Q[2] - Q[1]) == (Rp, 0)


def test_birth_assoc_rounding():
    assert oracle.birth_assoc(1000, 10, np.float32(0.3)) == (3, int(1000 * float(np.float32(0.3))))
    assert oracle.birth_assoc(1000, 10, 0.0) == (0, 0)
    assert oracle.birth_assoc(1000, 2, 0.25) == (1, 250)          # 0.5 rounds half up
    assert oracle.birth_assoc(1000, 10, 1.0) == (10, 1000)
    assert oracle.birth_assoc(777, 3, 0.9) == (3, 777)            # nu_A = nb: all mass associated
    assert oracle.birth_assoc(777, 3, 0.1) == (0, 0)              # nu_A = 0: all mass unassociated


# ---------------------------------------------------------------- whole cycle
def scene(w=24, h=16, nu=3000, nu_b=300, seed=5):
    p = oracle.Params(width=w, height=h, nu=nu, nu_b=nu_b, cell_size=0.1, seed=seed, v_max=20.0)
    rng = np.random.default_rng(seed)
    x = rng.uniform(2, w - 2, nu).astype(np.float32); y = rng.uniform(2, h - 2, nu).astype(np.float32)
    x[:10] = SENT; y[:10] = SENT
    vx = rng.normal(0, 3, nu).astype(np.float32); vy = rng.normal(0, 3, nu).astype(np.float32)
    mf = rng.uniform(0, 0.5, w * h).astype(np.float32)
    meas = np.zeros((w * h, 2), np.float32)
    occ = rng.random(w * h) < 0.4
    meas[occ, 0] = 0.9
    meas[~occ, 1] = 0.6
    state = (x, y, vx, vy, np.float32(1.0 / nu), mf, 3)
    return p, state, meas


def doppler_grid(C, seed, frac=0.5, pA=None):
    rng = np.random.default_rng(seed)
    ang = rng.uniform(0, 2 * np.pi, C)
    dop = np.stack([np.cos(ang), np.sin(ang), rng.normal(0, 3, C), rng.uniform(0.3, 1.5, C)], 1).astype(np.float32)
    a = np.where(rng.random(C) < frac, rng.uniform(0.05, 1.0, C), 0.0).astype(np.float32) if pA is None else pA
    return dop, a


def fresh(p, state):
    o = oracle.Oracle(p)
    o.set_state(*state)
    return o


def test_pA_zero_is_the_plain_cycle():
    p, state, meas = scene()
    a, b = fresh(p, state), fresh(p, state)
    dop, _ = doppler_grid(p.width * p.height, 1)
    a.step(meas, 0.1)
    b.step_doppler(meas, dop, np.zeros(p.width * p.height, np.float32), 0.1)
    sa, sb = a.get_state(), b.get_state()
    for k in ("x", "y", "vx", "vy", "m_free"):
        assert np.array_equal(sa[k].view(np.uint32), sb[k].view(np.uint32)), k
    ra, rb = a.read_cells(), b.read_cells()
    assert np.array_equal(ra["mean"], rb["mean"]) and np.array_equal(ra["cov"], rb["cov"])


def joint_weights(o, p, pA):
    """Per-member fixed-point weights rebuilt from the dumps (PERM, OFFSETS, RP, GFX, GS)."""
    off, perm, Rp = o.dump("OFFSETS"), o.dump("PERM"), o.dump("RP")
    gfx, GS = o.dump("GFX"), o.dump("GS")
    out = {}
    for c in range(p.width * p.height):
        a, b = int(off[c]), int(off[c + 1])
        if b == a or GS[c] == 0:
            continue
        n = b - a
        pre = np.concatenate([[0], np.cumsum(gfx[perm[a:b]].astype(np.uint64))])
        Q = [oracle.doppler_Q(int(Rp[c]), float(pA[c]), int(pre[j]), int(GS[c]), j, n) for j in range(n + 1)]
        out[c] = (perm[a:b], np.diff(np.array(Q, np.uint64)).astype(np.int64))
    return out


def test_cell_mass_and_total_weight_unchanged():
    p, state, meas = scene()
    C = p.width * p.height
    dop, pA = doppler_grid(C, 2)
    a, b = fresh(p, state), fresh(p, state)
    a.step(meas, 0.1)
    b.step_doppler(meas, dop, pA, 0.1)
    assert a.scalars()["W"] == b.scalars()["W"]                  # sum over cells of R_p + gated R_b
    Rp = b.dump("RP")
    jw = joint_weights(b, p, pA)
    assert len(jw) > 20
    for c, (_, q) in jw.items():
        assert q.sum() == int(Rp[c]) and (q >= 0).all()
    nA, RbA, Rb, nb = b.dump("NA"), b.dump("RBA"), b.dump("RB"), b.dump("NB")
    assert (nA <= nb).all() and (RbA <= Rb).all()
    assert ((pA == 0) <= (nA == 0)).all()


def test_incompatible_members_get_no_copies():
    """p_A = 1 everywhere with a measured radial speed far from every particle's but one per cell: the
    resampled persistent particles all come from members with nonzero likelihood."""
    p, state, meas = scene(seed=7)
    C = p.width * p.height
    dop, _ = doppler_grid(C, 3)
    dop[:, 3] = 0.05                                             # sharp likelihood: most members get gfx 0
    o = fresh(p, state)
    o.step_doppler(meas, dop, np.ones(C, np.float32), 0.1)
    gfx, jidx = o.dump("GFX"), o.dump("JOINT_IDX")
    off, perm, GS = o.dump("OFFSETS"), o.dump("PERM"), o.dump("GS")
    n_in = int(off[C])
    # joint order: cell by cell, members then births -> map joint index -> input particle or birth
    joint_src = []
    nb = o.dump("NB")
    for c in range(C):
        joint_src += [int(i) for i in perm[off[c]:off[c + 1]]]
        joint_src += [-1] * int(nb[c])
    picked = [joint_src[j] for j in jidx if j != 0xFFFFFFFF]
    pers = [i for i in picked if i >= 0]
    assert len(pers) > 100
    cell_of = np.full(p.nu, C, np.int64)
    for c in range(C):
        cell_of[perm[off[c]:off[c + 1]]] = c
    for i in pers:
        if GS[cell_of[i]] > 0:
            assert gfx[i] > 0
    assert n_in > 0


def test_associated_births_follow_the_radial_speed():
    p, state, meas = scene(seed=9)
    C = p.width * p.height
    dop, _ = doppler_grid(C, 4)
    dop[:, 3] = 1e-4                                             # sd -> 0: radial component = v_r
    o = fresh(p, state)
    o.step_doppler(meas, dop, np.full(C, 0.7, np.float32), 0.1)
    nA, nb, bcell = o.dump("NA"), o.dump("NB"), o.dump("BIRTH_CELL")
    bvx, bvy = o.dump("BIRTH_VX"), o.dump("BIRTH_VY")
    j, seen = 0, 0
    for c in range(C):
        for r in range(int(nb[c])):
            assert bcell[j] == c
            if r < nA[c] and abs(dop[c, 2]) < 15:
                proj = bvx[j] * dop[c, 0] + bvy[j] * dop[c, 1]
                if abs(bvx[j]) < p.v_max and abs(bvy[j]) < p.v_max:   # not clamped
                    assert abs(proj - dop[c, 2]) < 1e-3
                    seen += 1
            j += 1
    assert seen > 20


def test_single_compatible_member_sets_the_mean():
    """A Doppler cell with p_A = 1 whose likelihood is nonzero for exactly one member reports that
    member's velocity as the mean and zero variance (Eqs. 81-84 with all weight on one member)."""
    p, state, meas = scene(seed=11)
    C = p.width * p.height
    dop, _ = doppler_grid(C, 5)
    dop[:, 3] = 0.02
    o = fresh(p, state)
    o.step_doppler(meas, dop, np.ones(C, np.float32), 0.1)
    gfx, GS, perm, off = o.dump("GFX"), o.dump("GS"), o.dump("PERM"), o.dump("OFFSETS")
    pvx, pvy = o.dump("PRED_VX"), o.dump("PRED_VY")
    cells = o.read_cells()
    hits = 0
    for c in range(C):
        mem = perm[off[c]:off[c + 1]]
        nz = [i for i in mem if gfx[i] > 0]
        if GS[c] > 0 and len(nz) == 1 and cells["occ"][c] > 0:
            i = nz[0]
            assert abs(cells["mean"][c, 0] - pvx[i]) < 1e-4 * max(1, abs(pvx[i]))
            assert abs(cells["mean"][c, 1] - pvy[i]) < 1e-4 * max(1, abs(pvy[i]))
            assert abs(cells["cov"][c, 0]) < 1e-4 * max(1, pvx[i] ** 2)
            hits += 1
    assert hits > 3
