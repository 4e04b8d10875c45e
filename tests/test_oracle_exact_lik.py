"""Pins of the oracle's exact PHD/MIB filter with a single-object likelihood (NEXT-3 general form;
multi-object likelihood Eq. 38, particle update Eqs. 49-52; A-38):

* p_A = 0 everywhere is the uniform-likelihood exact filter (orc_step_exact) bit for bit;
* the births' expected likelihood under the birth prior against numerical integration;
* the cell update against the paper's formulas evaluated independently in fp64 from explicit members
  (the persistent sum of Eq. 51 over the members, the born term by its expectation);
* the members' shares of rho_p against g_A(z|x_j) / sum g_A in fp64, also when every likelihood is
  far below the old absolute quantum;
* an uninformative measurement (g = p_cl for everything) reduces to the uniform form;
* the births: nu_A of the rule, the associated slots' radial speeds from the closed-form posterior
  (statistical), the even split kept by the associated / unassociated mass division (brute force)."""
import math

import numpy as np
import pytest

import oracle

SENT = -1073741824.0


def npdf(x, s):
    return math.exp(-0.5 * (x / s) ** 2) / (s * math.sqrt(2 * math.pi))


def test_birth_mean_likelihood_vs_quadrature():
    for vr, sd, sb in ((0.0, 0.25, 4.0), (3.0, 0.5, 4.0), (-7.5, 1.0, 2.0), (12.0, 0.1, 4.0)):
        # E over the radial component r ~ N(0, sb^2) of N(r - vr; 0, sd^2), by a fine Riemann sum
        r = np.linspace(-12 * sb, 12 * sb, 400001)
        ref = float(np.sum(np.exp(-0.5 * (r / sb) ** 2) / (sb * math.sqrt(2 * math.pi))
                           * np.exp(-0.5 * ((r - vr) / sd) ** 2) / (sd * math.sqrt(2 * math.pi))) * (r[1] - r[0]))
        got = oracle.birth_mean_lik(vr, sd, sb)
        assert abs(got / ref - 1) < 2e-6, (vr, sd, sb, got, ref)


def test_birth_assoc_exact_keeps_the_single_even_split():
    rng = np.random.default_rng(3)
    for _ in range(500):
        nb = int(rng.integers(1, 40))
        Rb = int(rng.integers(0, 1 << 40))
        pi = float(np.float32(rng.random()))
        na, ra = oracle.birth_assoc_exact(Rb, nb, pi)
        assert na == min(nb, math.floor(pi * nb + 0.5))
        single = [Rb // nb + (1 if r < Rb % nb else 0) for r in range(nb)]
        assert ra == sum(single[:na])                        # the first nu_A slots' part of the even split
        if na:                                               # and the two-set even splits reproduce it
            a = [ra // na + (1 if r < ra % na else 0) for r in range(na)]
            rest = Rb - ra
            b = [rest // (nb - na) + (1 if r < rest % (nb - na) else 0) for r in range(nb - na)] if nb > na else []
            assert a + b == single


def cell_reference(S, occ_max, p_b, pTP, pFP, pcl, pA, g_members, vr, sd, sb):
    """Eqs. 38, 49-52 from explicit members, fp64: (rho_p, rho_b, member shares)."""
    n = len(g_members)
    rpp = min(S, occ_max)
    rbp = p_b * (1 - rpp)
    rplus = rpp + rbp
    gA = [pA * g + (1 - pA) * pcl for g in g_members]
    w = rpp / n if n else 0.0
    sum_p = sum(pTP * ga * w for ga in gA)                   # Eq. 50 summed over the persistent members
    Eb = npdf(vr, math.sqrt(sd * sd + sb * sb))
    sum_b = pTP * rbp * (pA * Eb + (1 - pA) * pcl)          # the born particles' sum, by its expectation
    mu = pFP * pcl * (1 - rplus) + sum_p + sum_b             # Eq. 51
    shares = [ga / sum(gA) for ga in gA] if n else []
    return sum_p / mu, sum_b / mu, shares


def gfx_of(gs):
    g32 = [float(np.float32(g)) for g in gs]
    gmax = max(g32)
    return [oracle.doppler_gfx(g, gmax) for g in g32], gmax


def test_cell_update_vs_the_paper_formulas():
    rng = np.random.default_rng(7)
    for _ in range(300):
        n = int(rng.integers(1, 30))
        sd = float(np.float32(rng.uniform(0.1, 2.0)))
        vr = float(np.float32(rng.normal(0, 5)))
        v = rng.normal(vr, 3 * sd, n)                        # members' radial speeds around the measurement
        g = [float(np.float32(oracle.doppler_g(float(np.float32(x)), 0.0, 1.0, 0.0, vr, sd))) for x in v]
        S = float(np.float32(rng.uniform(0.0, 1.2)))
        p_b, pTP, pFP = (float(np.float32(x)) for x in (rng.uniform(0, 0.1), rng.uniform(0.5, 0.99),
                                                       rng.uniform(0.001, 0.3)))
        pcl = float(np.float32(rng.uniform(0.001, 0.5)))
        pA = float(np.float32(rng.uniform(0.05, 1.0)))
        gfx, gmax = gfx_of(g)
        rp, rb, pAe, pi = oracle.exact_lik_cell(S, 1.0, p_b, pTP, pFP, pcl, pA, sum(gfx), gmax, n, vr, sd, 4.0)
        rp_ref, rb_ref, shares = cell_reference(S, 1.0, p_b, pTP, pFP, pcl, pA, g, vr, sd, 4.0)
        assert abs(rp - rp_ref) <= 2e-6 * max(rp_ref, 1e-30) + 1e-12, (rp, rp_ref)
        assert abs(rb - rb_ref) <= 2e-6 * max(rb_ref, 1e-30) + 1e-12, (rb, rb_ref)
        assert rp + rb <= 1.0 + 1e-6
        # member j's share through the Doppler Q_j form with the effective pAe (A-35)
        Rp = 1 << 40
        pre = np.concatenate([[0], np.cumsum(gfx)]).astype(np.uint64)
        Q = [oracle.doppler_Q(Rp, pAe, int(pre[j]), sum(gfx), j, n) for j in range(n + 1)]
        got = np.diff(np.array(Q, np.float64)) / Rp
        assert np.allclose(got, shares, rtol=2e-6, atol=2e-9), (got, shares)
        Eb = npdf(vr, math.sqrt(sd * sd + 16.0))
        assert abs(pi - pA * Eb / (pA * Eb + (1 - pA) * pcl)) < 2e-6


def test_tiny_likelihoods_keep_their_shares():
    """Every member 6..10 SD from the measured radial speed (g far below 2^-24): the shares still follow
    g_A / sum g_A (the relative fixed point of A-34) -- p_A = 1, p_cl = 0."""
    sd = 0.25
    t = [6.0, 7.0, 8.0, 9.0, 10.0]
    g = [float(np.float32(oracle.doppler_g(x * sd, 0.0, 1.0, 0.0, 0.0, sd))) for x in t]
    gfx, gmax = gfx_of(g)
    rp, rb, pAe, pi = oracle.exact_lik_cell(0.5, 1.0, 0.0, 0.9, 0.05, 0.0, 1.0, sum(gfx), gmax, 5, 0.0, sd, 4.0)
    assert pAe == 1.0 and rp > 0.99
    Rp = 1 << 40
    pre = np.concatenate([[0], np.cumsum(gfx)]).astype(np.uint64)
    Q = [oracle.doppler_Q(Rp, pAe, int(pre[j]), sum(gfx), j, 5) for j in range(6)]
    share = np.diff(np.array(Q, np.float64)) / Rp
    ref = np.array([npdf(x * sd, sd) for x in t]); ref /= ref.sum()
    assert np.allclose(share, ref, rtol=1e-6, atol=2.0 ** -30) and share[0] > 0.998   # quantum 2^-31 of the max


def test_uninformative_measurement_is_the_uniform_update():
    """p_A = 0: g_A(z|x) = p_cl for every member and every birth (Eq. 38), so the likelihood cancels from
    Eqs. 50-51 and the update is the uniform form of orc_exact_cell (Eqs. 38-41)."""
    pcl = float(np.float32(0.2))
    for S in (0.0, 0.3, 0.9):
        rp, rb, pAe, pi = oracle.exact_lik_cell(S, 1.0, 0.05, 0.9, 0.1, pcl, 0.0, 3 << 31, pcl, 3, 1.0, 0.5, 4.0)
        up, ub = oracle.exact_cell(S, 1.0, 0.05, 1.0, 0.9, 0.1)
        assert abs(rp - up) < 2e-7 and abs(rb - ub) < 2e-7 and pAe == 0.0 and pi == 0.0


def scene(w=20, h=16, nu=4000, nu_b=400, seed=5):
    p = oracle.Params(width=w, height=h, nu=nu, nu_b=nu_b, cell_size=0.1, seed=seed, v_max=20.0)
    rng = np.random.default_rng(seed)
    x = rng.uniform(2, w - 2, nu).astype(np.float32); y = rng.uniform(2, h - 2, nu).astype(np.float32)
    vx = rng.normal(0, 3, nu).astype(np.float32); vy = rng.normal(0, 3, nu).astype(np.float32)
    C = w * h
    occ = (rng.random(C) < 0.5).astype(np.float32)
    obs = np.stack([occ, rng.uniform(0.6, 0.95, C), rng.uniform(0.01, 0.2, C), rng.uniform(0.01, 0.3, C)],
                   1).astype(np.float32)
    ang = rng.uniform(0, 2 * np.pi, C)
    lik = np.stack([np.cos(ang), np.sin(ang), rng.normal(0, 3, C), rng.uniform(0.3, 1.5, C)], 1).astype(np.float32)
    pA = np.where(rng.random(C) < 0.7, rng.uniform(0.2, 1.0, C), 0.0).astype(np.float32)
    state = (x, y, vx, vy, np.float32(0.8 / nu), np.zeros(C, np.float32), 3)
    return p, state, obs, lik, pA


def fresh(p, state):
    o = oracle.Oracle(p)
    o.set_state(*state)
    return o


def test_pA_zero_is_the_uniform_exact_cycle():
    p, state, obs, lik, _ = scene()
    a, b = fresh(p, state), fresh(p, state)
    a.step_exact(obs, 0.1)
    b.step_exact_lik(obs, lik, np.zeros(p.width * p.height, np.float32), 0.1)
    sa, sb = a.get_state(), b.get_state()
    for k in ("x", "y", "vx", "vy"):
        assert np.array_equal(sa[k].view(np.uint32), sb[k].view(np.uint32)), k
    assert np.array_equal(a.read_cells()["occ"], b.read_cells()["occ"])


def test_cycle_masses_and_weights():
    """One cycle: every likelihood cell's posterior masses equal A-38's cell update from the cycle's own
    dumps, its members' fixed-point weights sum to R_p, and occupancy = rho_p + rho_b (Eq. 52)."""
    p, state, obs, lik, pA = scene(seed=11)
    o = fresh(p, state)
    o.step_exact_lik(obs, lik, pA, 0.1)
    C = p.width * p.height
    off, perm, Rp = o.dump("OFFSETS"), o.dump("PERM"), o.dump("RP")
    gfx, GS = o.dump("GFX"), o.dump("GS")
    pvx, pvy = o.dump("PRED_VX"), o.dump("PRED_VY")
    cells = o.read_cells()
    rho_p, rho_b = o.dump("RHO_P"), o.dump("RHO_B")
    w_pred = np.float32(p.p_s) * np.float32(0.8 / p.nu)
    checked = 0
    for c in range(C):
        a, b = int(off[c]), int(off[c + 1])
        if not (obs[c, 0] > 0 and pA[c] > 0) or b == a:
            continue
        mem = perm[a:b]
        g = [oracle.doppler_g(float(pvx[i]), float(pvy[i]), *map(float, lik[c])) for i in mem]
        gmax = max(g)
        S = float(np.float32(np.float64(b - a) * np.float64(w_pred)))
        rp, rb, pAe, pi = oracle.exact_lik_cell(S, 1.0, p.p_b, *map(float, obs[c, 1:4]), float(pA[c]), int(GS[c]),
                                                gmax, b - a, float(lik[c, 2]), float(lik[c, 3]), p.sigma_birth_vel)
        assert rho_p[c] == np.float32(rp) and rho_b[c] == np.float32(rb)
        assert cells["occ"][c] == np.float32(np.float32(rp) + np.float32(rb))
        if GS[c] > 0 and Rp[c] > 0:
            pre = np.concatenate([[0], np.cumsum(gfx[mem].astype(np.uint64))])
            Q = [oracle.doppler_Q(int(Rp[c]), pAe, int(pre[j]), int(GS[c]), j, b - a) for j in range(b - a + 1)]
            assert Q[0] == 0 and Q[-1] == int(Rp[c])
        checked += 1
    assert checked > 20


def test_associated_births_follow_the_posterior():
    """Births in likelihood cells: nu_A = round(pi nb); the associated slots' radial speed is drawn from
    the closed-form posterior N(v_r sb^2 / (sb^2 + sd^2), sb^2 sd^2 / (sb^2 + sd^2)) (statistical over
    all associated slots of the cycle, standardised)."""
    p, state, obs, lik, pA = scene(w=40, h=40, nu=30000, nu_b=20000, seed=13)
    obs[:, 0] = 1.0
    pA[:] = 1.0
    o = fresh(p, state)
    o.step_exact_lik(obs, lik, pA, 0.1)
    nA, nb = o.dump("NA"), o.dump("NB")
    bvx, bvy = o.dump("BIRTH_VX"), o.dump("BIRTH_VY")
    sb2 = p.sigma_birth_vel ** 2
    z, j = [], 0
    for c in range(p.width * p.height):
        for r in range(int(nb[c])):
            if r < nA[c]:
                u = lik[c, :2]
                rad = bvx[j] * u[0] + bvy[j] * u[1]
                sd2 = float(lik[c, 3]) ** 2
                mu = float(lik[c, 2]) * sb2 / (sb2 + sd2)
                s = math.sqrt(sb2 * sd2 / (sb2 + sd2))
                if abs(bvx[j]) < p.v_max and abs(bvy[j]) < p.v_max:
                    z.append((rad - mu) / s)
            j += 1
    z = np.array(z)
    assert z.size > 500
    assert abs(z.mean()) < 4 / math.sqrt(z.size) + 0.02 and abs(z.std() - 1) < 0.05


def test_no_measurement_no_likelihood():
    """The likelihood enters only where a measurement occurred (Eq. 38 applies to the measured cell): with
    p_A > 0 everywhere but no cell holding a measurement, the cycle is orc_step_exact bit for bit."""
    p, state, obs, lik, pA = scene(seed=17)
    obs[:, 0] = 0.0
    pA[:] = 0.9
    a, b = fresh(p, state), fresh(p, state)
    a.step_exact(obs, 0.1)
    b.step_exact_lik(obs, lik, pA, 0.1)
    sa, sb = a.get_state(), b.get_state()
    for k in ("x", "y", "vx", "vy"):
        assert np.array_equal(sa[k].view(np.uint32), sb[k].view(np.uint32)), k
    assert np.array_equal(a.read_cells()["occ"], b.read_cells()["occ"])
