"""Pins of the CPU oracle's primitives against what the paper / mathematics fix (not against itself).

Each test names the passage it pins.  None of these compute an expected value with the oracle's own
formula: expected values are printed examples (tests/golden), closed forms of a DIFFERENT
formulation (e.g. Dempster's rule by explicit set intersection), library routines (math.log,
scipy.stats) within stated error bounds, or brute-force enumeration.
"""
import json
import math
import os
import struct
from fractions import Fraction

import numpy as np
import pytest

from pinlib import dempster_by_sets, f32, gold, ulp32  # noqa: E402


# ------------------------------------------------------------------ Philox (A-20)
def test_philox_known_answers(orc):
    """P-KAT: the three Random123 known-answer vectors (tests/golden/philox_kat.json)."""
    for v in gold("philox_kat.json")["vectors"]:
        ctr = [int(h, 16) for h in v["ctr"]]
        key = [int(h, 16) for h in v["key"]]
        out = orc.philox(ctr, key)
        assert [f"{x:08x}" for x in out] == v["out"]


def test_uniform_transforms_exact(orc):
    """u(r) = (r>>8) 2^-24 in [0,1), u°(r) in (0,1): exact dyadic values (A-20)."""
    for r in [0, 1, 255, 256, 0xFFFFFFFF, 0x80000000, 0x12345678]:
        assert orc.u01(r) == (r >> 8) * 2.0 ** -24
        assert orc.u01_open(r) == ((r >> 8) | 1) * 2.0 ** -24
        assert 0.0 <= orc.u01(r) < 1.0 and 0.0 < orc.u01_open(r) < 1.0


# ------------------------------------------------------------------ written transcendental spec
def test_ln_spec_accuracy(orc):
    """ln spec vs math.log in fp64: the written f32 polynomial is within 2 ulp (+1e-9 abs) on a
    dense sample of odd m and at every power-of-two boundary (range-reduction edges)."""
    ms = list(range(1, 4097, 2)) + list(range((1 << 24) - 8193, 1 << 24, 2))
    ms += [((1 << e) + d) | 1 for e in range(1, 24) for d in (-3, -1, 1, 3) if ((1 << e) + d) > 0]
    rng = np.random.default_rng(5)
    ms += [int(m) | 1 for m in rng.integers(1, 1 << 24, 20000)]
    worst = 0.0
    for m in ms:
        m = min(m, (1 << 24) - 1)
        got = orc.ln_u24(m)
        ref = math.log(m * 2.0 ** -24)
        err = abs(got - ref)
        assert err <= 2 * ulp32(ref) + 1e-9, (m, got, ref)
        worst = max(worst, err / ulp32(ref))
    assert worst < 2.0


def test_sincos_spec_accuracy(orc):
    """sin/cos(2 pi n 2^-24) vs math.sin/cos: within 2e-7 absolute everywhere, exact at the
    quadrant points (range reduction by integer arithmetic)."""
    assert orc.sincos_2pi_u24(0) == (0.0, 1.0)
    s, c = orc.sincos_2pi_u24(1 << 22)
    assert s == 1.0 and c == 0.0
    s, c = orc.sincos_2pi_u24(2 << 22)
    assert s == 0.0 and c == -1.0
    s, c = orc.sincos_2pi_u24(3 << 22)
    assert s == -1.0 and c == 0.0
    rng = np.random.default_rng(7)
    ns = [int(n) for n in rng.integers(0, 1 << 24, 30000)] + [(1 << 24) - 1, (1 << 21), (1 << 21) - 1, 3 << 21]
    for n in ns:
        s, c = orc.sincos_2pi_u24(n)
        a = 2 * math.pi * n * 2.0 ** -24
        assert abs(s - math.sin(a)) <= 2e-7 and abs(c - math.cos(a)) <= 2e-7, n
        assert abs(s * s + c * c - 1.0) <= 5e-7


def test_box_muller_normal_ks(orc):
    """P-BM (statistical; the paper fixes no generator): normals from the Philox stream pass
    a KS test against N(0,1), the two outputs of a pair are uncorrelated, and the radius is
    Rayleigh-distributed."""
    from scipy import stats
    z0, z1 = [], []
    for i in range(40000):
        r = orc.philox([i, 17, 1, 0], [2406, 0])
        a, b = orc.box_muller(int(r[0]), int(r[1]))
        z0.append(a); z1.append(b)
    z0, z1 = np.array(z0), np.array(z1)
    assert stats.kstest(z0, "norm").pvalue > 0.01
    assert stats.kstest(z1, "norm").pvalue > 0.01
    assert abs(np.corrcoef(z0, z1)[0, 1]) < 0.02
    assert stats.kstest(np.hypot(z0, z1), "rayleigh").pvalue > 0.01


# ------------------------------------------------------------------ Dempster's rule (Eq. 63)
def test_dempster_examples(orc):
    """P-DS: SPEC worked examples (tests/golden/spec_examples.json)."""
    for ex in gold("spec_examples.json")["dempster"]:
        mo, mf = orc.dempster(*ex["a"], *ex["b"])
        assert abs(mo - f32(ex["out"][0])) <= ex["tol"], ex["cite"]
        assert abs(mf - f32(ex["out"][1])) <= ex["tol"], ex["cite"]


def test_dempster_vs_set_definition(orc):
    """P-DS: the oracle's closed form equals the set-intersection definition within f32 rounding,
    is commutative bit for bit, keeps m_O, m_F >= 0 and m_O + m_F <= 1 (BBA normalisation)."""
    rng = np.random.default_rng(11)
    for _ in range(3000):
        a0, a1, b0, b1 = (f32(v) for v in rng.random(4))
        a1 = f32(a1 * (1 - a0)); b1 = f32(b1 * (1 - b0))
        if rng.random() < 0.2:
            b0, b1 = 0.0, f32(rng.random())
        mo, mf = orc.dempster(a0, a1, b0, b1)
        k = a0 * b1 + a1 * b0
        if 1 - k < 1e-3:
            continue
        eo, ef = dempster_by_sets((a0, a1), (b0, b1))
        tol = 8 * 2.0 ** -24 / (1 - k)
        assert abs(mo - eo) <= tol and abs(mf - ef) <= tol, (a0, a1, b0, b1)
        mo2, mf2 = orc.dempster(b0, b1, a0, a1)
        assert (mo, mf) == (mo2, mf2)
        assert mo >= 0 and mf >= 0 and mo + mf <= 1 + 4e-7


def test_dempster_total_conflict_returns_measurement(orc):
    """A-10: 1 - K <= 0 (total conflict, e.g. (1,0) + (0,1)) yields the measurement BBA."""
    assert orc.dempster(1.0, 0.0, 0.0, 1.0) == (0.0, 1.0)


def test_dempster_is_bbf_for_bayesian_bbas(orc):
    """P-BBF (one combination): for Bayesian BBAs (m_O + m_F = 1) Dempster's rule IS the binary
    Bayes filter update, Eq. 1 `eq:BBF`: p' = z p / (z p + (1-z)(1-p)); includes the
    printed example S:349 (p = 0.5, alpha = 3 -> 0.75)."""
    ex = gold("spec_examples.json")["bbf"][0]
    z = ex["alpha"] / (1 + ex["alpha"])
    mo, mf = orc.dempster(ex["p"], 1 - ex["p"], z, 1 - z)
    assert abs(mo - ex["out"]) < 1e-6
    rng = np.random.default_rng(3)
    for _ in range(2000):
        p, z = f32(rng.random()), f32(rng.random())
        mo, mf = orc.dempster(p, f32(1 - p), z, f32(1 - z))
        bbf = z * p / (z * p + (1 - z) * (1 - p))
        tol = 16 * 2.0 ** -24 / (z * p + (1 - z) * (1 - p))   # f32 rounding amplified by 1/(1-K)
        assert abs(mo - bbf) <= tol and abs(mo + mf - 1) <= 2 * tol


# ------------------------------------------------------------------ birth split (Eqs. 64-68)
def test_birth_split_examples(orc):
    for ex in gold("spec_examples.json")["birth_split"]:
        rb, rp = orc.birth_split(ex["m_p"], ex["m_O"], ex["p_b"])
        assert abs(rb - f32(ex["rho_b"])) <= ex["tol"], ex["cite"]
        assert abs(rp - f32(ex["rho_p"])) <= ex["tol"], ex["cite"]


def test_birth_split_relation(orc):
    """Eq. 64 (rho_p + rho_b = m_O) and the mass relation of Eq. 65/67 with the PREDICTED mass
    (A-11): rho_b / rho_p = p_B (1 - m_p) / m_p, checked in exact arithmetic within f32 rounding."""
    rng = np.random.default_rng(4)
    for _ in range(3000):
        m_p, m_O, p_b = f32(rng.random()), f32(rng.random()), f32(rng.random() * 0.2)
        if m_p < 1e-3:
            continue
        rb, rp = orc.birth_split(m_p, m_O, p_b)
        assert abs((rb + rp) - m_O) <= 2 * ulp32(m_O)
        q = Fraction(p_b) * (1 - Fraction(m_p))
        exact_rb = Fraction(m_O) * q / (Fraction(m_p) + q)
        assert abs(rb - float(exact_rb)) <= 4 * ulp32(float(exact_rb)) + 1e-30
        if rp > 1e-6:
            assert abs(rb / rp - float(q / Fraction(m_p))) <= 1e-5 * max(1.0, float(q / Fraction(m_p)))


# ------------------------------------------------------------------ birth slots (Alg. 5, A-15)
def test_slots_spec_example(orc):
    ex = gold("spec_examples.json")["slots"][0]
    Rb = [int(Fraction(f32(v)) * 2 ** 40) for v in ex["rho_b"]]
    assert orc.birth_slots(Rb, ex["nu_b"]).tolist() == ex["nb"]


def test_slots_brute_force(orc):
    """P-SLOT: exactly nu_b slots; every cell gets floor or ceil of its exact share; zero mass gives
    zero; the cumulative count equals round-half-up(nu_b A_c / A) computed with Fractions."""
    rng = np.random.default_rng(8)
    for trial in range(300):
        C = int(rng.integers(1, 40))
        nu_b = int(rng.integers(0, 200))
        Rb = rng.integers(0, 2 ** 40, C).astype(np.uint64)
        Rb[rng.random(C) < 0.4] = 0
        nb = orc.birth_slots(Rb, nu_b)
        A = int(sum(int(v) for v in Rb))
        if A == 0 or nu_b == 0:
            assert nb.sum() == 0
            continue
        assert int(nb.sum()) == nu_b
        acc = 0
        for c in range(C):
            share = Fraction(nu_b * int(Rb[c]), A)
            assert math.floor(share) <= int(nb[c]) <= math.ceil(share)
            if Rb[c] == 0:
                assert nb[c] == 0
            acc += int(Rb[c])
            assert int(nb[: c + 1].sum()) == math.floor(Fraction(nu_b * acc, A) + Fraction(1, 2))


# ------------------------------------------------------------------ systematic resampling (Alg. 7)
def test_resample_copy_counts_bruteforce(orc):
    """P-RES: for many U, every weight gets floor or ceil of nu q_j / W copies, zero weights are never
    drawn, copies sum to nu and indices are non-decreasing (systematic resampling, A-24)."""
    rng = np.random.default_rng(9)
    for trial in range(60):
        n = int(rng.integers(1, 30))
        nu = int(rng.integers(1, 200))
        q = rng.integers(0, 1000, n).astype(np.uint64)
        q[rng.random(n) < 0.3] = 0
        if q.sum() == 0:
            q[0] = 1
        W = int(q.sum())
        for U in [0, 1, 2 ** 31, 2 ** 32 - 1] + [int(u) for u in rng.integers(0, 2 ** 32, 8)]:
            idx, Wr = orc.systematic_resample(q, nu, U)
            assert Wr == W
            assert np.all(np.diff(idx.astype(np.int64)) >= 0)
            copies = np.bincount(idx, minlength=n)
            assert copies.sum() == nu
            for j in range(n):
                share = Fraction(nu * int(q[j]), W)
                assert math.floor(share) <= copies[j] <= math.ceil(share), (q, nu, U, j)
                if q[j] == 0:
                    assert copies[j] == 0


def test_resample_unbiased_over_offsets(orc):
    """E_U[copies_j] = nu q_j / W (Eq. 57 unbiasedness): averaging over an even grid of 2^12 offsets
    U reproduces the share to within 1/2^12 per particle."""
    q = np.array([3, 0, 7, 1, 13, 5], np.uint64)
    nu, W = 10, int(q.sum())
    tot = np.zeros(len(q))
    M = 4096
    for m in range(M):
        idx, _ = orc.systematic_resample(q, nu, m * (2 ** 32 // M))
        tot += np.bincount(idx, minlength=len(q))
    mean = tot / M
    for j in range(len(q)):
        assert abs(mean[j] - nu * int(q[j]) / W) <= 2.0 / M + 1e-12


def test_resample_one_particle_holds_all(orc):
    """one particle holding all weight -> nu copies."""
    q = np.array([0, 0, 123456789, 0], np.uint64)
    idx, W = orc.systematic_resample(q, 1000, 98765)
    assert W == 123456789 and np.all(idx == 2)


# ------------------------------------------------------------------ per-step scalars
def test_step_scalars(orc):
    """c.1: Tc = T / cell, s_p = sigma_pos T / cell, s_v = sigma_vel T, alpha = exp(-T/tau)
    (Table I units per (T/s), A-1; A-9), each rounded once to f32."""
    p = orc.Params(width=4, height=4, nu=1, nu_b=0, cell_size=0.1, sigma_pos=0.02, sigma_vel=0.8, free_tau=2.0)
    Tc, s_p, s_v, al = orc.step_scalars(p, 0.1)
    assert Tc == f32(0.1 / f32(0.1) * 1.0) or abs(Tc - 1.0) <= ulp32(1.0)
    assert abs(s_p - 0.02) <= ulp32(0.02)
    assert abs(s_v - 0.08) <= ulp32(0.08)
    assert abs(al - math.exp(-0.05)) <= ulp32(al)
    p.free_tau = float("inf")
    assert orc.step_scalars(p, 0.1)[3] == 1.0


def test_fixed_point_exponent_keeps_totals_below_2_64():
    """A-23: a cell contributes R_p + R_b <= (rho_p + rho_b) 2^FX, and rho_p + rho_b <= 1 + 2^-24 (DS:
    rho_p = fl(m_O - rho_b), off by at most half an ulp below 1; exact filter: two quotients of a sum <= 1,
    each within a relative 2^-24), so a total over C cells is at most C 2^FX (1 + 2^-24); FX = 40 for every
    grid below 2^24 cells (the pinned examples), 63 - bitlen(C) beyond, never more than one bit given away."""
    import oracle
    for C in [1, 2, 1000, (1 << 24) - 1, 1 << 24, (1 << 24) + 1, (1 << 25) - 1, 4096 * 4096, 8192 * 8192,
              (1 << 31) - 2]:
        fx = oracle.fx_bits(C)
        if C < (1 << 24):
            assert fx == 40
        bound = Fraction(C) * 2 ** fx * (1 + Fraction(1, 2 ** 24))
        assert bound < 2 ** 64, (C, fx)
        if fx < 40:                                      # the next larger exponent would not be safe
            assert Fraction(C) * 2 ** (fx + 2) >= 2 ** 64, (C, fx)
