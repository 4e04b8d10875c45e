"""Pins of the oracle's ego-motion compensation (NEXT-2, SPEC S:171-179 ego_scroll), against
the SPEC's worked examples and plain properties (scroll semantics by brute force, conservation)."""
import numpy as np
import pytest

import oracle


def make(w=16, h=12, nu=500, seed=3):
    o = oracle.Oracle(oracle.Params(width=w, height=h, nu=nu, nu_b=50, cell_size=0.1, seed=seed))
    rng = np.random.default_rng(seed)
    x = rng.uniform(0, w, nu).astype(np.float32); y = rng.uniform(0, h, nu).astype(np.float32)
    x[:20] = -1073741824.0; y[:20] = -1073741824.0          # sentinel particles
    vx = rng.normal(0, 2, nu).astype(np.float32); vy = rng.normal(0, 2, nu).astype(np.float32)
    mf = rng.uniform(0, 1, w * h).astype(np.float32)
    o.set_state(x, y, vx, vy, 1.0 / nu, mf, 7)
    return o, (x, y, vx, vy, mf)


def test_zero_delta_changes_nothing():                       # SPEC: delta (0,0) -> unchanged bitwise
    o, (x, y, vx, vy, mf) = make()
    assert o.ego_scroll(0.0, 0.0) == (0, 0)
    st = o.get_state()
    for a, b in ((st["x"], x), (st["y"], y), (st["vx"], vx), (st["vy"], vy), (st["m_free"], mf)):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert o.ego_residual() == (0.0, 0.0)


def test_integer_fraction_split():                          # SPEC: 0.25 m with 0.1 m cells -> 2 cells, 0.05 m kept
    o, _ = make()
    assert o.ego_scroll(0.25, 0.0) == (2, 0)
    rx, ry = o.ego_residual()
    cs = float(np.float32(0.1))                              # the f32 cell size as the filter holds it
    assert rx == 0.25 - 2 * cs and abs(rx - 0.05) < 1e-8 and ry == 0.0
    assert o.ego_scroll(0.06, 0.0) == (1, 0)                 # the residual is carried: 0.05 + 0.06 -> 1 cell
    assert abs(o.ego_residual()[0] - 0.01) < 1e-8
    assert o.ego_scroll(-0.25, -0.34) == (-2, -3)            # truncation toward zero (A-32)


def test_scroll_semantics_brute_force():
    w, h = 16, 12
    o, (x, y, vx, vy, mf) = make(w, h)
    sx, sy = o.ego_scroll(0.21, -0.31)                       # (+2, -3) cells (0.2 itself is 1.99999 f32 cells)
    assert (sx, sy) == (2, -3)
    st = o.get_state()
    g_old, g_new = mf.reshape(h, w), st["m_free"].reshape(h, w)
    for r in range(h):
        for c in range(w):
            r0, c0 = r - sy, c - sx
            exp = g_old[r0, c0] if (0 <= r0 < h and 0 <= c0 < w) else 0.0   # leading edge vacuous
            assert g_new[r, c] == exp
    sent = np.float32(-1073741824.0)
    for i in range(x.size):
        if x[i] == sent:
            assert st["x"][i] == sent and st["y"][i] == sent
            continue
        xn, yn = np.float32(x[i] + np.float32(sx)), np.float32(y[i] + np.float32(sy))
        if 0 <= xn < w and 0 <= yn < h:
            assert st["x"][i] == xn and st["y"][i] == yn and st["vx"][i] == vx[i] and st["vy"][i] == vy[i]
        else:                                                # left the grid: sentinel (A-19)
            assert st["x"][i] == sent and st["y"][i] == sent and st["vx"][i] == 0 and st["vy"][i] == 0
    # conservation: every particle is either in the grid or a sentinel
    inside = (st["x"] >= 0) & (st["x"] < w) & (st["y"] >= 0) & (st["y"] < h)
    assert np.count_nonzero(inside) + np.count_nonzero(st["x"] == sent) == x.size


def test_too_large_displacement_is_refused():
    o, (x, y, vx, vy, mf) = make(16, 12)
    assert o.ego_scroll(0.81, 0.0) is None                   # 8 cells = half of 16 columns
    st = o.get_state()
    assert np.array_equal(st["x"].view(np.uint32), x.view(np.uint32))
    assert np.array_equal(st["m_free"].view(np.uint32), mf.view(np.uint32))
    assert o.ego_residual() == (0.0, 0.0)
    assert o.ego_scroll(0.79, 0.0) == (7, 0)
