"""GPU parity of the evaluation workload (NEXT-4): dog_eval_cells vs the oracle's orc_eval_cells on the
same seeded synthetic readouts -- Mahalanobis distances bit-identical, classification counts exact,
cluster sums within 1e-12 relative (fp64, summation order differs).  Requires a CUDA device."""
import numpy as np
import pytest
import torch

import oracle
from paper_1605_02406_b200 import inputs as I

pytestmark = pytest.mark.gpu


def synthetic_readouts(C, seed):
    rng = np.random.default_rng(seed)
    mean = rng.normal(0, 3, (C, 2)).astype(np.float32)
    a = rng.normal(0, 1, (C, 2, 2))
    P = a @ np.transpose(a, (0, 2, 1)) * rng.uniform(0.01, 4, (C, 1, 1))
    cov = np.stack([P[:, 0, 0], P[:, 1, 1], P[:, 0, 1]], 1).astype(np.float32)
    sing = rng.random(C) < 0.05                      # singular: one particle (var 0) -> regularised
    cov[sing] = 0.0
    valid = (rng.random(C) < 0.7).astype(np.uint8)
    mean[valid == 0] = 0.0; cov[valid == 0] = 0.0
    zero_v = rng.random(C) < 0.02                     # moments with an exactly zero estimate
    mean[zero_v] = 0.0; cov[zero_v] = 0.0
    labels = rng.integers(0, 3, C).astype(np.uint8)
    mask = (rng.random(C) < 0.1).astype(np.uint8)
    return mean, cov, valid, labels, mask


@pytest.mark.parametrize("path", ["tma", "direct"])
def test_eval_matches_oracle(path, monkeypatch):
    """Both paths (bulk-copy staged tiles + direct tail; direct loads) against the oracle."""
    from paper_1605_02406_b200 import dog
    if path == "direct":
        monkeypatch.setenv("DOG_EVAL_NO_TMA", "1")
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    cfg = I.config("cfg1", width=300, height=211, nu=5000, nu_b=100)   # ragged cell count
    g = dog.Filter.from_config(cfg)
    thr = np.r_[0.0, np.logspace(-3, 3, 40), 3.4e38].astype(np.float32)
    for seed in (1, 2):
        mean, cov, valid, labels, mask = synthetic_readouts(cfg.C, seed)
        for use_valid in (True, False):
            mo, co, so = oracle.eval_cells(mean, cov, valid=valid if use_valid else None, labels=labels, mask=mask,
                                           thresholds=thr)
            t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
            r = g.evaluate(labels=t(labels), mask=t(mask), thresholds=thr, mean=t(mean), cov=t(cov),
                           valid=t(valid) if use_valid else None)
            mg = r["m"].cpu().numpy()
            bad = np.nonzero(mg.view(np.uint32) != mo.view(np.uint32))[0]
            assert bad.size == 0, (seed, use_valid, bad[:5], mg[bad[:5]], mo[bad[:5]])
            assert np.array_equal(r["counts"], co)
            assert np.allclose(r["sums"], so, rtol=1e-12, atol=1e-9)


def test_eval_on_live_filter():
    """Filter.evaluate on the filter's own readouts: counts add up to the labelled cells, m >= 0, and
    cells without moments are static (m = 0)."""
    from paper_1605_02406_b200 import dog
    cfg = I.CONFIGS["cfg1"]
    sc = I.scene(cfg)
    g = dog.Filter.from_config(cfg)
    for k in range(6):
        g.step(sc.frame(k, device="cuda"), cfg.dt)
    cells = g.read_cells()
    labels = torch.ones(cfg.C, dtype=torch.uint8, device="cuda")
    labels[cells["occ"] > 0.5] = 2
    thr = np.array([0.0, 1.0, 10.0], np.float32)
    r = g.evaluate(labels=labels, mask=(cells["occ"] > 0.5).to(torch.uint8), thresholds=thr)
    m = r["m"]
    assert bool((m >= 0).all())
    assert r["counts"].sum(axis=1).tolist() == [cfg.C] * 3
    nomom = (cells["mean"].abs().sum(1) == 0) & (cells["cov"].abs().sum(1) == 0)
    assert bool((m[nomom] == 0).all())


def test_eval_threshold_order_and_reset():
    """Thresholds in any order, with duplicates, +-inf and NaN (never met), give the oracle's counts in the
    caller's order; a call that leaves the reductions on the device does not leak into the next call
    (the accumulator resets itself); an empty label set gives all-zero counts."""
    from paper_1605_02406_b200 import dog
    cfg = I.config("cfg1", width=257, height=129, nu=4000, nu_b=64)
    g = dog.Filter.from_config(cfg)
    rng = np.random.default_rng(7)
    thr = np.r_[np.logspace(-2, 2, 20), 1.0, 1.0, 0.0, -0.0, -1.0, -np.inf, np.inf, np.nan, 5.0,
                2.0 + 1e-4 * np.arange(30)].astype(np.float32)          # 30 thresholds in one rank bucket
    thr = thr[rng.permutation(thr.size)]
    mean, cov, valid, labels, mask = synthetic_readouts(cfg.C, 11)
    neg = np.random.default_rng(3).random(cfg.C) < 0.05                 # indefinite P: negative m
    cov[neg, 2] = 0.0; cov[neg, 0] = -np.abs(cov[neg, 0]) - 0.5; cov[neg, 1] = np.abs(cov[neg, 1]) + 0.5
    _, co, so = oracle.eval_cells(mean, cov, valid=valid, labels=labels, mask=mask, thresholds=thr)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    args = dict(labels=t(labels), mask=t(mask), thresholds=thr, mean=t(mean), cov=t(cov), valid=t(valid))
    for _ in range(3):
        g.evaluate(fetch=False, **args)
    r = g.evaluate(**args)
    assert np.array_equal(r["counts"], co)
    assert np.allclose(r["sums"], so, rtol=1e-12, atol=1e-9)
    r0 = g.evaluate(labels=t(np.zeros(cfg.C, np.uint8)), mask=t(mask), thresholds=thr, mean=t(mean), cov=t(cov),
                    valid=t(valid))
    assert not r0["counts"].any()
    assert np.allclose(r0["sums"], so, rtol=1e-12, atol=1e-9)


def test_eval_unaligned_inputs():
    """Readouts that are not 16-byte aligned take the scalar-load path and give the same results."""
    from paper_1605_02406_b200 import dog
    cfg = I.config("cfg1", width=131, height=67, nu=2000, nu_b=32)
    g = dog.Filter.from_config(cfg)
    mean, cov, valid, labels, mask = synthetic_readouts(cfg.C, 5)
    thr = np.logspace(-2, 2, 9).astype(np.float32)
    mo, co, so = oracle.eval_cells(mean, cov, valid=valid, labels=labels, mask=mask, thresholds=thr)
    def shifted(a):                                   # same values, base address offset by one element
        b = torch.zeros((a.shape[0] + 1,) + a.shape[1:], dtype=torch.from_numpy(a).dtype, device="cuda")
        b[1:] = torch.from_numpy(a).cuda()
        return b[1:]
    r = g.evaluate(labels=shifted(labels), mask=shifted(mask), thresholds=thr, mean=shifted(mean), cov=shifted(cov),
                   valid=shifted(valid))
    assert np.array_equal(r["m"].cpu().numpy().view(np.uint32), mo.view(np.uint32))
    assert np.array_equal(r["counts"], co)
    assert np.allclose(r["sums"], so, rtol=1e-12, atol=1e-9)
