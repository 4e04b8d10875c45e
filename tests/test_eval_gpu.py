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


def test_eval_matches_oracle():
    from paper_1605_02406_b200 import dog
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
