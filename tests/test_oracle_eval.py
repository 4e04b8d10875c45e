"""Pins of the evaluation workload (NEXT-4; PAPER section VIII Eqs. 85-88, SPEC S:456-543 examples):
the oracle's per-cell Mahalanobis distance / classification counts / cluster sums, with the host-side
statistics of paper_1605_02406_b200.evaluate."""
import math

import numpy as np
import pytest

import oracle
from paper_1605_02406_b200 import evaluate as E


def one(v, P, valid=True):
    mean = np.array([v], np.float32)
    cov = np.array([[P[0][0], P[1][1], P[0][1]]], np.float32)
    m, _, _ = oracle.eval_cells(mean, cov, valid=np.array([valid], np.uint8))
    return float(m[0])


def test_mahalanobis_examples():
    assert one((0, 0), [[1, 0], [0, 1]]) == 0.0
    assert one((2, 0), [[1, 0], [0, 1]]) == 4.0
    assert one((2, 0), [[4, 0], [0, 4]]) == 1.0      # scaling P by 4 divides m by 4
    assert one((3, 4), [[1, 0], [0, 1]], valid=False) == 0.0   # no moments reported: no velocity estimate (A-33)


def test_mahalanobis_closed_form_and_rotation_invariance():
    rng = np.random.default_rng(5)
    for _ in range(200):
        v = rng.normal(0, 3, 2)
        A = rng.normal(0, 1, (2, 2)); P = A @ A.T + 0.1 * np.eye(2)
        exact = float(v @ np.linalg.solve(P, v))
        assert abs(one(v, P) - exact) <= 2e-6 * exact + 1e-6
        th = rng.uniform(0, 2 * math.pi); R = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]])
        assert abs(one(R @ v, R @ P @ R.T) - exact) <= 1e-4 * exact + 1e-5   # invariant up to f32 inputs


def test_regularised_singular_covariance():       # det <= 1e-12 -> P + 1e-6 I
    assert abs(one((1e-3, 0), [[0, 0], [0, 0]]) - 1.0) < 1e-6
    assert abs(one((0, 2e-3), [[0, 0], [0, 0]]) - 4.0) < 1e-5


def test_cluster_statistics_examples():          # SPEC S:476-491 (Eqs. 85-86)
    mean = np.array([[1, 0], [3, 0], [7, 7]], np.float32)
    cov = np.zeros((3, 3), np.float32)
    _, _, sums = oracle.eval_cells(mean, cov, valid=[1, 1, 1], mask=[1, 1, 0])
    st = E.cluster_stats(sums)
    assert st["cells"] == 2 and st["mean_vx"] == 2.0 and st["var_vx"] == 1.0
    mean2 = np.array([[2, 1]] * 4, np.float32); cov2 = np.array([[0.5, 0.25, 0.1]] * 4, np.float32)
    st2 = E.cluster_stats(oracle.eval_cells(mean2, cov2, valid=[1] * 4, mask=[1] * 4)[2])
    assert abs(st2["var_vx"] - 0.5) < 1e-12 and abs(st2["var_vy"] - 0.25) < 1e-12   # identical cells
    with pytest.raises(ValueError):
        E.cluster_stats(oracle.eval_cells(mean2, cov2, valid=[1] * 4, mask=[0] * 4)[2])


def test_nees_examples():                         # SPEC S:496-500 (Eq. 87)
    assert E.nees(5.0, 1.0, 5.0) == 0.0
    assert E.nees(6.0, 1.0, 5.0) == 1.0
    assert E.nees(6.0, 0.25, 5.0) == 4.0


def test_roc_examples_and_monotonicity():
    rng = np.random.default_rng(2)
    n = 400
    labels = rng.integers(1, 3, n).astype(np.uint8)
    v = np.where(labels[:, None] == 2, rng.normal(0, 3, (n, 2)), rng.normal(0, 0.3, (n, 2))).astype(np.float32)
    cov = np.tile(np.array([[1, 1, 0]], np.float32), (n, 1))
    thr = np.r_[0.0, np.logspace(-3, 3, 30), 1e30].astype(np.float32)
    m, counts, _ = oracle.eval_cells(v, cov, valid=np.ones(n, np.uint8), labels=labels, thresholds=thr)
    r = E.roc(counts, thr)
    assert r["tpr"][0] == 1.0 and r["fpr"][0] == 1.0 and r["tpr"][-1] == 0.0 and r["fpr"][-1] == 0.0
    assert all(a >= b for a, b in zip(r["tpr"], r["tpr"][1:])) and all(a >= b for a, b in zip(r["fpr"], r["fpr"][1:]))
    # brute force counts
    for t, row in zip(thr, counts):
        dyn = labels == 2
        assert row[0] == np.count_nonzero(dyn & (m >= t)) and row[2] == np.count_nonzero(~dyn & (m >= t))
    # perfectly separated -> AUC 1
    v2 = np.where(labels[:, None] == 2, 10.0, 0.01).astype(np.float32) * np.array([[1, 0]], np.float32)
    m2, c2, _ = oracle.eval_cells(v2, cov, valid=np.ones(n, np.uint8), labels=labels, thresholds=thr)
    assert E.roc(c2, thr)["auc"] == 1.0
