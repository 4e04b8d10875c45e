"""Evaluation statistics of the filter output (PAPER section VIII): host-side
arithmetic on the device reductions of ``Filter.evaluate`` (include/dog.h ``dog_eval_cells``).

* cluster mean (Eq. 85 `eq:mean_cluster`):  v_S = (1/|S|) sum_c v_c
* cluster variance as a Gaussian mixture (Eq. 86 `eq:gaussian_mixture_x`):
  sigma2_S = (1/|S|) sum_c (sigma2_c + v_c^2) - v_S^2
* NEES (Eq. 87 `eq:NEES_x`): (v_S - v_true)^2 / sigma2_S, 95 % level for 1 DoF = 3.84
* ROC of the static/dynamic classification by Mahalanobis distance: per threshold
  TPR = dynamic cells with m >= tau / dynamic cells, FPR = static cells with m >= tau / static cells,
  AUC by the trapezoid rule over (FPR, TPR) sorted by FPR.
"""
from __future__ import annotations

import numpy as np

CHI2_95_1DOF = 3.84


def cluster_stats(sums) -> dict:
    """From the cluster sums (|S|, sum mean_x, sum var_x + mean_x^2, sum mean_y, sum var_y + mean_y^2)."""
    n = float(sums[0])
    if n <= 0:
        raise ValueError("empty cluster")
    mx, my = sums[1] / n, sums[3] / n
    return {"cells": int(n), "mean_vx": mx, "mean_vy": my,
            "var_vx": sums[2] / n - mx * mx, "var_vy": sums[4] / n - my * my}


def nees(mean: float, var: float, truth: float) -> float:
    if not var > 0:
        raise ValueError("variance must be positive")
    return (mean - truth) ** 2 / var


def roc(counts, thresholds) -> dict:
    """counts[t] = (TP, FN, FP, TN) per threshold (dynamic detection = m >= tau)."""
    c = np.asarray(counts, np.float64).reshape(-1, 4)
    pos, neg = c[:, 0] + c[:, 1], c[:, 2] + c[:, 3]
    if np.any(pos <= 0) or np.any(neg <= 0):
        raise ValueError("ROC needs dynamic and static cells")
    tpr, fpr = c[:, 0] / pos, c[:, 2] / neg
    o = np.lexsort((tpr, fpr))                              # by FPR, then TPR (a monotone staircase)
    f, t = np.r_[0.0, fpr[o], 1.0], np.r_[0.0, tpr[o], 1.0]
    auc = float(np.sum((f[1:] - f[:-1]) * (t[1:] + t[:-1]) / 2.0))
    return {"thresholds": list(map(float, thresholds)), "tpr": tpr.tolist(), "fpr": fpr.tolist(), "auc": auc}
