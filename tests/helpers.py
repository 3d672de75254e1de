"""Comparison helpers for the GPU-vs-oracle parity tests (test-only)."""
from __future__ import annotations

import numpy as np

NEAR_TIE = 1e-5  # BASELINE north_star: relative distance gap below which an argmin flip is excused


def rel_fro(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def align_signs(X, Xref):
    """Flip columns of X to best match Xref (sign ambiguity of singular pairs, Z5)."""
    X = np.array(X, np.float64, copy=True)
    for c in range(min(X.shape[1], Xref.shape[1])):
        if np.dot(X[:, c], Xref[:, c]) < 0:
            X[:, c] = -X[:, c]
    return X


def label_mismatches(gpu_labels, ref_labels, ref_gaps, log, what=""):
    """Indices where labels differ; every difference must be a near tie (gap < 1e-5) and is logged."""
    g = np.asarray(gpu_labels)
    r = np.asarray(ref_labels)
    bad = np.nonzero(g != r)[0]
    for i in bad:
        log.append((what, int(i), int(r[i]), int(g[i]), float(ref_gaps[i])))
    unexcused = [int(i) for i in bad if not (ref_gaps[i] < NEAR_TIE)]
    return bad, unexcused
