"""Shared test helpers: parity metrics of the north_star contract."""
import numpy as np


def subspace_sin(a: np.ndarray, b: np.ndarray) -> float:
    """sin of the largest principal angle: |a - b (b^T a)|_2 (metrics.cpp:59-66)."""
    r = a - b @ (b.T @ a)
    return float(np.linalg.norm(r, 2)) if r.size else 0.0


def canonical_cols(u: np.ndarray) -> np.ndarray:
    """Sign rule of linalg.cpp:18-32 (largest |entry| >= 0, lowest index on ties)."""
    u = u.copy()
    for c in range(u.shape[1]):
        p = int(np.argmax(np.abs(u[:, c])))
        if u[p, c] < 0:
            u[:, c] = -u[:, c]
    return u


def align_core(core_a, factors_a, factors_b):
    """Express core_a in the column signs of factors_b (sign alignment)."""
    core = core_a.copy()
    for m, (fa, fb) in enumerate(zip(factors_a, factors_b)):
        s = np.sign((fa * fb).sum(axis=0))
        s[s == 0] = 1
        shape = [1] * core.ndim
        shape[m] = -1
        core = core * s.reshape(shape)
    return core


def rel(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))
