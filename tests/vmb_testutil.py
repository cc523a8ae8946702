import numpy as np


def relfro(a, b):
    """Relative Frobenius error ||a - b|| / ||b|| (bench_main.cpp:64-76)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
