"""Shared test helpers (no method arithmetic)."""
import numpy as np

EPS = 2.0 ** -52  # DBL_EPSILON (reading R9)


def nrel(a, b):
    """Normwise relative difference ||a - b||_F / ||b||_F."""
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)
