"""Seeded random vectors for parity checks (U(-1, 1) over the
interleaved N-vector)."""
import numpy as np


def seeded_vector(n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    return np.random.Generator(np.random.PCG64(seed)).uniform(lo, hi, n)
