import numpy as np

SMALL_CASES = [(1, 0), (2, 0), (2, 1), (3, -2), (4, 3), (8, 0), (8, -5), (16, 2),
               (32, 0), (32, 10)]


def max_abs(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))))


def rel(a, b):
    b = np.asarray(b)
    d = float(np.max(np.abs(b))) if b.size else 1.0
    return max_abs(a, b) / max(d, 1e-300)


def random_signal(L, spin, seed):
    """Same generator as tests/golden/make_golden.py."""
    rng = np.random.Generator(np.random.PCG64(50_000 + seed))
    shape = (L, 2 * L - 1)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def checksums(x):
    x = np.asarray(x)
    return np.array([x.real.sum(), np.imag(x).sum(), (np.abs(x) ** 2).sum(),
                     np.abs(x).max()], dtype=np.float64)
