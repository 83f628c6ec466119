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


def subsample_idx(n, k, seed):
    """Same index sets as tests/golden/make_golden.py."""
    rng = np.random.Generator(np.random.PCG64(10_000 + seed))
    return np.sort(rng.choice(n, size=min(n, k), replace=False))


def table_weights(n, seed):
    """Unit complex weights e^{2 pi i u}, u ~ U[0,1) from PCG64(seed)."""
    u = np.random.Generator(np.random.PCG64(seed)).random(n)
    return np.exp(2j * np.pi * u)


def table_sums(x, seed):
    """Row and column checksums of a 2-D array with seeded unit weights:
    rows[i] = sum_j x[i, j] w_c[j], cols[j] = sum_i x[i, j] w_r[i].  A change
    e at one entry moves one row sum and one column sum by |e|."""
    x = np.asarray(x)
    wc = table_weights(x.shape[1], seed)
    wr = table_weights(x.shape[0], seed + 1)
    return x @ wc, wr @ x


def checksum_dev(x, rows_ref, cols_ref, seed):
    """Deviation of x's row/column checksums from the stored ones, per sqrt of
    the number of terms: independent per-entry errors of size <= e move a
    checksum by ~sqrt(n) e, while one entry off by d moves it by d."""
    rows, cols = table_sums(x, seed)
    x = np.asarray(x)
    dr = np.max(np.abs(rows - rows_ref)) / np.sqrt(x.shape[1])
    dc = np.max(np.abs(cols - cols_ref)) / np.sqrt(x.shape[0])
    return float(max(dr, dc))
