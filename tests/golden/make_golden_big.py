"""Generate the large-L golden vectors (round 2): forward of RAW (not
band-limited) signals and the headline config C5, at the sizes bench.py runs.

Run in the build container:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_big.py [--only NAME]

Fixtures (tests/golden/big_<name>.npz), each with a deterministic subsample
of every output array plus row and column checksums of the whole array
(tests/helpers.py: ``table_sums``), so a localized error anywhere in the
array moves at least one checksum:

  L2048_s0_risbo_raw   forward of a seeded raw signal, produced by the
                       REFERENCE itself (torusht.forward, recursion="risbo",
                       mw.py:365-375 + kernels/_numba.py:132-166).
  L1100_s2_risbo       inverse of seeded coefficients and forward of a raw
                       signal, spin 2, the REFERENCE (risbo).
  L4096_s0_risbo /     C5: inverse of the seeded BASELINE coefficients and
  L4096_s2_risbo       forward of a raw signal, produced by oracle/ (the C
                       restatement of the reference's numba Risbo cores +
                       the reference's numpy FFT stages; bit-identical to the
                       reference on every fixture of tests/golden/, see
                       tests/test_oracle.py).  The reference itself would take
                       ~1 h per spin here; the oracle runs threaded.
"""

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle import mw_oracle as O  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "tests"))
from helpers import random_signal, subsample_idx, table_sums  # noqa: E402

K_SUB = 1 << 16


def _coeff_table(v, L):
    return O.from_flat(v, L)  # (L, N), zeros for |m| > l


def save(name, L, spin, seed, rec, producer, seconds, samples=None, fwd=None, raw_seed=None):
    out = dict(L=L, spin=spin, seed=seed, recursion=rec, producer=producer, seconds=seconds)
    if samples is not None:
        si = subsample_idx(samples.size, K_SUB, 3 * L + abs(spin))
        rs, cs = table_sums(samples, 1000 + L)
        out.update(samples_idx=si, samples_sub=samples.reshape(-1)[si],
                   samples_rowsum=rs, samples_colsum=cs, samples_max=np.abs(samples).max())
    if fwd is not None:
        bi = subsample_idx(fwd.size, K_SUB, 4 * L + abs(spin))
        rs, cs = table_sums(_coeff_table(fwd, L), 2000 + L)
        out.update(raw_seed=raw_seed, fwd_idx=bi, fwd_sub=fwd[bi], fwd_rowsum=rs,
                   fwd_colsum=cs, fwd_max=np.abs(fwd).max())
    np.savez_compressed(os.path.join(HERE, f"big_{name}.npz"), **out)
    print(f"{name}: {seconds:.1f}s", flush=True)


def ref_case(L, spin, with_inverse, raw_seed, seed=0):
    import torusht as ref
    t0 = time.time()
    samples = None
    if with_inverse:
        v = O.gaussian_coeffs(L, spin, seed)
        samples = np.asarray(ref.inverse(ref.HarmonicCoeffs(L, spin, v.copy()),
                                         recursion="risbo").samples)
    raw = random_signal(L, spin, raw_seed)
    fwd = np.asarray(ref.forward(ref.MwSignal(L, spin, raw), recursion="risbo").values)
    return samples, fwd, time.time() - t0


def oracle_case(L, spin, raw_seed, seed=0):
    t0 = time.time()
    v = O.gaussian_coeffs(L, spin, seed)
    samples = O.inverse(v, L, spin, "risbo")
    raw = random_signal(L, spin, raw_seed)
    fwd = O.forward(raw, L, spin, "risbo")
    return samples, fwd, time.time() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    jobs = {
        "L1100_s2_risbo": lambda: ("reference", 1100, 2, *ref_case(1100, 2, True, 11)),
        "L2048_s0_risbo_raw": lambda: ("reference", 2048, 0, *ref_case(2048, 0, False, 20)),
        "L4096_s0_risbo": lambda: ("oracle", 4096, 0, *oracle_case(4096, 0, 40)),
        "L4096_s2_risbo": lambda: ("oracle", 4096, 2, *oracle_case(4096, 2, 42)),
    }
    raw_seeds = {"L1100_s2_risbo": 11, "L2048_s0_risbo_raw": 20, "L4096_s0_risbo": 40,
                 "L4096_s2_risbo": 42}
    for name, job in jobs.items():
        if args.only and name != args.only:
            continue
        producer, L, spin, samples, fwd, dt = job()
        save(name, L, spin, 0, "risbo", producer, dt, samples, fwd, raw_seeds[name])


if __name__ == "__main__":
    main()
