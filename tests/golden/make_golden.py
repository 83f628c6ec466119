"""Generate the golden vectors in tests/golden/ by running the REFERENCE.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py [--big]

Every fixture stores the reference's own outputs (torusht.forward / inverse /
forward_real / inverse_real, and the numba kernels fmm_core / flm_core) on
seeded inputs; tests/test_oracle.py pins oracle/ against them (CPU) and
tests/test_gpu_parity.py pins the CUDA path against them (GPU).  Inputs are
regenerated from their seeds by oracle.mw_oracle.gaussian_coeffs /
gaussian_real_coeffs (numpy PCG64, BASELINE.json configs), and the generator
recomputes them here so the stored vectors and the regenerated ones are
checked equal by the tests.

Large fixtures keep a deterministic subsample (index set stored alongside)
plus whole-array checksums, so they stay small enough to commit.
"""

import argparse
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import torusht as ref  # noqa: E402  (the reference, from PYTHONPATH)
from torusht.kernels import _numba as ref_kernels  # noqa: E402

from oracle.mw_oracle import gaussian_coeffs, gaussian_real_coeffs  # noqa: E402

SMALL_CASES = [(1, 0), (2, 0), (2, 1), (3, -2), (4, 3), (8, 0), (8, -5), (16, 2),
               (32, 0), (32, 10)]   # test_mw.py:46-48


def checksums(x):
    x = np.asarray(x)
    return np.array([x.real.sum(), np.imag(x).sum(), (np.abs(x) ** 2).sum(),
                     np.abs(x).max()], dtype=np.float64)


def subsample_idx(n, k, seed):
    rng = np.random.Generator(np.random.PCG64(10_000 + seed))
    return np.sort(rng.choice(n, size=min(n, k), replace=False))


def random_signal(L, spin, seed):
    rng = np.random.Generator(np.random.PCG64(50_000 + seed))
    shape = (L, 2 * L - 1)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def small():
    out = {}
    for L, s in SMALL_CASES:
        for rec in ("trapani", "risbo"):
            v = gaussian_coeffs(L, s, L + abs(s))
            sig = ref.inverse(ref.HarmonicCoeffs(L, s, v.copy()), recursion=rec).samples
            back = ref.forward(ref.MwSignal(L, s, np.array(sig)), recursion=rec).values
            raw = random_signal(L, s, L + abs(s))
            fwd_raw = ref.forward(ref.MwSignal(L, s, raw.copy()), recursion=rec).values
            key = f"L{L}_s{s}_{rec}"
            out[key + "_samples"] = np.asarray(sig)
            out[key + "_back"] = np.asarray(back)
            out[key + "_fwdraw"] = np.asarray(fwd_raw)
    # kernel-level (test_kernels.py:52-92 shapes): L = 9, s in {0, 2, -1}
    L = 9
    cl = np.sqrt((2.0 * np.arange(L) + 1.0) / (4.0 * math.pi))
    for s in (0, 2, -1):
        rng = np.random.Generator(np.random.PCG64(700 + s + 3))
        flm2d = rng.standard_normal((L, 2 * L - 1)) + 1j * rng.standard_normal((L, 2 * L - 1))
        gfold = rng.standard_normal((2 * L - 1, L)) + 1j * rng.standard_normal((2 * L - 1, L))
        for tr in (True, False):
            key = f"k9_s{s}_{'trapani' if tr else 'risbo'}"
            out[key + "_flm2d"] = flm2d
            out[key + "_gfold"] = gfold
            out[key + "_fmm"] = ref_kernels.fmm_core(flm2d, cl, L, s, tr)
            out[key + "_flm"] = ref_kernels.flm_core(gfold, L, s, tr)
    rng = np.random.Generator(np.random.PCG64(777))
    half = rng.standard_normal((8, 8)) + 1j * rng.standard_normal((8, 8))
    gfh = rng.standard_normal((8, 8)) + 1j * rng.standard_normal((8, 8))
    cl8 = np.sqrt((2.0 * np.arange(8) + 1.0) / (4.0 * math.pi))
    out["k8real_in"] = half
    out["k8real_gf"] = gfh
    out["k8real_fmm"] = ref_kernels.fmm_core_real(half, cl8, 8, True)
    out["k8real_flm"] = ref_kernels.flm_core_real(gfh, 8, True)
    # real path, L = 16 (test_mw.py:246-254)
    v = gaussian_real_coeffs(16, 6)
    sr = ref.inverse_real(ref.HarmonicCoeffs(16, 0, v.copy())).samples
    out["real16_samples"] = np.asarray(sr)
    out["real16_back"] = ref.forward_real(ref.MwSignal(16, 0, np.array(sr))).values
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)


def config(L, spin, rec, real=False, seed=0, k=4096, name=None):
    """One BASELINE config: inverse of the seeded coefficients, then forward of
    those samples (round trip), subsampled + checksummed."""
    t0 = time.time()
    if real:
        v = gaussian_real_coeffs(L, seed)
        sig = np.asarray(ref.inverse_real(ref.HarmonicCoeffs(L, 0, v.copy()), recursion=rec).samples)
        back = np.asarray(ref.forward_real(ref.MwSignal(L, 0, sig.copy()), recursion=rec).values)
    else:
        v = gaussian_coeffs(L, spin, seed)
        sig = np.asarray(ref.inverse(ref.HarmonicCoeffs(L, spin, v.copy()), recursion=rec).samples)
        back = np.asarray(ref.forward(ref.MwSignal(L, spin, sig.copy()), recursion=rec).values)
    dt = time.time() - t0
    si = subsample_idx(sig.size, k, L + abs(spin))
    bi = subsample_idx(back.size, k, 2 * L + abs(spin))
    name = name or f"L{L}_s{spin}_{rec}{'_real' if real else ''}"
    np.savez_compressed(
        os.path.join(HERE, f"cfg_{name}.npz"),
        L=L, spin=spin, seed=seed, real=real, recursion=rec,
        input_checksums=checksums(v),
        samples_idx=si, samples_sub=sig.reshape(-1)[si], samples_checksums=checksums(sig),
        back_idx=bi, back_sub=back[bi], back_checksums=checksums(back),
        roundtrip_err=np.max(np.abs(back - v)), ref_seconds=dt,
    )
    print(f"{name}: {dt:.1f}s roundtrip {np.max(np.abs(back - v)):.3e}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also L=2048 risbo (~10 min)")
    args = ap.parse_args()
    small()
    config(64, 0, "trapani")             # C1
    config(256, 2, "trapani")            # C2
    config(256, -2, "trapani")           # C2, s=-2 same seed
    config(1024, 0, "trapani", real=True)  # C3
    config(1100, 0, "risbo")             # past the reference Trapani breakdown
    if args.big:
        config(2048, 0, "risbo")         # C4 map 0


if __name__ == "__main__":
    main()
