"""ORACLE — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).

CPU restatement of the reference's MW transform pipeline
(/root/reference/pkg/src/torusht/mw.py) on plain numpy arrays.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` arm may import it.  The shipped package
``paper_1110_6298_b200`` never imports this module and fails loudly when its
CUDA library is missing.

The FFT stages call the same numpy (pocketfft) routines with the same
arguments as the reference, and the O(L^3) cores run the C restatement in
``oracle/cores.c`` (bit-identical to the reference's numba kernels), so the
oracle reproduces the reference's outputs exactly; tests/test_oracle.py pins
that against tests/golden/*.npz, which tests/golden/make_golden.py produced
by importing the reference itself.

Array conventions (reference layout contract, _numpy.py:8-17):
  flat coefficients: index l(l+1)+m, length L^2
  samples: (L, 2L-1), theta rows by phi columns
  2-D coefficient tables: (L, 2L-1), column L-1+m
  Fourier planes: (2L-1, 2L-1), [m, m'], both offset L-1
"""

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle_cores.so")
_lib = None

RECURSIONS = ("trapani", "risbo")


def build():
    """Compile the C cores (oracle/Makefile)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        ci = ctypes.c_int
        lib.oracle_fmm_core.argtypes = [dp, dp, ci, ci, ci, dp, ci]
        lib.oracle_fmm_core_real.argtypes = [dp, dp, ci, ci, dp, ci]
        lib.oracle_flm_core.argtypes = [dp, ci, ci, ci, dp, ci]
        lib.oracle_flm_core_real.argtypes = [dp, ci, ci, dp, ci]
        lib.oracle_trapani_step.argtypes = [dp, ci, ci]
        lib.oracle_risbo_step_into.argtypes = [dp, dp, ci, ci]
        for f in (lib.oracle_fmm_core, lib.oracle_fmm_core_real, lib.oracle_flm_core,
                  lib.oracle_flm_core_real):
            f.restype = ci
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def default_threads():
    return int(os.environ.get("MWSHT_ORACLE_THREADS", "1"))


# ----------------------------------------------------------- cores (C) ---

def fmm_core(flm2d, cl, L, spin, use_trapani, threads=None):
    """_numba.py:74-105 — T[m', L-1+m] = sum_l cl D_m'm D_m',-s f_lm."""
    flm2d = np.ascontiguousarray(flm2d, dtype=np.complex128)
    cl = np.ascontiguousarray(cl, dtype=np.float64)
    out = np.zeros((L, 2 * L - 1), dtype=np.complex128)
    rc = _load().oracle_fmm_core(_p(flm2d), _p(cl), L, spin, int(bool(use_trapani)), _p(out),
                                 threads or default_threads())
    if rc:
        raise MemoryError("oracle fmm_core failed")
    return out


def fmm_core_real(flm_half, cl, L, use_trapani, threads=None):
    """_numba.py:108-128."""
    flm_half = np.ascontiguousarray(flm_half, dtype=np.complex128)
    cl = np.ascontiguousarray(cl, dtype=np.float64)
    out = np.zeros((L, L), dtype=np.complex128)
    rc = _load().oracle_fmm_core_real(_p(flm_half), _p(cl), L, int(bool(use_trapani)), _p(out),
                                      threads or default_threads())
    if rc:
        raise MemoryError("oracle fmm_core_real failed")
    return out


def flm_core(gfold, L, spin, use_trapani, threads=None):
    """_numba.py:131-166 — R[l, L-1+m] = sum_m' D_m'm D_m',-s gfold[L-1+m, m']."""
    gfold = np.ascontiguousarray(gfold, dtype=np.complex128)
    out = np.zeros((L, 2 * L - 1), dtype=np.complex128)
    rc = _load().oracle_flm_core(_p(gfold), L, spin, int(bool(use_trapani)), _p(out),
                                 threads or default_threads())
    if rc:
        raise MemoryError("oracle flm_core failed")
    return out


def flm_core_real(gfold, L, use_trapani, threads=None):
    """_numba.py:169-188."""
    gfold = np.ascontiguousarray(gfold, dtype=np.complex128)
    out = np.zeros((L, L), dtype=np.complex128)
    rc = _load().oracle_flm_core_real(_p(gfold), L, int(bool(use_trapani)), _p(out),
                                      threads or default_threads())
    if rc:
        raise MemoryError("oracle flm_core_real failed")
    return out


def trapani_quadrants(L):
    """Degree-l pi/2 quadrants from trapani_step (_numba.py:53-71), l < L."""
    lib = _load()
    quad = np.zeros((L, L))
    out = []
    for ell in range(L):
        lib.oracle_trapani_step(_p(quad), L, ell)
        out.append(quad[: ell + 1, : ell + 1].copy())
    return out


# ------------------------------------------------- small exact helpers ---

def cl_table(L):
    """sqrt((2l+1)/4pi) — mw.py:144-146."""
    return np.sqrt((2.0 * np.arange(L) + 1.0) / (4.0 * math.pi))


def parity(L, spin):
    """(-1)^(m+s) for m = -(L-1)..L-1 — mw.py:129-132."""
    m = np.arange(-(L - 1), L)
    return np.where((m + spin) % 2 == 0, 1.0, -1.0)


_IPOW = np.array([1.0 + 0.0j, 1.0j, -1.0 + 0.0j, -1.0j])


def ipow(L, spin, sign):
    """i^(sign (m+s)) for m = -(L-1)..L-1 — mw.py:135-141."""
    m = np.arange(-(L - 1), L)
    return _IPOW[(sign * (m + spin)) % 4]


def weights_w(k):
    """w(k) = int_0^pi sin(t) e^{ikt} dt over an integer array — quadrature.py:66-74."""
    k = np.asarray(k)
    out = np.zeros(k.shape, dtype=np.complex128)
    even = k % 2 == 0
    out[even] = 2.0 / (1.0 - k[even].astype(np.float64) ** 2)
    out[k == 1] = 0.5j * math.pi
    out[k == -1] = -0.5j * math.pi
    return out


def smooth5(n):
    """Smallest 2^a 3^b 5^c >= n — mw.py:254-270."""
    best = 1 << max(0, (n - 1).bit_length())
    p5 = 1
    while p5 < best:
        p3 = p5
        while p3 < best:
            p2 = p3
            while p2 < n:
                p2 *= 2
            if n <= p2 < best:
                best = p2
            p3 *= 3
        p5 *= 5
    return best


def flat_maps(L):
    """(row l, column L-1+m) of every flat index l(l+1)+m — mw.py:341-350."""
    ell = np.arange(L)
    rows = np.repeat(ell, 2 * ell + 1)
    cols = np.arange(L * L) - rows * rows + (L - 1 - rows)
    return rows, cols


def to_flat(table, L):
    r, c = flat_maps(L)
    return table[r, c]


def from_flat(values, L):
    r, c = flat_maps(L)
    out = np.zeros((L, 2 * L - 1), dtype=np.complex128)
    out[r, c] = values
    return out


# ------------------------------------------------------ FFT stages -------

def phi_fft(samples, L):
    """mw.py:149-158: G_m(theta_t), columns L-1+m."""
    out = np.fft.fftshift(np.fft.fft(samples, axis=1), axes=1)
    out *= 2.0 * math.pi / (2 * L - 1)
    return out


def periodic_extend(gm, spin):
    """mw.py:161-177: rows t >= L get (-1)^(m+s) G_m(theta_{2L-2-t})."""
    L = gm.shape[0]
    ext = np.empty((2 * L - 1, 2 * L - 1), dtype=np.complex128)
    ext[:L] = gm
    if L > 1:
        ext[L:] = gm[L - 2::-1, :] * parity(L, spin)[None, :]
    return ext


def theta_transform(ext):
    """mw.py:180-192: FFT over rows with e^{-im' theta0}/(2 pi N); rows m'."""
    N = ext.shape[0]
    L = (N + 1) // 2
    mp = np.arange(-(L - 1), L)
    raw = np.fft.fftshift(np.fft.fft(ext, axis=0), axes=0)
    raw *= (np.exp(-1j * mp * (math.pi / N)) / (2.0 * math.pi * N))[:, None]
    return raw


_CONV = {}


def conv_operator(L):
    """mw.py:225-241 (direct matrix up to L=128, else FFT at a 5-smooth length)."""
    op = _CONV.get(L)
    if op is None:
        if L <= 128:
            mp = np.arange(-(L - 1), L)
            data = weights_w(mp[:, None] - mp[None, :])
        else:
            M = smooth5(6 * L - 5)
            data = np.fft.fft(weights_w(np.arange(2 * (L - 1), -2 * L + 1, -1)), n=M)
        data *= 2.0 * math.pi
        op = (L <= 128, data)
        _CONV[L] = op
    return op


def convolve_rows(rows, L):
    """mw.py:244-251: G(m') = 2 pi sum_k F(k) w(k - m') per row."""
    direct, data = conv_operator(L)
    if direct:
        return rows @ data
    M = data.shape[0]
    full = np.fft.ifft(np.fft.fft(rows, n=M, axis=1) * data[None, :], axis=1)
    return full[:, 2 * L - 2: 4 * L - 3].copy()


def fourier_plane(samples, L, spin):
    """forward stages 1-3 (mw.py:371-374): F[m, m'] (FourierPlane layout)."""
    return theta_transform(periodic_extend(phi_fft(samples, L), spin)).T.copy()


def fold_mprime(G, L, spin):
    """mw.py:273-285."""
    fold = np.empty((2 * L - 1, L), dtype=np.complex128)
    fold[:, 0] = G[:, L - 1]
    if L > 1:
        fold[:, 1:] = G[:, L:] + parity(L, spin)[:, None] * G[:, L - 2::-1]
    return fold


def gfold_of(samples, L, spin):
    """Forward pipeline up to the core input: gfold (2L-1, L)."""
    return fold_mprime(convolve_rows(fourier_plane(samples, L, spin), L), L, spin)


# --------------------------------------------------------- transforms ----

def forward(samples, L, spin, recursion="trapani", threads=None):
    """mw.py:365-375 + assemble_flm :299-320 -> flat coefficients (L^2,)."""
    gf = gfold_of(np.asarray(samples), L, spin)
    R = flm_core(gf, L, spin, recursion == "trapani", threads)
    out2d = R * (cl_table(L)[:, None] * ipow(L, spin, +1)[None, :])
    if spin % 2:
        out2d = -out2d
    return to_flat(out2d, L)


def fourier_plane_inverse(values, L, spin, recursion="trapani", threads=None):
    """compute_Fmm, mw.py:378-402 -> F[m, m'] (2L-1, 2L-1)."""
    T = fmm_core(from_flat(values, L), cl_table(L), L, spin, recursion == "trapani", threads)
    phase = ipow(L, spin, -1)
    if spin % 2:
        phase = -phase
    F = np.empty((2 * L - 1, 2 * L - 1), dtype=np.complex128)
    F[:, L - 1:] = T.T * phase[:, None]
    if L > 1:
        F[:, : L - 1] = (F[:, L:] * parity(L, spin)[:, None])[:, ::-1]
    return F


def theta_synthesis(F, L):
    """mw.py:441-446: rows F_m(theta_t) over extended t."""
    mp = np.arange(-(L - 1), L)
    spect = F * (np.exp(1j * mp * (math.pi / (2 * L - 1))) * (2 * L - 1))[None, :]
    return np.fft.ifft(np.fft.ifftshift(spect, axes=1), axis=1)


def inverse(values, L, spin, recursion="trapani", threads=None):
    """mw.py:419-438 -> samples (L, 2L-1) complex."""
    F = fourier_plane_inverse(values, L, spin, recursion, threads)
    rows = theta_synthesis(F, L)[:, :L]
    samples = np.fft.ifft(np.fft.ifftshift(rows, axes=0), axis=0)
    return samples.T * (2 * L - 1)


def _half_signs(n):
    return np.where(np.arange(n) % 2 == 0, 1.0, -1.0)


def forward_real(samples, L, recursion="trapani", threads=None):
    """mw.py:469-501 (spin 0, real samples) -> flat coefficients."""
    samples = np.asarray(samples)
    if np.iscomplexobj(samples):
        samples = samples.real
    gm = np.fft.rfft(samples, axis=1) * (2.0 * math.pi / (2 * L - 1))
    ext = np.empty((2 * L - 1, L), dtype=np.complex128)
    ext[:L] = gm
    if L > 1:
        ext[L:] = gm[L - 2::-1, :] * _half_signs(L)[None, :]
    ghalf = convolve_rows(theta_transform(ext).T, L)
    gf = np.empty((L, L), dtype=np.complex128)                 # mw.py:504-511
    gf[:, 0] = ghalf[:, L - 1]
    if L > 1:
        gf[:, 1:] = ghalf[:, L:] + _half_signs(L)[:, None] * ghalf[:, L - 2::-1]
    R = flm_core_real(gf, L, recursion == "trapani", threads)
    half = R * (cl_table(L)[:, None] * _IPOW[np.arange(L) % 4][None, :])
    out2d = np.zeros((L, 2 * L - 1), dtype=np.complex128)     # mw.py:514-521
    out2d[:, L - 1:] = half
    if L > 1:
        s = np.where(np.arange(1, L) % 2 == 0, 1.0, -1.0)
        out2d[:, : L - 1] = (np.conj(half[:, 1:]) * s[None, :])[:, ::-1]
    return to_flat(out2d, L)


def reality_residual(values, L):
    """(worst, tol) of the reality check, mw.py:537-547."""
    flm2d = from_flat(values, L)
    signs = np.where(np.arange(-(L - 1), L) % 2 == 0, 1.0, -1.0)
    residual = np.conj(flm2d) - signs[None, :] * flm2d[:, ::-1]
    peak = float(np.max(np.abs(values))) if values.size else 0.0
    return float(np.max(np.abs(residual))), 1e-12 * max(1.0, peak)


def inverse_real(values, L, recursion="trapani", threads=None):
    """mw.py:524-559 -> real samples (L, 2L-1) float64."""
    flm2d = from_flat(values, L)
    half = np.ascontiguousarray(flm2d[:, L - 1:])
    T = fmm_core_real(half, cl_table(L), L, recursion == "trapani", threads)
    fhalf = T.T * _IPOW[(-np.arange(L)) % 4][:, None]
    full = np.empty((L, 2 * L - 1), dtype=np.complex128)
    full[:, L - 1:] = fhalf
    if L > 1:
        full[:, : L - 1] = (full[:, L:] * _half_signs(L)[:, None])[:, ::-1]
    rows = theta_synthesis(full, L)[:, :L]
    return np.fft.irfft(rows.T, n=2 * L - 1, axis=1, norm="forward")


# ------------------------------------------- reduced grid, quadrature -----

def synthesize_reduced(values, L, spin, recursion="trapani", threads=None):
    """mw.py:449-466: samples on the reduced (L, L) grid (theta_t, 2 pi p/L):
    theta synthesis, orders folded by residue mod L, an L-point inverse DFT."""
    F = fourier_plane_inverse(values, L, spin, recursion, threads)
    rows = theta_synthesis(F, L)[:, :L]                   # (N orders, L rings)
    m = np.arange(-(L - 1), L)
    bins = np.zeros((L, L), dtype=np.complex128)
    np.add.at(bins, m % L, rows)
    return (np.fft.ifft(bins, axis=0) * L).T.copy()


def ring_weights_v(L):
    """quadrature.py:77-93: v(theta_t) = (1/N) sum_{|m'|<L} w(-m') e^{i m' theta_t}."""
    mp = np.arange(-(L - 1), L)
    theta0 = math.pi / (2 * L - 1)
    spectrum = weights_w(-mp) * np.exp(1j * mp * theta0)
    return np.fft.ifft(np.fft.ifftshift(spectrum))


def quad_weights_q(L, spin):
    """quadrature.py:96-111: q(theta_t) = 2pi/L [v(theta_t) + (-1)^s v(theta_{2L-2-t})]."""
    v = ring_weights_v(L)
    q = v[:L].copy()
    if L > 1:
        q[: L - 1] += (-1.0 if spin % 2 else 1.0) * v[2 * L - 2: L - 1: -1]
    return q * (2.0 * math.pi / L)


def integrate(samples, q):
    """quadrature.py:123-139: sum_t q_t sum_p f[t, p] on the reduced grid."""
    return complex(np.sum(np.asarray(samples).sum(axis=1) * q))


# ------------------------------------------------------------ inputs -----

def gaussian_coeffs(L, spin, seed):
    """BASELINE.json configs / SURVEY 8(d): PCG64(seed); re then im N(0,1);
    entries l < |s| zeroed."""
    rng = np.random.Generator(np.random.PCG64(seed))
    re = rng.standard_normal(L * L)
    im = rng.standard_normal(L * L)
    v = re + 1j * im
    v[: spin * spin] = 0.0
    return v


def gaussian_real_coeffs(L, seed):
    """Config C3: f_l0 = a (real), f_lm = a + ib for m > 0,
    f_l,-m = (-1)^m conj(f_lm)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    a = rng.standard_normal(L * L)
    b = rng.standard_normal(L * L)
    v = np.zeros(L * L, dtype=np.complex128)
    for ell in range(L):
        base = ell * (ell + 1)
        v[base] = a[base]
        if ell:
            m = np.arange(1, ell + 1)
            pos = a[base + m] + 1j * b[base + m]
            v[base + m] = pos
            v[base - m] = np.where(m % 2 == 0, 1.0, -1.0) * np.conj(pos)
    return v


# ------------------------------------------------ Gauss-Legendre comparator
# Restatement of the reference's gl_flm_core / gl_fm_core (_numba.py:191-268),
# vectorised over the order rows mi with the reference's per-element operation
# order (every (l, mi) sum runs over the nodes i in increasing i, as there).

def _libm():
    """The C math library's lgamma/exp: the reference's numba _seed_d
    (_numba.py:191-208) calls these, not CPython's own math.lgamma."""
    import ctypes
    import ctypes.util
    lib = ctypes.CDLL(ctypes.util.find_library("m") or "libm.so.6")
    for name in ("lgamma", "exp"):
        getattr(lib, name).restype = ctypes.c_double
        getattr(lib, name).argtypes = [ctypes.c_double]
    return lib


_LIBM = _libm()


def _gl_seeds(L, spin):
    n = -spin
    N = 2 * L - 1
    cst, ec, es, l0 = np.zeros(N), np.zeros(N), np.zeros(N), np.zeros(N, dtype=np.int64)
    for mi in range(N):
        m = mi - (L - 1)
        if n >= abs(m):
            mm, nn, sign = m, n, 1.0
        elif n <= -abs(m):
            mm, nn, sign = -m, -n, (-1.0 if (m - n) % 2 else 1.0)
        elif m >= abs(n):
            mm, nn, sign = n, m, (-1.0 if (m - n) % 2 else 1.0)
        else:
            mm, nn, sign = -n, -m, 1.0
        cst[mi] = sign * _LIBM.exp(0.5 * (_LIBM.lgamma(2 * nn + 1.0) - _LIBM.lgamma(nn + mm + 1.0)
                                          - _LIBM.lgamma(nn - mm + 1.0)))
        ec[mi], es[mi], l0[mi] = nn + mm, nn - mm, nn
    return cst, ec, es, l0


def _int_power(a, e):
    """float ** int as numba evaluates it (exponentiation by squaring from
    r = 1, the reference's ch[i] ** ec with integer ec)."""
    e = np.asarray(e, dtype=np.int64).copy()
    r = np.ones(e.shape)
    base = np.full(e.shape, float(a))
    while np.any(e != 0):
        odd = (e & 1) == 1
        r = np.where(odd, r * base, r)
        e >>= 1
        base = base * base
    return r


def _gl_chains(L, spin, x, ch, sh, visit):
    """Run every (mi, node) chain; visit(el, i, dl, active) per degree."""
    n = -spin
    N = 2 * L - 1
    m = np.arange(N) - (L - 1)
    cst, ec, es, l0 = _gl_seeds(L, spin)
    mf = m.astype(np.float64)
    for i in range(L):
        xi = x[i]
        dl = np.zeros(N)
        dlm1 = np.zeros(N)
        for el in range(L):
            start = l0 == el
            if np.any(start):
                dl[start] = cst[start] * _int_power(ch[i], ec[start]) * _int_power(sh[i], es[start])
                dlm1[start] = 0.0
            active = l0 <= el
            visit(el, i, dl, active)
            if el == L - 1:
                break
            if el == 0:
                nxt = xi * dl
            else:
                with np.errstate(invalid="ignore"):
                    den = el * np.sqrt(((el + 1.0) ** 2 - mf * mf) * ((el + 1.0) ** 2 - n * n))
                    t = ((2.0 * el + 1.0) * (el * (el + 1.0) * xi - m * n) * dl
                         - (el + 1.0) * np.sqrt((el * el - mf * mf) * (el * el - n * n)) * dlm1)
                    nxt = t / den
            dlm1 = np.where(active, dl, dlm1)
            dl = np.where(active, nxt, dl)


def gl_flm_core(a, x, ch, sh, L, spin):
    R = np.zeros((L, 2 * L - 1), dtype=np.complex128)

    def visit(el, i, dl, active):
        R[el, active] += dl[active] * a[active, i]

    _gl_chains(L, spin, x, ch, sh, visit)
    return R


def gl_fm_core(flm_scaled, x, ch, sh, L, spin):
    F = np.zeros((2 * L - 1, L), dtype=np.complex128)
    acc = {}

    def visit(el, i, dl, active):
        if el == 0:
            acc[i] = np.zeros(2 * L - 1, dtype=np.complex128)
        acc[i][active] += flm_scaled[el, active] * dl[active]
        if el == L - 1:
            F[:, i] = acc.pop(i)

    _gl_chains(L, spin, x, ch, sh, visit)
    return F


def gl_forward(samples, L, spin, nodes, weights):
    """gl.py:114-148 with the oracle's core."""
    gm = np.fft.fftshift(np.fft.fft(samples, axis=1), axes=1) * (2.0 * math.pi / (2 * L - 1))
    a = np.ascontiguousarray(gm.T * weights[None, :])
    ch, sh = np.sqrt((1.0 + nodes) / 2.0), np.sqrt((1.0 - nodes) / 2.0)
    out2d = gl_flm_core(a, nodes, ch, sh, L, spin) * cl_table(L)[:, None]
    if spin % 2:
        out2d = -out2d
    return to_flat(out2d, L)


def gl_inverse(values, L, spin, nodes):
    """gl.py:151-178 with the oracle's core."""
    flm_scaled = from_flat(values, L) * cl_table(L)[:, None]
    if spin % 2:
        flm_scaled = -flm_scaled
    ch, sh = np.sqrt((1.0 + nodes) / 2.0), np.sqrt((1.0 - nodes) / 2.0)
    F = gl_fm_core(flm_scaled, nodes, ch, sh, L, spin)
    return np.fft.ifft(np.fft.ifftshift(F.T, axes=1), axis=1) * (2 * L - 1)
