"""SSHC / SSHS files: harmonic coefficients and MW samples on disk.

Byte-compatible with the reference's formats (pkg/src/torusht/io.py:1-14,
SPEC.md:296): a 14-byte little-endian header

    offset 0   4 bytes  magic b"SSHC" (coefficients) or b"SSHS" (samples)
    offset 4   u8       format version (1)
    offset 5   u32      band limit L
    offset 9   i32      spin
    offset 13  u8       grid code (0 = MW equiangular, 1 = Gauss-Legendre)

then the payload, little-endian complex128: L^2 coefficients in flat
l(l+1)+m order, or the (L, 2L-1) samples row-major (theta rows).

Beyond the reference's numpy readers, ``read_coeffs_to`` / ``read_signal_to``
read a payload straight into page-locked host memory and start an
asynchronous copy to a CUDA device, so a file feeds ``forward`` / ``inverse``
(or ``HostPipeline``) without an extra host copy.  Errors follow the
reference: every malformed file raises ``ContractViolationError``.
"""

import os

import numpy as np

from .errors import ContractViolationError

COEFFS_MAGIC = b"SSHC"
SIGNAL_MAGIC = b"SSHS"
VERSION = 1
HEADER_BYTES = 14
GRIDS = ("mw", "gl")  # code = index


def _header(magic, L, spin, grid):
    if grid not in GRIDS:
        raise ContractViolationError(f"grid must be one of {list(GRIDS)}, got {grid!r}")
    h = bytearray(HEADER_BYTES)
    h[0:4] = magic
    h[4] = VERSION
    h[5:9] = int(L).to_bytes(4, "little", signed=False)
    h[9:13] = int(spin).to_bytes(4, "little", signed=True)
    h[13] = GRIDS.index(grid)
    return bytes(h)


def _parse(h, magic, path):
    """(L, spin, grid) from the first bytes of a file, validated."""
    if len(h) < HEADER_BYTES:
        raise ContractViolationError(f"{path}: truncated header")
    if bytes(h[0:4]) != magic:
        raise ContractViolationError(f"{path}: expected magic {magic!r}, found {bytes(h[0:4])!r}")
    if h[4] != VERSION:
        raise ContractViolationError(f"{path}: unsupported format version {h[4]}")
    if h[13] >= len(GRIDS):
        raise ContractViolationError(f"{path}: unknown grid code {h[13]}")
    L = int.from_bytes(bytes(h[5:9]), "little", signed=False)
    spin = int.from_bytes(bytes(h[9:13]), "little", signed=True)
    return L, spin, GRIDS[h[13]]


def _count(magic, L):
    return L * L if magic == COEFFS_MAGIC else L * (2 * L - 1)


def _open_payload(path, magic):
    """Open `path`, validate header and payload size; returns (file, L, spin, grid, count)."""
    fh = open(path, "rb")
    try:
        L, spin, grid = _parse(fh.read(HEADER_BYTES), magic, path)
        count = _count(magic, L)
        size = os.fstat(fh.fileno()).st_size - HEADER_BYTES
        if size != 16 * count:
            raise ContractViolationError(
                f"{path}: expected {16 * count} payload bytes, found {size}")
    except BaseException:
        fh.close()
        raise
    return fh, L, spin, grid, count


def _write(path, header, values):
    data = np.ascontiguousarray(values, dtype="<c16")
    with open(path, "wb") as fh:
        fh.write(header)
        data.tofile(fh)


# ------------------------------------------------------ the reference's API

def save_coeffs(path, coeffs, grid="mw"):
    """Write a HarmonicCoeffs (numpy or CUDA tensor values) as an SSHC file."""
    _write(path, _header(COEFFS_MAGIC, coeffs.band_limit, coeffs.spin, grid),
           _host(coeffs.values))


def load_coeffs(path):
    """Read an SSHC file: (HarmonicCoeffs, grid name)."""
    from .mw import HarmonicCoeffs
    fh, L, spin, grid, count = _open_payload(path, COEFFS_MAGIC)
    with fh:
        values = np.fromfile(fh, dtype="<c16", count=count).astype(np.complex128)
    return HarmonicCoeffs(L, spin, values), grid


def save_signal(path, samples, spin, grid="mw"):
    """Write (L, 2L-1) samples (array, CUDA tensor or MwSignal) as an SSHS file."""
    from .mw import MwSignal
    if isinstance(samples, MwSignal):
        if samples.spin != spin:
            raise ContractViolationError(
                f"spin {spin} does not match the signal's spin {samples.spin}")
        samples = samples.samples
    arr = _host(samples)
    if arr.ndim != 2 or arr.shape[1] != 2 * arr.shape[0] - 1:
        raise ContractViolationError(f"samples must have shape (L, 2L-1), got {arr.shape}")
    _write(path, _header(SIGNAL_MAGIC, arr.shape[0], spin, grid), arr)


def load_signal(path):
    """Read an SSHS file: (samples (L, 2L-1) complex128, spin, grid name)."""
    fh, L, spin, grid, count = _open_payload(path, SIGNAL_MAGIC)
    with fh:
        arr = np.fromfile(fh, dtype="<c16", count=count).astype(np.complex128)
    return arr.reshape(L, 2 * L - 1), spin, grid


# ------------------------------------------------ pinned / device readers

def _read_pinned(fh, count):
    import torch
    buf = torch.empty(count, dtype=torch.complex128)
    if torch.cuda.is_available():  # page-locked so the device copy is asynchronous
        buf = buf.pin_memory()
    view = buf.numpy().view(np.uint8)
    got = fh.readinto(memoryview(view))
    if got != view.nbytes:
        raise ContractViolationError(f"short read: {got} of {view.nbytes} bytes")
    return buf


def read_coeffs_to(path, device=None):
    """SSHC payload read into pinned host memory, then copied asynchronously to
    `device` (None: stay pinned).  Returns (values tensor, L, spin, grid);
    build HarmonicCoeffs(L, spin, values) to transform it."""
    fh, L, spin, grid, count = _open_payload(path, COEFFS_MAGIC)
    with fh:
        buf = _read_pinned(fh, count)
    return (buf if device is None else buf.to(device, non_blocking=True)), L, spin, grid


def read_signal_to(path, device=None):
    """SSHS payload into pinned memory (and asynchronously onto `device`):
    (samples tensor (L, 2L-1), spin, grid)."""
    fh, L, spin, grid, count = _open_payload(path, SIGNAL_MAGIC)
    with fh:
        buf = _read_pinned(fh, count).view(L, 2 * L - 1)
    return (buf if device is None else buf.to(device, non_blocking=True)), spin, grid


def _host(x):
    """numpy view/copy of an array-like or (CUDA) tensor."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x)
