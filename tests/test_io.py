"""SSHC/SSHS files (paper_1110_6298_b200.io) against files the reference wrote
(tests/golden/make_io_fixtures.py, pkg/src/torusht/io.py) -- CPU only, except
the device reader."""

import os

import numpy as np
import pytest

from conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def io():
    from paper_1110_6298_b200 import io as m
    return m


def _read(name):
    with open(os.path.join(GOLD, name), "rb") as fh:
        return fh.read()


def test_reads_reference_files(io):
    from oracle.mw_oracle import gaussian_coeffs
    c, grid = io.load_coeffs(os.path.join(GOLD, "io_L6_s-2.sshc"))
    assert (c.band_limit, c.spin, grid) == (6, -2, "mw")
    assert np.array_equal(np.asarray(c.values), gaussian_coeffs(6, -2, 9))
    s, spin, grid = io.load_signal(os.path.join(GOLD, "io_L6_s-2.sshs"))
    assert s.shape == (6, 11) and spin == -2 and grid == "mw"
    c3, grid = io.load_coeffs(os.path.join(GOLD, "io_L3_s0_gl.sshc"))
    assert (c3.band_limit, c3.spin, grid) == (3, 0, "gl")


def test_writes_reference_bytes(io, tmp_path):
    c, _ = io.load_coeffs(os.path.join(GOLD, "io_L6_s-2.sshc"))
    io.save_coeffs(tmp_path / "a.sshc", c)
    assert (tmp_path / "a.sshc").read_bytes() == _read("io_L6_s-2.sshc")
    s, spin, _ = io.load_signal(os.path.join(GOLD, "io_L6_s-2.sshs"))
    io.save_signal(tmp_path / "a.sshs", s, spin)
    assert (tmp_path / "a.sshs").read_bytes() == _read("io_L6_s-2.sshs")
    c3, grid = io.load_coeffs(os.path.join(GOLD, "io_L3_s0_gl.sshc"))
    io.save_coeffs(tmp_path / "b.sshc", c3, grid=grid)
    assert (tmp_path / "b.sshc").read_bytes() == _read("io_L3_s0_gl.sshc")


def test_malformed_files_raise(io, tmp_path):
    import paper_1110_6298_b200 as mw
    good = _read("io_L6_s-2.sshc")
    cases = {
        "truncated": good[:10],
        "magic": b"SSHS" + good[4:],
        "version": good[:4] + bytes([2]) + good[5:],
        "grid": good[:13] + bytes([7]) + good[14:],
        "payload": good[:-16],
    }
    for name, data in cases.items():
        p = tmp_path / f"{name}.sshc"
        p.write_bytes(data)
        with pytest.raises(mw.ContractViolationError):
            io.load_coeffs(p)
    with pytest.raises(mw.ContractViolationError):
        io.save_coeffs(tmp_path / "x.sshc", io.load_coeffs(os.path.join(GOLD, "io_L6_s-2.sshc"))[0],
                       grid="healpix")
    with pytest.raises(mw.ContractViolationError):
        io.save_signal(tmp_path / "x.sshs", np.zeros((4, 6), complex), 0)


def test_pinned_reader_matches(io):
    import torch
    vals, L, spin, grid = io.read_coeffs_to(os.path.join(GOLD, "io_L6_s-2.sshc"))
    assert (L, spin, grid) == (6, -2, "mw")
    ref, _ = io.load_coeffs(os.path.join(GOLD, "io_L6_s-2.sshc"))
    assert np.array_equal(vals.numpy(), np.asarray(ref.values))
    s, spin, grid = io.read_signal_to(os.path.join(GOLD, "io_L6_s-2.sshs"))
    assert tuple(s.shape) == (6, 11) and isinstance(s, torch.Tensor)


@pytest.mark.gpu
def test_file_to_gpu_transform(io):
    import torch
    import paper_1110_6298_b200 as mw
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    vals, L, spin, _ = io.read_coeffs_to(os.path.join(GOLD, "io_L6_s-2.sshc"), device="cuda:0")
    sig = mw.inverse(mw.HarmonicCoeffs(L, spin, vals)).samples
    s_ref, _, _ = io.load_signal(os.path.join(GOLD, "io_L6_s-2.sshs"))
    assert np.max(np.abs(sig.cpu().numpy() - s_ref)) < 1e-12
