"""HostPipeline: pipelined host-resident transforms give the same results as
the per-call public API (which is itself parity-tested against the oracle)."""

import numpy as np
import pytest
import torch

import paper_1110_6298_b200 as mw
from oracle import mw_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["inverse", "forward", "roundtrip"])
@pytest.mark.parametrize("L,spin,real", [(64, 0, False), (48, 2, False), (64, 0, True)])
def test_pipeline_matches_api(kind, L, spin, real):
    from paper_1110_6298_b200.pipeline import HostPipeline
    nmaps = 5
    N = 2 * L - 1
    coeffs = [O.gaussian_real_coeffs(L, 10 + i) if real else O.gaussian_coeffs(L, spin, 10 + i)
              for i in range(nmaps)]
    inv = mw.inverse_real if real else mw.inverse
    fwd = mw.forward_real if real else mw.forward
    sigs = [np.asarray(inv(mw.HarmonicCoeffs(L, spin, c.copy())).samples) for c in coeffs]
    if kind == "forward":
        h_in = [torch.from_numpy(s.copy()).pin_memory() for s in sigs]
        want = [np.asarray(fwd(mw.MwSignal(L, spin, s.copy())).values) for s in sigs]
        h_out = [torch.empty(L * L, dtype=torch.complex128).pin_memory() for _ in range(nmaps)]
    else:
        h_in = [torch.from_numpy(c.copy()).pin_memory() for c in coeffs]
        if kind == "inverse":
            want = sigs
            dt = torch.float64 if real else torch.complex128
            h_out = [torch.empty((L, N), dtype=dt).pin_memory() for _ in range(nmaps)]
        else:
            want = [np.asarray(fwd(mw.MwSignal(L, spin, s.copy())).values) for s in sigs]
            h_out = [torch.empty(L * L, dtype=torch.complex128).pin_memory() for _ in range(nmaps)]
    pipe = HostPipeline(L, spin, kind=kind, real=real, device=0, depth=2)
    for _ in range(2):  # twice: slots are reused
        for i in range(nmaps):
            pipe.submit(h_in[i], h_out[i])
        pipe.synchronize()
        for i in range(nmaps):
            np.testing.assert_array_equal(h_out[i].numpy(), want[i])


def test_pipeline_rejects_bad_shape():
    from paper_1110_6298_b200.pipeline import HostPipeline
    pipe = HostPipeline(16, 0, kind="roundtrip", device=0)
    with pytest.raises(mw.ContractViolationError):
        pipe.submit(torch.zeros(15 * 15, dtype=torch.complex128), torch.zeros(256))


def test_pipeline_rejects_low_degree_for_spin():
    from paper_1110_6298_b200.pipeline import HostPipeline
    L = 16
    pipe = HostPipeline(L, 2, kind="inverse", device=0)
    bad = torch.zeros(L * L, dtype=torch.complex128)
    bad[1] = 1.0
    with pytest.raises(mw.ContractViolationError):
        pipe.submit(bad, torch.empty((L, 2 * L - 1), dtype=torch.complex128))


def test_pipeline_defers_reality_check_to_synchronize():
    # inverse_real raises SymmetryError for a non-real coefficient set (mw.py:537-547);
    # the pipeline reports it at synchronize() and names the submission
    import torch
    from oracle import mw_oracle as O
    import paper_1110_6298_b200 as mw
    from paper_1110_6298_b200.pipeline import HostPipeline
    L = 24
    good = torch.from_numpy(O.gaussian_real_coeffs(L, 3)).pin_memory()
    bad = torch.from_numpy(O.gaussian_coeffs(L, 0, 4)).pin_memory()
    outs = [torch.empty((L, 2 * L - 1), dtype=torch.float64).pin_memory() for _ in range(3)]
    pipe = HostPipeline(L, 0, kind="inverse", real=True, device=0, depth=2)
    pipe.submit(good, outs[0])
    pipe.submit(bad, outs[1])
    pipe.submit(good, outs[2])
    with pytest.raises(mw.SymmetryError, match="submission 1"):
        pipe.synchronize()
    ref = mw.inverse_real(mw.HarmonicCoeffs(L, 0, good.numpy().copy())).samples
    assert np.max(np.abs(outs[0].numpy() - ref)) == 0.0
    assert np.max(np.abs(outs[2].numpy() - ref)) == 0.0
    pipe.submit(good, outs[0])
    pipe.synchronize()  # the error was reported once; the pipeline keeps working


def test_pipeline_batched_submissions():
    # HostPipeline(batch=B): each submission is B maps through forward_batch /
    # inverse_batch (one recursion shared by the maps); results as per map
    import numpy as np
    import torch
    import paper_1110_6298_b200 as mw
    from paper_1110_6298_b200.pipeline import HostPipeline
    from oracle import mw_oracle as O
    L, s, B = 96, 2, 3
    vals = np.stack([O.gaussian_coeffs(L, s, 20 + k) for k in range(B)])
    h_in = torch.from_numpy(vals).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    h_sig = torch.empty((B, L, 2 * L - 1), dtype=torch.complex128).pin_memory()
    pipe = HostPipeline(L, s, kind="roundtrip", batch=B)
    inv = HostPipeline(L, s, kind="inverse", batch=B)
    for _ in range(3):
        pipe.submit(h_in, h_out)
        inv.submit(h_in, h_sig)
    pipe.synchronize()
    inv.synchronize()
    assert float((h_out - h_in).abs().max()) < 1e-12
    for b in range(B):
        ref = O.inverse(vals[b], L, s)
        assert float(np.max(np.abs(h_sig[b].numpy() - ref))) < 1e-12 * float(np.max(np.abs(ref)))
