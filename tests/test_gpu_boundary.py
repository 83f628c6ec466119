"""Boundary semantics of the drop-in (round 2): reentrancy across threads and
streams (the reference CLI's thread pool cli.py:205-207), the
documented band-limit cap (UnsupportedDegreeError, errors.py:24-25), and that
an entry point leaves the caller's current device alone."""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mw():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_1110_6298_b200 as m
    return m


@pytest.mark.parametrize("L", [512, 640])  # 640: H = 2048, the tensor-memory theta stage
def test_two_threads_two_streams_share_one_plan(mw, L):
    # both threads hit the same cached (L, device) plan, each on its own torch
    # stream; the library's event hand-off keeps their scratch use ordered
    import torch
    from oracle import mw_oracle as O
    spin, reps = 2, 6
    vals = [torch.from_numpy(O.gaussian_coeffs(L, spin, 60 + k)).cuda() for k in range(2)]
    expect = []
    for v in vals:
        s = mw.inverse(mw.HarmonicCoeffs(L, spin, v)).samples
        expect.append((s, mw.forward(mw.MwSignal(L, spin, s)).values))
    torch.cuda.synchronize()
    errors = []

    def worker(k):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(reps):
                    s = mw.inverse(mw.HarmonicCoeffs(L, spin, vals[k])).samples
                    f = mw.forward(mw.MwSignal(L, spin, s)).values
                st.synchronize()
                if not (torch.equal(s, expect[k][0]) and torch.equal(f, expect[k][1])):
                    errors.append(k)
        except Exception as exc:  # pragma: no cover - reported below
            errors.append(repr(exc))

    th = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors


def test_band_limit_above_cap_raises_unsupported_degree(mw):
    import torch
    L = 8193
    with pytest.raises(mw.UnsupportedDegreeError):
        mw.get_plan(L)
    assert torch.cuda.current_device() == 0


def test_current_device_is_restored(mw):
    import torch
    from paper_1110_6298_b200 import _lib
    before = torch.cuda.current_device()
    v = np.zeros(16 * 16, complex)
    v[5] = 1.0
    mw.inverse(mw.HarmonicCoeffs(16, 0, v))
    assert torch.cuda.current_device() == before
    assert _lib.load() is not None


def test_plan_cache_keeps_one_plan_per_band_limit(mw):
    from paper_1110_6298_b200 import mw as core
    L = 40
    p1 = core.get_plan(L, 0, max_batch=3)
    assert p1.max_batch == 4
    assert core.get_plan(L, 0, max_batch=2) is p1
    p2 = core.get_plan(L, 0, max_batch=5)
    assert p2.max_batch == 8
    assert sum(1 for (l_, d_) in core._PLANS if l_ == L and d_ == 0) == 1
