"""Pipelined transforms of maps that live in host memory.

The reference's callers transform maps one by one from host arrays
(cli.py:144-224). Through ``mw.inverse`` / ``mw.forward`` with numpy arrays,
each call copies its input to the device, runs, and copies back with the GPU
idle during the copies. At L = 4096 one copy is 268 MB (coefficients) to
537 MB (samples), several milliseconds over PCIe each way.

``HostPipeline`` keeps ``depth`` device slots and three streams:
* an H2D copy stream;
* the compute stream, which is the caller's current stream, where the public
  API calls run;
* a D2H copy stream.

``submit(h_in, h_out)`` enqueues three steps, ordered by events:
* the H2D copy of map k into its slot;
* the transform(s), through the public API on device tensors;
* the D2H copy of the result into ``h_out``.

Because the slots are ordered only by events, the copies of maps k-1 and k+1
run on the copy engines while map k computes. Both host buffers should be
pinned (``torch.Tensor.pin_memory()``). Otherwise the copies are synchronous
and nothing overlaps.

The results in ``h_out`` are valid after ``synchronize()``, or after ``join()``
followed by a sync of the caller's stream.

The real path's reality check (``inverse_real`` raises ``SymmetryError``,
mw.py:537-547) needs a device reduction; ``inverse_real`` waits for it, which
would stall the pipeline every map.  The pipeline instead reduces each map's
residual into its own device slot and checks the slots in ``synchronize()``,
which raises ``SymmetryError`` naming the offending submissions.  A violating
map's output is still computed (like every other map in flight).
"""

import struct

import torch

from . import _lib, mw

KINDS = ("inverse", "forward", "roundtrip")


class HostPipeline:
    def __init__(self, band_limit, spin=0, kind="roundtrip", real=False, device=None,
                 depth=2, recursion="trapani", fn=None, batch=None):
        """fn: optional callable (device input) -> device result that replaces
        the public-API transform(s), e.g. a sharded round trip.  batch=B: each
        submission is B maps of one spin (leading dimension B), transformed by
        forward_batch / inverse_batch, which share every Wigner recursion
        between maps (complex maps only)."""
        if kind not in KINDS:
            raise ValueError(f"kind must be one of {KINDS}, got {kind!r}")
        if real and spin != 0:
            from .errors import InvalidSpinError
            raise InvalidSpinError(f"the real-signal path supports spin 0 only, got {spin}")
        if depth < 1:
            raise ValueError("depth must be >= 1")
        if batch is not None and (real or batch < 1):
            raise ValueError("batch needs complex maps and batch >= 1")
        self.batch = batch
        mw.check_band_limit(band_limit)
        self.L, self.spin, self.kind, self.real = band_limit, spin, kind, real
        self.recursion = recursion
        self.fn = fn
        self.device = torch.cuda.current_device() if device is None else int(device)
        dev = torch.device("cuda", self.device)
        L, N = band_limit, 2 * band_limit - 1
        if kind == "forward":
            shape, dtype = (L, N), (torch.float64 if real else torch.complex128)
        else:
            shape, dtype = (L * L,), torch.complex128
        if batch is not None:
            shape = (batch,) + shape
        self.in_shape, self.in_dtype = shape, dtype
        self.h2d = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        self.slots = [dict(buf=torch.empty(shape, dtype=dtype, device=dev),
                           loaded=torch.cuda.Event(), consumed=None) for _ in range(depth)]
        self.k = 0
        self.pending = []  # (submission index, device (2,) uint64 worst/peak) of real inverses
        self.plan = mw.get_plan(L, self.device)

    def _run(self, x):
        L, s, rec = self.L, self.spin, self.recursion
        if self.batch is not None:
            if self.kind == "forward":
                return mw.forward_batch(x, L, s, rec)
            sig = mw.inverse_batch(x, L, s, rec)
            return sig if self.kind == "inverse" else mw.forward_batch(sig, L, s, rec)
        if self.kind in ("inverse", "roundtrip"):
            # the l < |spin| zeros were checked on the host copy in submit()
            if self.real:
                # deferred reality check (see the module docstring)
                red = torch.zeros(2, dtype=torch.int64, device=x.device)
                _lib.call("mwsht_reality_residual_async", self.plan.handle, x.data_ptr(),
                          red.data_ptr(), torch.cuda.current_stream(self.device).cuda_stream)
                self.pending.append((self.k - 1, red))
                mw._check_recursion(rec)
                samples = mw._inverse_real_unchecked(x, L, rec)
                if self.kind == "inverse":
                    return samples
                sig = mw._trusted(mw.MwSignal, L, 0, samples)
            else:
                c = mw._trusted(mw.HarmonicCoeffs, L, s, x, lead_checked=True)
                sig = mw.inverse(c, rec)
                if self.kind == "inverse":
                    return sig.samples
        else:
            sig = mw.MwSignal(L, s, x)
        out = mw.forward_real(sig, rec) if self.real else mw.forward(sig, rec)
        return out.values

    def fence(self):
        """Copies submitted from now on start after the work already on the
        caller's stream (e.g. a timing event recorded there)."""
        cur = torch.cuda.current_stream(self.device)
        self.h2d.wait_stream(cur)
        self.d2h.wait_stream(cur)

    def submit(self, h_in, h_out):
        """Transform host map h_in into host buffer h_out (asynchronously)."""
        if tuple(h_in.shape) != self.in_shape:
            from .errors import ContractViolationError
            raise ContractViolationError(f"pipeline input must have shape {self.in_shape}, "
                                         f"got {tuple(h_in.shape)}")
        if self.kind != "forward" and self.fn is None and self.batch is None and \
                mw._lead_nonzero(h_in.cpu() if h_in.is_cuda else h_in, self.spin * self.spin):
            from .errors import ContractViolationError
            raise ContractViolationError(f"coefficients with degree below |spin|={abs(self.spin)} "
                                         "must be exactly zero")
        cur = torch.cuda.current_stream(self.device)
        slot = self.slots[self.k % len(self.slots)]
        self.k += 1
        if slot["consumed"] is not None:  # the previous map in this slot has been read
            self.h2d.wait_event(slot["consumed"])
        with torch.cuda.stream(self.h2d):
            slot["buf"].copy_(h_in, non_blocking=True)
            slot["loaded"].record(self.h2d)
        cur.wait_event(slot["loaded"])
        out = self.fn(slot["buf"]) if self.fn is not None else self._run(slot["buf"])
        done = torch.cuda.Event()
        done.record(cur)
        slot["consumed"] = done
        self.d2h.wait_event(done)
        with torch.cuda.stream(self.d2h):
            h_out.copy_(out, non_blocking=True)
        out.record_stream(self.d2h)
        return h_out

    def join(self):
        """Make the caller's stream wait for every submitted copy (no host sync)."""
        cur = torch.cuda.current_stream(self.device)
        cur.wait_stream(self.h2d)
        cur.wait_stream(self.d2h)

    def synchronize(self):
        self.join()
        torch.cuda.current_stream(self.device).synchronize()
        self._check_reality()

    def _check_reality(self):
        pending, self.pending = self.pending, []
        bad = []
        for k, red in pending:
            w, pk = (struct.unpack("<d", struct.pack("<q", int(v)))[0] for v in red.tolist())
            tol = 1e-12 * max(1.0, pk)
            if w > tol:
                bad.append(f"submission {k}: residual {w:.3e} > tolerance {tol:.3e}")
        if bad:
            from .errors import SymmetryError
            raise SymmetryError("coefficients violate the reality condition: " + "; ".join(bad))
