#!/usr/bin/env python
"""bench.py — MW fwd+inv spherical-harmonic transform throughput on B200.

Driver contract (one JSON line from rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c5s0|c5s2|c3|c4|c2|c1] [--no-extra]

A "step" is one inverse + one forward transform (a fwd+inv pair, as in the
reference's round-trip benchmark cli.py:144-156) of the workload's maps.
`value` = pairs/s over all ranks, inputs resident in HBM, L2 flushed between
steps (or inputs > L2), device-timed with CUDA events, max over ranks.
`e2e` = the same through the public API (HostPipeline over
paper_1110_6298_b200.inverse / forward, or the sharded transforms) with
pinned host buffers: H2D of the coefficients and D2H of the result inside the
timed region.

Workloads (BASELINE.json configs; seeded synthetic N(0,1) coefficients,
PCG64):
  c5s0 (default headline)  L=4096, spin 0, complex, one map; N>1: m-column
                           sharded over the ranks
  c5s2                     L=4096, spin 2, same
  c3                       L=1024, spin 0, real path (inverse_real incl. its
                           reality check, forward_real)
  c4                       L=2048, spin 0, 8 maps sharded by map over ranks
  c2 / c1                  L=256 s=2 / L=64 s=0
The default run also measures c5s2, c3, c4, c2 and c1 and reports each
under "workloads" (compact, at the end of the line).

Multi-GPU: `--gpus N` with N > 1 and no torchrun environment re-launches
itself under torch.distributed.run (N ranks, 127.0.0.1, NCCL); under torchrun
(WORLD_SIZE set) it runs as one rank.

--impl reference times the reference algorithm on the host CPU: oracle/, the
C restatement of the reference's numba cores (bit-identical to them, see
tests/test_oracle.py) plus the reference's numpy FFT stages.  L <= 1024: the
reference's default Trapani recursion; L >= 2048: its Risbo recursion (its
Trapani diverges there).  The headline figure is ONE full, un-extrapolated
fwd+inv pair on all host threads; a serial (1-core, like the stock numba
reference) figure is estimated from a degree prefix and reported beside it.
Rank 0 only.
"""

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "MW fwd+inv SHT transforms/sec at L=1024 & 4096; % of FP64/HBM roofline"
UNIT = "fwd+inv pairs/s"
DATA = "synthetic: seeded N(0,1) coefficients (PCG64), BASELINE.json configs"

WORKLOADS = {
    "c5s0": dict(L=4096, spin=0, real=False, maps=1, shard="mcolumn",
                 name="C5: L=4096 spin 0 complex128, single map"),
    "c5s2": dict(L=4096, spin=2, real=False, maps=1, shard="mcolumn",
                 name="C5: L=4096 spin 2 complex128, single map"),
    "c3": dict(L=1024, spin=0, real=True, maps=1, shard="replica",
               name="C3: L=1024 spin 0 real signal (inverse_real incl. reality check, forward_real)"),
    "c4": dict(L=2048, spin=0, real=False, maps=8, shard="maps",
               name="C4: L=2048 spin 0 complex128, batch of 8 maps sharded by map"),
    "c2": dict(L=256, spin=2, real=False, maps=1, shard="replica",
               name="C2: L=256 spin 2 complex128"),
    "c1": dict(L=64, spin=0, real=False, maps=1, shard="replica",
               name="C1: L=64 spin 0 complex128"),
}
EXTRAS = ("c5s2", "c3", "c4", "c2", "c1")

L2_BYTES = 126 * 1024 * 1024


def wnz(L, spin, real):
    """Useful FP64 work per direction: structurally nonzero
    contraction terms (4 flop each) + the quadrant recursion 4(l+1)^2."""
    ls = np.arange(L, dtype=np.float64)
    sel = ls >= abs(spin)
    n_m = (ls + 1) if real else (2 * ls + 1)
    n_mp = (ls + 1) if spin != 0 else (np.floor(ls / 2) + 1)
    return float(np.sum(4 * n_m[sel] * n_mp[sel]) + np.sum(4 * (ls + 1) ** 2))


def stage_bytes(L, real):
    """§8(d) algorithmic HBM bytes of the forward FFT stages (phi FFT,
    extension + theta FFT, convolution, fold), core term excluded."""
    N = 2 * L - 1
    b = 16 * (2 * L * N + (L * N + N * N) + 2 * N * N + (N * N + N * L))
    return b / 2 if real else b


def inv_stage_bytes(L, real):
    """§8(d) algorithmic HBM bytes of the inverse stages around the core
    (mirror fill, theta synthesis, phi synthesis; no convolution there)."""
    N = 2 * L - 1
    b = 16 * ((N * L + N * N) + (N * N + L * N) + 2 * L * N)
    return b / 2 if real else b


def inv_stage_flops(L, real):
    """5 n log2 n flops of the inverse FFT stages per map: the theta DFT_N of
    each order row and the phi DFT_N of each ring."""
    N = 2 * L - 1
    f = (N + L) * 5.0 * N * math.log2(N)
    return f / 2 if real else f


def stage_flops(L, real):
    """Algorithmic FP64 flops of the forward FFT stages per map, counting an
    n-point complex FFT as 5 n log2 n: the phi DFT_N of L rings, then per
    order row the theta DFT_N and the weight correlation as one forward and
    one inverse FFT of the power-of-two length M >= 4L-3 (the weights'
    spectrum is precomputed).  Real path: half the rows."""
    N = 2 * L - 1
    M = 1 << int(math.ceil(math.log2(4 * L - 3)))
    fft = lambda n: 5.0 * n * math.log2(n)
    f = L * fft(N) + N * (fft(N) + 2 * fft(M))
    return f / 2 if real else f


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def n_maps_total(wl, ws):
    if wl["shard"] == "maps":
        return wl["maps"]
    if wl["shard"] == "mcolumn":
        return 1
    return ws  # replicas: one map per rank


def config_of(wl, ws):
    """The config dict, identical in both arms (same_config)."""
    par = {"maps": f"{wl['maps']} maps sharded by map over {ws} rank(s), no data-path collective",
           "mcolumn": (f"one map, m-column sharded over {ws} ranks (work-balanced |m| ranges, "
                       "NCCL all-to-all ring<->order transposes, all-gather of coefficients)"
                       if ws > 1 else "one map on one GPU"),
           "replica": f"{ws} independent replica(s), one map per rank"}[wl["shard"]]
    maps_total = n_maps_total(wl, ws)
    N = 2 * wl["L"] - 1
    per_map = wl["L"] ** 2 * 16 + wl["L"] * N * (8 if wl["real"] else 16)
    return {"workload": wl["name"], "L": wl["L"], "spin": wl["spin"], "real": wl["real"],
            "maps_total": maps_total, "parallelism": par,
            "l2": ("inputs larger than L2" if per_map * max(1, maps_total // ws) > 2 * L2_BYTES
                   else "L2 flushed between steps"),
            "recursion": "trapani (drop-in default; same GPU recursion as risbo)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, ValueError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
                power.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# ------------------------------------------------------------ CPU reference

def _ref_rec(L):
    # the reference's Trapani diverges above l ~ 1040: Risbo there
    return "trapani" if L <= 1024 else "risbo"


def cpu_full_pair(wl, threads):
    """One full, un-extrapolated inverse + forward of map 0 with the port.
    Returns seconds."""
    from oracle import mw_oracle as O
    L, spin, real = wl["L"], wl["spin"], wl["real"]
    rec = _ref_rec(L)
    v = O.gaussian_real_coeffs(L, 0) if real else O.gaussian_coeffs(L, spin, 0)
    t0 = time.perf_counter()
    if real:
        s = O.inverse_real(v, L, rec, threads=threads)
        O.forward_real(s, L, rec, threads=threads)
    else:
        s = O.inverse(v, L, spin, rec, threads=threads)
        O.forward(s, L, spin, rec, threads=threads)
    return time.perf_counter() - t0


def cpu_prefix_estimate(wl, threads, budget_s, lp_fixed=None):
    """Seconds per pair estimated from the FFT stages at full L plus the
    cores on a degree prefix l < L' scaled by (L/L')^3 (bounded sample)."""
    from oracle import mw_oracle as O
    L, spin = wl["L"], wl["spin"]
    rec = _ref_rec(L)
    N = 2 * L - 1
    rng = np.random.default_rng(0)
    sig = rng.standard_normal((L, N)) + 1j * rng.standard_normal((L, N))
    t0 = time.perf_counter()
    O.gfold_of(sig, L, spin)
    F = rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N))
    rows = O.theta_synthesis(F, L)[:, :L]
    np.fft.ifft(np.fft.ifftshift(rows, axes=0), axis=0)
    t_fft = time.perf_counter() - t0
    if wl["real"]:
        t_fft *= 0.5
    remaining = max(2.0, budget_s - t_fft)
    Lp = lp_fixed or 128
    while True:
        v = O.gaussian_coeffs(Lp, spin, 0)
        flm2d = O.from_flat(v, Lp)
        gf = rng.standard_normal((2 * Lp - 1, Lp)) + 1j * rng.standard_normal((2 * Lp - 1, Lp))
        t0 = time.perf_counter()
        O.fmm_core(flm2d, O.cl_table(Lp), Lp, spin, rec == "trapani", threads=threads)
        O.flm_core(gf, Lp, spin, rec == "trapani", threads=threads)
        t_core = time.perf_counter() - t0
        if wl["real"]:
            t_core *= 0.5
        if lp_fixed or t_core * 8 > remaining or Lp * 2 > L:
            break
        Lp *= 2
    scale = (L / Lp) ** 3
    per_pair = t_fft + t_core * scale
    desc = (f"numpy FFT stages at full L={L} ({t_fft:.1f} s) + {rec} cores (oracle C, "
            f"{threads} thread(s)) on the degree prefix l<{Lp} ({t_core:.2f} s) scaled by "
            f"(L/L')^3={scale:.0f}")
    return per_pair, desc, t_fft, t_core


def cpu_baseline_sample(wl, budget_s):
    """Bounded CPU sample for the GPU arm's `cpu_baseline` (rank 0, N=1)."""
    threads = os.cpu_count() or 1
    if wl["L"] <= 1024:
        dt = cpu_full_pair(wl, threads)
        return {"value": 1.0 / dt, "unit": UNIT, "cores": threads, "kind": "port",
                "sample": (f"one full inverse+forward of map 0 (oracle: reference numpy FFT "
                           f"stages + C restatement of its {_ref_rec(wl['L'])} cores, {threads} "
                           f"threads): {dt:.2f} s")}
    per_pair, desc, _, _ = cpu_prefix_estimate(wl, threads, budget_s)
    return {"value": 1.0 / per_pair, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": "bounded sample, extrapolated: " + desc +
                      "; the reference arm (--impl reference) times a full pair"}


def run_reference(args, wl, ws):
    """--impl reference: the reference algorithm on the host CPU (rank 0)."""
    threads = os.cpu_count() or 1
    L = wl["L"]
    maps = wl["maps"] if wl["shard"] == "maps" else 1
    full_runs = []
    if L <= 1024:  # seconds per pair: warm-up + K timed pairs fit in minutes
        for _ in range(args.warmup):
            cpu_full_pair(wl, threads)
        for _ in range(args.steps):
            full_runs.append(cpu_full_pair(wl, threads))
        t_pair = float(np.median(full_runs))
        how = (f"{args.steps} full inverse+forward pairs of map 0, median (after {args.warmup} "
               "warm-up)")
    else:  # one pair is minutes: time exactly one full pair (no extrapolation)
        t_pair = cpu_full_pair(wl, threads)
        full_runs = [t_pair]
        how = ("ONE full inverse+forward pair of map 0 (un-extrapolated; one pair takes "
               f"{t_pair:.0f} s, so --steps/--warmup are not repeated)")
    value = 1.0 / t_pair
    if maps > 1:
        how += f"; C4's {maps} maps cost {maps} pairs (value = pairs/s)"
    # serial (1 core, like the stock numba reference): the same degree prefix
    # timed on 1 thread and on all threads gives the threading speed-up of the
    # cores, which scales the measured full pair's core time (the FFT stages are
    # single-threaded numpy either way).  At L <= 1024 the prefix is the whole
    # range, so the serial figure is a full measurement.
    serial_pp, serial_desc, t_fft, core_1 = cpu_prefix_estimate(wl, 1, budget_s=20.0)
    if L > 1024:
        lp = int(serial_desc.split("prefix l<")[1].split(" ")[0])
        _, _, _, core_n = cpu_prefix_estimate(wl, threads, budget_s=20.0, lp_fixed=lp)
        speedup = max(1.0, core_1 / max(1e-9, core_n))
        serial_pp = t_fft + (t_pair - t_fft) * speedup
        serial_desc = (f"estimated: the measured full pair's core time x the {threads}-thread "
                       f"speed-up of the cores on a degree prefix ({speedup:.1f}x); " + serial_desc)
    sample = (f"oracle port (reference numpy FFT stages + C restatement of its numba "
              f"{_ref_rec(L)} cores, bit-identical to the reference) on {threads} threads: "
              f"{how}; {t_pair:.1f} s per pair")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_pair * 1e3,
        "higher_is_better": True,
        "scaling": "strong" if wl["shard"] in ("maps", "mcolumn") else "weak",
        "vs_baseline": None, "dtype": "f64 (complex128)", "data": DATA,
        "config": config_of(wl, ws),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample,
                         "serial_1core": {"value": 1.0 / serial_pp, "unit": UNIT, "cores": 1,
                                          "sample": serial_desc}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "pair_seconds": full_runs,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GPU arm

def make_inputs(wl, rank, ws):
    from oracle import mw_oracle as O  # seeded input generation only (before timing)
    L, spin, real = wl["L"], wl["spin"], wl["real"]
    if wl["shard"] == "maps":
        from paper_1110_6298_b200.shard import shard_maps
        mine = shard_maps(wl["maps"], ws, rank)
    elif wl["shard"] == "mcolumn":
        mine = [0]  # one map split over all ranks by order columns and rings
    else:
        mine = [rank]
    vals = [O.gaussian_real_coeffs(L, s) if real else O.gaussian_coeffs(L, spin, s) for s in mine]
    return np.stack(vals), len(mine)


def _unpack_max(red):
    import struct
    return [struct.unpack("<d", struct.pack("<q", int(v)))[0] for v in red.tolist()]


def run_gpu(wl, steps, warmup, rank, ws, local, want_e2e=True, want_clocks=True,
            e2e_steps=None):
    import torch
    import paper_1110_6298_b200 as mw
    from paper_1110_6298_b200 import _lib
    dev = local
    L, spin, real = wl["L"], wl["spin"], wl["real"]
    N = 2 * L - 1
    host, nm = make_inputs(wl, rank, ws)
    plan = mw.get_plan(L, dev, max_batch=nm)
    lib = _lib.load()
    _lib.check(lib.mwsht_plan_set_timing(plan.handle, 0), "set_timing")
    stream = torch.cuda.current_stream(dev)
    sp = _lib._P(stream.cuda_stream)
    flm = torch.from_numpy(host).to(f"cuda:{dev}")                       # (nm, L^2)
    sig = torch.empty((nm, L, N), dtype=torch.float64 if real else torch.complex128,
                      device=f"cuda:{dev}")
    back = torch.empty_like(flm)
    red = torch.zeros((nm, 2), dtype=torch.int64, device=f"cuda:{dev}")
    working = host.nbytes + sig.numel() * sig.element_size() + back.numel() * 16
    flush = torch.empty(L2_BYTES * 2 // 4, dtype=torch.float32, device=f"cuda:{dev}") \
        if working < 4 * L2_BYTES else None
    rec = _lib.TRAPANI

    def step():
        launches = 0
        if real:
            for b in range(nm):
                # inverse_real's reality check (mw.py:537-547), reduced on the device
                _lib.check(lib.mwsht_reality_residual_async(plan.handle, flm[b].data_ptr(),
                                                            red[b].data_ptr(), sp), "reality")
                _lib.check(lib.mwsht_inverse_real_d(plan.handle, flm[b].data_ptr(),
                                                    sig[b].data_ptr(), rec, sp), "inv")
                launches += 1 + plan.last_launches()
                _lib.check(lib.mwsht_forward_real_d(plan.handle, sig[b].data_ptr(),
                                                    back[b].data_ptr(), rec, sp), "fwd")
                launches += plan.last_launches()
        else:
            _lib.check(lib.mwsht_inverse_z_batch(plan.handle, nm, flm.data_ptr(), sig.data_ptr(),
                                                 spin, rec, sp), "inv")
            launches += plan.last_launches()
            _lib.check(lib.mwsht_forward_z_batch(plan.handle, nm, sig.data_ptr(), back.data_ptr(),
                                                 spin, rec, sp), "fwd")
            launches += plan.last_launches()
        return launches

    def core_times():
        c, s = _lib.ctypes.c_float(), _lib.ctypes.c_float()
        lib.mwsht_plan_last_timing(plan.handle, 1, _lib.ctypes.byref(c), _lib.ctypes.byref(s))
        inv_core, inv_stage = c.value, s.value
        lib.mwsht_plan_last_timing(plan.handle, 0, _lib.ctypes.byref(c), _lib.ctypes.byref(s))
        return inv_core, c.value, s.value, inv_stage

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    err = float((back - flm).abs().max().item())
    if real:
        for w, pk in (_unpack_max(r) for r in red.cpu()):
            assert w <= 1e-12 * max(1.0, pk), "reality check failed on the bench input"

    barrier(ws)
    torch.cuda.synchronize()
    clocks = ClockSampler(dev) if want_clocks else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    launches = 0
    for k in range(steps):
        if flush is not None:
            flush.zero_()
        e0[k].record(stream)
        launches += step()
        e1[k].record(stream)
    torch.cuda.synchronize()
    step_ms = [e0[k].elapsed_time(e1[k]) for k in range(steps)]
    clk = clocks.stop() if clocks else None
    # per-kernel attribution pass (not part of `value`): events around the cores
    _lib.check(lib.mwsht_plan_set_timing(plan.handle, 1), "set_timing")
    inv_core = fwd_core = fwd_stage = inv_stage = 0.0
    for k in range(steps):
        if flush is not None:
            flush.zero_()
        step()
        torch.cuda.synchronize()
        a, b, c, d = core_times()
        inv_core += a
        fwd_core += b
        fwd_stage += c
        inv_stage += d
    _lib.check(lib.mwsht_plan_set_timing(plan.handle, 0), "set_timing")
    total_ms = max_over_ranks(float(np.sum(step_ms)), ws)
    # the attribution pass times the last map of each step's batch/loop only for
    # the real path (one map per call); batched calls time the whole batch
    per = nm if real else 1
    out = dict(total_ms=total_ms, steps=steps, maps_per_rank=nm, launches=launches // steps,
               inv_core_ms=inv_core / steps * per, fwd_core_ms=fwd_core / steps * per,
               fwd_stages_ms=fwd_stage / steps * per, inv_stages_ms=inv_stage / steps * per,
               roundtrip_err=err, clocks=clk, plan_bytes=plan.device_bytes())

    if want_e2e:
        # Public API with pinned host buffers: every step copies its coefficients
        # H2D and its result D2H inside the timed region.  HostPipeline (the
        # package's host-streaming API) double-buffers the maps so the copies of
        # neighbouring maps/steps run on the copy engines while one computes.
        from paper_1110_6298_b200.pipeline import HostPipeline
        h_in = torch.from_numpy(host).pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()
        # C4: the step's maps go through the pipeline as batch submissions of
        # `sub` maps (two maps share each Wigner recursion in the cores, so
        # pairs lose nothing against one batch of all maps, and the pipeline's
        # fill and drain -- one H2D and one D2H without overlap -- shrink with
        # the submission size)
        batched = nm > 1 and not real
        sub = int(os.environ.get("MWSHT_BENCH_SUB", "2"))
        sub = sub if batched and nm % sub == 0 else nm
        pipe = HostPipeline(L, spin, kind="roundtrip", real=real, device=dev, depth=2,
                            batch=sub if batched else None)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def e2e_step():
            if batched:
                for b in range(0, nm, sub):
                    pipe.submit(h_in[b:b + sub], h_out[b:b + sub])
                return
            for b in range(nm):
                pipe.submit(h_in[b], h_out[b])

        for _ in range(max(1, warmup)):
            e2e_step()
        pipe.synchronize()
        barrier(ws)
        if flush is not None:
            flush.zero_()
        ev0.record(stream)
        pipe.fence()
        e2e_steps = e2e_steps or steps
        for _ in range(e2e_steps):
            e2e_step()
        pipe.join()
        ev1.record(stream)
        ev1.synchronize()
        pipe.synchronize()  # raises SymmetryError if a real map failed the check
        out["e2e_total_ms"] = max_over_ranks(ev0.elapsed_time(ev1), ws)
        out["e2e_steps"] = e2e_steps
        out["h2d"] = host.nbytes
        out["d2h"] = host.nbytes
        out["e2e_err"] = float(np.max(np.abs(h_out.numpy() - host)))
    return out


def run_gpu_mcolumn(wl, steps, warmup, rank, ws, local, want_clocks=True):
    """C5 over ws GPUs: one map, m-column sharded.  A step is
    inverse (core + theta synthesis of own orders, all-to-all, phi synthesis of
    own rings) then forward (phi DFT of own rings, all-to-all, theta stage + core
    of own orders, all-gather of the coefficient blocks)."""
    import torch
    from paper_1110_6298_b200.shard import MColumnSharding
    L, spin = wl["L"], wl["spin"]
    host, _ = make_inputs(wl, rank, ws)
    sh = MColumnSharding(L, ws, rank, local)
    flm = torch.from_numpy(host[0]).to(f"cuda:{local}")
    stream = torch.cuda.current_stream(local)

    def step():
        rings = sh.inverse(flm, spin)
        return sh.forward(rings, spin)

    for _ in range(warmup):
        out = step()
    torch.cuda.synchronize()
    err = float((out - flm).abs().max().item())
    barrier(ws)
    torch.cuda.synchronize()
    clocks = ClockSampler(local) if want_clocks else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    sh.launches = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        out = step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = sh.launches // steps
    clk = clocks.stop() if clocks else None
    total = max_over_ranks(e0.elapsed_time(e1), ws)
    # e2e: coefficients from pinned host memory, result back to the host, every
    # step; HostPipeline overlaps the copies of neighbouring steps with compute
    from paper_1110_6298_b200.pipeline import HostPipeline
    h_in = torch.from_numpy(host[0]).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    pipe = HostPipeline(L, spin, kind="roundtrip", device=local, depth=2,
                        fn=lambda x: sh.forward(sh.inverse(x, spin), spin))
    pipe.submit(h_in, h_out)
    pipe.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    e0.record(stream)
    pipe.fence()
    for _ in range(steps):
        pipe.submit(h_in, h_out)
    pipe.join()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_total = max_over_ranks(e0.elapsed_time(e1), ws)
    return dict(total_ms=total, steps=steps, maps_per_rank=1, launches=launches, inv_core_ms=0.0,
                fwd_core_ms=0.0, fwd_stages_ms=0.0, roundtrip_err=err, clocks=clk,
                plan_bytes=sh.plan.device_bytes(), e2e_total_ms=e2e_total, h2d=host.nbytes,
                d2h=host.nbytes, e2e_err=float(np.max(np.abs(h_out.numpy() - host[0]))),
                splits=sh.bounds)


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, ws):
    if ws <= 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def fp64_peak(dev):
    from paper_1110_6298_b200 import _lib
    tf, ms = _lib.ctypes.c_double(), _lib.ctypes.c_double()
    _lib.check(_lib.load().mwsht_fp64_probe(dev, _lib.ctypes.byref(tf), _lib.ctypes.byref(ms)),
               "fp64_probe")
    return tf.value


def measured_peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def traffic_table():
    try:
        with open(os.path.join(HERE, "profiles", "traffic.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def summarize(key, wl, r, ws, peak_tf, steps, warmup):
    L, spin, real = wl["L"], wl["spin"], wl["real"]
    maps_total = n_maps_total(wl, ws)
    pairs = maps_total * steps
    value = pairs / (r["total_ms"] / 1e3)
    w = wnz(L, spin, real)
    nm = r["maps_per_rank"]
    fwd_tf = w * nm / (r["fwd_core_ms"] / 1e3) / 1e12 if r["fwd_core_ms"] > 0 else None
    inv_tf = w * nm / (r["inv_core_ms"] / 1e3) / 1e12 if r["inv_core_ms"] > 0 else None
    dom = "forward_core" if r["fwd_core_ms"] >= r["inv_core_ms"] else "inverse_core"
    ach = fwd_tf if dom == "forward_core" else inv_tf
    if ach is None:  # sharded run: whole-step rate per GPU (both directions' W_nz)
        dom = "whole step, per GPU"
        ach = 2 * w * maps_total * steps / (r["total_ms"] / 1e3) / ws / 1e12
    hbm = measured_peaks().get("hbm_gbs")
    st_gbs = (stage_bytes(L, real) * nm / (r["fwd_stages_ms"] / 1e3) / 1e9
              if r["fwd_stages_ms"] > 0 else None)
    st_tf = (stage_flops(L, real) * nm / (r["fwd_stages_ms"] / 1e3) / 1e12
             if r["fwd_stages_ms"] > 0 else None)
    ims = r.get("inv_stages_ms", 0.0)
    ist_gbs = inv_stage_bytes(L, real) * nm / (ims / 1e3) / 1e9 if ims > 0 else None
    ist_tf = inv_stage_flops(L, real) * nm / (ims / 1e3) / 1e12 if ims > 0 else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": steps,
        "warmup": warmup, "ms_per_step": r["total_ms"] / steps, "higher_is_better": True,
        "scaling": "strong" if wl["shard"] in ("maps", "mcolumn") else "weak",
        "vs_baseline": None, "dtype": "f64 (complex128)", "data": DATA,
        "config": config_of(wl, ws),
        "roofline": {"bound": "fp64", "kernel": dom, "achieved": ach, "peak": peak_tf,
                     "unit": "TFLOP/s", "frac": (ach / peak_tf) if (ach and peak_tf) else None,
                     "traffic": traffic_table().get(f"{key}:{dom}"),
                     "work_per_launch_flop": w * nm,
                     "peak_source": "DFMA probe in bench.py (mwsht_fp64_probe, measured live); "
                                    "MEASURED_PEAKS.json has no FP64 entry",
                     "kernels": {
                         "forward_core": {"ms": r["fwd_core_ms"], "tflops": fwd_tf},
                         "inverse_core": {"ms": r["inv_core_ms"], "tflops": inv_tf},
                         "forward_fft_stages": {
                             "ms": r["fwd_stages_ms"], "gbs": st_gbs, "hbm_peak_gbs": hbm,
                             "frac": (st_gbs / hbm) if (st_gbs and hbm) else None,
                             "bytes": "SURVEY §8(d) stage bytes, core term excluded",
                             "fp64_tflops": st_tf,
                             "fp64_frac": (st_tf / peak_tf) if (st_tf and peak_tf) else None,
                             "flops": "5 n log2 n per FFT (bench.stage_flops)"},
                         "inverse_fft_stages": {
                             "ms": ims, "gbs": ist_gbs, "hbm_peak_gbs": hbm,
                             "frac": (ist_gbs / hbm) if (ist_gbs and hbm) else None,
                             "bytes": "SURVEY §8(d): fill + theta synthesis + phi synthesis",
                             "fp64_tflops": ist_tf,
                             "fp64_frac": (ist_tf / peak_tf) if (ist_tf and peak_tf) else None}}},
        "gpu_launches": r["launches"] * steps,
        "roundtrip_max_abs_err": r["roundtrip_err"],
        "clocks": r["clocks"],
        "plan_device_bytes": r["plan_bytes"],
    }
    if "e2e_total_ms" in r:
        e2e_pairs = maps_total * r.get("e2e_steps", steps)
        line["e2e"] = {"value": e2e_pairs / (r["e2e_total_ms"] / 1e3), "unit": UNIT,
                       "steps": r.get("e2e_steps", steps),
                       "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"],
                       "path": "paper_1110_6298_b200.pipeline.HostPipeline (public API), "
                               "pinned host buffers", "max_abs_err": r["e2e_err"]}
    return line


def compact(line):
    """Short per-workload summary for the end of the JSON line."""
    rf = line["roofline"]
    out = {"value": round(line["value"], 3), "ms_per_step": round(line["ms_per_step"], 4),
           "e2e": round(line["e2e"]["value"], 3) if "e2e" in line else None,
           "frac": round(rf["frac"], 4) if rf.get("frac") else None, "kernel": rf["kernel"],
           "fwd_core_ms": round(rf["kernels"]["forward_core"]["ms"], 4),
           "inv_core_ms": round(rf["kernels"]["inverse_core"]["ms"], 4),
           "fwd_stages_ms": round(rf["kernels"]["forward_fft_stages"]["ms"], 4),
           "inv_stages_ms": round(rf["kernels"]["inverse_fft_stages"]["ms"], 4),
           "roundtrip_err": line["roundtrip_max_abs_err"], "launches": line["gpu_launches"]}
    if "cpu_baseline" in line:
        out["cpu_pairs_s"] = line["cpu_baseline"]["value"]
    return out


def relaunch(args):
    """--gpus N > 1 outside torchrun: re-run this script as N NCCL ranks."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    port = env.get("MASTER_PORT") or str(29500 + os.getpid() % 2000)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5s0", choices=sorted(WORKLOADS))
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=25.0)
    ap.add_argument("--band-limit", type=int, default=None,
                    help="harness tests only: override the workload's L")
    args = ap.parse_args()
    ws, rank, local = dist_env()
    if args.band_limit:
        for w in WORKLOADS.values():
            w["L"] = args.band_limit
    wl = WORKLOADS[args.workload]

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, wl, max(ws, args.gpus))
        return

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))

    import torch
    if args.gpus > 1 and ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    # harness self-test only (tests/test_gpu_bench_harness.py): every rank on
    # cuda:0 with a host-staged gloo exchange, so the N-rank code path runs on a
    # one-GPU box; its timings are not scaling figures
    if os.environ.get("MWSHT_BENCH_SAME_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        backend = os.environ.get("MWSHT_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    peak = fp64_peak(local)

    def measure(key, steps, want_clocks, e2e_steps=None):
        w = WORKLOADS[key]
        if w["shard"] == "mcolumn" and ws > 1:
            r = run_gpu_mcolumn(w, steps, args.warmup, rank, ws, local, want_clocks=want_clocks)
        else:
            r = run_gpu(w, steps, args.warmup, rank, ws, local, want_clocks=want_clocks,
                        e2e_steps=e2e_steps)
        return summarize(key, w, r, ws, peak, steps, args.warmup)

    line = measure(args.workload, args.steps, True)
    if rank == 0 and ws == 1:
        line["cpu_baseline"] = cpu_baseline_sample(wl, args.cpu_budget)
    line["fp64_peak_tflops_measured"] = peak
    if not args.no_extra:
        extra = {}
        for key in EXTRAS:
            if key == args.workload:
                continue
            small = WORKLOADS[key]["L"] <= 256
            # sub-millisecond steps: the e2e pipeline's fill and drain (one H2D
            # and one D2H without overlap) would dominate a few steps, so the
            # e2e figure of these runs averages 100 pipelined steps
            e2e_k = 100 if WORKLOADS[key]["L"] <= 1024 else None
            sub = measure(key, max(20, args.steps) if small else max(3, args.steps // 2), False,
                          e2e_steps=e2e_k)
            if rank == 0 and ws == 1 and key == "c3":
                sub["cpu_baseline"] = cpu_baseline_sample(WORKLOADS[key], 15.0)
            extra[key] = compact(sub)
        line["workloads"] = extra
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
