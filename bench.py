#!/usr/bin/env python
"""bench.py — MW fwd+inv spherical-harmonic transform throughput on B200.

Driver contract (one JSON line from rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c5s0|c5s2|c3|c4|c2|c1] [--no-extra]

A "step" is one inverse + one forward transform (a fwd+inv pair, as in the
reference's round-trip benchmark cli.py:144-156) of the workload's maps.
`value` = pairs/s over all ranks, inputs resident in HBM, L2 flushed between
steps (or inputs > L2), device-timed with CUDA events, max over ranks.
`e2e` = the same through the public API (paper_1110_6298_b200.inverse /
forward) with pinned host buffers: H2D of the coefficients and D2H of the
result inside the timed region.

Workloads (BASELINE.json configs; seeded synthetic N(0,1) coefficients,
PCG64):
  c5s0 (default headline)  L=4096, spin 0, complex, one map per rank
  c5s2                     L=4096, spin 2
  c3                       L=1024, spin 0, real path (inverse_real/forward_real)
  c4                       L=2048, spin 0, 8 maps sharded by map over ranks
  c2 / c1                  L=256 s=2 / L=64 s=0
The default run also measures c3, c5s2 and c4 briefly and reports them
under "workloads".

--impl reference times the reference algorithm on the host CPU: the oracle/
C restatement of the reference's numba cores (bit-identical to it) with all
host threads + the reference's numpy FFT stages, as a bounded sample (see
"sample" in the line).  Rank 0 only.
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

WORKLOADS = {
    "c5s0": dict(L=4096, spin=0, real=False, maps=1, shard="mcolumn",
                 name="C5: L=4096 spin 0 complex128, single map"),
    "c5s2": dict(L=4096, spin=2, real=False, maps=1, shard="mcolumn",
                 name="C5: L=4096 spin 2 complex128, single map"),
    "c3": dict(L=1024, spin=0, real=True, maps=1, shard="replica",
               name="C3: L=1024 spin 0 real signal (forward_real/inverse_real)"),
    "c4": dict(L=2048, spin=0, real=False, maps=8, shard="maps",
               name="C4: L=2048 spin 0 complex128, batch of 8 maps sharded by map"),
    "c2": dict(L=256, spin=2, real=False, maps=1, shard="replica",
               name="C2: L=256 spin 2 complex128"),
    "c1": dict(L=64, spin=0, real=False, maps=1, shard="replica",
               name="C1: L=64 spin 0 complex128"),
}

L2_BYTES = 126 * 1024 * 1024


def wnz(L, spin, real):
    """Useful FP64 work per direction."""
    ls = np.arange(L, dtype=np.float64)
    sel = ls >= abs(spin)
    n_m = (ls + 1) if real else (2 * ls + 1)
    n_mp = (ls + 1) if spin != 0 else (np.floor(ls / 2) + 1)
    return float(np.sum(4 * n_m[sel] * n_mp[sel]) + np.sum(4 * (ls + 1) ** 2))


def stage_bytes(L, real):
    """Algorithmic HBM bytes per direction of the FFT-stage pipeline (§8d)."""
    N = 2 * L - 1
    b = 16 * (2 * L * N + (L * N + N * N) + 2 * N * N + (N * N + N * L) + (N * L + L * L))
    return b / 2 if real else b


# ------------------------------------------------------------ environment

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


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

def cpu_reference(wl, budget_s=25.0, threads=None):
    """Time the reference algorithm on the host (oracle/), bounded sample.

    Returns (pairs_per_s, sample_description, cores).  L <= 1024: full
    inverse+forward with the reference's default Trapani recursion.  Larger
    L: the reference Trapani diverges, so the Risbo cores are
    timed on a degree prefix l < L' and scaled by (L/L')^3 (their cost is
    sum_l O(l^2)), while the numpy FFT stages run at full L.
    """
    from oracle import mw_oracle as O
    threads = threads or os.cpu_count() or 1
    L, spin, real = wl["L"], wl["spin"], wl["real"]
    if L <= 1024:
        v = O.gaussian_real_coeffs(L, 0) if real else O.gaussian_coeffs(L, spin, 0)
        t0 = time.perf_counter()
        if real:
            s = O.inverse_real(v, L, "trapani", threads=threads)
            O.forward_real(s, L, "trapani", threads=threads)
        else:
            s = O.inverse(v, L, spin, "trapani", threads=threads)
            O.forward(s, L, spin, "trapani", threads=threads)
        dt = time.perf_counter() - t0
        return 1.0 / dt, (
            f"full inverse+forward of one map (oracle: numpy FFT stages + C cores, trapani, "
            f"{threads} threads), {dt:.2f} s"), threads
    # FFT stages at full L
    N = 2 * L - 1
    rng = np.random.default_rng(0)
    sig = rng.standard_normal((L, N)) + 1j * rng.standard_normal((L, N))
    t0 = time.perf_counter()
    O.gfold_of(sig, L, spin)
    t_fwd_fft = time.perf_counter() - t0
    F = rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N))
    t0 = time.perf_counter()
    rows = O.theta_synthesis(F, L)[:, :L]
    np.fft.ifft(np.fft.ifftshift(rows, axes=0), axis=0)
    t_inv_fft = time.perf_counter() - t0
    # Risbo core prefix, sized to the remaining budget
    remaining = max(2.0, budget_s - t_fwd_fft - t_inv_fft)
    Lp = 256
    t_core = None
    while True:
        v = O.gaussian_coeffs(Lp, spin, 0)
        flm2d = O.from_flat(v, Lp)
        gf = rng.standard_normal((2 * Lp - 1, Lp)) + 1j * rng.standard_normal((2 * Lp - 1, Lp))
        t0 = time.perf_counter()
        O.fmm_core(flm2d, O.cl_table(Lp), Lp, spin, False, threads=threads)
        O.flm_core(gf, Lp, spin, False, threads=threads)
        t_core = time.perf_counter() - t0
        if t_core * 8 > remaining or Lp * 2 > L:
            break
        Lp *= 2
    scale = (L / Lp) ** 3
    per_pair = t_fwd_fft + t_inv_fft + t_core * scale
    return 1.0 / per_pair, (
        f"numpy FFT stages at full L={L} ({t_fwd_fft + t_inv_fft:.1f} s) + reference Risbo cores "
        f"(oracle C restatement, {threads} threads) on the degree prefix l<{Lp} ({t_core:.2f} s) "
        f"scaled by (L/L')^3={scale:.0f}; one pair = {per_pair:.1f} s"), threads


# ------------------------------------------------------------ GPU arm

def make_inputs(wl, rank, ws, torch, dev):
    from oracle import mw_oracle as O
    L, spin, real = wl["L"], wl["spin"], wl["real"]
    if wl["shard"] == "maps":
        from paper_1110_6298_b200.shard import shard_maps
        mine = shard_maps(wl["maps"], ws, rank)
    elif wl["shard"] == "mcolumn":
        mine = [0]  # one map split over all ranks by order columns and rings
    else:
        mine = [rank]
    vals = []
    for seed in mine:
        v = O.gaussian_real_coeffs(L, seed) if real else O.gaussian_coeffs(L, spin, seed)
        vals.append(v)
    host = np.stack(vals)
    return host, len(mine)


def run_gpu(wl, steps, warmup, rank, ws, local, want_e2e=True, want_clocks=True):
    import torch
    import paper_1110_6298_b200 as mw
    from paper_1110_6298_b200 import _lib
    torch.cuda.set_device(local)
    dev = local
    L, spin, real = wl["L"], wl["spin"], wl["real"]
    N = 2 * L - 1
    host, nm = make_inputs(wl, rank, ws, torch, dev)
    plan = mw.get_plan(L, dev, max_batch=nm)
    lib = _lib.load()
    # the plan's per-core timing events sit between kernels and would serialise
    # the programmatic-dependent-launch overlap: off for the timed loop, on for a
    # separate pass that attributes time to the cores (roofline)
    _lib.check(lib.mwsht_plan_set_timing(plan.handle, 0), "set_timing")
    stream = torch.cuda.current_stream(dev)
    sp = _lib._P(stream.cuda_stream)
    flm = torch.from_numpy(host).to(f"cuda:{dev}")                       # (nm, L^2)
    if real:
        sig = torch.empty((nm, L, N), dtype=torch.float64, device=f"cuda:{dev}")
    else:
        sig = torch.empty((nm, L, N), dtype=torch.complex128, device=f"cuda:{dev}")
    back = torch.empty_like(flm)
    working = host.nbytes + sig.numel() * sig.element_size() + back.numel() * 16
    flush = torch.empty(L2_BYTES * 2 // 4, dtype=torch.float32, device=f"cuda:{dev}") \
        if working < 4 * L2_BYTES else None
    rec = _lib.TRAPANI

    def step():
        launches = 0
        if real:
            for b in range(nm):
                _lib.check(lib.mwsht_inverse_real_d(plan.handle, flm[b].data_ptr(),
                                                    sig[b].data_ptr(), rec, sp), "inv")
                launches += plan.last_launches()[0]
                _lib.check(lib.mwsht_forward_real_d(plan.handle, sig[b].data_ptr(),
                                                    back[b].data_ptr(), rec, sp), "fwd")
                launches += plan.last_launches()[0]
        else:
            _lib.check(lib.mwsht_inverse_z_batch(plan.handle, nm, flm.data_ptr(), sig.data_ptr(),
                                                 spin, rec, sp), "inv")
            launches += plan.last_launches()[0]
            _lib.check(lib.mwsht_forward_z_batch(plan.handle, nm, sig.data_ptr(), back.data_ptr(),
                                                 spin, rec, sp), "fwd")
            launches += plan.last_launches()[0]
        return launches

    def core_times():
        c = _lib.ctypes.c_float()
        s = _lib.ctypes.c_float()
        lib.mwsht_plan_last_timing(plan.handle, 1, _lib.ctypes.byref(c), _lib.ctypes.byref(s))
        inv_core = c.value
        lib.mwsht_plan_last_timing(plan.handle, 0, _lib.ctypes.byref(c), _lib.ctypes.byref(s))
        return inv_core, c.value, s.value

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    err = float((back - flm).abs().max().item())

    barrier(ws)
    torch.cuda.synchronize()
    clocks = ClockSampler(dev) if want_clocks else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    launches = 0
    inv_core = fwd_core = fwd_stage = 0.0
    step_ms = []
    for k in range(steps):
        if flush is not None:
            flush.zero_()
        e0[k].record(stream)
        launches += step()
        e1[k].record(stream)
    torch.cuda.synchronize()
    for k in range(steps):
        step_ms.append(e0[k].elapsed_time(e1[k]))
    clk = clocks.stop() if clocks else None
    # per-kernel attribution pass (not part of `value`)
    _lib.check(lib.mwsht_plan_set_timing(plan.handle, 1), "set_timing")
    for k in range(steps):
        if flush is not None:
            flush.zero_()
        step()
        torch.cuda.synchronize()
        if not real or nm == 1:
            a, b, c = core_times()
            inv_core += a
            fwd_core += b
            fwd_stage += c
    _lib.check(lib.mwsht_plan_set_timing(plan.handle, 0), "set_timing")
    total_ms = float(np.sum(step_ms))
    total_ms = max_over_ranks(total_ms, ws)

    out = dict(total_ms=total_ms, steps=steps, maps_per_rank=nm, launches=launches // steps,
               inv_core_ms=inv_core / steps, fwd_core_ms=fwd_core / steps,
               fwd_stages_ms=fwd_stage / steps, roundtrip_err=err, clocks=clk,
               l2="inputs larger than L2" if flush is None else "L2 flushed between steps")
    out["plan_bytes"] = plan.device_bytes()

    if want_e2e:
        # Public API with pinned host buffers: every step copies its coefficients
        # H2D and its result D2H inside the timed region.  HostPipeline (the
        # package's host-streaming API) double-buffers the maps so the copies of
        # neighbouring maps/steps run on the copy engines while one computes.
        from paper_1110_6298_b200.pipeline import HostPipeline
        h_in = torch.from_numpy(host).pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()
        pipe = HostPipeline(L, spin, kind="roundtrip", real=real, device=dev, depth=2)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def e2e_step():
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
        for k in range(steps):
            e2e_step()
        pipe.join()
        ev1.record(stream)
        ev1.synchronize()
        ms = [ev0.elapsed_time(ev1)]
        e2e_ms = max_over_ranks(float(np.sum(ms)), ws)
        out["e2e_total_ms"] = e2e_ms
        out["h2d"] = host.nbytes
        out["d2h"] = host.nbytes
        out["e2e_err"] = float(np.max(np.abs(h_out.numpy() - host)))
    return out


def run_gpu_mcolumn(wl, steps, warmup, rank, ws, local):
    """C5 over ws GPUs: one map, m-column sharded.  A step is
    inverse (core + theta synthesis of own orders, all-to-all, phi synthesis of
    own rings) then forward (phi DFT of own rings, all-to-all, theta stage + core
    of own orders, all-reduce of the coefficients)."""
    import torch
    from paper_1110_6298_b200.shard import MColumnSharding
    torch.cuda.set_device(local)
    L, spin = wl["L"], wl["spin"]
    host, _ = make_inputs(wl, rank, ws, torch, local)
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
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        out = step()
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
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
    return dict(total_ms=total, steps=steps, maps_per_rank=1, launches=8, inv_core_ms=0.0,
                fwd_core_ms=0.0, fwd_stages_ms=0.0, roundtrip_err=err, clocks=clk,
                l2="inputs larger than L2", plan_bytes=sh.plan.device_bytes(),
                e2e_total_ms=e2e_total, h2d=host.nbytes, d2h=host.nbytes,
                e2e_err=float(np.max(np.abs(h_out.numpy() - host[0]))),
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
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
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


def summarize(key, wl, r, ws, peak_tf, steps, warmup, with_cpu, cpu_budget):
    L, spin, real = wl["L"], wl["spin"], wl["real"]
    maps_total = (wl["maps"] if wl["shard"] == "maps" else
                  (1 if (wl["shard"] == "mcolumn" and ws > 1) else ws))
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
    traffic = traffic_table().get(f"{key}:{dom}")
    line = {
        "metric": "MW fwd+inv SHT transforms/sec at L=1024 & 4096; % of FP64/HBM roofline",
        "value": value,
        "unit": "fwd+inv pairs/s",
        "n_gpus": ws,
        "steps": steps,
        "warmup": warmup,
        "ms_per_step": r["total_ms"] / steps,
        "higher_is_better": True,
        "scaling": "strong" if wl["shard"] in ("maps", "mcolumn") else "weak",
        "vs_baseline": None,
        "dtype": "f64 (complex128)",
        "data": "synthetic: seeded N(0,1) coefficients (PCG64), BASELINE.json configs",
        "config": {"workload": wl["name"], "L": L, "spin": spin, "real": real,
                   "maps_per_rank": nm, "maps_total": maps_total,
                   "parallelism": (f"maps sharded over {ws} ranks" if wl["shard"] == "maps" else
                                   (f"one map, m-column sharded over {ws} ranks (orders "
                                    f"{r.get('splits')}), NCCL all-to-all transposes"
                                    if (wl["shard"] == "mcolumn" and ws > 1) else
                                    f"{ws} independent replicas (one map per rank)")),
                   "l2": r["l2"], "recursion": "trapani (drop-in default; same GPU recursion "
                                               "as risbo)"},
        "roofline": {"bound": "fp64", "kernel": dom, "achieved": ach, "peak": peak_tf,
                     "unit": "TFLOP/s", "frac": (ach / peak_tf) if (ach and peak_tf) else None,
                     "traffic": traffic,
                     "work_per_launch_flop": w * nm,
                     "peak_source": "DFMA probe in bench.py (mwsht_fp64_probe); "
                                    "MEASURED_PEAKS.json has no FP64 entry",
                     "kernels": {
                         "forward_core": {"ms": r["fwd_core_ms"], "tflops": fwd_tf},
                         "inverse_core": {"ms": r["inv_core_ms"], "tflops": inv_tf},
                         "forward_fft_stages": {
                             "ms": r["fwd_stages_ms"],
                             "gbs": stage_bytes(L, real) * nm / (r["fwd_stages_ms"] / 1e3) / 1e9
                             if r["fwd_stages_ms"] > 0 else None,
                             "hbm_peak_gbs": measured_peaks().get("hbm_gbs")},
                     }},
        "gpu_launches": r["launches"] * steps,
        "roundtrip_max_abs_err": r["roundtrip_err"],
        "clocks": r["clocks"],
    }
    if "e2e_total_ms" in r:
        line["e2e"] = {"value": pairs / (r["e2e_total_ms"] / 1e3), "unit": "fwd+inv pairs/s",
                       "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"],
                       "path": "paper_1110_6298_b200.pipeline.HostPipeline (public API; "
                               "inverse/forward or the *_real pair per map), pinned host buffers", "max_abs_err": r["e2e_err"]}
    if with_cpu:
        v, sample, cores = cpu_reference(wl, budget_s=cpu_budget)
        line["cpu_baseline"] = {"value": v, "unit": "fwd+inv pairs/s", "cores": cores,
                                "kind": "port", "sample": sample}
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5s0", choices=sorted(WORKLOADS))
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=25.0)
    args = ap.parse_args()
    ws, rank, local = dist_env()
    wl = WORKLOADS[args.workload]

    if args.impl == "reference":
        if rank != 0:
            return
        vals, sample, cores = [], None, None
        for _ in range(args.warmup if wl["L"] <= 256 else 0):
            cpu_reference(wl, budget_s=args.cpu_budget)
        for _ in range(args.steps):
            v, sample, cores = cpu_reference(wl, budget_s=args.cpu_budget)
            vals.append(v)
        value = float(np.mean(vals))
        print(json.dumps({
            "impl": "reference", "metric": "MW fwd+inv SHT transforms/sec at L=1024 & 4096; "
                                           "% of FP64/HBM roofline",
            "value": value, "unit": "fwd+inv pairs/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong" if wl["shard"] in ("maps", "mcolumn") else "weak",
            "vs_baseline": None, "dtype": "f64 (complex128)",
            "data": "synthetic: seeded N(0,1) coefficients (PCG64), BASELINE.json configs",
            "config": {"workload": wl["name"], "L": wl["L"], "spin": wl["spin"],
                       "real": wl["real"]},
            "cpu_baseline": {"value": value, "unit": "fwd+inv pairs/s", "cores": cores,
                             "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "fwd+inv pairs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }), flush=True)
        return

    import torch
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    peak = fp64_peak(local)
    if wl["shard"] == "mcolumn" and ws > 1:
        r = run_gpu_mcolumn(wl, args.steps, args.warmup, rank, ws, local)
    else:
        r = run_gpu(wl, args.steps, args.warmup, rank, ws, local)
    line = summarize(args.workload, wl, r, ws, peak, args.steps, args.warmup,
                     with_cpu=(rank == 0 and ws == 1), cpu_budget=args.cpu_budget)
    line["fp64_peak_tflops_measured"] = peak
    if not args.no_extra and args.workload == "c5s0" and ws == 1:
        extra = {}
        for key in ("c3", "c5s2", "c4"):
            wk = WORKLOADS[key]
            rr = run_gpu(wk, max(3, args.steps // 2), args.warmup, rank, ws, local,
                         want_e2e=True, want_clocks=False)
            sub = summarize(key, wk, rr, ws, peak, max(3, args.steps // 2), args.warmup,
                            with_cpu=(rank == 0 and ws == 1 and key == "c3"), cpu_budget=15)
            extra[key] = {k: sub[k] for k in ("value", "unit", "ms_per_step", "config", "roofline",
                                              "e2e", "roundtrip_max_abs_err", "gpu_launches")
                          if k in sub}
            if "cpu_baseline" in sub:
                extra[key]["cpu_baseline"] = sub["cpu_baseline"]
        line["workloads"] = extra
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
