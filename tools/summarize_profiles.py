"""Summarise an ncu capture (tools/capture_profiles.sh) into profiles/<round>/.

    python tools/summarize_profiles.py gpurun_out/prof profiles/round1 [--L 4096]

Writes launches_L<L>.csv (the launch list), cores_L<L>_details.csv and
fft_L<L>_details.csv (ncu --page details), a kernel table
(kernels_L<L>.md) and updates profiles/traffic.json with the cores' DRAM bytes.
"""
import argparse
import csv
import io
import json
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
W_NZ = {4096: 1.8332e11, 2048: 2.29e10, 1024: 2.87e9}  # spin 0 complex, per direction


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    out = {}
    order = []
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        key = (d["ID"], d["Kernel Name"])
        if key not in out:
            out[key] = {}
            order.append(key)
        out[key][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return [(k[1], out[k]) for k in order]


def details(rep, kernel_regex):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv", "-k",
                          "regex:" + kernel_regex], capture_output=True, text=True).stdout
    return txt


def raw_metrics(rep, names):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "s": 1e3}
    res = []
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        d = {"kernel": r[h.index("Kernel Name")]}
        for n in names:
            if n in h:
                j = h.index(n)
                try:
                    d[n] = float(r[j].replace(",", "")) * scale.get(units[j], 1.0)
                except ValueError:
                    d[n] = r[j]
        res.append(d)
    return res


def short(name):
    s = name.replace("void ", "").replace("mwsht::", "").replace("fft::", "")
    return s.split("(")[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("dst")
    ap.add_argument("--L", type=int, default=4096)
    a = ap.parse_args()
    L = a.L
    os.makedirs(a.dst, exist_ok=True)
    lpath = os.path.join(a.src, f"launches_L{L}.csv")
    shutil.copy(lpath, os.path.join(a.dst, f"launches_L{L}.csv"))
    ls = [(n, m) for n, m in launches(lpath) if "mwsht" in n or "fft::" in n]
    total = sum(m.get("gpu__time_duration.sum", 0) for _, m in ls)
    lines = [f"# Launch list, L={L} spin 0, one inverse + one forward (ncu, cold, serialised)", "",
             "| kernel | ms | share | DRAM read GB | DRAM write GB |", "|---|---|---|---|---|"]
    for n, m in ls:
        t = m.get("gpu__time_duration.sum", 0)
        unit = 1e-6  # ns -> ms
        lines.append(f"| {short(n)} | {t * unit:.3f} | {t / total:.1%} | "
                     f"{m.get('dram__bytes_read.sum', 0) / 1e9:.2f} | "
                     f"{m.get('dram__bytes_write.sum', 0) / 1e9:.2f} |")
    lines.append(f"| total (our kernels) | {total * 1e-6:.3f} | | | |")
    names = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
             "smsp__issue_active.avg.pct_of_peak_sustained_active",
             "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
             "l1tex__throughput.avg.pct_of_peak_sustained_active",
             "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"]
    traffic = {}
    for tag in ("cores", "fft"):
        rep = os.path.join(a.src, f"{tag}_L{L}.ncu-rep")
        if not os.path.exists(rep):
            continue
        regex = "k_inverse_core|k_forward_core" if tag == "cores" else "k_theta_fwd|k_phi_inv"
        with open(os.path.join(a.dst, f"{tag}_L{L}_details.csv"), "w") as f:
            f.write(details(rep, regex))
        lines += ["", f"# ncu --set full: {tag}", "",
                  "| kernel | ms | FP64 pipe % | issue % | L1TEX % | DRAM GB | stalls/issue: wait, long_sb, math, barrier |",
                  "|---|---|---|---|---|---|---|"]
        for d in raw_metrics(rep, names):
            ms = d.get("gpu__time_duration.sum", 0)  # converted to ms
            dram = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0))
            lines.append(
                f"| {short(d['kernel'])} | {ms:.3f} | "
                f"{d.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                f"{d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                f"{d.get('l1tex__throughput.avg.pct_of_peak_sustained_active', 0):.1f} | "
                f"{dram / 1e9:.2f} | "
                f"{d.get('smsp__average_warps_issue_stalled_wait_per_issue_active.ratio', 0):.2f}, "
                f"{d.get('smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio', 0):.2f}, "
                f"{d.get('smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio', 0):.2f}, "
                f"{d.get('smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio', 0):.2f} |")
            if tag == "cores":
                k = "inverse_core" if "inverse" in d["kernel"] else "forward_core"
                traffic[f"c5s0:{k}"] = dram
    with open(os.path.join(a.dst, f"kernels_L{L}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic and L == 4096:
        traffic["_source"] = (f"{a.dst}/cores_L{L}_details.csv (ncu --set full, L={L} spin 0, one "
                              "launch each); bytes per launch = dram__bytes_read.sum + "
                              "dram__bytes_write.sum")
        with open(os.path.join(HERE, "profiles", "traffic.json"), "w") as f:
            json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
