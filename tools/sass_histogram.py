"""Static SASS opcode histogram per kernel of the built library.

    python tools/sass_histogram.py [paper_1110_6298_b200/libmwsht.so] > profiles/<round>/sass_histogram.md

Runs `cuobjdump -sass` and counts opcodes (the mnemonic before the first '.')
per function, for the kernels on the hot path.  Evidence of the instruction
choice: DFMA/DMUL/DADD for the FP64 work, UBLKCP (TMA bulk copies) and SYNCS
(mbarriers) in the cores' producer/consumer ring, USETMAXREG (warpgroup
register hand-off), and no tensor-core MMA (the contraction is a matvec).
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1110_6298_b200/libmwsht.so"
KEEP = ("k_forward_core", "k_inverse_core", "k_theta_fwd", "k_theta_inv", "k_phi_fwd",
        "k_phi_inv", "k_inv_prescale", "k_reality", "k_flm_unpack", "k_gl_fm", "k_gl_flm")
SHOW = ("DFMA", "DMUL", "DADD", "FFMA", "HMMA", "UTCHMMA", "UTCQMMA", "UTCMMA", "DMMA", "UBLKCP",
        "UTMALDG", "SYNCS", "USETMAXREG", "LDS", "STS", "LDG", "STG", "LDL", "STL", "SHFL",
        "BAR", "LDTM", "STTM")

txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = collections.OrderedDict()
cur = None
for line in txt.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs.setdefault(cur, collections.Counter())
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and cur:
        funcs[cur][m.group(2)] += 1


def short(name):
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    return re.sub(r"\(.*", "", d.replace("mwsht::", "").replace("fft::", ""))


rows = []
for f, c in funcs.items():
    s = short(f)
    if not any(k in s for k in KEEP):
        continue
    if "k_theta" in s or "k_phi" in s:
        if not re.search(r"<false, 1[23], false>", s):  # large-L complex instances
            continue
    rows.append((s, c))

print(f"# Static SASS opcode counts per kernel (`cuobjdump -sass {LIB}`)\n")
print("Instruction counts in the kernel body (static, not executed). Large-L complex")
print("instances of the FFT stage kernels only (H = 4096, 8192).\n")
print("| kernel | total | " + " | ".join(SHOW) + " |")
print("|---|---|" + "---|" * len(SHOW))
for s, c in rows:
    print(f"| `{s}` | {sum(c.values())} | " + " | ".join(str(c.get(k, 0)) for k in SHOW) + " |")
