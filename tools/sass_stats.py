"""Static evidence for the hot kernels (profiles/<round>/): ptxas -v register / spill report
of the N = 2^14 instantiation unit and the pointwise kernels, and SASS opcode histograms
(cuobjdump -sass of the built libedl.so) -- counts of IMAD.WIDE / DFMA / LDG / LDS / STL /
UBLKCP / UTMALDG ... per kernel.

Usage: python tools/sass_stats.py profiles/round2"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2110_13638_b200", "csrc")
LIB = os.path.join(ROOT, "paper_2110_13638_b200", "libedl.so")
HOT = ["k_relin_modup", "k_rescale_ntt", "k_relin_moddown_ntt", "k_relin_moddown_intt", "k_relin_intt_d2",
       "k_rescale_intt", "k_relin_mac3", "k_cc_mac4", "k_cc_mac2", "k_dense_mac3", "k_relin_ks", "k_ntt_limbs"]


def demangle(sym):
    d = subprocess.run(["c++filt"], input=sym, capture_output=True, text=True).stdout.strip()
    d = re.sub(r"\(anonymous namespace\)::", "", d.split("(")[0].replace("void ", "").replace("edl::", ""))
    return d


def ptxas(out_dir):
    lines = []
    for src in ("ntt_inst_14.cu", "pointwise.cu"):
        r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                            "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "--expt-relaxed-constexpr", "-Xptxas", "-v",
                            "-c", os.path.join(CSRC, src), "-o", "/tmp/_sass_stats.o"], capture_output=True, text=True)
        cur, spill = None, (0, 0)
        for ln in r.stderr.splitlines():
            m = re.search(r"Compiling entry function '(\S+)'", ln)
            if m:
                cur, spill = demangle(m.group(1)), (0, 0)
            m2 = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
            if m2 and cur:
                spill = (int(m2.group(1)), int(m2.group(2)))
            m3 = re.search(r"Used (\d+) registers", ln)
            if m3 and cur and any(h in cur for h in HOT):
                lines.append("%-84s regs %3s  spill st/ld %4d/%4d B" % (cur[:84], m3.group(1), *spill))
    with open(os.path.join(out_dir, "ptxas_v_hot.txt"), "w") as f:
        f.write("ptxas -v, sm_100a (ntt_inst_14.cu: the N = 2^14 kernels; pointwise.cu)\n")
        f.write("\n".join(lines) + "\n")
    return lines


def sass(out_dir):
    dump = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    hist = {}
    cur, cnt = None, None
    for ln in dump.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            if cur and cnt is not None:
                hist[cur] = cnt
            name = demangle(m.group(1))
            keep = any(h in name for h in HOT) and ("NttCfg<14" in name or
                                                     any(h in name for h in ("k_relin_mac3", "k_cc_mac4", "k_cc_mac2", "k_dense_mac3")))
            cur = name if keep else None
            cnt = collections.Counter() if keep else None
            continue
        if cnt is not None:
            m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*(\.[A-Z0-9_]+)*)", ln)
            if m:
                op = m.group(2)
                base = op.split(".")[0]
                cnt[op if base in ("IMAD", "SYNCS", "LDG", "STG", "LDS", "STS") else base] += 1
    if cur and cnt is not None:
        hist[cur] = cnt
    out = {k: dict(v.most_common(40)) for k, v in hist.items()}
    json.dump(out, open(os.path.join(out_dir, "sass_opcode_hist.json"), "w"), indent=1)
    return out


if __name__ == "__main__":
    od = sys.argv[1]
    os.makedirs(od, exist_ok=True)
    for ln in ptxas(od):
        print(ln)
    h = sass(od)
    rows = []
    for k, v in h.items():
        tma = sum(n for op, n in v.items() if op.startswith(("UBLKCP", "UTMALDG", "UTMASTG")))
        rows.append("%-72s IMAD.WIDE %4d  DFMA %4d  STL %3d  LDL %3d  bulk/TMA %d" % (
            k[:72], sum(n for op, n in v.items() if op.startswith("IMAD.WIDE")), v.get("DFMA", 0), v.get("STL", 0),
            v.get("LDL", 0), tma))
    with open(os.path.join(od, "sass_summary.txt"), "w") as f:
        f.write("\n".join(rows) + "\n")
    print("\n".join(rows))
