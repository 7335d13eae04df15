"""Summarise an `ncu --set full` capture of ONE C1 step (tools/prof_step.py --step-only):
  * per launch: duration (ms), DRAM MB, issue-active %, FP64 / fmaheavy / ALU pipe %,
    warps active %, top stall reasons (per issue);
  * per kernel, summed over the step's launches: DRAM bytes per step and launches per step
    (bench.py's roofline.traffic source: profiles/<round>/ncu_traffic.json).
Units come from the CSV's unit row (round-1's tool printed ns as us and MB as 0).

Usage: python tools/ncu_step_summary.py rep.ncu-rep out_dir
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
         "s": 1e3, "%": 1.0, "": 1.0}


def short(name):
    return name.split("(")[0].split("<")[0].replace("void ", "").replace("edl::", "").split("::")[-1].strip()


def main(rep, out_dir):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    os.makedirs(out_dir, exist_ok=True)
    H = {h: i for i, h in enumerate(hdr)}

    def val(d, k, unit_to=None):
        if k not in H or d[H[k]] in ("", "n/a"):
            return None
        v = float(d[H[k]].replace(",", ""))
        return v * SCALE.get(units[H[k]], 1.0)

    def first(d, keys):   # the integer-multiply pipe metric's name differs between ncu versions
        for k in keys:
            v = val(d, k)
            if v is not None:
                return v
        return None

    FMA_KEYS = [k for k in ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
                            "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
                            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active") if k in H]
    with open(os.path.join(out_dir, "ncu_pipe_metric_names.txt"), "w") as f:   # what this ncu reports
        f.write("\n".join(h for h in hdr if "pipe" in h) + "\n")
    stall_keys = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    lines, agg = [], collections.OrderedDict()
    for d in data:
        name = short(d[H["Kernel Name"]])
        ms = val(d, "gpu__time_duration.sum")
        dram = (val(d, "dram__bytes_read.sum") or 0.0) + (val(d, "dram__bytes_write.sum") or 0.0)
        st = sorted(((k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                      val(d, k) or 0.0) for k in stall_keys), key=lambda kv: -kv[1])[:4]
        e = {"kernel": name, "ms": ms, "dram_MB": dram / 1e6,
             "issue_active_pct": val(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
             "fp64_pipe_pct": val(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
             "fmaheavy_pipe_pct": first(d, FMA_KEYS),
             "alu_pipe_pct": val(d, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
             "warps_active_pct": val(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
             "registers": val(d, "launch__registers_per_thread"),
             "top_stalls_per_issue": st}
        lines.append(e)
        a = agg.setdefault(name, {"launches_per_step": 0, "dram_bytes_per_step": 0.0, "ncu_ms_per_step": 0.0})
        a["launches_per_step"] += 1
        a["dram_bytes_per_step"] += dram
        a["ncu_ms_per_step"] += ms or 0.0
    for a in agg.values():
        a["source"] = "ncu --set full --clock-control none, one C1 step (tools/prof_step.py --step-only), cold/serialised"
    json.dump(agg, open(os.path.join(out_dir, "ncu_traffic.json"), "w"), indent=1)
    with open(os.path.join(out_dir, "ncu_step_summary.txt"), "w") as f:
        f.write("kernel                    ms      DRAM_MB  issue%  fp64%  fma%       alu%  warps%  regs  top stalls/issue\n")
        for e in lines:
            f.write("%-24s %7.4f %9.1f %6.1f %6.1f %9.1f %6.1f %6.1f %5.0f  %s\n" % (
                e["kernel"][:24], e["ms"] or 0, e["dram_MB"], e["issue_active_pct"] or 0, e["fp64_pipe_pct"] or 0,
                e["fmaheavy_pipe_pct"] or 0, e["alu_pipe_pct"] or 0, e["warps_active_pct"] or 0, e["registers"] or 0,
                ", ".join("%s %.2f" % kv for kv in e["top_stalls_per_issue"])))
        f.write("\nper kernel, summed over one step:\n")
        for k, a in agg.items():
            f.write("%-24s launches %2d  ncu_ms %.4f  DRAM %.1f MB\n" % (k, a["launches_per_step"], a["ncu_ms_per_step"],
                                                                        a["dram_bytes_per_step"] / 1e6))
    json.dump(lines, open(os.path.join(out_dir, "ncu_step_launches.json"), "w"), indent=1)
    print(open(os.path.join(out_dir, "ncu_step_summary.txt")).read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
