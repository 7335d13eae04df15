"""Summarise an `ncu --page raw --csv` export: per kernel launch, duration, issue activity,
pipe utilisation (FP64, ALU, FMA, fmaheavy, LSU), DRAM bytes and the top warp-stall reasons.

Usage: python tools/ncu_summary.py RAW.csv [--top 6]
"""
import argparse
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("--top", type=int, default=6)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.raw)))
    h = rows[0]
    for r in rows[2:]:
        d = {h[i]: r[i] for i in range(len(h))}

        def f(k):
            try:
                return float(d.get(k, "nan").replace(",", ""))
            except ValueError:
                return float("nan")
        print("==", d["Kernel Name"][:70])
        print("   dur_us %.1f  issue %.1f%%  fp64 %.1f%%  alu %.1f%%  fma %.1f%%  fmaheavy(elapsed) %.1f%%  lsu %.1f%%  dram %.0f MB  occ %.1f%%" % (
            f("gpu__time_duration.sum") / 1e3, f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            f("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            f("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            f("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            f("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
            (f("dram__bytes_read.sum") + f("dram__bytes_write.sum")) / 1e6,
            f("sm__warps_active.avg.pct_of_peak_sustained_active")))
        st = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): f(k)
              for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
        top = sorted(st.items(), key=lambda kv: -kv[1])[: a.top]
        print("   stalls/issue: " + ", ".join("%s %.2f" % kv for kv in top))


if __name__ == "__main__":
    main()
