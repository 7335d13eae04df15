"""Summarise DRAM traffic per launch from an `ncu --page raw --csv` export into
profiles/<round>/ncu_traffic.json (bench.py's roofline.traffic source).

Usage: python tools/ncu_traffic.py <raw.csv> <out.json>
"""
import csv
import json
import sys
from collections import defaultdict


def main(src, dst):
    rows = list(csv.reader(open(src)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    k = hdr.index("Kernel Name")
    rd, wr, dur = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum"), hdr.index("gpu__time_duration.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tscale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    agg = defaultdict(lambda: {"launches": 0, "dram_read_bytes": 0.0, "dram_write_bytes": 0.0, "ncu_ms": 0.0})
    for d in data:
        name = d[k].split("(")[0].split("<")[0].replace("void ", "").replace("edl::", "").split("::")[-1].strip()
        a = agg[name]
        a["launches"] += 1
        a["dram_read_bytes"] += float(d[rd]) * scale[units[rd]]
        a["dram_write_bytes"] += float(d[wr]) * scale[units[wr]]
        a["ncu_ms"] += float(d[dur]) * tscale[units[dur]]
    out = {}
    for name, a in agg.items():
        n = a["launches"]
        out[name] = {"launches": n, "dram_bytes_per_launch": (a["dram_read_bytes"] + a["dram_write_bytes"]) / n,
                     "dram_read_bytes_per_launch": a["dram_read_bytes"] / n,
                     "dram_write_bytes_per_launch": a["dram_write_bytes"] / n, "ncu_ms_per_launch": a["ncu_ms"] / n,
                     "source": "ncu --set full --clock-control none (tools/prof_step.py: one C1 step)"}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
