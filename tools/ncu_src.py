"""Summarise an ncu source page (SASS) per kernel: stall samples by reason, by opcode,
and the hottest instructions.  Usage: python tools/ncu_src.py rep.ncu-rep <kernel regex> [top]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    body = []
    for r in rows:
        if len(r) > 5 and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            body.append(r)
    # ncu repeats the whole table for some captures (same rows twice): count each row once
    seen, uniq = set(), []
    for r in body:
        k = tuple(r)
        if k not in seen:
            seen.add(k)
            uniq.append(r)
    body = uniq
    if not hdr:
        print("no source page"); return
    H = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    by_op = collections.Counter()
    by_op_reason = collections.defaultdict(collections.Counter)
    insts = []
    for r in body:
        src = r[H["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        n = int(r[H["Warp Stall Sampling (All Samples)"]] or 0)
        by_op[op] += n
        for c in stall_cols:
            v = int(r[H[c]] or 0)
            tot[c] += v
            by_op_reason[op][c] += v
        insts.append((n, r[H["Address"]], src, {c: int(r[H[c]] or 0) for c in stall_cols}))
    total = sum(tot.values())
    print(f"total samples {total}")
    print("by reason:", ", ".join(f"{k[6:]} {v / total:.1%}" for k, v in tot.most_common(10)))
    print("by opcode:")
    for op, n in by_op.most_common(15):
        rs = by_op_reason[op].most_common(3)
        print(f"  {op:10s} {n / total:6.1%}   " + ", ".join(f"{k[6:]} {v / total:.1%}" for k, v in rs))
    ex = collections.Counter()
    for r in body:
        src = r[H["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        try:
            ex[op] += int(r[H["Instructions Executed"]] or 0)
        except (KeyError, ValueError):
            pass
    te = sum(ex.values())
    if te:
        print("executed warp-instructions %d; by opcode:" % te)
        print("  " + ", ".join("%s %.1f%%" % (k, 100.0 * v / te) for k, v in ex.most_common(22)))
    print("hottest instructions:")
    for n, a, src, st in sorted(insts, key=lambda x: -x[0])[:top]:
        rs = sorted(st.items(), key=lambda kv: -kv[1])[:2]
        print(f"  {n / total:5.1%} {a[-5:]} {src[:60]:60s} " + ", ".join(f"{k[6:]} {v}" for k, v in rs))


if __name__ == "__main__":
    main()
