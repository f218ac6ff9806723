"""Per-phase stall reasons of one kernel launch from an ncu source page export
(ncu -i REP --page source --csv --print-source sass > X.csv): the SASS in address
order cut at every BAR.SYNC; for each phase the executed warp instructions per unit,
its share of the stall samples and its top stall reasons (share of the phase's samples).

  python tools/stall_phases.py X.csv [units]
"""
import csv
import re
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r)
    hdr = rows[hi]
    iS, iI, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    rs = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    segs, cur, seen = [], None, set()
    tot = defaultdict(int)
    for r in rows[hi + 1:]:
        if len(r) <= iI or not r[iI].isdigit():
            continue
        if r[0] in seen:
            break
        seen.add(r[0])
        if cur is None:
            cur = {"start": r[0][-5:], "inst": 0, "stall": 0, "why": defaultdict(int), "ops": defaultdict(int)}
        src = r[iS].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0].split(".")[0] if src else "?"
        cur["inst"] += int(r[iI])
        cur["ops"][op] += int(r[iI])
        cur["stall"] += int(r[iW] or 0)
        for i, h in rs:
            v = int(r[i] or 0)
            cur["why"][h[6:]] += v
            tot[h[6:]] += v
        if op == "BAR":
            segs.append(cur)
            cur = None
    if cur:
        segs.append(cur)
    S = sum(g["stall"] for g in segs)
    print("| phase | warp inst/unit | stall share | top stall reasons (share of phase) | top opcodes |")
    print("|---|---|---|---|---|")
    for g in segs:
        if g["inst"] == 0:
            continue
        w = sorted(g["why"].items(), key=lambda kv: -kv[1])[:5]
        gs = max(1, sum(g["why"].values()))
        ops = sorted(g["ops"].items(), key=lambda kv: -kv[1])[:6]
        print("| %s | %.1f | %.1f%% | %s | %s |" % (g["start"], g["inst"] / units, 100.0 * g["stall"] / max(S, 1),
              ", ".join("%s %.0f%%" % (k, 100.0 * v / gs) for k, v in w),
              ", ".join("%s %.0f" % (k, v / units) for k, v in ops)))
    T = max(1, sum(tot.values()))
    print("\nwhole launch: " + ", ".join("%s %.1f%%" % (k, 100.0 * v / T)
                                          for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]))


if __name__ == "__main__":
    main()
