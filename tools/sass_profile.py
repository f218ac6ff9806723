"""Per-opcode / per-region breakdown of an ncu source page (SASS view):
  ncu -i rep --page source --csv --print-source=sass -k regex:K --launch-skip S --launch-count 1 > x.csv
  python tools/sass_profile.py x.csv [--regions]"""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    out = []
    hdr = None
    for r in rows:
        if len(r) > 5 and r[0] == "Address":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or len(r) < len(hdr) - 5:
            continue
        try:
            n = int(r[hdr["Instructions Executed"]] or 0)
        except ValueError:
            continue
        src = r[hdr["Source"]].strip()
        toks = src.split()
        op = "?"
        if toks:
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        out.append(dict(addr=r[0], src=src, op=op.split(".")[0], n=n,
                        s=int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0),
                        e=int(r[hdr["L1 Wavefronts Shared Excessive"]] or 0)))
    return out


def main():
    d = load(sys.argv[1])
    tot = sum(x["n"] for x in d) or 1
    tots = sum(x["s"] for x in d) or 1
    inst, samp, exc = defaultdict(int), defaultdict(int), defaultdict(int)
    for x in d:
        inst[x["op"]] += x["n"]
        samp[x["op"]] += x["s"]
        exc[x["op"]] += x["e"]
    print("total warp-inst %d, stall samples %d" % (tot, tots))
    for op in sorted(inst, key=lambda o: -inst[o])[:22]:
        print("%-8s inst %5.1f%%  samples %5.1f%%  excess-wavefronts %d" % (op, 100 * inst[op] / tot,
                                                                          100 * samp[op] / tots, exc[op]))
    if "--regions" in sys.argv:
        # split at BAR instructions
        reg, cur = [], dict(n=0, s=0, e=0, start=d[0]["addr"] if d else "")
        for x in d:
            cur["n"] += x["n"]; cur["s"] += x["s"]; cur["e"] += x["e"]
            if x["op"] == "BAR":
                cur["end"] = x["addr"]; reg.append(cur); cur = dict(n=0, s=0, e=0, start=x["addr"])
        cur["end"] = "end"; reg.append(cur)
        for i, r in enumerate(reg):
            print("region %2d %s..%s inst %5.1f%% samples %5.1f%% excess %d" % (i, r["start"][-5:], r["end"][-5:],
                  100 * r["n"] / tot, 100 * r["s"] / tots, r["e"]))


if __name__ == "__main__":
    main()
