"""Render the Table 1 readings study (tools/table1_study.py JSON lines) against the paper.

For every (post, penalty, solver) combination and both level readings (A5: row L = 2^L
cells per direction; SPEC: 2^{L+1}), prints the grid ours / paper, the mean |nu - paper|,
the number of cells within +-0.5, and the level trend: the mean over degrees of
nu(L_max) - nu(L=3) for ours and for the paper (the paper's counts fall with L).

  python tools/render_table1_study.py profiles/tables/r02_study.jsonl > profiles/r02_table1_study.md
"""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TABLE1 = {}
for line in open(os.path.join(ROOT, "tests", "golden", "table1_full_kernel.txt")):
    line = line.split("#", 1)[0].split()
    if line:
        for j, v in enumerate(line[1:]):
            if v != "---":
                TABLE1[(int(line[0]), 3 + j)] = float(v)


def main(path):
    runs = collections.defaultdict(dict)
    for line in open(path):
        r = json.loads(line)
        runs[(r["post"], r["pen"], r["solver"], r["vcycle"])][(r["L"], r["k"])] = r["nu"]
    summary = []
    for key in sorted(runs):
        grid = runs[key]
        for shift, name in ((0, "A5 (2^L cells)"), (1, "SPEC (2^{L+1} cells)")):
            cells = {(L, k): grid[(L + shift, k)] for (L, k) in TABLE1 if (L + shift, k) in grid}
            if not cells:
                continue
            d = [abs(v - TABLE1[c]) for c, v in cells.items()]
            within = sum(x <= 0.5 for x in d)
            trend_o, trend_p = [], []
            for k in range(3, 8):
                Ls = sorted(L for (L, kk) in cells if kk == k and L >= 3)
                if len(Ls) >= 2:
                    trend_o.append(cells[(Ls[-1], k)] - cells[(Ls[0], k)])
                    trend_p.append(TABLE1[(Ls[-1], k)] - TABLE1[(Ls[0], k)])
            summary.append((sum(d) / len(d), key, name, within, len(d),
                            sum(trend_o) / max(len(trend_o), 1), sum(trend_p) / max(len(trend_p), 1)))
            print("#### post %s, penalty %s, %s GMRES/CG, %s V-cycle, level reading %s\n" % (key + (name,)))
            print("| L | " + " | ".join("Q%d" % k for k in range(3, 8)) + " |")
            print("|---" * 6 + "|")
            for L in range(2, 8):
                row = []
                for k in range(3, 8):
                    c = (L, k)
                    row.append("%.2f / %.1f" % (cells[c], TABLE1[c]) if c in cells else "")
                if any(row):
                    print("| %d | %s |" % (L, " | ".join(row)))
            print("\nmean |nu - paper| = %.2f, within 0.5: %d/%d, level trend L=3..max (ours / paper): %+.2f / %+.2f\n"
                  % (summary[-1][0], within, len(d), summary[-1][5], summary[-1][6]))
    print("### Summary (sorted by mean |nu - paper|)\n")
    print("| post | penalty (interior x boundary) | solver | V-cycle | level reading | mean abs dev | within 0.5 "
          "| trend ours | trend paper |")
    print("|---|---|---|---|---|---|---|---|---|")
    for m, key, name, w, n, to, tp in sorted(summary):
        print("| %s | %s | %s | %s | %s | %.2f | %d/%d | %+.2f | %+.2f |" % (key + (name, m, w, n, to, tp)))


if __name__ == "__main__":
    main(sys.argv[1])
