"""Render the C3 sweep and the configs runs (tools/sweep_c3.py, tools/configs.py
jsonl output) as the markdown tables kept under profiles/.

  python tools/render_tables.py c3.jsonl configs.jsonl > profiles/rNN_tables.md
"""
import json
import sys


def c3(path):
    rows = [json.loads(l) for l in open(path) if l.strip()]
    out = ["### C3 sweep (BASELINE.json configs[2]): 3D SIPG k=1..7, ~130M dofs, one B200", "",
           "`python tools/sweep_c3.py` (CUDA events, 3 warm-up + 10 timed calls, vectors > L2). Roofline: algorithmic "
           "bytes (vmult 2s, smoother step 2^d*3s per dof) vs MEASURED_PEAKS hbm_gbs; flops (vmult 14(k+1)+48, "
           "smoother `bench.smoother_flops_per_dof`) vs the CUDA-core peaks measured live (ipmg_alu_peak: FFMA2 for fp32, DFMA for fp64).", "",
           "| k | cells | dofs | vmult fp64 GDoF/s (bound, frac) | vmult fp32 | smoother step fp64 | smoother step fp32 "
           "| mixed GMG-CG solve ms (its) |", "|---|---|---|---|---|---|---|---|"]
    for r in rows:
        def c(key):
            d = r[key]
            return "%.1f (%s %.2f)" % (d["gdofs"], d["roofline"]["bound"], d["roofline"]["frac"])
        out.append("| %d | %s | %d | %s | %s | %s | %s | %.1f (%d) |" % (
            r["k"], "x".join(str(v) for v in r["cells"]), r["ndofs"], c("vmult_fp64"), c("vmult_fp32"),
            c("smooth_fp64"), c("smooth_fp32"), r["solve_mixed"]["ms"], r["solve_mixed"]["iterations"]))
    return "\n".join(out)


def configs(path):
    rows = [json.loads(l) for l in open(path) if l.strip()]
    out = ["### BASELINE.json configs on one B200 (`python tools/configs.py`)", "",
           "f == 1, x0 = 0, CG to ||r|| <= 1e-8 ||b|| (PAPER.md:331); CUDA-event time of complete solves after a "
           "warm-up solve (setup excluded).", "",
           "| config | smoother | V-cycle | levels | dofs | time to solution (ms) | GDoF/s | CG its | nu |",
           "|---|---|---|---|---|---|---|---|---|"]
    tput = []
    for r in rows:
        if r["config"] == "T":
            tput.append(r)
            continue
        out.append("| %s | %s | %s | %d | %d | %.2f | %.3f | %d | %.2f |" % (
            r["config"], r.get("smoother", "multiplicative"), r.get("vcycle", "fp32" if r["config"] != "C1" else "fp64"),
            r["levels"], r["dofs"], r["ms"], r["gdofs"], r["iterations"], r["nu"]))
    if tput:
        out += ["", "### Throughput vs problem size (NEXT-4), 3D k = 4", "",
                "| levels | dofs | operator vmult fp64 GDoF/s | smoother step fp32 GDoF/s |", "|---|---|---|---|"]
        for r in tput:
            out.append("| %d | %d | %.1f | %.1f |" % (r["levels"], r["dofs"], r["vmult_fp64_gdofs"], r["smooth_fp32_gdofs"]))
    return "\n".join(out)


if __name__ == "__main__":
    print(c3(sys.argv[1]))
    print()
    print(configs(sys.argv[2]))
