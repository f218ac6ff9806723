"""Summarise ncu reports into a small JSON/markdown table (run here, no GPU).

  python profiles/ncu_summary.py gpurun_out/prof_smooth_r01.ncu-rep [...] > profiles/xxx.md
  python profiles/ncu_summary.py --launches gpurun_out/launches_r01.csv

Per kernel launch: duration, dram bytes (read+write), achieved DRAM %, issue
slots, registers, occupancy, FP32/FP64 pipe utilisation, shared-memory bank
conflicts (excess wavefronts) -- the evidence DESIGN.md cites.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

WANT = [
    ("Duration", "gpu__time_duration.sum"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("SM busy %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("Issue active %", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("Registers", "launch__registers_per_thread"),
    ("Occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("FMA pipe %", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("FP64 pipe %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("Inst executed", "smsp__inst_executed.sum"),
    ("FFMA thread-inst", "sm__sass_thread_inst_executed_op_ffma_pred_on.sum"),
    ("DFMA thread-inst", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum"),
    ("smem ld bank conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
    ("smem st bank conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"),
    ("L2 hit %", "lts__t_sector_hit_rate.pct"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], stdout=subprocess.PIPE,
                         stderr=subprocess.DEVNULL, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        res.append((d, u))
    return res


def summarise(rep):
    lines = ["### %s" % rep, "", "| launch | kernel | " + " | ".join(w[0] for w in WANT) + " |",
             "|---" * (len(WANT) + 2) + "|"]
    for i, (d, u) in enumerate(raw(rep)):
        name = d.get("Kernel Name", "?")[:48]
        vals = []
        for label, m in WANT:
            v = d.get(m, "n/a")
            unit = u.get(m, "")
            vals.append("%s %s" % (v, unit) if v != "n/a" else "n/a")
        lines.append("| %d | %s | %s |" % (i, name, " | ".join(vals)))
    return "\n".join(lines) + "\n"


# flops per predicated-on thread instruction of the SASS opcodes that do floating-point work
FLOPS = {"FFMA": 2, "FFMA2": 4, "FADD": 1, "FADD2": 2, "FMUL": 1, "FMUL2": 2, "DFMA": 2, "DADD": 1, "DMUL": 1,
         "HFMA2": 0}


def sass_mix(rep, launch=0):
    """Per-opcode warp instructions and achieved flops of one launch, from the SASS source
    page (ncu -i --page source --print-source sass): counters 'Instructions Executed' and
    'Predicated-On Thread Instructions Executed' per SASS instruction."""
    import re
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(launch), "--launch-count", "1"], stdout=subprocess.PIPE,
                         stderr=subprocess.DEVNULL, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r)
    hdr = rows[hi]
    iS, iI = hdr.index("Source"), hdr.index("Instructions Executed")
    iP = hdr.index("Predicated-On Thread Instructions Executed")
    ops, flops, seen = defaultdict(int), defaultdict(float), set()
    for r in rows[hi + 1:]:
        if len(r) <= iP or not r[iI].strip().isdigit():
            continue
        if r[0] in seen:      # the page can list a function twice
            continue
        seen.add(r[0])
        src = r[iS].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0].split(".")[0] if src else "?"
        ops[op] += int(r[iI])
        flops[op] += FLOPS.get(op, 0) * int(r[iP] or 0)
    return ops, flops


def summarise_mix(rep, launch=0, top=16):
    ops, flops = sass_mix(rep, launch)
    tot = sum(ops.values())
    fl = sum(flops.values())
    lines = ["#### SASS mix of launch %d of %s (ncu source page)" % (launch, rep), "",
             "warp instructions %d; floating-point work %.4g flop (FFMA/DFMA 2, FFMA2 4, FADD/FMUL 1, "
             "packed x2 2 per thread instruction)" % (tot, fl), "",
             "| opcode | warp inst | share | flop |", "|---|---|---|---|"]
    for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:top]:
        lines.append("| %s | %d | %.1f%% | %.4g |" % (k, v, 100.0 * v / tot, flops.get(k, 0)))
    return "\n".join(lines) + "\n", tot, fl


def phases(rep, launch=0, units=1.0, top=8):
    """Per-phase warp instructions of one launch: the SASS (ncu source page, in address
    order) cut at every BAR.SYNC; counts are divided by `units` (e.g. the patches of the
    launch).  Columns: executed warp instructions, stall samples, excess shared-memory
    wavefronts (bank conflicts), L1 global tag requests, top opcodes."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(launch), "--launch-count", "1"], stdout=subprocess.PIPE,
                         stderr=subprocess.DEVNULL, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r)
    hdr = rows[hi]
    iS, iI = hdr.index("Source"), hdr.index("Instructions Executed")
    iW = hdr.index("Warp Stall Sampling (All Samples)")
    iX = hdr.index("L1 Wavefronts Shared Excessive")
    iL = hdr.index("L1 Tag Requests Global")
    segs, cur, seen = [], None, set()
    import re
    for r in rows[hi + 1:]:
        if len(r) <= iI or not r[iI].isdigit():
            continue
        if r[0] in seen:   # the page may list a launch twice
            break
        seen.add(r[0])
        if cur is None:
            cur = {"start": r[0][-5:], "inst": 0, "stall": 0, "exc": 0, "tag": 0, "ops": defaultdict(int)}
        src = r[iS].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0].split(".")[0] if src else "?"
        n = int(r[iI])
        cur["inst"] += n
        cur["stall"] += int(r[iW] or 0)
        cur["exc"] += int(r[iX] or 0)
        cur["tag"] += int(r[iL] or 0)
        cur["ops"][op] += n
        if op == "BAR":
            segs.append(cur)
            cur = None
    if cur:
        segs.append(cur)
    lines = ["#### Phases of launch %d of %s (per unit, unit = 1/%g of the launch)" % (launch, rep, units), "",
             "| phase start | warp inst | stall samples | smem excess wavefronts | L1 global tags | top opcodes |",
             "|---|---|---|---|---|---|"]
    for g in segs:
        if g["inst"] == 0:
            continue
        topo = ", ".join("%s %.0f" % (k, v / units) for k, v in sorted(g["ops"].items(), key=lambda kv: -kv[1])[:top])
        lines.append("| %s | %.1f | %d | %.1f | %.1f | %s |" % (g["start"], g["inst"] / units, g["stall"],
                                                             g["exc"] / units, g["tag"] / units, topo))
    lines.append("| **total** | %.1f | | | | |" % (sum(g["inst"] for g in segs) / units))
    return "\n".join(lines) + "\n"


def launches(path):
    """Per-kernel share of the device time in an ncu --metrics gpu__time_duration.sum CSV."""
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r.get("Metric Unit", "us"), 1.0)
        tot[name] += v * scale
        cnt[name] += 1
    T = sum(tot.values())
    out = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append("| %s | %d | %.1f | %.1f%% |" % (k, cnt[k], v, 100 * v / T))
    out.append("| **total** | %d | %.1f | 100%% |" % (sum(cnt.values()), T))
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        for p in sys.argv[2:]:
            print("### %s\n" % p)
            print(launches(p))
    elif sys.argv[1] == "--phases":   # --phases REP LAUNCH UNITS
        print(phases(sys.argv[2], int(sys.argv[3]), float(sys.argv[4])))
    elif sys.argv[1] == "--mix":
        for p in sys.argv[2:]:
            print(summarise_mix(p)[0])
    else:
        for p in sys.argv[1:]:
            print(summarise(p))
