"""Summarise the -Xptxas -v output of the in-tree build: registers, stack and
spills per kernel (paper_2405_18982_b200/_build/*.log)."""
import glob
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pat_fn = re.compile(r"Compiling entry function '(\S+)'")
pat_st = re.compile(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads")
pat_rg = re.compile(r"Used (\d+) registers")
only = sys.argv[1] if len(sys.argv) > 1 else ""
for log in sorted(glob.glob(os.path.join(ROOT, "paper_2405_18982_b200", os.environ.get("IPMG_BUILD_DIR", "_build"), "*.log"))):
    fn = None
    st = None
    for line in open(log):
        m = pat_fn.search(line)
        if m:
            fn = m.group(1)
            continue
        m = pat_st.search(line)
        if m:
            st = m.groups()
            continue
        m = pat_rg.search(line)
        if m and fn:
            short = re.sub(r"_ZN4ipmg5kdeg(\d)\d+(\w+?)ILi(\d)E([fd]).*", r"k\1 \2<\3,\4>", fn)
            short = re.sub(r"_ZN4ipmg12_GLOBAL__N_1\d+", "", short)
            if only in short:
                print("%-40s regs=%-4s stack=%-5s spill_st=%-5s spill_ld=%s" % (short[:40], m.group(1), *(st or ("?",) * 3)))
            fn = None
