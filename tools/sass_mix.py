"""Instruction mix of one kernel from an ncu report's SASS source page.
usage: python tools/sass_mix.py REP.ncu-rep KERNEL_REGEX"""
import collections
import csv
import io
import subprocess
import signal
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k",
                      "regex:" + sys.argv[2], "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
hdr = rows[h]
si, ii, ss = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
mix, stall = collections.Counter(), collections.Counter()
tot = 0
for r in rows[h + 1:]:
    if len(r) <= ii or not r[ii].isdigit():
        continue
    toks = r[si].split()
    op = (toks[1] if toks and toks[0].startswith("@") else toks[0]) if toks else "?"
    op = op.split(".")[0]
    n = int(r[ii])
    mix[op] += n
    stall[op] += int(r[ss] or 0)
    tot += n
st = sum(stall.values()) or 1
print(f"total warp instructions {tot}")
for op, n in mix.most_common(30):
    print(f"  {op:10s} {n:12d} {n / tot:6.1%}  stall-samples {stall[op] / st:6.1%}")
