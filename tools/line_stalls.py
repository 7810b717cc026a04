"""Aggregate warp-stall samples and executed instructions per CUDA source line
from an ncu report (mixed cuda,sass source page).
usage: python tools/line_stalls.py REP.ncu-rep KERNEL_REGEX [top]"""
import collections
import csv
import io
import signal
import subprocess
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k",
                      "regex:" + sys.argv[2], "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
fname, cur = "?", None
samp, inst, src = collections.Counter(), collections.Counter(), {}
reasons = collections.defaultdict(collections.Counter)
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0].strip():  # a CUDA line row
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()[:70]
    if cur is None or not r[3].strip():
        continue
    try:
        s = int(r[4] or 0)
        n = int(r[7] or 0)
    except ValueError:
        continue
    samp[cur] += s
    inst[cur] += n
    for k, v in zip(hdr, r):
        if k.startswith("stall_") and "Not Issued" not in k and v not in ("", "0"):
            try:
                reasons[cur][k[6:]] += int(v)
            except ValueError:
                pass
tot = sum(samp.values()) or 1
itot = sum(inst.values()) or 1
print(f"samples {tot}, instructions {itot}")
for k, v in samp.most_common(top):
    rs = ", ".join(f"{a}:{b / v:.0%}" for a, b in reasons[k].most_common(3))
    print(f"{v / tot:6.1%} {inst[k] / itot:6.1%}  {k[0]}:{k[1]:<5d} {src.get(k, '')[:60]:60s} [{rs}]")
