"""Per-family DRAM traffic per launch (dram__bytes_read.sum + write.sum) from an
ncu --set full capture of one GP iteration -> profiles/ncu_traffic.json, which
bench.py reports as roofline.traffic.  usage: python tools/ncu_traffic.py REP.ncu-rep [config]"""
import csv
import io
import json
import os
import subprocess
import sys

FAMILY = [("fused_net", "K1"), ("generic_net", "K1"), ("fused_gather", "K1"), ("gather_warp", "K1"),
          ("tile_", "K2"), ("scatter", "K2"), ("spec_", "K3"), ("dens_kernel", "K4"),
          ("gmax0", "K5"), ("advance", "K5")]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
# a kernel captured more than once (the window straddles two iterations)
# counts once, at its mean
fam, kern, seen, famof = {}, {}, {}, {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    b = sum(float(d[m]) * scale[u[m]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    name = d["Kernel Name"]
    f = next((f for k, f in FAMILY if k in name), None)
    if f is None:
        continue
    short = name.split("(")[0].split("::")[-1]
    kern[short] = kern.get(short, 0) + b
    seen[short] = seen.get(short, 0) + 1
    famof[short] = f
kern = {k: v / seen[k] for k, v in kern.items()}
for k, v in kern.items():
    fam[famof[k]] = fam.get(famof[k], 0) + v
res = {k: int(v) for k, v in fam.items()}
res["per_kernel"] = {k: int(v) for k, v in kern.items()}
res["source"] = os.path.basename(sys.argv[1])
res["config"] = int(sys.argv[2]) if len(sys.argv) > 2 else 3  # bench --config of the capture
dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                   "ncu_traffic.json")
with open(dst, "w") as fh:
    json.dump(res, fh, indent=1)
print(json.dumps(res, indent=1))
