"""Copy an evidence run's artefacts (tools/gpu_final.sh TAG) from gpurun_out/
into profiles/ under the round-2 names.  usage: python tools/refresh_profiles.py TAG"""
import json
import shutil
import sys

tag = sys.argv[1]
g = "gpurun_out"
d = json.load(open(f"{g}/ncu_traffic_{tag}.json"))
pk = d["per_kernel"]
if pk.get("gmax0_kernel", 0) > 1e6:  # the capture's first iteration ran iteration 0's step
    d["K5"] = pk["advance_kernel"]
    d["note"] = ("steady-state families; the capture's gmax0_kernel launch was iteration 0's "
                 "(real work, absent from steady iterations) and is not counted in K5")
json.dump(d, open("profiles/ncu_traffic.json", "w"), indent=1)
lines = []
for f in ["", "_ref", "_c1", "_c2", "_c4", "_b4", "_sh1"]:
    ln = open(f"{g}/bench_{tag}{f}.log").read().strip().splitlines()[-1]
    json.loads(ln)
    lines.append(ln)
open("profiles/round2_bench.jsonl", "w").write("\n".join(lines) + "\n")
shutil.copy(f"{g}/launches_{tag}.csv", "profiles/round2_launches.csv")
shutil.copy(f"{g}/launch_summary_{tag}.txt", "profiles/round2_launch_summary.txt")
shutil.copy(f"{g}/ncu_summary_{tag}.txt", "profiles/round2_ncu_summary.txt")
shutil.copy(f"{g}/next_{tag}.jsonl", "profiles/round2_next_rows.jsonl")
print("profiles refreshed from", tag)
