"""Summarise an ncu report: headline metrics, instruction mix and top stall lines."""
import csv, io, subprocess, sys
from collections import Counter

rep = sys.argv[1]
def page(name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))

det = page("details")
hdr = det[0]
want = {"Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Executed Instructions",
        "Registers Per Thread", "Achieved Occupancy", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction", "SM Frequency"}
for r in det[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']:>14s} {d['Metric Unit']}")
raw = page("raw")
rh = raw[0]
vals = dict(zip(rh, raw[2])) if len(raw) > 2 else {}
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "gpu__time_duration.sum"):
    if k in vals:
        print(f"{k:40s} {vals[k]:>14s} {raw[1][rh.index(k)]}")
src = page("source", ("--print-source", "sass"))
if len(src) > 2:
    h = src[1]
    data = [dict(zip(h, r)) for r in src[2:] if len(r) == len(h)]
    tot = sum(int(d["Instructions Executed"]) for d in data)
    op = Counter()
    for d in data:
        ins = d["Source"].strip()
        name = (ins.split()[1] if ins.startswith("@") else ins.split()[0]).split(".")[0]
        op[name] += int(d["Instructions Executed"])
    print("total warp instructions", tot)
    print("mix:", ", ".join(f"{k} {v/tot*100:.1f}%" for k, v in op.most_common(16)))
    data.sort(key=lambda d: -int(d["Warp Stall Sampling (All Samples)"]))
    print("top stall instructions:")
    for d in data[:12]:
        print("  ", d["Warp Stall Sampling (All Samples)"].rjust(6), d["Instructions Executed"].rjust(9), d["Source"].strip()[:80])
