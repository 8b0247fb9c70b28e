"""Turn gpurun_out/{launches,prof,bench}_<tag>.* into committed summaries under profiles/."""
import csv, io, json, subprocess, sys
from collections import defaultdict
from pathlib import Path

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
root = Path(__file__).resolve().parents[1]
out, prof = root / "gpurun_out", root / "profiles"
prof.mkdir(exist_ok=True)

# 1. launch list -> per-kernel shares
rows = list(csv.reader(io.StringIO((out / f"launches_{tag}.csv").read_text().split("\n", 0)[0])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
per = defaultdict(lambda: [0, 0.0])
for r in rows[hdr_i + 1:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].split("<")[0]
    unit = d["Metric Unit"]
    v = float(d["Metric Value"].replace(",", ""))
    v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[unit]  # -> us
    per[name][0] += 1
    per[name][1] += v
tot = sum(v[1] for v in per.values())
lines = [f"# launch list of `python bench.py --steps 20 --warmup 5 --no-cpu --no-o1280` under ncu "
         f"(--metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)",
         "kernel,launches,total_us,mean_us,share_of_gpu_time"]
for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"{k},{n},{t:.1f},{t / n:.2f},{t / tot:.3f}")
(prof / f"launches_{tag}_summary.csv").write_text("\n".join(lines) + "\n")
(prof / f"launches_{tag}.csv").write_text((out / f"launches_{tag}.csv").read_text())

# 2. full captures -> key metrics: the persistent loop kernel (10 steps per launch) and a
# single flushed step
def capture(rep, title):
    summ = subprocess.run([sys.executable, str(root / "tools" / "ncu_summary.py"), str(rep)],
                          capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    vals, units = dict(zip(rr[0], rr[2])), dict(zip(rr[0], rr[1]))

    def mb(k):
        v = float(vals[k].replace(",", ""))
        return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[units[k]]

    dur = float(vals["gpu__time_duration.sum"].replace(",", ""))
    dur *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(units["gpu__time_duration.sum"], 1.0)
    return title + "\n" + summ, mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum"), dur


text, rd, wr, dur = capture(out / f"prof_{tag}.ncu-rep",
                            "# ncu --set full --clock-control none --import-source on -k regex:mpdata_dyn: ONE "
                            "persistent launch of 10 steps at 279x256x80 (tools/prof_loop.py 10); per step = / 10")
(prof / f"ncu_loop_{tag}.txt").write_text(text)
steps = 10
traffic = {"tag": tag, "dram_read_MB_per_step": rd / steps, "dram_write_MB_per_step": wr / steps,
           "dram_bytes_per_step": int((rd + wr) * 1e6 / steps),
           "algorithmic_bytes_per_step": 319408128, "algorithmic_read_bytes_per_step": 273696768,
           "duration_us_per_step": dur / steps,
           "source": f"profiles/ncu_loop_{tag}.txt (one launch of {steps} steps / {steps})"}
sp = out / f"prof_step_{tag}.ncu-rep"
if sp.exists():
    text, rd1, wr1, dur1 = capture(sp, "# ncu --set full --clock-control none --import-source on -k regex:mpdata_dyn: "
                                       "one flushed single step at 279x256x80 (tools/prof_fused.py 0 4)")
    (prof / f"ncu_step_{tag}.txt").write_text(text)
    traffic["single_step"] = {"dram_read_MB": rd1, "dram_write_MB": wr1, "duration_us": dur1,
                              "source": f"profiles/ncu_step_{tag}.txt"}
(prof / "fused_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
b = out / f"bench_{tag}.json"
if b.exists():
    (prof / f"bench_{tag}.json").write_text(b.read_text().strip().splitlines()[-1] + "\n")
print(json.dumps(traffic, indent=1))
print("\n".join(lines[:8]))
