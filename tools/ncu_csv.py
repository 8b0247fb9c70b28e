"""Print an `ncu --csv --metrics ...` log as one line per launch: python tools/ncu_csv.py FILE"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, out = None, {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        out.setdefault(x["ID"], [x["Kernel Name"][:60], {}])[1][x["Metric Name"]] = x["Metric Value"]
for k, (name, m) in out.items():
    print(k, name, " ".join(f"{a.split('__')[1] if '__' in a else a}={v}" for a, v in m.items()))
