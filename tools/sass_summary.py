"""Per-kernel SASS instruction counts of libtsg.so (TMA / mbarrier / memory / fp64 mnemonics).

    python tools/sass_summary.py [paper_1908_06094_b200/libtsg.so] > profiles/sass_<round>.txt

The evidence that the hot kernels are TMA-fed (UTMALDG, SYNCS.* mbarrier waits) and use no
tensor-core or legacy mma instructions (fp64 stencil, bandwidth-bound)."""
import collections
import re
import subprocess
import sys

so = sys.argv[1] if len(sys.argv) > 1 else "paper_1908_06094_b200/libtsg.so"
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
demangle = lambda s: subprocess.run(["c++filt"], input=s, capture_output=True, text=True).stdout.strip()  # noqa: E731
KEYS = ["UTMALDG", "UTMASTG", "UTMACCTL", "UBLKCP", "SYNCS.ARRIVE", "SYNCS.PHASECHK", "LDS", "STS", "LDG", "STG",
        "DADD", "DMUL", "DFMA", "DSETP", "MUFU", "HMMA", "UTCHMMA", "BAR.SYNC", "MEMBAR", "ATOMG", "NANOSLEEP"]
funcs = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m and cur:
        op = m.group(1)
        funcs[cur]["_total"] += 1
        for k in KEYS:
            if op == k or op.startswith(k + ".") or (k.endswith(".") and op.startswith(k)) or op.startswith(k) and k in ("SYNCS.ARRIVE", "SYNCS.PHASECHK", "MEMBAR", "BAR.SYNC"):
                funcs[cur][k] += 1
                break
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else re.compile(r"mpdata_fused_kernel|reduce_tma_kernel")
print(f"# SASS instruction counts per kernel ({so}, cuobjdump -sass); kernels matching {pat.pattern!r}")
print("# columns: total " + " ".join(KEYS))
tot = collections.Counter()
n = 0
for name, c in funcs.items():
    dn = demangle(name)
    if not pat.search(dn):
        continue
    n += 1
    tot.update(c)
    print(f"{dn}\n    total={c['_total']} " + " ".join(f"{k}={c[k]}" for k in KEYS if c[k]))
print(f"# {n} matching instantiations; summed: total={tot['_total']} " + " ".join(f"{k}={tot[k]}" for k in KEYS if tot[k]))
print(f"# all {len(funcs)} kernels in the library: HMMA={sum(c['HMMA'] for c in funcs.values())} "
      f"UTCHMMA={sum(c['UTCHMMA'] for c in funcs.values())} (no tensor-core instructions: fp64, bandwidth-bound)")
