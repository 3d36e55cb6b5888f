"""Hot SASS lines of one kernel in an ncu report: stall samples per
instruction, the stall-reason columns summed, and the executed-instruction
mix. Usage: python tools/ncu_sass_hot.py report.ncu-rep kernel_regex [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if r and r[0].startswith("0x")]
stall_cols = [c for c in h if c.startswith("stall_")]
tot = collections.Counter()
for d in data:
    for c in stall_cols:
        try:
            tot[c] += float(d[c] or 0)
        except ValueError:
            pass
S = sum(float(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print(f"total samples {S:.0f}; stall reasons:", ", ".join(f"{k[6:]} {100*v/S:.1f}%" for k, v in tot.most_common(10)))
ex = sum(float(d["Instructions Executed"] or 0) for d in data)
print(f"warp instructions executed {ex:.3g}")
for i, d in enumerate(data):
    d["_i"] = i
hot = sorted(data, key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))[:top]
for d in sorted(hot, key=lambda d: d["_i"]):
    st = {c[6:]: float(d[c] or 0) for c in stall_cols if float(d[c] or 0) > 0}
    top2 = sorted(st.items(), key=lambda kv: -kv[1])[:2]
    print(f"{d['_i']:5d} {float(d['Warp Stall Sampling (All Samples)'] or 0):7.0f} "
          f"{float(d['Instructions Executed'] or 0):9.3g}  {d['Source'].strip()[:60]:60s} {top2}")
