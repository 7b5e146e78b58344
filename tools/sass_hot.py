"""Per-instruction hot spots from an ncu report: python tools/sass_hot.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ai, si = hdr.index("Address"), hdr.index("Source")
ei = hdr.index("Instructions Executed")
ti = hdr.index("Avg. Threads Executed")
wi = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ei]), float(r[ti]), int(r[wi]), r[si].strip()))
    except (ValueError, IndexError):
        continue
tot = sum(d[0] for d in data)
samp = sum(d[2] for d in data)
print(f"{len(data)} SASS lines, {tot / 1e6:.1f} M warp-instr executed, {samp} stall samples")
mode = sys.argv[3] if len(sys.argv) > 3 else "seq"
if mode == "seq":
    # instructions in program order with execution counts (loop bodies stand out)
    for i, (e, t, w, s) in enumerate(data):
        if e >= tot * 0.002:
            print(f"{i:5d} {e / 1e6:8.2f}M thr={t:5.1f} stall={w:6d}  {s}")
