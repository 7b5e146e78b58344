"""Group an ncu report's SASS lines into runs of equal execution count:
python tools/sass_groups.py rep.ncu-rep [min_sum_M]  (loop bodies and branch paths stand out)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 5.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ei, si, ti = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Avg. Threads Executed")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ei]), float(r[ti]), r[si].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print(f"{len(data)} lines, {tot / 1e6:.1f} M warp-instr")
prev, start, acc, thr_acc = None, 0, 0, 0.0
for i, (e, t, s) in enumerate(data + [(-1, 0, "")]):
    key = round(e / 1e5)
    if key != prev:
        if prev is not None and acc > thr * 1e6:
            print(f"{start:5d}-{i - 1:5d} n={i - start:3d} exec={prev / 10:6.2f}M thr={thr_acc / (i - start):4.1f} "
                  f"sum={acc / 1e6:7.1f}M")
        prev, start, acc, thr_acc = key, i, 0, 0.0
    acc += max(e, 0)
    thr_acc += t
