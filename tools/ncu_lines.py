"""Aggregate an ncu report's SASS metrics by CUDA source line:
  python tools/ncu_lines.py rep.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows[:6]) if "Address" in r)
h = rows[hi]
ei, st = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
src = {}
agg = collections.defaultdict(lambda: [0, 0])
cur = None
for r in rows[hi + 1:]:
    if len(r) < 4:
        continue
    if r[0].strip():
        cur = r[0].strip()
        src.setdefault(cur, r[1][:100])
    try:
        e, s = int(r[ei]), int(r[st])
    except ValueError:
        continue
    agg[cur][0] += e
    agg[cur][1] += s
tot = sum(v[0] for v in agg.values()) or 1
tots = sum(v[1] for v in agg.values()) or 1
print(f"{tot / 1e6:.1f} M warp-instr")
for ln, (e, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ln:>5} {100 * e / tot:5.1f}% instr {100 * s / tots:5.1f}% stall  {src.get(ln, '').strip()}")
