"""Top CUDA source lines of one kernel by executed warp instructions, from
`ncu -i rep --page source --print-source cuda --csv` output (file on argv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r]
h = rows[hi[0]]
ix = {n: i for i, n in enumerate(h)}
data = [r for r in rows[hi[0] + 1:] if len(r) == len(h)]
I, S = ix["Instructions Executed"], ix["Warp Stall Sampling (All Samples)"]
num = lambda v: int(v) if v.isdigit() else 0
tot = sum(num(r[I]) for r in data)
tots = sum(num(r[S]) for r in data)
print("warp instructions", tot, "stall samples", tots)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for r in sorted(data, key=lambda r: -num(r[I]))[:n]:
    print(f"{r[0]:>6} {num(r[I]):>10} {100 * num(r[I]) / max(tot, 1):5.1f}%  stall {100 * num(r[S]) / max(tots, 1):5.1f}%  "
          f"{r[ix['Source']].strip()[:105]}")
