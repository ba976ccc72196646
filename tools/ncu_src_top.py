"""Top SASS lines of one kernel by warp-stall samples, from
`ncu -i rep --page source --csv -k <kernel>` output (file given on argv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) != len(hdr) or not r[ix["Instructions Executed"]].isdigit():
        if data:
            break  # next kernel's block
        continue
    data.append(r)
tot_s = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
tot_i = sum(int(r[ix["Instructions Executed"]] or 0) for r in data)
print(f"samples {tot_s}  warp-instructions {tot_i}")
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
top = sorted(data, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for k, r in enumerate(data):
    pass
for r in top[:n]:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    st = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
    pos = data.index(r)
    print(f"{pos:5d} {s:6d} {100*s/max(tot_s,1):5.1f}% {int(r[ix['Instructions Executed']] or 0):10d} "
          f"{r[ix['Source']].strip()[:60]:60s} {st}")
