"""Per-CUDA-line executed warp instructions and stall samples of one kernel:
joins the SASS rows of `ncu -i rep --page source --csv` (argv[1]) with the
line markers of `nvdisasm -g -c <cubin>` (argv[2]) for the function whose
mangled name contains argv[3], by instruction order.  argv[4]: rows shown."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r][0]
h = rows[hi]
ix = {n: i for i, n in enumerate(h)}
sass = [r for r in rows[hi + 1:] if len(r) == len(h)]
# line markers per instruction, in order
lines, cur, inside, inl = [], None, False, None
for ln in open(sys.argv[2]):
    if ln.startswith(".text."):
        inside = sys.argv[3] in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*inlined at "([^"]+)", line (\d+))?', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
        lines.append(cur)
if len(lines) != len(sass):
    print(f"warning: {len(lines)} disassembled vs {len(sass)} profiled instructions", file=sys.stderr)
num = lambda v: int(v) if v.isdigit() else 0
agg = {}
for (loc, r) in zip(lines, sass):
    a = agg.setdefault(loc, [0, 0])
    a[0] += num(r[ix["Instructions Executed"]])
    a[1] += num(r[ix["Warp Stall Sampling (All Samples)"]])
ti = sum(a[0] for a in agg.values())
ts = sum(a[1] for a in agg.values())
print("warp instructions", ti, "stall samples", ts)
src = {}
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
for loc, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    f, l = loc if loc else ("?", 0)
    if f not in src:
        try:
            src[f] = open(f"paper_1805_11007_b200/csrc/{f}").read().split("\n")
        except OSError:
            src[f] = []
    text = src[f][l - 1].strip()[:80] if 0 < l <= len(src[f]) else ""
    print(f"{f}:{l:<5} {a[0]:>10} {100 * a[0] / max(ti, 1):5.1f}%  stall {100 * a[1] / max(ts, 1):5.1f}%  {text}")
