"""Hot SASS instructions of one kernel from an ncu --set full report, with
their dominant stall reasons.

    python tools/sass_stalls.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, kern, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    si, st, ie = (hdr.index(k) for k in ("Source", "Warp Stall Sampling (All Samples)",
                                          "Instructions Executed"))
    reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    data = []
    for r in rows[2:]:
        if len(r) != len(hdr) or not r[ie].isdigit():
            if data:
                break
            continue
        data.append(r)
    tot_s = sum(int(r[st]) for r in data)
    tot_i = sum(int(r[ie]) for r in data)
    agg = {hdr[i]: sum(int(r[i]) for r in data) for i in reasons}
    print(f"{len(data)} SASS lines, {tot_i} warp instructions, {tot_s} stall samples")
    print("kernel stall mix:", ", ".join(f"{k[6:]} {100 * v / tot_s:.0f}%"
                                         for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    for idx, r in sorted(enumerate(data), key=lambda x: -int(x[1][st]))[:top]:
        rs = sorted(((int(r[i]), hdr[i][6:]) for i in reasons), reverse=True)[:2]
        print(f"{idx:5d} {r[st]:>6} {r[ie]:>9}  {r[si].strip()[:60]:60s} "
              + " ".join(f"{n}:{v}" for v, n in rs if v))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
