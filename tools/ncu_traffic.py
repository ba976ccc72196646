"""Per-launch DRAM traffic of the force+update kernels from an ncu --set full
capture -> profiles/ncu_traffic_<config>.json (read by bench.py)."""
import csv
import json
import subprocess
import sys

TIME = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
        "s": 1.0, "second": 1.0}
KERNELS = {"k_fast_forces<": "forces", "k_fast_forces_generic": "forces_generic",
           "k_fast_update": "update", "k_scan": "scan",
           "k_bucket_sort": "bucket_sort", "k_fast_deposit_rows": "deposit_rows",
           "k_spec_cols": "spec_cols"}
# kernels of the bench's roofline stage (bin + force + update); the row
# deposit and the spectral pass are reported but belong to other stages
FU = ("forces", "forces_generic", "update", "scan", "bucket_sort")


def main(rep, out, config):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = rows[0]
    res = {"config": config, "source": rep, "kernels": {}}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "")
        for k, tag in KERNELS.items():
            if k in name:
                unit_r = rows[1][hdr.index("dram__bytes_read.sum")]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rd = float(d["dram__bytes_read.sum"]) * scale[rows[1][hdr.index("dram__bytes_read.sum")]]
                wr = float(d["dram__bytes_write.sum"]) * scale[rows[1][hdr.index("dram__bytes_write.sum")]]
                dur = float(d["gpu__time_duration.sum"]) * TIME[rows[1][hdr.index("gpu__time_duration.sum")]]
                res["kernels"][tag] = {"dram_read_bytes": rd, "dram_write_bytes": wr,
                                       "duration_s": dur, "name": name[:80]}
    res["fu_bytes_per_step"] = sum(v["dram_read_bytes"] + v["dram_write_bytes"]
                                   for k, v in res["kernels"].items() if k in FU)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
