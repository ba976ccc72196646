"""Generate tests/golden/cli_*/: the reference's own command line run on two
small ensembles, its output directories committed as fixtures.

Run in the build container (the reference is importable there, not on the
GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_cli.py

* ``cli_counts``: the reference test's FAST_RUN (pkg/tests/test_cli.py:12-18),
  field-free -- the device ensemble reproduces it bit for bit, so the CSVs
  must be byte-identical.
* ``cli_fig1``: fig1 (gaussian deposit, 52^2 neumann field, soft forces) cut
  to a few steps -- compared numerically (the device trajectories track the
  reference's within 1e-10).

``manifest.json`` keeps only the deterministic keys (wall clock and
timestamp dropped).
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

RUNS = {
    "cli_counts": "experiment = counts\nt_final = 0.005\nsamples = 2\nseed_base = 11\n",
    "cli_fig1": "experiment = fig1\nt_final = 1e-4\nsamples = 2\nseed_base = 3\n",
}


def main():
    from chemosim.cli import main as ref_main
    for name, text in RUNS.items():
        out = os.path.join(HERE, name)
        os.makedirs(out, exist_ok=True)
        cfg = os.path.join(out, "run.cfg")
        with open(cfg, "w") as fh:
            fh.write(text)
        assert ref_main(["--config", cfg, "--output-dir", out]) == 0
        mpath = os.path.join(out, "manifest.json")
        with open(mpath) as fh:
            manifest = json.load(fh)
        for key in ("wall_clock_seconds", "created"):
            manifest.pop(key)
        with open(mpath, "w") as fh:
            json.dump(manifest, fh, indent=2, sort_keys=True)
            fh.write("\n")
        print(name, sorted(os.listdir(out)))


if __name__ == "__main__":
    sys.exit(main())
