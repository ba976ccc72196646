"""Build the sm_100a CUDA library in-tree.

    python -m paper_1805_11007_b200.build

compiles csrc/*.cu with nvcc for ``-gencode arch=compute_100a,code=sm_100a``
(``-lineinfo`` for ncu source correlation) into
``paper_1805_11007_b200/_build/libchemo_b200.so``.  The .so is git-ignored but
travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_build")
SO = os.path.join(OUT_DIR, "libchemo_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(HERE, "..", "include", "*.h")))


def up_to_date() -> bool:
    if not os.path.exists(SO):
        return False
    t = os.path.getmtime(SO)
    return all(os.path.getmtime(f) <= t for f in sources() + headers())


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          extra: list[str] | None = None) -> str:
    """``out``/``extra``: an alternative output path and extra nvcc flags
    (tuning experiments, e.g. ``-DCS_SCATTER_U=8``; load one with CS_LIB)."""
    so = out or SO
    if not force and out is None and up_to_date():
        return SO
    os.makedirs(OUT_DIR, exist_ok=True)
    obj_dir = OUT_DIR if out is None else so + ".objs"
    os.makedirs(obj_dir, exist_ok=True)
    objs = []
    nv = nvcc()
    cuda_lib = os.path.join(os.path.dirname(os.path.dirname(nv)), "lib64")
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
              *ARCH, "--expt-relaxed-constexpr", "-I", os.path.join(HERE, "..", "include"),
              *(extra or [])]
    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
        hdr_t = max(os.path.getmtime(f) for f in headers())
        if (not force and os.path.exists(obj) and out is None
                and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t)):
            return obj, None
        r = subprocess.run([nv, "-c", src, "-o", obj, *common], capture_output=True, text=True)
        if r.returncode != 0:
            return None, r.stdout + r.stderr
        return obj, (r.stderr if verbose else None)

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as pool:
        results = list(pool.map(compile_one, sources()))
    for src, (obj, msg) in zip(sources(), results):
        if obj is None:
            sys.stderr.write(msg)
            raise RuntimeError(f"nvcc failed on {src}")
        if msg:
            sys.stderr.write(msg)
        objs.append(obj)
    tmp = so + ".tmp"
    cmd = [nv, "-shared", *ARCH, "-o", tmp, *objs, "-L", cuda_lib, "-lcufft",
           "-Xlinker", f"-rpath={cuda_lib}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, so)
    return so


if __name__ == "__main__":
    args = sys.argv[1:]
    out = None
    if "--out" in args:
        out = os.path.abspath(args[args.index("--out") + 1])
    extra = [a for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose="-v" in args, out=out, extra=extra))
