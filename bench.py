"""Throughput of the chemotaxis hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3]
                    [--impl ours|reference] [--no-cpu-baseline]

Workload (default): BASELINE config 3 -- N = 10^7 two-type cells (50/50,
radii 6.1804e-5 / 1.2361e-4 for area fraction 0.3, D 1.0 / 0.5, chi +1.0 /
-0.5), periodic unit box, 4096^2 periodic grid (D_c 1, decay 0.1, A
secretes k 0.1, B consumes k 0.03, CIC), dt 1e-5, fp32 storage with fp64
arithmetic and fp64 force sums.  Inputs: seeded uniform positions and a
pre-generated seeded N(0,1) increment array resident in HBM (synthetic; the
per-step working set, ~0.7 GB of particle state + 0.6 GB of grids, exceeds
the 126 MB L2, so no explicit flush is needed).

A step = the whole reference per-step pipeline (deposit, implicit field
step, gradient, drift refresh, cell list, pair forces, EM update,
boundaries) for all N particles.  value = N * K / (device time of K steps,
max over ranks).  With --gpus N > 1 every rank runs an independent replica
(weak scaling; the slab-decomposed single system is SURVEY 8e, see
DESIGN.md).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-steps/sec (force+update+PDE)"
UNIT = "particle-steps/s"

CONFIGS = {
    # name: BASELINE.json configs[i] mapped per SURVEY 8d
    "cfg0": dict(n=1000, n_c=0, prec="fp64", radii=None, eps=0.005, D=(1.0, 1.0),
                 chi=(0.0, 0.0), chi_pinned=(True, True), periodic=False, field=False,
                 types="beta", bound="launch"),
    "cfg1": dict(n=10_000, n_c=128, prec="fp64", radii=None, eps=0.005, D=(1.0, 1.0),
                 chi=(0.0, 1.0), chi_pinned=(True, False), periodic=False, field=True,
                 boundary="neumann", d_c=1.0, k_alpha=0.1, k_beta=0.0, gamma=0.1,
                 secretes=(False, True), consumes=(False, False), c0="linear_x",
                 types="beta", bound="launch"),
    "cfg2": dict(n=100_000, n_c=512, prec="fp64", radii=(0.005, 0.01), D=(1.0, 0.5),
                 chi=(1.0, -0.5), chi_pinned=(False, False), periodic=True, field=True,
                 boundary="periodic", d_c=1.0, k_alpha=0.1, k_beta=0.03, gamma=0.1,
                 secretes=(True, False), consumes=(False, True), c0="zero", types="half",
                 bound="fp64"),
    "cfg3": dict(n=10_000_000, n_c=4096, prec="fp32", radii=(6.1804e-5, 1.2361e-4),
                 D=(1.0, 0.5), chi=(1.0, -0.5), chi_pinned=(False, False), periodic=True,
                 field=True, boundary="periodic", d_c=1.0, k_alpha=0.1, k_beta=0.03,
                 gamma=0.1, secretes=(True, False), consumes=(False, True), c0="zero",
                 types="half"),
    # cfg2's fp32 variant (BASELINE configs[2]: "fp64 and fp32 variants")
    "cfg2f32": dict(n=100_000, n_c=512, prec="fp32", radii=(0.005, 0.01), D=(1.0, 0.5),
                    chi=(1.0, -0.5), chi_pinned=(False, False), periodic=True, field=True,
                    boundary="periodic", d_c=1.0, k_alpha=0.1, k_beta=0.03, gamma=0.1,
                    secretes=(True, False), consumes=(False, True), c0="zero", types="half"),
    # BASELINE configs[4] at one GPU (periodic, 64 seeded gaussian
    # clusters, sigma 0.02, wrapped periodically).  Rates: cfg2's, except the
    # consumption rate, scaled so that dt * k_beta * mean(rho_beta) equals
    # cfg2's 0.015: with cfg2's k_beta the explicit consumption factor
    # dt k_beta rho_beta reaches ~100 at the cluster nodes and the field step
    # diverges (x10 per step, sign alternating), as it would in the reference
    "cfg4": dict(n=80_000_000, n_c=8192, prec="fp32", radii=(2.1851e-5, 4.3702e-5),
                 D=(1.0, 0.5), chi=(1.0, -0.5), chi_pinned=(False, False), periodic=True,
                 field=True, boundary="periodic", d_c=1.0, k_alpha=0.1, k_beta=3.75e-5,
                 gamma=0.1, secretes=(True, False), consumes=(False, True), c0="zero",
                 types="half", init="clustered"),
}
DT = 1e-5
SEED = 20241805


# --------------------------------------------------------------------------
# algorithmic bytes
# --------------------------------------------------------------------------
def algorithmic_bytes(cfg: dict) -> dict:
    n = cfg["n"]
    s = 8 if cfg["prec"] == "fp64" else 4
    sg = s
    P = 1 if cfg["periodic"] else 0
    T = 1 if cfg["types"] == "half" else 0
    G = 1 if cfg["field"] else 0
    cut = 2.0 * (cfg["radii"][1] if cfg["radii"] else cfg["eps"])
    ncell = int(1.0 / cut) ** 2
    nc2 = cfg["n_c"] ** 2
    b_fu = n * (2 * s + 2 * s + 2 * s + T * 1 + P * 4 * s) + 8 * ncell \
        + G * min(4 * n, nc2) * 2 * sg
    F = 9 if (cfg["field"] and cfg["consumes"][1]) else 7
    b_pde = G * F * nc2 * sg
    return dict(fu=b_fu, pde=b_pde, total=b_fu + b_pde, n_cells=ncell)


# --------------------------------------------------------------------------
# clocks sampler (nvml, during the timed region)
# --------------------------------------------------------------------------
_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}


class ClockSampler:
    def __init__(self, device_index: int, period: float = 0.01):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self.period = period

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                for bit, name in _REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------
# setup
# --------------------------------------------------------------------------
def initial_positions(cfg: dict, rng) -> np.ndarray:
    """Uniform in the centred unit square, or (cfg4) 64 seeded uniform centres,
    each particle picking one uniformly, offset N(0, 0.02^2), wrapped
    periodically into [-0.5, 0.5)."""
    n = cfg["n"]
    if cfg.get("init") == "clustered":
        centres = -0.5 + rng.random((64, 2))
        pos = centres[rng.integers(0, 64, n)]
        pos += 0.02 * rng.standard_normal((n, 2))
        pos = np.mod(pos + 0.5, 1.0) - 0.5
        pos[pos >= 0.5] = -0.5
        return pos
    return (-0.5 + rng.random((n, 2))).astype(np.float64)


def make_state(cfg: dict, rank: int, xi_by_slot: bool = False, engine: str = "auto",
               build_sim: bool = True):
    """(DeviceSim, state tensors, initial positions, species) of a config;
    build_sim=False returns the cs_sim_params in place of the simulation."""
    import torch
    import paper_1805_11007_b200 as cs
    n, n_c = cfg["n"], max(cfg["n_c"], 3)
    rng = np.random.default_rng(SEED + rank)
    dt_ = torch.float64 if cfg["prec"] == "fp64" else torch.float32
    pos = initial_positions(cfg, rng)
    if cfg["types"] == "half":
        sp = (np.arange(n) >= n // 2).astype(np.uint8)
    else:
        sp = np.ones(n, np.uint8)
    dom = cs.Domain.square(1.0, periodic=cfg["periodic"])
    grid = cs.Grid.square(n_c, 1.0, cfg.get("boundary", "neumann"))
    if cfg.get("c0") == "linear_x":
        c0 = grid.node_positions()[:, 0].copy()
    else:
        c0 = np.zeros(n_c * n_c)
    dev = "cuda"
    st = dict(pos=torch.as_tensor(pos, device=dev).to(dt_).contiguous(),
              anchor=torch.as_tensor(pos, device=dev).to(dt_).contiguous(),
              next_pos=None,
              species=torch.as_tensor(sp, device=dev),
              drift=torch.zeros((n, 2), dtype=torch.float64, device=dev),
              local_c=None,
              c=torch.as_tensor(c0, device=dev).to(dt_).contiguous(),
              grad=torch.zeros((n_c * n_c, 2), dtype=dt_, device=dev),
              rho_a=torch.zeros(n_c * n_c, dtype=dt_, device=dev),
              rho_b=torch.zeros(n_c * n_c, dtype=dt_, device=dev))
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        if cfg["radii"]:
            mp = cs.MotionParams(d_alpha=cfg["D"][0], d_beta=cfg["D"][1], epsilon=cfg["radii"][0],
                                 cutoff=2 * cfg["radii"][0], dt=DT, radius_alpha=cfg["radii"][0],
                                 radius_beta=cfg["radii"][1])
        else:
            mp = cs.MotionParams(d_alpha=cfg["D"][0], d_beta=cfg["D"][1], epsilon=cfg["eps"],
                                 cutoff=2.0 * cfg["eps"], dt=DT)
    fp = cs.FieldParams(d_c=cfg.get("d_c", 0.0), k_alpha=cfg.get("k_alpha", 0.0),
                        k_beta=cfg.get("k_beta", 0.0), gamma=cfg.get("gamma", 0.0))
    if os.environ.get("CS_BENCH_NO_INTERACTION"):  # diagnostics only
        mp.interaction = "none"
    params = cs.sim_params_struct(
        n=n, prec=0 if cfg["prec"] == "fp64" else 1, domain=dom, motion=mp, dt=DT,
        field_active=cfg["field"], refresh_active=cfg["field"] or cfg.get("c0") == "linear_x",
        grid=grid, fparams=fp, kernel=cs.Kernel(kind="cic"),
        secretes=cfg.get("secretes", (False, False)), consumes=cfg.get("consumes", (False, False)),
        chi=cfg["chi"], chi_pinned=cfg["chi_pinned"], store_samples=False, store_next=False,
        xi_by_slot=xi_by_slot, engine=engine)
    if cfg["field"] or cfg.get("c0") == "linear_x":
        f = cs.Field(c=st["c"], grad=st["grad"], rho_alpha=st["rho_a"], rho_beta=st["rho_b"])
        cs.gradient(f, cs.build_operators(grid, fp, DT))
    if not build_sim:
        return params, st, pos, sp
    sim = cs.DeviceSim(params, st)
    return sim, st, pos, sp


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config_name: str):
    """Per-step DRAM bytes of the F+U kernels from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", f"ncu_traffic_{config_name}.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return None


# --------------------------------------------------------------------------
# CPU baseline / reference arm: the oracle port on host cores
# --------------------------------------------------------------------------
def oracle_sim(cfg: dict, pos, sp, nthreads: int):
    import oracle
    from oracle.sim import OracleSim
    n_c = max(cfg["n_c"], 3)
    if cfg["radii"]:
        e, c, cell = oracle.pair_table(radii=cfg["radii"])
    else:
        e, c, cell = oracle.pair_table(epsilon=cfg["eps"], cutoff=2.0 * cfg["eps"])
    field = None
    if cfg["field"]:
        per = cfg["boundary"] == "periodic"
        if cfg.get("c0") == "linear_x":
            xs = -0.5 + (1.0 / (n_c - 1)) * np.arange(n_c)
            c0 = np.tile(xs, n_c)
        else:
            c0 = np.zeros(n_c * n_c)
        field = dict(n_c=n_c, boundary=cfg["boundary"], d_c=cfg["d_c"], k_alpha=cfg["k_alpha"],
                     k_beta=cfg["k_beta"], gamma=cfg["gamma"], kernel="cic",
                     secretes=cfg["secretes"], consumes=cfg["consumes"], c0=c0,
                     splu_max=256 if per else 0)
    return OracleSim(pos, sp, lo=[-0.5] * 2, hi=[0.5] * 2,
                     periodic=(cfg["periodic"],) * 2, dt=DT, diffusion=cfg["D"], eps_tab=e,
                     cut_tab=c, cell_cutoff=cell, chi=cfg["chi"], chi_pinned=cfg["chi_pinned"],
                     field=field, fp32=cfg["prec"] == "fp32", nthreads=nthreads)


def config_dict(name: str, cfg: dict, world: int) -> dict:
    """The workload description both arms print (same keys and values)."""
    return {"workload": f"{name}: N={cfg['n']}, {cfg['n_c']}^2 "
                        f"{cfg.get('boundary', '-')} grid, {cfg['prec']} storage",
            "parallelism": "single" if world == 1 else f"replicas{world}",
            "l2": "per-step working set > 126 MB L2 (no flush needed)"
            if cfg["n"] >= 1_000_000 else
            "working set L2-resident (launch/latency-bound config; absolute numbers)"}


def reference_numba(name: str):
    """The reference's own functions timed on one core (tools/time_reference.py,
    build container: the reference does not travel to the GPU box)."""
    path = os.path.join(ROOT, "profiles", "r02", f"reference_numba_{name}.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return {k: d[k] for k in ("value_1core", "value_replicas", "unit", "cpu_model", "cores",
                                  "stage_s_per_step", "pde", "note") if k in d}
    except Exception:
        return None


def roofline_entry(name, cfg, fu_gbs, peak, peak_src, traffic, ab, t_fu, stages):
    """The F+U stage against the roof that bounds it: HBM for the binary32
    configs (cfg2f32, cfg3, cfg4); the FP64 pipe for cfg2 (binary64 pair
    terms: FLOPs per step counted by ncu, profiles/r02/fp64_<cfg>.json, over
    the measured DFMA peak); cfg0 / cfg1 are launch/latency-bound (L2-resident
    working sets of <= 2 MB): their HBM fraction is shown for completeness."""
    bound = cfg.get("bound", "hbm")
    e = {"bound": bound, "kernel": "force+update stage (bin, forces, update)",
         "achieved": fu_gbs, "peak": peak, "unit": "GB/s",
         "frac": (fu_gbs / peak) if fu_gbs else None,
         "traffic": traffic.get("fu_bytes_per_step") if traffic else None,
         "algorithmic_bytes_per_step": ab["fu"], "t_ms": t_fu, "peak_source": peak_src}
    if bound == "launch":
        e["note"] = ("launch/latency-bound: the per-step working set is L2-resident; "
                     "ms_per_step is the number that matters, the HBM fraction is not a roof")
    if bound == "fp64":
        try:
            with open(os.path.join(ROOT, "profiles", "r02", f"fp64_{name}.json")) as fh:
                f = json.load(fh)
            t = stages["force"]
            ach = f["force_fp64_flop_per_step"] / (t / 1e3) / 1e12
            e.update({"hbm": {"achieved": fu_gbs, "peak": peak, "unit": "GB/s",
                              "frac": (fu_gbs / peak) if fu_gbs else None},
                      "kernel": "pair forces (binary64 pair terms)",
                      "achieved": ach, "peak": f["fp64_fma_tflops"], "unit": "TFLOP/s",
                      "frac": ach / f["fp64_fma_tflops"], "t_ms": t,
                      "peak_source": f.get("peak_source", "measured DFMA microbenchmark"),
                      "flop_source": f.get("flop_source", "ncu")})
        except Exception:
            e["note"] = "FP64-bound; FLOP count not measured yet (profiles/r02/fp64_*.json)"
    return e


def cpu_model() -> str:
    """The host CPU's model name (for the CPU baseline lines)."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def run_oracle_steps(cfg, steps: int, warmup: int, budget_s: float, nthreads: int):
    rng = np.random.default_rng(SEED)
    n = cfg["n"]
    pos = initial_positions(cfg, rng)
    sp = (np.arange(n) >= n // 2).astype(np.uint8) if cfg["types"] == "half" \
        else np.ones(n, np.uint8)
    if n < 100_000:
        nthreads = 1  # thread start-up dominates small steps
    sim = oracle_sim(cfg, pos, sp, nthreads)
    xi_rng = np.random.default_rng(SEED + 1)
    for _ in range(warmup):
        sim.step(xi_rng.standard_normal((n, 2)))
    sim.timings = {}
    done, t_used = 0, 0.0
    while done < steps and (done == 0 or t_used < budget_s):
        xi = xi_rng.standard_normal((n, 2))
        if cfg["prec"] == "fp32":
            xi = xi.astype(np.float32).astype(np.float64)
        t0 = time.perf_counter()
        sim.step(xi)
        t_used += time.perf_counter() - t0
        done += 1
    return done, t_used, dict(sim.timings)


def reference_arm(args, cfg, rank):
    if rank != 0:
        return
    ncores = os.cpu_count() or 1
    # bounded sample: warm-up 0 (no JIT in the port), at most ~150 s timed
    done, t_used, stages = run_oracle_steps(cfg, args.steps, 0, 150.0, ncores)
    value = cfg["n"] * done / t_used
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": done, "warmup": 0,
        "ms_per_step": 1e3 * t_used / done, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64 (fp32 storage)" if cfg["prec"] == "fp32" else "f64",
        "data": "synthetic",
        "config": config_dict(args.config, cfg, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ncores, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{done} full step(s) of {args.config} (N={cfg['n']}) on the "
                                   f"oracle restatement (oracle/, C + numpy FFT), "
                                   f"{ncores} OpenMP threads; requested {args.steps}",
                         "stage_s": stages},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_numba": reference_numba(args.config),
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-perf-mode", action="store_true")
    ap.add_argument("--force-slabs", action="store_true",
                    help="run the N > 1 slab path (NCCL transports) even with one rank")
    ap.add_argument("--rebalance-every", type=int, default=25,
                    help="N > 1: re-balance the y-slabs every M steps (0: never)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        reference_arm(args, cfg, rank)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    slabs_on = (world > 1 or args.force_slabs) and cfg["prec"] == "fp32"
    if world > 1 or slabs_on:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if world > 1:
            dist.barrier()

    if slabs_on:
        run_slabs(args, cfg, rank, world, barrier)
        dist.destroy_process_group()
        return

    sim, st, pos_host, sp_host = make_state(cfg, rank)
    n = cfg["n"]
    K, W = args.steps, max(args.warmup, 0)
    dt_ = st["pos"].dtype
    # pre-generated seeded N(0,1) increments, resident in HBM
    blocks = K + W
    per_block = n * 2 * (8 if dt_ == torch.float64 else 4)
    if blocks * per_block > 40e9:
        blocks = max(1, int(40e9 // per_block))
    gen = torch.Generator(device="cuda").manual_seed(SEED + 17 * rank)
    xi = torch.randn((blocks, n, 2), generator=gen, device="cuda", dtype=torch.float32).to(dt_)
    stream = torch.cuda.current_stream()

    for w in range(W):
        sim.step(xi[w % blocks], 1)
    torch.cuda.synchronize()
    if sim.status().code != 0:
        raise RuntimeError(f"warm-up failed: status {sim.status().code}")

    launches = 0
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local_rank)
    with clocks:
        barrier()
        torch.cuda.synchronize()
        start.record(stream)
        if W + K <= blocks:  # the K steps' increments are contiguous: one call
            sim.step(xi[W:W + K], K)
            launches += sim.launches()
        else:
            for k in range(K):
                sim.step(xi[(W + k) % blocks], 1)
                launches += sim.launches()
        sim.export_state()  # the job's result back in the caller's (id-ordered) arrays
        launches += 1 if sim.engine == "sorted" else 0
        end.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = start.elapsed_time(end)
    st_ = sim.status()
    if st_.code != 0:
        raise RuntimeError(f"timed run failed: status {st_.code} at step {st_.step}")
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    value = n * world * K / (ms_max / 1e3)

    # ---- stage times (separate profiled pass, same stream, CUDA events)
    sim.set_profiling(True)
    KP = min(K, 10)
    if W + KP <= blocks:  # one call, as the timed run (the engine sees the coming step's block)
        sim.step(xi[W:W + KP], KP)
    else:
        for k in range(KP):
            sim.step(xi[(W + k) % blocks], 1)
    stages = {k: v / KP for k, v in sim.stage_times().items()}
    sim.set_profiling(False)
    t_fu = stages["bin"] + stages["force"] + stages["update"]
    t_pde = stages["deposit"] + stages["solve"] + stages["gradient"]
    ab = algorithmic_bytes(cfg)
    peak, peak_src = measured_peak()
    fu_gbs = ab["fu"] / (t_fu / 1e3) / 1e9 if t_fu > 0 else None
    step_gbs = ab["total"] / (ms_max / K / 1e3) / 1e9
    traffic = ncu_traffic(args.config)

    # ---- end to end: host-resident increments copied in every step, status
    # word read back every step, through the C-ABI sim call
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(sim, n, dt_, K, W, barrier, world)

    # ---- performance mode (SURVEY 7 hard part 6): the sorted engine reading
    # the increments by storage slot (coalesced) instead of by particle id;
    # same distribution (parity tier T4), not the same trajectory
    perf = None
    engine_name = sim.engine
    if engine_name == "sorted" and not args.no_perf_mode:
        del sim
        torch.cuda.empty_cache()
        sim2, _, _, _ = make_state(cfg, rank, xi_by_slot=True)
        for w in range(W):
            sim2.step(xi[w % blocks], 1)
        barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        if W + K <= blocks:
            sim2.step(xi[W:W + K], K)
        else:
            for k in range(K):
                sim2.step(xi[(W + k) % blocks], 1)
        sim2.export_state()
        b.record(stream)
        torch.cuda.synchronize()
        barrier()
        if sim2.status().code != 0:
            raise RuntimeError("performance-mode run failed")
        pms = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([pms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            pms = float(t.item())
        sim2.set_profiling(True)
        if W + KP <= blocks:
            sim2.step(xi[W:W + KP], KP)
        else:
            for k in range(KP):
                sim2.step(xi[(W + k) % blocks], 1)
        pst = {k: v / KP for k, v in sim2.stage_times().items()}
        sim2.set_profiling(False)
        p_fu = pst["bin"] + pst["force"] + pst["update"]
        perf = {"value": n * world * K / (pms / 1e3), "unit": UNIT, "ms_per_step": pms / K,
                "stage_ms": {k: round(v, 4) for k, v in pst.items()},
                "roofline_frac": (ab["fu"] / (p_fu / 1e3) / 1e9) / peak,
                "xi_order": "slot",
                "note": "performance mode: increments consumed in storage-slot order "
                        "(cs_sim_params.xi_by_slot); i.i.d. N(0,1), so the same dynamics in "
                        "distribution (tests/test_gpu_t4.py), not the reference's trajectory"}
        del sim2

    # ---- CPU baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ncores = os.cpu_count() or 1
        done, t_used, stg = run_oracle_steps(cfg, 1, 0, 30.0, ncores)
        cpu = {"value": cfg["n"] * done / t_used, "unit": UNIT, "cores": ncores, "kind": "port",
               "cpu_model": cpu_model(),
               "sample": f"{done} full step of {args.config} (N={cfg['n']}, "
                         f"{cfg['n_c']}^2 grid) on the oracle restatement "
                         f"(C + numpy FFT), {ncores} OpenMP threads",
               "stage_s": {k: round(v, 3) for k, v in stg.items()}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms_max / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f64" if cfg["prec"] == "fp64" else "f64 (fp32 storage)",
            "data": "synthetic",
            "config": config_dict(args.config, cfg, world),
            "roofline": roofline_entry(args.config, cfg, fu_gbs, peak, peak_src, traffic, ab,
                                       t_fu, stages),
            "step_roofline": {"achieved": step_gbs, "peak": peak, "unit": "GB/s",
                              "frac": step_gbs / peak, "algorithmic_bytes_per_step": ab["total"]},
            "stage_ms": {k: round(v, 4) for k, v in stages.items()},
            "engine": engine_name,
            "clocks": clocks.summary(),
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "reference_numba": reference_numba(args.config),
            "perf_mode": perf,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def slab_setup(cfg: dict, world: int):
    """(engine params, state tensors, cell-row bounds, field plan) of one
    system of the config split into world y-slabs: the seeded initial state
    (rank 0's seed on every rank), count-balanced on the initial cell-row
    histogram."""
    from paper_1805_11007_b200 import slabs
    params, st, pos, sp = make_state(cfg, 0, engine="sorted", build_sim=False)
    radii = cfg["radii"]
    cell = 2.0 * (radii[1] if radii else cfg["eps"])
    geom = slabs.CellGeometry.make(-0.5, 0.5, cell)
    counts = np.bincount(geom.row_of(pos[:, 1].astype(np.float64)), minlength=geom.n)
    bounds = slabs.SlabLayout.balanced(counts, world).bounds
    plan = slabs.FieldPlan.make(bounds, geom.n, cfg["n_c"], world) if cfg["field"] else None
    return params, st, bounds, plan


def run_slabs(args, cfg, rank, world, barrier):
    """N > 1: ONE system of the config decomposed into y-slabs over the N
    ranks (slabs.py): strong scaling, value = N_particles * K /
    (device time of K steps, max over ranks).  Every rank builds the same
    seeded initial state and increments (rank 0's seed), the layout is
    count-balanced on the initial cell-row histogram."""
    import torch
    import torch.distributed as dist
    from paper_1805_11007_b200 import slabs
    n, K, W = cfg["n"], args.steps, max(args.warmup, 0)
    params, st, bounds, plan = slab_setup(cfg, world)
    eng = slabs.SlabEngine(params, st, bounds, rank, world, field_plan=plan)
    # the warm-up steps go through the counted exchange (one host round trip
    # per step) and size the packed one the timed steps use (none)
    tr = slabs.PackedNcclTransport(world)
    blocks = K + W
    gen = torch.Generator(device="cuda").manual_seed(SEED)
    xi = torch.randn((blocks, n, 2), generator=gen, device="cuda", dtype=torch.float32)
    overlap = not os.environ.get("CS_SLAB_NO_OVERLAP")  # field step beside the pair forces
    for w in range(W):
        eng.step(xi[w], tr, overlap)
    if W > 0 and not os.environ.get("CS_SLAB_COUNTED"):
        tr.calibrate()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    launches = 0
    with clocks:
        barrier()
        torch.cuda.synchronize()
        a.record(stream)
        for k in range(K):
            eng.step(xi[W + k], tr, overlap)
            launches += eng.sim.launches()  # forces / update / sort / deposit of the step
            if args.rebalance_every and (k + 1) % args.rebalance_every == 0 and k + 1 < K:
                eng.rebalance(tr, eng.n1, cfg["n_c"] if cfg["field"] else None)
        b.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = a.elapsed_time(b)
    code = eng.status().code
    t = torch.tensor([ms, float(code != 0)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, failed = float(t[0].item()), bool(t[1].item())
    if failed:
        raise RuntimeError("slab run failed on some rank")
    lo, hi = eng.owned_range()
    if rank == 0:
        line = {
            "metric": METRIC, "value": n * K / (ms_max / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": ms_max / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64 (fp32 storage)",
            "data": "synthetic",
            "config": dict(config_dict(args.config, cfg, world),
                           parallelism=f"yslab{world}",
                           decomposition="one system, count-balanced y-slabs of cell rows "
                                         f"(re-balanced every {args.rebalance_every} steps), "
                                         "even grid-row split, NCCL all-to-all exchanges",
                           exchange=(f"packed, {tr.seg} slots per destination, no host sync"
                                     if tr.seg else "counted (one host round trip per step)")),
            "engine": "sorted (slab mode)", "clocks": clocks.summary(),
            "gpu_launches": launches,  # rank 0's particle kernels (the field passes not counted)
            "rank0_owned": hi - lo,
            "e2e": None,
            "note": "N > 1: one slab-decomposed system (strong scaling); the end-to-end "
                    "host-increment variant is measured at N = 1",
        }
        print(json.dumps(line), flush=True)
    eng.close()


def run_e2e(sim, n, dt_, K, W, barrier, world):
    """K steps with the step's increments in pinned host memory, copied H2D on
    a side stream (double-buffered, overlapping the previous step), and the
    status word copied D2H after every step."""
    import torch
    from paper_1805_11007_b200 import _native as N
    lib = N.load_library()
    es = 8 if dt_ == torch.float64 else 4
    nhost = min(K, 4)
    gen = torch.Generator().manual_seed(SEED + 99)
    host = [torch.randn((n, 2), generator=gen, dtype=torch.float32).to(dt_).pin_memory()
            for _ in range(nhost)]
    dev = [torch.empty((n, 2), dtype=dt_, device="cuda") for _ in range(2)]
    sbytes = int(lib.cs_sim_status_bytes())
    status_host = torch.empty(sbytes, dtype=torch.uint8).pin_memory()
    sdev = lib.cs_sim_status_device(sim._h)
    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]

    def one_pass(k_steps):
        for k in range(k_steps):
            b = k % 2
            with torch.cuda.stream(copy):
                copy.wait_event(free[b])
                dev[b].copy_(host[k % nhost], non_blocking=True)
                ready[b].record(copy)
            comp.wait_event(ready[b])
            sim.step(dev[b], 1)
            free[b].record(comp)
            # D2H of the step's result (status word) into pinned memory
            _d2h(status_host, sdev, sbytes)

    for b in range(2):
        free[b].record(comp)
    one_pass(min(W, 2))
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    start.record(comp)
    one_pass(K)
    end.record(comp)
    torch.cuda.synchronize()
    barrier()
    ms = start.elapsed_time(end)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": n * world * K / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": n * 2 * es, "d2h_bytes_per_step": sbytes,
            "ms_per_step": ms / K,
            "path": "DeviceSim.step (cs_sim_step C ABI) with pinned host increments, "
                    "side-stream H2D double-buffered, status D2H every step"}


_STATUS_VIEW = {}


def _d2h(host_tensor, dev_ptr, nbytes):
    """Asynchronous device->host copy of the library's status word (current
    stream), through a byte view aliasing the library-owned device memory."""
    key = (dev_ptr, nbytes)
    if key not in _STATUS_VIEW:
        _STATUS_VIEW[key] = _device_bytes(dev_ptr, nbytes)
    host_tensor.copy_(_STATUS_VIEW[key], non_blocking=True)


def _device_bytes(ptr, nbytes):
    """uint8 CUDA tensor aliasing library memory (via __cuda_array_interface__)."""
    import torch

    class _Alias:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                    "data": (int(ptr), False), "version": 3}
    return torch.as_tensor(_Alias(), device="cuda")


if __name__ == "__main__":
    main()
