"""ctypes binding of libchemo_b200.so (include/chemo_b200.h).

The library is the only compute path of this package: there is no CPU
fallback.  Importing works on a CPU-only host (so the API, parameter objects
and the C-ABI symbol table can be checked), but every compute call raises
``RuntimeError`` unless a CUDA device and the built library are present.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "_build", "libchemo_b200.so")
if os.environ.get("CS_LIB"):  # tuning experiments: an alternative build of the same sources
    SO_PATH = os.path.abspath(os.environ["CS_LIB"])

CS_OK, CS_NONFINITE, CS_OVERSHOOT, CS_UNSETTLED, CS_FIELD_NONFINITE = 0, 1, 2, 3, 4
CS_DEPOSIT_OVERFLOW = 5
CS_SORT_OVERFLOW = 6
CS_F64, CS_F32 = 0, 1
CS_GAUSSIAN, CS_CIC = 0, 1
CS_ENGINE_AUTO, CS_ENGINE_DIRECT, CS_ENGINE_SORTED, CS_ENGINE_CTA = 0, 1, 2, 3

C_i32, C_i64, C_f64, C_p = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class Domain_t(ctypes.Structure):
    _fields_ = [("lo", C_f64 * 2), ("hi", C_f64 * 2), ("periodic", C_i32 * 2)]


class PairParams_t(ctypes.Structure):
    _fields_ = [("eps", C_f64 * 4), ("cutoff", C_f64 * 4), ("cell_cutoff", C_f64)]


class Grid_t(ctypes.Structure):
    _fields_ = [("n_c", C_i32), ("periodic", C_i32), ("lo", C_f64 * 2), ("spacing", C_f64 * 2)]


class SimParams_t(ctypes.Structure):
    _fields_ = [("n", C_i64), ("prec", C_i32), ("n_types", C_i32), ("domain", Domain_t),
                ("interaction", C_i32), ("pairs", PairParams_t), ("amp", C_f64 * 2),
                ("dt", C_f64), ("field_active", C_i32), ("refresh_active", C_i32),
                ("grid", Grid_t), ("d_c", C_f64), ("k_alpha", C_f64), ("k_beta", C_f64),
                ("gamma", C_f64), ("deposit_kind", C_i32), ("kernel_h", C_f64),
                ("kernel_cutoff", C_f64), ("secretes", C_i32 * 2), ("consumes", C_i32 * 2),
                ("chi", C_f64 * 2), ("chi_pinned", C_i32 * 2), ("store_samples", C_i32),
                ("store_next", C_i32), ("engine", C_i32), ("react", C_i32),
                ("react_p_ab", C_f64), ("react_r_beta", C_f64), ("integrator", C_i32),
                ("hard_eps", C_f64), ("diffusion", C_f64 * 2), ("xi_by_slot", C_i32)]


class SimState_t(ctypes.Structure):
    _fields_ = [("pos", C_p), ("next_pos", C_p), ("anchor", C_p), ("type", C_p),
                ("drift", C_p), ("local_c", C_p), ("c", C_p), ("grad", C_p),
                ("rho_a", C_p), ("rho_b", C_p)]


class Status_t(ctypes.Structure):
    _fields_ = [("code", C_i32), ("step", C_i32), ("particle", C_i64), ("axis", C_i32),
                ("clamped", C_i64), ("neg_mass_steps", C_i64), ("first_neg_mass", C_f64),
                ("steps_done", C_i64), ("react_high_count", C_i64),
                ("react_high_max", C_f64)]


class EnsState_t(ctypes.Structure):
    _fields_ = [("pos", C_p), ("anchor", C_p), ("drift", C_p), ("local_c", C_p),
                ("type", C_p), ("c", C_p)]


# (name, restype, argtypes) -- every symbol include/chemo_b200.h declares
SIGNATURES = [
    ("cs_abi_version", C_i32, []),
    ("cs_last_error", ctypes.c_char_p, []),
    ("cs_ctx_create", C_i32, [C_i32, C_p, ctypes.POINTER(C_p)]),
    ("cs_ctx_set_stream", C_i32, [C_p, C_p]),
    ("cs_ctx_sync", C_i32, [C_p]),
    ("cs_ctx_destroy", C_i32, [C_p]),
    ("cs_soft_forces", C_i32, [C_p, C_i32, C_p, C_p, C_i64, ctypes.POINTER(Domain_t),
                               ctypes.POINTER(PairParams_t), C_p]),
    ("cs_soft_force_pairs", C_i32, [C_p, C_i32, C_p, C_p, C_i64, ctypes.POINTER(Domain_t),
                                    ctypes.POINTER(PairParams_t), C_p, C_i64,
                                    ctypes.POINTER(C_i64)]),
    ("cs_cell_index", C_i32, [C_p, C_i32, C_p, C_i64, ctypes.POINTER(Domain_t), C_f64, C_p,
                              C_p, C_p, C_p]),
    ("cs_index_forces", C_i32, [C_p, C_i32, C_p, C_i64, C_p, C_p, C_p,
                                ctypes.POINTER(Domain_t), C_p, C_f64, C_f64, C_p]),
    ("cs_deposit_gather", C_i32, [C_p, C_i32, C_p, C_i64, ctypes.POINTER(Grid_t), C_f64, C_f64,
                                  C_f64, C_f64, C_p]),
    ("cs_em_step", C_i32, [C_p, C_i32, C_p, C_p, C_p, C_p, C_p, C_f64, C_i64, C_p]),
    ("cs_tamed_step", C_i32, [C_p, C_i32, C_p, C_p, C_p, C_p, C_p, C_f64, C_i64, C_p]),
    ("cs_apply_boundaries", C_i32, [C_p, C_i32, C_p, C_p, C_p, C_i64, ctypes.POINTER(Domain_t),
                                    ctypes.POINTER(C_i64), ctypes.POINTER(C_i32)]),
    ("cs_deposit", C_i32, [C_p, C_i32, C_p, C_p, C_i64, ctypes.POINTER(Grid_t), C_i32, C_f64,
                           C_f64, C_p, C_p]),
    ("cs_bilinear", C_i32, [C_p, C_i32, C_p, C_i64, C_p, C_i32, ctypes.POINTER(Grid_t), C_p,
                            ctypes.POINTER(C_i64)]),
    ("cs_gradient", C_i32, [C_p, C_i32, C_p, ctypes.POINTER(Grid_t), C_p]),
    ("cs_field_ops_create", C_i32, [C_p, C_i32, ctypes.POINTER(Grid_t), C_f64, C_f64,
                                    ctypes.POINTER(C_p)]),
    ("cs_field_ops_destroy", C_i32, [C_p]),
    ("cs_field_solve", C_i32, [C_p, C_p, C_p]),
    ("cs_field_step", C_i32, [C_p, C_p, C_p, C_p, C_f64, C_f64, C_f64, ctypes.POINTER(C_i32),
                              ctypes.POINTER(C_f64)]),
    ("cs_exp_batch", C_i32, [C_p, C_p, C_p, C_i64]),
    ("cs_resolve_hard_sphere", C_i32, [C_p, C_i32, C_p, C_p, C_i64, ctypes.POINTER(Domain_t),
                                       C_f64, C_f64, C_f64]),
    ("cs_react", C_i32, [C_p, C_p, C_p, C_p, C_p, C_i64, C_f64, C_f64, C_f64,
                         ctypes.POINTER(C_i64), ctypes.POINTER(C_f64)]),
    ("cs_sim_create", C_i32, [C_p, ctypes.POINTER(SimParams_t), ctypes.POINTER(C_p)]),
    ("cs_sim_destroy", C_i32, [C_p]),
    ("cs_sim_step", C_i32, [C_p, ctypes.POINTER(SimState_t), C_p, C_i64, C_i32]),
    ("cs_sim_step_react", C_i32, [C_p, ctypes.POINTER(SimState_t), C_p, C_i64, C_p, C_i64,
                                  C_i32]),
    ("cs_sim_status", C_i32, [C_p, ctypes.POINTER(Status_t)]),
    ("cs_sim_reset_status", C_i32, [C_p]),
    ("cs_sim_launches", C_i64, [C_p]),
    ("cs_sim_set_profiling", C_i32, [C_p, C_i32]),
    ("cs_sim_stage_times", C_i32, [C_p, C_p, C_i32]),
    ("cs_sim_engine", C_i32, [C_p]),
    ("cs_sim_import", C_i32, [C_p, ctypes.POINTER(SimState_t)]),
    ("cs_slab_config", C_i32, [C_p, ctypes.POINTER(C_i32), C_i32, C_i32]),
    ("cs_slab_import", C_i32, [C_p, ctypes.POINTER(SimState_t)]),
    ("cs_slab_step_local", C_i32, [C_p, ctypes.POINTER(SimState_t), C_p]),
    ("cs_slab_step_part", C_i32, [C_p, ctypes.POINTER(SimState_t), C_p, C_i32]),
    ("cs_slab_outbox", C_i32, [C_p, ctypes.POINTER(C_p), ctypes.POINTER(C_p),
                               ctypes.POINTER(C_i64)]),
    ("cs_slab_claim", C_i32, [C_p, C_p, C_i64]),
    ("cs_slab_finish", C_i32, [C_p]),
    ("cs_slab_exchange_cap", C_i32, [C_p, C_i64]),
    ("cs_slab_outbox_packed", C_i32, [C_p, ctypes.POINTER(C_p), ctypes.POINTER(C_p),
                                      ctypes.POINTER(C_i64)]),
    ("cs_slab_claim_packed", C_i32, [C_p, C_p, C_p, C_i64]),
    ("cs_slab_range", C_i32, [C_p, ctypes.POINTER(C_i64), ctypes.POINTER(C_i64)]),
    ("cs_slab_field_config", C_i32, [C_p, C_i32, C_i32, C_i32, C_i32, C_i32, C_i32]),
    ("cs_slab_rho", C_p, [C_p]),
    ("cs_slab_field_rows", C_i32, [C_p, ctypes.POINTER(SimState_t), C_p, C_i32]),
    ("cs_slab_field_cols", C_i32, [C_p, C_p, C_i32, C_i32, C_i32]),
    ("cs_slab_field_grad", C_i32, [C_p, ctypes.POINTER(SimState_t)]),
    ("cs_slab_row_counts", C_i32, [C_p, C_p]),
    ("cs_slab_rebalance", C_i32, [C_p, ctypes.POINTER(C_i32)]),
    ("cs_slab_finish_rebalance", C_i32, [C_p]),
    ("cs_sim_export", C_i32, [C_p, ctypes.POINTER(SimState_t)]),
    ("cs_sim_status_device", C_p, [C_p]),
    ("cs_sim_status_bytes", C_i64, []),
    ("cs_ens_create", C_i32, [C_p, ctypes.POINTER(SimParams_t), C_i32, ctypes.POINTER(C_p)]),
    ("cs_ens_destroy", C_i32, [C_p]),
    ("cs_ens_step", C_i32, [C_p, ctypes.POINTER(EnsState_t), C_p, C_p, C_i32]),
    ("cs_ens_status", C_i32, [C_p, C_p]),
    ("cs_ens_observe", C_i32, [C_p, ctypes.POINTER(EnsState_t), C_p, C_p]),
    ("cs_rng_fill", C_i32, [C_p, C_p, C_i32, C_i32, C_i32, C_i64, C_p]),
    ("cs_rng_fill_stream", C_i32, [C_p, C_p, C_i32, C_i64, C_i32, C_p]),
    ("cs_msd", C_i32, [C_p, C_i32, C_p, C_p, C_i64, C_p]),
    ("cs_hist2d", C_i32, [C_p, C_i32, C_p, C_p, C_i64, C_i32, C_p, C_p, C_i32, C_i64, C_p]),
    ("cs_log1p_batch", C_i32, [C_p, C_p, C_p, C_i64]),
]

STAGES = ("deposit", "solve", "gradient", "bin", "force", "update")

_lib = None
_lock = threading.Lock()


def load_library():
    """Load (without requiring a GPU) and type the C-ABI library."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(SO_PATH):
                raise RuntimeError(
                    f"{SO_PATH} is missing: build it with "
                    "`python -m paper_1805_11007_b200.build` (nvcc, sm_100a)")
            lib = ctypes.CDLL(SO_PATH)
            for name, res, args in SIGNATURES:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class NativeError(RuntimeError):
    pass


def check(rc: int, what: str) -> int:
    if rc < 0:
        msg = load_library().cs_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed (code {rc}): {msg}")
    return rc


_ctx = {}


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1805_11007_b200 needs a CUDA device (sm_100a B200); there is no "
            "CPU fallback")
    load_library()
    return torch


def context(device=None):
    """The library context of the current device, bound to torch's current
    stream (rebound on every call, so callers may switch streams)."""
    torch = require_cuda()
    dev = torch.cuda.current_device() if device is None else int(device)
    stream = torch.cuda.current_stream(dev).cuda_stream
    lib = load_library()
    h = _ctx.get(dev)
    if h is None:
        p = C_p()
        with torch.cuda.device(dev):
            check(lib.cs_ctx_create(dev, C_p(stream), ctypes.byref(p)), "cs_ctx_create")
        h = p
        _ctx[dev] = h
    check(lib.cs_ctx_set_stream(h, C_p(stream)), "cs_ctx_set_stream")
    return h


def ptr(t) -> C_p:
    return C_p(0 if t is None else t.data_ptr())


def domain_struct(lo, hi, periodic) -> Domain_t:
    d = Domain_t()
    for a in range(2):
        d.lo[a] = float(lo[a])
        d.hi[a] = float(hi[a])
        d.periodic[a] = 1 if bool(periodic[a]) else 0
    return d


def pair_struct(eps_tab, cut_tab, cell_cutoff) -> PairParams_t:
    p = PairParams_t()
    for k in range(4):
        p.eps[k] = float(eps_tab[k])
        p.cutoff[k] = float(cut_tab[k])
    p.cell_cutoff = float(cell_cutoff)
    return p


def grid_struct(grid) -> Grid_t:
    g = Grid_t()
    g.n_c = int(grid.n_c)
    g.periodic = 1 if grid.boundary == "periodic" else 0
    sp = grid.spacing
    for a in range(2):
        g.lo[a] = float(grid.lo[a])
        g.spacing[a] = float(sp[a])
    return g


def prec_code(dtype) -> int:
    s = str(dtype)
    if s.endswith("float64"):
        return CS_F64
    if s.endswith("float32"):
        return CS_F32
    raise TypeError(f"unsupported dtype {dtype}")


def to_device(a, dtype=None, device=None):
    """(tensor on the CUDA device, was_host) for numpy or torch input."""
    torch = require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    if isinstance(a, torch.Tensor):
        t = a
        was_host = t.device.type != "cuda"
    else:
        t = torch.from_numpy(np.ascontiguousarray(a))
        was_host = True
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    t = t.to(dev).contiguous()
    return t, was_host
