"""ctypes binding of the in-tree C-ABI library ``libhep.so`` (include/hep.h).

The library is the product: there is no Python or CPU fallback.  If it is
missing, or no CUDA device is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os

from .core import STATUS_ERRORS, HarmonyError

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libhep.so")

c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
vp = ctypes.c_void_p


class HepSchedOut(ctypes.Structure):
    """``hep_sched_out`` (include/hep.h): device output buffers of one solve."""

    _fields_ = [
        ("d_m", vp),
        ("d_xq", vp),
        ("d_xi", vp),
        ("d_gpu_load", vp),
        ("d_ranges", vp),
        ("d_n_ranges", vp),
        ("d_transfer", vp),
        ("d_status", vp),
    ]


TUNING_FIELDS = ("st256", "pair_wait_cluster", "ffn_pair", "ffn_light_rows", "wgrad_order", "l2_policy",
                 "light_first", "raster_gm1", "raster_gm2", "sched_lexmin_warps", "lsu256", "ffn_clock",
                 "router_tile_rows", "pair_wave_sync", "lp_dsm", "light_wave_sync", "router_mc", "router_pair", "wgrad_wave_sync", "wgrad_raster",
                 "sched_route_serial")


class HepTuning(ctypes.Structure):
    """``hep_tuning`` (include/hep.h): process-wide launch tuning, -1 = default."""

    _fields_ = [(f, ctypes.c_int) for f in TUNING_FIELDS] + [("reserved", ctypes.c_int * 1)]


# (name, restype, argtypes) for every symbol declared in include/hep.h
SIGNATURES = {
    "hep_last_error": (ctypes.c_char_p, []),
    "hep_tuning_get": (ctypes.c_int, [ctypes.POINTER(HepTuning)]),
    "hep_tuning_set": (ctypes.c_int, [ctypes.POINTER(HepTuning)]),
    "hep_abi_version": (ctypes.c_int, []),
    "hep_device_sm_count": (ctypes.c_int, []),
    "hep_sched_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, c_i32p, c_i32p, c_i32p, ctypes.c_int, ctypes.POINTER(vp)]),
    "hep_sched_destroy": (ctypes.c_int, [vp]),
    "hep_sched_sizes": (ctypes.c_int, [vp, c_i64p, c_i64p, c_i64p, c_i64p]),
    "hep_sched_solve": (ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_int64, vp, ctypes.c_int, ctypes.POINTER(HepSchedOut), vp]),
    "hep_sched_integerize": (ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.POINTER(HepSchedOut), vp]),
    "hep_sched_pipelined": (ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, vp, ctypes.POINTER(HepSchedOut), ctypes.POINTER(HepSchedOut), vp, vp]),
    "hep_sched_route": (ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_int64, vp, ctypes.c_int, ctypes.POINTER(HepSchedOut), vp]),
    "hep_sched_debug_timing": (ctypes.c_int, [c_i64p, ctypes.c_int]),
    "hep_lp_workspace": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]),
    "hep_lp_solve": (ctypes.c_int, [vp, vp, vp, vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, vp, ctypes.c_double, ctypes.c_int64, vp, ctypes.c_size_t, vp, vp, vp, vp]),
    "hep_transfer_plan": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, vp, ctypes.c_int64, vp, vp, vp]),
    "hep_gate_topk": (ctypes.c_int, [vp, ctypes.c_int64, vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int, vp, vp, vp, vp]),
    "hep_gemm_bf16": (ctypes.c_int, [vp, vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, vp]),
    "hep_router_topk": (ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int, vp, vp, vp, vp, vp, vp]),
    "hep_router_topk_ws": (ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int, vp, vp, vp, vp, vp, vp, vp]),
    "hep_router_sync_bytes": (ctypes.c_size_t, []),
    "hep_gate_chunk_counts": (ctypes.c_int, [vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int, vp, vp]),
    "hep_moe_assign_precounted": (ctypes.c_int, [vp, ctypes.POINTER(HepSchedOut), vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]),
    "hep_moe_assign_chunk_offset": (ctypes.c_size_t, [vp, ctypes.c_int64, ctypes.c_int]),
    "hep_moe_assign": (ctypes.c_int, [vp, ctypes.POINTER(HepSchedOut), vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]),
    "hep_moe_assign_phase": (ctypes.c_int, [vp, ctypes.POINTER(HepSchedOut), vp, ctypes.c_int, vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]),
    "hep_moe_assign_workspace": (ctypes.c_size_t, [vp, ctypes.c_int64, ctypes.c_int]),
    "hep_moe_assign_ep": (ctypes.c_int, [vp, ctypes.POINTER(HepSchedOut), vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, vp, vp, vp, vp, ctypes.c_size_t, vp]),
    "hep_moe_assign_ep_phase": (ctypes.c_int, [vp, ctypes.POINTER(HepSchedOut), vp, ctypes.c_int, vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]),
    "hep_moe_assign_ep_workspace": (ctypes.c_size_t, [vp, ctypes.c_int64, ctypes.c_int]),
    "hep_sched_hosted": (ctypes.c_int, [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    "hep_moe_permute": (ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, vp, vp]),
    "hep_moe_permute_ex": (ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, vp, ctypes.c_int, vp]),
    "hep_moe_expert_ffn": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, vp, vp, vp, ctypes.c_size_t, vp, vp]),
    "hep_moe_expert_ffn_gather": (ctypes.c_int, [vp, ctypes.c_int64, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, vp, vp, vp, ctypes.c_size_t, vp, vp]),
    "hep_ffn_debug_clock": (ctypes.c_int, [c_i64p]),
    "hep_moe_ffn_workspace": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int64, ctypes.c_int]),
    "hep_moe_ffn_launches": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int, ctypes.c_int]),
    "hep_moe_ffn_bwd_launches": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int]),
    "hep_moe_combine": (ctypes.c_int, [vp, vp, vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, vp, vp]),
    "hep_moe_gather_sum": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, vp, vp]),
    "hep_moe_combine_bwd": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, vp, vp, vp]),
    "hep_moe_ep_train_layout": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int64, vp, vp, vp]),
    "hep_moe_rows_to_addr": (ctypes.c_int, [vp, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, vp, vp, vp]),
    "hep_moe_dispatch_p2p": (ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int64, vp, vp]),
    "hep_moe_return_addr": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int64, ctypes.c_int64, vp, vp]),
    "hep_moe_return_addr_map": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int64, ctypes.c_int64, vp, vp, vp]),
    "hep_moe_expert_ffn_p2p": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, vp, vp, vp, ctypes.c_size_t, vp, vp]),
    "hep_p2p_barrier": (ctypes.c_int, [vp, vp, ctypes.c_int, ctypes.c_int, vp]),
    "hep_p2p_allgather": (ctypes.c_int, [vp, ctypes.c_int64, vp, vp, vp, ctypes.c_int, ctypes.c_int, vp]),
    "hep_ipc_handle": (ctypes.c_int, [vp, vp, ctypes.POINTER(ctypes.c_int64)]),
    "hep_ipc_open": (ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_void_p)]),
    "hep_ipc_close": (ctypes.c_int, [vp]),
    "hep_moe_zero_padding": (ctypes.c_int, [vp, vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int64, vp]),
    "hep_moe_expert_ffn_bwd": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, vp, vp, vp, vp, vp, ctypes.c_size_t, vp, vp]),
    "hep_moe_expert_ffn_train": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, vp, vp, vp, vp, ctypes.c_size_t, vp, vp]),
    "hep_gate_bwd": (ctypes.c_int, [vp, vp, vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, vp, vp]),
    "hep_router_bwd": (ctypes.c_int, [vp, vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, vp, vp, vp]),
}

_LIB = None


def lib():
    """Load libhep.so once; raise if it was not built (no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2511_16947_b200.build` "
                "(the CUDA library is required; there is no CPU fallback)"
            )
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(rc: int, where: str) -> None:
    """Raise the reference exception class matching a C-ABI status code."""
    if rc == 0:
        return
    msg = (lib().hep_last_error() or b"").decode(errors="replace")
    cls = STATUS_ERRORS.get(rc)
    if cls is None:
        raise RuntimeError(f"{where}: status {rc}: {msg}")
    raise cls(f"{where}: {msg}")


def raise_status(code: int, where: str) -> None:
    """Raise for a device-detected status word (``d_status``)."""
    if code == 0:
        return
    cls = STATUS_ERRORS.get(int(code), HarmonyError)
    raise cls(f"{where}: device reported status {code}")


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("a CUDA (sm_100a) device is required: this package has no CPU path")
    lib()
    return torch


def get_tuning() -> dict:
    """The library's current launch tuning (``hep_tuning_get``)."""
    t = HepTuning()
    check(lib().hep_tuning_get(ctypes.byref(t)), "hep_tuning_get")
    return {f: getattr(t, f) for f in TUNING_FIELDS}


def set_tuning(**fields) -> dict:
    """Change launch-tuning fields (``hep_tuning_set``); returns the previous values of
    every field so the caller can restore them.  Unknown names raise."""
    old = get_tuning()
    bad = set(fields) - set(TUNING_FIELDS)
    if bad:
        raise ValueError(f"unknown tuning fields {sorted(bad)}")
    t = HepTuning(**{**old, **{k: int(v) for k, v in fields.items()}})
    check(lib().hep_tuning_set(ctypes.byref(t)), "hep_tuning_set")
    return old


class tuning:
    """``with tuning(ffn_pair=1): ...`` — set tuning fields for a block, then restore."""

    def __init__(self, **fields):
        self.fields = fields
        self.old = None

    def __enter__(self):
        self.old = set_tuning(**self.fields)
        return self

    def __exit__(self, *exc):
        set_tuning(**self.old)


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
