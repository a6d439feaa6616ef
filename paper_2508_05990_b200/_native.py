"""ctypes binding of libbmc_b200.so (the C ABI in include/bmc.h).

PyTorch is only the plumbing here: it owns device memory and streams; every
compute call goes through the C ABI into the hand-written sm_100a kernels.
There is no CPU fallback: if the library or a CUDA device is missing, the
product path raises.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "lib" / "libbmc_b200.so"
ABI_VERSION = 2  # must equal BMC_ABI_VERSION (include/bmc.h)

BMC_OK, BMC_E_ARG, BMC_E_CUDA, BMC_E_NOVALID, BMC_E_SMEM = 0, 1, 2, 3, 4
KIND_LUMA, KIND_BAYER = 0, 1
MAX_LEVELS = 8

i32, i64, f64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class FmeParams(ctypes.Structure):
    """Mirror of ``bmc_fme_params`` (include/bmc.h)."""

    _fields_ = [
        ("planes", i32), ("elem_bytes", i32), ("max_value", i32),
        ("real_h", i32), ("real_w", i32), ("pad_h", i32), ("pad_w", i32), ("pitch", i32),
        ("plane_stride", i64), ("frame_stride", i64),
        ("n_levels", i32), ("block_sizes", i32 * MAX_LEVELS),
        ("stage_range", i32 * 3), ("stage_step", i32 * 3),
        ("lam", f64), ("one_minus_lam", f64), ("sparsity_tolerance", f64),
        ("split_threshold", f64), ("refine_block_threshold", f64),
    ]


class LevelOut(ctypes.Structure):
    _fields_ = [("mv", vp), ("energy", vp), ("matched", vp), ("evals", vp)]


class SelectParams(ctypes.Structure):
    _fields_ = [
        ("grid_h", i32), ("grid_w", i32), ("factor", i32), ("coarse_h", i32), ("coarse_w", i32),
        ("statistic_mean", i32), ("policy_keyframe", i32), ("has_max_gop", i32), ("max_gop", i32),
        ("aem_threshold", f64),
    ]


class Session(ctypes.Structure):
    """Mirror of ``bmc_session`` (include/bmc_ext.h): the native chunked clip executor."""

    MAX_CHUNKS = 64
    _fields_ = [
        ("T", i32), ("H", i32), ("W", i32), ("elem_bytes", i32), ("kind", i32), ("n_chunks", i32), ("lag", i32),
        ("chunk_begin", i32 * 65),
        ("gh", i32), ("gw", i32), ("b_final", i32), ("scale", i32), ("deviation_threshold", i32),
        ("n_levels", i32), ("Hl", i32), ("Wl", i32), ("ring_vote", i32),
        ("params", FmeParams), ("select", SelectParams),
        ("raw", vp), ("planes", vp), ("cur_index", vp), ("ref_index", vp), ("levels", LevelOut * MAX_LEVELS),
        ("mv_ref", vp), ("e_ref", vp), ("replaced", vp), ("aem_state", vp), ("aem_state_bytes", i64),
        ("acc", vp), ("fsk", vp), ("last_key", vp), ("kind_out", vp), ("ref_out", vp), ("trigger", vp),
        ("labels", vp), ("key_labels", vp), ("chain_ws", vp),
        ("cabr_packed", vp), ("cabr_classes", i32), ("cabr_scratch", vp), ("cabr_ws", vp),
        ("host_raw", vp), ("host_keys", vp), ("host_labels", vp), ("host_kind", vp), ("host_ref", vp),
        ("host_trigger", vp), ("compute", vp), ("copy_in", vp), ("copy_out", vp),
        ("h2d_bytes", i64), ("d2h_bytes", i64), ("priv", vp),
    ]


_SIGNATURES = {
    "bmc_version": (ctypes.c_char_p, []),
    "bmc_abi_version": (ctypes.c_int, []),
    "bmc_struct_size": (ctypes.c_size_t, [ctypes.c_int]),
    "bmc_memset_async": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_size_t, vp]),
    "bmc_last_error": (ctypes.c_char_p, []),
    "bmc_fill_params": (ctypes.c_int, [ctypes.POINTER(FmeParams), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int, ctypes.POINTER(i32), ctypes.POINTER(i32),
                                       ctypes.POINTER(i32), f64, f64, f64, f64]),
    "bmc_plane_buffer_elems": (ctypes.c_size_t, [ctypes.POINTER(FmeParams), ctypes.c_int]),
    "bmc_pack_planes": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(FmeParams), vp, vp]),
    "bmc_estimate_motion": (ctypes.c_int, [vp, ctypes.c_int, ctypes.POINTER(FmeParams), ctypes.c_int, vp, vp,
                                           ctypes.POINTER(LevelOut), vp]),
    "bmc_search_stage": (ctypes.c_int, [vp, vp, ctypes.POINTER(FmeParams)] + [ctypes.c_int] * 7 + [vp, vp, vp, vp]),
    "bmc_block_energy_f64": (ctypes.c_int, [vp, vp, i64, f64, f64, vp, vp]),
    "bmc_refine_mvs": (ctypes.c_int, [vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      vp, ctypes.POINTER(FmeParams), vp, vp, vp, vp, vp, vp]),
    "bmc_decide": (ctypes.c_int, [vp, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.POINTER(SelectParams), vp, vp, vp, vp, vp, vp, i64, vp, i32, vp]),
    "bmc_predict_labels": (ctypes.c_int, [vp, i64, i64, vp, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int, i64,
                                          ctypes.c_int, ctypes.c_int, vp, i64, i64, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, vp]),
    "bmc_predict_labels_clip": (ctypes.c_int, [vp, i64, i64, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, i64,
                                               ctypes.c_int, ctypes.c_int, vp, i64, i64, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_int, ctypes.c_int, vp, vp, vp, vp]),
    "bmc_predict_features": (ctypes.c_int, [vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_int, ctypes.c_int, vp]),
    # include/bmc_ext.h: float64 plane stacks, ingest, reporting
    "bmc_estimate_motion_f64": (ctypes.c_int, [vp, vp] + [ctypes.c_int] * 6 + [ctypes.POINTER(i32)] * 3
                                + [f64] * 4 + [ctypes.POINTER(LevelOut), vp]),
    "bmc_search_stage_f64": (ctypes.c_int, [vp, vp] + [ctypes.c_int] * 10 + [f64, f64, vp, vp, vp, vp]),
    "bmc_unpack_raw": (ctypes.c_int, [vp, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, vp, vp]),
    "bmc_pack_be16": (ctypes.c_int, [vp, i64, vp, vp]),
    "bmc_confusion": (ctypes.c_int, [vp, vp, i64, ctypes.c_int, i64, ctypes.c_int, ctypes.c_int, vp, vp, vp]),
    # CaBR-Net (include/bmc_ext.h)
    "bmc_cabr_weight_floats": (ctypes.c_size_t, [ctypes.c_int]),
    "bmc_cabr_pack_weights": (ctypes.c_int, [vp, ctypes.c_int, vp, vp]),
    "bmc_cabr_forward_blocks": (ctypes.c_int, [vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int,
                                               ctypes.c_int, ctypes.c_int, vp, vp, vp, vp]),
    "bmc_cabr_forward_patches": (ctypes.c_int, [vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp]),
    "bmc_cabr_extract_patches": (ctypes.c_int, [vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int,
                                                ctypes.c_int, ctypes.c_int, vp, vp, vp]),
    "bmc_refine_blocks": (ctypes.c_int, [vp, ctypes.c_int, vp, vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp]),
    "bmc_cabr_chain_workspace": (ctypes.c_size_t, [ctypes.c_int] * 4),
    "bmc_session_init": (ctypes.c_int, [ctypes.POINTER(Session)]),
    "bmc_session_run": (ctypes.c_int, [ctypes.POINTER(Session)]),
    "bmc_session_destroy": (None, [ctypes.POINTER(Session)]),
    "bmc_cabr_chain": (ctypes.c_int, [vp, i64, i64, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, i64,
                                      ctypes.c_int, ctypes.c_int, vp, i64, i64, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int, i64, i64, ctypes.c_int, vp,
                                      vp, vp, vp]),
}

RAW_BE16, RAW_MIPI10, RAW_MIPI12 = 0, 1, 2

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None


def lib_path() -> Path:
    return _LIB_PATH


def load(build_if_missing: bool = True):
    """Load (and, in a source checkout, rebuild when stale) the shared library.

    A rebuild that was needed and failed raises: loading the previous .so
    would run kernels that no longer match the sources or the ctypes layouts.
    The loaded library's ABI version and struct sizes are checked against this
    module before any call is made.
    """
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if build_if_missing:
            from . import build as _build
            if _build.sources_present():
                _build.build()  # file-locked; raises on a compile error
        if not _LIB_PATH.exists():
            raise ImportError(f"libbmc_b200.so not found at {_LIB_PATH}; run paper_2508_05990_b200/build.py")
        lib = ctypes.CDLL(str(_LIB_PATH))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        abi = lib.bmc_abi_version()
        if abi != ABI_VERSION:
            raise ImportError(f"{_LIB_PATH} has ABI {abi}, the Python binding expects {ABI_VERSION}; rebuild it")
        for code, st in ((0, FmeParams), (1, LevelOut), (2, SelectParams), (3, Session)):
            if lib.bmc_struct_size(code) != ctypes.sizeof(st):
                raise ImportError(f"{_LIB_PATH}: {st.__name__} is {lib.bmc_struct_size(code)} bytes in C, "
                                  f"{ctypes.sizeof(st)} in the binding; rebuild it")
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Map a C status to the reference's exception types."""
    if rc == BMC_OK:
        return
    msg = load().bmc_last_error().decode(errors="replace")
    if rc in (BMC_E_ARG, BMC_E_NOVALID, BMC_E_SMEM):
        raise ValueError(msg)
    raise RuntimeError(msg)


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2508_05990_b200 runs on CUDA (sm_100a) only; no CUDA device is visible "
                           "and there is no CPU fallback")
    return torch


def memset_async(tensor, value: int, stream=None) -> None:
    """Byte fill of a device tensor on the current stream (a memset node under graph capture)."""
    check(load().bmc_memset_async(ptr(tensor), int(value), tensor.numel() * tensor.element_size(),
                                  stream_handle(stream)))


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())


def make_params(kind: int, elem_bytes: int, height: int, width: int, cfg) -> FmeParams:
    """Fill bmc_fme_params from an FmeConfig-like object (fme.py:49-76)."""
    lib = load()
    p = FmeParams()
    bs = (i32 * MAX_LEVELS)(*cfg.block_sizes)
    rs = (i32 * 3)(*[int(s.range) for s in cfg.stages])
    ss = (i32 * 3)(*[int(s.step) for s in cfg.stages])
    check(lib.bmc_fill_params(ctypes.byref(p), kind, elem_bytes, height, width, len(cfg.block_sizes), bs, rs, ss,
                              float(cfg.lam), float(cfg.sparsity_tolerance), float(cfg.split_threshold),
                              float(cfg.refine_block_threshold)))
    return p


def select_params(grid_h, grid_w, factor, coarse_h, coarse_w, statistic, policy, max_gop, aem_threshold):
    sp = SelectParams()
    sp.grid_h, sp.grid_w, sp.factor = grid_h, grid_w, factor
    sp.coarse_h, sp.coarse_w = coarse_h, coarse_w
    sp.statistic_mean = 1 if statistic == "mean" else 0
    sp.policy_keyframe = 1 if policy == "keyframe" else 0
    sp.has_max_gop = 0 if max_gop is None else 1
    sp.max_gop = 0 if max_gop is None else int(max_gop)
    sp.aem_threshold = float(aem_threshold)
    return sp
