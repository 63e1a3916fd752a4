"""ctypes binding of the sm_100a C-ABI library (include/blockfam_b200.h).

The library is built in-tree by paper_2604_07311_b200/build.py.  There is no
fallback: if it is missing, or a compute call is given non-CUDA storage, the
call raises DeviceError.  `declared_symbols()` parses the header so tests can
check that every declared entry point is exported.
"""
from __future__ import annotations

import ctypes
import os
import re
import threading
from pathlib import Path
from typing import Optional

import torch

from ..errors import DeviceError, ShapeError
from ..views import DType, MatrixView

__all__ = [
    "lib",
    "lib_path",
    "header_path",
    "declared_symbols",
    "BfView",
    "BfScatterView",
    "BfCholLevel",
    "BfModesView",
    "as_bfview",
    "stream_ptr",
    "check",
    "require_cuda",
]

_PKG = Path(__file__).resolve().parents[1]
_LIB_PATH = Path(os.environ["BF_LIB_PATH"]) if os.environ.get("BF_LIB_PATH") else _PKG / "_lib" / "libblockfam_b200.so"
_HEADER = _PKG.parent / "include" / "blockfam_b200.h"

BF_OK = 0
BF_ERR_SHAPE = -1


class BfView(ctypes.Structure):
    _fields_ = [
        ("base", ctypes.c_void_p),
        ("off", ctypes.c_int64),
        ("m", ctypes.c_int64),
        ("n", ctypes.c_int64),
        ("rs", ctypes.c_int64),
        ("cs", ctypes.c_int64),
    ]


class BfScatterView(ctypes.Structure):
    _fields_ = [
        ("base", ctypes.c_void_p),
        ("m", ctypes.c_int64),
        ("n", ctypes.c_int64),
        ("rscat", ctypes.c_void_p),
        ("cscat", ctypes.c_void_p),
    ]


class BfModesView(ctypes.Structure):
    _fields_ = [
        ("base", ctypes.c_void_p),
        ("off", ctypes.c_int64),
        ("nr", ctypes.c_int32),
        ("nc", ctypes.c_int32),
        ("rdim", ctypes.c_int64 * 2),
        ("rstr", ctypes.c_int64 * 2),
        ("cdim", ctypes.c_int64 * 2),
        ("cstr", ctypes.c_int64 * 2),
    ]


class BfCholLevel(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("pad_", ctypes.c_int32), ("bs", ctypes.c_int64), ("kc", ctypes.c_int64)]


_lock = threading.Lock()
_lib: Optional[ctypes.CDLL] = None

_P = ctypes.POINTER
_V = _P(BfView)
_SV = _P(BfScatterView)
_I = ctypes.c_int
_D = ctypes.c_double
_L = ctypes.c_int64
_VP = ctypes.c_void_p

_SIGNATURES = {
    "bf_abi_version": ([], _I),
    "bf_release_scratch": ([], _I),
    "bf_scratch_stats": ([_P(_L), _P(_L)], _I),
    "bf_scratch_reset_peak": ([], _I),
    "bf_launch_count": ([], _L),
    "bf_last_error": ([], ctypes.c_char_p),
    "bf_device_sm_count": ([], _I),
    "bf_set_option": ([ctypes.c_char_p, _L], _I),
    "bf_timeline": ([ctypes.POINTER(ctypes.c_float), _I], _I),
    "bf_gemm_d": ([_D, _V, _V, _D, _V, _I, _L, _VP, _VP], _I),
    "bf_gemm_s": ([_D, _V, _V, _D, _V, _I, _L, _VP, _VP], _I),
    "bf_gemm_sd": ([_D, _V, _V, _D, _V, _I, _L, _VP, _VP], _I),
    "bf_scale_d": ([_D, _V, _I, _VP], _I),
    "bf_scale_s": ([_D, _V, _I, _VP], _I),
    "bf_scale_sd": ([_D, _V, _I, _VP], _I),
    "bf_potrf_leaf_d": ([_V, _I, _L, _VP, _VP], _I),
    "bf_potrf_leaf_s": ([_V, _I, _L, _VP, _VP], _I),
    "bf_trsm_rltn_d": ([_D, _V, _V, _L, _VP, _VP], _I),
    "bf_trsm_rltn_s": ([_D, _V, _V, _L, _VP, _VP], _I),
    "bf_cholesky_d": ([_V, _P(BfCholLevel), _I, _VP, _VP], _I),
    "bf_sandwich_skew_d": ([_V, _V, _VP, _L, _VP], _I),
    "bf_sandwich_skew_s": ([_V, _V, _VP, _VP, _L, _VP], _I),
    "bf_ltlt_d": ([_V, _L, _L, _I, _L, _VP, _L, _VP, _VP, _VP, _VP, _VP], _I),
    "bf_ltlt_s": ([_V, _L, _L, _I, _L, _VP, _L, _VP, _VP, _VP, _VP, _VP], _I),
    "bf_qr_panel_d": ([_V, _VP, _VP], _I),
    "bf_gemm_splitk_d": ([_D, _V, _V, _D, _V, _VP], _I),
    "bf_gemm_splitk_s": ([_D, _V, _V, _D, _V, _VP], _I),
    "bf_qr_panel_s": ([_V, _VP, _VP], _I),
    "bf_qr_t_d": ([_V, _VP, _VP, _VP, _VP, _VP], _I),
    "bf_qr_t_s": ([_V, _VP, _VP, _VP, _VP, _VP], _I),
    "bf_reflector_apply_d": ([_V, _L, _D, _V, _VP], _I),
    "bf_reflector_apply_s": ([_V, _L, _D, _V, _VP], _I),
    "bf_lu_d": ([_V, _P(BfCholLevel), _I, _VP, _VP, _VP], _I),
    "bf_lu_s": ([_V, _P(BfCholLevel), _I, _VP, _VP, _VP], _I),
    "bf_trsm_llnu_d": ([_D, _V, _V, _L, _VP], _I),
    "bf_trsm_llnu_s": ([_D, _V, _V, _L, _VP], _I),
    "bf_trsm_lun_d": ([_V, _V, _L, _VP], _I),
    "bf_trsm_lun_s": ([_V, _V, _L, _VP], _I),
    "bf_apply_pivots_d": ([_V, _VP, _L, _I, _VP], _I),
    "bf_apply_pivots_s": ([_V, _VP, _L, _I, _VP], _I),
    "bf_cholesky_host_d": ([_VP, _L, _V, _P(BfCholLevel), _I, _VP, _VP], _I),
    "bf_cholesky_s": ([_V, _P(BfCholLevel), _I, _VP, _VP], _I),
    "bf_cholesky_ex_d": ([_V, _P(BfCholLevel), _I, _L, _VP, _VP], _I),
    "bf_trsm_rltn_ex_d": ([_D, _V, _V, _L, _VP, _VP, _VP], _I),
    "bf_gemm_bf16": ([_D, _VP, _L, _VP, _L, _D, _V, _L, _I, _VP], _I),
    "bf_split_tf32_s": ([_V, _VP, _L, _L, _VP], _I),
    "bf_split_tf32_d": ([_V, _VP, _L, _L, _VP], _I),
    "bf_gemm_tf32": ([_D, _VP, _L, _VP, _L, _D, _V, _L, _I, _VP], _I),
    "bf_gemm_f32_tc": ([_D, _V, _V, _D, _V, _I, _VP], _I),
    "bf_convert_f32_bf16": ([_V, _VP, _L, _I, _VP], _I),
    "bf_convert_f64_f32": ([_V, _V, _I, _VP], _I),
    "bf_convert_f32_f64": ([_V, _V, _I, _VP], _I),
    "bf_row_abs_sum_d": ([_VP, _L, _VP, _L, _VP], _I),
    "bf_convert_f64_bf16": ([_V, _VP, _L, _I, _VP], _I),
    "bf_residual_d": ([_VP, _L, _VP, _VP, _VP, _L, _VP], _I),
    "bf_potrs_f32_d": ([_VP, _L, _VP, _L, _VP], _I),
    "bf_potrs_blocked_f32_d": ([_VP, _L, _VP, _L, _VP, _L, _VP, _VP], _I),
    "bf_gemm_scatter_d": ([_D, _SV, _SV, _D, _SV, _L, _VP], _I),
    "bf_pack_scatter_d": ([_SV, _I, _VP, _VP], _I),
    "bf_gemm_scatter_s": ([_D, _SV, _SV, _D, _SV, _L, _VP], _I),
    "bf_gemm_scatter_sd": ([_D, _SV, _SV, _D, _SV, _L, _VP], _I),
    "bf_contract_bf16_d": ([_D, _V, _V, _D, _V, _VP], _I),
    "bf_contract_modes_d": ([_D, _P(BfModesView), _P(BfModesView), _D, _P(BfModesView), _L, _VP], _I),
    "bf_cholesky_mixed": ([_V, _VP, _L, _VP, _VP, _VP, _VP, _VP, _VP, _L, _P(BfCholLevel), _I, _I, _I, _VP, _VP],
                          _I),
    "bf_dist_available": ([], _I),
    "bf_dist_unique_id_bytes": ([], _I),
    "bf_dist_unique_id": ([_VP], _I),
    "bf_dist_init": ([_VP, _I, _I, _I, _I, _P(_VP)], _I),
    "bf_dist_set_option": ([_VP, ctypes.c_char_p, _L], _I),
    "bf_dist_finalize": ([_VP], _I),
    "bf_dist_local_elems": ([_L, _L, _I, _I, _I], _L),
    "bf_dist_panel_offset": ([_L, _L, _I, _I, _I, _L], _L),
    "bf_dist_fill_synthetic_d": ([_L, _L, _I, _I, _I, _VP, ctypes.c_uint64, _VP], _I),
    "bf_fill_synthetic_d": ([_V, ctypes.c_uint64, _VP], _I),
    "bf_chol_dist_d": ([_VP, _VP, _L, _P(BfCholLevel), _I, _VP, _VP], _I),
    "bf_cholesky_dist_d": ([_VP, _VP, _L, _P(BfCholLevel), _I, _VP, _VP], _I),
}


def lib_path() -> Path:
    return _LIB_PATH


def header_path() -> Path:
    return _HEADER


def declared_symbols() -> list[str]:
    """Function names declared in include/blockfam_b200.h."""
    text = _HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(bf_\w+)\s*\(", text, flags=re.M)))


def lib() -> ctypes.CDLL:
    """Load (once) the sm_100a library; raise loudly if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise DeviceError(
                    f"{_LIB_PATH} is missing: build it with `python -m paper_2604_07311_b200.build` "
                    "(there is no CPU fallback)"
                )
            handle = ctypes.CDLL(str(_LIB_PATH))
            for name, (args, res) in _SIGNATURES.items():
                fn = getattr(handle, name)
                fn.argtypes = args
                fn.restype = res
            _lib = handle
    return _lib


def require_cuda(*objs) -> None:
    """Every operand (a view or a raw tensor) must live in GPU memory."""
    for o in objs:
        st = o if isinstance(o, torch.Tensor) else o.storage
        if not st.is_cuda:
            raise DeviceError(
                "blockfam-b200 computes on the GPU only; operand storage is on "
                f"{st.device} (create views with make_view(..., device='cuda'))"
            )


def as_bfview(v: MatrixView) -> BfView:
    return BfView(v.storage.data_ptr(), v.offset, v.m, v.n, v.rs, v.cs)


def stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def check(rc: int, what: str) -> None:
    if rc == BF_OK:
        return
    msg = (lib().bf_last_error() or b"").decode(errors="replace")
    if rc == BF_ERR_SHAPE:
        raise ShapeError(f"{what}: {msg}")
    raise DeviceError(f"{what} failed (code {rc}): {msg}")


def suffix(dtype: DType, acc: DType) -> str:
    if dtype is DType.F64:
        return "d"
    return "sd" if acc is DType.F64 else "s"
