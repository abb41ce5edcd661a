"""ctypes binding of include/qweight_b200.h.

The library is built in-tree (paper_2311_16442_b200/lib/libqweight_b200.so).
There is no fallback: if the library is missing or a call fails, a
QWeightError is raised.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libqweight_b200.so"

QW_OK, QW_ERR_ARG, QW_ERR_LAYER, QW_ERR_CUDA, QW_ERR_NCCL = 0, 1, 2, 3, 4
QW_ERR_UNSUPPORTED, QW_ERR_NOMEM, QW_ERR_IO, QW_ERR_FORMAT = 5, 6, 7, 8


class QWeightError(RuntimeError):
    """Python face of qweight::Error (reference types.hpp:11-14)."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


u8p, u16p, u32p = C.POINTER(C.c_uint8), C.POINTER(C.c_uint16), C.POINTER(C.c_uint32)


class LayerView(C.Structure):
    _fields_ = [
        ("n", C.c_uint16), ("n2", C.c_uint16), ("group1", C.c_uint16),
        ("group2", C.c_uint16), ("tile", C.c_uint16),
        ("rows", C.c_uint32), ("cols", C.c_uint32), ("n4", C.c_uint32),
        ("pad2", C.c_uint32), ("outlier_count", C.c_uint32),
        ("alpha", C.c_float), ("outlier_ratio", C.c_float),
        ("plan_bits", u8p), ("plan_bits_len", C.c_uint64),
        ("plan_perm", u32p), ("plan_perm_len", C.c_uint64),
        ("main", u8p), ("main_len", C.c_uint64),
        ("tail2", u8p), ("tail2_len", C.c_uint64),
        ("tail4", u8p), ("tail4_len", C.c_uint64),
        ("secondary", u8p), ("secondary_len", C.c_uint64),
        ("meta", u16p), ("meta_len", C.c_uint64),
        ("sorder_zero2", u8p), ("sorder_scale2", u16p), ("sorder_len", C.c_uint64),
        ("fourbit_scale", u16p), ("fourbit_zero", u8p), ("fourbit_len", C.c_uint64),
        ("csr_row_ptr", u32p), ("csr_row_ptr_len", C.c_uint64),
        ("csr_col_ind", u16p), ("csr_values", u16p), ("csr_nnz", C.c_uint64),
    ]


class LayerInfo(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in (
        "rows", "cols", "padded_cols", "n2_padded", "n4", "triples", "blocks4",
        "groups", "group2", "row_blocks", "quads", "quad_bytes")] + [
        (n, C.c_uint64) for n in ("nnz", "payload_bytes", "device_bytes", "stream_bytes")]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_SIGS = {
    "qw_abi_version": (C.c_int, []),
    "qw_strerror": (C.c_char_p, [C.c_int]),
    "qw_last_error": (C.c_char_p, []),
    "qw_host_quantize": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_double,
                                   C.c_uint32, C.c_double, C.c_uint32, C.POINTER(C.c_void_p)]),
    "qw_device_quantize": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_double, C.c_uint32,
                                     C.c_double, C.c_int, C.POINTER(C.c_void_p)]),
    "qw_host_from_view": (C.c_int, [C.POINTER(LayerView), C.POINTER(C.c_void_p)]),
    "qw_host_view": (C.c_int, [C.c_void_p, C.POINTER(LayerView)]),
    "qw_host_free": (None, [C.c_void_p]),
    "qw_host_write": (C.c_int, [C.c_void_p, C.c_char_p]),
    "qw_host_read": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "qw_host_shard_rows": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]),
    "qw_host_shard_tiles": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p),
                                      C.POINTER(C.c_uint32)]),
    "qw_validate_layer": (C.c_int, [C.POINTER(LayerView)]),
    "qw_payload_bytes": (C.c_uint64, [C.POINTER(LayerView)]),
    "qw_layer_view_info": (C.c_int, [C.POINTER(LayerView), C.POINTER(LayerInfo)]),
    "qw_synth_gaussian": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p]),
    "qw_plant_outliers": (C.c_int, [C.c_void_p, C.c_uint64, C.c_double, C.c_float, C.c_uint64]),
    "qw_synth_calibration": (C.c_int, [C.c_uint32, C.c_uint64, C.c_void_p]),
    "qw_synth_activation": (C.c_int, [C.c_uint32, C.c_uint64, C.c_void_p]),
    "qw_layer_upload": (C.c_int, [C.POINTER(LayerView), C.c_int, C.POINTER(C.c_void_p)]),
    "qw_layer_upload_ex": (C.c_int, [C.POINTER(LayerView), C.c_int, C.c_uint32, C.POINTER(C.c_void_p)]),
    "qw_layer_uses_tensor_core": (C.c_int, [C.c_void_p]),
    "qw_layer_upload_qwl": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int, C.c_uint32, C.POINTER(C.c_void_p)]),
    "qw_layer_load": (C.c_int, [C.c_char_p, C.c_int, C.c_uint32, C.POINTER(C.c_void_p)]),
    "qw_layer_free": (C.c_int, [C.c_void_p]),
    "qw_layer_get_info": (C.c_int, [C.c_void_p, C.POINTER(LayerInfo)]),
    "qw_workspace_create": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]),
    "qw_workspace_free": (C.c_int, [C.c_void_p]),
    "qw_matvec": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "qw_matvec_ex": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_uint32]),
    "qw_dequant_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "qw_group_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32, C.POINTER(C.c_void_p)]),
    "qw_group_free": (C.c_int, [C.c_void_p]),
    "qw_group_matvec": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p, C.c_uint32]),
    "qw_group_matvec_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p), C.c_void_p,
                                        C.c_uint32]),
    "qw_layer_set_prefetch": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_uint32]),
    "qw_chain_create": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p)]),
    "qw_chain_run": (C.c_int, [C.c_void_p, C.c_void_p]),
    "qw_chain_free": (C.c_int, [C.c_void_p]),
    "qw_debug_chain_watch": (C.c_int, [C.POINTER(C.c_uint32), C.c_uint32]),
    "qw_debug_chain_timeline": (C.c_int, [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_uint64]),
    "qw_group_set_prefetch": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_uint32]),
    "qw_matvec_pdl": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p,
                                C.c_void_p]),
    "qw_matvec_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p,
                                 C.c_void_p, C.c_void_p]),
    "qw_matvec_host_ex": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]),
    "qw_dequant": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "qw_unpack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                            C.c_void_p]),
    "qw_layer_clone": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "qw_debug_timeline": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32,
                                      C.c_uint32, C.c_void_p]),
    "qw_debug_timeline_events": (C.c_int, []),
    "qw_debug_group_timeline": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p,
                                          C.c_uint32, C.c_void_p]),
    "qw_debug_gemm_timeline": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p,
                                         C.c_void_p]),
    "qw_launches_per_matvec": (C.c_int, [C.c_void_p, C.c_uint32]),
    "qw_launches_per_matvec_ex": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32]),
    "qw_matvec_push": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p),
                                 C.POINTER(C.c_void_p), C.c_uint32, C.c_void_p, C.c_uint32]),
    "qw_push_arrivals": (C.c_int, [C.c_void_p]),
    "qw_peer_wait": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p]),
    "qw_peer_reduce": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]),
    "qw_ipc_handle": (C.c_int, [C.c_void_p, C.c_char_p]),
    "qw_ipc_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "qw_ipc_close": (C.c_int, [C.c_void_p]),
    "qw_matvec_uses_gemm": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32]),
    "qw_debug_gemm_shift": (C.c_int, [C.c_void_p, C.POINTER(C.c_int)]),
    "qw_debug_knob": (C.c_uint32, [C.c_char_p, C.c_uint32]),
}

_lib = None


def lib_path() -> Path:
    return LIB_PATH


def lib() -> C.CDLL:
    """Load libqweight_b200.so (loudly: no silent fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise QWeightError(QW_ERR_UNSUPPORTED,
                               f"{LIB_PATH} is missing; run __graft_entry__.build() or "
                               "`python -m paper_2311_16442_b200.build`")
        handle = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.qw_abi_version() != 1:
            raise QWeightError(QW_ERR_UNSUPPORTED, "libqweight_b200 ABI version mismatch")
        _lib = handle
    return _lib


def check(status: int) -> None:
    if status != QW_OK:
        L = lib()
        detail = L.qw_last_error().decode(errors="replace")
        raise QWeightError(status, f"{L.qw_strerror(status).decode()}: {detail}")


def exported_symbols() -> list[str]:
    return list(_SIGS)
