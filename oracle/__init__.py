"""oracle -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

Python handles to
  * libqw_oracle.so  -- plain-C restatement of the reference hot path
                        (oracle/qw_oracle.c), and
  * libqweight_ref.so -- the unmodified reference library compiled from its
                        own sources (oracle/Makefile), behind ref_capi.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this package.  Nothing under paper_2311_16442_b200/ may.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libqw_oracle.so"
REF_SO = HERE / "_ref" / "libqweight_ref.so"


def build() -> None:
    """Compile the checkers (the reference part only where its sources exist)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def _view_type():
    from paper_2311_16442_b200._native import LayerView
    return LayerView


_oracle = None
_ref = None


def oracle_lib() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not ORACLE_SO.exists():
            build()
        L = C.CDLL(str(ORACLE_SO), mode=os.RTLD_LOCAL)
        V = C.POINTER(_view_type())
        L.qo_f16_to_f32.restype, L.qo_f16_to_f32.argtypes = C.c_float, [C.c_uint16]
        L.qo_f32_to_f16.restype, L.qo_f32_to_f16.argtypes = C.c_uint16, [C.c_float]
        L.qo_unpack.restype = None
        L.qo_unpack.argtypes = [V] + [C.c_void_p] * 4
        L.qo_reconstruct_dense.restype, L.qo_reconstruct_dense.argtypes = None, [V, C.c_void_p]
        L.qo_permute.restype, L.qo_permute.argtypes = C.c_int, [V, C.c_void_p, C.c_void_p]
        L.qo_matvec_oracle.restype, L.qo_matvec_oracle.argtypes = C.c_int, [V, C.c_void_p, C.c_void_p]
        L.qo_matvec_f64.restype, L.qo_matvec_f64.argtypes = C.c_int, [V, C.c_void_p, C.c_void_p]
        L.qo_matvec_oracle_rows.restype = C.c_int
        L.qo_matvec_oracle_rows.argtypes = [V, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p]
        L.qo_payload_bytes.restype, L.qo_payload_bytes.argtypes = C.c_uint64, [V]
        L.qo_pack_tile.restype = None
        L.qo_pack_tile.argtypes = [C.c_void_p] * 5
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return REF_SO.exists()


def ref_lib() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        L = C.CDLL(str(REF_SO), mode=os.RTLD_LOCAL)
        V = C.POINTER(_view_type())
        P = C.POINTER(C.c_void_p)
        sig = {
            "qwref_last_error": (C.c_char_p, []),
            "qwref_quantize": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_double,
                                         C.c_uint32, C.c_double, P]),
            "qwref_from_view": (C.c_int, [V, P]),
            "qwref_view": (C.c_int, [C.c_void_p, V]),
            "qwref_free": (None, [C.c_void_p]),
            "qwref_matvec_oracle": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                              C.POINTER(C.c_uint64)]),
            "qwref_matvec_pipelined": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32,
                                                 C.c_void_p, C.POINTER(C.c_uint64)]),
            "qwref_matvec_f64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
            "qwref_reconstruct": (C.c_int, [C.c_void_p, C.c_void_p]),
            "qwref_unpack": (C.c_int, [C.c_void_p] * 5),
            "qwref_payload_bytes": (C.c_uint64, [C.c_void_p]),
            "qwref_write": (C.c_int, [C.c_void_p, C.c_char_p]),
            "qwref_read": (C.c_int, [C.c_char_p, P]),
            "qwref_synth_gaussian": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p]),
            "qwref_plant_outliers": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_double,
                                               C.c_float, C.c_uint64]),
            "qwref_synth_calibration": (C.c_int, [C.c_uint32, C.c_uint64, C.c_void_p]),
            "qwref_synth_activation": (C.c_int, [C.c_uint32, C.c_uint64, C.c_void_p]),
            "qwref_pack_tile": (C.c_int, [C.c_void_p] * 5),
            "qwref_f32_to_f16": (C.c_uint16, [C.c_float]),
            "qwref_f16_to_f32": (C.c_float, [C.c_uint16]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _ref = L
    return _ref


def _ref_check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError("reference: " + ref_lib().qwref_last_error().decode())


# ------------------------------------------------------------ C oracle calls
def _geom(layer):
    c = layer.cfg
    return c.rows, c.n2_padded, c.padded_cols, 3 * c.triples, c.n4


def unpack(layer) -> dict:
    rows, n2p, pc, gpr, n4 = _geom(layer)
    out = {"codes2": np.zeros((rows, n2p), np.uint8), "zeros2": np.zeros((rows, gpr), np.uint8),
           "scodes": np.zeros((rows, gpr), np.uint8), "codes4": np.zeros((rows, n4), np.uint8)}
    oracle_lib().qo_unpack(C.byref(layer.view()), *(a.ctypes.data for a in out.values()))
    return out


def reconstruct_dense(layer) -> np.ndarray:
    rows, _, pc, _, _ = _geom(layer)
    w = np.zeros((rows, pc), np.float32)
    oracle_lib().qo_reconstruct_dense(C.byref(layer.view()), w.ctypes.data)
    return w


def matvec_oracle(layer, x) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    y = np.zeros(layer.cfg.rows, np.float32)
    if oracle_lib().qo_matvec_oracle(C.byref(layer.view()), x.ctypes.data, y.ctypes.data) != 0:
        raise ValueError("matvec: non-finite activation")
    return y


def matvec_f64(layer, x) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    y = np.zeros(layer.cfg.rows, np.float64)
    if oracle_lib().qo_matvec_f64(C.byref(layer.view()), x.ctypes.data, y.ctypes.data) != 0:
        raise ValueError("matvec: non-finite activation")
    return y


def matvec_oracle_rows(layer, x, r0: int, r1: int) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    y = np.zeros(r1 - r0, np.float32)
    oracle_lib().qo_matvec_oracle_rows(C.byref(layer.view()), x.ctypes.data, r0, r1, y.ctypes.data)
    return y


def payload_bytes(layer) -> int:
    return int(oracle_lib().qo_payload_bytes(C.byref(layer.view())))


def pack_tile(c2, c4, z, s) -> bytes:
    arrs = [np.ascontiguousarray(a, np.uint8) for a in (c2, c4, z, s)]
    out = np.zeros(22, np.uint8)
    oracle_lib().qo_pack_tile(*(a.ctypes.data for a in arrs), out.ctypes.data)
    return out.tobytes()


# ------------------------------------------------------------ reference calls
class RefLayer:
    """A reference qweight::PackedLayer owned by libqweight_ref.so."""

    def __init__(self, handle: C.c_void_p):
        self.h = handle

    @classmethod
    def quantize(cls, w, h, alpha=0.25, group2=16, ratio=0.002) -> "RefLayer":
        w = np.ascontiguousarray(w, np.float32)
        h = np.ascontiguousarray(h, np.float32)
        out = C.c_void_p()
        _ref_check(ref_lib().qwref_quantize(w.ctypes.data, w.shape[0], w.shape[1], h.ctypes.data,
                                            alpha, group2, ratio, C.byref(out)))
        return cls(out)

    @classmethod
    def from_layer(cls, layer) -> "RefLayer":
        out = C.c_void_p()
        _ref_check(ref_lib().qwref_from_view(C.byref(layer.view()), C.byref(out)))
        return cls(out)

    @classmethod
    def read(cls, path) -> "RefLayer":
        out = C.c_void_p()
        _ref_check(ref_lib().qwref_read(str(path).encode(), C.byref(out)))
        return cls(out)

    def to_layer(self):
        from paper_2311_16442_b200.layer import PackedLayer
        V = _view_type()
        v = V()
        ref_lib().qwref_view(self.h, C.byref(v))
        return PackedLayer.from_view(v)

    def matvec_oracle(self, x):
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros(self.rows(), np.float32)
        ns = C.c_uint64()
        _ref_check(ref_lib().qwref_matvec_oracle(self.h, x.ctypes.data, x.size, y.ctypes.data,
                                                 C.byref(ns)))
        return y, ns.value

    def matvec_pipelined(self, x, workers):
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros(self.rows(), np.float32)
        ns = C.c_uint64()
        _ref_check(ref_lib().qwref_matvec_pipelined(self.h, x.ctypes.data, x.size, workers,
                                                    y.ctypes.data, C.byref(ns)))
        return y, ns.value

    def matvec_f64(self, x):
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros(self.rows(), np.float64)
        _ref_check(ref_lib().qwref_matvec_f64(self.h, x.ctypes.data, x.size, y.ctypes.data))
        return y

    def reconstruct_dense(self):
        v = self._view()
        w = np.zeros((v.rows, v.cols - v.n4 + v.pad2 + v.n4), np.float32)
        _ref_check(ref_lib().qwref_reconstruct(self.h, w.ctypes.data))
        return w

    def unpack(self):
        v = self._view()
        n2p = v.cols - v.n4 + v.pad2
        gpr = 3 * (n2p // 48)
        out = {"codes2": np.zeros((v.rows, n2p), np.uint8), "zeros2": np.zeros((v.rows, gpr), np.uint8),
               "scodes": np.zeros((v.rows, gpr), np.uint8), "codes4": np.zeros((v.rows, v.n4), np.uint8)}
        _ref_check(ref_lib().qwref_unpack(self.h, *(a.ctypes.data for a in out.values())))
        return out

    def payload_bytes(self) -> int:
        return int(ref_lib().qwref_payload_bytes(self.h))

    def write(self, path) -> None:
        _ref_check(ref_lib().qwref_write(self.h, str(path).encode()))

    def _view(self):
        v = _view_type()()
        ref_lib().qwref_view(self.h, C.byref(v))
        return v

    def rows(self) -> int:
        return self._view().rows

    def __del__(self):
        try:
            if self.h:
                ref_lib().qwref_free(self.h)
        except Exception:
            pass


def ref_synth_gaussian(rows, cols, seed):
    out = np.zeros((rows, cols), np.float32)
    _ref_check(ref_lib().qwref_synth_gaussian(rows, cols, seed, out.ctypes.data))
    return out


def ref_synth_calibration(cols, seed):
    out = np.zeros(cols, np.float32)
    _ref_check(ref_lib().qwref_synth_calibration(cols, seed, out.ctypes.data))
    return out


def ref_synth_activation(cols, seed):
    out = np.zeros(cols, np.float32)
    _ref_check(ref_lib().qwref_synth_activation(cols, seed, out.ctypes.data))
    return out


def ref_plant_outliers(w, ratio, scale, seed):
    _ref_check(ref_lib().qwref_plant_outliers(w.ctypes.data, w.shape[0], w.shape[1], ratio, scale,
                                              seed))


def ref_pack_tile(c2, c4, z, s) -> bytes:
    arrs = [np.ascontiguousarray(a, np.uint8) for a in (c2, c4, z, s)]
    out = np.zeros(22, np.uint8)
    _ref_check(ref_lib().qwref_pack_tile(*(a.ctypes.data for a in arrs), out.ctypes.data))
    return out.tobytes()
