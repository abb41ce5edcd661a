"""B200 engine: device-resident layers and the quantized linear forward.

Mirrors the reference engine API (engine.hpp:19-70) on the GPU:

  reference                          here
  ---------------------------------  ------------------------------------------
  reconstruct_dense(layer)           DeviceLayer.reconstruct_dense()  (bit-exact)
  unpack_layer(layer)                DeviceLayer.unpack()             (bit-exact)
  matvec_oracle / matvec_pipelined   DeviceLayer.matvec(x)           (1e-2 rel)
  MatvecResult{y, stage_ns, wall_ns} matvec_checked(x) -> MatvecResult

PyTorch only supplies device memory and streams; every kernel is ours
(libqweight_b200.so).  A missing GPU raises QWeightError -- there is no CPU
path.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from ._native import LayerInfo, QWeightError, check, lib
from .layer import PackedLayer

try:  # torch is plumbing (device buffers, streams, events)
    import torch
except Exception:  # pragma: no cover
    torch = None


def _stream_handle(stream=None) -> int:
    if torch is None:
        return 0
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


class Workspace:
    """Per-stream activation scratch (qw_workspace_create)."""

    def __init__(self, device: int = 0, max_cols: int = 65536, max_batch: int = 16):
        self.device = device
        self.max_cols, self.max_batch = max_cols, max_batch
        self._h = C.c_void_p()
        check(lib().qw_workspace_create(device, max_cols, max_batch, C.byref(self._h)))

    def close(self):
        if self._h:
            lib().qw_workspace_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ws: dict = {}


def default_workspace(device: int) -> Workspace:
    ws = _default_ws.get(device)
    if ws is None:
        ws = _default_ws[device] = Workspace(device)
    return ws


@dataclass
class MatvecResult:
    """MatvecResult (engine.hpp:19-23): y plus timing.  stage_ns: [0] the
    host->device copy of x, [1] [2] 0 (the 2-order scales and the decode are
    fused into the kernel), [3] the fused kernel (CUDA events)."""
    y: np.ndarray
    stage_ns: list = field(default_factory=lambda: [0, 0, 0, 0])
    wall_ns: int = 0


class DeviceLayer:
    """A packed layer uploaded to HBM in the 4-row device format."""

    def __init__(self, layer: PackedLayer | None, device: int = 0, _handle=None, kernel: str = "auto"):
        """kernel (batch-1 path): "auto" -- the SIMT GEMV K2 except where the
        warp-MMA kernel K2m measured faster (dense outliers that overflow K2's
        CSR stage, very wide layers; qweight_b200.h); "simt" / "mma" force one."""
        if kernel not in ("auto", "simt", "mma"):
            raise ValueError("kernel must be 'auto', 'simt' or 'mma'")
        self.device = device
        self.kernel = kernel
        self._h = C.c_void_p()
        if _handle is not None:
            self._h = _handle
        else:
            self.layer_cfg = layer.cfg
            flags = {"auto": 0, "mma": 1, "simt": 2}[kernel]
            check(lib().qw_layer_upload_ex(C.byref(layer.view()), device, flags, C.byref(self._h)))
        inf = LayerInfo()
        check(lib().qw_layer_get_info(self._h, C.byref(inf)))
        self.info = inf.as_dict()

    @property
    def uses_tensor_core(self) -> bool:
        """True when batch-1 calls run the warp-MMA kernel K2m."""
        return bool(lib().qw_layer_uses_tensor_core(self._h))

    @property
    def rows(self): return self.info["rows"]
    @property
    def cols(self): return self.info["cols"]
    @property
    def padded_cols(self): return self.info["padded_cols"]

    def close(self):
        if self._h:
            lib().qw_layer_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- forward
    def matvec(self, x, out=None, workspace: Workspace | None = None, stream=None,
               pdl: bool = False, x_independent: bool = False, batched: str = "auto"):
        """y = W_q x on the GPU.  x: torch cuda fp32 [cols] or [batch, cols]
        in original channel order.  Returns fp32 [rows] / [batch, rows].
        pdl: programmatic dependent launch (weights stream under the previous
        kernel); x_independent: x was not produced by the previous kernel on
        the stream, so no dependency wait is needed before reading it."""
        if torch is None:
            raise QWeightError(3, "torch is required for device tensors")
        squeeze = x.dim() == 1
        xb = x.reshape(1, -1) if squeeze else x
        if xb.dtype != torch.float32 or not xb.is_cuda or not xb.is_contiguous():
            raise QWeightError(1, "matvec: x must be a contiguous cuda float32 tensor")
        if xb.device.index != self.device:
            raise QWeightError(1, f"matvec: x is on cuda:{xb.device.index}, the layer on cuda:{self.device}")
        batch = xb.shape[0]
        if xb.shape[1] != self.cols:
            raise QWeightError(1, "matvec: activation length != input channels")
        if out is None:
            out = torch.empty((batch, self.rows), dtype=torch.float32, device=xb.device)
        elif (out.dtype != torch.float32 or not out.is_cuda or not out.is_contiguous() or
              out.numel() != batch * self.rows or out.device != xb.device):
            # the kernel writes y[n * rows + row] from out.data_ptr(): anything
            # but a contiguous fp32 [batch, rows] buffer on x's device is wrong
            raise QWeightError(1, "matvec: out must be a contiguous cuda float32 tensor of batch * rows "
                                  "elements on the activation's device")
        ws = workspace or default_workspace(self.device)
        # batched: "auto" (K4 from 6 columns, the batch-1 kernel over the
        # columns below), "gemm" (force the tcgen05 GEMM K4), "columns"
        # (force the batch-1 kernel, up to 8 columns per launch)
        flags = (1 if pdl else 0) | (2 if x_independent else 0) | {"auto": 0, "gemm": 4, "columns": 8}[batched]
        check(lib().qw_matvec_ex(self._h, C.c_void_p(xb.data_ptr()), batch,
                                 C.c_void_p(out.data_ptr()), ws._h,
                                 C.c_void_p(_stream_handle(stream)), flags))
        return out.reshape(-1) if squeeze else out

    def matvec_checked(self, x: np.ndarray, workspace: Workspace | None = None) -> MatvecResult:
        """Host buffers in and out, with the reference's activation checks
        (engine.cpp:124-132): wrong length or a non-finite value raises."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        batch = 1 if x.ndim == 1 else x.shape[0]
        y = np.empty((batch, self.rows), dtype=np.float32)
        ws = workspace or default_workspace(self.device)
        stages = (C.c_uint64 * 4)()
        t0 = time.perf_counter_ns()
        check(lib().qw_matvec_host_ex(self._h, x.ctypes.data, x.size, batch, y.ctypes.data, ws._h,
                                      C.c_void_p(_stream_handle()), stages))
        wall = time.perf_counter_ns() - t0
        # stage_ns: [x copy, 0, 0, fused kernel] (device event times; the
        # scale and decode stages are fused into the kernel)
        return MatvecResult(y=y.reshape(-1) if x.ndim == 1 else y, wall_ns=wall, stage_ns=list(stages))

    # ------------------------------------------------------------ bit-exact
    def reconstruct_dense(self, stream=None):
        """reconstruct_dense (engine.hpp:26): rows x padded_cols fp32, permuted."""
        w = torch.empty((self.rows, self.padded_cols), dtype=torch.float32,
                        device=f"cuda:{self.device}")
        check(lib().qw_dequant(self._h, C.c_void_p(w.data_ptr()), C.c_void_p(_stream_handle(stream))))
        return w

    def unpack(self, stream=None) -> dict:
        """unpack_layer codes (bitpack.hpp:128): codes2, zeros2, scodes, codes4."""
        inf, dev = self.info, f"cuda:{self.device}"
        gpr = 3 * inf["triples"]
        codes2 = torch.empty((self.rows, max(inf["n2_padded"], 1)), dtype=torch.uint8, device=dev)
        zeros2 = torch.empty((self.rows, max(gpr, 1)), dtype=torch.uint8, device=dev)
        scodes = torch.empty((self.rows, max(gpr, 1)), dtype=torch.uint8, device=dev)
        codes4 = torch.empty((self.rows, max(inf["n4"], 1)), dtype=torch.uint8, device=dev)
        check(lib().qw_unpack(self._h, C.c_void_p(codes2.data_ptr()), C.c_void_p(zeros2.data_ptr()),
                              C.c_void_p(scodes.data_ptr()), C.c_void_p(codes4.data_ptr()),
                              C.c_void_p(_stream_handle(stream))))
        return {"codes2": codes2[:, :inf["n2_padded"]], "zeros2": zeros2[:, :gpr],
                "scodes": scodes[:, :gpr], "codes4": codes4[:, :inf["n4"]]}

    @classmethod
    def load(cls, path, device: int = 0, kernel: str = "auto") -> "DeviceLayer":
        """A QWL1 file (the reference's container, container.cpp:321-471)
        straight to HBM (qw_layer_load): parse, CRC, validate, repack, copy."""
        h = C.c_void_p()
        flags = {"auto": 0, "mma": 1, "simt": 2}[kernel]
        check(lib().qw_layer_load(str(path).encode(), device, flags, C.byref(h)))
        out = cls(None, device, _handle=h, kernel=kernel)
        return out

    @classmethod
    def from_qwl_bytes(cls, data: bytes, device: int = 0, kernel: str = "auto") -> "DeviceLayer":
        """QWL1 bytes in memory (e.g. a memory-mapped cache) -> HBM."""
        h = C.c_void_p()
        buf = (C.c_uint8 * len(data)).from_buffer_copy(data)
        flags = {"auto": 0, "mma": 1, "simt": 2}[kernel]
        check(lib().qw_layer_upload_qwl(buf, len(data), device, flags, C.byref(h)))
        return cls(None, device, _handle=h, kernel=kernel)

    def clone(self) -> "DeviceLayer":
        """Device-to-device copy (distinct HBM buffers, same content)."""
        h = C.c_void_p()
        check(lib().qw_layer_clone(self._h, C.byref(h)))
        out = DeviceLayer(None, self.device, _handle=h, kernel=self.kernel)
        out.layer_cfg = getattr(self, "layer_cfg", None)
        return out

    def set_prefetch(self, next_layers: list["DeviceLayer"]) -> None:
        """Decode chains: launches of this layer also stream `next_layers`'
        weights (the following launch on the stream) into L2.  [] clears."""
        check(lib().qw_layer_set_prefetch(self._h, _handles(next_layers), len(next_layers)))

    def launches_per_matvec(self, batch: int = 1, batched: str = "auto") -> int:
        return int(lib().qw_launches_per_matvec_ex(self._h, batch, {"auto": 0, "gemm": 4, "columns": 8}[batched]))

    def batched_path(self, batch: int, batched: str = "auto") -> str:
        """"gemm" (the tcgen05 GEMM K4) or "columns" (the batch-1 kernel over
        the columns, up to 8 per launch) for a matvec of `batch` columns."""
        r = lib().qw_matvec_uses_gemm(self._h, batch, {"auto": 0, "gemm": 4, "columns": 8}[batched])
        if r < 0:
            check(-r)
        return "gemm" if r else "columns"


class _ChainStep(C.Structure):
    _fields_ = [("layers", C.POINTER(C.c_void_p)), ("n", C.c_uint32), ("x", C.c_void_p),
                ("ys", C.POINTER(C.c_void_p)), ("depends", C.c_uint32)]


class DecodeChain:
    """A fixed sequence of batch-1 launch steps run by ONE persistent kernel
    (qw_chain_*): steps = [(layers, x, ys, depends)], layers of a step share
    geometry and read x (cuda fp32 [cols]); ys[i] receives layers[i] @ x;
    depends: x is the previous step's output (wait for every CTA's stores)."""

    def __init__(self, steps):
        self._keep = []
        arr = (_ChainStep * len(steps))()
        for i, (layers, x, ys, dep) in enumerate(steps):
            if len(layers) != len(ys):
                raise QWeightError(1, "chain: one output per layer")
            for o in ys:
                if o.dtype != torch.float32 or not o.is_cuda or not o.is_contiguous():
                    raise QWeightError(1, "chain: outputs must be contiguous cuda float32")
            if x.dtype != torch.float32 or not x.is_cuda or not x.is_contiguous() or x.numel() != layers[0].cols:
                raise QWeightError(1, "chain: x must be a contiguous cuda float32 [cols]")
            lh = _handles(layers)
            yh = (C.c_void_p * len(ys))(*[o.data_ptr() for o in ys])
            self._keep += [lh, yh, layers, x, ys]
            arr[i] = _ChainStep(C.cast(lh, C.POINTER(C.c_void_p)), len(layers), x.data_ptr(),
                                C.cast(yh, C.POINTER(C.c_void_p)), 1 if dep else 0)
        h = C.c_void_p()
        check(lib().qw_chain_create(C.cast(arr, C.c_void_p), len(steps), C.byref(h)))
        self._h = h
        self.steps = len(steps)

    def run(self, stream=None) -> None:
        check(lib().qw_chain_run(self._h, C.c_void_p(_stream_handle(stream))))

    def close(self):
        if getattr(self, "_h", None):
            lib().qw_chain_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _handles(layers):
    return (C.c_void_p * max(1, len(layers)))(*[d._h.value if hasattr(d._h, "value") else d._h for d in layers])


def upload(layer: PackedLayer, device: int = 0) -> DeviceLayer:
    return DeviceLayer(layer, device)


class LayerGroup:
    """Several DeviceLayers that read the same input (q/k/v, gate/up) computed
    by ONE fused batch-1 launch (qw_group_matvec): the dependency wait and the
    activation staging are paid once.  The layers share their columns,
    channel split and group2; the row counts may differ (GQA: q with k/v)."""

    def __init__(self, layers: list["DeviceLayer"]):
        self.layers = list(layers)
        arr = (C.c_void_p * len(layers))(*[d._h.value if hasattr(d._h, "value") else d._h for d in layers])
        h = C.c_void_p()
        check(lib().qw_group_create(arr, len(layers), C.byref(h)))
        self._h = h
        self.device = layers[0].device

    def close(self):
        if getattr(self, "_h", None):
            lib().qw_group_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_prefetch(self, next_layers: list["DeviceLayer"]) -> None:
        """Decode chains: this group's launches also stream `next_layers`'
        weights into L2 (see DeviceLayer.set_prefetch)."""
        check(lib().qw_group_set_prefetch(self._h, _handles(next_layers), len(next_layers)))

    def matvec(self, x, outs=None, stream=None, pdl: bool = False, x_independent: bool = False):
        """x: cuda fp32 [cols] or [batch, cols] (original order); returns one
        [rows] / [batch, rows] output per layer.  A batch runs up to 8 / n
        columns of every layer per launch (qw_group_matvec_batch)."""
        if x.dtype != torch.float32 or not x.is_cuda or not x.is_contiguous() or x.dim() not in (1, 2):
            raise QWeightError(1, "group matvec: x must be a contiguous 1-D or 2-D cuda float32 tensor")
        if x.shape[-1] != self.layers[0].cols:
            raise QWeightError(1, "group matvec: activation length != input channels")
        batch = 1 if x.dim() == 1 else x.shape[0]
        shape = (lambda r: (r,)) if x.dim() == 1 else (lambda r: (batch, r))
        if outs is None:
            outs = [torch.empty(shape(d.rows), dtype=torch.float32, device=x.device) for d in self.layers]
        for o, d in zip(outs, self.layers):
            if (o.dtype != torch.float32 or not o.is_cuda or not o.is_contiguous() or o.numel() != batch * d.rows
                    or o.device != x.device):
                raise QWeightError(1, "group matvec: every output must be a contiguous cuda float32 tensor of "
                                      "batch * rows elements on the activation's device")
        ptrs = (C.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        flags = (1 if pdl else 0) | (2 if x_independent else 0)
        if x.dim() == 1:
            check(lib().qw_group_matvec(self._h, C.c_void_p(x.data_ptr()), ptrs,
                                        C.c_void_p(_stream_handle(stream)), flags))
        else:
            check(lib().qw_group_matvec_batch(self._h, C.c_void_p(x.data_ptr()), batch, ptrs,
                                              C.c_void_p(_stream_handle(stream)), flags))
        return outs
