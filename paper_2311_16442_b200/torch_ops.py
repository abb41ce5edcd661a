"""PyTorch integration: the quantized linear as a
torch.library custom op and an nn.Module, so a decode step written in PyTorch
calls the B200 kernels (K2 / K2m at batch 1, K4 at 2..16) like any other op --
eagerly, inside torch.cuda.graph capture, and through torch.compile (the op
has a fake implementation for shape propagation and is opaque to the
compiler: the kernel is ours, not generated).

    lin = QuantizedLinear(packed_layer)          # upload once
    y = lin(x)                                   # x: [..., in] cuda fp32 -> [..., out]
    y = torch.ops.qweight_b200.quantized_linear(x, lin.layer_id)

The reference has no model layer; this is the host-side hook a
model would use.
"""
from __future__ import annotations

import itertools

import torch

from .engine import DeviceLayer, LayerGroup
from .layer import PackedLayer

_REGISTRY: dict[int, DeviceLayer] = {}
_GROUPS: dict[int, LayerGroup] = {}
_IDS = itertools.count(1)


@torch.library.custom_op("qweight_b200::quantized_linear", mutates_args=())
def quantized_linear(x: torch.Tensor, layer_id: int) -> torch.Tensor:
    """y = W_q x for the registered layer; x [..., cols] fp32 on the layer's GPU."""
    dl = _REGISTRY[layer_id]
    lead = x.shape[:-1]
    xb = x.reshape(-1, x.shape[-1]).contiguous()
    if xb.shape[0] == 0:
        return x.new_empty((*lead, dl.rows))
    ys = []
    for c0 in range(0, xb.shape[0], 16):  # the batched path takes at most 16 columns per call
        # programmatic dependent launch: the weight stream starts under the
        # previous kernel on the stream; x is read after it completes
        ys.append(dl.matvec(xb[c0:c0 + 16], pdl=True))
    return torch.cat(ys, 0).reshape(*lead, dl.rows)


@quantized_linear.register_fake
def _(x: torch.Tensor, layer_id: int) -> torch.Tensor:
    return x.new_empty((*x.shape[:-1], _REGISTRY[layer_id].rows))


@torch.library.custom_op("qweight_b200::quantized_linear_group", mutates_args=())
def quantized_linear_group(x: torch.Tensor, group_id: int) -> list[torch.Tensor]:
    """[W_i x for each layer of the registered group]: one fused launch for all
    the layers (q/k/v, gate/up: one dependency wait, one activation staging)
    per up to 8 / n columns while the batched policy keeps the batch-1
    kernel; larger batches run each layer's K4 GEMM."""
    grp = _GROUPS[group_id]
    lead = x.shape[:-1]
    xb = x.reshape(-1, x.shape[-1]).contiguous()
    if xb.shape[0] == 1:
        return [y.reshape(*lead, y.shape[0]) for y in grp.matvec(xb.reshape(-1), pdl=True)]
    if all(_REGISTRY[lid].batched_path(xb.shape[0]) == "columns" for lid in grp.layer_ids):
        # the batch-1 kernel: up to 8 / n columns of every layer per launch
        return [y.reshape(*lead, y.shape[-1]) for y in grp.matvec(xb, pdl=True)]
    return [quantized_linear(x, lid) for lid in grp.layer_ids]  # each layer's K4 GEMM


@quantized_linear_group.register_fake
def _(x: torch.Tensor, group_id: int) -> list[torch.Tensor]:
    return [x.new_empty((*x.shape[:-1], _REGISTRY[lid].rows)) for lid in _GROUPS[group_id].layer_ids]


class QuantizedLinearGroup(torch.nn.Module):
    """Several nn.Linear-shaped layers that read the same input (q/k/v,
    gate/up), computed by one fused launch at batch 1.  forward(x) returns
    the tuple of outputs."""

    def __init__(self, layers: list, device: int = 0, kernel: str = "auto"):
        super().__init__()
        self.members = torch.nn.ModuleList(QuantizedLinear(l, device, kernel) for l in layers)
        self.group = LayerGroup([m.dl for m in self.members])
        self.group.layer_ids = [m.layer_id for m in self.members]
        self.group_id = next(_IDS)
        _GROUPS[self.group_id] = self.group

    def forward(self, x: torch.Tensor):
        return tuple(torch.ops.qweight_b200.quantized_linear_group(x, self.group_id))

    def __del__(self):
        if _GROUPS is not None:
            _GROUPS.pop(getattr(self, "group_id", None), None)


class QuantizedLinear(torch.nn.Module):
    """nn.Linear-shaped module over one uploaded mixed 2/4-bit layer
    (no bias: the reference layer has none)."""

    def __init__(self, layer: PackedLayer | DeviceLayer, device: int = 0, kernel: str = "auto"):
        super().__init__()
        self.dl = layer if isinstance(layer, DeviceLayer) else DeviceLayer(layer, device, kernel=kernel)
        self.layer_id = next(_IDS)
        _REGISTRY[self.layer_id] = self.dl
        self.in_features, self.out_features = self.dl.cols, self.dl.rows

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return torch.ops.qweight_b200.quantized_linear(x, self.layer_id)

    def extra_repr(self) -> str:
        return (f"in_features={self.in_features}, out_features={self.out_features}, "
                f"kernel={'K2m' if self.dl.uses_tensor_core else 'K2'}")

    def __del__(self):
        if _REGISTRY is not None:  # (interpreter shutdown clears module globals)
            _REGISTRY.pop(getattr(self, "layer_id", None), None)
