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

from .engine import DeviceLayer
from .layer import PackedLayer

_REGISTRY: dict[int, DeviceLayer] = {}
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
        ys.append(dl.matvec(xb[c0:c0 + 16]))
    return torch.cat(ys, 0).reshape(*lead, dl.rows)


@quantized_linear.register_fake
def _(x: torch.Tensor, layer_id: int) -> torch.Tensor:
    return x.new_empty((*x.shape[:-1], _REGISTRY[layer_id].rows))


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
        _REGISTRY.pop(getattr(self, "layer_id", None), None)
