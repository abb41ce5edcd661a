"""paper_2311_16442_b200 -- B200-native quantized linear layer of arXiv 2311.16442.

y = W_q x with range-aware mixed 2/4-bit groups, 2-order group scales and
fp16 sparse outliers, behind the reference's host API.
"""
from ._native import QWeightError, exported_symbols, lib
from .layer import (PAD, LayerConfig, PackedLayer, payload_bytes, permute, plant_outliers,
                    quantize_layer, quantize_layer_gpu, read_packed_layer, shard_rows, shard_tiles,
                    synth_activation, synth_calibration, synth_gaussian, synth_layer,
                    validate_layer, write_packed_layer)

__all__ = [
    "QWeightError", "LayerConfig", "PackedLayer", "PAD", "lib", "exported_symbols",
    "payload_bytes", "permute", "plant_outliers", "quantize_layer", "quantize_layer_gpu", "read_packed_layer",
    "shard_rows", "shard_tiles", "synth_activation", "synth_calibration", "synth_gaussian",
    "synth_layer", "validate_layer", "write_packed_layer", "DeviceLayer", "Workspace",
    "MatvecResult", "upload", "LayerGroup", "DecodeChain",
]


def __getattr__(name):  # the engine imports torch lazily
    if name in ("DeviceLayer", "Workspace", "MatvecResult", "upload", "default_workspace", "LayerGroup",
                "DecodeChain"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)
