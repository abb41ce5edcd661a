#!/usr/bin/env python3
"""Regenerate tests/golden/ from the UNMODIFIED reference library.

Run in the build container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py

Writes
  tile_zero.bin / tile_ramp.bin / tile_meta.bin   22-byte pack_tile wire images
      (reference test_bitpack.cpp:30-60, acceptance.cpp:155-185)
  layer_<name>.qwl    layers quantized AND serialized by the reference
                      (quantize_layer + write_packed_layer)
  layer_<name>.npz    x, y_oracle (reference matvec_oracle), y_f64
                      (matvec_reference_f64), sha256 of reconstruct_dense and
                      of unpack_layer's code arrays
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

import oracle  # noqa: E402

# name, rows, cols, alpha, group2, ratio, seed, planted-outlier ratio
LAYERS = [
    ("pads_tails", 20, 80, 0.25, 16, 0.002, 1, 0.0),
    ("tail4_heavy", 24, 160, 0.5, 16, 0.005, 2, 0.0),
    ("pure2", 9, 96, 0.0, 16, 0.0, 7, 0.0),
    ("pure4", 9, 96, 1.0, 16, 0.0, 8, 0.0),
    ("odd_g2", 37, 256, 0.25, 5, 0.01, 13, 0.0),
    ("g2_128", 130, 512, 0.25, 128, 0.002, 17, 0.0),
    ("planted", 64, 512, 0.25, 16, 0.002, 21, 0.01),
]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    oracle.build()
    # golden tiles (A.4)
    z48, z16, z3 = np.zeros(48, np.uint8), np.zeros(16, np.uint8), np.zeros(3, np.uint8)
    (HERE / "tile_zero.bin").write_bytes(oracle.ref_pack_tile(z48, z16, z3, z3))
    ramp2 = (np.arange(48) % 4).astype(np.uint8)
    ramp4 = np.arange(16, dtype=np.uint8)
    (HERE / "tile_ramp.bin").write_bytes(oracle.ref_pack_tile(ramp2, ramp4, z3, z3))
    (HERE / "tile_meta.bin").write_bytes(
        oracle.ref_pack_tile(z48, z16, np.array([1, 2, 3], np.uint8), np.array([9, 5, 3], np.uint8)))
    for name, rows, cols, alpha, g2, ratio, seed, planted in LAYERS:
        w = oracle.ref_synth_gaussian(rows, cols, seed)
        if planted:
            oracle.ref_plant_outliers(w, planted, 8.0, seed)
        h = oracle.ref_synth_calibration(cols, seed)
        ref = oracle.RefLayer.quantize(w, h, alpha, g2, ratio)
        ref.write(HERE / f"layer_{name}.qwl")
        x = oracle.ref_synth_activation(cols, seed + 100)
        y, _ = ref.matvec_oracle(x)
        un = ref.unpack()
        np.savez_compressed(
            HERE / f"layer_{name}.npz", x=x, y_oracle=y, y_f64=ref.matvec_f64(x),
            recon_sha=sha(ref.reconstruct_dense()),
            unpack_sha=np.array([sha(un[k]) for k in ("codes2", "zeros2", "scodes", "codes4")]),
            w_sha=sha(w), payload=ref.payload_bytes(),
            params=np.array([rows, cols, alpha, g2, ratio, seed, planted], np.float64))
        print(name, rows, cols, "payload", ref.payload_bytes())


if __name__ == "__main__":
    main()
