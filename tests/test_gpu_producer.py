"""quantize_layer on the GPU: qw_device_quantize must
produce the same packed layer as the CPU producer -- which tests/test_producer.py
pins byte for byte to the reference's quantize_layer -- compared as the
serialized QWL1 bytes (every stream, the plan, the CSR, the 2-order params).
Covers the tie-break order of the global top-K (planted outliers with equal
magnitudes), dense outlier budgets, pads, odd group2, alpha 0 / 1 and a
Llama-2-7B shape."""
import numpy as np
import pytest

import paper_2311_16442_b200 as qw

pytestmark = pytest.mark.gpu


def qwl_bytes(layer, tmp_path, name):
    p = tmp_path / f"{name}.qwl"
    qw.write_packed_layer(layer, str(p))
    return p.read_bytes()


@pytest.mark.parametrize("rows,cols,alpha,g2,ratio,planted", [
    (64, 512, 0.25, 16, 0.002, False),
    (37, 160, 0.5, 16, 0.01, False),     # pads (n2 % 48 != 0), tails, odd rows
    (96, 1024, 0.0, 5, 0.005, False),    # pure 2-bit, odd group2
    (48, 256, 1.0, 16, 0.0, False),      # pure 4-bit, no outliers
    (128, 768, 0.25, 128, 0.02, True),   # planted equal-magnitude outliers: the tie-break
    (4096, 4096, 0.25, 16, 0.002, False),  # Llama-2-7B q_proj
])
def test_device_producer_is_bit_identical(rows, cols, alpha, g2, ratio, planted, tmp_path):
    w = qw.synth_gaussian(rows, cols, rows + cols)
    if planted:
        qw.plant_outliers(w, 0.01, 8.0, 5)
        w[3, 10] = w[5, 20] = w[7, 30] = 50.0  # exact ties in |w|
    h = qw.synth_calibration(cols, 9)
    cpu = qw.quantize_layer(w, h, alpha, g2, ratio)
    gpu = qw.quantize_layer_gpu(w, h, alpha, g2, ratio)
    assert qwl_bytes(gpu, tmp_path, "gpu") == qwl_bytes(cpu, tmp_path, "cpu")


def test_device_producer_rejects_bad_input():
    w = qw.synth_gaussian(16, 64, 1)
    h = qw.synth_calibration(64, 1)
    bad = w.copy()
    bad[2, 3] = np.nan
    with pytest.raises(qw.QWeightError):
        qw.quantize_layer_gpu(bad, h)
    with pytest.raises(qw.QWeightError):
        qw.quantize_layer_gpu(w, -h)
    with pytest.raises(qw.QWeightError):
        qw.quantize_layer_gpu(w, h, alpha=1.5)
