"""The host producer (quantize_layer & co, libqweight_b200.so) is
bit-identical to the compiled reference, and the QWL1 container interoperates
both ways (reference test_quantizer.cpp, test_container.cpp, AC2, AC6, AC9)."""
import numpy as np
import pytest

import oracle
import paper_2311_16442_b200 as qw
from paper_2311_16442_b200 import QWeightError

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("rows,cols,seed", [(1, 16, 1), (7, 48, 2), (33, 208, 3), (256, 1024, 4)])
def test_synth_matches_reference(rows, cols, seed):
    assert np.array_equal(qw.synth_gaussian(rows, cols, seed), oracle.ref_synth_gaussian(rows, cols, seed))
    assert np.array_equal(qw.synth_calibration(cols, seed), oracle.ref_synth_calibration(cols, seed))
    assert np.array_equal(qw.synth_activation(cols, seed), oracle.ref_synth_activation(cols, seed))
    w1 = qw.synth_gaussian(rows, cols, seed)
    w2 = w1.copy()
    qw.plant_outliers(w1, 0.05, 8.0, seed)
    oracle.ref_plant_outliers(w2, 0.05, 8.0, seed)
    assert np.array_equal(w1, w2)


GRID = [
    # rows, cols, alpha, group2, ratio, planted
    (20, 80, 0.25, 16, 0.002, 0.0),
    (24, 160, 0.5, 16, 0.005, 0.0),
    (9, 96, 0.0, 16, 0.0, 0.0),
    (9, 96, 1.0, 16, 0.0, 0.0),
    (37, 160, 0.25, 16, 0.01, 0.0),
    (64, 512, 0.25, 1, 0.01, 0.0),
    (64, 512, 0.25, 5, 0.05, 0.01),
    (50, 1024, 0.75, 128, 0.002, 0.01),
    (130, 1024, 0.25, 128, 0.002, 0.0),
    (1, 16, 0.25, 16, 1.0, 0.0),        # every real 2-bit slot an outlier
    (300, 2048, 0.25, 16, 0.002, 0.0),
]


@needs_ref
@pytest.mark.parametrize("rows,cols,alpha,g2,ratio,planted", GRID)
def test_quantize_layer_bit_identical(rows, cols, alpha, g2, ratio, planted):
    seed = rows * 7 + cols
    w = qw.synth_gaussian(rows, cols, seed)
    if planted:
        qw.plant_outliers(w, planted, 8.0, seed)
    h = qw.synth_calibration(cols, seed)
    ours = qw.quantize_layer(w, h, alpha, g2, ratio, threads=3)
    ref = oracle.RefLayer.quantize(w, h, alpha, g2, ratio).to_layer()
    assert ours.streams_equal(ref)
    assert ours.cfg.alpha == ref.cfg.alpha and ours.cfg.outlier_ratio == ref.cfg.outlier_ratio


@needs_ref
def test_quantize_threads_do_not_change_bits():
    w, h = qw.synth_gaussian(96, 512, 3), qw.synth_calibration(512, 3)
    a = qw.quantize_layer(w, h, threads=1)
    b = qw.quantize_layer(w, h, threads=7)
    assert a.streams_equal(b)


def test_llama_q_proj_payload_matches_survey():
    """Q7 payload 6,851,660 B, nnz 33,554, P = T2 = T4 = 64."""
    layer = qw.synth_layer(4096, 4096, seed=7)
    assert layer.nnz == 33554
    assert qw.payload_bytes(layer) == 6851660
    c = layer.cfg
    assert (c.triples, c.blocks4, c.paired, c.pad2) == (64, 64, 64, 0)


def test_outlier_slots_dequantize_to_zero_and_csr_holds_fp16():
    """AC6 (acceptance.cpp:273-339): dense slot exactly 0, sparse = f16(orig)."""
    w = qw.synth_gaussian(64, 512, 5)
    qw.plant_outliers(w, 0.002, 8.0, 5)
    h = qw.synth_calibration(512, 5)
    layer = qw.quantize_layer(w, h)
    recon = oracle.reconstruct_dense(layer)
    perm = layer.plan_perm.astype(np.int64)
    for r in range(64):
        for i in range(layer.row_ptr[r], layer.row_ptr[r + 1]):
            col = int(layer.col_ind[i])
            assert recon[r, col] == 0.0
            assert layer.values[i] == np.float16(w[r, perm[col]]).view(np.uint16)


def test_container_round_trip(tmp_path):
    layer = qw.synth_layer(40, 320, seed=9, outlier_ratio=0.01)
    p = tmp_path / "l.qwl"
    qw.write_packed_layer(layer, str(p))
    back = qw.read_packed_layer(str(p))
    assert back.streams_equal(layer)
    # corrupt one payload byte -> checksum mismatch (test_container.cpp:145-214)
    b = bytearray(p.read_bytes())
    b[400] ^= 0x5A
    p.write_bytes(bytes(b))
    with pytest.raises(QWeightError) as e:
        qw.read_packed_layer(str(p))
    assert e.value.status == 8
    with pytest.raises(QWeightError) as e:
        qw.read_packed_layer(str(tmp_path / "missing.qwl"))
    assert e.value.status == 7


@needs_ref
def test_container_interop_with_reference(tmp_path):
    layer = qw.synth_layer(33, 256, seed=4, outlier_ratio=0.01)
    p1, p2 = tmp_path / "ours.qwl", tmp_path / "ref.qwl"
    qw.write_packed_layer(layer, str(p1))
    ref = oracle.RefLayer.read(p1)          # reference reads our file
    assert ref.to_layer().streams_equal(layer)
    ref.write(p2)                            # and writes the same bytes
    assert p1.read_bytes() == p2.read_bytes()


def test_validate_layer_rejects_malformed():
    layer = qw.synth_layer(16, 128, seed=2, outlier_ratio=0.01)
    bad = qw.read_packed_layer.__globals__["PackedLayer"](**{**layer.__dict__, "_keep": []})
    bad.sorder_zero2 = layer.sorder_zero2.copy()
    bad.sorder_zero2[0] = 16                 # bitpack.cpp:235-237
    with pytest.raises(QWeightError) as e:
        qw.validate_layer(bad)
    assert e.value.status == 2
    bad.sorder_zero2 = layer.sorder_zero2
    bad.main = layer.main[:-1]               # stream size
    with pytest.raises(QWeightError):
        qw.validate_layer(bad)
    bad.main = layer.main
    bad.col_ind = layer.col_ind.copy()
    if bad.col_ind.size:
        bad.col_ind[0] = layer.cfg.n2_padded + 1  # outlier outside 2-bit region
        with pytest.raises(QWeightError):
            qw.validate_layer(bad)


def test_row_shards_reassemble_bitwise():
    """Column-parallel TP split: shards' oracle y concatenate to the full y."""
    layer = qw.synth_layer(96, 512, seed=12, outlier_ratio=0.01)
    x = qw.synth_activation(512, 13)
    full = oracle.matvec_oracle(layer, x)
    parts = [oracle.matvec_oracle(qw.shard_rows(layer, r0, r1), x)
             for r0, r1 in ((0, 32), (32, 64), (64, 96))]
    assert np.array_equal(np.concatenate(parts), full)
    with pytest.raises(QWeightError):
        qw.shard_rows(layer, 8, 40)          # not aligned to group2


def test_tile_shards_sum_to_full():
    """Row-parallel TP split: per-tile-range partial y sum to the full y."""
    layer = qw.synth_layer(64, 1024, seed=14, outlier_ratio=0.01)
    x = qw.synth_activation(1024, 15)
    xp = qw.permute(layer, x)
    ref = oracle.matvec_f64(layer, x)
    T = layer.cfg.triples
    total = np.zeros(64, np.float64)
    for t0, t1 in ((0, T // 2), (T // 2, T)):
        shard, slots = qw.shard_tiles(layer, t0, t1)
        total += oracle.matvec_f64(shard, xp[slots])
    assert np.max(np.abs(total - ref)) <= 1e-9 * np.max(np.abs(ref))
