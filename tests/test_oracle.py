"""Pin the C oracle (oracle/qw_oracle.c) before trusting it.

  * golden tile bytes (reference test_bitpack.cpp:30-85,
    acceptance.cpp:155-185)
  * IEEE half conversions against numpy and the compiled reference
  * golden layers quantized + serialized + evaluated by the reference itself
    (tests/golden/make_golden.py): matvec_oracle bitwise, reconstruct_dense
    and unpack_layer by hash, matvec_reference_f64
  * randomized layers (random_groups) against the compiled reference
"""
import hashlib
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_2311_16442_b200 as qw
from helpers import pack, random_csr, random_groups

GOLD = Path(__file__).resolve().parent / "golden"
GOLDEN_LAYERS = sorted(p.stem[len("layer_"):] for p in GOLD.glob("layer_*.qwl"))
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ------------------------------------------------------------------ tiles
def test_golden_tiles_match_survey_bytes():
    assert (GOLD / "tile_zero.bin").read_bytes() == bytes(22)
    assert (GOLD / "tile_ramp.bin").read_bytes() == bytes.fromhex(
        "e4" * 12 + "10325476" + "98badcfe" + "0000")
    assert (GOLD / "tile_meta.bin").read_bytes() == bytes(20) + bytes.fromhex("7976")


def test_oracle_pack_tile_golden():
    z48, z16, z3 = np.zeros(48, np.uint8), np.zeros(16, np.uint8), np.zeros(3, np.uint8)
    assert oracle.pack_tile(z48, z16, z3, z3) == (GOLD / "tile_zero.bin").read_bytes()
    ramp = oracle.pack_tile(np.arange(48) % 4, np.arange(16), z3, z3)
    assert ramp == (GOLD / "tile_ramp.bin").read_bytes()
    meta = oracle.pack_tile(z48, z16, [1, 2, 3], [9, 5, 3])
    assert meta == (GOLD / "tile_meta.bin").read_bytes()
    assert meta[20] | (meta[21] << 8) == 0x7679


def test_lsb_first_and_nibble_order():
    """test_bitpack.cpp:62-85"""
    c2 = np.zeros(48, np.uint8)
    c2[0], c2[5] = 3, 2
    z16, z3 = np.zeros(16, np.uint8), np.zeros(3, np.uint8)
    t = oracle.pack_tile(c2, z16, z3, z3)
    assert t[0] == 0x03 and t[1] == 0x08
    c4 = np.zeros(16, np.uint8)
    c4[0], c4[1], c4[8] = 0xF, 0xA, 0x1
    t = oracle.pack_tile(np.zeros(48, np.uint8), c4, z3, z3)
    assert t[12] == 0xAF and t[16] == 0x01


# ------------------------------------------------------------------ fp16
def test_f16_to_f32_exhaustive():
    L = oracle.oracle_lib()
    h = np.arange(65536, dtype=np.uint32)
    ours = np.array([L.qo_f16_to_f32(int(v)) for v in h], np.float32)
    ref = h.astype(np.uint16).view(np.float16).astype(np.float32)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(ours), nan)
    assert np.array_equal(ours[~nan].view(np.uint32), ref[~nan].view(np.uint32))


def test_f32_to_f16_round_to_nearest_even():
    L = oracle.oracle_lib()
    rng = np.random.default_rng(0)
    vals = np.concatenate([
        rng.standard_normal(20000).astype(np.float32) * np.float32(10) ** rng.integers(-8, 6, 20000),
        np.array([0.0, -0.0, 65504.0, 65520.0, 65519.99, 6e-8, 3e-8, 2.98e-8, 1e-40, np.inf, -np.inf],
                 np.float32)])
    ours = np.array([L.qo_f32_to_f16(float(v)) for v in vals], np.uint16)
    with np.errstate(over="ignore"):
        ref = vals.astype(np.float16).view(np.uint16)
    assert np.array_equal(ours, ref)
    assert L.qo_f32_to_f16(float("nan")) & 0x7E00 == 0x7E00  # quieted NaN


@needs_ref
def test_f16_conversions_match_reference():
    L, R = oracle.oracle_lib(), oracle.ref_lib()
    for v in range(0, 65536, 7):
        a, b = L.qo_f16_to_f32(v), R.qwref_f16_to_f32(v)
        assert (np.isnan(a) and np.isnan(b)) or np.float32(a).view(np.uint32) == np.float32(b).view(np.uint32)
    rng = np.random.default_rng(1)
    for v in rng.standard_normal(5000).astype(np.float32) * np.float32(300):
        assert L.qo_f32_to_f16(float(v)) == R.qwref_f32_to_f16(float(v))


# ------------------------------------------------------------------ golden layers
@pytest.mark.parametrize("name", GOLDEN_LAYERS)
def test_golden_layer_oracle(name):
    layer = qw.read_packed_layer(str(GOLD / f"layer_{name}.qwl"))
    d = np.load(GOLD / f"layer_{name}.npz")
    # matvec_oracle is bit-exact with the reference's own output
    y = oracle.matvec_oracle(layer, d["x"])
    assert np.array_equal(y.view(np.uint32), d["y_oracle"].view(np.uint32))
    y64 = oracle.matvec_f64(layer, d["x"])
    assert np.array_equal(y64, d["y_f64"])
    assert sha(oracle.reconstruct_dense(layer)) == str(d["recon_sha"])
    un = oracle.unpack(layer)
    assert [sha(un[k]) for k in ("codes2", "zeros2", "scodes", "codes4")] == list(d["unpack_sha"])
    assert oracle.payload_bytes(layer) == int(d["payload"]) == qw.payload_bytes(layer)


# ------------------------------------------------------------------ random layers
@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_random_groups_oracle_vs_reference(seed):
    rng = np.random.default_rng(100 + seed)
    rows = int(rng.integers(1, 40))
    ic = 16 * int(rng.integers(1, 40))
    n4 = 16 * int(rng.integers(0, ic // 16 + 1))
    g2 = int(rng.choice([1, 3, 4, 16, 128]))
    g = random_groups(rows, ic, n4, g2, rng, big_scales=True)
    csr = random_csr(rows, ic - n4, rng)
    layer = pack(rows, ic, n4, g2, g, csr)
    qw.validate_layer(layer)
    ref = oracle.RefLayer.from_layer(layer)
    # unpack_layer and reconstruct_dense bit for bit
    un, run = oracle.unpack(layer), ref.unpack()
    for k in run:
        assert np.array_equal(un[k], run[k]), k
    assert np.array_equal(un["codes2"], g["codes2"])
    assert np.array_equal(un["codes4"], g["codes4"])
    w, rw = oracle.reconstruct_dense(layer), ref.reconstruct_dense()
    assert np.array_equal(w.view(np.uint32), rw.view(np.uint32))
    x = np.random.default_rng(seed).standard_normal(ic).astype(np.float32)
    y, _ = ref.matvec_oracle(x)
    ours = oracle.matvec_oracle(layer, x)
    assert np.array_equal(np.isnan(ours), np.isnan(y))
    fin = np.isfinite(y)
    assert np.array_equal(ours[fin].view(np.uint32), y[fin].view(np.uint32))


def test_oracle_rejects_nonfinite_activation():
    """engine.cpp:126-130 via the C restatement."""
    layer = qw.read_packed_layer(str(GOLD / "layer_pads_tails.qwl"))
    x = np.zeros(80, np.float32)
    x[3] = np.inf
    with pytest.raises(ValueError):
        oracle.matvec_oracle(layer, x)


def test_oracle_known_answer_dequant():
    """dequantize_scale(3, 1, f16(2.0)) = 4 and (7, 7, .) = 0 (test_quant.cpp:174-177);
    codes {0,2,3} with z=1 -> {-1,1,2} x s (109-118)."""
    rows, ic, n4 = 1, 48, 0
    rng = np.random.default_rng(0)
    g = random_groups(rows, ic, n4, 16, rng)
    g["codes2"][:] = 0
    g["codes2"][0, :3] = [0, 2, 3]
    g["zeros2"][:] = [1, 0, 0]
    g["scodes"][:] = [3, 0, 0]
    g["zero2"][:] = [1, 7, 0]
    g["scale2"][:] = [np.float16(2.0).view(np.uint16)] * 3
    layer = pack(rows, ic, n4, 16, g)
    w = oracle.reconstruct_dense(layer)[0]
    # group 0: s1 = (3-1)*2 = 4; w = (c - 1) * 4
    assert list(w[:3]) == [-4.0, 4.0, 8.0]
    # group 1: eff = 0 << 1 = 0, zero2 = 7 -> s1 = -14; codes 0, z 0 -> 0
    assert np.all(w[16:32] == 0.0)
