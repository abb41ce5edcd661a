"""Test helpers mirroring the reference's tests/helpers.hpp.

manual_plan (helpers.hpp:46-63), make_cfg (65-73), random_groups (77-108),
random_csr (112-136), plus a numpy pack of logical groups into the
reference stream layout (bitpack.cpp:91-147) so tests can build layers with
arbitrary codes / zero2 / scales and check every path against them.
"""
import numpy as np

import paper_2311_16442_b200 as qw

PAD = 0xFFFFFFFF


def manual_plan(ic: int, n4: int):
    n2 = ic - n4
    pad2 = (48 - n2 % 48) % 48
    bits = np.full(ic, 2, np.uint8)
    bits[n2:] = 4
    perm = np.concatenate([np.arange(n2), np.full(pad2, PAD), np.arange(n2, ic)]).astype(np.uint32)
    return bits, perm, pad2


def random_groups(rows, ic, n4, group2, rng, big_scales=False):
    """Structurally valid random content.  big_scales=True draws fp16 scales
    over the reference's full 0..0x7bff range (pack/unpack tests only)."""
    n2 = ic - n4
    pad2 = (48 - n2 % 48) % 48
    n2p = n2 + pad2
    T2, T4 = n2p // 48, n4 // 16
    gpr = 3 * T2
    rb = (rows + group2 - 1) // group2
    g = {}
    g["codes2"] = rng.integers(0, 4, (rows, n2p), dtype=np.uint8)
    g["zeros2"] = rng.integers(0, 4, (rows, gpr), dtype=np.uint8)
    sc = np.zeros((rows, gpr), np.uint8)
    for j in range(gpr):
        sc[:, j] = rng.integers(0, 16 if j % 3 == 0 else 8, rows)
    g["scodes"] = sc
    g["zero2"] = rng.integers(0, 16, rb * gpr, dtype=np.uint8)
    g["codes4"] = rng.integers(0, 16, (rows, n4), dtype=np.uint8)
    g["z4"] = rng.integers(0, 16, rows * T4, dtype=np.uint8)
    if big_scales:
        g["scale2"] = rng.integers(0, 0x7BFF, rb * gpr, dtype=np.uint16)
        g["s4"] = rng.integers(0, 0x7BFF, rows * T4, dtype=np.uint16)
    else:
        g["scale2"] = np.float16(rng.uniform(0.01, 0.2, rb * gpr)).view(np.uint16)
        g["s4"] = np.float16(rng.uniform(0.01, 0.5, rows * T4)).view(np.uint16)
    return g


def random_csr(rows, n2, rng, max_per_row=3):
    """random_csr (helpers.hpp:112-136): sorted unique real 2-bit slots."""
    row_ptr = [0]
    cols, vals = [], []
    for _ in range(rows):
        k = int(rng.integers(0, max_per_row + 1)) if n2 else 0
        c = np.unique(rng.integers(0, max(n2, 1), k)) if k else np.zeros(0, np.int64)
        cols.extend(c.tolist())
        vals.extend(np.float16(rng.normal(0, 4, c.size)).view(np.uint16).tolist())
        row_ptr.append(len(cols))
    return (np.array(row_ptr, np.uint32), np.array(cols, np.uint16), np.array(vals, np.uint16))


def pack(rows, ic, n4, group2, g, csr=None, perm_bits=None) -> qw.PackedLayer:
    """pack_layer (bitpack.cpp:91-147) in numpy."""
    n2 = ic - n4
    pad2 = (48 - n2 % 48) % 48
    n2p = n2 + pad2
    T2, T4 = n2p // 48, n4 // 16
    P = min(T2, T4)
    bits, perm = (perm_bits if perm_bits is not None else manual_plan(ic, n4)[:2])
    c2 = g["codes2"].reshape(rows, T2, 48)
    # 48 2-bit codes -> 12 bytes, code k at bits 2(k%4) of byte k/4
    b2 = (c2.reshape(rows, T2, 12, 4).astype(np.uint32) << np.array([0, 2, 4, 6])).sum(-1).astype(np.uint8)
    c4 = g["codes4"].reshape(rows, T4, 2, 4, 2)
    b4 = (c4[..., 0] | (c4[..., 1] << 4)).astype(np.uint8)  # rows, T4, half, 4 bytes
    main = np.zeros((rows, P, 16), np.uint8)
    main[:, :, :12] = b2[:, :P]
    main[:, :, 12:] = b4[:, :P, 0]
    tail2 = b2[:, P:].reshape(-1)
    tail4 = b4[:, P:, 0].reshape(-1)
    secondary = b4[:, :, 1].reshape(-1)
    z, s = g["zeros2"].reshape(rows, T2, 3), g["scodes"].reshape(rows, T2, 3)
    meta = (z[..., 0] | (z[..., 1] << 2) | (z[..., 2] << 4) | (s[..., 0].astype(np.uint16) << 6) |
            (s[..., 1].astype(np.uint16) << 10) | (s[..., 2].astype(np.uint16) << 13)).astype(np.uint16)
    if csr is None:
        csr = (np.zeros(rows + 1, np.uint32), np.zeros(0, np.uint16), np.zeros(0, np.uint16))
    cfg = qw.LayerConfig(rows=rows, cols=ic, n4=n4, pad2=pad2, outlier_count=int(csr[1].size),
                         group2=group2)
    layer = qw.PackedLayer(cfg=cfg, plan_bits=bits, plan_perm=perm, main=main.reshape(-1),
                           tail2=tail2, tail4=tail4, secondary=secondary, meta=meta.reshape(-1),
                           sorder_zero2=g["zero2"], sorder_scale2=g["scale2"],
                           fourbit_scale=g["s4"], fourbit_zero=g["z4"],
                           row_ptr=csr[0], col_ind=csr[1], values=csr[2])
    return layer
