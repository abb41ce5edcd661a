"""The torch.library custom op / nn.Module over the B200 quantized linear
(SURVEY §8(f) rank 4): eager, under CUDA-graph capture and under
torch.compile it runs this repository's kernels and matches the f64 oracle."""
import numpy as np
import pytest

import oracle
import paper_2311_16442_b200 as qw

pytestmark = pytest.mark.gpu


def rel_l2(y, ref):
    return float(np.linalg.norm(np.asarray(y, np.float64) - ref) / np.linalg.norm(ref))


def test_quantized_linear_module_eager_graph_compile():
    import torch
    from paper_2311_16442_b200.torch_ops import QuantizedLinear
    layers = [qw.synth_layer(512, 1024, seed=31), qw.synth_layer(1024, 512, seed=32)]
    mlp = torch.nn.Sequential(QuantizedLinear(layers[0]), torch.nn.ReLU(), QuantizedLinear(layers[1]))
    x = torch.from_numpy(np.stack([qw.synth_activation(1024, 33 + b) for b in range(3)])).cuda()
    # eager: batch 3 (the tcgen05 path) and the reference composition
    y = mlp(x)
    for b in range(3):
        h = np.maximum(oracle.matvec_f64(layers[0], x[b].cpu().numpy()), 0).astype(np.float32)
        assert rel_l2(y[b].cpu().numpy(), oracle.matvec_f64(layers[1], h)) <= 2e-2
    # batch 1 under CUDA-graph capture
    x1 = x[:1].clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        y1 = mlp(x1)
    g.replay()
    torch.cuda.synchronize()
    assert torch.allclose(y1, mlp(x1), rtol=0, atol=0)
    # torch.compile: the op is opaque (fake impl for shapes), the kernel stays ours
    f = torch.compile(mlp, fullgraph=True)
    assert torch.equal(f(x1), mlp(x1))
    # leading dims and batches > 16 are split into <= 16-column calls
    xl = torch.from_numpy(np.stack([qw.synth_activation(1024, 60 + b) for b in range(20)])).cuda()
    yl = mlp[0](xl.reshape(4, 5, 1024))
    assert yl.shape == (4, 5, 512)
    assert rel_l2(yl.reshape(20, 512)[17].cpu().numpy(), oracle.matvec_f64(layers[0], xl[17].cpu().numpy())) <= 1e-2


def test_quantized_linear_group_module():
    """q/k/v as one QuantizedLinearGroup: one fused launch at batch 1 (also
    under CUDA-graph capture), each layer's batched path above; every output
    matches its own QuantizedLinear and the f64 oracle."""
    import torch
    from paper_2311_16442_b200.torch_ops import QuantizedLinear, QuantizedLinearGroup
    layers = [qw.synth_layer(r, 1024, seed=40 + i, outlier_ratio=0.005) for i, r in enumerate((512, 256, 256))]
    grp = QuantizedLinearGroup(layers)
    singles = [QuantizedLinear(m.dl) for m in grp.members]
    for b in (1, 3):
        x = torch.from_numpy(np.stack([qw.synth_activation(1024, 50 + i) for i in range(b)])).cuda()
        outs = grp(x)
        assert [o.shape for o in outs] == [(b, 512), (b, 256), (b, 256)]
        for L, o, m in zip(layers, outs, singles):
            ref_single = m(x)
            assert float((o - ref_single).abs().max()) <= 1e-6 * float(ref_single.abs().max())
            for i in range(b):
                assert rel_l2(o[i].cpu().numpy(), oracle.matvec_f64(L, x[i].cpu().numpy())) <= 1e-2
    # batch 1 under CUDA-graph capture
    x1 = torch.from_numpy(qw.synth_activation(1024, 70)).cuda().reshape(1, 1024)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        outs = grp(x1)
    g.replay()
    torch.cuda.synchronize()
    for o, e in zip(outs, grp(x1)):
        assert torch.equal(o, e)
    # torch.compile: the group op is opaque (fake impl for the list of outputs)
    f = torch.compile(lambda t: [o * 2.0 for o in grp(t)], fullgraph=True)
    for o, e in zip(f(x1), grp(x1)):
        assert torch.equal(o, e * 2.0)
