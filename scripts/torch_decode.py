"""µs per token of a Llama-2-7B-shaped decode step written
in PyTorch, with the 7 linears of each of the 32 decoder layers as
QuantizedLinear modules (torch.ops.qweight_b200.quantized_linear -> this
repository's kernels) and everything else in torch: RMSNorm, a stand-in for
attention (q + k + v: the attention kernel is not part of this path), the
residual adds and SiLU(gate) * up.  The whole step is captured in one CUDA
graph; batch 1 (K2), 4 (column launches) and 8 (K4).  Weights: 7 distinct
layers quantized by the GPU producer, cloned per decoder layer (every linear
its own HBM copy, 2.65 GB, > L2).
usage: python scripts/torch_decode.py [layers] [batches...]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2311_16442_b200 as qw  # noqa: E402
from paper_2311_16442_b200.torch_ops import QuantizedLinear, QuantizedLinearGroup  # noqa: E402

NL = int(sys.argv[1]) if len(sys.argv) > 1 else 32
BATCHES = [int(b) for b in sys.argv[2:] if not b.startswith("--")] or [1, 4, 8]
D, F = 4096, 11008
SHAPES = {"q": (D, D), "k": (D, D), "v": (D, D), "o": (D, D), "gate": (F, D), "up": (F, D), "down": (D, F)}

t0 = time.perf_counter()
base = {}
for i, (name, (rows, cols)) in enumerate(SHAPES.items()):
    layer = qw.quantize_layer_gpu(qw.synth_gaussian(rows, cols, 7 + i), qw.synth_calibration(cols, 7 + i))
    base[name] = qw.DeviceLayer(layer)
prep_s = time.perf_counter() - t0


GROUPED = "--ungrouped" not in sys.argv


class DecoderLayer(torch.nn.Module):
    def __init__(self):
        super().__init__()
        self.lin = torch.nn.ModuleDict({n: QuantizedLinear(base[n].clone()) for n in SHAPES})
        if GROUPED:  # q/k/v and gate/up: one fused launch each at batch 1
            self.qkv = QuantizedLinearGroup([self.lin[n].dl for n in ("q", "k", "v")])
            self.gu = QuantizedLinearGroup([self.lin[n].dl for n in ("gate", "up")])
        self.n1 = torch.nn.RMSNorm(D, device="cuda")
        self.n2 = torch.nn.RMSNorm(D, device="cuda")

    def forward(self, x):
        h = self.n1(x)
        q, k, v = self.qkv(h) if GROUPED else (self.lin["q"](h), self.lin["k"](h), self.lin["v"](h))
        x = x + self.lin["o"](q + k + v)  # attention stand-in
        h = self.n2(x)
        g, u = self.gu(h) if GROUPED else (self.lin["gate"](h), self.lin["up"](h))
        return x + self.lin["down"](torch.nn.functional.silu(g) * u)


model = torch.nn.Sequential(*[DecoderLayer() for _ in range(NL)])
for b in BATCHES:
    x = torch.randn(b, D, device="cuda") * 0.1
    with torch.no_grad():
        y = model(x)  # warm-up (eager)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                model(x)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            y = model(x)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        R = 20
        e0.record()
        for _ in range(R):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / R
    print(json.dumps({"batch": b, "layers": NL, "ms_per_step": round(ms, 4), "us_per_token": round(1e3 * ms / b, 1),
                      "finite": bool(torch.isfinite(y).all()), "grouped": GROUPED, "path": qw.DeviceLayer.batched_path(base["q"], b)
                      if b > 1 else "batch-1", "prep_s": round(prep_s, 1)}), flush=True)
