"""LinearStack: a decode step over many quantized linears, captured once.

The reference has no model layer; this is the thinnest runner
that exercises the hot path the way a decoder does: every linear of every
layer runs once per token.  All activations live in one device buffer and
all outputs in another, so a host round trip is two copies; the launches
(one fused kernel per linear, chained with programmatic dependent launch)
are captured in one CUDA graph.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .engine import DecodeChain, DeviceLayer, LayerGroup, Workspace

try:
    import torch
except Exception:  # pragma: no cover
    torch = None


@dataclass
class _Slot:
    layer: DeviceLayer
    x_off: int
    y_off: int


class LinearStack:
    def __init__(self, layers: list[DeviceLayer], device: int = 0, batch: int = 1,
                 pdl: bool = True, depends: list[bool] | None = None,
                 groups: list[list[int]] | None = None, prefetch: bool = False):
        """groups: consecutive index lists of linears that read the same input
        (q/k/v, gate/up) and run as ONE fused launch (batch 1); default one
        launch per linear.  depends[i] (per launch): launch i reads an input
        produced by launch i-1 (it waits for it); False lets it read its input
        at once (it came from the host or an earlier, finished kernel).
        prefetch: each launch streams the next launch's weights into L2
        (qw_*_set_prefetch), so HBM never idles between dependent launches."""
        self.device, self.batch, self.pdl = device, batch, pdl
        self.groups = groups if groups is not None else [[i] for i in range(len(layers))]
        assert [i for g in self.groups for i in g] == list(range(len(layers))), "groups must tile the layers in order"
        self.depends = list(depends) if depends is not None else [True] * len(self.groups)
        self.fused = [LayerGroup([layers[i] for i in g]) if len(g) > 1 and batch == 1 else None
                      for g in self.groups]
        self.dev = torch.device(f"cuda:{device}")
        self.prefetch = prefetch and batch == 1
        self._layers = layers
        self.set_prefetch()
        xo = yo = 0
        self.slots = []
        for dl in layers:
            self.slots.append(_Slot(dl, xo, yo))
            xo += batch * dl.cols
            yo += batch * dl.rows
        self.x = torch.zeros(xo, dtype=torch.float32, device=self.dev)
        self.y = torch.zeros(yo, dtype=torch.float32, device=self.dev)
        self.x_host = torch.zeros(xo, dtype=torch.float32).pin_memory()
        self.y_host = torch.zeros(yo, dtype=torch.float32).pin_memory()
        max_cols = max(dl.padded_cols for dl in layers)
        self.ws = Workspace(device, max_cols, batch)
        self.graph = None
        self.gemv_graph = None
        self.chain = None

    def set_prefetch(self, select=None):
        """Every launch (of those whose first layer `select` accepts) streams the
        following launch's weights into L2 -- the last one the first's, i.e. the
        next decode step.  Launch parameters are captured by value, so a graph
        keeps the setting it was captured with."""
        if not self.prefetch:
            return
        order = []  # launches in stream order: (fused group | layer, its layers)
        for gi, g in enumerate(self.groups):
            if select is not None and not select(self._layers[g[0]]):
                continue
            if self.fused[gi] is not None:
                order.append((self.fused[gi], [self._layers[i] for i in g]))
            else:
                order.extend((self._layers[i], [self._layers[i]]) for i in g)
        for k, (launch, _) in enumerate(order):
            launch.set_prefetch(order[(k + 1) % len(order)][1])

    # ------------------------------------------------------------ views
    def x_of(self, i: int):
        s = self.slots[i]
        return self.x[s.x_off:s.x_off + self.batch * s.layer.cols].view(self.batch, s.layer.cols)

    def y_of(self, i: int):
        s = self.slots[i]
        return self.y[s.y_off:s.y_off + self.batch * s.layer.rows].view(self.batch, s.layer.rows)

    # ------------------------------------------------------------ launches
    def _launch(self, gi, stream=None):
        g, dep = self.groups[gi], self.depends[gi]
        if self.fused[gi] is not None:  # one input, one fused launch
            self.fused[gi].matvec(self.x_of(g[0])[0], outs=[self.y_of(i)[0] for i in g], stream=stream,
                                  pdl=self.pdl, x_independent=not dep)
            return
        for k, i in enumerate(g):
            self.slots[i].layer.matvec(self.x_of(g[0] if len(g) > 1 else i), out=self.y_of(i),
                                       workspace=self.ws, stream=stream, pdl=self.pdl,
                                       x_independent=(not dep) or k > 0)

    def make_chain(self, depends: list[bool] | None = None) -> DecodeChain:
        """The whole step as ONE persistent kernel (qw_chain_*, batch 1): one
        chain step per launch of the grouped sequence; depends per launch."""
        assert self.batch == 1, "the decode chain is batch 1"
        dep = self.depends if depends is None else depends
        steps = []
        for gi, g in enumerate(self.groups):
            lay = [self.slots[i].layer for i in g]
            if self.fused[gi] is not None:
                steps.append((lay, self.x_of(g[0])[0], [self.y_of(i)[0] for i in g], dep[gi]))
            else:
                for k, i in enumerate(g):
                    src = g[0] if len(g) > 1 else i
                    steps.append(([self.slots[i].layer], self.x_of(src)[0], [self.y_of(i)[0]], dep[gi] and k == 0))
        return DecodeChain(steps)

    def use_chain(self, on: bool = True):
        """launch_step / capture / run go through the persistent decode-chain kernel."""
        self.chain = self.make_chain() if on else None
        self.graph = None

    def launch_step(self, stream=None):
        if self.chain is not None:
            self.chain.run(stream)
            return
        for gi in range(len(self.groups)):
            self._launch(gi, stream)

    def launch_subset(self, select, stream=None):
        """Launch only the launches whose first layer `select(layer)` accepts (kernel-only timing)."""
        for gi, g in enumerate(self.groups):
            if select(self.slots[g[0]].layer):
                self._launch(gi, stream)

    def capture(self):
        """Capture one decode step into a CUDA graph (after a warm run)."""
        self.launch_step()
        torch.cuda.synchronize(self.dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.launch_step()
        torch.cuda.synchronize(self.dev)
        self.graph = g
        return g

    def capture_subset(self, select):
        self.set_prefetch(select)
        self.launch_subset(select)
        torch.cuda.synchronize(self.dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.launch_subset(select)
        torch.cuda.synchronize(self.dev)
        self.set_prefetch()
        return g

    def replay(self):
        if self.graph is None:
            self.capture()
        self.graph.replay()

    # ------------------------------------------------------------ host API
    def _io_range(self, gi):
        """Contiguous x and y element ranges of launch group gi's layers."""
        g = self.groups[gi]
        a, b = self.slots[g[0]], self.slots[g[-1]]
        return ((a.x_off, b.x_off + self.batch * b.layer.cols),
                (a.y_off, b.y_off + self.batch * b.layer.rows))

    def capture_e2e(self):
        """The step with its host copies overlapped, as one CUDA graph.  The
        inputs go host -> HBM on a copy stream in a few chunks of growing size
        (the first covers the first launches only), each launch chunk waits for
        its inputs; the outputs go HBM -> host on a second copy stream in
        chunks of shrinking size as soon as their launches finished.  The
        step's critical path gains only the first input chunk and the last
        output chunk, and only a handful of launches carry a cross-stream wait
        (the others keep their programmatic dependent launch edge)."""
        self.launch_step()
        torch.cuda.synchronize(self.dev)
        n = len(self.groups)
        cuts_in = sorted({0, min(n, 2), min(n, 8), min(n, 32), n})
        cuts_out = sorted({0, max(0, n - 32), max(0, n - 8), max(0, n - 2), n})
        s_in, s_out = torch.cuda.Stream(self.dev), torch.cuda.Stream(self.dev)

        def span(lo, hi):  # x and y element ranges of launch groups [lo, hi)
            (x0, _), (y0, _) = self._io_range(lo)
            (_, x1), (_, y1) = self._io_range(hi - 1)
            return x0, x1, y0, y1

        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            cap = torch.cuda.current_stream(self.dev)
            s_in.wait_stream(cap)
            s_out.wait_stream(cap)
            ready = {}
            with torch.cuda.stream(s_in):
                for lo, hi in zip(cuts_in[:-1], cuts_in[1:]):
                    x0, x1, _, _ = span(lo, hi)
                    self.x[x0:x1].copy_(self.x_host[x0:x1], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(s_in)
                    ready[lo] = e
            out_end = {hi: lo for lo, hi in zip(cuts_out[:-1], cuts_out[1:])}
            for gi in range(n):
                if gi in ready:
                    cap.wait_event(ready[gi])
                self._launch(gi)
                if gi + 1 in out_end:
                    done = torch.cuda.Event()
                    done.record(cap)
                    _, _, y0, y1 = span(out_end[gi + 1], gi + 1)
                    s_out.wait_event(done)
                    with torch.cuda.stream(s_out):
                        self.y_host[y0:y1].copy_(self.y[y0:y1], non_blocking=True)
            cap.wait_stream(s_in)
            cap.wait_stream(s_out)
        torch.cuda.synchronize(self.dev)
        self.e2e_graph = g
        return g

    def run(self, x_host: np.ndarray | None = None) -> np.ndarray:
        """One decode step end to end: pinned host -> HBM copy of every
        activation, the step, HBM -> pinned host copy of every output,
        synchronise.  Returns the outputs (flat, slot order).  Per-launch
        launches overlap the copies with the step (capture_e2e); the chain
        kernel (use_chain) copies around it."""
        if x_host is not None:
            self.x_host.numpy()[:] = x_host
        stream = torch.cuda.current_stream(self.dev)
        if self.chain is None:
            if getattr(self, "e2e_graph", None) is None:
                self.capture_e2e()
            self.e2e_graph.replay()
        else:
            self.x.copy_(self.x_host, non_blocking=True)
            self.replay()
            self.y_host.copy_(self.y, non_blocking=True)
        stream.synchronize()
        return self.y_host.numpy()

    @property
    def h2d_bytes(self) -> int:
        return self.x.numel() * 4

    @property
    def d2h_bytes(self) -> int:
        return self.y.numel() * 4
