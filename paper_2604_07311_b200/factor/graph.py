"""CUDA-graph replay of the native Cholesky driver.

The native driver (bf_cholesky_*) issues a few hundred launches per
factorization on two streams (main + the high-priority panel stream of the
lookahead schedule, forked and joined by events).  For repeated
factorizations of the same view and tree — a solver loop, the CLI's
repeats, small orders where launch latency shows — CholeskyGraph records
that launch sequence once into a CUDA graph (torch.cuda.CUDAGraph; the
fork/join becomes graph edges) and replays it: same kernels, same
arguments, same bits (tests/test_graph.py), without per-launch host work.
The reference has no counterpart (its driver is a Python loop,
factor/cholesky.py:118-158); this replaces a tracing compiler.
"""
from __future__ import annotations

from typing import Optional

import torch

from ..control import ControlNode, default_tree
from ..errors import NotPositiveDefiniteError
from ..views import MatrixView, make_view
from .cholesky import cholesky_async

__all__ = ["CholeskyGraph"]


class CholeskyGraph:
    """Capture cholesky_async(a, uplo, tree) once; run() replays it on the
    same storage (refill `a` between runs) and returns the device pivot flag."""

    def __init__(self, a: MatrixView, uplo: str = "lower", tree: Optional[ControlNode] = None) -> None:
        if tree is None:
            tree = default_tree("cholesky", a.n, a.dtype)
        self.a, self.uplo, self.tree = a, uplo, tree
        # one-time driver state (streams, kernel attributes) outside the capture:
        # a small identity factorization through the same tree shape
        bs = tree.bs or 128
        nw = min(a.n, 2 * bs + 64)
        if nw > 0:
            w = make_view(nw, nw, a.dtype, device=a.device)
            w.storage.view(nw, nw).diagonal().fill_(1.0)
            cholesky_async(w, uplo, tree)
            torch.cuda.synchronize(a.device)
        self.graph = torch.cuda.CUDAGraph()
        stream = torch.cuda.Stream(a.device)
        stream.wait_stream(torch.cuda.current_stream(a.device))
        with torch.cuda.graph(self.graph, stream=stream):
            self.info = cholesky_async(a, uplo, tree)

    def run(self) -> torch.Tensor:
        """Replay on the current stream's device; returns the pivot flag tensor."""
        self.graph.replay()
        return self.info

    def __call__(self) -> None:
        """Replay and raise NotPositiveDefiniteError like cholesky()."""
        bad = int(self.run().item())
        if bad >= 0:
            raise NotPositiveDefiniteError(bad)
