"""CUDA-graph capture of hot-path calls (iterative DMRG/CTMRG-style reuse).

The engine's host layer does per-call bookkeeping in Python (label checks, plan
lookup); for loops that repeat the same contraction on the same buffers (the
Lanczos matvec L.A.W.R, a CTMRG move) the whole launch sequence can be captured
once and replayed with a single graph launch. Inputs are the bound tensors'
buffers (update them in place, e.g. ``t.get_block_().storage().copy_(x)``);
the output object returned by ``replay`` is the one produced at capture time
(its buffer is rewritten by every replay).
"""
import torch


class CapturedCall:
    def __init__(self, fn, warmup=2):
        self._fn = fn
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(warmup):  # builds plans / sets kernel attributes outside capture
                fn()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self._graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self._graph):
            self._out = fn()

    def replay(self):
        self._graph.replay()
        return self._out

    @property
    def output(self):
        return self._out


def capture(fn, warmup=2):
    """Capture ``fn()`` (a sequence of engine calls on fixed buffers) into a CUDA graph."""
    return CapturedCall(fn, warmup)
