"""CUDA-graph capture of a fixed-shape orthogonalization (launch-bound small problems).

configs[0] (512 x 128) and configs[1] (16 x 2048 x 512) are dominated by host-side launch
overhead (ctypes call, tensor-map encoding, ~6-20 kernel launches).  `GraphedOrthogonalize`
records one `orthogonalize` call into a CUDA graph (stream capture of the library's launches:
TMA descriptors and workspace pointers are baked into the kernel nodes) and replays it for new
inputs copied into the captured input buffer -- one graph launch per call.
"""

from __future__ import annotations

import torch

from .ortho import MethodSpec, orthogonalize


class GraphedOrthogonalize:
    """Replayable orthogonalize(x, spec) for one shape/dtype/device.

    Usage:
        g = GraphedOrthogonalize(example, spec, precision="bf16")
        y = g(x)            # copies x into the captured buffer, replays, returns the output buffer
    The returned tensor is reused by the next call (clone it to keep a result).  Device-side
    status checks are skipped (check=False semantics); validate inputs beforehand if needed.
    """

    def __init__(self, example: torch.Tensor, spec: MethodSpec, precision=None, warmup: int = 2):
        if not example.is_cuda:
            raise ValueError("example must be a CUDA tensor")
        self.spec = spec
        self.precision = precision
        self.x = example.detach().clone(memory_format=torch.contiguous_format)
        side = torch.cuda.Stream(device=self.x.device)
        side.wait_stream(torch.cuda.current_stream(self.x.device))
        with torch.cuda.stream(side):
            for _ in range(max(warmup, 1)):  # first calls configure kernels / size the workspace
                orthogonalize(self.x, spec, precision=precision, check=False)
        torch.cuda.current_stream(self.x.device).wait_stream(side)
        torch.cuda.synchronize(self.x.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.y = orthogonalize(self.x, spec, precision=precision, check=False).y

    def __call__(self, x: torch.Tensor | None = None) -> torch.Tensor:
        if x is not None:
            if x.shape != self.x.shape or x.dtype != self.x.dtype:
                raise ValueError("input must match the captured shape and dtype")
            self.x.copy_(x)
        self.graph.replay()
        return self.y


__all__ = ["GraphedOrthogonalize"]
