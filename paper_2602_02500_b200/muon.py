"""Muon-style optimizer step around the batched orthogonalizer (BASELINE configs[2],
SURVEY §8f item 2).

For every 2-D parameter: momentum buffer M <- mu M + G (Nesterov: update = G + mu M), the update
is orthogonalized, rescaled by sqrt(max(1, rows/cols)) and applied with learning rate lr and
decoupled weight decay.  Parameters of equal shape and dtype are stacked and orthogonalized in ONE
grouped call (one launch per kernel stage for the whole group), which is what makes a 32-layer
transformer step (224 matrices of 4096 x {4096, 14336}) tensor-core bound instead of launch bound.

The orthogonalizer is any MethodSpec of this package: the learned UNSO polynomial (default) or the
NS/Muon quintic iteration.  Non-2-D parameters are updated with plain momentum SGD.

Data-parallel use (BASELINE configs[2] "grouped batch distributed across 1/2/4/8 GPUs"): with
``process_group`` set (or the default group initialised and ``distribute=True``), every rank holds
the same (all-reduced) gradients, each shape group is split into contiguous, equal shares of its
matrices, every rank orthogonalizes only its share, and the results are all-gathered before the
identical update on every rank.  Equal shapes cost the same, so equal shares are the LPT optimum
within a group; no communication besides the one all-gather per group.
"""

from __future__ import annotations

import math
from collections import defaultdict
from typing import Callable, Iterable

import torch
import torch.distributed as dist

from .ortho import MethodKind, MethodSpec, orthogonalize
from .scalarpoly import default_coefficients


def default_spec(kind: str = "unso") -> MethodSpec:
    if kind == "unso":
        return MethodSpec(MethodKind.UNSO, coeffs=default_coefficients())
    if kind == "muon":
        return MethodSpec(MethodKind.MUON_NS, iterations=5)
    raise ValueError(f"unknown orthogonalizer {kind!r}")


class Muon(torch.optim.Optimizer):
    """Momentum + orthogonalized update, grouped by shape.

    Args:
        params: iterable of parameters or parameter groups.
        lr: learning rate.
        momentum: momentum coefficient mu.
        nesterov: use the Nesterov form G + mu M.
        weight_decay: decoupled weight decay.
        spec: MethodSpec of the orthogonalizer (default: UNSO with the shipped coefficients).
        precision: "bf16" (tensor cores) or "fp32" (fp64-grade parity path).
        orthogonalize_fn: override (stacked 3-D tensor -> stacked result); for testing.
        process_group: process group over which the orthogonalizations are shared (data parallel).
        distribute: share the work over the default group when it is initialised (default False;
            implied by process_group).
    """

    def __init__(self, params: Iterable, lr: float = 0.02, momentum: float = 0.95, nesterov: bool = True,
                 weight_decay: float = 0.0, spec: MethodSpec | None = None, precision: str = "bf16",
                 orthogonalize_fn: Callable | None = None, process_group=None, distribute: bool = False):
        if lr <= 0.0:
            raise ValueError("lr must be positive")
        if not 0.0 <= momentum < 1.0:
            raise ValueError("momentum must be in [0, 1)")
        defaults = dict(lr=lr, momentum=momentum, nesterov=nesterov, weight_decay=weight_decay)
        super().__init__(params, defaults)
        self.spec = spec or default_spec()
        self.precision = precision
        self._ortho = orthogonalize_fn or (
            lambda u: orthogonalize(u, self.spec, precision=self.precision, check=False).y)
        self.process_group = process_group
        self.distribute = distribute or process_group is not None

    def _orthogonalize_group(self, stacked: torch.Tensor) -> torch.Tensor:
        """Orthogonalize a stacked group; under data parallelism each rank does an equal contiguous
        share and the shares are all-gathered (same result on every rank)."""
        if not self.distribute or not (dist.is_available() and dist.is_initialized()):
            return self._ortho(stacked)
        world, rank = dist.get_world_size(self.process_group), dist.get_rank(self.process_group)
        n = stacked.shape[0]
        per = -(-n // world)
        lo, hi = min(n, rank * per), min(n, (rank + 1) * per)
        mine = torch.zeros((per,) + tuple(stacked.shape[1:]), dtype=stacked.dtype, device=stacked.device)
        if hi > lo:
            mine[: hi - lo] = self._ortho(stacked[lo:hi])
        if dist.get_backend(self.process_group) == "nccl":
            full = torch.empty((world * per,) + tuple(stacked.shape[1:]), dtype=stacked.dtype, device=stacked.device)
            dist.all_gather_into_tensor(full, mine, group=self.process_group)
        else:
            parts = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(parts, mine, group=self.process_group)
            full = torch.cat(parts)
        return full[:n]

    @torch.no_grad()
    def step(self, closure=None):
        loss = None
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        for group in self.param_groups:
            lr, mu, nesterov, wd = group["lr"], group["momentum"], group["nesterov"], group["weight_decay"]
            buckets: dict = defaultdict(list)
            for p in group["params"]:
                if p.grad is None:
                    continue
                g = p.grad
                state = self.state[p]
                buf = state.get("momentum_buffer")
                if buf is None:
                    buf = state["momentum_buffer"] = torch.zeros_like(g)
                if p.dim() == 2:  # momentum in the group pass (fused on CUDA)
                    buckets[(tuple(p.shape), g.dtype, g.device)].append(p)
                else:
                    torch.add(g, buf, alpha=mu, out=buf)  # M <- mu M + G
                    if wd:
                        p.mul_(1.0 - lr * wd)
                    p.add_(g.add(buf, alpha=mu) if nesterov else buf, alpha=-lr)
            for (shape, dtype, device), items in buckets.items():
                rows, cols = shape
                scale = math.sqrt(max(1.0, rows / cols))
                if _fused_ok(items, self.state):
                    self._fused_group(items, rows, cols, mu, nesterov, 1.0 - lr * wd, -lr * scale)
                    continue
                # the update of every matrix of the group is written straight into the stacked batch
                stacked = torch.empty((len(items), rows, cols), dtype=dtype, device=device)
                for i, p in enumerate(items):
                    buf = self.state[p]["momentum_buffer"]
                    torch.add(p.grad, buf, alpha=mu, out=buf)  # M <- mu M + G
                    if nesterov:
                        torch.add(p.grad, buf, alpha=mu, out=stacked[i])
                    else:
                        stacked[i].copy_(buf)
                zero = torch.linalg.vector_norm(stacked.flatten(1), ord=float("inf"), dim=1) == 0
                ortho = self._orthogonalize_group(stacked)
                if bool(zero.any()):  # zero update -> zero step (not a degenerate input)
                    ortho = torch.where(zero[:, None, None], torch.zeros_like(ortho), ortho)
                if wd:
                    torch._foreach_mul_(items, 1.0 - lr * wd)
                torch._foreach_add_(items, [o.to(items[0].dtype) for o in ortho.unbind(0)], alpha=-lr * scale)
        return loss

    def _fused_group(self, items, rows, cols, mu, nesterov, decay, alpha):
        """CUDA bf16/fp32 groups: momentum, Nesterov stacking and the zero check in one multi-tensor
        kernel, the decayed update in another (csrc/muon_update.cuh), no host synchronisation."""
        from . import _native as N
        p0 = items[0]
        dev, n, numel = p0.device, len(items), rows * cols
        dt = N.DTYPE_BF16 if p0.dtype == torch.bfloat16 else N.DTYPE_F32
        # Parameter and momentum-buffer addresses are stable across steps: their device pointer
        # lists are cached.  Gradients are usually reallocated every step (zero_grad(set_to_none=True)),
        # so their list goes through a reused pinned staging buffer and a non-blocking copy.
        key = tuple((self.state[p]["momentum_buffer"].data_ptr(), p.data_ptr()) for p in items)
        cache = self.__dict__.setdefault("_ptr_lists", {})
        ent = cache.get(key)
        if ent is None:
            stable = torch.tensor(list(zip(*key)), dtype=torch.int64).to(dev)
            ent = (stable, torch.empty(n, dtype=torch.int64, pin_memory=True),
                   torch.empty(n, dtype=torch.int64, device=dev), torch.cuda.Event())
            if len(cache) > 64:
                cache.clear()
            cache[key] = ent
        stable, g_host, g_dev, g_ready = ent
        g_ready.synchronize()  # the previous step's copy out of the staging buffer has finished
        g_host.numpy()[:] = [p.grad.data_ptr() for p in items]
        g_dev.copy_(g_host, non_blocking=True)
        g_ready.record(torch.cuda.current_stream(dev))
        stacked = torch.empty((n, rows, cols), dtype=p0.dtype, device=dev)
        maxabs = torch.empty(n, dtype=torch.float32, device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        lib = N.lib()
        N.check(lib.unso_muon_prepare(n, g_dev.data_ptr(), stable[0].data_ptr(), stacked.data_ptr(), numel, dt,
                                      float(mu), 1 if nesterov else 0, maxabs.data_ptr(), stream), "unso_muon_prepare")
        ortho = self._orthogonalize_group(stacked).contiguous()
        N.check(lib.unso_muon_update(n, stable[1].data_ptr(), ortho.data_ptr(), numel, dt, maxabs.data_ptr(),
                                     float(decay), float(alpha), stream), "unso_muon_update")


#: use the fused CUDA passes where _fused_ok allows (tests switch it off to compare with the torch ops)
FUSED_PASSES = True


def _fused_ok(items, state) -> bool:
    """Every tensor of the group on one CUDA device, contiguous, bf16 or fp32, 16-byte aligned."""
    p0 = items[0]
    if (not FUSED_PASSES or not p0.is_cuda or p0.dtype not in (torch.bfloat16, torch.float32) or p0.numel() % 8
            or len(items) > 65535):
        return False
    for p in items:
        for t in (p, p.grad, state[p]["momentum_buffer"]):
            if t.dtype != p0.dtype or t.device != p0.device or not t.is_contiguous() or t.data_ptr() % 16:
                return False
    return True


__all__ = ["Muon", "default_spec"]
