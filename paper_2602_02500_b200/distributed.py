"""Multi-GPU partitioning of the orthogonalization (one process per GPU).

Two schemes (BASELINE.json north_star):

* Row sharding of one very tall matrix (configs[3]): rank r owns rows
  [r*w/P, (r+1)*w/P) of the w x h input.  Each rank computes its local Gram
  X_r^T X_r (``unso_gram``), ONE all-reduce (sum) of the h x h Gram over the
  process group (NCCL over NVLink on B200), then forms the scale and P(A)
  redundantly and applies it to its own rows (``unso_orthogonalize_from_gram``).
  The output stays row-sharded.  This is exact: sum_r X_r^T X_r = X^T X.

  ``collective="nvlink"`` replaces the all-reduce by the peer-memory reduction
  of ``unso_gram_push`` / ``_reduce`` / ``_wait``: the Gram
  kernel stores each partial tile straight into its owner rank's buffer over
  NVLink, owners sum their tiles in a fixed order and write the result into
  every rank's Gram buffer (torch symmetric memory provides the peer mappings).

* Batch distribution of independent matrices (configs[1,2,4]): longest-
  processing-time assignment by reference-model FLOPs, no communication.

The stage functions are injectable so the protocol can be exercised on CPU
(gloo) in tests; the product default is the CUDA library.
"""

from __future__ import annotations

import ctypes
import heapq
from dataclasses import dataclass
from typing import Callable, Sequence

import torch
import torch.distributed as dist

from . import _native as N
from .errors import DegenerateInputError, ShapeError
from .ortho import (MethodKind, MethodSpec, _DTYPES, _SCALING, _matrix_desc, _method_desc, _resolve_precision,
                    _row_major, kernel_model_flops, workspace_pool)


def row_shard_bounds(w: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced split of w rows over `world` ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(w, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def lpt_assignment(costs: Sequence[float], world: int) -> list[list[int]]:
    """Longest-processing-time-first: items sorted by cost, each to the least-loaded rank.
    Deterministic (ties broken by rank, then item index)."""
    heap = [(0.0, r) for r in range(world)]
    out: list[list[int]] = [[] for _ in range(world)]
    for i in sorted(range(len(costs)), key=lambda j: (-costs[j], j)):
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(v) for v in out]


# --------------------------------------------------------------------------- native stages

def native_gram(x_local: torch.Tensor, spec: MethodSpec, precision) -> torch.Tensor:
    """Un-normalised short-side Gram of a row shard (rows = long side)."""
    x_local = _row_major(x_local)
    xd = _matrix_desc(x_local)
    xd.orientation = 1
    prec = _resolve_precision(spec, x_local, precision)
    md, co = _method_desc(spec, prec, _SCALING[spec.effective_scaling])
    lib = N.lib()
    h = x_local.shape[-1]
    gdtype = torch.float64 if lib.unso_gram_dtype(ctypes.byref(md)) == N.DTYPE_F64 else torch.float32
    shape = (h, h) if x_local.dim() == 2 else (x_local.shape[0], h, h)
    g = torch.empty(shape, dtype=gdtype, device=x_local.device)
    nbytes = lib.unso_workspace_size(ctypes.byref(xd), ctypes.byref(md))
    stream = torch.cuda.current_stream(x_local.device)
    ws = workspace_pool.get(nbytes, x_local.device, stream)
    code = lib.unso_gram(ctypes.byref(xd), ctypes.c_void_p(x_local.data_ptr()), ctypes.c_void_p(g.data_ptr()),
                         ctypes.byref(md), ctypes.c_void_p(ws.data_ptr()), ctypes.c_size_t(ws.numel()),
                         ctypes.c_void_p(stream.cuda_stream))
    del co
    N.check(code, "unso_gram")
    return g


def native_finish(x_local: torch.Tensor, g: torch.Tensor, spec: MethodSpec, precision,
                  out: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """Scale, squaring chain and apply on the local rows, given the reduced Gram."""
    x_local = _row_major(x_local)
    xd = _matrix_desc(x_local)
    xd.orientation = 1
    prec = _resolve_precision(spec, x_local, precision)
    md, co = _method_desc(spec, prec, _SCALING[spec.effective_scaling])
    lib = N.lib()
    nbytes = lib.unso_workspace_size(ctypes.byref(xd), ctypes.byref(md))
    stream = torch.cuda.current_stream(x_local.device)
    ws = workspace_pool.get(nbytes, x_local.device, stream)
    y = out if out is not None else torch.empty_like(x_local, memory_format=torch.contiguous_format)
    status = torch.zeros(xd.batch, dtype=torch.int32, device=x_local.device)
    code = lib.unso_orthogonalize_from_gram(ctypes.byref(xd), ctypes.c_void_p(x_local.data_ptr()),
                                            ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                            ctypes.byref(md), ctypes.c_void_p(ws.data_ptr()),
                                            ctypes.c_size_t(ws.numel()), ctypes.c_void_p(status.data_ptr()),
                                            ctypes.c_void_p(stream.cuda_stream))
    del co
    N.check(code, "unso_orthogonalize_from_gram")
    return y, status


# --------------------------------------------------------------------------- NVLink Gram reduction

def gram_push_splits(h: int, w_local: int) -> int:
    """Split-K slices of the pushed Gram: enough CTA-pair work items for the 74 pairs, <= 4, and at
    least 64 local rows per slice.  A pure function of (h, w_local); every rank must use the same
    value, so callers pass the smallest shard's row count."""
    nt = (h + 255) // 256
    tiles = nt * (nt + 1) // 2
    return max(1, min(4, 74 // max(tiles, 1), max(w_local // 64, 1)))


class NvlinkGramReducer:
    """One rank's view of the peer-memory Gram reduction (unso_gram_push / _reduce / _wait).

    ``buffers`` lists, for every rank, the (slots, g, flags) device addresses as seen from THIS
    process; ``g`` is this rank's reduced h x h fp32 Gram as a tensor.  Build with
    :meth:`symmetric` (torch symmetric memory over the process group) or :meth:`emulated` (all
    ranks' buffers on one GPU, for tests).  Calls must follow push -> reduce -> wait on every rank."""

    def __init__(self, h: int, rank: int, world: int, splits: int, buffers, g: torch.Tensor, keep=()):
        if not 1 <= world <= N.MAX_PEERS:
            raise ValueError(f"world size {world} outside 1..{N.MAX_PEERS}")
        self.h, self.rank, self.world, self.splits, self.g = h, rank, world, splits, g
        self.peers = N.GramPeers()
        for r, (sl, gg, fl) in enumerate(buffers):
            self.peers.slots[r], self.peers.g[r], self.peers.flags[r] = sl, gg, fl
        self.epoch = 0
        self._keep = keep  # owns the underlying allocations
        self._done = torch.zeros(4, dtype=torch.int32, device=g.device)

    @staticmethod
    def _sizes(h: int, world: int, splits: int):
        lib = N.lib()
        return tuple(int(lib.unso_gram_peer_bytes(h, world, splits, i)) for i in range(3))

    @classmethod
    def emulated(cls, h: int, world: int, splits: int, device) -> list["NvlinkGramReducer"]:
        """All ranks on one device (ordinary allocations standing in for peer mappings)."""
        s_b, g_b, f_b = cls._sizes(h, world, splits)
        slots = [torch.empty(s_b // 4, dtype=torch.float32, device=device) for _ in range(world)]
        gs = [torch.empty(h, h, dtype=torch.float32, device=device) for _ in range(world)]
        flags = [torch.zeros(f_b // 4, dtype=torch.int32, device=device) for _ in range(world)]
        buffers = [(slots[r].data_ptr(), gs[r].data_ptr(), flags[r].data_ptr()) for r in range(world)]
        keep = (slots, gs, flags)
        return [cls(h, r, world, splits, buffers, gs[r], keep) for r in range(world)]

    @classmethod
    def symmetric(cls, h: int, splits: int, group=None, device=None) -> "NvlinkGramReducer":
        """Peer buffers from torch symmetric memory over ``group`` (NVLink P2P mappings)."""
        import torch.distributed._symmetric_memory as symm
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        device = device or torch.device("cuda", torch.cuda.current_device())
        s_b, g_b, f_b = cls._sizes(h, world, splits)
        f_pad = 256
        total = f_pad + g_b + s_b
        buf = symm.empty(total, dtype=torch.uint8, device=device)
        buf[:f_pad].zero_()
        grp = group if group is not None else dist.group.WORLD
        hdl = symm.rendezvous(buf, grp.group_name if hasattr(grp, "group_name") else grp)
        ptrs = list(hdl.buffer_ptrs)
        buffers = [(p + f_pad + g_b, p + f_pad, p) for p in ptrs]
        g = buf[f_pad:f_pad + g_b].view(torch.float32).view(h, h)
        torch.cuda.synchronize(device)
        dist.barrier(group)  # every rank's flags are zero before anyone signals
        return cls(h, rank, world, splits, buffers, g, keep=(buf, hdl))

    def push(self, x_local: torch.Tensor, spec: MethodSpec, precision=None) -> None:
        x_local = _row_major(x_local)
        xd = _matrix_desc(x_local)
        xd.orientation = 1
        prec = _resolve_precision(spec, x_local, precision)
        md, co = _method_desc(spec, prec, _SCALING[spec.effective_scaling])
        lib = N.lib()
        stream = torch.cuda.current_stream(x_local.device)
        ws = workspace_pool.get(lib.unso_workspace_size(ctypes.byref(xd), ctypes.byref(md)), x_local.device, stream)
        self.epoch += 1
        N.check(lib.unso_gram_push(ctypes.byref(xd), ctypes.c_void_p(x_local.data_ptr()), ctypes.byref(md),
                                   ctypes.byref(self.peers), self.rank, self.world, self.splits, self.epoch,
                                   ctypes.c_void_p(ws.data_ptr()), ctypes.c_size_t(ws.numel()),
                                   ctypes.c_void_p(stream.cuda_stream)), "unso_gram_push")

    def reduce(self) -> None:
        stream = torch.cuda.current_stream(self.g.device)
        N.check(N.lib().unso_gram_reduce(self.h, ctypes.byref(self.peers), self.rank, self.world, self.splits,
                                         self.epoch, ctypes.c_void_p(self._done.data_ptr()),
                                         ctypes.c_size_t(self._done.numel() * 4),
                                         ctypes.c_void_p(stream.cuda_stream)), "unso_gram_reduce")

    def wait(self) -> torch.Tensor:
        stream = torch.cuda.current_stream(self.g.device)
        N.check(N.lib().unso_gram_wait(self.h, ctypes.byref(self.peers), self.rank, self.world, self.epoch,
                                       ctypes.c_void_p(stream.cuda_stream)), "unso_gram_wait")
        return self.g


_REDUCERS: dict = {}
_SPLITS: dict = {}


def _nvlink_reducer(h: int, w_local: int, group, device) -> NvlinkGramReducer:
    """The cached reducer for this (h, local rows).  The split count must be the same on every rank
    (it is derived from the smallest shard), which costs one MIN all-reduce + host read -- done once
    per (h, local rows, group, device), not per call: calls run in lockstep on every rank, so every
    rank meets a new shape in the same call and the collective stays matched."""
    skey = (h, w_local, id(group), device)
    splits = _SPLITS.get(skey)
    if splits is None:
        wmin = torch.tensor([w_local], dtype=torch.int64, device=device)
        dist.all_reduce(wmin, op=dist.ReduceOp.MIN, group=group)
        splits = _SPLITS[skey] = gram_push_splits(h, int(wmin.item()))
    key = (h, splits, id(group), device)
    if key not in _REDUCERS:
        _REDUCERS[key] = NvlinkGramReducer.symmetric(h, splits, group, device)
    return _REDUCERS[key]


@dataclass
class ShardStages:
    gram: Callable
    finish: Callable


NATIVE_STAGES = ShardStages(native_gram, native_finish)


def orthogonalize_row_sharded(x_local: torch.Tensor, spec: MethodSpec, *, group=None, precision=None,
                              out: torch.Tensor | None = None, check: bool = True,
                              stages: ShardStages = NATIVE_STAGES, collective: str = "nccl") -> torch.Tensor:
    """UNSO on a tall matrix whose rows are sharded over the process group.

    x_local holds this rank's contiguous block of rows (the long side); every
    rank must pass the same column count h.  Returns this rank's rows of Y."""
    if spec.kind is not MethodKind.UNSO:
        raise ShapeError("row sharding is implemented for the UNSO method (one Gram all-reduce)")
    if collective not in ("nccl", "nvlink"):
        raise ValueError("collective must be 'nccl' or 'nvlink'")
    if collective == "nvlink":
        if not (dist.is_available() and dist.is_initialized()):
            raise ValueError("collective='nvlink' needs an initialised process group")
        red = _nvlink_reducer(x_local.shape[-1], x_local.shape[-2], group, x_local.device)
        red.push(x_local, spec, precision)
        red.reduce()
        g = red.wait()
        y, status = stages.finish(x_local, g, spec, precision, out)
        if check and status is not None and bool((status != 0).any()):
            raise DegenerateInputError("input is identically zero or the scaling denominator is not positive finite")
        return y
    g = stages.gram(x_local, spec, precision)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(g, op=dist.ReduceOp.SUM, group=group)
    y, status = stages.finish(x_local, g, spec, precision, out)
    if check and status is not None and bool((status != 0).any()):
        raise DegenerateInputError("input is identically zero or the scaling denominator is not positive finite")
    return y


def orthogonalize_batch_distributed(mats: Sequence[torch.Tensor], spec: MethodSpec, *, rank: int, world: int,
                                    orthogonalize_fn=None, precision=None) -> dict[int, torch.Tensor]:
    """Process this rank's LPT share of independent matrices; no communication.
    Returns {global index: Y}.  Equal shapes are grouped into one batched call."""
    from .ortho import orthogonalize
    fn = orthogonalize_fn or (lambda m: orthogonalize(m, spec, precision=precision, check=False).y)
    costs = []
    for m in mats:
        r, c = m.shape[-2], m.shape[-1]
        h, w = (c, r) if r > c else (r, c)
        costs.append(float(kernel_model_flops(h, w, spec)))
    mine = lpt_assignment(costs, world)[rank]
    groups: dict = {}
    for i in mine:
        groups.setdefault((tuple(mats[i].shape), mats[i].dtype), []).append(i)
    out = {}
    for _, idx in sorted(groups.items(), key=lambda kv: str(kv[0])):
        stacked = torch.stack([mats[i] for i in idx]) if len(idx) > 1 else mats[idx[0]]
        y = fn(stacked)
        if len(idx) == 1:
            out[idx[0]] = y
        else:
            for j, i in enumerate(idx):
                out[i] = y[j]
    return out


__all__ = ["row_shard_bounds", "lpt_assignment", "orthogonalize_row_sharded", "orthogonalize_batch_distributed",
           "native_gram", "native_finish", "ShardStages", "NATIVE_STAGES", "NvlinkGramReducer", "gram_push_splits",
           "_DTYPES"]
