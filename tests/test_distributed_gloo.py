"""Multi-process (gloo, world size 2, CPU) tests of the multi-GPU host protocol in
paper_2602_02500_b200/distributed.py.  The CUDA stages are replaced by oracle-based
stand-ins (test-only injection); the product default is the native library."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_02500_b200 import MethodKind, MethodSpec, default_coefficients
from paper_2602_02500_b200.distributed import (ShardStages, lpt_assignment, orthogonalize_batch_distributed,
                                               orthogonalize_row_sharded, row_shard_bounds)
from oracle import unso_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_gram(x_local, spec, precision):
    x = x_local.double().numpy()
    return torch.from_numpy(x.T @ x)           # local X_r^T X_r (rows = long side)


def _oracle_finish(x_local, g, spec, precision, out):
    G = g.numpy()
    denom = float(np.sqrt(float(np.sqrt(np.sum(G * G)))))
    a, order = O.DEFAULT_A, O.DEFAULT_ORDER
    b = O.final_coefficient(order, a, "exact")
    bk = np.eye(G.shape[0]) - G / denom ** 2
    p = np.eye(G.shape[0])
    for k in range(1, order):
        p = p + a[k - 1] * bk
        bk = bk @ bk
    p = p + b * bk
    return torch.from_numpy((x_local.double().numpy() / denom) @ p), torch.zeros(1, dtype=torch.int32)


def _worker_row_shard(rank, world, port, m, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r0, r1 = row_shard_bounds(m.shape[0], world, rank)
    spec = MethodSpec(MethodKind.UNSO, coeffs=default_coefficients())
    y = orthogonalize_row_sharded(torch.from_numpy(m[r0:r1]), spec, stages=ShardStages(_oracle_gram, _oracle_finish))
    q.put((rank, r0, r1, y.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _worker_batch(rank, world, port, mats, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = MethodSpec(MethodKind.UNSO, coeffs=default_coefficients())
    def fn(t):
        if t.dim() == 2:
            return torch.from_numpy(O.run(t.numpy(), "unso")["y"])
        return torch.from_numpy(np.stack([O.run(a.numpy(), "unso")["y"] for a in t]))

    out = orthogonalize_batch_distributed([torch.from_numpy(x) for x in mats], spec, rank=rank, world=world,
                                          orthogonalize_fn=fn)
    gathered = [None] * world
    dist.all_gather_object(gathered, {k: v.numpy() for k, v in out.items()})
    if rank == 0:
        q.put(gathered)
    dist.destroy_process_group()


def _muon_params(seed):
    g = torch.Generator().manual_seed(seed)
    shapes = [(24, 16)] * 5 + [(16, 40)] * 2 + [(9,)]
    params = [torch.nn.Parameter(torch.randn(*sh, generator=g, dtype=torch.float64)) for sh in shapes]
    grads = [torch.randn(*sh, generator=g, dtype=torch.float64) for sh in shapes]
    return params, grads


def _oracle_stacked(calls):
    def fn(t):
        calls.append(int(t.shape[0]))
        return torch.from_numpy(np.stack([O.run(a.numpy(), "unso")["y"] for a in t]))
    return fn


def _worker_muon(rank, world, port, q):
    from paper_2602_02500_b200.muon import Muon
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    params, grads = _muon_params(3)
    calls = []
    opt = Muon(params, lr=0.05, momentum=0.9, weight_decay=0.01, orthogonalize_fn=_oracle_stacked(calls),
               distribute=True)
    for step in range(2):                      # two steps: the momentum buffer carries over
        for p, g in zip(params, grads):
            p.grad = g * (step + 1)
        opt.step()
    q.put((rank, calls, [p.detach().numpy() for p in params]))
    dist.barrier()
    dist.destroy_process_group()


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = []
    n_expected = world if target in (_worker_row_shard, _worker_muon) else 1
    for _ in range(n_expected):
        results.append(q.get(timeout=120))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return results


def test_row_shard_bounds_cover_exactly():
    for w in (1, 7, 262144, 1000003):
        for world in (1, 2, 3, 8):
            spans = [row_shard_bounds(w, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == w
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_lpt_assignment_balanced_and_deterministic():
    costs = [5, 3, 3, 2, 2, 2, 1, 1, 9, 4]
    parts = lpt_assignment(costs, 3)
    assert sorted(i for p in parts for i in p) == list(range(len(costs)))
    loads = [sum(costs[i] for i in p) for p in parts]
    assert max(loads) - min(loads) <= max(costs)
    assert parts == lpt_assignment(costs, 3)
    # configs[2]: 32 layers x {4 x 4096^2, 3 x 14336x4096}, 8 ranks -> equal FLOP split
    from paper_2602_02500_b200 import kernel_model_flops
    spec = MethodSpec(MethodKind.UNSO, coeffs=default_coefficients())
    cfg3 = [kernel_model_flops(4096, 4096, spec)] * 128 + [kernel_model_flops(4096, 14336, spec)] * 96
    parts = lpt_assignment(cfg3, 8)
    loads = [sum(cfg3[i] for i in p) for p in parts]
    assert max(loads) / min(loads) < 1.01


def test_row_sharded_unso_matches_unsharded_oracle_gloo():
    m = O.gaussian_matrix(301, 24, 5)                  # ragged split: 151 + 150 rows
    results = _spawn(_worker_row_shard, 2, m)
    y = np.zeros_like(m)
    for rank, r0, r1, ys in results:
        y[r0:r1] = ys
    ref = O.run(m, "unso")["y"]
    assert np.max(np.abs(y - ref)) < 1e-10


def test_batch_distribution_gloo():
    mats = [O.gaussian_matrix(40, 12, s) for s in range(5)] + [O.gaussian_matrix(16, 48, 9)]
    gathered = _spawn(_worker_batch, 2, mats)[0]
    merged = {}
    for part in gathered:
        assert not (set(part) & set(merged))          # disjoint shares
        merged.update(part)
    assert sorted(merged) == list(range(len(mats)))
    for i, m in enumerate(mats):
        assert np.max(np.abs(merged[i] - O.run(m, "unso")["y"])) < 1e-12


def test_sharded_requires_unso():
    with pytest.raises(ValueError):
        orthogonalize_row_sharded(torch.zeros(4, 2), MethodSpec(MethodKind.MUON_NS))


def test_muon_data_parallel_split_gloo():
    """Muon(distribute=True) on 2 ranks: each rank orthogonalizes half of every shape group (5 -> 3 + 2,
    2 -> 1 + 1) and after the all-gather both ranks hold exactly the single-process result."""
    from paper_2602_02500_b200.muon import Muon
    results = _spawn(_worker_muon, 2)
    params, grads = _muon_params(3)
    calls = []
    opt = Muon(params, lr=0.05, momentum=0.9, weight_decay=0.01, orthogonalize_fn=_oracle_stacked(calls))
    for step in range(2):
        for p, g in zip(params, grads):
            p.grad = g * (step + 1)
        opt.step()
    assert sorted(calls) == [2, 2, 5, 5]
    by_rank = {r: (c, ps) for r, c, ps in results}
    assert sorted(by_rank[0][0]) == [1, 1, 3, 3] and sorted(by_rank[1][0]) == [1, 1, 2, 2]
    for r in (0, 1):
        for got, want in zip(by_rank[r][1], params):
            assert np.array_equal(got, want.detach().numpy())
