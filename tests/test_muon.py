"""Muon-style optimizer around the batched orthogonalizer: grouping and update rule (CPU, with an
oracle stand-in for the device orthogonalizer) and one real device step (GPU)."""

import math

import numpy as np
import pytest
import torch

from paper_2602_02500_b200.muon import Muon
from oracle import unso_oracle as O


def oracle_ortho(calls):
    def fn(stacked):
        calls.append(tuple(stacked.shape))
        return torch.from_numpy(np.stack([O.run(m.double().numpy(), "unso")["y"] for m in stacked])).to(stacked.dtype)
    return fn


def test_grouping_and_update_rule_cpu():
    torch.manual_seed(0)
    shapes = [(24, 16), (24, 16), (16, 40), (24, 16), (7,)]
    params = [torch.nn.Parameter(torch.randn(*s, dtype=torch.float64)) for s in shapes]
    for p in params:
        p.grad = torch.randn_like(p)
    before = [p.detach().clone() for p in params]
    calls = []
    opt = Muon(params, lr=0.1, momentum=0.9, nesterov=True, weight_decay=0.01, orthogonalize_fn=oracle_ortho(calls))
    opt.step()
    assert sorted(calls) == sorted([(3, 24, 16), (1, 16, 40)])     # one grouped call per shape
    for p, p0 in zip(params, before):
        g = p.grad
        upd = g + 0.9 * g                                          # buffer = g after one step; Nesterov
        if p.dim() == 2:
            o = torch.from_numpy(O.run(upd.numpy(), "unso")["y"])
            exp = p0 * (1 - 0.1 * 0.01) - 0.1 * math.sqrt(max(1.0, p.shape[0] / p.shape[1])) * o
        else:
            exp = p0 * (1 - 0.1 * 0.01) - 0.1 * upd
        assert torch.allclose(p.detach(), exp, atol=1e-12)


def test_zero_gradient_gives_zero_step():
    p = torch.nn.Parameter(torch.randn(8, 4, dtype=torch.float64))
    p.grad = torch.zeros_like(p)
    p0 = p.detach().clone()
    Muon([p], lr=0.1, orthogonalize_fn=lambda s: torch.full_like(s, float("nan"))).step()
    assert torch.equal(p.detach(), p0)


@pytest.mark.gpu
def test_muon_step_on_device():
    torch.manual_seed(1)
    dev = torch.device("cuda:0")
    params = [torch.nn.Parameter(torch.randn(512, 256, device=dev) * 0.02) for _ in range(3)]
    params.append(torch.nn.Parameter(torch.randn(256, 1024, device=dev) * 0.02))
    for p in params:
        p.grad = torch.randn_like(p) * 0.02
    before = [p.detach().clone() for p in params]
    Muon(params, lr=0.05, momentum=0.0, nesterov=False, precision="bf16").step()
    for p, p0 in zip(params, before):
        step = (p0 - p.detach()).double().cpu().numpy() / 0.05 / math.sqrt(max(1.0, p.shape[0] / p.shape[1]))
        ref = O.run(p.grad.to(torch.bfloat16).double().cpu().numpy(), "unso")["y"]
        assert np.linalg.norm(step - ref) / np.linalg.norm(ref) <= 2e-2


@pytest.mark.gpu
def test_muon_distribute_over_nccl_group_world1():
    """The data-parallel path (equal shares + NCCL all_gather_into_tensor) on a real one-rank NCCL
    group gives the same parameters as the plain step."""
    import socket
    import torch.distributed as dist
    dev = torch.device("cuda:0")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{port}", device_id=dev)
    try:
        g = torch.Generator(device=dev).manual_seed(5)
        base = [torch.randn(512, 256, generator=g, device=dev) * 0.02 for _ in range(3)]
        grads = [torch.randn(512, 256, generator=g, device=dev) * 0.02 for _ in range(3)]
        results = []
        for distribute in (False, True):
            params = [torch.nn.Parameter(b.clone()) for b in base]
            for p, gr in zip(params, grads):
                p.grad = gr.clone()
            Muon(params, lr=0.05, precision="bf16", distribute=distribute).step()
            results.append([p.detach() for p in params])
        for a, b in zip(*results):
            assert torch.equal(a, b)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_fused_passes_match_torch_ops(dtype):
    """The fused multi-tensor momentum / Nesterov / zero-check and update kernels
    (csrc/muon_update.cuh) against the plain torch ops of the same step: two steps with weight
    decay, one all-zero gradient in the group (zero step), an odd-sized group, a 1-D parameter."""
    import paper_2602_02500_b200.muon as M
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(3)
    shapes = [(384, 256)] * 3 + [(256, 640)] + [(64,)]
    base = [torch.randn(s, generator=g, device=dev).to(dtype) * 0.02 for s in shapes]
    grads = [[torch.randn(s, generator=g, device=dev).to(dtype) * 0.02 for s in shapes] for _ in range(2)]
    grads[0][1].zero_()
    grads[1][1].zero_()
    out = []
    for fused in (True, False):
        M.FUSED_PASSES = fused
        try:
            params = [torch.nn.Parameter(b.clone()) for b in base]
            opt = M.Muon(params, lr=0.05, momentum=0.9, weight_decay=0.1, precision="bf16")
            for step in range(2):
                for p, gr in zip(params, grads[step]):
                    p.grad = gr.clone()
                opt.step()
            out.append([p.detach().double() for p in params] +
                       [opt.state[p]["momentum_buffer"].double() for p in params])
        finally:
            M.FUSED_PASSES = True
    for a, b in zip(*out):
        assert torch.isfinite(a).all()
        # bf16: the torch ops round twice (decay, then update), the fused kernel once: <= ~2 ulps apart
        tol = 1e-2 if dtype == torch.bfloat16 else 1e-5
        assert float(torch.linalg.norm(a - b)) <= tol * float(torch.linalg.norm(b)) + 1e-12
    # the zero-gradient matrix only decayed: p = base * (1 - lr wd)^2
    assert torch.allclose(out[0][1], base[1].double() * (1 - 0.05 * 0.1) ** 2, rtol=1e-2 if dtype == torch.bfloat16 else 1e-6)


def test_fused_passes_only_for_cuda_bf16_fp32_groups():
    """The fused optimizer kernels take CUDA bf16/fp32 groups only; CPU tensors (and other dtypes)
    run the torch ops, so this CPU step must not touch the native library."""
    import paper_2602_02500_b200.muon as M
    p = torch.nn.Parameter(torch.randn(16, 8))
    p.grad = torch.randn(16, 8)
    state = {p: {"momentum_buffer": torch.zeros(16, 8)}}
    assert not M._fused_ok([p], state)
    q = torch.nn.Parameter(torch.randn(16, 8, dtype=torch.float64))
    q.grad = torch.randn(16, 8, dtype=torch.float64)
    assert not M._fused_ok([q], {q: {"momentum_buffer": torch.zeros_like(q)}})
