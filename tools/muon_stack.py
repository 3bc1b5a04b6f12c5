"""BASELINE configs[2] measured directly: one Muon optimizer step (paper_2602_02500_b200.Muon) over
a synthetic 32-layer transformer stack -- per layer q, k, v, o (4096 x 4096), up, gate (14336 x 4096)
and down (4096 x 14336) -- bf16 parameters, gradients i.i.d. N(0, 0.02^2) (seeded).  The optimizer
groups equal shapes into one batched orthogonalize call per group (three calls per step).

Under torchrun (WORLD_SIZE > 1, one rank per GPU, NCCL) every rank holds the same gradients (as after
a data-parallel all-reduce) and Muon(distribute=True) splits each shape group into equal shares, one
per rank, then all-gathers the orthogonalized updates; the step time is the max over ranks.

usage: python tools/muon_stack.py [layers] [steps]                       (prints one JSON line)
       python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/muon_stack.py
"""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2602_02500_b200 as U  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 32
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
distributed = "WORLD_SIZE" in os.environ
if distributed:
    dist.init_process_group("nccl", device_id=dev)
g = torch.Generator(device=dev).manual_seed(7)   # same seed on every rank: replicated gradients
shapes = [(4096, 4096)] * 4 + [(14336, 4096)] * 2 + [(4096, 14336)]
params = []
for _ in range(layers):
    for s in shapes:
        p = torch.nn.Parameter(torch.zeros(s, dtype=torch.bfloat16, device=dev))
        p.grad = (torch.randn(s, generator=g, device=dev) * 0.02).to(torch.bfloat16)
        params.append(p)
opt = U.Muon(params, lr=0.02, momentum=0.95, distribute=distributed)
spec = opt.spec
flops = sum(U.kernel_model_flops(min(p.shape), max(p.shape), spec) for p in params)
opt.step()  # warm-up: allocates momentum buffers and workspaces
torch.cuda.synchronize()
if distributed:
    dist.barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    opt.step()
e1.record()
torch.cuda.synchronize()
ms_t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
if distributed:
    dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
ms = float(ms_t.item())
peak_path = os.path.join(REPO, "MEASURED_PEAKS.json")
peak = json.load(open(peak_path))["bf16_tflops"] if os.path.exists(peak_path) else 1639.3
groups = None
if not distributed:
    from paper_2602_02500_b200._native import PROFILE_STAGES, StageProfiler  # noqa: E402
    with StageProfiler(8) as prof:  # per orthogonalize call (one per shape group) of one more step
        opt.step()
        torch.cuda.synchronize()
        st = prof.read()
    groups = [{k: round(float(v), 2) for k, v in zip(PROFILE_STAGES, row)} for row in st]
tf = flops / (ms / 1e3) / 1e12
if rank == 0:
    print(json.dumps({"config": f"configs[2]: Muon step over {layers} layers ({len(params)} matrices)",
                      "n_gpus": world, "parallelism": f"data-parallel orthogonalization shares x{world}",
                      "ms_per_step": ms, "matrices_per_s": len(params) / (ms / 1e3), "model_tflops": tf,
                      "pct_bf16_peak_per_gpu": tf / peak / world, "model_flops_per_step": flops,
                      "orthogonalize_ms_per_group": groups,
                      "max_memory_gb": torch.cuda.max_memory_allocated() / 2 ** 30}), flush=True)
if distributed:
    dist.destroy_process_group()
