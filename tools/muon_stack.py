"""BASELINE configs[2] measured directly: one Muon optimizer step (paper_2602_02500_b200.Muon) over
a synthetic 32-layer transformer stack -- per layer q, k, v, o (4096 x 4096), up, gate (14336 x 4096)
and down (4096 x 14336) -- bf16 parameters, gradients i.i.d. N(0, 0.02^2) (seeded).  The optimizer
groups equal shapes into one batched orthogonalize call per group (three calls per step).

usage: python tools/muon_stack.py [layers] [steps]     (prints one JSON line)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_02500_b200 as U  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 32
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(7)
shapes = [(4096, 4096)] * 4 + [(14336, 4096)] * 2 + [(4096, 14336)]
params = []
for _ in range(layers):
    for s in shapes:
        p = torch.nn.Parameter(torch.zeros(s, dtype=torch.bfloat16, device=dev))
        p.grad = (torch.randn(s, generator=g, device=dev) * 0.02).to(torch.bfloat16)
        params.append(p)
opt = U.Muon(params, lr=0.02, momentum=0.95)
spec = opt.spec
flops = sum(U.kernel_model_flops(min(p.shape), max(p.shape), spec) for p in params)
opt.step()  # warm-up: allocates momentum buffers and workspaces
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    opt.step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["bf16_tflops"] if os.path.exists(
    os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 1639.3
from paper_2602_02500_b200._native import PROFILE_STAGES, StageProfiler  # noqa: E402
with StageProfiler(8) as prof:  # per orthogonalize call (one per shape group) of one more step
    opt.step()
    torch.cuda.synchronize()
    st = prof.read()
groups = [{k: round(float(v), 2) for k, v in zip(PROFILE_STAGES, row)} for row in st]
tf = flops / (ms / 1e3) / 1e12
print(json.dumps({"config": f"configs[2]: Muon step over {layers} layers ({len(params)} matrices)",
                  "ms_per_step": ms, "matrices_per_s": len(params) / (ms / 1e3), "model_tflops": tf,
                  "pct_bf16_peak": tf / peak, "model_flops_per_step": flops,
                  "orthogonalize_ms_per_group": groups,
                  "max_memory_gb": torch.cuda.max_memory_allocated() / 2 ** 30}), flush=True)
