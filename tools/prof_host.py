import cProfile, pstats, sys, os, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2602_02500_b200 as U
x = torch.randn(512, 128, device="cuda").to(torch.bfloat16)
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
for _ in range(20): U.orthogonalize(x, spec, check=False)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(500): U.orthogonalize(x, spec, check=False)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host submit {1e6*(t1-t0)/500:.1f} us/call, total {1e6*(t2-t0)/500:.1f} us/call")
pr = cProfile.Profile(); pr.enable()
for _ in range(500): U.orthogonalize(x, spec, check=False)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
