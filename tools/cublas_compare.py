"""Dev tool: cuBLAS (torch.matmul, bf16 in / fp32 accumulate / bf16 out) on the headline's two long-side
shapes next to this library's kernels: the apply Y = X R (262144 x 2048 @ 2048 x 2048) and the Gram
X^T X (full product; our SYRK executes the upper half).  CUDA-event timed, inputs resident."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

w, h = 262144, 2048
x = torch.randn(w, h, device="cuda").to(torch.bfloat16)
r = (torch.randn(h, h, device="cuda") * 0.02).to(torch.bfloat16)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


y = torch.empty(w, h, device="cuda", dtype=torch.bfloat16)
g = torch.empty(h, h, device="cuda", dtype=torch.bfloat16)
t_apply = timeit(lambda: torch.matmul(x, r, out=y))
t_gram = timeit(lambda: torch.matmul(x.T, x, out=g))
f = 2.0 * w * h * h
print(f"cuBLAS apply X @ R: {t_apply:.3f} ms = {f / t_apply / 1e9:.0f} TFLOP/s")
print(f"cuBLAS Gram X^T X (full product): {t_gram:.3f} ms = {f / t_gram / 1e9:.0f} TFLOP/s "
      f"(a SYRK executing half would take {t_gram / 2:.3f} ms at that rate)")
