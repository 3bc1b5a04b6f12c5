mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import torch, sys
sys.path.insert(0, ".")
import paper_2602_02500_b200 as U
x = (torch.randn(4, 16384, 8192, device="cuda") * 0.02).to(torch.bfloat16)
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
U.orthogonalize(x, spec)
torch.cuda.synchronize()
PY
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none -k chain_pair_f8_kernel -s 6 -c 1 -o gpurun_out/cfg5_chain_f8 -f python /tmp/one.py > gpurun_out/cfg5_ncu.log 2>&1; tail -1 gpurun_out/cfg5_ncu.log
