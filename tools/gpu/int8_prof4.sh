mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import torch, sys
sys.path.insert(0, ".")
import paper_2602_02500_b200 as U
x = torch.randn(16, 2048, 512, device="cuda")
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
for i in range(2):
    U.orthogonalize(x, spec, precision="fp32")
torch.cuda.synchronize()
PY
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k oz_gemm_kernel -s 29 -c 1 -o gpurun_out/int8_cfg2_out -f python /tmp/one.py > gpurun_out/int8_ncu_full4.log 2>&1
