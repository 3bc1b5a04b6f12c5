mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import torch, sys
sys.path.insert(0, ".")
import paper_2602_02500_b200 as U
x = torch.randn(1, 16384, 8192, device="cuda")
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
U.orthogonalize(x, spec, precision="fp32")
torch.cuda.synchronize()
PY
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv python /tmp/one.py > gpurun_out/int8_cfg5_launches.csv 2>/dev/null
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k oz_gemm_kernel -s 3 -c 1 -o gpurun_out/int8_cfg5_chain -f python /tmp/one.py > gpurun_out/int8_ncu5.log 2>&1; tail -1 gpurun_out/int8_ncu5.log
