mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import torch, sys
sys.path.insert(0, ".")
import paper_2602_02500_b200 as U
x = torch.randn(16, 2048, 512, device="cuda")
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
for i in range(2):
    try:
        U.orthogonalize(x, spec, precision="fp32")
    except Exception as e:
        print("ignored", type(e).__name__)
torch.cuda.synchronize()
PY
for d in 0 1 2 3; do
UNSO_LIB=exp/dev.so UNSO_OZ_DEBUG=$d timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum -k oz_gemm_kernel --clock-control none --csv python /tmp/one.py > gpurun_out/dbg3_$d.csv 2>/dev/null
done
