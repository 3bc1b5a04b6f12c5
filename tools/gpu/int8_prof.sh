mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
import paper_2602_02500_b200 as U
import numpy as np
which = sys.argv[1]
if which == "cfg2":
    x = torch.randn(16, 2048, 512, device="cuda")
else:
    x = torch.randn(1, 16384, 8192, device="cuda")
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
for i in range(2):
    U.orthogonalize(x, spec, precision="fp32")
torch.cuda.synchronize()
PY
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv python /tmp/one.py cfg2 > gpurun_out/int8_launches_cfg2.csv 2> gpurun_out/int8_launches_cfg2.err
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:oz_gemm -s 20 -c 2 -o gpurun_out/int8_cfg2_gemm -f python /tmp/one.py cfg2 > gpurun_out/int8_ncu_full.log 2>&1
tail -2 gpurun_out/int8_ncu_full.log
