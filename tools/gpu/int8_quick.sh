mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import torch, sys
sys.path.insert(0, ".")
import paper_2602_02500_b200 as U
x = torch.randn(16, 2048, 512, device="cuda") if sys.argv[1] == "cfg2" else torch.randn(2, 8192, 4096, device="cuda")
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
for i in range(2):
    try:
        U.orthogonalize(x, spec, precision="fp32")
    except Exception as e:
        print("ignored", type(e).__name__)
torch.cuda.synchronize()
PY
timeout 600 python -m pytest tests/test_gpu_fp32_int8.py -x -q > gpurun_out/int8_tests.log 2>&1; tail -2 gpurun_out/int8_tests.log
for cfg in cfg2 big; do
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv python /tmp/one.py $cfg > gpurun_out/launch_${cfg}.csv 2>/dev/null
done
timeout 300 python bench.py --workload cfg2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg2_int8.json 2> gpurun_out/bench_cfg2_int8.err; tail -2 gpurun_out/bench_cfg2_int8.err
python -c "import json;d=json.loads(open('gpurun_out/bench_cfg2_int8.json').read().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms'])"
