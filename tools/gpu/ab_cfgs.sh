mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_poisoned_workspace.py -x -q > gpurun_out/ab_tests.log 2>&1; tail -1 gpurun_out/ab_tests.log
for wl in "cfg1 --steps 200" "cfg2 --precision bf16 --steps 50" "cfg5 --steps 3 --warmup 2"; do
for i in 1 2; do for L in exp/base.so exp/new.so; do
UNSO_LIB=$L timeout 600 python bench.py --workload $wl --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().splitlines()[-1]);print('$wl $L',round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['stages_ms'].items()},d['clocks']['sm_mhz'])"
done; done; done
