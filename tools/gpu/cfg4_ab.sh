mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -x -q > gpurun_out/ab_tests.log 2>&1; tail -1 gpurun_out/ab_tests.log
for i in 1 2; do
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-projection > gpurun_out/ab_cfg4_$i.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ab_cfg4_$i.json').read().splitlines()[-1]);print(d['ms_per_step'],{k:round(v,4) for k,v in d['stages_ms'].items()},d['clocks']['sm_mhz'])"
done
timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ab_cfg5.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ab_cfg5.json').read().splitlines()[-1]);print('cfg5',d['ms_per_step'],{k:round(v,3) for k,v in d['stages_ms'].items()},d['clocks']['sm_mhz'])"
